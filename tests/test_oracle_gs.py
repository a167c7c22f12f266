"""Pins of the Gauss-Seidel AMG smoother of the oracle (NEXT-f2; "one sweep of hybrid forward l1-Gauss-
Seidel for the down cycle and one sweep of hybrid backward l1-Gauss-Seidel for the up cycle"; DESIGN.md R-gs):
the colourings against their definitions, the sweeps against the dense matrices that define them, the V-cycle
against the textbook two-grid error propagation, symmetry for SPD inputs and the special cases.  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from test_oracle import _laplacian7 as _lap7


def _fmix(i):
    x = int(i) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def _block_colouring(A, B):
    """First fit in descending (fmix32(i), i) inside each block of B rows (the definition, in Python)."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    col = -np.ones(n, int)
    for b0 in range(0, n, B):
        b1 = min(n, b0 + B)
        for v in sorted(range(b0, b1), key=lambda i: (_fmix(i), i), reverse=True):
            used = {col[u] for u in A.indices[A.indptr[v]:A.indptr[v + 1]] if u != v and b0 <= u < b1 and col[u] >= 0}
            c = 0
            while c in used:
                c += 1
            col[v] = c
    return col


def _sweep_matrices(A, col, B, dh):
    """(D^ + L^, D^ + U^) of the hybrid sweep: L^ / U^ = in-block entries to rows of a lower / higher colour,
    D^ = the hybrid l1 diagonal (B = n and dh = diag(A): the multicolour sweep of a whole level)."""
    Ad = A.toarray()
    n = Ad.shape[0]
    blk = np.arange(n) // B
    same = blk[:, None] == blk[None, :]
    Lm = np.where(same & (col[None, :] < col[:, None]), Ad, 0.0)
    Um = np.where(same & (col[None, :] > col[:, None]), Ad, 0.0)
    return np.diag(dh) + Lm, np.diag(dh) + Um


def test_level0_geometric_colourings_are_proper():
    """R-gs level 0: node colour = parity of (x, y, z) (8 colours) for the 27-point mechanics graph, cell colour
    = parity of x + y + z (2 colours) for the 7-point S_pp: no stored coupling joins two rows of one colour."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb, amg_smoother=1).setup()
    for which, ncol in ((0, 8), (1, 2)):
        L0 = o.level(which, 0)
        col, nc = o.colour(which, 0)
        assert nc == ncol
        rows = np.repeat(np.arange(L0["n"]), np.diff(L0["A_rp"]))
        off = rows != L0["A_ci"]
        assert np.all(col[rows[off]] != col[L0["A_ci"][off]])
    n = np.arange(pb.Nn)
    x, y, z = n % (pb.nx + 1), (n // (pb.nx + 1)) % (pb.ny + 1), n // ((pb.nx + 1) * (pb.ny + 1))
    assert np.array_equal(o.colour(0, 0)[0], (x & 1) + 2 * (y & 1) + 4 * (z & 1))


@pytest.mark.parametrize("B", [64, 1024])
def test_hybrid_block_colouring_is_first_fit_by_priority(B):
    """Coarse levels: each block of B rows coloured by first fit in descending (fmix32(i), i) (checked against
    an independent Python statement), proper inside every block."""
    A = _lap7(9, 8, 7, neumann=False)
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_smoother=1, amg_gs_block=B, amg_coarse_max=8)
    for lvl, L in enumerate(amg.levels()[:-1]):
        col, nc = amg.colour(lvl)
        Al = sp.csr_matrix((L["A_v"][:, 0], L["A_ci"], L["A_rp"]), shape=(L["n"], L["n"]))
        ref = _block_colouring(Al, B)
        assert np.array_equal(col, ref) and nc == ref.max() + 1
        r, c = Al.nonzero()
        inb = (r // B == c // B) & (r != c)
        assert np.all(col[r[inb]] != col[c[inb]])


def _two_level(A, amg, B, lvl0_block):
    L0, L1 = amg.levels()[:2]
    n = L0["n"]
    P = sp.csr_matrix((L0["P_v"][:, 0], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
    col, _ = amg.colour(0)
    gsb, dh = amg.gs(0)
    assert gsb == lvl0_block
    dh = dh[:, 0] if gsb else A.diagonal()
    F, Bk = _sweep_matrices(A, col, gsb if gsb else n, dh)
    Ad = A.toarray()
    I = np.eye(n)
    return (I - np.linalg.solve(Bk, Ad)) @ (I - P @ np.linalg.solve(P.T @ Ad @ P, P.T @ Ad)) @ (I - np.linalg.solve(F, Ad))


def test_hybrid_two_grid_error_propagation():
    """V(1,1) with hybrid l1-GS (Baker et al. 2011) on a two-level hierarchy: E = I - M A equals
    (I - (D^+U^)^-1 A)(I - P A_c^-1 P^T A)(I - (D^+L^)^-1 A), D^ = a_ii + sign(a_ii) sum_{off-block}|a_ij|."""
    A = _lap7(7, 6, 6, neumann=False)
    B = 64
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_smoother=1, amg_gs_block=B, amg_coarse_max=60)
    assert len(amg.levels()) == 2 and amg.levels()[1]["coarsest"]
    _, dh = amg.gs(0)
    Ad = A.toarray()
    blk = np.arange(A.shape[0]) // B
    off = np.where(blk[:, None] != blk[None, :], np.abs(Ad), 0.0).sum(1)
    np.testing.assert_allclose(dh[:, 0], np.diag(Ad) + off, rtol=1e-15)      # positive diagonal here
    E_ref = _two_level(A, amg, B, B)
    n = A.shape[0]
    M = np.stack([amg.vcycle(e) for e in np.eye(n)], 1)
    assert np.abs(np.eye(n) - M @ Ad - E_ref).max() <= 1e-11


def test_multicolour_two_grid_error_propagation():
    """A level with a given colouring (level 0 of the coupled problem) is swept by plain multicolour GS:
    E = (I - (D+U^)^-1 A)(I - P A_c^-1 P^T A)(I - (D+L^)^-1 A) with L^ / U^ the couplings to lower / higher
    colours over the whole level (red-black here)."""
    nx, ny, nz = 7, 6, 6
    A = _lap7(nx, ny, nz, neumann=False)
    i = np.arange(nx * ny * nz)
    rb = ((i % nx) + (i // nx) % ny + i // (nx * ny)) % 2
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, colour0=rb, amg_smoother=1, amg_coarse_max=60)
    assert amg.colour(0)[1] == 2
    E_ref = _two_level(A, amg, None, 0)
    n = A.shape[0]
    M = np.stack([amg.vcycle(e) for e in np.eye(n)], 1)
    assert np.abs(np.eye(n) - M @ A.toarray() - E_ref).max() <= 1e-11


def test_gs_vcycle_symmetric_for_spd_and_faster_than_l1_jacobi():
    """Forward GS down, backward GS up: the V-cycle is a symmetric operator for SPD A; as a
    stationary iteration on 3-D Poisson it contracts faster than the l1-Jacobi cycle (measured 0.46 vs 0.62)."""
    A = _lap7(12, 12, 12, neumann=False)
    rng = np.random.default_rng(7)
    v, w = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    rates = {}
    for sm in (0, 1):
        amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_smoother=sm, amg_gs_block=256)
        assert abs(amg.vcycle(v) @ w - v @ amg.vcycle(w)) <= 1e-12 * abs(amg.vcycle(v) @ w)
        x = np.zeros(A.shape[0]); b = rng.standard_normal(A.shape[0])
        r0 = np.linalg.norm(b)
        for _ in range(10):
            x = x + amg.vcycle(b - A @ x)
        rates[sm] = (np.linalg.norm(b - A @ x) / r0) ** 0.1
    assert rates[1] < 0.8 * rates[0], rates


def test_gs_isolated_rows_exact_after_the_first_sweep():
    """A row with no off-diagonal (Dirichlet, D11) has d_i = a_ii and no coupling: the forward sweep sets
    x_i = b_i / a_ii, the coarse correction (zero P row) and the backward sweep keep it."""
    A = _lap7(6, 5, 6, neumann=False).tolil()
    dirichlet = np.arange(0, 30)
    for i in dirichlet:
        A[i, :] = 0.0
        A[:, i] = 0.0
        A[i, i] = 3.0
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_smoother=1, amg_gs_block=64, amg_coarse_max=8)
    b = np.random.default_rng(9).uniform(-1, 1, A.shape[0])
    np.testing.assert_allclose(amg.vcycle(b)[dirichlet], b[dirichlet] / 3.0, rtol=1e-15)


def test_gs_cycle_is_sign_equivariant():
    """R-l1 sign convention carries over to the hybrid diagonal: V(-A) = -V(A) exactly."""
    A = _lap7(7, 6, 5, neumann=False)
    b = np.random.default_rng(4).uniform(-1, 1, A.shape[0])
    xa = oracle.Amg(A.indptr, A.indices, A.data, None, amg_smoother=1, amg_gs_block=64, amg_coarse_max=20).vcycle(b)
    xn = oracle.Amg(A.indptr, A.indices, -A.data, None, amg_smoother=1, amg_gs_block=64, amg_coarse_max=20).vcycle(b)
    assert np.array_equal(xn, -xa)


def test_gs_preconditioner_fewer_fgmres_iterations():
    """On the coupled problem (C2) the GS smoothers of P:711 need fewer FGMRES iterations than l1-Jacobi
    (measured 61 -> 47); both converge with a verified true residual."""
    pb = synth.generate("C2")
    its = {}
    for sm in (0, 1):
        o = oracle.Oracle(pb, amg_smoother=sm).setup()
        x, info = o.solve(pb.b, rtol=1e-8)
        assert info["status"] == 0 and info["true_relres"] <= 1e-8
        its[sm] = info["iterations"]
    assert its[1] <= 0.85 * its[0], its

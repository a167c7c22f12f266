"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics
fix -- closed forms, exact limits, textbook equivalences, invariants and brute
force on tiny inputs (never against itself).  Each test names the passage.
CPU only (no `gpu` marker)."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth


def _dense_blocks(pb, fs=True):
    A, (Auu, Auf, Afu, Aff) = synth.to_scipy(pb)
    Auu, Auf, Afu, Aff = (M.toarray() for M in (Auu, Auf, Afu, Aff))
    Sfs = Aff.copy()
    if fs:
        Sfs[0::2, 1::2] += np.diag(pb.fs[:, 0])
        Sfs[1::2, 1::2] += np.diag(pb.fs[:, 1])
    return A.toarray(), Auu, Auf, Afu, Aff, Sfs


@pytest.fixture(scope="module")
def tiny():
    return synth.generate(nx=3, ny=3, nz=3, recipe=2, perm_sigma=2.0)


# ---------------------------------------------------------------- operator (a12)
def test_operator_equals_assembled_matvec():
    """eq:jac_system: the oracle's block loops = scipy's BSR matvec."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb)
    A, _ = synth.to_scipy(pb)
    x = np.random.default_rng(3).uniform(-1, 1, pb.n)
    y = o.operator(x)
    assert np.linalg.norm(y - A @ x) <= 1e-14 * np.linalg.norm(y)


# ---------------------------------------------------------------- exact limits (Algorithm 1 structure)
def test_exact_limit_is_block_lower_inverse(tiny):
    """M_uu = A_uu^-1 and M_ff = S_ff^-1 (exact, eq:LU P:366) => M^-1 = L^-1
    (P:371-378).  z is compared with the dense L^-1 v."""
    pb = tiny
    A, Auu, Auf, Afu, Aff, _ = _dense_blocks(pb)
    o = oracle.Oracle(pb, mech_mode=1, ff_mode=1).setup()
    nu = Auu.shape[0]
    S = Aff - Afu @ np.linalg.solve(Auu, Auf)
    Linv = np.zeros_like(A)
    Auu_inv = np.linalg.inv(Auu)
    S_inv = np.linalg.inv(S)
    Linv[:nu, :nu] = Auu_inv
    Linv[nu:, :nu] = -S_inv @ Afu @ Auu_inv
    Linv[nu:, nu:] = S_inv
    rng = np.random.default_rng(1)
    for _ in range(3):
        v = rng.uniform(-1, 1, pb.n)
        z = o.apply(v)
        assert np.linalg.norm(z - Linv @ v) <= 1e-9 * np.linalg.norm(Linv @ v)


def test_exact_limit_fgmres_two_iterations(tiny):
    """L^-1 A = U has the single eigenvalue 1 and (U - I)^2 = 0, so
    FGMRES converges in <= 2 iterations (assert <= 3)."""
    o = oracle.Oracle(tiny, mech_mode=1, ff_mode=1).setup()
    x, info = o.solve(tiny.b, rtol=1e-10)
    assert info["status"] == 0 and info["iterations"] <= 3


def test_exact_local_stage_gives_exact_fs_inverse(tiny):
    """M_L = (S_ff^FS)^-1 => M_ff = M_G + M_L (I - S M_G) = (S_ff^FS)^-1 for
    any M_G (eq:mult_prec_op); with M_uu exact, step 2
    gives z_f = (S^FS)^-1 (v_f - A_fu A_uu^-1 v_u)."""
    pb = tiny
    _, Auu, _, Afu, _, Sfs = _dense_blocks(pb)
    o = oracle.Oracle(pb, mech_mode=1, local_mode=1).setup()
    nu = Auu.shape[0]
    v = np.random.default_rng(2).uniform(-1, 1, pb.n)
    z = o.apply(v)
    zu = np.linalg.solve(Auu, v[:nu])
    zf = np.linalg.solve(Sfs, v[nu:] - Afu @ zu)
    assert np.linalg.norm(z[:nu] - zu) <= 1e-10 * np.linalg.norm(zu)
    assert np.linalg.norm(z[nu:] - zf) <= 1e-8 * np.linalg.norm(zf)


def test_global_stage_composition(tiny):
    """With M_pp exact and no local stage, M_ff = M_G of eq:S1_prec:
    diag(I, S_pp^-1) [[I,0],[-A_ps, I]] diag(D_ss^-1, I), full A_ps,
    D_ss = diagm(A_ss) and S_pp = A_pp^FS - D_ps D_ss^-1 A_sp^FS."""
    pb = tiny
    _, Auu, _, Afu, Aff, Sfs = _dense_blocks(pb)
    o = oracle.Oracle(pb, mech_mode=1, pres_mode=1, local_mode=2).setup()
    nu, nc = Auu.shape[0], pb.Nc
    Ass, Aps = Aff[0::2, 0::2], Aff[1::2, 0::2]
    Asp_fs, App_fs = Sfs[0::2, 1::2], Sfs[1::2, 1::2]
    Dss, Dps = np.diag(np.diag(Ass)), np.diag(np.diag(Aps))
    Spp = App_fs - Dps @ np.linalg.inv(Dss) @ Asp_fs
    MG = np.block([[np.eye(nc), np.zeros((nc, nc))], [np.zeros((nc, nc)), np.linalg.inv(Spp)]]) \
        @ np.block([[np.eye(nc), np.zeros((nc, nc))], [-Aps, np.eye(nc)]]) \
        @ np.block([[np.linalg.inv(Dss), np.zeros((nc, nc))], [np.zeros((nc, nc)), np.eye(nc)]])
    v = np.random.default_rng(4).uniform(-1, 1, pb.n)
    z = o.apply(v)
    yf = v[nu:] - Afu @ np.linalg.solve(Auu, v[:nu])
    yp = np.concatenate([yf[0::2], yf[1::2]])            # P^T: partitioned (s; p)
    zp = MG @ yp
    got = np.concatenate([z[nu:][0::2], z[nu:][1::2]])
    assert np.linalg.norm(got - zp) <= 1e-8 * np.linalg.norm(zp)


def test_quasi_impes_exact_when_blocks_diagonal():
    """With g = 0 and no flow (hydrostatic, every Phi = 0) A_ss and A_ps are
    diagonal, so quasi-IMPES S_pp equals the exact second-level Schur complement
    A_pp^FS - A_ps A_ss^-1 A_sp^FS (P:555 vs P:579)."""
    pb = synth.generate(nx=3, ny=3, nz=2, recipe=1, gravity=0.0)
    _, _, _, _, Aff, Sfs = _dense_blocks(pb)
    Ass, Aps = Aff[0::2, 0::2], Aff[1::2, 0::2]
    assert np.count_nonzero(Ass - np.diag(np.diag(Ass))) == 0
    exact = Sfs[1::2, 1::2] - Aps @ np.linalg.solve(Ass, Sfs[0::2, 1::2])
    o = oracle.Oracle(pb).setup()
    Dss, rp, ci, v = o.spp()
    got = sp.csr_matrix((v, ci, rp), shape=(pb.Nc, pb.Nc)).toarray()
    assert np.abs(got - exact).max() <= 1e-12 * np.abs(exact).max()
    assert np.array_equal(Dss, np.diag(Ass))


def test_sparsity_preserved_by_reductions(tiny):
    """pattern(S_pp) = pattern(A_pp)."""
    o = oracle.Oracle(tiny).setup()
    _, rp, ci, _ = o.spp()
    assert np.array_equal(rp, tiny.ff_rowptr) and np.array_equal(ci, tiny.ff_col)


def test_identity_subsolvers_trace():
    """Decoupled problem (b = 0, g = 0 => A_fu = 0): z_u depends on
    v_u only and z_f on v_f only."""
    pb = synth.generate(nx=3, ny=3, nz=3, recipe=1, biot=0.0, gravity=0.0)
    o = oracle.Oracle(pb).setup()
    nu = 3 * pb.Nn
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, pb.n)
    w = v.copy(); w[nu:] = 0
    z1, z2 = o.apply(v), o.apply(w)
    assert np.array_equal(z1[:nu], z2[:nu])
    assert np.all(z2[nu:] == 0)


def test_apply_is_linear():
    """Every stage of Algorithm 1 is a fixed linear operator (V-cycles with zero
    initial guess, ILU solves) -- FGMRES relies on it only for the iteration
    count; M(a v + w) = a M v + M w to rounding."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb).setup()
    rng = np.random.default_rng(6)
    v, w = rng.uniform(-1, 1, pb.n), rng.uniform(-1, 1, pb.n)
    lhs = o.apply(2.5 * v + w)
    rhs = 2.5 * o.apply(v) + o.apply(w)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(lhs)


# ---------------------------------------------------------------- MIS(2) / aggregation (a4)
def _grid_graph(nx, ny, nz, stencil=27):
    idx = np.arange(nx * ny * nz).reshape(nz, ny, nx)
    rows = [[] for _ in range(nx * ny * nz)]
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                for dk in (-1, 0, 1):
                    for dj in (-1, 0, 1):
                        for di in (-1, 0, 1):
                            if (di, dj, dk) == (0, 0, 0):
                                continue
                            if stencil == 7 and abs(di) + abs(dj) + abs(dk) != 1:
                                continue
                            ii, jj, kk = i + di, j + dj, k + dk
                            if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                                rows[idx[k, j, i]].append(idx[kk, jj, ii])
    rp = np.zeros(len(rows) + 1, np.int32)
    rp[1:] = np.cumsum([len(r) for r in rows])
    return rp, np.concatenate([sorted(r) for r in rows]).astype(np.int32)


def _random_graph(n, deg, seed):
    rng = np.random.default_rng(seed)
    adj = [set() for _ in range(n)]
    for _ in range(n * deg // 2):
        a, b = rng.integers(0, n, 2)
        if a != b:
            adj[a].add(b); adj[b].add(a)
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum([len(s) for s in adj])
    ci = np.concatenate([sorted(s) for s in adj] + [np.zeros(0, int)]).astype(np.int32)
    return rp, ci


def _dist(rp, ci, src, maxd):
    seen = {src: 0}
    frontier = [src]
    for d in range(1, maxd + 1):
        nxt = []
        for u in frontier:
            for w in ci[rp[u]:rp[u + 1]]:
                if w not in seen:
                    seen[w] = d; nxt.append(w)
        frontier = nxt
    return seen


@pytest.mark.parametrize("graph", ["grid27", "grid7", "rand4", "rand9"])
def test_mis2_greedy_equals_rounds_and_is_maximal(graph):
    """Greedy MIS(2) by descending priority == parallel local-max rounds (the
    lexicographically-first MIS of the distance-2 graph), and the
    result is a distance-2 independent, maximal set."""
    if graph == "grid27":
        rp, ci = _grid_graph(7, 6, 5, 27)
    elif graph == "grid7":
        rp, ci = _grid_graph(9, 8, 7, 7)
    else:
        rp, ci = _random_graph(400, int(graph[4:]), seed=int(graph[4:]))
    n = len(rp) - 1
    h = oracle.fmix32(np.arange(n))
    g, _ = oracle.mis2(rp, ci, h, rounds=False)
    r, nrounds = oracle.mis2(rp, ci, h, rounds=True)
    assert np.array_equal(g, r) and nrounds >= 1
    roots = np.flatnonzero(g == 1)
    near = np.zeros(n, bool)
    for v in roots:
        d = _dist(rp, ci, v, 2)
        assert all(g[u] != 1 for u in d if u != v)       # independence at distance 2
        near[list(d)] = True
    nonisolated = np.diff(rp) > 0
    assert np.all(near[nonisolated])                      # maximality
    assert np.all(g[~nonisolated] == -1)


def _laplacian7(nx, ny, nz, neumann=True):
    rp, ci = _grid_graph(nx, ny, nz, 7)
    n = nx * ny * nz
    rows = np.repeat(np.arange(n), np.diff(rp))
    A = sp.csr_matrix((-np.ones(len(ci)), ci, rp), shape=(n, n)).toarray()
    np.fill_diagonal(A, -A.sum(1) + (0.0 if neumann else 1e-3))
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def test_aggregates_partition_connected_confined():
    """Aggregates partition the non-isolated nodes, are connected in the
    strength graph and lie inside one z-block."""
    nx, ny, nz = 8, 7, 12
    A = _laplacian7(nx, ny, nz, neumann=False)
    zb = (np.arange(nx * ny * nz) // (nx * ny) // 5).astype(np.int32)
    amg = oracle.Amg(A.indptr, A.indices, A.data, zb, amg_coarse_max=4)
    L0 = amg.levels()[0]
    agg = L0["agg"]
    assert agg.min() >= 0 and agg.max() == L0["nagg"] - 1
    for J in range(L0["nagg"]):
        mem = np.flatnonzero(agg == J)
        assert len(set(zb[mem])) == 1
        sub = A[mem][:, mem].toarray() != 0
        reach = {0}; stack = [0]
        while stack:
            u = stack.pop()
            for w in np.flatnonzero(sub[u]):
                if w not in reach:
                    reach.add(w); stack.append(w)
        assert len(reach) == len(mem)


def test_prolongator_preserves_constants_and_galerkin():
    """Zero row sums in A^F => (P 1)_i = 1 (near-null space preserved, SURVEY
    c.4); A_c equals the dense Galerkin product P^T A P; symmetric A => A_c
    symmetric."""
    A = _laplacian7(9, 8, 7, neumann=True)
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=8)
    Ls = amg.levels()
    L0, L1 = Ls[0], Ls[1]
    P = sp.csr_matrix((L0["P_v"][:, 0], L0["P_ci"], L0["P_rp"]), shape=(L0["n"], L0["nagg"])).toarray()
    np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-13)
    Ac = sp.csr_matrix((L1["A_v"][:, 0], L1["A_ci"], L1["A_rp"]), shape=(L1["n"], L1["n"])).toarray()
    ref = P.T @ A.toarray() @ P
    assert np.abs(Ac - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.abs(Ac - Ac.T).max() <= 1e-13 * np.abs(Ac).max()


def test_two_grid_error_propagation_formula():
    """The V(1,1) l1-Jacobi cycle on a two-level hierarchy has the textbook
    error propagation E = I - M A = (I - D^-1 A)(I - P A_c^-1 P^T A)(I - D^-1 A)."""
    A = _laplacian7(6, 5, 6, neumann=False)
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=60)
    Ls = amg.levels()
    assert len(Ls) == 2 and Ls[1]["coarsest"]
    n = A.shape[0]
    L0 = Ls[0]
    P = sp.csr_matrix((L0["P_v"][:, 0], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
    Ad = A.toarray()
    D = np.abs(Ad).sum(1)
    S = np.eye(n) - Ad / D[:, None]
    Ac = P.T @ Ad @ P
    E_ref = S @ (np.eye(n) - P @ np.linalg.solve(Ac, P.T @ Ad)) @ S
    M = np.stack([amg.vcycle(e) for e in np.eye(n)], 1)
    E = np.eye(n) - M @ Ad
    assert np.abs(E - E_ref).max() <= 1e-11


def test_vcycle_symmetric_for_spd_and_converges():
    """SPD A => the V-cycle is a symmetric operator and, as a
    stationary iteration on a 3-D Poisson problem, contracts the error."""
    A = _laplacian7(12, 12, 12, neumann=False)
    amg = oracle.Amg(A.indptr, A.indices, A.data, None)
    rng = np.random.default_rng(7)
    v, w = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    assert abs(amg.vcycle(v) @ w - v @ amg.vcycle(w)) <= 1e-12 * abs(amg.vcycle(v) @ w)
    x = np.zeros(A.shape[0]); b = rng.standard_normal(A.shape[0])
    r0 = np.linalg.norm(b)
    for _ in range(10):
        x = x + amg.vcycle(b - A @ x)
    assert np.linalg.norm(b - A @ x) <= 0.75 ** 10 * r0   # measured factor ~0.62 per cycle


def test_sdc_components_use_one_graph():
    """Three SDC components share one node aggregation; each
    component's coarse operator is its own Galerkin product."""
    A = _laplacian7(6, 6, 6, neumann=False)
    v = np.stack([A.data, 2.0 * A.data, 0.5 * A.data], 1)
    amg3 = oracle.Amg(A.indptr, A.indices, v, None, amg_coarse_max=20)
    amg1 = oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=20)
    L3, L1 = amg3.levels(), amg1.levels()
    assert np.array_equal(L3[0]["agg"], L1[0]["agg"])
    np.testing.assert_allclose(L3[1]["A_v"][:, 1], 2.0 * L1[1]["A_v"][:, 0], rtol=1e-13)


# ---------------------------------------------------------------- ILU(0) (a5)
def test_ilu0_defining_property_and_tile_blocking():
    """(L U)_ij = A_ij on the in-tile pattern (the definition of ILU(0)); entries
    coupling different tiles are not represented (block Jacobi over tiles,
    SURVEY D7)."""
    pb = synth.generate(nx=4, ny=3, nz=4, recipe=2, perm_sigma=2.0)
    rp, ci, v = pb.ff_rowptr, pb.ff_col, pb.ff_val
    tile = (2, 3, 2)
    ilu = oracle.Ilu(pb.nx, pb.ny, pb.nz, tile, rp, ci, v)
    n2 = 2 * pb.Nc
    Minv = np.stack([ilu.apply(e) for e in np.eye(n2)], 1)
    M = np.linalg.inv(Minv)
    A = sp.bsr_matrix((v, ci, rp), shape=(n2, n2)).toarray()

    def tile_of(c):
        i, j, k = c % pb.nx, (c // pb.nx) % pb.ny, c // (pb.nx * pb.ny)
        return (i // tile[0], j // tile[1], k // tile[2])

    for K in range(pb.Nc):
        for q in range(rp[K], rp[K + 1]):
            J = ci[q]
            blk = M[2 * K:2 * K + 2, 2 * J:2 * J + 2]
            if tile_of(K) == tile_of(J):
                np.testing.assert_allclose(blk, A[2 * K:2 * K + 2, 2 * J:2 * J + 2], rtol=1e-8, atol=1e-12 * np.abs(A).max())
            else:
                assert np.abs(blk).max() <= 1e-8 * np.abs(A).max()


def test_ilu0_exact_on_a_column_tile():
    """A 1 x 1 x nz column is block tridiagonal: ILU(0) has no fill and is the
    exact LU (SURVEY c.4)."""
    pb = synth.generate(nx=1, ny=1, nz=6, recipe=1)
    n2 = 2 * pb.Nc
    ilu = oracle.Ilu(1, 1, 6, (1, 1, 16), pb.ff_rowptr, pb.ff_col, pb.ff_val)
    A = sp.bsr_matrix((pb.ff_val, pb.ff_col, pb.ff_rowptr), shape=(n2, n2)).toarray()
    w = np.random.default_rng(8).uniform(-1, 1, n2)
    x = ilu.apply(w)
    assert np.linalg.norm(A @ x - w) <= 1e-10 * np.linalg.norm(w)


# ---------------------------------------------------------------- FGMRES (a14)
def test_fgmres_solves_c1_and_estimate_is_true_residual():
    """FGMRES(64) to 1e-8 (north star); the Arnoldi estimate equals the true
    residual (right preconditioning preserves it); x -> x_rand."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb).setup()
    x, info = o.solve(pb.b, rtol=1e-8, m=64)
    assert info["status"] == 0 and info["true_relres"] <= 1e-8
    assert abs(info["est_relres"] - info["true_relres"]) <= 1e-3 * info["true_relres"]
    assert np.linalg.norm(x - pb.x_rand) <= 1e-3 * np.linalg.norm(pb.x_rand)


def test_fgmres_restart_path():
    """A short restart length still reaches the tolerance (restart logic)."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb).setup()
    x, info = o.solve(pb.b, rtol=1e-8, m=8, maxit=2000)
    assert info["status"] == 0 and info["restarts"] >= 1 and info["true_relres"] <= 1e-8


def test_fgmres_reports_non_convergence():
    """Non-convergence is an explicit result, never a silent answer."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb).setup()
    x, info = o.solve(pb.b, rtol=1e-14, m=4, maxit=6)
    assert info["status"] == 1 and info["iterations"] == 6


def test_vcycle_is_sign_equivariant():
    """R-l1: d_i = sign(a_ii) sum_j |a_ij|.  Strength, aggregation and the prolongator depend on |a_ij| and
    D^-1 A only, so the V-cycle of -A must be exactly minus the V-cycle of A (the unsigned l1 scaling breaks
    this: a negative-diagonal row would be 'smoothed' uphill).  Exact in IEEE arithmetic (negation)."""
    A = _laplacian7(7, 6, 5, neumann=False)
    b = np.random.default_rng(4).uniform(-1, 1, A.shape[0])
    xa = oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=20).vcycle(b)
    xn = oracle.Amg(A.indptr, A.indices, -A.data, None, amg_coarse_max=20).vcycle(b)
    assert len(oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=20).levels()) >= 3
    assert np.array_equal(xn, -xa)

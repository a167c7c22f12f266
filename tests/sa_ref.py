"""Second, numpy-only statement of ONE smoothed-aggregation level (DESIGN.md R-strength,
R-mis2, R-agg, R-prolong), written from the readings' text and NOT from oracle/oracle.c.  It is used to
write tests/golden/sa_level.txt (tests/golden/make_sa_level.py) and to re-derive the oracle's prolongator on
random inputs (tests/test_oracle_sa.py).  Dense matrices and whole-array numpy operations; no oracle import.

  strength  (D2)  S_ij  iff  j != i, zb(i) == zb(j), m_i > 0, meas_ij >= theta * m_i,
                  meas_ij = sum_c |a^c_ij|,  m_i = max_{k != i} meas_ik;   E = S or S^T
  MIS(2)    (D3)  greedy over the non-isolated nodes by descending (fmix32(i), i): a node still undecided
                  becomes a root and every node within strong-graph distance 2 of it is decided
  aggregate (D3)  phase 1: root + its strong neighbours, aggregates numbered by ascending root id;
                  phase 2: a remaining non-isolated node joins the phase-1 aggregate of its strong neighbour
                  of maximal meas, ties to the smallest aggregate id
  prolong   (D5)  A^F_c = strong entries of A_c, weak off-diagonal entries added to the diagonal;
                  rho_c = max_i sum_j |A^F_c,ij| / |A^F_c,ii|;  omega_c = 4 / (3 rho_c);
                  P_c = P_tent - omega_c D_F,c^-1 A^F_c P_tent  (P_tent 0/1, zero rows for unaggregated nodes,
                  rows with A^F_ii = 0 keep P_tent)
"""
import numpy as np

ISOLATED, UNDECIDED, ROOT, OUT = -1, 0, 1, 2


def fmix32(i):
    """MurmurHash3's fmix32 finaliser (the fixed priority hash of D3), in plain Python integers."""
    x = int(i) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    x ^= x >> 16
    return x


def strength(A, zb, theta=0.25):
    """A: (nc, n, n) dense values, zero = no entry; returns the symmetrised strong-edge matrix E (bool)."""
    M = np.abs(A).sum(0)
    n = M.shape[0]
    off = M.copy()
    np.fill_diagonal(off, 0.0)
    m = off.max(1) if n else np.zeros(0)
    S = (off >= theta * m[:, None]) & (m[:, None] > 0) & (zb[:, None] == zb[None, :]) & (off != 0)
    np.fill_diagonal(S, False)
    return S | S.T


def mis2(E):
    n = E.shape[0]
    st = np.where(E.any(1), UNDECIDED, ISOLATED)
    order = sorted(np.flatnonzero(st == UNDECIDED), key=lambda i: (fmix32(i), i), reverse=True)
    E1 = E | np.eye(n, dtype=bool)
    reach2 = (E1.astype(int) @ E1.astype(int)) > 0
    for v in order:
        if st[v] != UNDECIDED:
            continue
        st[v] = ROOT
        st[(st == UNDECIDED) & reach2[v]] = OUT
    return st


def aggregate(A, E, st):
    M = np.abs(A).sum(0)
    n = len(st)
    roots = np.flatnonzero(st == ROOT)
    ph1 = np.full(n, -1)
    for a, r in enumerate(roots):
        ph1[r] = a
        ph1[E[r]] = a
    agg = ph1.copy()
    for v in range(n):
        if st[v] == ISOLATED or ph1[v] >= 0:
            continue
        cand = [(M[v, j], -ph1[j]) for j in np.flatnonzero(E[v]) if ph1[j] >= 0]
        agg[v] = -max(cand)[1] if cand else -1
    return ph1, agg, len(roots)


def prolongator(A, E, agg, nagg):
    """Returns (P (nc, n, nagg), rho (nc), omega (nc), AF (nc, n, n))."""
    nc, n, _ = A.shape
    Pt = np.zeros((n, nagg))
    rows = np.flatnonzero(agg >= 0)
    Pt[rows, agg[rows]] = 1.0
    off = ~np.eye(n, dtype=bool)
    P, rho, omega, AF = [], [], [], []
    for c in range(nc):
        F = np.where(E, A[c], 0.0)
        d = np.diag(A[c]) + np.where(off & ~E, A[c], 0.0).sum(1)
        F[np.arange(n), np.arange(n)] = d
        nzd = d != 0
        r = (np.abs(F[nzd]).sum(1) / np.abs(d[nzd])).max() if nzd.any() else 0.0
        w = 4.0 / (3.0 * r) if r > 0 else 0.0
        scale = np.where(nzd, w / np.where(nzd, d, 1.0), 0.0)
        P.append(Pt - scale[:, None] * (F @ Pt))
        rho.append(r)
        omega.append(w)
        AF.append(F)
    return np.array(P), np.array(rho), np.array(omega), np.array(AF)


def level(A, zb, theta=0.25):
    E = strength(A, zb, theta)
    st = mis2(E)
    ph1, agg, nagg = aggregate(A, E, st)
    P, rho, omega, _ = prolongator(A, E, agg, nagg)
    # the aggregated rows of P only keep the aggregates of {i} U strong(i): the others are exact zeros
    return dict(E=E, st=st, ph1=ph1, agg=agg, nagg=nagg, P=P, rho=rho, omega=omega)

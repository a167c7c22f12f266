"""The identity behind the fused tile-ILU kernel (paper_1812_05540_b200/csrc/ilu.cu), checked in
numpy on a small ragged multi-tile grid with 2x2 blocks: for M = (D + L) D^-1 (D + U) on each tile (D = the DILU
pivots U_KK of the 7-point pattern, L / U = the in-tile lower / upper blocks) and S = L + S_KK + U + C (C = the
couplings that leave the tile), steps 6-8 of Algorithm 1,
    z + M^-1 (y - S z)  =  z + (I + D^-1 U)^-1 [ (D + L)^-1 (y - E z - U z - C z) - z ],   E = S_KK - D,
for ANY block diagonal D (so also for perturbed pivots and for the hybrid block Gauss-Seidel stage, D = S_KK, E = 0,
where the new z is the forward solve itself).  No GPU, no oracle: plain linear algebra."""
import numpy as np
import pytest


def _system(seed, nx=5, ny=4, nz=6, tx=3, ty=2, tz=4):
    rng = np.random.default_rng(seed)
    N = nx * ny * nz
    idx = lambda i, j, k: i + nx * (j + ny * k)   # noqa: E731
    S = np.zeros((2 * N, 2 * N))
    tile = np.empty(N, dtype=np.int64)
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                c = idx(i, j, k)
                tile[c] = (i // tx) + 100 * (j // ty) + 10000 * (k // tz)
                S[2 * c:2 * c + 2, 2 * c:2 * c + 2] = np.array([[6.0, 0.5], [-0.3, 7.0]]) + rng.uniform(0, 1, (2, 2))
                for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
                    a, b, e = i + d[0], j + d[1], k + d[2]
                    if 0 <= a < nx and 0 <= b < ny and 0 <= e < nz:
                        q = idx(a, b, e)
                        S[2 * c:2 * c + 2, 2 * q:2 * q + 2] = -rng.uniform(0.1, 1.0, (2, 2))
    same = np.kron((tile[:, None] == tile[None, :]).astype(float), np.ones((2, 2)))
    blk = np.kron(np.eye(N), np.ones((2, 2)))
    lower = np.kron(np.tril(np.ones((N, N)), -1), np.ones((2, 2)))
    L, U = S * same * lower, S * same * lower.T
    SKK = S * blk
    C = S - SKK - L - U
    return N, S, SKK, L, U, C


def _dilu(N, SKK, L, U):
    D = np.zeros_like(SKK)
    for K in range(N):
        B = SKK[2 * K:2 * K + 2, 2 * K:2 * K + 2].copy()
        for J in range(K):
            A = L[2 * K:2 * K + 2, 2 * J:2 * J + 2]
            if A.any():
                B -= A @ np.linalg.solve(D[2 * J:2 * J + 2, 2 * J:2 * J + 2], U[2 * J:2 * J + 2, 2 * K:2 * K + 2])
        D[2 * K:2 * K + 2, 2 * K:2 * K + 2] = B
    return D


@pytest.mark.parametrize("kind", ["dilu", "block_gs", "perturbed"])
def test_eisenstat_form_of_steps_6_to_8(kind):
    N, S, SKK, L, U, C = _system(3)
    rng = np.random.default_rng(7)
    y, z = rng.normal(size=2 * N), rng.normal(size=2 * N)
    if kind == "dilu":
        D = _dilu(N, SKK, L, U)
        # the 7-point ILU(0) only updates diagonal blocks: (D + L) D^-1 (D + U) reproduces S on the in-tile pattern
        M = (D + L) @ np.linalg.solve(D, D + U)
        mask = (np.abs(SKK + L + U) > 0)
        assert np.abs((M - (SKK + L + U))[mask]).max() <= 1e-12
    elif kind == "block_gs":
        D = SKK.copy()
    else:
        D = _dilu(N, SKK, L, U) + 0.37 * np.kron(np.eye(N), np.eye(2))
    I = np.eye(2 * N)
    if kind == "block_gs":                     # M_L = D + L: the forward sweep is the whole stage
        ref = z + np.linalg.solve(D + L, y - S @ z)
        s = np.linalg.solve(D + L, y - (SKK - D) @ z - U @ z - C @ z)
        assert np.abs(s - ref).max() <= 1e-12 * np.abs(ref).max()
        return
    M = (D + L) @ np.linalg.solve(D, D + U)
    ref = z + np.linalg.solve(M, y - S @ z)
    E = SKK - D
    s = np.linalg.solve(D + L, y - E @ z - U @ z - C @ z)
    x = np.linalg.solve(I + np.linalg.solve(D, U), s - z)
    assert np.abs(z + x - ref).max() <= 1e-12 * np.abs(ref).max()

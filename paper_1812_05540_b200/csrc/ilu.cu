// ilu.cu -- row a5 (factorisation) and rows a10-a11 (steps 6-8 of Algorithm 1,
// P:629-634) as one fused kernel: the second-stage local preconditioner M_L of
// P:606-612 read as tile-local 2x2-block ILU(0) of the interleaved S_ff^FS
// (DESIGN.md R-ilu: block Jacobi over fixed 16^3 tiles, natural order inside).
//
// On the 7-point pattern ILU(0) only updates diagonal blocks (a lower
// neighbour's upper neighbours are never neighbours of the row), so with
// D_K = U_KK^-1:
//   U_KK = A_KK - sum_{J<K, same tile} A_KJ D_J A_JK
//   forward   yhat_K = D_K (w_K - sum_{J<K} A_KJ yhat_J)
//   backward  x_K    = yhat_K - D_K sum_{J>K} A_KJ x_J
// Steps 6-8 without streaming the in-tile lower blocks twice (Eisenstat's trick for M = (D + L) D^-1 (D + U), D = U_KK,
// L / U = the in-tile lower / upper blocks, S^FS = L + S_KK + U + C with C the couplings that leave the tile):
//   M^-1 (y - S z) = (I + D^-1 U)^-1 [ (D + L)^-1 (y - E z - U z - C z) - z ],   E = S_KK - U_KK,
// so the residual phase reads the diagonal slot (holding E after the factorisation), the upper blocks and the few
// lower blocks that cross the tile boundary; L is streamed once, by the forward sweep.  The same operator as
// w = y - S z followed by the two sweeps, in a different association of the sums (TSP_ILU_PLAIN_RESID: the old form).
// B200 mapping: one CTA per tile; the tile is swept by x-LINES in (j+k)
// wavefront order (31 levels for 16^3 instead of 46 cell levels), each line
// held by a W-lane warp segment.  Inside a line the x-recurrence is affine,
//   yhat_i = M_i yhat_{i-1} + c_i,  M_i = -D_i A_{i,-x},  c_i = D_i (w_i - y/z terms),
// and is solved by a log2(W)-step segmented shuffle scan of (M, c) pairs (same
// ILU(0) operator, different association of the products).  Every global access
// is along x: coalesced.  The tile vector lives in shared memory.  The oracle
// runs textbook IKJ block ILU(0) cell by cell.
#include <algorithm>

#include "tsp_internal.cuh"

namespace tsp {

// slot order: 0 -z, 1 -y, 2 -x, 3 self, 4 +x, 5 +y, 6 +z
// nx, ny, nz: LOCAL slab grid (nz = owned cell planes); k0: first owned global plane
struct TileGeo {
    int nx, ny, nz, tx, ty, tz, ntx, nty, ntz, W, nlev, k0, nlo, nhi;
};

__device__ __forceinline__ int64_t vidx(const TileGeo &g, int64_t t, int lk, int lj, int s, int e, int li)
{
    return (((((t * g.tz + lk) * g.ty + lj) * 7 + s) * 4 + e) * g.W) + li;
}
__device__ __forceinline__ int64_t didx(const TileGeo &g, int64_t t, int lk, int lj, int e, int li)
{
    return ((((t * g.tz + lk) * g.ty + lj) * 4 + e) * g.W) + li;
}
__device__ __forceinline__ int sidx(const TileGeo &g, int lk, int lj, int li) { return ((lk * g.ty + lj) * g.tx + li) * 2; }

// line `slot` of wavefront level l (lj + lk = l, lk ascending; same order as the host's line table)
__device__ __forceinline__ bool line_at(const TileGeo &g, int l, int slot, int &lj, int &lk)
{
    const int lo = max(0, l - g.ty + 1), hi = min(l, g.tz - 1);
    lk = lo + slot; lj = l - lk;
    if (lk > hi) { lj = lk = 0; return false; }
    return true;
}

// fill the tile-ordered S_ff^FS = A_ff + diag(D_sp, D_pp) blocks (a1 folded in)
// (column ids are GLOBAL cell ids: neighbours in the ranks below/above keep their stencil slot)
__global__ void k_ilu_fill(TileGeo g, int nyg, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const double *__restrict__ fs, double *__restrict__ ival)
{
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)g.nx * g.ny * g.nz) return;
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / ((int64_t)g.nx * g.ny);
    const int TI = i / g.tx, TJ = j / g.ty, TK = k / g.tz;
    const int64_t t = ((int64_t)TK * g.nty + TJ) * g.ntx + TI;
    const int li = i - TI * g.tx, lj = j - TJ * g.ty, lk = k - TK * g.tz;
    for (int s = 0; s < 7; ++s)
        for (int e = 0; e < 4; ++e) ival[vidx(g, t, lk, lj, s, e, li)] = 0.0;
    const int dxs[7] = {0, 0, -1, 0, 1, 0, 0}, dys[7] = {0, -1, 0, 0, 0, 1, 0}, dzs[7] = {-1, 0, 0, 0, 0, 0, 1};
    for (int64_t q = rp[c]; q < rp[c + 1]; ++q) {
        const int64_t d = ci[q];
        const int di = (int)(d % g.nx) - i, dj = (int)((d / g.nx) % nyg) - j, dk = (int)(d / ((int64_t)g.nx * nyg)) - (k + g.k0);
        int s = -1;
        for (int u = 0; u < 7; ++u) if (dxs[u] == di && dys[u] == dj && dzs[u] == dk) s = u;
        if (s < 0) continue;
        for (int e = 0; e < 4; ++e) {
            double a = v[q * 4 + e];
            if (s == 3 && e == 1) a += fs[2 * c];      // A_sp^FS = A_sp + D_sp
            if (s == 3 && e == 3) a += fs[2 * c + 1];  // A_pp^FS = A_pp + D_pp
            ival[vidx(g, t, lk, lj, s, e, li)] = a;
        }
    }
}

__device__ __forceinline__ void ld2x2(const double *__restrict__ a, const TileGeo &g, int64_t t, int lk, int lj, int s, int li, double r[4])
{
#pragma unroll
    for (int e = 0; e < 4; ++e) r[e] = a[vidx(g, t, lk, lj, s, e, li)];
}
__device__ __forceinline__ void mm2(const double a[4], const double b[4], double r[4])
{
    r[0] = a[0] * b[0] + a[1] * b[2]; r[1] = a[0] * b[1] + a[1] * b[3];
    r[2] = a[2] * b[0] + a[3] * b[2]; r[3] = a[2] * b[1] + a[3] * b[3];
}

// a5: one thread per x-line, lines in (j+k) order, cells along x sequential
// plain = 1 (second stage = hybrid block GS): D_K = A_KK^-1 without the ILU Schur updates
// eis = 1: slot 3 of `ival` (the diagonal block S_KK, read by this cell only) is replaced by E_K = S_KK - U_KK
__global__ void k_ilu_factor(TileGeo g, const int32_t *__restrict__ lines, const int32_t *__restrict__ lvlptr,
                             double *__restrict__ ival, double *__restrict__ dinv, unsigned long long *__restrict__ npert,
                             int plain, int eis)
{
    const int64_t t = blockIdx.x;
    const int TI = t % g.ntx, TJ = (t / g.ntx) % g.nty, TK = t / ((int64_t)g.ntx * g.nty);
    for (int l = 0; l < g.nlev; ++l) {
        for (int idx = lvlptr[l] + threadIdx.x; idx < lvlptr[l + 1]; idx += blockDim.x) {
            const int lj = lines[idx] & 0xffff, lk = lines[idx] >> 16;
            if (TJ * g.ty + lj >= g.ny || TK * g.tz + lk >= g.nz) continue;
            const int len = min(g.tx, g.nx - TI * g.tx);
            for (int li = 0; li < len; ++li) {
                double U[4], S0[4];
                ld2x2(ival, g, t, lk, lj, 3, li, U);
                for (int e = 0; e < 4; ++e) S0[e] = U[e];
                for (int s = 0; s < (plain ? 0 : 3); ++s) {
                    int nlk = lk, nlj = lj, nli = li;
                    if (s == 0) nlk--; else if (s == 1) nlj--; else nli--;
                    if (nlk < 0 || nlj < 0 || nli < 0) continue;   // outside the tile: dropped (block Jacobi)
                    double A[4], B[4], D[4], L[4], T[4];
                    ld2x2(ival, g, t, lk, lj, s, li, A);          // A_KJ
                    ld2x2(ival, g, t, nlk, nlj, 6 - s, nli, B);   // A_JK
                    for (int e = 0; e < 4; ++e) D[e] = dinv[didx(g, t, nlk, nlj, e, nli)];
                    mm2(A, D, L); mm2(L, B, T);
                    for (int e = 0; e < 4; ++e) U[e] -= T[e];
                }
                const double sc = fmax(fmax(fabs(U[0]), fabs(U[1])), fmax(fabs(U[2]), fabs(U[3])));
                double det = U[0] * U[3] - U[1] * U[2];
                if (sc == 0.0 || fabs(det) <= 1e-14 * sc * sc) {   // singular pivot: perturb
                    const double dl = 1e-12 * (sc > 0.0 ? sc : 1.0);
                    U[0] += dl; U[3] += dl;
                    det = U[0] * U[3] - U[1] * U[2];
                    atomicAdd(npert, 1ULL);
                }
                dinv[didx(g, t, lk, lj, 0, li)] = U[3] / det;
                dinv[didx(g, t, lk, lj, 1, li)] = -U[1] / det;
                dinv[didx(g, t, lk, lj, 2, li)] = -U[2] / det;
                dinv[didx(g, t, lk, lj, 3, li)] = U[0] / det;
                if (eis)
                    for (int e = 0; e < 4; ++e) ival[vidx(g, t, lk, lj, 3, e, li)] = S0[e] - U[e];
            }
        }
        __syncthreads();
    }
}

// segmented affine scan over lanes of width W: x_i = M_i x_{i-dir} + c_i
template <bool FORWARD>
__device__ __forceinline__ void affine_scan(double M[4], double c[2], int lseg, int W)
{
    for (int off = 1; off < W; off <<= 1) {
        double Mp[4], cp[2];
#pragma unroll
        for (int e = 0; e < 4; ++e) Mp[e] = FORWARD ? __shfl_up_sync(0xffffffffu, M[e], off, W) : __shfl_down_sync(0xffffffffu, M[e], off, W);
#pragma unroll
        for (int e = 0; e < 2; ++e) cp[e] = FORWARD ? __shfl_up_sync(0xffffffffu, c[e], off, W) : __shfl_down_sync(0xffffffffu, c[e], off, W);
        const bool take = FORWARD ? (lseg >= off) : (lseg + off < W);
        if (take) {
            const double c0 = M[0] * cp[0] + M[1] * cp[1] + c[0];
            const double c1 = M[2] * cp[0] + M[3] * cp[1] + c[1];
            double R[4];
            mm2(M, Mp, R);
            c[0] = c0; c[1] = c1;
#pragma unroll
            for (int e = 0; e < 4; ++e) M[e] = R[e];
        }
    }
}

// register prefetch of a line's 3 off-diagonal blocks (forward: -y,-z,-x; backward: +y,+z,+x) and D_K
__device__ __forceinline__ void pf_load_dir(const double *__restrict__ ival, const double *__restrict__ dinv, const TileGeo &g,
                                            int64_t t, int lk, int lj, int li, bool ok, bool fwd, double P[16])
{
    if (!ok) return;
    const int s3[3] = {fwd ? 1 : 5, fwd ? 0 : 6, fwd ? 2 : 4};
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) P[4 * q + e] = ival[vidx(g, t, lk, lj, s3[q], e, li)];
#pragma unroll
    for (int e = 0; e < 4; ++e) P[12 + e] = dinv[didx(g, t, lk, lj, e, li)];
}

// phase-0 slot batch [S0, S1): loads first, then the accumulation in slot order (same rounding as slot by slot)
#define P0_BATCH(S0, S1)                                                                                         \
    {                                                                                                            \
        constexpr int dxs[7] = {0, 0, -1, 0, 1, 0, 0}, dys[7] = {0, -1, 0, 0, 0, 1, 0}, dzs[7] = {-1, 0, 0, 0, 0, 0, 1}; \
        double Z0[7], Z1[7], AA[7][4];                                                                           \
        bool use[7];                                                                                             \
        _Pragma("unroll") for (int s = S0; s < S1; ++s) {                                                        \
            const int ni = gi + dxs[s], nj = gj + dys[s], nk = gk + dzs[s];                                      \
            use[s] = ni >= 0 && nj >= 0 && ni < g.nx && nj < g.ny;                                               \
            if (EIS && ((s == 0 && lk > 0) || (s == 1 && lj > 0) || (s == 2 && li > 0))) use[s] = false;         \
            const double *p0 = zs, *p1 = zp;                                                                     \
            int64_t q = gc + dxs[s] + dys[s] * sy + dzs[s] * sz;                                                 \
            if (dzs[s] < 0 && nk < 0) {                                                                          \
                use[s] = use[s] && g.nlo; p0 = zs_gh; p1 = zp_gh; q = (int64_t)nj * g.nx + ni;                   \
            } else if (dzs[s] > 0 && nk >= g.nz) {                                                               \
                use[s] = use[s] && g.nhi; p0 = zs_gh + g.nlo; p1 = zp_gh + g.nlo; q = (int64_t)nj * g.nx + ni;   \
            }                                                                                                    \
            if (!use[s]) { p0 = zs; p1 = zp; q = gc; }                                                           \
            Z0[s] = __ldg(p0 + q); Z1[s] = __ldg(p1 + q);                                                        \
            /* a skipped slot re-reads the cell's diagonal slot (needed anyway, a cache hit): no branch */      \
            const int sl = (EIS && !use[s]) ? 3 : s;                                                             \
            _Pragma("unroll") for (int e = 0; e < 4; ++e) AA[s][e] = __ldg(ival + vidx(g, t, lk, lj, sl, e, li)); \
        }                                                                                                        \
        _Pragma("unroll") for (int s = S0; s < S1; ++s)                                                          \
            if (use[s]) {                                                                                        \
                r0 -= AA[s][0] * Z0[s] + AA[s][1] * Z1[s];                                                       \
                r1 -= AA[s][2] * Z0[s] + AA[s][3] * Z1[s];                                                       \
            }                                                                                                    \
    }
#define P0B 4   // slots per load batch (all 7 at once costs occupancy; measured on C5)

// steps 6-8 fused, pipelined form:
//  phase 0 (fully parallel, coalesced): w = y - S^FS z for every cell of the tile -> shared memory,
//  each cell's loads issued in two batches (phase 0 was latency bound with one round trip per slot)
//  forward / backward line wavefronts: per level only 4 blocks per cell (and z for step 8) are read
//  from global memory, prefetched into registers one level ahead and issued before the scan, so the
//  load overlaps the scan and the barrier.  3 CTAs per SM (the shared-memory limit) matter more than
//  a deeper prefetch: at 2 CTAs per SM the kernel is 1.5x slower (measured on C5).
// One line per W-lane segment; requires (lines per level) <= segments per CTA.
#ifdef TSP_ILU_TIMING
__device__ unsigned long long g_ilu_t[8192][4];
__device__ __forceinline__ unsigned long long gtimer() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
#define ILU_T(k) do { if (threadIdx.x == 0 && blockIdx.x < 8192) g_ilu_t[blockIdx.x][k] = gtimer(); } while (0)
#else
#define ILU_T(k) do { } while (0)
#endif
template <bool BGS, bool EIS>
__global__ void __launch_bounds__(256, 3) k_ilu_apply2(TileGeo g, const int32_t *__restrict__ lines, const int32_t *__restrict__ lvlptr,
                                                    const double *__restrict__ ival, const double *__restrict__ dinv,
                                                    const double *__restrict__ yf, const double *__restrict__ zs,
                                                    const double *__restrict__ zp, const double *__restrict__ zs_gh,
                                                    const double *__restrict__ zp_gh, double *__restrict__ zout)
{
    extern __shared__ double sm[];   // [lk][lj][li][2]: w, then yhat, then x
    const int64_t t = blockIdx.x;
    const int TI = t % g.ntx, TJ = (t / g.ntx) % g.nty, TK = t / ((int64_t)g.ntx * g.nty);
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const int W = g.W, lane = threadIdx.x & 31, lseg = lane & (W - 1);
    const int slot0 = (threadIdx.x >> 5) * (32 / W) + lane / W, nslots = (blockDim.x >> 5) * (32 / W);
    const int li = lseg, gi = TI * g.tx + li;
    const bool xin = li < g.tx && gi < g.nx;
    ILU_T(0);
    // ---------------- phase 0: w = y - S^FS z (step 6); EIS: y - E z - U z - C z
    for (int line = slot0; line < g.ty * g.tz; line += nslots) {
        const int lj = line % g.ty, lk = line / g.ty;
        const int gj = TJ * g.ty + lj, gk = TK * g.tz + lk;
        if (!(xin && gj < g.ny && gk < g.nz)) continue;
        const int64_t gc = gi + sy * gj + sz * gk;
        double r0 = yf[2 * gc], r1 = yf[2 * gc + 1];
        // all loads of a batch of slots are issued before the first use (branch-free addressing: absent
        // neighbours read a dummy and are masked), so a cell costs P0B round trips instead of 7
        P0_BATCH(0, P0B)
        P0_BATCH(P0B, 7)
        sm[sidx(g, lk, lj, li)] = r0;
        sm[sidx(g, lk, lj, li) + 1] = r1;
    }
    // ---------------- forward
    double P[16], zn0 = 0, zn1 = 0;   // zn: z at the backward sweep's next cell (step 8)
    {
        int lj, lk;
        const bool lv = line_at(g, 0, slot0, lj, lk);
        pf_load_dir(ival, dinv, g, t, lk, lj, li, lv && xin && TJ * g.ty + lj < g.ny && TK * g.tz + lk < g.nz, true, P);
    }
    __syncthreads();
    ILU_T(1);
    for (int l = 0; l < g.nlev; ++l) {
        int lj, lk;
        const bool lv = line_at(g, l, slot0, lj, lk);
        const bool ok = lv && xin && TJ * g.ty + lj < g.ny && TK * g.tz + lk < g.nz;
        double M[4] = {0, 0, 0, 0}, c[2] = {0, 0};
        if (ok) {
            double r0 = sm[sidx(g, lk, lj, li)], r1 = sm[sidx(g, lk, lj, li) + 1];
            if (lj > 0) {
                const double y0 = sm[sidx(g, lk, lj - 1, li)], y1 = sm[sidx(g, lk, lj - 1, li) + 1];
                r0 -= P[0] * y0 + P[1] * y1; r1 -= P[2] * y0 + P[3] * y1;
            }
            if (lk > 0) {
                const double y0 = sm[sidx(g, lk - 1, lj, li)], y1 = sm[sidx(g, lk - 1, lj, li) + 1];
                r0 -= P[4] * y0 + P[5] * y1; r1 -= P[6] * y0 + P[7] * y1;
            }
            const double *D = P + 12;
            c[0] = D[0] * r0 + D[1] * r1;
            c[1] = D[2] * r0 + D[3] * r1;
            if (li > 0) {
                double T[4]; mm2(D, P + 8, T);
                M[0] = -T[0]; M[1] = -T[1]; M[2] = -T[2]; M[3] = -T[3];
            }
        }
        // prefetch the next level's blocks (or the backward sweep's first level) while the scan runs
        {
            const int ln = l + 1 < g.nlev ? l + 1 : g.nlev - 1;
            int ljn, lkn;
            const bool lvn = line_at(g, ln, slot0, ljn, lkn);
            const bool okn = lvn && xin && TJ * g.ty + ljn < g.ny && TK * g.tz + lkn < g.nz && (!BGS || l + 1 < g.nlev);
            pf_load_dir(ival, dinv, g, t, lkn, ljn, li, okn, l + 1 < g.nlev, P);
            if (!BGS && l + 1 == g.nlev && okn) {
                const int64_t gcn = gi + sy * (TJ * g.ty + ljn) + sz * (TK * g.tz + lkn);
                zn0 = zs[gcn]; zn1 = zp[gcn];
            }
        }
        affine_scan<true>(M, c, lseg, W);
        if (ok) { sm[sidx(g, lk, lj, li)] = c[0]; sm[sidx(g, lk, lj, li) + 1] = c[1]; }
        if (BGS && ok) {                          // hybrid block GS: the forward sweep is the whole M_L (step 8)
            const int64_t gc = gi + sy * (TJ * g.ty + lj) + sz * (TK * g.tz + lk);
            zout[2 * gc] = EIS ? c[0] : zs[gc] + c[0];          // EIS: z + ((D + L)^-1 (..) - z)
            zout[2 * gc + 1] = EIS ? c[1] : zp[gc] + c[1];
        }
        __syncthreads();
    }
    ILU_T(2);
    // ---------------- backward (ILU only)
    if constexpr (!BGS)
    for (int l = g.nlev - 1; l >= 0; --l) {
        int lj, lk;
        const bool lv = line_at(g, l, slot0, lj, lk);
        const int gj = TJ * g.ty + lj, gk = TK * g.tz + lk;
        const bool ok = lv && xin && gj < g.ny && gk < g.nz;
        double M[4] = {0, 0, 0, 0}, c[2] = {0, 0};
        if (ok) {
            double t0 = 0, t1 = 0;
            if (lj + 1 < g.ty && gj + 1 < g.ny) {
                const double x0 = sm[sidx(g, lk, lj + 1, li)], x1 = sm[sidx(g, lk, lj + 1, li) + 1];
                t0 += P[0] * x0 + P[1] * x1; t1 += P[2] * x0 + P[3] * x1;
            }
            if (lk + 1 < g.tz && gk + 1 < g.nz) {
                const double x0 = sm[sidx(g, lk + 1, lj, li)], x1 = sm[sidx(g, lk + 1, lj, li) + 1];
                t0 += P[4] * x0 + P[5] * x1; t1 += P[6] * x0 + P[7] * x1;
            }
            const double *D = P + 12;
            c[0] = (EIS ? sm[sidx(g, lk, lj, li)] - zn0 : sm[sidx(g, lk, lj, li)]) - (D[0] * t0 + D[1] * t1);
            c[1] = (EIS ? sm[sidx(g, lk, lj, li) + 1] - zn1 : sm[sidx(g, lk, lj, li) + 1]) - (D[2] * t0 + D[3] * t1);
            if (li + 1 < g.tx && gi + 1 < g.nx) {
                double T[4]; mm2(D, P + 8, T);
                M[0] = -T[0]; M[1] = -T[1]; M[2] = -T[2]; M[3] = -T[3];
            }
        }
        const double zc0 = zn0, zc1 = zn1;
        if (l > 0) {
            int ljn, lkn;
            const bool lvn = line_at(g, l - 1, slot0, ljn, lkn);
            const bool okn = lvn && xin && TJ * g.ty + ljn < g.ny && TK * g.tz + lkn < g.nz;
            pf_load_dir(ival, dinv, g, t, lkn, ljn, li, okn, false, P);
            if (okn) {
                const int64_t gcn = gi + sy * (TJ * g.ty + ljn) + sz * (TK * g.tz + lkn);
                zn0 = zs[gcn]; zn1 = zp[gcn];
            }
        }
        affine_scan<false>(M, c, lseg, W);
        if (ok) {
            sm[sidx(g, lk, lj, li)] = c[0]; sm[sidx(g, lk, lj, li) + 1] = c[1];
            const int64_t gc = gi + sy * gj + sz * gk;
            zout[2 * gc] = zc0 + c[0];           // step 8
            zout[2 * gc + 1] = zc1 + c[1];
        }
        __syncthreads();
    }
    ILU_T(3);
}
#ifdef TSP_ILU_TIMING
extern "C" int tsp_dev_ilu_timers(unsigned long long *out, int n)
{
    return (int)cudaMemcpyFromSymbol(out, g_ilu_t, sizeof(unsigned long long) * 4 * (size_t)n);
}
#endif

static TileGeo geo(const Ctx &c)
{
    TileGeo g;
    g.nx = c.nx; g.ny = c.ny; g.nz = c.nz;   // local slab
    g.tx = std::min(c.o.tile_x, c.nx); g.ty = std::min(c.o.tile_y, c.ny); g.tz = std::min(c.o.tile_z, std::max(c.nz, 1));
    g.ntx = (c.nx + g.tx - 1) / g.tx; g.nty = (c.ny + g.ty - 1) / g.ty; g.ntz = (c.nz + g.tz - 1) / g.tz;
    g.W = 1; while (g.W < g.tx) g.W <<= 1;
    g.nlev = g.ty + g.tz - 1;
    g.k0 = c.k0;
    g.nlo = c.hf.nrecv[0]; g.nhi = c.hf.nrecv[1];
    return g;
}

void ilu_setup(Ctx &c, const double *)
{
    TileGeo g = geo(c);
    TSP_REQUIRE(g.tx <= 32 && g.ty <= 0xffff && g.tz <= 0x7fff, TSP_ERR_INVALID_ARG, "ILU tile_x must be <= 32");
    TSP_REQUIRE(std::min(g.ty, g.tz) <= 8 * (32 / g.W), TSP_ERR_INVALID_ARG, "ILU tile: too many lines per wavefront level");
    TSP_REQUIRE(c.nranks == 1 || (c.o.zblock % c.o.tile_z == 0 && c.o.tile_z <= c.o.zblock), TSP_ERR_INVALID_ARG,
                "multi-GPU: tile_z must divide zblock (tiles may not cross slabs)");
    if (c.ilu_tsize != g.tx * g.ty * g.tz) {
        std::vector<int32_t> lines, lvlptr;
        for (int l = 0; l < g.nlev; ++l) {
            lvlptr.push_back((int32_t)lines.size());
            for (int lk = 0; lk < g.tz; ++lk)
                for (int lj = 0; lj < g.ty; ++lj)
                    if (lj + lk == l) lines.push_back(lj | (lk << 16));
        }
        lvlptr.push_back((int32_t)lines.size());
        c.ilu_nlev = g.nlev; c.ilu_tsize = g.tx * g.ty * g.tz;
        c.ilu_cells.alloc(lines.size()); c.ilu_lvlptr.alloc(lvlptr.size());
        TSP_CUDA(cudaMemcpyAsync(c.ilu_cells, lines.data(), sizeof(int32_t) * lines.size(), cudaMemcpyHostToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(c.ilu_lvlptr, lvlptr.data(), sizeof(int32_t) * lvlptr.size(), cudaMemcpyHostToDevice, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
    }
    // per handle (the attribute is per device; tsp_setup runs on the handle's device)
    TSP_CUDA(cudaFuncSetAttribute(k_ilu_apply2<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    TSP_CUDA(cudaFuncSetAttribute(k_ilu_apply2<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    TSP_CUDA(cudaFuncSetAttribute(k_ilu_apply2<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    TSP_CUDA(cudaFuncSetAttribute(k_ilu_apply2<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    c.ilu_eis = getenv("TSP_ILU_PLAIN_RESID") == nullptr;       // read per setup: slot 3 then holds E = S_KK - U_KK
    c.ntx = g.ntx; c.nty = g.nty; c.ntz = g.ntz;
    c.ntiles = g.ntx * g.nty * g.ntz;
    const size_t per_tile = (size_t)g.tz * g.ty * g.W;
    c.ilu_val.alloc((size_t)c.ntiles * per_tile * 28);
    c.ilu_dinv.alloc((size_t)c.ntiles * per_tile * 4);
    c.ilu_val.zero(c.s);
    c.ilu_dinv.zero(c.s);
    if (c.Nc) k_ilu_fill<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(g, c.ny, c.ff.rp, c.ff.gci.p ? c.ff.gci.p : c.ff.ci.p, c.ff.v, c.fs_eff,
                                                             c.ilu_val);
    c.dcount.zero(c.s);
    k_ilu_factor<<<c.ntiles, 32, 0, c.s>>>(g, c.ilu_cells, c.ilu_lvlptr, c.ilu_val, c.ilu_dinv, c.dcount, c.o.second_stage == 1, c.ilu_eis);
    TSP_CUDA(cudaGetLastError());
    unsigned long long np = 0;
    TSP_CUDA(cudaMemcpyAsync(&np, c.dcount, sizeof(np), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.perturbed += (int64_t)np;
    c.launches += 2;
}

void ilu_apply_fused(Ctx &c, const double *yf, const double *zs, const double *zp, double *zf_out)
{
    TileGeo g = geo(c);
    const size_t smem = sizeof(double) * 2 * (size_t)g.tx * g.ty * g.tz;
    TSP_REQUIRE(smem <= 227 * 1024, TSP_ERR_INVALID_ARG, "ILU tile too large for shared memory");
    const double *zs_gh = c.gh_f2.p, *zp_gh = c.gh_f2.p ? c.gh_f2.p + c.hf.nghost() : nullptr;
    prof_begin(c, PK_ILU);
    if (c.ntiles)
        (c.o.second_stage == 1 ? (c.ilu_eis ? k_ilu_apply2<true, true> : k_ilu_apply2<true, false>)
                               : (c.ilu_eis ? k_ilu_apply2<false, true> : k_ilu_apply2<false, false>))<<<c.ntiles, 256, smem, c.s>>>(
            g, c.ilu_cells, c.ilu_lvlptr, c.ilu_val, c.ilu_dinv, yf, zs, zp, zs_gh, zp_gh, zf_out);
    prof_end(c, PK_ILU, (28.0 * 8 + 32 + 16 + 16 + 16) * c.Nc);
    c.launches += 1;
    TSP_CUDA(cudaGetLastError());
}

}  // namespace tsp

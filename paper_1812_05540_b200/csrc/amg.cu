// amg.cu -- row a4 (AMG setup on the GPU) and rows a6/a9 (V-cycles).
//
// Method (DESIGN.md R-amg, R-strength, R-mis2, R-agg, R-prolong, R-rap,
// R-cycle): smoothed aggregation with MIS(2) aggregates,
// Galerkin R = P^T, one V(1,1) l1-Jacobi cycle, dense coarsest solve.  The
// setup is bit-identical to the oracle: every floating-point sum is a left fold
// in the oracle's canonical order with IEEE round-to-nearest intrinsics
// (__dadd_rn/__dmul_rn/__ddiv_rn, no FMA contraction) and no atomics on values.
// Apply kernels are free (FMA, any order).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <ctime>

#include <climits>

#include "tsp_internal.cuh"

namespace tsp {

// lanes per row from the GLOBAL mean row length (0: sliced-ELL thread per row); measured at C5:
// 8/16 lanes beat a full warp by 20-35 % on the pressure levels 1-2 and the level-0 restriction
// A level too small to fill the GPU even at a full warp per row (rows x 32 <= the SMs' resident threads) is
// latency-bound, not bandwidth-bound: there every row gets 32 lanes, which shortens each lane's chain of
// dependent loads (row pointer -> column -> gathered x) to one or two steps.  Measured at C5: the restrictions
// into mechanics levels 4-6 took 7-28 us with a thread per row (sliced ELL, 8-20 dependent steps).
static int lanes_for(int64_t nnz, int64_t rows, int sms)
{
    if (rows <= 0) return 0;
    if (rows * 32 <= (int64_t)sms * 2048) return 32;
    if (nnz < 12 * rows) return 0;
    return nnz < 40 * rows ? 8 : nnz < 96 * rows ? 16 : 32;
}
// test knob TSP_FORCE_LANES=0|8|16|32: every level uses that vector-CSR variant (parity coverage of each
// lanes_for choice on small grids; the setup products are unaffected, apply sums change order only)
static int lanes_forced(int lanes)
{
    const char *e = getenv("TSP_FORCE_LANES");
    return e ? atoi(e) : lanes;
}
static int lanes_idx(int lanes) { return lanes == 0 ? 0 : lanes == 8 ? 1 : lanes == 16 ? 2 : 3; }


__device__ __forceinline__ uint32_t fmix32(uint32_t x)
{
    x ^= x >> 16; x *= 0x85ebca6bU; x ^= x >> 13; x *= 0xc2b2ae35U; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint64_t prio(int i) { return ((uint64_t)fmix32((uint32_t)i) << 32) | (uint64_t)(uint32_t)i; }

// ------------------------------------------------------------------ l1 norms: d_i = fold_j |a_ij|
// thread per (row, component): the fold of each component stays serial in q order
__global__ void k_l1(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                     double *dl1, double *dinv)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * nc) return;
    const int i = (int)(t / nc), c = (int)(t % nc);
    double s = 0.0, aii = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        s = __dadd_rn(s, fabs(v[q * nc + c]));
        if (ci[q] == i) aii = v[q * nc + c];
    }
    if (aii < 0.0) s = -s;                                 // R-l1: the sign of the diagonal
    dl1[t] = s;
    dinv[t] = s != 0.0 ? 1.0 / s : 0.0;
}

__device__ __forceinline__ double meas(const double *__restrict__ v, int64_t q, int nc)
{
    double s = 0.0;
    for (int c = 0; c < nc; ++c) s = __dadd_rn(s, fabs(v[q * nc + c]));
    return s;
}

// ------------------------------------------------------------------ strength (R-strength)
// 8 lanes per row: the row max is order independent (exact), each entry's flag is its own
constexpr int kStrG = 8;
__global__ void k_strength(int n, int nc, int nown, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const int32_t *__restrict__ zb, double theta, uint8_t *S)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int i = (int)(t / kStrG), sub = (int)(t % kStrG);
    const bool ok = i < n;
    const int64_t q0 = ok ? rp[i] : 0, q1 = ok ? rp[i + 1] : 0;
    double m = 0.0;
    for (int64_t q = q0 + sub; q < q1; q += kStrG)
        if (ci[q] != i) { double u = meas(v, q, nc); if (u > m) m = u; }
#pragma unroll
    for (int o = kStrG / 2; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o, kStrG));
    if (!ok) return;
    const double thr = __dmul_rn(theta, m);
    const int zi = zb[i];
    for (int64_t q = q0 + sub; q < q1; q += kStrG) {
        const int j = ci[q];
        // columns of other ranks (j >= nown) lie in other z-blocks by construction
        S[q] = (j != i && m > 0.0 && j < nown && zi == zb[j] && meas(v, q, nc) >= thr) ? 1 : 0;
    }
}

// kStrG lanes per row, one entry (and its transpose search) per lane at a time
__global__ void k_symm(int n, int nown, int linear, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                       const uint8_t *__restrict__ S, uint8_t *E, int *err)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int i = (int)(t / kStrG), sub = (int)(t % kStrG);
    if (i >= n) return;
    for (int64_t q = rp[i] + sub; q < rp[i + 1]; q += kStrG) {
        int j = ci[q];
        if (j == i || j >= nown) { E[q] = 0; continue; }
        int64_t lo = rp[j], hi = rp[j + 1] - 1, qt = -1;
        if (linear) {   // distributed level: local ids in a row are not monotone (ghosts first/last)
            for (int64_t u = lo; u <= hi; ++u) if (ci[u] == i) { qt = u; break; }
            lo = 1; hi = 0;
        }
        while (lo <= hi) {
            int64_t mid = (lo + hi) >> 1;
            int cm = ci[mid];
            if (cm == i) { qt = mid; break; }
            if (cm < i) lo = mid + 1; else hi = mid - 1;
        }
        if (qt < 0) { *err = 1; E[q] = 0; continue; }
        E[q] = (S[q] || S[qt]) ? 1 : 0;
    }
}

// ------------------------------------------------------------------ MIS(2) rounds (R-mis2)
enum { ST_ISO = -1, ST_UND = 0, ST_ROOT = 1, ST_OUT = 2 };

__global__ void k_mis_init(int n, const int32_t *__restrict__ rp, const uint8_t *__restrict__ E, int8_t *st)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = 0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) d |= E[q];
    st[i] = d ? ST_UND : ST_ISO;
}
__global__ void k_mis_t1(int n, int off, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                         const int8_t *__restrict__ st, uint64_t *t1)
{
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    uint64_t m = st[x] == ST_UND ? prio(off + x) + 1 : 0;   // priorities of GLOBAL row ids
    for (int64_t q = rp[x]; q < rp[x + 1]; ++q)
        if (E[q]) { int u = ci[q]; if (st[u] == ST_UND) { uint64_t p = prio(off + u) + 1; if (p > m) m = p; } }
    t1[x] = m;
}
__global__ void k_mis_root(int n, int off, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                           const int8_t *__restrict__ st, const uint64_t *__restrict__ t1, uint8_t *newr)
{
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint8_t r = 0;
    if (st[v] == ST_UND) {
        uint64_t m = t1[v];
        for (int64_t q = rp[v]; q < rp[v + 1]; ++q) if (E[q]) { uint64_t t = t1[ci[q]]; if (t > m) m = t; }
        r = (m == prio(off + v) + 1);
    }
    newr[v] = r;
}
__global__ void k_mis_near(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                           const uint8_t *__restrict__ newr, int8_t *st, uint8_t *near1)
{
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    uint8_t h = newr[x];
    for (int64_t q = rp[x]; q < rp[x + 1] && !h; ++q) if (E[q] && newr[ci[q]]) h = 1;
    near1[x] = h;
    if (newr[x]) st[x] = ST_ROOT;
}
__global__ void k_mis_out(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                          const uint8_t *__restrict__ near1, int8_t *st, unsigned long long *undecided)
{
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    if (st[v] != ST_UND) return;
    uint8_t h = near1[v];
    for (int64_t q = rp[v]; q < rp[v + 1] && !h; ++q) if (E[q] && near1[ci[q]]) h = 1;
    if (h) st[v] = ST_OUT;
    else atomicAdd(undecided, 1ULL);
}

// ------------------------------------------------------------------ aggregates (R-agg)
__global__ void k_rootflag(int n, const int8_t *__restrict__ st, int32_t *flag)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = st[i] == ST_ROOT;
}
__global__ void k_phase1(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                         const int8_t *__restrict__ st, const int32_t *__restrict__ rid, const int32_t *__restrict__ zb,
                         int32_t *agg, int32_t *zbc)
{
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || st[r] != ST_ROOT) return;
    int a = rid[r];
    agg[r] = a;
    zbc[a] = zb[r];
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q) if (E[q]) agg[ci[q]] = a;
}
__global__ void k_phase2(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                         const uint8_t *__restrict__ E, const int8_t *__restrict__ st, const int32_t *__restrict__ ph1, int32_t *agg)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (st[i] == ST_ISO || ph1[i] >= 0) { agg[i] = ph1[i]; return; }
    int best = -1; double bw = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        if (!E[q]) continue;
        int a = ph1[ci[q]];
        if (a < 0) continue;
        double w = meas(v, q, nc);
        if (best < 0 || w > bw || (w == bw && a < best)) { best = a; bw = w; }
    }
    agg[i] = best;
}

// ------------------------------------------------------------------ smoothed prolongator (R-prolong)
// d_i = a_ii + fold_{weak j} a_ij ; ratio_i = fold_j |a^F_ij| / |d_i|
// thread per (row, component), each fold serial in q order; rho reduced per block first (measured at C5: 2-4x
// faster than a warp per row with the entries broadcast by shuffles)
__global__ void __launch_bounds__(256) k_pdiag(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                 const double *__restrict__ v, const uint8_t *__restrict__ E, double *d,
                                                 unsigned long long *rho_bits)
{
    __shared__ unsigned long long bm[3];
    if (threadIdx.x < 3) bm[threadIdx.x] = 0ULL;
    __syncthreads();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n * nc) {
        const int i = (int)(t / nc), c = (int)(t % nc);
        const int64_t q0 = rp[i], q1 = rp[i + 1];
        int64_t qd = -1;
        for (int64_t q = q0; q < q1; ++q) if (ci[q] == i) { qd = q; break; }
        double di = qd >= 0 ? v[qd * nc + c] : 0.0;
        for (int64_t q = q0; q < q1; ++q)
            if (ci[q] != i && !E[q]) di = __dadd_rn(di, v[q * nc + c]);
        d[(int64_t)i * nc + c] = di;
        if (di != 0.0) {
            double s = 0.0;
            for (int64_t q = q0; q < q1; ++q) {
                const double a = (ci[q] == i) ? di : (E[q] ? v[q * nc + c] : 0.0);
                s = __dadd_rn(s, fabs(a));
            }
            const double r = __ddiv_rn(s, fabs(di));
            atomicMax(&bm[c], (unsigned long long)__double_as_longlong(r));   // r >= 0: bit order = value order
        }
    }
    __syncthreads();
    if (threadIdx.x < nc && bm[threadIdx.x]) atomicMax(rho_bits + threadIdx.x, bm[threadIdx.x]);
}
struct Omega { double w[3]; };
#define PMAX 512
__device__ int collect_aggs(int i, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                            const int32_t *__restrict__ agg, int32_t *tmp, int *overflow)
{
    int cnt = 0;
    if (agg[i] < 0) return 0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        int j = ci[q];
        if ((j == i || E[q]) && agg[j] >= 0) {
            int a = agg[j];
            bool dup = false;
            for (int t = 0; t < cnt; ++t) if (tmp[t] == a) { dup = true; break; }
            if (dup) continue;
            if (cnt >= PMAX) { *overflow = 1; break; }
            int t = cnt++;
            while (t > 0 && tmp[t - 1] > a) { tmp[t] = tmp[t - 1]; --t; }   // insertion sort
            tmp[t] = a;
        }
    }
    return cnt;
}
// one (row, component): the aggregates of the row (every component's thread collects them; component 0
// writes the column ids), then one pass over the row -- each sum is still the fold over the row in q order
// restricted to its aggregate (R-prolong)
__device__ void pfill_row(int i, int c, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                          const double *__restrict__ v, const uint8_t *__restrict__ E, const int32_t *__restrict__ agg,
                          const double *__restrict__ d, const Omega &om, const int32_t *__restrict__ prp, int32_t *pci,
                          double *pv, int *overflow)
{
    int32_t tmp[PMAX];
    double s[PMAX];
    const int cnt = collect_aggs(i, rp, ci, E, agg, tmp, overflow);
    const int64_t o = prp[i];
    if (c == 0) for (int t = 0; t < cnt; ++t) pci[o + t] = tmp[t];
    if (!cnt) return;
    const int ai = agg[i];
    const double di = d[(int64_t)i * nc + c];
    const double w = (di != 0.0) ? __ddiv_rn(om.w[c], di) : 0.0;
    for (int t = 0; t < cnt; ++t) s[t] = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        const int j = ci[q];
        if (!((j == i) || E[q])) continue;
        const int J = agg[j];
        if (J < 0) continue;
        int t = 0;
        while (t < cnt && tmp[t] != J) ++t;
        if (t == cnt) continue;   // only after an overflow (the row is then rejected)
        const double a = (j == i) ? di : v[q * nc + c];
        s[t] = __dadd_rn(s[t], a);
    }
    for (int t = 0; t < cnt; ++t) {
        const double delta = (tmp[t] == ai) ? 1.0 : 0.0;
        pv[(o + t) * nc + c] = __dsub_rn(delta, __dmul_rn(w, s[t]));
    }
}

// thread per row (a warp-per-row variant with the folds kept in q order was measured slower at C5)
__global__ void k_pcount(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const uint8_t *__restrict__ E,
                         const int32_t *__restrict__ agg, int32_t *cnt, int *overflow)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t tmp[PMAX];
    cnt[i] = collect_aggs(i, rp, ci, E, agg, tmp, overflow);
}
__global__ void k_pfill(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                        const uint8_t *__restrict__ E, const int32_t *__restrict__ agg, const double *__restrict__ d, Omega om,
                        const int32_t *__restrict__ prp, int32_t *pci, double *pv, int *overflow)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n * nc) pfill_row((int)(t / nc), (int)(t % nc), nc, rp, ci, v, E, agg, d, om, prp, pci, pv, overflow);
}

// ------------------------------------------------------------------ transpose helpers
__global__ void k_expand_rows(int n, const int32_t *__restrict__ rp, int32_t *row)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) row[q] = i;
}
__global__ void k_iota(int64_t n, int32_t *a)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}
__global__ void k_col_count(int64_t nnz, const int32_t *__restrict__ ci, int32_t *cnt)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) atomicAdd(cnt + ci[q], 1);
}
__global__ void k_transpose_fill(int64_t nnz, int nc, const int32_t *__restrict__ perm, const int32_t *__restrict__ row,
                                 const double *__restrict__ pv, int32_t *rci, double *rv)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nnz) return;
    int q = perm[t];
    rci[t] = row[q];
    for (int c = 0; c < nc; ++c) rv[t * nc + c] = pv[(int64_t)q * nc + c];
}

// ------------------------------------------------------------------ deterministic SpGEMM (R-rap)
// C = X Y; C_ik = fold over X's row i (ascending) of x_ij * y_jk, starting at 0.0.
// One warp per row; the X row is walked sequentially (canonical order), lanes
// split Y's row j (unique columns, so no two lanes touch one accumulator).
// Latency: the X row's (j, x_ij, Y-row bounds) are fetched lane-parallel 32 entries at
// a time and broadcast by shuffles, and the first 32 entries of the next Y row are
// loaded while the current one is merged into the warp's shared-memory hash table.
template <int NC>
__device__ __forceinline__ void spg_insert(int k, const double *yq, const double *x, int *keys, double *acc, int HS, bool fill,
                                           int &nfull)
{
    unsigned h = ((unsigned)k * 2654435761u) & (HS - 1);
    int probes = 0;
    for (;;) {
        const int old = atomicCAS(&keys[h], -1, k);
        if (old == -1) {
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[h * NC + c] = 0.0;
            break;
        }
        if (old == k) break;
        h = (h + 1) & (HS - 1);
        if (++probes >= HS) { nfull = 1; return; }
    }
    if (fill) {
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[h * NC + c] = __dadd_rn(acc[h * NC + c], __dmul_rn(x[c], yq[c]));
    }
}

// G lanes per row (G | 32): a group walks its X row in order, its lanes split each Y row.
// G < 32 when Y's rows are short (A P: P has ~4 entries per row), so several rows share a warp.
template <int NC, int G, int HS>
__global__ void k_spgemm(int n, const int32_t *__restrict__ xrp, const int32_t *__restrict__ xci, const double *__restrict__ xv,
                         const int32_t *__restrict__ yrp, const int32_t *__restrict__ yci, const double *__restrict__ yv,
                         int fill, int32_t *cnt, const int32_t *__restrict__ crp, int32_t *cci, double *cv, int *overflow)
{
    extern __shared__ unsigned char smraw[];
    constexpr int GPW = 32 / G;                     // groups (rows) per warp
    const int lane = threadIdx.x & 31, sub = lane & (G - 1), gid = lane / G;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << (gid * G));
    const int ngroups = blockDim.x / G, grp = threadIdx.x / G;
    // per-group tables padded by one word / one double so the groups of a warp hit different banks
    int *keys = (int *)smraw + grp * (HS + 1);
    double *acc = (double *)(smraw + (((size_t)ngroups * (HS + 1) * sizeof(int) + 15) & ~(size_t)15)) + (size_t)grp * (HS * NC + 1);
    (void)GPW;
    for (int i = blockIdx.x * ngroups + grp; i < n; i += gridDim.x * ngroups) {
        for (int t = sub; t < HS; t += G) keys[t] = -1;
        __syncwarp(gmask);
        int nfull = 0;
        const int q0 = xrp[i], q1 = xrp[i + 1];
        for (int qb = q0; qb < q1 && !nfull; qb += G) {
            const int nb = min(G, q1 - qb);
            int ysl = 0, yel = 0;
            double xl[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) xl[c] = 0.0;
            if (sub < nb) {
                const int j = xci[qb + sub];
                ysl = yrp[j]; yel = yrp[j + 1];
                if (fill)
#pragma unroll
                    for (int c = 0; c < NC; ++c) xl[c] = xv[(int64_t)(qb + sub) * NC + c];
            }
            // first chunk of Y row t (prefetched one step ahead)
            int ys = __shfl_sync(gmask, ysl, 0, G), ye = __shfl_sync(gmask, yel, 0, G);
            int ck = -1;
            double cy[NC];
            if (ys + sub < ye) {
                ck = yci[ys + sub];
                if (fill)
#pragma unroll
                    for (int c = 0; c < NC; ++c) cy[c] = yv[(int64_t)(ys + sub) * NC + c];
            }
            for (int t = 0; t < nb; ++t) {
                double x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) x[c] = __shfl_sync(gmask, xl[c], t, G);
                const int cys = ys, cye = ye;
                int nk = -1;
                double ny[NC];
                if (t + 1 < nb) {
                    ys = __shfl_sync(gmask, ysl, t + 1, G); ye = __shfl_sync(gmask, yel, t + 1, G);
                    if (ys + sub < ye) {
                        nk = yci[ys + sub];
                        if (fill)
#pragma unroll
                            for (int c = 0; c < NC; ++c) ny[c] = yv[(int64_t)(ys + sub) * NC + c];
                    }
                }
                if (ck >= 0) spg_insert<NC>(ck, cy, x, keys, acc, HS, fill, nfull);
                for (int p = cys + G + sub; p < cye && !nfull; p += G) {
                    double yq[NC];
                    if (fill)
#pragma unroll
                        for (int c = 0; c < NC; ++c) yq[c] = yv[(int64_t)p * NC + c];
                    spg_insert<NC>(yci[p], yq, x, keys, acc, HS, fill, nfull);
                }
                __syncwarp(gmask);
                ck = nk;
#pragma unroll
                for (int c = 0; c < NC; ++c) cy[c] = ny[c];
            }
            nfull = __any_sync(gmask, nfull);
        }
        // count occupied slots
        int mine = 0;
        for (int t = sub; t < HS; t += G) mine += keys[t] >= 0;
#pragma unroll
        for (int o = G / 2; o; o >>= 1) mine += __shfl_xor_sync(gmask, mine, o, G);
        if (__any_sync(gmask, nfull) || mine > (HS * 3) / 4) { if (sub == 0) *overflow = 1; }
        if (!fill) {
            if (sub == 0) cnt[i] = mine;
        } else {
            const int64_t base = crp[i];
            for (int t = sub; t < HS; t += G) {
                int k = keys[t];
                if (k < 0) continue;
                int rank = 0;
                for (int u = 0; u < HS; ++u) { int kk = keys[u]; rank += (kk >= 0 && kk < k); }
                cci[base + rank] = k;
#pragma unroll
                for (int c = 0; c < NC; ++c) cv[(base + rank) * NC + c] = acc[t * NC + c];
            }
        }
        __syncwarp(gmask);
    }
}

// ------------------------------------------------------------------ coarsest dense LU -> inverse (one CTA per component)
// LU with partial pivoting, pivot = first maximal |a| in the column (lowest row on ties),
// zero pivot -> 1e-12 * max|A| (R-coarse).  Then inverse columns by forward/back substitution.
__global__ void k_dense_inv(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                            double *work, int *piv, double *inv, unsigned long long *npert)
{
    const int c = blockIdx.x;
    double *a = work + (size_t)c * n * n;
    int *pv = piv + (size_t)c * n;
    double *out = inv + (size_t)c * n * n;
    for (int64_t t = threadIdx.x; t < (int64_t)n * n; t += blockDim.x) a[t] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q) a[(int64_t)i * n + ci[q]] = v[q * nc + c];
    __syncthreads();
    __shared__ double s_scale;
    __shared__ int s_p;
    if (threadIdx.x == 0) {
        double sc = 0.0;
        for (int64_t t = 0; t < (int64_t)n * n; ++t) sc = fmax(sc, fabs(a[t]));
        s_scale = sc == 0.0 ? 1.0 : sc;
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (threadIdx.x == 0) {
            int p = k; double best = fabs(a[(int64_t)k * n + k]);
            for (int i = k + 1; i < n; ++i) { double t = fabs(a[(int64_t)i * n + k]); if (t > best) { best = t; p = i; } }
            s_p = p; pv[k] = p;
        }
        __syncthreads();
        int p = s_p;
        if (p != k)
            for (int j = threadIdx.x; j < n; j += blockDim.x) { double t = a[(int64_t)k * n + j]; a[(int64_t)k * n + j] = a[(int64_t)p * n + j]; a[(int64_t)p * n + j] = t; }
        __syncthreads();
        if (threadIdx.x == 0 && a[(int64_t)k * n + k] == 0.0) { a[(int64_t)k * n + k] = 1e-12 * s_scale; atomicAdd(npert, 1ULL); }
        __syncthreads();
        double dkk = a[(int64_t)k * n + k];
        for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) a[(int64_t)i * n + k] /= dkk;
        __syncthreads();
        for (int64_t t = threadIdx.x; t < (int64_t)(n - k - 1) * (n - k - 1); t += blockDim.x) {
            int i = k + 1 + (int)(t / (n - k - 1)), j = k + 1 + (int)(t % (n - k - 1));
            a[(int64_t)i * n + j] -= a[(int64_t)i * n + k] * a[(int64_t)k * n + j];
        }
        __syncthreads();
    }
    // inverse: column e of A^-1 solves A x = e_e (row swaps applied in order)
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        double *x = out + (size_t)e;   // column e, stride n: out[i*n + e]
        for (int i = 0; i < n; ++i) x[(size_t)i * n] = (i == e) ? 1.0 : 0.0;
        for (int k = 0; k < n; ++k) if (pv[k] != k) { double t = x[(size_t)k * n]; x[(size_t)k * n] = x[(size_t)pv[k] * n]; x[(size_t)pv[k] * n] = t; }
        for (int i = 0; i < n; ++i) { double s = x[(size_t)i * n]; for (int j = 0; j < i; ++j) s -= a[(int64_t)i * n + j] * x[(size_t)j * n]; x[(size_t)i * n] = s; }
        for (int i = n - 1; i >= 0; --i) { double s = x[(size_t)i * n]; for (int j = i + 1; j < n; ++j) s -= a[(int64_t)i * n + j] * x[(size_t)j * n]; x[(size_t)i * n] = s / a[(int64_t)i * n + i]; }
    }
}

// ------------------------------------------------------------------ host helpers
template <class T>
static void exclusive_scan(Ctx &c, const T *in, T *out, int64_t n)
{
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, c.s);
    void *t = scratch(c, tb);
    cub::DeviceScan::ExclusiveSum(t, tb, in, out, n, c.s);
}
template <class T>
static T d2h1(Ctx &c, const T *p)
{
    T v;
    TSP_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    return v;
}

// rp from per-row counts (n+1 entries, counts in [0,n), last = 0)
static int64_t rowptr_from_counts(Ctx &c, DBuf<int32_t> &cnt, DBuf<int32_t> &rp, int n)
{
    TSP_CUDA(cudaMemsetAsync(cnt.p + n, 0, sizeof(int32_t), c.s));
    rp.alloc(n + 1);
    exclusive_scan<int32_t>(c, cnt, rp, n + 1);
    return d2h1(c, rp.p + n);
}

// one k_spgemm launch with (value sets, lanes per row, hash slots) chosen at run time
static void spgemm_launch(Ctx &c, int ncv, int G, int HS, int fill, const Csr &X, const Csr &Y, int32_t *cnt, Csr &C, int *ovf)
{
    const int threads = HS >= 4096 ? 32 : HS >= 512 ? 128 : 256;
    const int groups = threads / G;
    const size_t smem = (((size_t)groups * (HS + 1) * sizeof(int) + 15) & ~(size_t)15) + (size_t)groups * (HS * ncv + 1) * sizeof(double);
    const int grid = std::max(1, std::min((int)((X.n + groups - 1) / groups), c.sm_count * 64));
#define SPG(NCV, GV_, HSV)                                                                                                \
    do {                                                                                                                  \
        cudaFuncSetAttribute(k_spgemm<NCV, GV_, HSV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
        k_spgemm<NCV, GV_, HSV><<<grid, threads, smem, c.s>>>(X.n, X.rp, X.ci, X.v, Y.rp, Y.ci, Y.v, fill, cnt, C.rp,     \
                                                              C.ci, C.v, ovf);                                            \
    } while (0)
#define SPG_NC(NCV)                                                                                                       \
    do {                                                                                                                  \
        if (G == 4 && HS == 64) SPG(NCV, 4, 64);                                                                          \
        else if (G == 8 && HS == 64) SPG(NCV, 8, 64);                                                                     \
        else if (HS == 128) SPG(NCV, 32, 128);                                                                            \
        else if (HS == 512) SPG(NCV, 32, 512);                                                                            \
        else SPG(NCV, 32, 4096);                                                                                          \
    } while (0)
    if (ncv == 1) SPG_NC(1);
    else SPG_NC(3);
#undef SPG_NC
#undef SPG
    TSP_CUDA(cudaGetLastError());
    c.launches++;
    c.variants[TSP_VAR_SPGEMM_HS64 + (HS == 64 ? 0 : HS == 128 ? 1 : HS == 512 ? 2 : 3)]++;
    c.variants[TSP_VAR_SPGEMM_G4 + (G == 4 ? 0 : G == 8 ? 1 : 2)]++;
}

static void spgemm(Ctx &c, const Csr &X, const Csr &Y, Csr &C, int nc)
{
    C.n = X.n; C.m = Y.m; C.nc = nc;
    DBuf<int32_t> cnt; cnt.alloc(X.n + 1);
    DBuf<int> ovf; ovf.alloc(1);
    // Lanes per row from Y's mean row length (8 for the prolongators, whose rows are ~4 long -- 4 for the
    // scalar 7-point A P; 32 otherwise);
    // attempts grow the per-row hash table on overflow.  The symbolic pass (counts) touches no values and
    // runs the scalar kernel.  Measured at C5: 8 lanes beat 32 for the prolongator products (mechanics level-0
    // A P: 73.6 -> 36.2 ms for both passes); for the scalar 7-point A P 4 lanes beat 8 (pressure level 0:
    // 10.8 -> 9.7 ms).
    const double ymean = Y.n ? (double)Y.nnz / Y.n : 0.0, xmean = X.n ? (double)X.nnz / X.n : 0.0;
    const int G0 = ymean > 8.0 ? 32 : (nc == 1 && xmean <= 8.0 && ymean <= 4.0) ? 4 : 8;   // 4: 7-point A P
    // test knob TSP_SPGEMM_MIN_SLOTS=512|4096: start at the overflow tables (bitwise the same products; lets
    // the parity tests cover the paths the full-size configs take)
    const char *ms = getenv("TSP_SPGEMM_MIN_SLOTS");
    const int first = !ms ? 0 : atoi(ms) >= 4096 ? 2 : atoi(ms) >= 512 ? 1 : 0;
    for (int attempt = first; attempt < 3; ++attempt) {
        const int Gs = attempt == 0 ? G0 : 32;
        const int HSs = attempt == 0 ? (G0 < 32 ? 64 : 128) : attempt == 1 ? 512 : 4096;
        const int Gf = Gs, HSf = HSs;
        ovf.zero(c.s);
        spgemm_launch(c, 1, Gs, HSs, 0, X, Y, cnt, C, ovf);
        if (d2h1(c, ovf.p)) continue;
        C.nnz = rowptr_from_counts(c, cnt, C.rp, X.n);
        C.ci.alloc(C.nnz); C.v.alloc(C.nnz * nc);
        spgemm_launch(c, nc, Gf, HSf, 1, X, Y, cnt, C, ovf);
        TSP_REQUIRE(!d2h1(c, ovf.p), TSP_ERR_INVALID_ARG, "spgemm: row too dense");
        return;
    }
    throw Error{TSP_ERR_INVALID_ARG, "spgemm: coarse row exceeds 3072 distinct columns"};
}

static void transpose(Ctx &c, const Csr &P, Csr &R, int nc)
{
    R.n = P.m; R.m = P.n; R.nc = nc; R.nnz = P.nnz;
    DBuf<int32_t> row, keys_out, perm_in, perm_out, cnt;
    row.alloc(P.nnz + 1); keys_out.alloc(P.nnz + 1); perm_in.alloc(P.nnz + 1); perm_out.alloc(P.nnz + 1);
    cnt.alloc(R.n + 1); cnt.zero(c.s);
    if (P.nnz) {
        k_expand_rows<<<grid_for(P.n, 256), 256, 0, c.s>>>(P.n, P.rp, row);
        k_iota<<<grid_for(P.nnz, 256), 256, 0, c.s>>>(P.nnz, perm_in);
        k_col_count<<<grid_for(P.nnz, 256), 256, 0, c.s>>>(P.nnz, P.ci, cnt);
        size_t tb = 0;
        int bits = 1; while ((1LL << bits) < (int64_t)R.n + 1) ++bits;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, P.ci.p, keys_out.p, perm_in.p, perm_out.p, (int)P.nnz, 0, bits, c.s);
        void *t = scratch(c, tb);
        cub::DeviceRadixSort::SortPairs(t, tb, P.ci.p, keys_out.p, perm_in.p, perm_out.p, (int)P.nnz, 0, bits, c.s);
        c.launches += 5;
    }
    rowptr_from_counts(c, cnt, R.rp, R.n);
    R.ci.alloc(R.nnz); R.v.alloc(R.nnz * nc);
    if (P.nnz) k_transpose_fill<<<grid_for(P.nnz, 256), 256, 0, c.s>>>(P.nnz, nc, perm_out, row, P.v, R.ci, R.v);
    TSP_CUDA(cudaGetLastError());
}

static void make_coarsest(Ctx &c, Hier &H, Level &L)
{
    TSP_REQUIRE(L.n <= 4096, TSP_ERR_SINGULAR, "coarsest AMG level exceeds the dense limit (4096 rows)");
    L.coarsest = 1;
    int n = std::max(L.n, 1);
    DBuf<double> work; work.alloc((size_t)L.nc * n * n);
    DBuf<int> piv; piv.alloc((size_t)L.nc * n);
    L.cinv.alloc((size_t)L.nc * n * n);
    c.dcount.zero(c.s);
    if (L.n) k_dense_inv<<<L.nc, 256, 0, c.s>>>(L.n, L.nc, L.A.rp, L.A.ci, L.A.v, work, piv, L.cinv, c.dcount);
    TSP_CUDA(cudaGetLastError());
    H.perturbed += (int64_t)d2h1(c, c.dcount.p);
    c.launches++;
}

// TSP_DEBUG=1: synchronise and print the wall time of each setup phase
void dbg_mark(Ctx &c, const char *what, int lvl)
{
    static const bool on = getenv("TSP_DEBUG") != nullptr;
    static double last = 0;
    if (!on) return;
    cudaStreamSynchronize(c.s);
    timespec t; clock_gettime(CLOCK_MONOTONIC, &t);
    double now = t.tv_sec + 1e-9 * t.tv_nsec;
    if (lvl >= 0 || lvl == -2) {
        cudaMemPool_t pool;
        uint64_t res = 0, used = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        }
        fprintf(stderr, "[tsp setup] level %d %-12s %8.3f ms  pool reserved %.2f GB used %.2f GB\n", lvl, what,
                (now - last) * 1e3, res / 1e9, used / 1e9);
    }
    last = now;
}


// ------------------------------------------------------------------ distributed-setup helpers
__global__ void k_add_off(int64_t nnz, const int32_t *__restrict__ a, int64_t off, int32_t *__restrict__ b)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) b[q] = (int32_t)(a[q] + off);
}
__global__ void k_row_lens(int n, const int32_t *__restrict__ idx, const int32_t *__restrict__ rp, int32_t *__restrict__ len)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) { const int r = idx ? idx[k] : k; len[k] = rp[r + 1] - rp[r]; }
}
// copy rows idx[k] of (rp, ci, v) to a packed buffer at offsets o[k]
__global__ void k_pack_rows(int n, int nc, const int32_t *__restrict__ idx, const int32_t *__restrict__ rp,
                            const int32_t *__restrict__ ci, const double *__restrict__ v, const int32_t *__restrict__ o,
                            int32_t *__restrict__ pci, double *__restrict__ pv)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int r = idx ? idx[k] : k;
    int64_t d = o[k];
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q, ++d) {
        pci[d] = ci[q];
        for (int e = 0; e < nc; ++e) pv[d * nc + e] = v[q * nc + e];
    }
}

static std::vector<int32_t> d2h_vec(Ctx &c, const int32_t *p, size_t n)
{
    std::vector<int32_t> h(n);
    if (n) TSP_CUDA(cudaMemcpyAsync(h.data(), p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    return h;
}

// P rows of the ghost rows of a distributed level: the owners send the rows listed in the
// halo plan; result = P_ext with rows [own rows | ghost rows] and GLOBAL coarse columns.
static void ghost_rows(Ctx &c, Halo &H, const Csr &Pg, Csr &Pext, int nc)
{
    const int ns = H.nsend[0] + H.nsend[1], ng = H.nghost();
    DBuf<int32_t> slen, rlen;
    slen.alloc(std::max(ns, 1)); rlen.alloc(std::max(ng, 1));
    if (ns) k_row_lens<<<grid_for(ns, 256), 256, 0, c.s>>>(ns, H.sidx, Pg.rp, slen);
    c.comm->neighbor_exchange(slen.p, 4 * H.nsend[0], rlen.p, 4 * H.nrecv[0], slen.p + H.nsend[0], 4 * H.nsend[1],
                              rlen.p + H.nrecv[0], 4 * H.nrecv[1], c.s);
    std::vector<int32_t> sl = d2h_vec(c, slen, ns), rl = d2h_vec(c, rlen, ng);
    std::vector<int32_t> so(ns + 1, 0), ro(ng + 1, 0);
    for (int k = 0; k < ns; ++k) so[k + 1] = so[k] + sl[k];
    for (int k = 0; k < ng; ++k) ro[k + 1] = ro[k] + rl[k];
    const int64_t sn_lo = so[H.nsend[0]], sn = so[ns], rn_lo = ro[H.nrecv[0]], rn = ro[ng];
    DBuf<int32_t> sof, sci, rci;
    DBuf<double> sv, rv;
    sof.alloc(ns + 1); sci.alloc(std::max<int64_t>(sn, 1)); sv.alloc(std::max<int64_t>(sn, 1) * nc);
    rci.alloc(std::max<int64_t>(rn, 1)); rv.alloc(std::max<int64_t>(rn, 1) * nc);
    TSP_CUDA(cudaMemcpyAsync(sof, so.data(), sizeof(int32_t) * (ns + 1), cudaMemcpyHostToDevice, c.s));
    if (ns) k_pack_rows<<<grid_for(ns, 128), 128, 0, c.s>>>(ns, nc, H.sidx, Pg.rp, Pg.ci, Pg.v, sof, sci, sv);
    c.comm->neighbor_exchange(sci.p, 4 * sn_lo, rci.p, 4 * rn_lo, sci.p + sn_lo, 4 * (sn - sn_lo), rci.p + rn_lo, 4 * (rn - rn_lo), c.s);
    c.comm->neighbor_exchange(sv.p, 8 * nc * sn_lo, rv.p, 8 * nc * rn_lo, sv.p + sn_lo * nc, 8 * nc * (sn - sn_lo),
                              rv.p + rn_lo * nc, 8 * nc * (rn - rn_lo), c.s);
    // assemble P_ext
    Pext.n = Pg.n + ng; Pext.m = Pg.m; Pext.nc = nc; Pext.nnz = Pg.nnz + rn;
    Pext.rp.alloc(Pext.n + 1); Pext.ci.alloc(std::max<int64_t>(Pext.nnz, 1)); Pext.v.alloc(std::max<int64_t>(Pext.nnz, 1) * nc);
    std::vector<int32_t> prp = d2h_vec(c, Pg.rp, Pg.n + 1);
    for (int k = 0; k < ng; ++k) prp.push_back((int32_t)(Pg.nnz + ro[k + 1]));
    TSP_CUDA(cudaMemcpyAsync(Pext.rp, prp.data(), sizeof(int32_t) * prp.size(), cudaMemcpyHostToDevice, c.s));
    if (Pg.nnz) {
        TSP_CUDA(cudaMemcpyAsync(Pext.ci, Pg.ci, 4 * Pg.nnz, cudaMemcpyDeviceToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(Pext.v, Pg.v, 8 * nc * Pg.nnz, cudaMemcpyDeviceToDevice, c.s));
    }
    if (rn) {
        TSP_CUDA(cudaMemcpyAsync(Pext.ci.p + Pg.nnz, rci, 4 * rn, cudaMemcpyDeviceToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(Pext.v.p + Pg.nnz * nc, rv, 8 * nc * rn, cudaMemcpyDeviceToDevice, c.s));
    }
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.launches += 2;
}

// allgather the rows of a distributed matrix (global columns) into one full copy per rank
static void gather_rows(Ctx &c, const Csr &A, const int32_t *zb, Csr &F, DBuf<int32_t> &zbF, int nc,
                        std::vector<int64_t> &counts)
{
    std::vector<int64_t> me = {(int64_t)A.n, A.nnz};
    std::vector<int64_t> all = host_allgather<int64_t>(c, me);
    const int P = c.nranks;
    int64_t mxn = 1, mxz = 1, N = 0, Z = 0;
    counts.assign(P, 0);
    for (int r = 0; r < P; ++r) {
        counts[r] = all[2 * r];
        mxn = std::max(mxn, all[2 * r]); mxz = std::max(mxz, all[2 * r + 1]);
        N += all[2 * r]; Z += all[2 * r + 1];
    }
    DBuf<int32_t> slen, rlen, sci, rci, szb, rzb;
    DBuf<double> sv, rv;
    slen.alloc(mxn); rlen.alloc(mxn * P); sci.alloc(mxz); rci.alloc(mxz * P); szb.alloc(mxn); rzb.alloc(mxn * P);
    sv.alloc(mxz * nc); rv.alloc(mxz * nc * P);
    if (A.n) {
        k_row_lens<<<grid_for(A.n, 256), 256, 0, c.s>>>(A.n, nullptr, A.rp, slen);
        TSP_CUDA(cudaMemcpyAsync(szb, zb, 4 * A.n, cudaMemcpyDeviceToDevice, c.s));
    }
    if (A.nnz) {
        TSP_CUDA(cudaMemcpyAsync(sci, A.ci, 4 * A.nnz, cudaMemcpyDeviceToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(sv, A.v, 8 * nc * A.nnz, cudaMemcpyDeviceToDevice, c.s));
    }
    c.comm->allgather(slen.p, rlen.p, 4 * mxn, c.s);
    c.comm->allgather(szb.p, rzb.p, 4 * mxn, c.s);
    c.comm->allgather(sci.p, rci.p, 4 * mxz, c.s);
    c.comm->allgather(sv.p, rv.p, 8 * nc * mxz, c.s);
    F.n = (int)N; F.m = (int)N; F.nc = nc; F.nnz = Z;
    F.rp.alloc(N + 1); F.ci.alloc(std::max<int64_t>(Z, 1)); F.v.alloc(std::max<int64_t>(Z, 1) * nc);
    zbF.alloc(std::max<int64_t>(N, 1));
    std::vector<int32_t> lens((size_t)mxn * P);
    TSP_CUDA(cudaMemcpyAsync(lens.data(), rlen, 4 * lens.size(), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    std::vector<int32_t> rp(1, 0);
    int64_t rowo = 0, nzo = 0;
    for (int r = 0; r < P; ++r) {
        for (int64_t k = 0; k < all[2 * r]; ++k) rp.push_back(rp.back() + lens[(size_t)r * mxn + k]);
        if (all[2 * r]) TSP_CUDA(cudaMemcpyAsync(zbF.p + rowo, rzb.p + r * mxn, 4 * all[2 * r], cudaMemcpyDeviceToDevice, c.s));
        if (all[2 * r + 1]) {
            TSP_CUDA(cudaMemcpyAsync(F.ci.p + nzo, rci.p + r * mxz, 4 * all[2 * r + 1], cudaMemcpyDeviceToDevice, c.s));
            TSP_CUDA(cudaMemcpyAsync(F.v.p + nzo * nc, rv.p + r * mxz * nc, 8 * nc * all[2 * r + 1], cudaMemcpyDeviceToDevice, c.s));
        }
        rowo += all[2 * r]; nzo += all[2 * r + 1];
    }
    TSP_CUDA(cudaMemcpyAsync(F.rp, rp.data(), 4 * rp.size(), cudaMemcpyHostToDevice, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.launches++;
}

// ------------------------------------------------------------------ hierarchy build (row a4)
// Level 0 arrives distributed when nranks > 1 (halo plan `fine_halo`, global row offset
// `row_off0`).  A coarse level stays distributed while its global size exceeds
// opts.replicate_rows; below that it is gathered onto every rank and the rest of the
// hierarchy is built redundantly (identical data => identical results on all ranks).
//
// refresh = true (frozen aggregation, NEXT-f1, DESIGN.md R-refresh): A0 holds new values on the pattern the
// hierarchy H was built from; the strength flags, MIS(2) roots, aggregates and every pattern of H are kept and
// every value is recomputed in the build's own order and arithmetic (l1 norms, filtered diagonal with the KEPT
// strength flags, rho and omega, P, R = P^T, A_c = R (A P), the coarsest inverse) -- the oracle's amg_refresh.
void amg_build(Ctx &c, Hier &H, Csr &A0, DBuf<int32_t> &zb0, int nc, Halo *fine_halo, int64_t row_off0, int64_t nglob0,
               bool refresh)
{
    dbg_mark(c, "start", -1);
    H.smoother = (nc == 1 && c.o.amg_smoother_p >= 0) ? c.o.amg_smoother_p : c.o.amg_smoother;
    if (refresh) {
        TSP_REQUIRE(!H.L.empty() && H.nc == nc && H.L[0].A.n == A0.n && H.L[0].A.nnz == A0.nnz, TSP_ERR_STATE,
                    "refresh: no hierarchy of this pattern to refresh");
        H.perturbed = 0;
        H.L[0].A = std::move(A0);          // same pattern (checked by the caller), new values
    } else {
        H.L.clear();
        dbg_mark(c, "free old", -2);
        H.L.reserve(16);
        H.nc = nc;
        H.L.emplace_back();
        Level &L0 = H.L[0];
        L0.A = std::move(A0);
        L0.zb = std::move(zb0);
        L0.dist = c.comm != nullptr;
        L0.row_off = row_off0;
        L0.nglob = nglob0;
        L0.hp = fine_halo;
    }
    const int maxl = std::min(std::max(c.o.amg_max_levels, 1), 16);
    const int64_t rep_rows = c.o.replicate_rows > 0 ? c.o.replicate_rows : 32768;
    DBuf<int> err; err.alloc(1);
    for (int lvl = 0;; ++lvl) {
        Level &L = H.L[lvl];
        L.n = L.A.n; L.nc = nc;
        if (!L.dist) { L.nglob = L.n; L.row_off = 0; }
        const int n = L.n;
        const int nown = n;   // rows of this rank; columns >= nown are ghosts
        L.dl1.alloc((size_t)std::max(n, 1) * nc); L.dinv.alloc((size_t)std::max(n, 1) * nc);
        if (n) k_l1<<<grid_for((int64_t)n * nc, 256), 256, 0, c.s>>>(n, nc, L.A.rp, L.A.ci, L.A.v, L.dl1, L.dinv);
        c.launches++;
        if (L.dist && L.hp->any()) {
            L.dinv_gh.alloc((size_t)std::max(L.hp->nghost(), 1) * nc);
            halo_exchange(c, *L.hp, nc, L.dinv, L.dinv_gh);
        }
        if (refresh ? L.coarsest != 0 : (L.nglob <= c.o.amg_coarse_max || lvl == maxl - 1)) {
            TSP_REQUIRE(!L.dist, TSP_ERR_INVALID_ARG, "the distributed fine level is too small for this many ranks");
            make_coarsest(c, H, L);
            break;
        }
        int nagg = L.nagg;
        int64_t nagg_glob = L.nagg_glob, coarse_off = L.coarse_off;
        if (!refresh) {
            // strength + symmetrisation (the flags E are kept for a later refresh)
            DBuf<uint8_t> S; S.alloc(L.A.nnz + 1);
            DBuf<uint8_t> &E = L.E; E.alloc(L.A.nnz + 1);
            err.zero(c.s);
            if (n) {
                k_strength<<<grid_for((int64_t)n * kStrG, 256), 256, 0, c.s>>>(n, nc, nown, L.A.rp, L.A.ci, L.A.v, L.zb, c.o.amg_theta, S);
                k_symm<<<grid_for((int64_t)n * kStrG, 256), 256, 0, c.s>>>(n, nown, L.dist ? 1 : 0, L.A.rp, L.A.ci, S, E, err);
            }
            c.launches += 2;
            TSP_REQUIRE(!d2h1(c, err.p), TSP_ERR_INVALID_ARG, "AMG input pattern is not structurally symmetric");
            // MIS(2) rounds: the strength graph never leaves a z-block, so each rank runs its own rounds
            DBuf<int8_t> st; st.alloc(std::max(n, 1));
            DBuf<uint64_t> t1; t1.alloc(std::max(n, 1));
            DBuf<uint8_t> newr, near1; newr.alloc(std::max(n, 1)); near1.alloc(std::max(n, 1));
            if (n) k_mis_init<<<grid_for(n, 256), 256, 0, c.s>>>(n, L.A.rp, E, st);
            c.launches++;
            const int off = (int)L.row_off;
            for (int round = 0; round < 1000 && n; ++round) {
                k_mis_t1<<<grid_for(n, 256), 256, 0, c.s>>>(n, off, L.A.rp, L.A.ci, E, st, t1);
                k_mis_root<<<grid_for(n, 256), 256, 0, c.s>>>(n, off, L.A.rp, L.A.ci, E, st, t1, newr);
                k_mis_near<<<grid_for(n, 256), 256, 0, c.s>>>(n, L.A.rp, L.A.ci, E, newr, st, near1);
                c.dcount.zero(c.s);
                k_mis_out<<<grid_for(n, 256), 256, 0, c.s>>>(n, L.A.rp, L.A.ci, E, near1, st, c.dcount);
                c.launches += 4;
                if (d2h1(c, c.dcount.p) == 0) break;
            }
            dbg_mark(c, "strength+mis", lvl);
            // aggregates: local numbering by ascending root, global = coarse_off + local
            DBuf<int32_t> flag, rid, ph1;
            flag.alloc(n + 1); rid.alloc(n + 1); ph1.alloc(std::max(n, 1));
            if (n) k_rootflag<<<grid_for(n, 256), 256, 0, c.s>>>(n, st, flag);
            TSP_CUDA(cudaMemsetAsync(flag.p + n, 0, sizeof(int32_t), c.s));
            exclusive_scan<int32_t>(c, flag, rid, n + 1);
            nagg = d2h1(c, rid.p + n);
            nagg_glob = nagg; coarse_off = 0;
            if (L.dist) {
                std::vector<int64_t> all = host_allgather<int64_t>(c, std::vector<int64_t>{(int64_t)nagg});
                nagg_glob = 0;
                for (int r = 0; r < c.nranks; ++r) { if (r < c.rank) coarse_off += all[r]; nagg_glob += all[r]; }
            }
            if (nagg_glob == 0 || (double)nagg_glob > 0.8 * (double)L.nglob) {   // stagnation: direct solve here
                TSP_REQUIRE(!L.dist, TSP_ERR_SINGULAR, "coarsening stagnated on a distributed level");
                H.fallbacks++;
                make_coarsest(c, H, L);
                break;
            }
            L.nagg = nagg;
            L.nagg_glob = nagg_glob;
            L.coarse_off = coarse_off;
            L.agg.alloc(std::max(n, 1));
            H.L.emplace_back();
            Level &Lc = H.L[lvl + 1];
            Level &Lf = H.L[lvl];   // re-fetch after emplace_back
            Lc.zb.alloc(std::max(nagg, 1));
            TSP_CUDA(cudaMemsetAsync(ph1, 0xff, sizeof(int32_t) * std::max(n, 1), c.s));
            if (n) {
                k_phase1<<<grid_for(n, 256), 256, 0, c.s>>>(n, Lf.A.rp, Lf.A.ci, Lf.E, st, rid, Lf.zb, ph1, Lc.zb);
                k_phase2<<<grid_for(n, 256), 256, 0, c.s>>>(n, nc, Lf.A.rp, Lf.A.ci, Lf.A.v, Lf.E, st, ph1, Lf.agg);
            }
            c.launches += 3;
        }
        Level &Lc = H.L[lvl + 1];
        Level &Lf = H.L[lvl];
        const uint8_t *E = Lf.E.p;
        // prolongator
        DBuf<double> d; d.alloc((size_t)std::max(n, 1) * nc);
        DBuf<unsigned long long> rho; rho.alloc(3); rho.zero(c.s);
        if (n) k_pdiag<<<grid_for((int64_t)n * nc, 256), 256, 0, c.s>>>(n, nc, Lf.A.rp, Lf.A.ci, Lf.A.v, E, d, rho);
        unsigned long long rb[3] = {0, 0, 0};
        TSP_CUDA(cudaMemcpyAsync(rb, rho.p, sizeof(rb), cudaMemcpyDeviceToHost, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
        std::vector<double> rhos(3);
        for (int k = 0; k < 3; ++k) memcpy(&rhos[k], &rb[k], sizeof(double));
        if (Lf.dist) {   // global max (exact, order independent)
            std::vector<double> all = host_allgather<double>(c, rhos);
            for (int r = 0; r < c.nranks; ++r)
                for (int k = 0; k < 3; ++k) rhos[k] = std::max(rhos[k], all[3 * r + k]);
        }
        Omega om;
        for (int k = 0; k < 3; ++k) {
            const double r = rhos[k];
            volatile double three_r = 3.0 * r;   // IEEE: 4 / (3 rho), same expression as the oracle
            om.w[k] = (k < nc && r > 0.0) ? 4.0 / three_r : 0.0;
        }
        DBuf<int32_t> cnt; cnt.alloc(n + 1);
        err.zero(c.s);
        if (n) k_pcount<<<grid_for(n, 128), 128, 0, c.s>>>(n, Lf.A.rp, Lf.A.ci, E, Lf.agg, cnt, err);
        Lf.P.n = n; Lf.P.m = nagg; Lf.P.nc = nc;
        Lf.P.nnz = rowptr_from_counts(c, cnt, Lf.P.rp, n);
        Lf.P.ci.alloc(std::max<int64_t>(Lf.P.nnz, 1)); Lf.P.v.alloc(std::max<int64_t>(Lf.P.nnz, 1) * nc);
        if (n) k_pfill<<<grid_for((int64_t)n * nc, 128), 128, 0, c.s>>>(n, nc, Lf.A.rp, Lf.A.ci, Lf.A.v, E, Lf.agg, d, om, Lf.P.rp, Lf.P.ci, Lf.P.v, err);
        c.launches += 3;
        TSP_REQUIRE(!d2h1(c, err.p), TSP_ERR_INVALID_ARG, "prolongator row exceeds 512 aggregates");
        dbg_mark(c, "agg+P", lvl);
        transpose(c, Lf.P, Lf.R, nc);     // local coarse rows x local fine columns
        dbg_mark(c, "transpose", lvl);
        // P with GLOBAL coarse columns (and the ghost rows on a distributed level)
        Csr Pg;
        Pg.n = Lf.P.n; Pg.m = (int)nagg_glob; Pg.nc = nc; Pg.nnz = Lf.P.nnz;
        Pg.rp.alloc(n + 1); Pg.ci.alloc(std::max<int64_t>(Pg.nnz, 1)); Pg.v.alloc(std::max<int64_t>(Pg.nnz, 1) * nc);
        TSP_CUDA(cudaMemcpyAsync(Pg.rp, Lf.P.rp, 4 * (n + 1), cudaMemcpyDeviceToDevice, c.s));
        if (Pg.nnz) {
            k_add_off<<<grid_for(Pg.nnz, 256), 256, 0, c.s>>>(Pg.nnz, Lf.P.ci, coarse_off, Pg.ci);
            TSP_CUDA(cudaMemcpyAsync(Pg.v, Lf.P.v, 8 * nc * Pg.nnz, cudaMemcpyDeviceToDevice, c.s));
        }
        Csr AP;
        if (Lf.dist && Lf.hp->any()) {
            Csr Pext;
            ghost_rows(c, *Lf.hp, Pg, Pext, nc);
            spgemm(c, Lf.A, Pext, AP, nc);
        } else {
            spgemm(c, Lf.A, Pg, AP, nc);
        }
        AP.m = (int)nagg_glob;
        dbg_mark(c, "AP", lvl);
        Csr Ac;
        spgemm(c, Lf.R, AP, Ac, nc);       // local coarse rows, global coarse columns
        Ac.m = (int)nagg_glob;
        dbg_mark(c, "RAP", lvl);
        if (Lf.dist && nagg_glob > rep_rows) {
            // next level stays distributed: remap its columns to local + ghosts
            Lc.dist = true; Lc.nglob = nagg_glob; Lc.row_off = coarse_off;
            Lc.A = std::move(Ac);
            DBuf<int32_t> gcol; gcol.alloc(std::max<int64_t>(Lc.A.nnz, 1));
            if (Lc.A.nnz) TSP_CUDA(cudaMemcpyAsync(gcol, Lc.A.ci, 4 * Lc.A.nnz, cudaMemcpyDeviceToDevice, c.s));
            halo_build(c, Lc.halo, nagg, coarse_off, gcol, Lc.A.nnz, Lc.A.ci);
            Lc.A.gci = std::move(gcol);
            Lc.A.m = nagg + Lc.halo.nghost();
            Lc.hp = &Lc.halo;
            Lf.next_dist = true;
        } else if (Lf.dist) {
            // gather the coarse level onto every rank; the prolongator then addresses the full vector
            DBuf<int32_t> zbF;
            // (refresh: Lc.zb is already the gathered copy; this rank's rows start at coarse_off)
            gather_rows(c, Ac, refresh ? Lc.zb.p + coarse_off : Lc.zb.p, Lc.A, zbF, nc, Lf.rep_counts);
            Lc.zb = std::move(zbF);
            Lc.dist = false;
            Lf.rep_offs.assign(c.nranks + 1, 0);
            for (int r = 0; r < c.nranks; ++r) Lf.rep_offs[r + 1] = Lf.rep_offs[r] + Lf.rep_counts[r];
            int64_t mx = 1;
            for (auto v : Lf.rep_counts) mx = std::max(mx, v);
            Lf.rep_buf.alloc((size_t)mx * nc * (c.nranks + 1));
            Lf.rep_offs_d.alloc(c.nranks + 1);           // uploaded once, read by every V-cycle's gather
            TSP_CUDA(cudaMemcpyAsync(Lf.rep_offs_d, Lf.rep_offs.data(), sizeof(int64_t) * (c.nranks + 1),
                                     cudaMemcpyHostToDevice, c.s));
            TSP_CUDA(cudaStreamSynchronize(c.s));
            Lf.P.m = (int)nagg_glob;
            if (Lf.P.nnz) TSP_CUDA(cudaMemcpyAsync(Lf.P.ci, Pg.ci, 4 * Lf.P.nnz, cudaMemcpyDeviceToDevice, c.s));
        } else {
            Lc.A = std::move(Ac);
        }
    }
    // apply-side layouts and work vectors
    for (size_t l = 0; l < H.L.size(); ++l) {
        Level &L = H.L[l];
        if (l == 0 && nc == 1 && !L.coarsest) p7_build(c, L.A);            // pressure level 0: p7.cu when 7-point
        const bool structured = l == 0 && !L.coarsest && ((nc == 3 && c.sym_sdc.ok) || (nc == 1 && c.p7_ok));
        if (!structured) sell_from_csr(c, L.A, L.sA, nc);                  // sym.cu / p7.cu cover level 0
        else L.sA = Sell{};
        if (!L.coarsest) {
            sell_from_csr(c, L.P, L.sP, nc);
            sell_from_csr(c, L.R, L.sR, nc);
        }
        size_t m = (size_t)std::max(L.n, 1) * nc;
        L.b.alloc(m); L.x.alloc(m); L.x2.alloc(m); L.r.alloc(m);
        if (H.smoother == 2) { L.dcheb.alloc(m); L.xc.alloc(m); } else { L.dcheb.release(); L.xc.release(); }
        {   // kernel choice from global mean row lengths, so every rank computes a row exactly like P = 1
            std::vector<int64_t> st = {L.A.nnz, (int64_t)L.n, L.coarsest ? 0 : L.R.nnz, L.coarsest ? 0 : (int64_t)L.R.n};
            if (L.dist) {
                std::vector<int64_t> all = host_allgather<int64_t>(c, st);
                st.assign(4, 0);
                for (int r = 0; r < c.nranks; ++r) for (int k = 0; k < 4; ++k) st[k] += all[4 * r + k];
            }
            L.warpA = l > 0 ? lanes_forced(lanes_for(st[0], st[1], c.sm_count)) : 0;
            L.warpR = lanes_forced(lanes_for(st[2], st[3], c.sm_count));
            if (l > 0 && !L.coarsest) c.variants[TSP_VAR_LANES_A0 + lanes_idx(L.warpA)]++;
            if (!L.coarsest) c.variants[TSP_VAR_LANES_R0 + lanes_idx(L.warpR)]++;
        }
        if (L.dist) {
            const size_t g = (size_t)std::max(L.hp->nghost(), 1) * nc;
            L.gh_b.alloc(g); L.gh_x.alloc(g);
        }
    }
    gs_setup(c, H, nc);                    // Gauss-Seidel smoother layouts (amg_smoother = 1)
    dbg_mark(c, "sell+vectors", 99);
    TSP_CUDA(cudaStreamSynchronize(c.s));
}

// ------------------------------------------------------------------ V-cycle kernels (apply; free arithmetic)
// x = D^-1 b over the own values and, on a distributed level, over the ghost values (xg = bg dg): the first
// half of pre-smoothing from zero on the coarse levels, whose residual r = b - A x then gathers ONE vector
// (a fused pre-smoothing kernel gathering b and D^-1 per entry was L1-bound: C5 mechanics level 1
// 152 us against 98 us for the same product in post-smoothing).  The same products b_j D^-1_j as the fused
// form: results are bitwise unchanged.
__global__ void k_dscale(int64_t m, const double *__restrict__ b, const double *__restrict__ dinv, double *__restrict__ x,
                         int64_t mg, const double *__restrict__ bg, const double *__restrict__ dg, double *__restrict__ xg)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < m) x[t] = b[t] * dinv[t];
    else if (t - m < mg) xg[t - m] = bg[t - m] * dg[t - m];
}
// y = S x  (restriction R r; rows and columns local)
template <int NC>
__global__ void __launch_bounds__(256) k_sell_mv(int n, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                 const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = i >> 5, lane = i & 31;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const int64_t b0 = off[s], b1 = off[s + 1];
#pragma unroll 2
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), __ldg(x + (int64_t)j * NC + c), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) y[(int64_t)i * NC + c] = acc[c];
}
// x += P xc
template <int NC>
__global__ void __launch_bounds__(256) k_prolong(int n, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                 const double *__restrict__ val, const double *__restrict__ xc, double *__restrict__ x)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = i >> 5, lane = i & 31;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = x[(int64_t)i * NC + c];
    const int64_t b0 = off[s], b1 = off[s + 1];
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), __ldg(xc + (int64_t)j * NC + c), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) x[(int64_t)i * NC + c] = acc[c];
}
// post-smooth: xo = x + D^-1 (b - A x)   (x ghost-aware)
template <int NC, bool D>
__global__ void __launch_bounds__(256) k_vc_post(int n, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                 const double *__restrict__ val, const double *__restrict__ dinv,
                                                 const double *__restrict__ b, GV x, double *__restrict__ xo)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = i >> 5, lane = i & 31;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const int64_t b0 = off[s], b1 = off[s + 1];
#pragma unroll 2
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), gvld<D>(x, j, c, NC), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int64_t t = (int64_t)i * NC + c;
        xo[t] = x.own[t] + dinv[t] * (b[t] - acc[c]);
    }
}
// residual r = b - A x (Gauss-Seidel smoother after the forward sweep; Chebyshev steps; x ghost-aware)
template <int NC, bool D>
__global__ void __launch_bounds__(256) k_sell_resid(int n, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                    const double *__restrict__ val, const double *__restrict__ b,
                                                    GV x, double *__restrict__ r)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = i >> 5, lane = i & 31;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const int64_t b0 = off[s], b1 = off[s + 1];
#pragma unroll 2
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), gvld<D>(x, j, c, NC), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) r[(int64_t)i * NC + c] = b[(int64_t)i * NC + c] - acc[c];
}
// fused Chebyshev step on a SELL operator (R-cheb, cheb_epi): PRE gathers sc dinv_j b_j, STEP gathers x_j
template <int NC, bool D, bool PRE>
__global__ void __launch_bounds__(256) k_cheb_sell(int n, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                   const double *__restrict__ val, GV dinv, GV b, GV x, ChebArgs ca,
                                                   double *__restrict__ xo)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = i >> 5, lane = i & 31;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const int64_t b0 = off[s], b1 = off[s + 1];
#pragma unroll 2
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const double xv = PRE ? ca.sc * (gvld<D>(dinv, j, c, NC) * gvld<D>(b, j, c, NC)) : gvld<D>(x, j, c, NC);
            acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), xv, acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int64_t t = (int64_t)i * NC + c;
        cheb_epi<PRE>(t, acc[c], b.own[t], dinv.own[t], PRE ? 0.0 : x.own[t], ca, xo);
    }
}
// one Chebyshev step after its residual (R-cheb): d = alpha d + beta D^-1 r (alpha ignored when first);
// xo = x + d (x == nullptr: from zero).  In place (xo == x) is fine: every entry is its own.
__global__ void k_cheb_upd(int64_t m, const double *__restrict__ r, const double *__restrict__ dinv, double *__restrict__ d,
                           const double *x, double *xo, double alpha, double beta, int first)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    const double dn = (first ? 0.0 : alpha * d[t]) + beta * (dinv[t] * r[t]);
    d[t] = dn;
    xo[t] = (x ? x[t] : 0.0) + dn;
}
// coarsest: x = A_c^-1 b per component
template <int NC>
__global__ void k_coarse(int n, const double *__restrict__ inv, const double *__restrict__ b, double *__restrict__ x)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int c = blockIdx.y;
    if (i >= n) return;
    const double *row = inv + ((size_t)c * n + i) * n;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(row[j], b[(int64_t)j * NC + c], s);
    x[(int64_t)i * NC + c] = s;
}

// ---- vector-CSR variants for operators with long rows (coarse levels, restriction): a
// group of G lanes (G | 32) per row strides the row's entries (coalesced [q][c] values),
// then a fixed shuffle tree inside the group.  32/G rows per warp keep several dependent
// load chains in flight.
// MODE 0: y = A x ; MODE 2: post (xo = x + D^-1 (b - A x));
// MODE 3: residual r = b - A x ; MODE 4 / 5: fused Chebyshev PRE / STEP (cheb_epi, R-cheb)
template <int NC, int MODE, bool D, int G>
__global__ void __launch_bounds__(256) k_csr_vec(int n, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                 const double *__restrict__ v, GV dinv, GV b, GV x,
                                                 double *__restrict__ out1, double *__restrict__ out2, ChebArgs ca)
{
    const int sub = threadIdx.x & (G - 1);
    const int i = blockIdx.x * (blockDim.x / G) + (threadIdx.x / G);
    const bool ok = i < n;
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    if (ok) {
        const int64_t q1 = rp[i + 1];
#pragma unroll 2
        for (int64_t q = rp[i] + sub; q < q1; q += G) {
            const int j = ci[q];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double xv = MODE == 4 ? ca.sc * (gvld<D>(dinv, j, c, NC) * gvld<D>(b, j, c, NC)) : gvld<D>(x, j, c, NC);
                acc[c] = fma(__ldcs(v + q * NC + c), xv, acc[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int o = G / 2; o; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (ok && sub < NC) {
        double a = acc[0];
#pragma unroll
        for (int c = 1; c < NC; ++c) if (sub == c) a = acc[c];
        const int64_t t = (int64_t)i * NC + sub;
        if (MODE == 0) out1[t] = a;
        else if (MODE == 3) out1[t] = b.own[t] - a;
        else if (MODE == 4 || MODE == 5) cheb_epi<MODE == 4>(t, a, b.own[t], dinv.own[t], MODE == 5 ? x.own[t] : 0.0, ca, out1);
        else out1[t] = x.own[t] + dinv.own[t] * (b.own[t] - a);
    }
}
template <int NC, int MODE, bool D>
static void csr_vec(int G, cudaStream_t s, int n, const Csr &A, GV dinv, GV b, GV x, double *o1, double *o2,
                    const ChebArgs &ca)
{
    if (!n) return;
    const int rows = 256 / G;
    const dim3 grid((unsigned)((n + rows - 1) / rows));
    if (G == 8) k_csr_vec<NC, MODE, D, 8><<<grid, 256, 0, s>>>(n, A.rp, A.ci, A.v, dinv, b, x, o1, o2, ca);
    else if (G == 16) k_csr_vec<NC, MODE, D, 16><<<grid, 256, 0, s>>>(n, A.rp, A.ci, A.v, dinv, b, x, o1, o2, ca);
    else k_csr_vec<NC, MODE, D, 32><<<grid, 256, 0, s>>>(n, A.rp, A.ci, A.v, dinv, b, x, o1, o2, ca);
}
// compact the padded allgather [rank][mx*nc] into the full replicated vector
__global__ void k_rep_compact(int nranks, int nc, int64_t mx, const int64_t *__restrict__ offs, const double *__restrict__ buf,
                              double *__restrict__ out)
{
    const int r = blockIdx.y;
    const int64_t cnt = (offs[r + 1] - offs[r]) * nc;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x)
        out[offs[r] * nc + k] = buf[r * mx * nc + k];
}

static double sbytes(const Sell &S) { return (double)S.slots * 32 * (4.0 + 8.0 * S.bs); }
static double cbytes(const Csr &A) { return (double)A.nnz * (4.0 + 8.0 * A.nc); }

// r = b - A x on level l (x's ghosts exchanged first on a distributed level)
template <int NC>
static void level_resid(Ctx &c, Level &L, bool sym0, const double *b, const double *x, double *r)
{
    const int n = L.n;
    if (L.dist) halo_exchange(c, *L.hp, NC, x, L.gh_x);
    const GV gx = gv(x, n, L.dist ? L.gh_x.p : nullptr);
    if (NC == 1 && &L == &c.pres.L[0] && c.p7_ok) p7_launch(c, 3, gv(nullptr, 0), gv(b, n), gx, r, nullptr, ChebArgs{});
    else if (sym0) sym_vcycle_resid(c, n, b, gx, r);
    else if (L.warpA) (L.dist ? csr_vec<NC, 3, true> : csr_vec<NC, 3, false>)(L.warpA, c.s, n, L.A, gv(nullptr, 0), gv(b, n), gx, r, nullptr, ChebArgs{});
    else if (n) (L.dist ? k_sell_resid<NC, true> : k_sell_resid<NC, false>)<<<grid_for(n, 256), 256, 0, c.s>>>(
        n, L.sA.off, L.sA.col, L.sA.val, b, gx, r);
    c.launches++;
}

// Chebyshev smoother (R-cheb; the oracle's cheb_smooth): `amg_cheb_degree` steps of the Chebyshev iteration on
// D_l1^-1 A over [lower, 1].  Fused kernels (cheb_epi): pre-smoothing from zero does steps 0 and 1 in ONE product
// (PRE), every further step and each post-smoothing step is one product + epilogue (STEP); degree 1 pre-smoothing
// is the elementwise x = D^-1 b / theta.  x_0 = xin (post) or 0 (pre); the result lands in `x` (!= xin); `tmp` is
// the ping-pong buffer.
template <int NC>
static void cheb_step(Ctx &c, Level &L, bool sym0, bool pre, const double *b, const double *xk, const ChebArgs &a, double *xo)
{
    const int n = L.n;
    const GV gd = gv(L.dinv, n, L.dist ? L.dinv_gh.p : nullptr);
    GV gb = gv(b, n), gx = gv(nullptr, 0);
    if (pre) {
        if (L.dist) { halo_exchange(c, *L.hp, NC, b, L.gh_b); gb = gv(b, n, L.gh_b.p); }
    } else {
        if (L.dist) halo_exchange(c, *L.hp, NC, xk, L.gh_x);
        gx = gv(xk, n, L.dist ? L.gh_x.p : nullptr);
    }
    if (NC == 1 && &L == &c.pres.L[0] && c.p7_ok) p7_launch(c, pre ? 4 : 5, gd, gb, gx, xo, nullptr, a);
    else if (sym0) sym_vcycle_cheb(c, n, pre, gd, gb, gx, a, xo);
    else if (L.warpA) {
        if (pre) (L.dist ? csr_vec<NC, 4, true> : csr_vec<NC, 4, false>)(L.warpA, c.s, n, L.A, gd, gb, gx, xo, nullptr, a);
        else (L.dist ? csr_vec<NC, 5, true> : csr_vec<NC, 5, false>)(L.warpA, c.s, n, L.A, gd, gb, gx, xo, nullptr, a);
    } else if (n) {
#define CHS(DD, PP) k_cheb_sell<NC, DD, PP><<<grid_for(n, 256), 256, 0, c.s>>>(n, L.sA.off, L.sA.col, L.sA.val, gd, gb, gx, a, xo)
        if (L.dist) { if (pre) CHS(true, true); else CHS(true, false); }
        else { if (pre) CHS(false, true); else CHS(false, false); }
#undef CHS
    }
    c.launches++;
}

template <int NC>
static void cheb_run(Ctx &c, Level &L, bool sym0, const double *b, const double *xin, double *x, double *tmp, bool from_zero)
{
    const int64_t m = (int64_t)L.n * NC;
    const int deg = c.o.amg_cheb_degree;
    const double bb = 1.0, aa = c.o.amg_cheb_lower * bb;
    const double theta = 0.5 * (bb + aa), delta = 0.5 * (bb - aa), sigma = theta / delta;
    std::vector<double> al(deg, 0.0), be(deg, 1.0 / theta);   // step k: d_k = al[k] d_{k-1} + be[k] D^-1 r_k
    double rho = 1.0 / sigma;
    for (int k = 1; k < deg; ++k) {
        const double rn = 1.0 / (2.0 * sigma - rho);
        al[k] = rn * rho; be[k] = 2.0 * rn / delta;
        rho = rn;
    }
    // buffers: the steps alternate between x and tmp so that the last one writes x
    int k = 0;
    const double *cur = xin;
    const int launches = from_zero ? deg - 1 : deg;   // PRE covers steps 0 and 1
    double *dst = (launches % 2 == 1) ? x : tmp;      // alternate so that the last launch writes x
    if (from_zero) {
        if (deg == 1) {
            if (m) k_cheb_upd<<<grid_for(m, 256), 256, 0, c.s>>>(m, b, L.dinv, L.dcheb, nullptr, x, 0.0, 1.0 / theta, 1);
            c.launches++;
            return;
        }
        ChebArgs a{nullptr, deg > 2 ? L.dcheb.p : nullptr, al[1], be[1], 1.0 / theta};
        cheb_step<NC>(c, L, sym0, true, b, nullptr, a, dst);
        cur = dst; dst = (dst == x) ? tmp : x;
        k = 2;
    }
    for (; k < deg; ++k) {
        ChebArgs a{k == 0 ? nullptr : L.dcheb.p, k + 1 < deg ? L.dcheb.p : nullptr, al[k], be[k], 0.0};
        cheb_step<NC>(c, L, sym0, false, b, cur, a, dst);
        cur = dst; dst = (dst == x) ? tmp : x;
    }
}

template <int NC>
static void vcycle_rec(Ctx &c, Hier &H, int l, const double *b, double *xout)
{
    Level &L = H.L[l];
    const bool mech = NC == 3;
    const int l0 = l == 0 ? PK_VC_L0 : 0;    // level 0 has profile classes of its own
    if (L.coarsest) {
        prof_begin(c, PK_COARSE);
        if (L.n) k_coarse<NC><<<dim3(grid_for(L.n, 128), NC), 128, 0, c.s>>>(L.n, L.cinv, b, xout);
        prof_end(c, PK_COARSE, 8.0 * L.n * L.n * NC);
        c.launches++;
        return;
    }
    const int n = L.n;
    const double vec = 8.0 * NC * n;
    const int wA = L.warpA, wR = L.warpR;
    const double bA = wA ? cbytes(L.A) : sbytes(L.sA), bR = wR ? cbytes(L.R) : sbytes(L.sR);
    const double *ghd = L.dist ? L.dinv_gh.p : nullptr;
    // pre-smooth + residual (needs b and D^-1 of the ghost rows)
    if (L.dist) halo_exchange(c, *L.hp, NC, b, L.gh_b);
    const GV gb = gv(b, n, L.dist ? L.gh_b.p : nullptr), gd = gv(L.dinv, n, ghd);
    const bool sym0 = mech && l == 0 && c.sym_sdc.ok;     // structured symmetric level 0 (sym.cu)
    const bool p70 = !mech && l == 0 && c.p7_ok;          // structured 7-point pressure level 0 (p7.cu)
    const double bA0 = sym0 ? sym_bytes(c, 3) : p70 ? p7_bytes(c) : bA;
    const bool gs = H.smoother == 1;         // Gauss-Seidel (gs.cu, R-gs): single GPU, never distributed
    const bool cheb = H.smoother == 2;       // Chebyshev (R-cheb)
    const int deg = c.o.amg_cheb_degree;
    prof_begin(c, (mech ? PK_VC_PRE_U : PK_VC_PRE_P) + l0);
    if (gs) {
        gs_sweep<NC>(c, L, false, b, nullptr, L.x2);                      // forward sweep from zero
        level_resid<NC>(c, L, sym0, b, L.x2, L.r);
    } else if (cheb) {
        cheb_run<NC>(c, L, sym0, b, nullptr, L.x2, L.xc, true);
        level_resid<NC>(c, L, sym0, b, L.x2, L.r);
    }
    else if (p70) p7_launch(c, 1, gd, gb, gv(nullptr, 0), L.x2, L.r, ChebArgs{});
    else if (n) {                        // x = D^-1 b (k_dscale), then r = b - A x (one gathered vector)
        const int64_t m = (int64_t)n * NC, mg = L.dist ? (int64_t)L.hp->nghost() * NC : 0;
        k_dscale<<<grid_for(m + mg, 256), 256, 0, c.s>>>(m, b, L.dinv, L.x2, mg, L.gh_b.p, ghd, L.gh_x.p);
        c.launches++;
        const GV gx = gv(L.x2, n, L.dist ? L.gh_x.p : nullptr);
        if (sym0) sym_vcycle_resid(c, n, b, gx, L.r);
        else if (wA) (L.dist ? csr_vec<NC, 3, true> : csr_vec<NC, 3, false>)(wA, c.s, n, L.A, gv(nullptr, 0), gb, gx, L.r, nullptr, ChebArgs{});
        else (L.dist ? k_sell_resid<NC, true> : k_sell_resid<NC, false>)<<<grid_for(n, 256), 256, 0, c.s>>>(
            n, L.sA.off, L.sA.col, L.sA.val, b, gx, L.r);
    }
    prof_end(c, (mech ? PK_VC_PRE_U : PK_VC_PRE_P) + l0, gs ? gs_sweep_bytes(L, NC) + bA0 + 3 * vec
                                                  : cheb ? (deg - 1) * (bA0 + 5 * vec) + bA0 + 3 * vec : bA0 + 4 * vec);
    // restriction (local rows of R); a replicated next level is gathered on every rank
    Level &Lc = H.L[l + 1];
    const bool gather = L.dist && !L.next_dist;
    const int nr = L.sR.nrows;
    double *rdst = gather ? L.rep_buf.p + (size_t)c.nranks * 0 : Lc.b.p;
    prof_begin(c, (mech ? PK_VC_RESTR_U : PK_VC_RESTR_P) + l0);
    if (wR) csr_vec<NC, 0, false>(wR, c.s, nr, L.R, gv(nullptr, 0), gv(nullptr, 0), gv(L.r, n), rdst, nullptr, ChebArgs{});
    else if (nr) k_sell_mv<NC><<<grid_for(nr, 256), 256, 0, c.s>>>(nr, L.sR.off, L.sR.col, L.sR.val, L.r, rdst);
    prof_end(c, (mech ? PK_VC_RESTR_U : PK_VC_RESTR_P) + l0, bR + vec + 8.0 * NC * nr);
    if (gather) {
        int64_t mx = 1;
        for (auto v : L.rep_counts) mx = std::max(mx, v);
        double *recv = L.rep_buf.p + (size_t)mx * NC;
        c.comm->allgather(L.rep_buf.p, recv, sizeof(double) * mx * NC, c.s);
        k_rep_compact<<<dim3(grid_for(mx * NC, 256), c.nranks), 256, 0, c.s>>>(c.nranks, NC, mx, L.rep_offs_d, recv, Lc.b);
        c.launches++;
    }
    vcycle_rec<NC>(c, H, l + 1, Lc.b, Lc.x);
    prof_begin(c, (mech ? PK_VC_PROL_U : PK_VC_PROL_P) + l0);
    if (n) k_prolong<NC><<<grid_for(n, 256), 256, 0, c.s>>>(n, L.sP.off, L.sP.col, L.sP.val, Lc.x, L.x2);
    prof_end(c, (mech ? PK_VC_PROL_U : PK_VC_PROL_P) + l0, sbytes(L.sP) + 2 * vec + 8.0 * NC * Lc.n);
    // post-smooth (needs x of the ghost rows)
    if (L.dist && !cheb) halo_exchange(c, *L.hp, NC, L.x2, L.gh_x);
    const GV gx = gv(L.x2, n, L.dist ? L.gh_x.p : nullptr);
    prof_begin(c, (mech ? PK_VC_POST_U : PK_VC_POST_P) + l0);
    if (gs) gs_sweep<NC>(c, L, true, b, L.x2, xout);                      // backward sweep
    else if (cheb) cheb_run<NC>(c, L, sym0, b, L.x2, xout, L.xc, false);
    else if (p70) p7_launch(c, 2, gv(L.dinv, n), gv(b, n), gx, xout, nullptr, ChebArgs{});
    else if (sym0) sym_vcycle_post(c, n, L.dinv, b, gx, xout);
    else if (wA) (L.dist ? csr_vec<NC, 2, true> : csr_vec<NC, 2, false>)(wA, c.s, n, L.A, gv(L.dinv, n), gv(b, n), gx, xout, nullptr, ChebArgs{});
    else if (n) (L.dist ? k_vc_post<NC, true> : k_vc_post<NC, false>)<<<grid_for(n, 256), 256, 0, c.s>>>(
        n, L.sA.off, L.sA.col, L.sA.val, L.dinv, b, gx, xout);
    prof_end(c, (mech ? PK_VC_POST_U : PK_VC_POST_P) + l0, gs ? gs_sweep_bytes(L, NC) : cheb ? deg * (bA0 + 5 * vec) : bA0 + 4 * vec);
    c.launches += 4;
}

void amg_vcycle(Ctx &c, Hier &H, const double *b, double *x, bool mech)
{
    if (mech) vcycle_rec<3>(c, H, 0, b, x);
    else vcycle_rec<1>(c, H, 0, b, x);
    TSP_CUDA(cudaGetLastError());
}

}  // namespace tsp

// krylov.cu -- rows a13/a14: right-preconditioned flexible GMRES(m)
// with classical Gram-Schmidt applied twice, the second pass DELAYED by one
// iteration (DCGS2, DESIGN.md R-krylov): iteration j holds v_0..v_{j-1} final and
// u_j once-orthogonalised; ONE pass over the basis computes [V_{j-1} u_j]^T [u_j w]
// (w = A M^-1 u_j), which both re-orthogonalises u_j into v_j (Pythagorean norm)
// and projects w; ONE fused pass then updates u_j -> v_j and w -> u_{j+1} (+ its
// norm).  Two basis passes per iteration instead of CGS2's three.  FGMRES keeps
// z_j = M^-1 u_j, so A Z = V H holds exactly with the Hessenberg column of step j-1
// completed at step j (H[:, j-1] += rho_{j-1} [s_j; alpha_j - 1 at row j]) and the
// last column completed by one extra projection of u_{k} at the end of the cycle.
//
// Deterministic reductions (R-reduce): every dot product is a sum of per-chunk
// partials (fixed chunks of the GLOBAL vector, halo.cu), each reduced by a fixed
// tree; the partials of all ranks are allgathered and summed in global chunk order,
// so the Hessenberg matrix -- hence the whole iteration -- is bitwise identical for
// any number of ranks.  Givens rotations and the small least-squares solve run on
// the host of every rank (identical data, identical control flow).
#include <cmath>
#include <vector>

#include "tsp_internal.cuh"

namespace tsp {

constexpr int KB = 256;        // threads per block for vector kernels
constexpr int KG = 8;          // vectors per multi-dot group

__device__ __forceinline__ double block_sum(double x, double *red)   // fixed tree over KB threads
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane == 0) red[wid] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int u = 0; u < KB / 32; ++u) s += red[u];
    return s;
}

// NV values per thread (NV a power of two <= 32) -> thread t < NV returns the block total of value t.
// Warp stage: transpose-reduce (log2 NV halving exchanges, NV-1 shuffles instead of 5 NV), after which
// lane L holds the warp total of value bitrev(L mod NV); then a fixed sum over the warps.
template <int NV>
__device__ __forceinline__ double block_sum_multi(double (&d)[NV], double (*red)[NV])
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int h = NV / 2, m = 1; h >= 1; h >>= 1, m <<= 1) {
        const bool up = lane & m;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double snd = up ? d[i] : d[i + h], kp = up ? d[i + h] : d[i];
            d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, m);
        }
    }
    double x = d[0];
#pragma unroll
    for (int o = NV; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    int idx = 0;
#pragma unroll
    for (int bit = 1, t = NV / 2; bit < NV; bit <<= 1, t >>= 1) if (lane & bit) idx |= t;
    if (lane < NV) red[wid][idx] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < NV)
        for (int u = 0; u < KB / 32; ++u) s += red[u][threadIdx.x];
    __syncthreads();
    return s;
}

// part[t*cmax + chunk] = sum_{r in chunk} V_t[r] w[r].  One block per chunk does every vector: the w
// chunk is staged once in shared memory, the vectors are streamed in groups of KG with the row loop
// unrolled by 2 (16 independent loads in flight per thread), then one fixed-tree block sum per vector.
__global__ void __launch_bounds__(KB) k_mdot(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ w,
                                             const int64_t *__restrict__ be, double *__restrict__ part, int cmax)
{
    __shared__ double ws[kRedChunk];
    __shared__ double red[KB / 32];
    const int k = blockIdx.x;
    const int64_t beg = be[2 * k];
    const int len = (int)(be[2 * k + 1] - beg);
    for (int i = threadIdx.x; i < len; i += KB) ws[i] = __ldcs(w + beg + i);
    __syncthreads();
    for (int v0 = 0; v0 < nv; v0 += KG) {
        const int cnt = min(KG, nv - v0);
        const double *Vg = V + v0 * ldv + beg;
        double acc[KG];
#pragma unroll
        for (int t = 0; t < KG; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + KB < len; i += 2 * KB) {
#pragma unroll
            for (int t = 0; t < KG; ++t)
                if (t < cnt) {
                    acc[t] = fma(__ldcs(Vg + t * ldv + i), ws[i], acc[t]);
                    acc[t] = fma(__ldcs(Vg + t * ldv + i + KB), ws[i + KB], acc[t]);
                }
        }
        for (; i < len; i += KB) {
#pragma unroll
            for (int t = 0; t < KG; ++t) if (t < cnt) acc[t] = fma(__ldcs(Vg + t * ldv + i), ws[i], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < KG; ++t)
            if (t < cnt) {
                const double s = block_sum(acc[t], red);
                if (threadIdx.x == 0) part[(int64_t)(v0 + t) * cmax + k] = s;
            }
    }
}

// DCGS2 pass 1: part[t] = V_t . u, part[nv + t] = V_t . w for t < nv (V_{nv-1} is u itself), per chunk.
// u and w chunks staged interleaved in shared memory (one 16-B load per row); KG2 vectors per group,
// rows unrolled by 2, both products share each V load.
#ifndef TSP_KG2
#define TSP_KG2 4
#endif
#ifndef TSP_MDOT2_MINB
#define TSP_MDOT2_MINB 1
#endif
constexpr int KG2 = TSP_KG2;
__global__ void __launch_bounds__(KB, TSP_MDOT2_MINB) k_mdot2(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ u,
                                              const double *__restrict__ w, const int64_t *__restrict__ be,
                                              double *__restrict__ part, int cmax)
{
    __shared__ double2 uw[kRedChunk];
    __shared__ double red[KB / 32][2 * KG2];
    const int k = blockIdx.x;
    const int64_t beg = be[2 * k];
    const int len = (int)(be[2 * k + 1] - beg);
    for (int i = threadIdx.x; i < len; i += KB) uw[i] = make_double2(__ldcs(u + beg + i), __ldcs(w + beg + i));
    __syncthreads();
    for (int v0 = 0; v0 < nv; v0 += KG2) {
        const int cnt = min(KG2, nv - v0);
        const double *Vg = V + v0 * ldv + beg;
        double acc[2 * KG2];
#pragma unroll
        for (int t = 0; t < 2 * KG2; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + KB < len; i += 2 * KB) {
            const double2 x0 = uw[i], x1 = uw[i + KB];
#pragma unroll
            for (int t = 0; t < KG2; ++t)
                if (t < cnt) {
                    const double va = __ldcs(Vg + t * ldv + i), vb = __ldcs(Vg + t * ldv + i + KB);
                    acc[t] = fma(va, x0.x, acc[t]); acc[t] = fma(vb, x1.x, acc[t]);
                    acc[KG2 + t] = fma(va, x0.y, acc[KG2 + t]); acc[KG2 + t] = fma(vb, x1.y, acc[KG2 + t]);
                }
        }
        for (; i < len; i += KB) {
            const double2 x0 = uw[i];
#pragma unroll
            for (int t = 0; t < KG2; ++t)
                if (t < cnt) {
                    const double va = __ldcs(Vg + t * ldv + i);
                    acc[t] = fma(va, x0.x, acc[t]);
                    acc[KG2 + t] = fma(va, x0.y, acc[KG2 + t]);
                }
        }
        const double s = block_sum_multi<2 * KG2>(acc, red);
        const int q = threadIdx.x;
        if (q < 2 * KG2 && (q % KG2) < cnt) part[(int64_t)((q < KG2 ? 0 : nv) + v0 + q % KG2) * cmax + k] = s;
    }
}

// ---- the same pass with its operands moved by the TMA bulk-copy engine (cp.async.bulk + mbarrier) ----
// One CTA per chunk as k_mdot2; one thread issues 1-D bulk copies of u and w (one each) and of the basis
// vectors in ITEMS of (group of KG2 vectors) x (half chunk of 1024 rows) into a two-slot shared-memory ring
// (slot = half), each slot completing an mbarrier by byte count; every thread waits on the slot's barrier
// (phase = group parity).  The copy engine keeps the next item in flight while the CTA multiplies and
// reduces the current one (k_mdot2 stalls on its own loads at every group's block reduction), and no
// thread spends issue slots on address arithmetic for the stream.  Each thread still accumulates its rows
// in the same order (tid, tid + 256, ...) and the same block_sum_multi<2 KG2> tree finishes every group:
// the result is BITWISE k_mdot2's.  Requirements (checked by the caller): V, u, w 16-byte aligned, ldv
// even; bulk copies start at the even row at or below the chunk start (off = 0 or 1 leading row) and end
// at the even row at or above its end, which stays inside the ld-padded basis columns.
constexpr int HR = kRedChunk / 2;         // rows per half chunk
constexpr int HS = HR + 2;                // half-chunk slot length in doubles (+ the odd-offset row, 16-B multiple)
constexpr int CS = kRedChunk + 2;         // u / w staging length
constexpr size_t kMdotTmaSmem = sizeof(double) * (2 * CS + 2 * KG2 * HS);

__global__ void __launch_bounds__(KB, 2) k_mdot2_tma(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ u,
                                                     const double *__restrict__ w, const int64_t *__restrict__ be,
                                                     double *__restrict__ part, int cmax)
{
    extern __shared__ __align__(128) double dsm[];
    double *uS = dsm, *wS = dsm + CS, *ring = dsm + 2 * CS;          // ring[h][t][HS]
    __shared__ __align__(8) uint64_t bar[3];                        // bar[h]: half h of the current group; bar[2]: u, w
    __shared__ double red[KB / 32][2 * KG2];
    const int k = blockIdx.x;
    const int64_t beg = be[2 * k];
    const int len = (int)(be[2 * k + 1] - beg);
    const int64_t a0 = beg & ~(int64_t)1;
    const int off = (int)(beg - a0);
    const int ngroups = (nv + KG2 - 1) / KG2;
    const int nh = len > HR ? 2 : 1;
    auto half_bytes = [&](int h) {                                   // bytes of one vector's copy of half h
        const int64_t r1 = beg + min(len, (h + 1) * HR);
        return (uint32_t)(8 * (((r1 + 1) & ~(int64_t)1) - (a0 + h * HR)));
    };
    auto issue = [&](int g, int h) {                                 // thread 0: item (group g, half h) -> slot h
        const int cnt = min(KG2, nv - g * KG2);
        const uint32_t nb = half_bytes(h);
        mbar_expect(&bar[h], nb * cnt);
        for (int t = 0; t < cnt; ++t)
            bulk_g2s(ring + (h * KG2 + t) * HS, V + (int64_t)(g * KG2 + t) * ldv + a0 + h * HR, nb, &bar[h]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nb = (uint32_t)(8 * (((beg + len + 1) & ~(int64_t)1) - a0));
        mbar_expect(&bar[2], 2 * nb);
        bulk_g2s(uS, u + a0, nb, &bar[2]);
        bulk_g2s(wS, w + a0, nb, &bar[2]);
        for (int h = 0; h < nh; ++h) issue(0, h);
    }
    mbar_wait(&bar[2], 0);
    for (int g = 0; g < ngroups; ++g) {
        const int v0 = g * KG2, cnt = min(KG2, nv - v0);
        double acc[2 * KG2];
#pragma unroll
        for (int t = 0; t < 2 * KG2; ++t) acc[t] = 0.0;
        for (int h = 0; h < nh; ++h) {
            mbar_wait(&bar[h], g & 1);
            const double *sl = ring + h * KG2 * HS + off - h * HR;
            const int r1 = min(len, (h + 1) * HR);
            for (int i = h * HR + threadIdx.x; i < r1; i += KB) {
                const double x = uS[off + i], y = wS[off + i];
#pragma unroll
                for (int t = 0; t < KG2; ++t)
                    if (t < cnt) {
                        const double va = sl[t * HS + i];
                        acc[t] = fma(va, x, acc[t]);
                        acc[KG2 + t] = fma(va, y, acc[KG2 + t]);
                    }
            }
            if (h == 0 && nh == 2) {                                 // slot 0 read by all: refill it
                __syncthreads();
                if (threadIdx.x == 0 && g + 1 < ngroups) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(g + 1, 0);
                }
            }
        }
        const double s = block_sum_multi<2 * KG2>(acc, red);          // its barriers: the last slot read by all
        if (threadIdx.x == 0 && g + 1 < ngroups) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (nh == 2) issue(g + 1, 1);
            else issue(g + 1, 0);
        }
        const int q = threadIdx.x;
        if (q < 2 * KG2 && (q % KG2) < cnt) part[(int64_t)((q < KG2 ? 0 : nv) + v0 + q % KG2) * cmax + k] = s;
    }
}

// DCGS2 scalars from the pass-1 dots d = [V_{j-1} u ; u.u | V_{j-1} w ; u.w] (2(j+1) values):
// s = d[0..j), gamma = d[j], a = d[j+1..2j+1), b = d[2j+1];
// alpha = sqrt(gamma - s.s) (norm of the re-orthogonalised u), h_j = (b - s.a) / alpha (= v_j . w).
// sc[0] = alpha, sc[1] = h_j.  When the Pythagorean difference loses more than 6 digits to cancellation
// (gamma - s.s <= 1e-6 gamma: u nearly inside span V) or is not finite, sc[0] = 0 flags the iteration for
// the explicit two-pass fallback on the host (k_dcgs_update then leaves u and w untouched).
constexpr double kPythagorasMin = 1e-6;
__global__ void k_dcgs_coef(int j, const double *__restrict__ d, double *__restrict__ sc, int force_fallback)
{
    if (threadIdx.x) return;
    double ss = 0.0, sa = 0.0;
    for (int t = 0; t < j; ++t) { ss = fma(d[t], d[t], ss); sa = fma(d[t], d[j + 1 + t], sa); }
    const double a2 = d[j] - ss;
    if (force_fallback || !(a2 > kPythagorasMin * d[j]) || !isfinite(a2)) { sc[0] = 0.0; sc[1] = 0.0; return; }
    const double alpha = sqrt(a2);
    sc[0] = alpha;
    sc[1] = (d[2 * j + 1] - sa) / alpha;
}

// w -= sum_t h[t] V_t (t < nv): the explicit Gram-Schmidt subtraction of the fallback
__global__ void __launch_bounds__(KB) k_gs_sub(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ h,
                                               double *__restrict__ w, int64_t n)
{
    __shared__ double hs[128];
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    for (int64_t r = blockIdx.x * (int64_t)KB + threadIdx.x; r < n; r += (int64_t)gridDim.x * KB) {
        double acc = 0.0;
        for (int t = 0; t < nv; ++t) acc = fma(hs[t], __ldcs(V + t * ldv + r), acc);
        w[r] -= acc;
    }
}

// DCGS2 pass 2 (fused): v_j = (u - V_{j-1} s) / alpha (in place of u); w <- w - V_{j-1} a - h_j v_j;
// part[chunk] = sum w^2.  8 independent basis loads in flight per row, both sums share them.
__global__ void __launch_bounds__(KB) k_dcgs_update(int j, const double *__restrict__ V, int64_t ldv,
                                                    const double *__restrict__ d, const double *__restrict__ sc,
                                                    double *__restrict__ u, double *__restrict__ w,
                                                    const int64_t *__restrict__ be, double *__restrict__ part)
{
    constexpr int UL = 8;
    __shared__ double ss[128], as[128];
    __shared__ double red[KB / 32];
    const int k = blockIdx.x;
    const int64_t beg = be[2 * k], end = be[2 * k + 1];
    const double alpha = sc[0], hj = sc[1];
    if (alpha == 0.0) {                                    // fallback flagged by k_dcgs_coef: touch nothing
        if (threadIdx.x == 0) part[k] = 0.0;
        return;
    }
    for (int t = threadIdx.x; t < j; t += KB) { ss[t] = d[t]; as[t] = d[j + 1 + t]; }
    __syncthreads();
    double nrm = 0.0;
    for (int64_t r = beg + threadIdx.x; r < end; r += KB) {
        double su = 0.0, sa = 0.0;
        const double ur = u[r], wr = w[r];                 // in flight with the first basis loads
        int t = 0;
        for (; t + UL <= j; t += UL) {
            double vv[UL];
#pragma unroll
            for (int q = 0; q < UL; ++q) vv[q] = __ldcs(V + (t + q) * ldv + r);
#pragma unroll
            for (int q = 0; q < UL; ++q) { su = fma(ss[t + q], vv[q], su); sa = fma(as[t + q], vv[q], sa); }
        }
        if (t < j) {                                       // the last j % UL columns: loads issued together, same fma order
            double vv[UL];
#pragma unroll
            for (int q = 0; q < UL; ++q) vv[q] = t + q < j ? __ldcs(V + (t + q) * ldv + r) : 0.0;
#pragma unroll
            for (int q = 0; q < UL; ++q)
                if (t + q < j) { su = fma(ss[t + q], vv[q], su); sa = fma(as[t + q], vv[q], sa); }
        }
        const double v = (ur - su) / alpha;
        const double wn = (wr - sa) - hj * v;
        u[r] = v;
        w[r] = wn;
        nrm = fma(wn, wn, nrm);
    }
    const double s = block_sum(nrm, red);
    if (threadIdx.x == 0) part[k] = s;
}

// per-segment sums of the chunk partials, fixed tree: segp[t*smax + s] = sum_{k in seg s} part[t*cmax + k]
__global__ void __launch_bounds__(KB) k_seg_reduce(const double *__restrict__ part, int cmax, const int32_t *__restrict__ segc,
                                                   double *__restrict__ segp, int smax)
{
    const int sg = blockIdx.x, t = blockIdx.y;
    const int k0 = segc[sg], k1 = segc[sg + 1];
    double x = 0.0;
    for (int k = k0 + threadIdx.x; k < k1; k += KB) x += part[(int64_t)t * cmax + k];
    __shared__ double red[KB / 32];
    const double s = block_sum(x, red);
    if (threadIdx.x == 0) segp[(int64_t)t * smax + sg] = s;
}

// out[t] = (sqrt of) the sum over the global segments, in global order, of the allgathered
// segment sums; seg_all layout [rank][nv][smax], perm[g] = rank * smax + local segment
__global__ void k_final(int nv, const double *__restrict__ seg_all, int smax, const int32_t *__restrict__ perm, int nglob,
                        double *__restrict__ out, int mode)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nv) return;
    double s = 0.0;
    for (int g = 0; g < nglob; ++g) {
        const int slot = perm[g], r = slot / smax, k = slot - r * smax;
        s += seg_all[((int64_t)r * nv + t) * smax + k];
    }
    if (mode == 0) out[t] = s;
    else out[t] = sqrt(s);
}

// x += Z y
__global__ void __launch_bounds__(KB) k_update(int64_t n, int k, const double *__restrict__ Z, int64_t ldz,
                                               const double *__restrict__ y, double *__restrict__ x)
{
    __shared__ double ys[128];
    for (int t = threadIdx.x; t < k; t += KB) ys[t] = y[t];
    __syncthreads();
    for (int64_t r = blockIdx.x * (int64_t)KB + threadIdx.x; r < n; r += (int64_t)gridDim.x * KB) {
        double acc = x[r];
        int t = 0;
        for (; t + 8 <= k; t += 8) {
            double zz[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) zz[u] = __ldcs(Z + (t + u) * ldz + r);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = fma(ys[t + u], zz[u], acc);
        }
        for (; t < k; ++t) acc = fma(ys[t], __ldcs(Z + t * ldz + r), acc);
        x[r] = acc;
    }
}
// y = x / *s (nothing when *s == 0: a lucky breakdown leaves w as it is)
__global__ void k_scale_inv(int64_t n, const double *__restrict__ s, const double *__restrict__ x, double *__restrict__ y)
{
    if (*s == 0.0) return;
    const double a = 1.0 / *s;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) y[r] = a * x[r];
}
// r = b - r
__global__ void k_bminus(int64_t n, const double *__restrict__ b, double *__restrict__ r)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) r[i] = b[i] - r[i];
}

struct Kr {
    Ctx &c;
    int64_t n, ld;                    // basis vectors are ld = n rounded up to 32 apart (256-B aligned)
    int nblk;
    double bytes = 0;                 // algorithmic bytes of the Krylov kernels (tsp_solve_info.bytes_krylov)
    int force_fallback = 0;           // test knob TSP_DCGS2_FALLBACK: every iteration takes the explicit path
    bool tma = true;                  // pass 1 by k_mdot2_tma (test knob TSP_NO_TMA, read per solve: k_mdot2)
    DBuf<double> pall;
    Kr(Ctx &c_, int maxv) : c(c_), n(c_.n), ld((c_.n + 31) & ~(int64_t)31)
    {
        nblk = (int)std::max<int64_t>(1, std::min<int64_t>((n + KB - 1) / KB, (int64_t)c.sm_count * 4));
        pall.alloc((size_t)std::max(c.nranks, 1) * maxv * std::max(c.nseg_max, 1) + 16);
        static const bool smem_ok =
            cudaFuncSetAttribute(k_mdot2_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMdotTmaSmem) == cudaSuccess;
        tma = smem_ok && getenv("TSP_NO_TMA") == nullptr;
    }
    // chunk partials `kpart` ([nv][nchunk_loc]) -> segment sums -> (allgather) -> out[nv]
    void finish(int nv, double *out, int mode)
    {
        if (c.nseg_loc) {
            dim3 g(c.nseg_loc, nv);
            k_seg_reduce<<<g, KB, 0, c.s>>>(c.kpart, c.nchunk_loc, c.seg_chunk, c.seg_part, c.nseg_max);
        }
        const double *src = c.seg_part;
        if (c.comm) {
            c.comm->allgather(c.seg_part.p, pall.p, sizeof(double) * nv * c.nseg_max, c.s);
            src = pall;
        }
        k_final<<<(nv + 63) / 64, 64, 0, c.s>>>(nv, src, c.nseg_max, c.seg_perm, c.nseg_glob, out, mode);
        c.launches += 2;
    }
    void mdot(const double *V, int nv, const double *w, double *h)
    {
        prof_begin(c, PK_DOT);
        k_mdot<<<c.nchunk_loc, KB, 0, c.s>>>(nv, V, ld, w, c.chunk_beg, c.kpart, c.nchunk_loc);
        finish(nv, h, 0);
        prof_end(c, PK_DOT, 8.0 * n * (nv + 1));
        bytes += 8.0 * n * (nv + 1);
        c.launches++;
    }
    // pass 1: d = [V_0..V_j]^T [u_j, w] (V_j = u_j), then alpha / h_j into sc
    void mdot2(const double *V, int j, const double *w, double *d, double *sc)
    {
        prof_begin(c, PK_DOT);
        // bulk copies: basis columns 16-B aligned (cudaMalloc base, ld a multiple of 32)
        if (tma && ((uintptr_t)V & 15) == 0 && (ld & 1) == 0 && ((uintptr_t)w & 15) == 0)
            k_mdot2_tma<<<c.nchunk_loc, KB, kMdotTmaSmem, c.s>>>(j + 1, V, ld, V + (size_t)j * ld, w, c.chunk_beg, c.kpart,
                                                                 c.nchunk_loc);
        else
            k_mdot2<<<c.nchunk_loc, KB, 0, c.s>>>(j + 1, V, ld, V + (size_t)j * ld, w, c.chunk_beg, c.kpart, c.nchunk_loc);
        finish(2 * (j + 1), d, 0);
        k_dcgs_coef<<<1, 32, 0, c.s>>>(j, d, sc, force_fallback);
        prof_end(c, PK_DOT, 8.0 * n * (j + 2));
        bytes += 8.0 * n * (j + 2);
        c.launches += 2;
    }
    // pass 2: v_j = (u_j - V s)/alpha, w -= V a + h_j v_j, rho = ||w||
    void dcgs_update(const double *V, int j, const double *d, const double *sc, double *w, double *rho)
    {
        prof_begin(c, PK_AXPY);
        k_dcgs_update<<<c.nchunk_loc, KB, 0, c.s>>>(j, V, ld, d, sc, (double *)V + (size_t)j * ld, w, c.chunk_beg, c.kpart);
        finish(1, rho, 2);
        prof_end(c, PK_AXPY, 8.0 * n * (j + 4));
        bytes += 8.0 * n * (j + 4);
        c.launches++;
    }
    // w -= V_{0..nv-1} h (h on the device)
    void gs_sub(const double *V, int nv, const double *h, double *w)
    {
        prof_begin(c, PK_AXPY);
        k_gs_sub<<<nblk, KB, 0, c.s>>>(nv, V, ld, h, w, n);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        bytes += 8.0 * n * (nv + 2);
        c.launches++;
    }
    void norm(const double *w, double *nrm)
    {
        prof_begin(c, PK_NORM);
        k_mdot<<<c.nchunk_loc, KB, 0, c.s>>>(1, w, ld, w, c.chunk_beg, c.kpart, c.nchunk_loc);
        finish(1, nrm, 2);
        prof_end(c, PK_NORM, 8.0 * n);
        bytes += 8.0 * n;
        c.launches++;
    }
    void scale_inv(const double *s, const double *x, double *y)
    {
        prof_begin(c, PK_VEC);
        k_scale_inv<<<nblk, KB, 0, c.s>>>(n, s, x, y);
        prof_end(c, PK_VEC, 16.0 * n);
        bytes += 16.0 * n;
        c.launches++;
    }
};

// Hessenberg bookkeeping on the host: raw columns (completed one step late, see the header),
// their Givens-rotated copies and the rotated right-hand side g.  gin[i] is g[i] before
// rotation i, so a column whose rotation changes can be re-rotated exactly.
struct Hess {
    int m;
    std::vector<std::vector<double>> raw, rot;
    std::vector<double> cs, sn, g, gin;
    explicit Hess(int m_) : m(m_), raw(m_), rot(m_), cs(m_), sn(m_), g(m_ + 1), gin(m_ + 1) {}
    void reset(double beta)
    {
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = gin[0] = beta;
    }
    // (re)compute the rotation of column i from its raw entries and rotations 0..i-1
    void rotate(int i)
    {
        std::vector<double> R = raw[i];
        for (int t = 0; t < i; ++t) {
            const double a = R[t], b = R[t + 1];
            R[t] = cs[t] * a + sn[t] * b;
            R[t + 1] = -sn[t] * a + cs[t] * b;
        }
        const double rho = std::hypot(R[i], R[i + 1]);
        cs[i] = R[i] / rho; sn[i] = R[i + 1] / rho;
        R[i] = rho; R[i + 1] = 0.0;
        rot[i] = R;
        g[i] = cs[i] * gin[i];
        g[i + 1] = -sn[i] * gin[i];
        gin[i + 1] = g[i + 1];
    }
    // complete column i with the delayed re-orthogonalisation of u_{i+1}: u_{i+1} = alpha v_{i+1} + V s
    void complete(int i, double rho, const double *s, double alpha)
    {
        for (int t = 0; t <= i; ++t) raw[i][t] += rho * s[t];
        raw[i][i + 1] = rho * alpha;
        rotate(i);
    }
};

void krylov_graphs_drop(Ctx &c)
{
    for (auto &g : c.kgraph)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    c.kgraph.assign(c.kgraph.size(), Ctx::KGraph{});
}

// Iteration j's body: eager the first time (one-time attribute settings happen there), then captured into a
// graph and replayed -- ~70 dependent launches per iteration become one, which is what bounds small problems.
template <class F>
static void run_body(Ctx &c, Kr &K, int j, bool use_graph, F &body)
{
    if (!use_graph || j >= (int)c.kgraph.size()) { body(); return; }
    auto &G = c.kgraph[j];
    if (!G.exec && !G.seen) { body(); G.seen = true; return; }
    if (G.failed) { body(); return; }
    if (!G.exec) {
        const int64_t l0 = c.launches;
        const double b0 = K.bytes;
        cudaGraph_t graph = nullptr;
        // capture on a private stream (the API stream may be the legacy default stream, which cannot capture);
        // the body launches on c.s, so c.s points at it meanwhile
        if (!c.cap_stream) TSP_CUDA(cudaStreamCreateWithFlags(&c.cap_stream, cudaStreamNonBlocking));
        // the capture is ended and c.s restored on every exit path, exceptions included
        struct CaptureScope {
            Ctx &c; cudaStream_t api; bool open = false;
            ~CaptureScope()
            {
                if (open) { cudaGraph_t g = nullptr; cudaStreamEndCapture(c.s, &g); if (g) cudaGraphDestroy(g); (void)cudaGetLastError(); }
                c.s = api;
            }
        } scope{c, c.s};
        c.s = c.cap_stream;
        TSP_CUDA(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
        scope.open = true;
        try {
            body();
        } catch (const Error &e) {                  // not capturable here: end the capture, run eagerly from now on
            cudaStreamEndCapture(c.s, &graph);
            scope.open = false;
            c.s = scope.api;
            if (graph) cudaGraphDestroy(graph);
            (void)cudaGetLastError();
            if (getenv("TSP_DEBUG")) fprintf(stderr, "[tsp graph] capture of iteration %d failed: %s\n", j, e.msg.c_str());
            G.failed = true;
            c.launches = l0; K.bytes = b0;
            body();
            return;
        }
        const cudaError_t ec = cudaStreamEndCapture(c.s, &graph);
        scope.open = false;
        c.s = scope.api;
        TSP_CUDA(ec);
        TSP_CUDA(cudaGraphInstantiate(&G.exec, graph, 0));
        cudaGraphDestroy(graph);
        G.launches = c.launches - l0;
        G.bytes = K.bytes - b0;
        c.launches = l0; K.bytes = b0;
    }
    TSP_CUDA(cudaGraphLaunch(G.exec, c.s));
    c.launches += G.launches;
    K.bytes += G.bytes;
}

// the solver workspace of restart length m: basis V (m + 1 columns), Z (m), residual, scalars, reduction partials
static void krylov_reserve(Ctx &c, int m)
{
    const int64_t n = c.n, ld = (n + 31) & ~(int64_t)31;
    if (c.kcap == m && c.V.n == (size_t)(m + 1) * ld) return;
    krylov_graphs_drop(c);
    c.V.alloc((size_t)(m + 1) * ld);
    c.Z.alloc((size_t)m * ld);
    c.kr.alloc(std::max<int64_t>(n, 1));
    c.kh.alloc(5 * (m + 2) + 16);
    c.kpart.alloc((size_t)2 * (m + 2) * std::max(c.nchunk_loc, 1) + 64);
    c.seg_part.alloc((size_t)2 * (m + 2) * std::max(c.nseg_max, 1) + 64);
    c.kcap = m;
}

// x += z
__global__ void k_xpz(int64_t n, const double *__restrict__ z, double *__restrict__ x)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = x[i] + z[i];
}

// The "sequential" embedding of the remark at P:640-642 (SURVEY NEXT-f4 iii): stationary Richardson iteration
// x <- x + M^-1 (b - A x) with Algorithm 1 as M^-1, from x0 (zero if o.x0_zero), stopped on the TRUE residual
// ||b - A x|| <= rtol ||b||, after max_iters preconditioner applications, or on a non-finite residual norm
// (TSP_ERR_NUMERIC, x = the last finite iterate's successor as computed).  Per iteration: the operator, r = b - r,
// one norm (allgathered over the ranks), Algorithm 1, x += z -- the FGMRES kernels, no basis.
void richardson_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info)
{
    const int64_t n = c.n;
    krylov_reserve(c, c.kcap > 0 ? c.kcap : 1);
    Kr K(c, 4);
    double *r = c.kr, *z = c.Z, *dh = c.kh;
    struct Events {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        ~Events() { if (e0) cudaEventDestroy(e0); if (e1) cudaEventDestroy(e1); }
    } ev;
    TSP_CUDA(cudaEventCreate(&ev.e0)); TSP_CUDA(cudaEventCreate(&ev.e1));
    TSP_CUDA(cudaEventRecord(ev.e0, c.s));
    double bn;
    K.norm(b, dh);
    TSP_CUDA(cudaMemcpyAsync(&bn, dh, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    TSP_REQUIRE(std::isfinite(bn), TSP_ERR_NUMERIC, "non-finite ||b||");
    if (o.x0_zero && n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
    int it = 0, status = TSP_NOT_CONVERGED;
    for (;;) {
        op_apply(c, x, r);
        k_bminus<<<K.nblk, KB, 0, c.s>>>(n, b, r);
        c.launches++;
        K.norm(r, dh);
        double rn;
        TSP_CUDA(cudaMemcpyAsync(&rn, dh, sizeof(double), cudaMemcpyDeviceToHost, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
        info.true_relres = bn > 0.0 ? rn / bn : 0.0;
        info.est_relres = info.true_relres;
        if (rn <= o.rtol * bn) { status = TSP_OK; break; }
        if (!std::isfinite(rn)) { status = TSP_ERR_NUMERIC; break; }
        if (it >= o.max_iters) { status = TSP_NOT_CONVERGED; break; }
        prec_apply(c, r, z);
        prof_begin(c, PK_VEC);
        k_xpz<<<K.nblk, KB, 0, c.s>>>(n, z, x);
        prof_end(c, PK_VEC, 24.0 * n);
        K.bytes += 24.0 * n;
        c.launches++;
        ++it;
    }
    TSP_CUDA(cudaEventRecord(ev.e1, c.s));
    TSP_CUDA(cudaEventSynchronize(ev.e1));
    float ms = 0;
    TSP_CUDA(cudaEventElapsedTime(&ms, ev.e0, ev.e1));
    info.iterations = it;
    info.restarts = 0;
    info.status = status;
    info.t_solve_s = ms * 1e-3;
    info.bytes_krylov = K.bytes;
}

void krylov_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info)
{
    const int m = std::max(1, std::min(o.restart, 120));
    const int64_t n = c.n, ld = (n + 31) & ~(int64_t)31;
    krylov_reserve(c, m);
    Kr K(c, 2 * (m + 2));
    double *V = c.V, *Z = c.Z, *r = c.kr;
    // device scalars: d = pass-1 dots [0, 2(j+1)), then alpha, h_j, rho right behind them
    double *dh = c.kh;
    struct Events {                                  // destroyed on every exit path
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        ~Events() { if (e0) cudaEventDestroy(e0); if (e1) cudaEventDestroy(e1); }
    } ev;
    TSP_CUDA(cudaEventCreate(&ev.e0)); TSP_CUDA(cudaEventCreate(&ev.e1));
    cudaEvent_t e0 = ev.e0, e1 = ev.e1;
    TSP_CUDA(cudaEventRecord(e0, c.s));

    Hess H(m);
    std::vector<double> yv(m), col(2 * (m + 2) + 8);
    if (!c.kcol_host) TSP_CUDA(cudaMallocHost((void **)&c.kcol_host, sizeof(double) * (2 * (120 + 2) + 8)));
    if ((int)c.kgraph.size() != m) { krylov_graphs_drop(c); c.kgraph.resize(m); }
    // CUDA graphs for the iteration body: one rank, no profiling (its events are per launch)
    const bool no_graph = getenv("TSP_NO_GRAPH") != nullptr;
    // sharded handles: only on request (TSP_NCCL_GRAPH=1) and only over a transport whose calls are pure stream
    // work (NCCL; the halo overlap's comm stream forks from and rejoins the capturing stream through its two
    // events).  Off by default: this build had one GPU, so the captured NCCL iteration was never executed.
    const bool comm_graph = c.comm && c.comm->capturable() && getenv("TSP_NCCL_GRAPH") != nullptr;
    const bool use_graph = (!c.comm || comm_graph) && !c.prof.on && !no_graph;
    const bool no_fuse = getenv("TSP_NO_OP_FUSE") != nullptr;   // test knob (read per solve): the full operator every iteration
    double bn;
    K.norm(b, dh);
    TSP_CUDA(cudaMemcpyAsync(&bn, dh, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    TSP_REQUIRE(std::isfinite(bn), TSP_ERR_NUMERIC, "non-finite ||b||");
    if (o.x0_zero && n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
    int it = 0, status = TSP_NOT_CONVERGED;
    info.restarts = 0; info.est_relres = 0; info.true_relres = 0; info.reorth = 0; info.dcgs_fallbacks = 0;
    K.force_fallback = getenv("TSP_DCGS2_FALLBACK") != nullptr;
    if (bn == 0.0) {
        if (n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
        status = TSP_OK;
    } else {
        for (;;) {
            op_apply(c, x, r);                         // r = b - A x ; beta = ||r||
            k_bminus<<<K.nblk, KB, 0, c.s>>>(n, b, r);
            c.launches++;
            K.norm(r, dh);
            double beta;
            TSP_CUDA(cudaMemcpyAsync(&beta, dh, sizeof(double), cudaMemcpyDeviceToHost, c.s));
            TSP_CUDA(cudaStreamSynchronize(c.s));
            TSP_REQUIRE(std::isfinite(beta), TSP_ERR_NUMERIC, "non-finite residual norm");
            info.true_relres = beta / bn;
            if (beta <= o.rtol * bn) { status = TSP_OK; break; }
            if (it >= o.max_iters) { status = TSP_NOT_CONVERGED; break; }
            if (it > 0) info.restarts++;
            K.scale_inv(dh, r, V);                     // u_0 = r / beta
            H.reset(beta);
            int k = 0;
            double rho_prev = 0.0;
            bool lucky = false;
            for (int j = 0; j < m; ++j) {
                double *uj = V + (size_t)j * ld, *zj = Z + (size_t)j * ld, *w = V + (size_t)(j + 1) * ld;
                double *d = dh, *sc = dh + 2 * (j + 1), *rho = sc + 2;
                // the iteration body: device work only, ending with the scalars copied to pinned host memory
                auto body = [&]() {
                    prec_apply(c, uj, zj);                 // z_j = M^-1 u_j (Algorithm 1)
                    if (no_fuse) op_apply(c, zj, w);       // w = A z_j
                    else op_apply_after_prec(c, uj, zj, w);   // (A_fu z_u reused from Algorithm 1's step 2)
                    K.mdot2(V, j, w, d, sc);               // [V_{j-1} u_j]^T [u_j w], alpha_j, h_j
                    K.dcgs_update(V, j, d, sc, w, rho);    // v_j, w -> w - V_j h, rho = ||w||
                    K.scale_inv(rho, w, w);                // u_{j+1} = w / rho (skipped when rho == 0)
                    TSP_CUDA(cudaMemcpyAsync(c.kcol_host, dh, sizeof(double) * (2 * (j + 1) + 3), cudaMemcpyDeviceToHost, c.s));
                };
                run_body(c, K, j, use_graph, body);
                TSP_CUDA(cudaStreamSynchronize(c.s));
                const double *dd = c.kcol_host;
                double alpha = dd[2 * (j + 1)], hj = dd[2 * (j + 1) + 1], rj = dd[2 * (j + 1) + 2];
                TSP_REQUIRE(std::isfinite(alpha) && std::isfinite(hj) && std::isfinite(rj), TSP_ERR_NUMERIC,
                            "non-finite Arnoldi coefficients");
                std::vector<double> s_j(dd, dd + j), a_j(dd + j + 1, dd + 2 * j + 1);
                if (alpha == 0.0) {
                    // k_dcgs_coef flagged the Pythagorean norm (u_j nearly inside span V, or the test knob): u_j
                    // and w are untouched.  Explicit two-pass path: v_j = (u_j - V s)/||u_j - V s||, then
                    // classical Gram-Schmidt of w against V_0..V_j applied twice, rho = ||w||.
                    info.dcgs_fallbacks++;
                    double *fb = dh + 4 * (m + 2) + 8;       // device scratch of m + 2 values
                    double host[2 * (120 + 2)];
                    K.gs_sub(V, j, dh, uj);                   // dh[0..j) = s
                    K.norm(uj, fb);
                    TSP_CUDA(cudaMemcpyAsync(host, fb, sizeof(double), cudaMemcpyDeviceToHost, c.s));
                    TSP_CUDA(cudaStreamSynchronize(c.s));
                    alpha = host[0];
                    TSP_REQUIRE(alpha > 0.0 && std::isfinite(alpha), TSP_ERR_NUMERIC, "Arnoldi vector inside the Krylov basis");
                    K.scale_inv(fb, uj, uj);
                    std::vector<double> h(j + 1, 0.0);
                    for (int pass = 0; pass < 2; ++pass) {
                        K.mdot(V, j + 1, w, fb);
                        K.gs_sub(V, j + 1, fb, w);
                        TSP_CUDA(cudaMemcpyAsync(host, fb, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, c.s));
                        TSP_CUDA(cudaStreamSynchronize(c.s));
                        for (int t = 0; t <= j; ++t) h[t] += host[t];
                    }
                    K.norm(w, fb);
                    K.scale_inv(fb, w, w);
                    TSP_CUDA(cudaMemcpyAsync(host, fb, sizeof(double), cudaMemcpyDeviceToHost, c.s));
                    TSP_CUDA(cudaStreamSynchronize(c.s));
                    rj = host[0];
                    TSP_REQUIRE(std::isfinite(rj), TSP_ERR_NUMERIC, "non-finite Arnoldi norm");
                    for (int t = 0; t < j; ++t) a_j[t] = h[t];
                    hj = h[j];
                }
                info.reorth++;
                if (j > 0) H.complete(j - 1, rho_prev, s_j.data(), alpha);   // column j-1 now exact
                else {                                                  // u_0 = r/beta: v_0 = u_0/alpha
                    H.g[0] = H.gin[0] = beta * alpha;
                }
                H.raw[j].assign(j + 2, 0.0);
                for (int t = 0; t < j; ++t) H.raw[j][t] = a_j[t];
                H.raw[j][j] = hj;
                H.raw[j][j + 1] = rj;                  // provisional: u_{j+1} taken as v_{j+1}
                H.rotate(j);
                rho_prev = rj;
                ++it; k = j + 1;
                info.est_relres = std::fabs(H.g[j + 1]) / bn;
                if (rj == 0.0) { lucky = true; break; }
                if (std::fabs(H.g[j + 1]) <= o.rtol * bn || it >= o.max_iters) break;
            }
            // complete the last column: one projection of u_k against V_0..V_{k-1} (+ u_k . u_k)
            if (!lucky) {
                K.mdot(V, k + 1, V + (size_t)k * ld, dh);
                TSP_CUDA(cudaMemcpyAsync(col.data(), dh, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, c.s));
                TSP_CUDA(cudaStreamSynchronize(c.s));
                double ss = 0.0;
                for (int t = 0; t < k; ++t) ss = std::fma(col[t], col[t], ss);
                double a2 = col[k] - ss;
                if (!(a2 > 1e-6 * col[k]) || K.force_fallback) {      // explicit norm of u_k - V s (see above)
                    info.dcgs_fallbacks++;
                    double *fb = dh + 4 * (m + 2) + 8;
                    double *uk = V + (size_t)k * ld;
                    K.gs_sub(V, k, dh, uk);
                    K.norm(uk, fb);
                    double an;
                    TSP_CUDA(cudaMemcpyAsync(&an, fb, sizeof(double), cudaMemcpyDeviceToHost, c.s));
                    TSP_CUDA(cudaStreamSynchronize(c.s));
                    a2 = an * an;
                }
                TSP_REQUIRE(a2 > 0.0 && std::isfinite(a2), TSP_ERR_NUMERIC, "loss of orthogonality in the last Arnoldi vector");
                H.complete(k - 1, rho_prev, col.data(), std::sqrt(a2));
                info.est_relres = std::fabs(H.g[k]) / bn;
            }
            for (int i = k - 1; i >= 0; --i) {
                double sacc = H.g[i];
                for (int t = i + 1; t < k; ++t) sacc -= H.rot[t][i] * yv[t];
                yv[i] = sacc / H.rot[i][i];
            }
            double *dy = dh + 2 * (m + 2) + 4;
            TSP_CUDA(cudaMemcpyAsync(dy, yv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
            prof_begin(c, PK_AXPY);
            k_update<<<K.nblk, KB, 0, c.s>>>(n, k, Z, ld, dy, x);
            prof_end(c, PK_AXPY, 8.0 * n * (k + 2));
            K.bytes += 8.0 * n * (k + 2);
            c.launches++;
        }
    }
    TSP_CUDA(cudaEventRecord(e1, c.s));
    TSP_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    TSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    info.iterations = it;
    info.status = status;
    info.t_solve_s = ms * 1e-3;
    info.bytes_krylov = K.bytes;
}

}  // namespace tsp

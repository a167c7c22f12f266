// krylov.cu -- rows a13/a14: right-preconditioned flexible GMRES(m)
// with classical Gram-Schmidt applied twice (CGS2, DESIGN.md R-krylov).
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

// CGS2 pass-1 update fused with the pass-2 projections: w -= V h ; part[t] = V_t . w (per chunk).
// Per 256-row slab: thread-per-row update (UL independent loads in flight), the updated slab staged in
// shared memory, then warp `wid` takes vectors t = wid + 8q and re-reads its slab rows (L1/L2-resident,
// just streamed by the update) into per-lane partials; one warp tree per vector at the end of the chunk.
template <int MAXQ>
__global__ void __launch_bounds__(KB) k_maxpy_mdot(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ h,
                                                   double *__restrict__ w, const int64_t *__restrict__ be,
                                                   double *__restrict__ part, int cmax)
{
    constexpr int UL = 4;
    __shared__ double hs[128];
    __shared__ double ws[KB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = blockIdx.x;
    const int64_t beg = be[2 * k], end = be[2 * k + 1];
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    double p[MAXQ];
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) p[q] = 0.0;
    for (int64_t r0 = beg; r0 < end; r0 += KB) {
        const int64_t r = r0 + threadIdx.x;
        double acc = 0.0;
        if (r < end) {
            acc = w[r];
            int t = 0;
            for (; t + UL <= nv; t += UL) {
                double vv[UL];
#pragma unroll
                for (int u = 0; u < UL; ++u) vv[u] = V[(t + u) * ldv + r];
#pragma unroll
                for (int u = 0; u < UL; ++u) acc = fma(-hs[t + u], vv[u], acc);
            }
            for (; t < nv; ++t) acc = fma(-hs[t], V[t * ldv + r], acc);
            w[r] = acc;
        }
        ws[threadIdx.x] = acc;
        __syncthreads();
        const int m = (int)min((int64_t)KB, end - r0);
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
            const int t = wid + 8 * q;
            if (t < nv) {
                const double *vt = V + t * ldv + r0;
                if (m == KB) {
#pragma unroll
                    for (int e = 0; e < KB / 32; ++e) p[q] = fma(vt[lane + 32 * e], ws[lane + 32 * e], p[q]);
                } else {
                    for (int e = lane; e < m; e += 32) p[q] = fma(vt[e], ws[e], p[q]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
        const int t = wid + 8 * q;
        if (t < nv) {
            double x = p[q];
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) part[(int64_t)t * cmax + k] = x;
        }
    }
}

// w -= V h and the per-chunk partial of ||w||^2 (8 independent loads in flight per row)
__global__ void __launch_bounds__(KB) k_maxpy_norm(int nv, const double *__restrict__ V, int64_t ldv, const double *__restrict__ h,
                                                   double *__restrict__ w, const int64_t *__restrict__ be,
                                                   double *__restrict__ part)
{
    constexpr int UL = 8;
    __shared__ double hs[128];
    __shared__ double red[KB / 32];
    const int k = blockIdx.x;
    const int64_t beg = be[2 * k], end = be[2 * k + 1];
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    double nrm = 0.0;
    for (int64_t r = beg + threadIdx.x; r < end; r += KB) {
        double acc = w[r];
        int t = 0;
        for (; t + UL <= nv; t += UL) {
            double vv[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) vv[u] = __ldcs(V + (t + u) * ldv + r);
#pragma unroll
            for (int u = 0; u < UL; ++u) acc = fma(-hs[t + u], vv[u], acc);
        }
        for (; t < nv; ++t) acc = fma(-hs[t], __ldcs(V + t * ldv + r), acc);
        w[r] = acc;
        nrm = fma(acc, acc, nrm);
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
// y = x / *s
__global__ void k_scale_inv(int64_t n, const double *__restrict__ s, const double *__restrict__ x, double *__restrict__ y)
{
    const double a = 1.0 / *s;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) y[r] = a * x[r];
}
// r = b - r
__global__ void k_bminus(int64_t n, const double *__restrict__ b, double *__restrict__ r)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) r[i] = b[i] - r[i];
}
__global__ void k_add_into(int nv, const double *__restrict__ a, double *__restrict__ b) { int i = threadIdx.x; if (i < nv) b[i] += a[i]; }

struct Kr {
    Ctx &c;
    int64_t n, ld;                    // basis vectors are ld = n rounded up to 32 apart (256-B aligned)
    int nblk;
    DBuf<double> pall;
    Kr(Ctx &c_, int maxv) : c(c_), n(c_.n), ld((c_.n + 31) & ~(int64_t)31)
    {
        nblk = (int)std::max<int64_t>(1, std::min<int64_t>((n + KB - 1) / KB, (int64_t)c.sm_count * 4));
        pall.alloc((size_t)std::max(c.nranks, 1) * maxv * std::max(c.nseg_max, 1) + 16);
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
        c.launches++;
    }
    void maxpy_mdot(const double *V, int nv, const double *h1, double *w, double *h2)
    {
        prof_begin(c, PK_AXPY);
        (nv <= 64 ? k_maxpy_mdot<8> : k_maxpy_mdot<16>)<<<c.nchunk_loc, KB, 0, c.s>>>(nv, V, ld, h1, w, c.chunk_beg, c.kpart,
                                                                                        c.nchunk_loc);
        finish(nv, h2, 0);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        c.launches++;
    }
    void maxpy_norm(const double *V, int nv, const double *h, double *w, double *nrm)
    {
        prof_begin(c, PK_AXPY);
        k_maxpy_norm<<<c.nchunk_loc, KB, 0, c.s>>>(nv, V, ld, h, w, c.chunk_beg, c.kpart);
        finish(1, nrm, 2);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        c.launches++;
    }
    void norm(const double *w, double *nrm)
    {
        prof_begin(c, PK_NORM);
        k_mdot<<<c.nchunk_loc, KB, 0, c.s>>>(1, w, ld, w, c.chunk_beg, c.kpart, c.nchunk_loc);
        finish(1, nrm, 2);
        prof_end(c, PK_NORM, 8.0 * n);
        c.launches++;
    }
    void scale_inv(const double *s, const double *x, double *y)
    {
        prof_begin(c, PK_VEC);
        k_scale_inv<<<nblk, KB, 0, c.s>>>(n, s, x, y);
        prof_end(c, PK_VEC, 16.0 * n);
        c.launches++;
    }
};

void krylov_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info)
{
    const int m = std::max(1, std::min(o.restart, 120));
    const int64_t n = c.n, ld = (n + 31) & ~(int64_t)31;
    if (c.kcap != m || c.V.n != (size_t)(m + 1) * ld) {
        c.V.alloc((size_t)(m + 1) * ld);
        c.Z.alloc((size_t)m * ld);
        c.kr.alloc(std::max<int64_t>(n, 1));
        c.kh.alloc(4 * (m + 2));
        c.kpart.alloc((size_t)(m + 2) * std::max(c.nchunk_loc, 1) + 64);
        c.seg_part.alloc((size_t)(m + 2) * std::max(c.nseg_max, 1) + 64);
        c.kcap = m;
    }
    Kr K(c, m + 2);
    double *V = c.V, *Z = c.Z, *r = c.kr;
    double *dh = c.kh;                // [0, m+2): h column; [m+2, 2m+4): second pass; then scalars
    double *dh2 = dh + (m + 2), *dsc = dh + 2 * (m + 2);
    cudaEvent_t e0, e1;
    TSP_CUDA(cudaEventCreate(&e0)); TSP_CUDA(cudaEventCreate(&e1));
    TSP_CUDA(cudaEventRecord(e0, c.s));

    std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), yv(m), col(m + 2);
    double bn;
    K.norm(b, dsc);
    TSP_CUDA(cudaMemcpyAsync(&bn, dsc, sizeof(double), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    TSP_REQUIRE(std::isfinite(bn), TSP_ERR_NUMERIC, "non-finite ||b||");
    if (o.x0_zero && n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
    int it = 0, status = TSP_NOT_CONVERGED;
    info.restarts = 0; info.est_relres = 0; info.true_relres = 0; info.reorth = 0;
    if (bn == 0.0) {
        if (n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
        status = TSP_OK;
    } else {
        for (;;) {
            op_apply(c, x, r);                         // r = b - A x ; beta = ||r||
            k_bminus<<<K.nblk, KB, 0, c.s>>>(n, b, r);
            c.launches++;
            K.norm(r, dsc);
            double beta;
            TSP_CUDA(cudaMemcpyAsync(&beta, dsc, sizeof(double), cudaMemcpyDeviceToHost, c.s));
            TSP_CUDA(cudaStreamSynchronize(c.s));
            TSP_REQUIRE(std::isfinite(beta), TSP_ERR_NUMERIC, "non-finite residual norm");
            info.true_relres = beta / bn;
            if (beta <= o.rtol * bn) { status = TSP_OK; break; }
            if (it >= o.max_iters) { status = TSP_NOT_CONVERGED; break; }
            if (it > 0) info.restarts++;
            K.scale_inv(dsc, r, V);
            std::fill(g.begin(), g.end(), 0.0);
            g[0] = beta;
            int k = 0;
            for (int j = 0; j < m; ++j) {
                double *vj = V + (size_t)j * ld, *zj = Z + (size_t)j * ld, *w = V + (size_t)(j + 1) * ld;
                prec_apply(c, vj, zj);                 // z_j = M^-1 v_j (Algorithm 1)
                op_apply(c, zj, w);                    // w = A z_j
                // CGS2 (DESIGN.md R-krylov).  A DGKS-selective second pass was measured to be needed
                // in 99% of the iterations here (the new direction is nearly in the Krylov space), so the
                // projection is always repeated; the first update is fused with the second projection.
                K.mdot(V, j + 1, w, dh);
                K.maxpy_mdot(V, j + 1, dh, w, dh2);
                K.maxpy_norm(V, j + 1, dh2, w, dh + j + 1);
                k_add_into<<<1, 128, 0, c.s>>>(j + 1, dh2, dh);
                c.launches++;
                info.reorth++;
                TSP_CUDA(cudaMemcpyAsync(col.data(), dh, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, c.s));
                TSP_CUDA(cudaStreamSynchronize(c.s));
                const double hn = col[j + 1];
                TSP_REQUIRE(std::isfinite(hn), TSP_ERR_NUMERIC, "non-finite Arnoldi norm");
                if (hn != 0.0) K.scale_inv(dh + j + 1, w, w);
                for (int i = 0; i <= j + 1; ++i) H[(size_t)j * (m + 1) + i] = col[i];
                for (int i = 0; i < j; ++i) {
                    double a = H[(size_t)j * (m + 1) + i], cc = H[(size_t)j * (m + 1) + i + 1];
                    H[(size_t)j * (m + 1) + i] = cs[i] * a + sn[i] * cc;
                    H[(size_t)j * (m + 1) + i + 1] = -sn[i] * a + cs[i] * cc;
                }
                double a = H[(size_t)j * (m + 1) + j], cc = H[(size_t)j * (m + 1) + j + 1];
                double rho = std::hypot(a, cc);
                cs[j] = a / rho; sn[j] = cc / rho;
                H[(size_t)j * (m + 1) + j] = rho; H[(size_t)j * (m + 1) + j + 1] = 0.0;
                g[j + 1] = -sn[j] * g[j]; g[j] = cs[j] * g[j];
                ++it; k = j + 1;
                info.est_relres = std::fabs(g[j + 1]) / bn;
                if (std::fabs(g[j + 1]) <= o.rtol * bn || it >= o.max_iters || hn == 0.0) break;
            }
            for (int i = k - 1; i >= 0; --i) {
                double s = g[i];
                for (int t = i + 1; t < k; ++t) s -= H[(size_t)t * (m + 1) + i] * yv[t];
                yv[i] = s / H[(size_t)i * (m + 1) + i];
            }
            TSP_CUDA(cudaMemcpyAsync(dh2, yv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
            prof_begin(c, PK_AXPY);
            k_update<<<K.nblk, KB, 0, c.s>>>(n, k, Z, ld, dh2, x);
            prof_end(c, PK_AXPY, 8.0 * n * (k + 2));
            c.launches++;
        }
    }
    TSP_CUDA(cudaEventRecord(e1, c.s));
    TSP_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    TSP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    info.iterations = it;
    info.status = status;
    info.t_solve_s = ms * 1e-3;
}

}  // namespace tsp

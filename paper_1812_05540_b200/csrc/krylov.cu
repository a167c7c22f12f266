// krylov.cu -- rows a13/a14: right-preconditioned flexible GMRES(m)
// with classical Gram-Schmidt applied twice (CGS2: two reductions per
// iteration instead of j+1, DESIGN.md R-krylov).  Reductions are per-block
// partial sums with a fixed tree, summed in a fixed order by one kernel, so
// every run is bitwise reproducible.  Givens rotations and the small
// least-squares solve live on the host (a (j+2)-double D2H copy per iteration).
#include <cmath>
#include <vector>

#include "tsp_internal.cuh"

namespace tsp {

constexpr int KB = 256;        // threads per block for vector kernels
constexpr int KG = 8;          // vectors per multi-dot group

// partial[g*KG + t][blockIdx.x] = sum over this block's rows of V_{g*KG+t} . w
__global__ void __launch_bounds__(KB) k_mdot(int64_t n, int nv, const double *__restrict__ V, int64_t ldv,
                                             const double *__restrict__ w, double *__restrict__ part, int nblk)
{
    const int g = blockIdx.y;
    const int v0 = g * KG, cnt = min(KG, nv - v0);
    double acc[KG];
#pragma unroll
    for (int t = 0; t < KG; ++t) acc[t] = 0.0;
    for (int64_t r = blockIdx.x * (int64_t)KB + threadIdx.x; r < n; r += (int64_t)nblk * KB) {
        const double wr = __ldg(w + r);
#pragma unroll
        for (int t = 0; t < KG; ++t)
            if (t < cnt) acc[t] = fma(__ldcs(V + (v0 + t) * ldv + r), wr, acc[t]);
    }
    __shared__ double red[KG][KB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int t = 0; t < KG; ++t) {
        double x = acc[t];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[t][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
        double x = 0.0;
        for (int u = 0; u < KB / 32; ++u) x += red[threadIdx.x][u];
        part[(int64_t)(v0 + threadIdx.x) * nblk + blockIdx.x] = x;
    }
}

// out[i] (+)= sum_b part[i][b], fixed order; mode 0: out = s, 1: out += s, 2: out = sqrt(s)
__global__ void k_reduce(int nv, const double *__restrict__ part, int nblk, double *out, int mode)
{
    int i = blockIdx.x;
    if (i >= nv) return;
    __shared__ double red[32];
    double x = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) x += part[(int64_t)i * nblk + b];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int u = 0; u < (int)(blockDim.x >> 5); ++u) s += red[u];
        if (mode == 0) out[i] = s;
        else if (mode == 1) out[i] += s;
        else out[i] = sqrt(s);
    }
}

// w -= V h (h: nv coefficients on device); optional partial of ||w||^2
template <bool NORM>
__global__ void __launch_bounds__(KB) k_maxpy(int64_t n, int nv, const double *__restrict__ V, int64_t ldv,
                                              const double *__restrict__ h, double *__restrict__ w, double *__restrict__ part,
                                              int nblk)
{
    __shared__ double hs[128];
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    double nrm = 0.0;
    for (int64_t r = blockIdx.x * (int64_t)KB + threadIdx.x; r < n; r += (int64_t)nblk * KB) {
        double acc = w[r];
        for (int t = 0; t < nv; ++t) acc = fma(-hs[t], __ldcs(V + t * ldv + r), acc);
        w[r] = acc;
        if (NORM) nrm = fma(acc, acc, nrm);
    }
    if (NORM) {
        __shared__ double red[KB / 32];
        for (int o = 16; o; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int u = 0; u < KB / 32; ++u) s += red[u];
            part[blockIdx.x] = s;
        }
    }
}

// CGS2 pass 1 axpy fused with pass 2 dots: w -= V h ; part[t][blk] = sum_r V_t[r] w[r]
// (V is read once for both; the second read hits L1/L2).  Per-warp shuffle
// reductions accumulated in a fixed order: deterministic.
__global__ void __launch_bounds__(KB) k_maxpy_mdot(int64_t n, int nv, const double *__restrict__ V, int64_t ldv,
                                                   const double *__restrict__ h, double *__restrict__ w,
                                                   double *__restrict__ part, int nblk)
{
    __shared__ double hs[128];
    __shared__ double sacc[KB / 32][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    for (int t = lane; t < nv; t += 32) sacc[wid][t] = 0.0;
    __syncthreads();
    const int64_t stride = (int64_t)nblk * KB;
    const int64_t nround = (n + stride - 1) / stride;
    for (int64_t k = 0; k < nround; ++k) {
        const int64_t r = k * stride + blockIdx.x * (int64_t)KB + threadIdx.x;
        const bool ok = r < n;
        double acc = ok ? w[r] : 0.0;
        if (ok) {
            for (int t = 0; t < nv; ++t) acc = fma(-hs[t], V[t * ldv + r], acc);
            w[r] = acc;
        }
        for (int t = 0; t < nv; ++t) {
            double d = ok ? V[t * ldv + r] * acc : 0.0;
            for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) sacc[wid][t] += d;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nv; t += KB) {
        double s = 0.0;
        for (int u = 0; u < KB / 32; ++u) s += sacc[u][t];
        part[(int64_t)t * nblk + blockIdx.x] = s;
    }
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
        for (int t = 0; t < k; ++t) acc = fma(ys[t], Z[t * ldz + r], acc);
        x[r] = acc;
    }
}

// y = a * x  (a = 1 / *s, read on device)
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

struct Kr {
    Ctx &c;
    int64_t n;
    int nblk;
    Kr(Ctx &c_) : c(c_), n(c_.n) { nblk = std::min<int64_t>((n + KB - 1) / KB, (int64_t)c.sm_count * 4); if (nblk < 1) nblk = 1; }
    int vgrid() const { return nblk; }
    // h[0..nv) = V[0..nv)^T w  (mode: 0 set, 1 add)
    void mdot(const double *V, int nv, const double *w, double *h, int mode) {
        prof_begin(c, PK_DOT);
        dim3 g(nblk, (nv + KG - 1) / KG);
        k_mdot<<<g, KB, 0, c.s>>>(n, nv, V, n, w, c.kpart, nblk);
        k_reduce<<<nv, 256, 0, c.s>>>(nv, c.kpart, nblk, h, mode);
        prof_end(c, PK_DOT, 8.0 * n * (nv + (nv + KG - 1) / KG));
        c.launches += 2;
    }
    void maxpy(const double *V, int nv, const double *h, double *w) {
        prof_begin(c, PK_AXPY);
        k_maxpy<false><<<nblk, KB, 0, c.s>>>(n, nv, V, n, h, w, nullptr, nblk);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        c.launches++;
    }
    // w -= V h1 ; h2 = V^T w  (CGS2 pass-1 update fused with pass-2 projections)
    void maxpy_mdot(const double *V, int nv, const double *h1, double *w, double *h2) {
        prof_begin(c, PK_AXPY);
        k_maxpy_mdot<<<nblk, KB, 0, c.s>>>(n, nv, V, n, h1, w, c.kpart, nblk);
        k_reduce<<<nv, 256, 0, c.s>>>(nv, c.kpart, nblk, h2, 0);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        c.launches += 2;
    }
    // w -= V h and ||w|| -> *nrm
    void maxpy_norm(const double *V, int nv, const double *h, double *w, double *nrm) {
        prof_begin(c, PK_AXPY);
        k_maxpy<true><<<nblk, KB, 0, c.s>>>(n, nv, V, n, h, w, c.kpart, nblk);
        k_reduce<<<1, 256, 0, c.s>>>(1, c.kpart, nblk, nrm, 2);
        prof_end(c, PK_AXPY, 8.0 * n * (nv + 2));
        c.launches += 2;
    }
    void norm(const double *w, double *nrm) {
        prof_begin(c, PK_NORM);
        dim3 g(nblk, 1);
        k_mdot<<<g, KB, 0, c.s>>>(n, 1, w, n, w, c.kpart, nblk);
        k_reduce<<<1, 256, 0, c.s>>>(1, c.kpart, nblk, nrm, 2);
        prof_end(c, PK_NORM, 8.0 * n);
        c.launches += 2;
    }
    void scale_inv(const double *s, const double *x, double *y) {
        prof_begin(c, PK_VEC);
        k_scale_inv<<<nblk, KB, 0, c.s>>>(n, s, x, y);
        prof_end(c, PK_VEC, 16.0 * n);
        c.launches++;
    }
};

__global__ void k_add_into(int nv, const double *__restrict__ a, double *__restrict__ b) { int i = threadIdx.x; if (i < nv) b[i] += a[i]; }

void krylov_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info)
{
    const int m = std::max(1, std::min(o.restart, 120));
    const int64_t n = c.n;
    if (c.kcap != m || c.V.n != (size_t)(m + 1) * n) {
        c.V.alloc((size_t)(m + 1) * n);
        c.Z.alloc((size_t)m * n);
        c.kr.alloc(n);
        c.kh.alloc(4 * (m + 2));
        c.kpart.alloc((size_t)(m + 2) * c.sm_count * 4 + 64);
        c.kcap = m;
    }
    Kr K(c);
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
    if (o.x0_zero) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
    int it = 0, status = TSP_NOT_CONVERGED;
    info.restarts = 0; info.est_relres = 0; info.true_relres = 0;
    if (bn == 0.0) {
        TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
        status = TSP_OK;
    } else {
        for (;;) {
            // r = b - A x ; beta = ||r||
            op_apply(c, x, r);
            k_bminus<<<K.vgrid(), KB, 0, c.s>>>(n, b, r);
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
            bool done = false;
            for (int j = 0; j < m; ++j) {
                double *vj = V + (size_t)j * n, *zj = Z + (size_t)j * n, *w = V + (size_t)(j + 1) * n;
                prec_apply(c, vj, zj);                 // z_j = M^-1 v_j (Algorithm 1)
                op_apply(c, zj, w);                    // w = A z_j
                // CGS2
                K.mdot(V, j + 1, w, dh, 0);
                K.maxpy_mdot(V, j + 1, dh, w, dh2);
                K.maxpy_norm(V, j + 1, dh2, w, dh + j + 1);
                k_add_into<<<1, 128, 0, c.s>>>(j + 1, dh2, dh);
                c.launches++;
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
                if (std::fabs(g[j + 1]) <= o.rtol * bn || it >= o.max_iters || hn == 0.0) { done = true; break; }
            }
            (void)done;
            for (int i = k - 1; i >= 0; --i) {
                double s = g[i];
                for (int t = i + 1; t < k; ++t) s -= H[(size_t)t * (m + 1) + i] * yv[t];
                yv[i] = s / H[(size_t)i * (m + 1) + i];
            }
            TSP_CUDA(cudaMemcpyAsync(dh2, yv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
            prof_begin(c, PK_AXPY);
            k_update<<<K.vgrid(), KB, 0, c.s>>>(n, k, Z, n, dh2, x);
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

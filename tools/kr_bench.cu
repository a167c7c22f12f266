// Developer microbenchmark: variants of the CGS2 kernels on synthetic vectors.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kr_bench tools/kr_bench.cu && ./kr_bench 42000000 30
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

constexpr int KB = 256;

__device__ __forceinline__ double block_sum(double x, double *red)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane == 0) red[wid] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) for (int u = 0; u < KB / 32; ++u) s += red[u];
    return s;
}

// A: grid (chunks, groups of G vectors), row loop unrolled by U
template <int G, int U>
__global__ void __launch_bounds__(KB) mdot(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ w, long CH,
                                           long n, double *__restrict__ part)
{
    const int k = blockIdx.x, v0 = blockIdx.y * G, cnt = min(G, nv - v0);
    const long beg = k * CH, end = min(n, beg + CH);
    double acc[G];
#pragma unroll
    for (int t = 0; t < G; ++t) acc[t] = 0.0;
    long r = beg + threadIdx.x;
    for (; r + (U - 1) * KB < end; r += U * KB) {
        double wr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) wr[u] = __ldg(w + r + u * KB);
#pragma unroll
        for (int t = 0; t < G; ++t)
            if (t < cnt) {
#pragma unroll
                for (int u = 0; u < U; ++u) acc[t] = fma(__ldcs(V + (v0 + t) * ldv + r + u * KB), wr[u], acc[t]);
            }
    }
    for (; r < end; r += KB) {
        const double wr = __ldg(w + r);
#pragma unroll
        for (int t = 0; t < G; ++t) if (t < cnt) acc[t] = fma(__ldcs(V + (v0 + t) * ldv + r), wr, acc[t]);
    }
    __shared__ double red[KB / 32];
#pragma unroll
    for (int t = 0; t < G; ++t) {
        const double s = block_sum(acc[t], red);
        if (threadIdx.x == 0 && t < cnt) part[(long)(v0 + t) * gridDim.x + k] = s;
    }
}

// maxpy + norm, loads unrolled by 8
template <int UL>
__global__ void __launch_bounds__(KB) maxpy_norm(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ h,
                                                 double *__restrict__ w, long CH, long n, double *__restrict__ part)
{
    __shared__ double hs[128];
    __shared__ double red[KB / 32];
    const int k = blockIdx.x;
    const long beg = k * CH, end = min(n, beg + CH);
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    double nrm = 0.0;
    for (long r = beg + threadIdx.x; r < end; r += KB) {
        double acc = w[r];
        int t = 0;
        if (UL > 1)
            for (; t + UL <= nv; t += UL) {
                double vv[UL > 1 ? UL : 1];
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

// mdot with the w chunk staged in shared memory; each block does ALL vectors of its chunk
template <int G, int U>
__global__ void __launch_bounds__(KB) mdot_s(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ w, long CH,
                                             long n, double *__restrict__ part, int nch)
{
    __shared__ double ws[2048];
    __shared__ double red[KB / 32];
    const int k = blockIdx.x;
    const long beg = k * CH, end = min(n, beg + CH);
    const int len = (int)(end - beg);
    for (int i = threadIdx.x; i < len; i += KB) ws[i] = __ldcs(w + beg + i);
    __syncthreads();
    for (int v0 = 0; v0 < nv; v0 += G) {
        const int cnt = min(G, nv - v0);
        double acc[G];
#pragma unroll
        for (int t = 0; t < G; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + (U - 1) * KB < len; i += U * KB) {
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
#pragma unroll
                    for (int u = 0; u < U; ++u) acc[t] = fma(__ldcs(V + (v0 + t) * ldv + beg + i + u * KB), ws[i + u * KB], acc[t]);
                }
        }
        for (; i < len; i += KB) {
#pragma unroll
            for (int t = 0; t < G; ++t) if (t < cnt) acc[t] = fma(__ldcs(V + (v0 + t) * ldv + beg + i), ws[i], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
            if (t < cnt) {
                const double s = block_sum(acc[t], red);
                if (threadIdx.x == 0) part[(long)(v0 + t) * nch + k] = s;
            }
        }
    }
}

__device__ __forceinline__ int brev4(int l) { return ((l & 1) << 3) | ((l & 2) << 1) | ((l & 4) >> 1) | ((l & 8) >> 3); }
// transpose-reduce: lane L returns sum over the warp of d[brev4(L & 15)]
__device__ __forceinline__ double tr16(double (&d)[16])
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const bool up = lane & 1;
        const double snd = up ? d[i] : d[i + 8], kp = up ? d[i + 8] : d[i];
        d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 1);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool up = lane & 2;
        const double snd = up ? d[i] : d[i + 4], kp = up ? d[i + 4] : d[i];
        d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 2);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const bool up = lane & 4;
        const double snd = up ? d[i] : d[i + 2], kp = up ? d[i + 2] : d[i];
        d[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
    }
    {
        const bool up = lane & 8;
        const double snd = up ? d[0] : d[1], kp = up ? d[1] : d[0];
        d[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
    }
    return d[0] + __shfl_xor_sync(0xffffffffu, d[0], 16);
}

// current library fused update + second projection
__global__ void __launch_bounds__(KB) maxpy_mdot0(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ h,
                                                  double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double hs[128];
    __shared__ double sacc[KB / 32][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = blockIdx.x;
    const long beg = k * CH, end = min(n, beg + CH);
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    for (int t = lane; t < nv; t += 32) sacc[wid][t] = 0.0;
    __syncthreads();
    for (long r0 = beg; r0 < end; r0 += KB) {
        const long r = r0 + threadIdx.x;
        const bool ok = r < end;
        double acc = ok ? w[r] : 0.0;
        if (ok) {
            for (int t = 0; t < nv; ++t) acc = fma(-hs[t], V[t * ldv + r], acc);
            w[r] = acc;
        }
        int t = 0;
        for (; t + 4 <= nv; t += 4) {
            double d0 = ok ? V[(t + 0) * ldv + r] * acc : 0.0, d1 = ok ? V[(t + 1) * ldv + r] * acc : 0.0;
            double d2 = ok ? V[(t + 2) * ldv + r] * acc : 0.0, d3 = ok ? V[(t + 3) * ldv + r] * acc : 0.0;
            for (int o = 16; o; o >>= 1) {
                d0 += __shfl_xor_sync(0xffffffffu, d0, o); d1 += __shfl_xor_sync(0xffffffffu, d1, o);
                d2 += __shfl_xor_sync(0xffffffffu, d2, o); d3 += __shfl_xor_sync(0xffffffffu, d3, o);
            }
            if (lane == 0) { sacc[wid][t] += d0; sacc[wid][t + 1] += d1; sacc[wid][t + 2] += d2; sacc[wid][t + 3] += d3; }
        }
        for (; t < nv; ++t) {
            double d = ok ? V[t * ldv + r] * acc : 0.0;
            for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) sacc[wid][t] += d;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nv; t += KB) {
        double s = 0.0;
        for (int u = 0; u < KB / 32; ++u) s += sacc[u][t];
        part[(long)t * cmax + k] = s;
    }
}

// unrolled update loads + transpose-reduced projections
template <int UL>
__global__ void __launch_bounds__(KB) maxpy_mdot1(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ h,
                                                  double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double hs[128];
    __shared__ double sacc[KB / 32][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = blockIdx.x;
    const long beg = k * CH, end = min(n, beg + CH);
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    for (int t = lane; t < 128; t += 32) sacc[wid][t] = 0.0;
    __syncthreads();
    const int vi = brev4(lane & 15);
    for (long r0 = beg; r0 < end; r0 += KB) {
        const long r = r0 + threadIdx.x;
        const bool ok = r < end;
        double acc = ok ? w[r] : 0.0;
        if (ok) {
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
        for (int g0 = 0; g0 < nv; g0 += 16) {
            double d[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) d[i] = (ok && g0 + i < nv) ? V[(g0 + i) * ldv + r] * acc : 0.0;
            const double s = tr16(d);
            if (lane < 16) sacc[wid][g0 + vi] += s;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nv; t += KB) {
        double s = 0.0;
        for (int u = 0; u < KB / 32; ++u) s += sacc[u][t];
        part[(long)t * cmax + k] = s;
    }
}

// update pass thread-per-row; dot pass warp-per-vector over the 256-row slab (w' staged in smem)
template <int UL, int MAXK>
__global__ void __launch_bounds__(KB) maxpy_mdot2(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ h,
                                                  double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double hs[128];
    __shared__ double ws[KB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, k = blockIdx.x;
    const long beg = k * CH, end = min(n, beg + CH);
    for (int t = threadIdx.x; t < nv; t += KB) hs[t] = h[t];
    __syncthreads();
    double p[MAXK];
#pragma unroll
    for (int q = 0; q < MAXK; ++q) p[q] = 0.0;
    for (long r0 = beg; r0 < end; r0 += KB) {
        const long r = r0 + threadIdx.x;
        const bool ok = r < end;
        double acc = 0.0;
        if (ok) {
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
        const int m = (int)min((long)KB, end - r0);
#pragma unroll
        for (int q = 0; q < MAXK; ++q) {
            const int t = wid + 8 * q;
            if (t < nv) {
                const double *vt = V + t * ldv + r0;
                if (m == KB) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) p[q] = fma(vt[lane + 32 * e], ws[lane + 32 * e], p[q]);
                } else {
                    for (int e = lane; e < m; e += 32) p[q] = fma(vt[e], ws[e], p[q]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < MAXK; ++q) {
        const int t = wid + 8 * q;
        if (t < nv) {
            double x = p[q];
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) part[(long)t * cmax + k] = x;
        }
    }
}

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
    for (int b = 1, t = NV / 2; b < NV; b <<= 1, t >>= 1) if (lane & b) idx |= t;
    if (lane < NV) red[wid][idx] = x;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x < NV)
        for (int u = 0; u < KB / 32; ++u) s += red[u][threadIdx.x];
    __syncthreads();
    return s;
}
template <int G, int U>
__global__ void __launch_bounds__(KB) mdot2(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ u,
                                            const double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double us[2048], ws[2048];
    __shared__ double red[KB / 32][2 * G];
    const int k = blockIdx.x;
    const long beg = k * CH;
    const int len = (int)(min(n, beg + CH) - beg);
    for (int i = threadIdx.x; i < len; i += KB) { us[i] = __ldcs(u + beg + i); ws[i] = __ldcs(w + beg + i); }
    __syncthreads();
    for (int v0 = 0; v0 < nv; v0 += G) {
        const int cnt = min(G, nv - v0);
        const double *Vg = V + v0 * ldv + beg;
        double acc[2 * G];
#pragma unroll
        for (int t = 0; t < 2 * G; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + (U - 1) * KB < len; i += U * KB) {
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const double vv = __ldcs(Vg + t * ldv + i + q * KB);
                        acc[t] = fma(vv, us[i + q * KB], acc[t]);
                        acc[G + t] = fma(vv, ws[i + q * KB], acc[G + t]);
                    }
                }
        }
        for (; i < len; i += KB) {
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
                    const double vv = __ldcs(Vg + t * ldv + i);
                    acc[t] = fma(vv, us[i], acc[t]);
                    acc[G + t] = fma(vv, ws[i], acc[G + t]);
                }
        }
        const double s = block_sum_multi<2 * G>(acc, red);
        const int q = threadIdx.x;
        if (q < 2 * G && (q % G) < cnt) part[(long)((q < G ? 0 : nv) + v0 + q % G) * cmax + k] = s;
    }
}

// interleaved staging {u_i, w_i}
template <int G, int U>
__global__ void __launch_bounds__(KB) mdot2i(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ u,
                                             const double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double2 uw[2048];
    __shared__ double red[KB / 32][2 * G];
    const int k = blockIdx.x;
    const long beg = k * CH;
    const int len = (int)(min(n, beg + CH) - beg);
    for (int i = threadIdx.x; i < len; i += KB) uw[i] = make_double2(__ldcs(u + beg + i), __ldcs(w + beg + i));
    __syncthreads();
    for (int v0 = 0; v0 < nv; v0 += G) {
        const int cnt = min(G, nv - v0);
        const double *Vg = V + v0 * ldv + beg;
        double acc[2 * G];
#pragma unroll
        for (int t = 0; t < 2 * G; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + (U - 1) * KB < len; i += U * KB) {
            double2 x[U];
#pragma unroll
            for (int q = 0; q < U; ++q) x[q] = uw[i + q * KB];
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const double vv = __ldcs(Vg + t * ldv + i + q * KB);
                        acc[t] = fma(vv, x[q].x, acc[t]);
                        acc[G + t] = fma(vv, x[q].y, acc[G + t]);
                    }
                }
        }
        for (; i < len; i += KB) {
            const double2 x = uw[i];
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
                    const double vv = __ldcs(Vg + t * ldv + i);
                    acc[t] = fma(vv, x.x, acc[t]);
                    acc[G + t] = fma(vv, x.y, acc[G + t]);
                }
        }
        const double s = block_sum_multi<2 * G>(acc, red);
        const int q = threadIdx.x;
        if (q < 2 * G && (q % G) < cnt) part[(long)((q < G ? 0 : nv) + v0 + q % G) * cmax + k] = s;
    }
}
// no staging: u, w through L1
template <int G, int U>
__global__ void __launch_bounds__(KB) mdot2n(int nv, const double *__restrict__ V, long ldv, const double *__restrict__ u,
                                             const double *__restrict__ w, long CH, long n, double *__restrict__ part, int cmax)
{
    __shared__ double red[KB / 32][2 * G];
    const int k = blockIdx.x;
    const long beg = k * CH;
    const int len = (int)(min(n, beg + CH) - beg);
    for (int v0 = 0; v0 < nv; v0 += G) {
        const int cnt = min(G, nv - v0);
        const double *Vg = V + v0 * ldv + beg;
        double acc[2 * G];
#pragma unroll
        for (int t = 0; t < 2 * G; ++t) acc[t] = 0.0;
        int i = threadIdx.x;
        for (; i + (U - 1) * KB < len; i += U * KB) {
            double xu[U], xw[U];
#pragma unroll
            for (int q = 0; q < U; ++q) { xu[q] = __ldg(u + beg + i + q * KB); xw[q] = __ldg(w + beg + i + q * KB); }
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const double vv = __ldcs(Vg + t * ldv + i + q * KB);
                        acc[t] = fma(vv, xu[q], acc[t]);
                        acc[G + t] = fma(vv, xw[q], acc[G + t]);
                    }
                }
        }
        for (; i < len; i += KB) {
            const double xu = __ldg(u + beg + i), xw = __ldg(w + beg + i);
#pragma unroll
            for (int t = 0; t < G; ++t)
                if (t < cnt) {
                    const double vv = __ldcs(Vg + t * ldv + i);
                    acc[t] = fma(vv, xu, acc[t]);
                    acc[G + t] = fma(vv, xw, acc[G + t]);
                }
        }
        const double s = block_sum_multi<2 * G>(acc, red);
        const int q = threadIdx.x;
        if (q < 2 * G && (q % G) < cnt) part[(long)((q < G ? 0 : nv) + v0 + q % G) * cmax + k] = s;
    }
}

__global__ void fillk(double *a, long n, double s)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        a[i] = s * (double)((i * 2654435761UL) % 1000003) / 1000003.0 - 0.5;
}
// plain copy for reference
__global__ void copyk(const double *__restrict__ a, double *__restrict__ b, long n)
{
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char **argv)
{
    long n = argc > 1 ? atol(argv[1]) : 42000000;
    int nv = argc > 2 ? atoi(argv[2]) : 30;
    double *V, *w, *part, *h;
    // optional extra device footprint (GB) to mimic the solver's ~110 GB working set (TLB reach)
    const double extra_gb = argc > 3 ? atof(argv[3]) : 0.0;
    std::vector<void *> extra;
    for (double gb = 0; gb < extra_gb; gb += 4.0) {
        void *p = nullptr;
        if (cudaMalloc(&p, (size_t)4 << 30) != cudaSuccess) break;
        cudaMemset(p, 0, (size_t)4 << 30);
        extra.push_back(p);
    }
    cudaMalloc(&V, sizeof(double) * n * (nv + 1));
    cudaMalloc(&w, sizeof(double) * n);
    cudaMalloc(&part, sizeof(double) * 200000 * 70);
    cudaMalloc(&h, sizeof(double) * 128);
    fillk<<<148 * 8, 256>>>(V, n * (nv + 1), 1.0);
    fillk<<<148 * 8, 256>>>(w, n, 2.0);
    fillk<<<1, 128>>>(h, 128, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char *name, double bytes, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        cudaEventRecord(e0);
        const int R = 10;
        for (int i = 0; i < R; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms / R, bytes / (ms / R * 1e-3) / 1e9);
    };
    const double vb = 8.0 * n;
    {
        const long CH = 2048; int nch = (int)((n + CH - 1) / CH);
        double *w2; cudaMalloc(&w2, sizeof(double) * n);
        std::vector<double> p0((size_t)nv * nch), p1((size_t)nv * nch);
        auto cmp = [&](const char *nm) {
            double mx = 0; for (size_t i = 0; i < p0.size(); ++i) mx = fmax(mx, fabs(p0[i] - p1[i]) / (fabs(p0[i]) + 1e-300));
            printf("check %-20s max rel diff %.3e\n", nm, mx);
        };
        cudaMemcpy(w2, w, 8 * n, cudaMemcpyDeviceToDevice);
        maxpy_mdot0<<<nch, KB>>>(nv, V, n, h, w2, CH, n, part, nch);
        cudaMemcpy(p0.data(), part, 8 * p0.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(p0.data(), part, 8 * p0.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(w2, w, 8 * n, cudaMemcpyDeviceToDevice);
        maxpy_mdot1<8><<<nch, KB>>>(nv, V, n, h, w2, CH, n, part, nch);
        cudaMemcpy(p1.data(), part, 8 * p1.size(), cudaMemcpyDeviceToHost);
        cmp("maxpy_mdot1");
        cudaMemcpy(w2, w, 8 * n, cudaMemcpyDeviceToDevice);
        maxpy_mdot2<8, 16><<<nch, KB>>>(nv, V, n, h, w2, CH, n, part, nch);
        cudaMemcpy(p1.data(), part, 8 * p1.size(), cudaMemcpyDeviceToHost);
        cmp("maxpy_mdot2");
        mdot<8, 1><<<dim3(nch, (nv + 7) / 8), KB>>>(nv, V, n, w, CH, n, part);
        cudaMemcpy(p0.data(), part, 8 * p0.size(), cudaMemcpyDeviceToHost);
        mdot_s<4, 2><<<nch, KB>>>(nv, V, n, w, CH, n, part, nch);
        cudaMemcpy(p1.data(), part, 8 * p1.size(), cudaMemcpyDeviceToHost);
        cmp("mdot_s");
        mdot2<8, 1><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch);
        {
            std::vector<double> p2((size_t)2 * nv * nch);
            cudaMemcpy(p2.data(), part, 8 * p2.size(), cudaMemcpyDeviceToHost);
            double mx = 0;
            for (size_t i = 0; i < p0.size(); ++i) mx = fmax(mx, fabs(p2[(size_t)nv * nch + i] - p0[i]) / (fabs(p0[i]) + 1e-300));
            printf("check mdot2 (w part) max rel diff %.3e\n", mx);
        }
        cudaFree(w2);
    }
    timeit("copy (r+w)", 2 * vb, [&] { copyk<<<148 * 8, 256>>>(V, w, n); });
    for (long CH : {2048L}) {
        int nch = (int)((n + CH - 1) / CH);
        char nm[64];
        snprintf(nm, 64, "mdot G8 U1 CH%ld", CH);
        timeit(nm, vb * (nv + (nv + 7) / 8), [&] { mdot<8, 1><<<dim3(nch, (nv + 7) / 8), KB>>>(nv, V, n, w, CH, n, part); });
        snprintf(nm, 64, "mdot G8 U2 CH%ld", CH);
        if (0) timeit(nm, vb * (nv + (nv + 7) / 8), [&] { mdot<8, 2><<<dim3(nch, (nv + 7) / 8), KB>>>(nv, V, n, w, CH, n, part); });
        snprintf(nm, 64, "mdot G4 U2 CH%ld", CH);
        timeit(nm, vb * (nv + (nv + 3) / 4), [&] { mdot<4, 2><<<dim3(nch, (nv + 3) / 4), KB>>>(nv, V, n, w, CH, n, part); });
        snprintf(nm, 64, "mdot G16 U1 CH%ld", CH);
        if (0) timeit(nm, vb * (nv + (nv + 15) / 16), [&] { mdot<16, 1><<<dim3(nch, (nv + 15) / 16), KB>>>(nv, V, n, w, CH, n, part); });
        snprintf(nm, 64, "mdot_s G8 U1 CH%ld", CH);
        timeit(nm, vb * (nv + (nv + 7) / 8), [&] { mdot_s<8, 1><<<nch, KB>>>(nv, V, n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot_s G4 U2 CH%ld", CH);
        timeit(nm, vb * (nv + (nv + 7) / 8), [&] { mdot_s<4, 2><<<nch, KB>>>(nv, V, n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot_s G8 U2 CH%ld", CH);
        timeit(nm, vb * (nv + (nv + 7) / 8), [&] { mdot_s<8, 2><<<nch, KB>>>(nv, V, n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2 G8 U1");
        timeit(nm, vb * (nv + 1), [&] { mdot2<8, 1><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2 G8 U2");
        timeit(nm, vb * (nv + 1), [&] { mdot2<8, 2><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2 G4 U2");
        timeit(nm, vb * (nv + 1), [&] { mdot2<4, 2><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2 G4 U4");
        timeit(nm, vb * (nv + 1), [&] { mdot2<4, 4><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2i G4 U2");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<4, 2><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2i G4 U2 misaligned+5");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<4, 2><<<nch, KB>>>(nv, V + 5, n, V + (nv - 1) * n + 5, w + 5, CH, n - 8, part, nch); });
        snprintf(nm, 64, "mdot2i G4 U4");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<4, 4><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2i G2 U8");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<2, 8><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2i G2 U4");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<2, 4><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2i G8 U2");
        timeit(nm, vb * (nv + 1), [&] { mdot2i<8, 2><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2n G4 U2");
        timeit(nm, vb * (nv + 1), [&] { mdot2n<4, 2><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2n G8 U1");
        timeit(nm, vb * (nv + 1), [&] { mdot2n<8, 1><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "mdot2 G2 U4");
        timeit(nm, vb * (nv + 1), [&] { mdot2<2, 4><<<nch, KB>>>(nv, V, n, V + (nv - 1) * n, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot0 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_mdot0<<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot1 UL4 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_mdot1<4><<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot1 UL8 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_mdot1<8><<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot2 UL8 K8 CH%ld", CH);
        if (nv <= 64) timeit(nm, vb * (nv + 2), [&] { maxpy_mdot2<8, 8><<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot2 UL8 K16 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_mdot2<8, 16><<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_mdot2 UL4 K8 CH%ld", CH);
        if (nv <= 64) timeit(nm, vb * (nv + 2), [&] { maxpy_mdot2<4, 8><<<nch, KB>>>(nv, V, n, h, w, CH, n, part, nch); });
        snprintf(nm, 64, "maxpy_norm UL1 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_norm<1><<<nch, KB>>>(nv, V, n, h, w, CH, n, part); });
        snprintf(nm, 64, "maxpy_norm UL8 CH%ld", CH);
        timeit(nm, vb * (nv + 2), [&] { maxpy_norm<8><<<nch, KB>>>(nv, V, n, h, w, CH, n, part); });
    }
    return 0;
}

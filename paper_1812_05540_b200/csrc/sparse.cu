// sparse.cu -- device CSR upload and the sliced-ELL (SELL-32) repack used by
// every apply-path kernel (DESIGN.md R-layout).
#include <cub/cub.cuh>

#include "tsp_internal.cuh"

namespace tsp {

void csr_upload(Ctx &c, Csr &A, int n, int m, int nc, const int32_t *rp, const int32_t *ci, const double *v, bool on_device)
{
    A.n = n; A.m = m; A.nc = nc;
    int64_t nnz;
    if (on_device) {
        int32_t last;
        TSP_CUDA(cudaMemcpyAsync(&last, rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
        nnz = last;
    } else {
        nnz = rp[n];
    }
    TSP_REQUIRE(nnz >= 0, TSP_ERR_INVALID_ARG, "rowptr[n] < 0");
    A.nnz = nnz;
    A.rp.alloc(n + 1); A.ci.alloc(nnz); A.v.alloc(nnz * nc);
    cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    TSP_CUDA(cudaMemcpyAsync(A.rp, rp, sizeof(int32_t) * (n + 1), k, c.s));
    if (nnz) {
        TSP_CUDA(cudaMemcpyAsync(A.ci, ci, sizeof(int32_t) * nnz, k, c.s));
        TSP_CUDA(cudaMemcpyAsync(A.v, v, sizeof(double) * nnz * nc, k, c.s));
    }
}

// validation on the device (one flag back to the host): rowptr[0] == 0, monotone row pointers inside
// [0, nnz] (a row outside is flagged and not read), in-range and strictly increasing (sorted, unique)
// columns in every row
__global__ void k_check_csr(int n, int m, int64_t nnz, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            unsigned *flag)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    unsigned f = 0;
    if (i == 0 && rp[0] != 0) f |= 1u;
    if (i < n) {
        const int64_t a = rp[i], b = rp[i + 1];
        if (b < a || a < 0 || b > nnz) { atomicOr(flag, f | 2u); return; }
        for (int64_t q = a; q < b; ++q) {
            const int j = ci[q];
            if (j < 0 || j >= m) f |= 4u;
            if (q > a && j <= ci[q - 1]) f |= 8u;
        }
    }
    if (f) atomicOr(flag, f);
}

void check_csr(Ctx &c, const Csr &A, const char *name)
{
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    k_check_csr<<<grid_for(A.n + 1, 256), 256, 0, c.s>>>(A.n, A.m, A.nnz, A.rp, A.ci, flag);
    c.launches++;
    unsigned f = 0;
    TSP_CUDA(cudaMemcpyAsync(&f, flag.p, sizeof(f), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    TSP_REQUIRE(!(f & 1u), TSP_ERR_INVALID_ARG, std::string(name) + ": rowptr[0] != 0");
    TSP_REQUIRE(!(f & 2u), TSP_ERR_INVALID_ARG, std::string(name) + ": rowptr not monotone or outside [0, nnz]");
    TSP_REQUIRE(!(f & 4u), TSP_ERR_INVALID_ARG, std::string(name) + ": column out of range");
    TSP_REQUIRE(!(f & 8u), TSP_ERR_INVALID_ARG, std::string(name) + ": columns not sorted/unique in a row");
}

// every value >= 0 (the fixed-stress diagonal)
__global__ void k_check_nonneg(int64_t n, const double *__restrict__ v, unsigned *flag)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n && !(v[k] >= 0.0)) atomicOr(flag, 1u);
}
bool all_nonneg(Ctx &c, const double *v, int64_t n)
{
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    if (n) k_check_nonneg<<<grid_for(n, 256), 256, 0, c.s>>>(n, v, flag);
    c.launches++;
    unsigned f = 0;
    TSP_CUDA(cudaMemcpyAsync(&f, flag.p, sizeof(f), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    return f == 0;
}

__global__ void k_sell_width(int n, const int32_t *__restrict__ rp, int64_t *__restrict__ w)
{
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    int nsl = (n + 31) / 32;
    if (s >= nsl) return;
    int mx = 0;
    for (int l = 0; l < 32; ++l) {
        int i = s * 32 + l;
        if (i < n) mx = max(mx, rp[i + 1] - rp[i]);
    }
    w[s] = mx;
}

struct ValMap { int m[16]; };

__global__ void k_sell_fill(int n, int nc, int bs, ValMap vm, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            const double *__restrict__ v, const int64_t *__restrict__ off, int32_t *__restrict__ scol,
                            double *__restrict__ sval)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int s = i >> 5, lane = i & 31;
    int64_t base = off[s], width = off[s + 1] - off[s];
    int64_t q0 = rp[i], len = rp[i + 1] - q0;
    for (int64_t k = 0; k < width; ++k) {
        int64_t slot = base + k;
        bool real = k < len;
        scol[slot * 32 + lane] = real ? ci[q0 + k] : (len ? ci[q0 + len - 1] : 0);   // padding: a valid column, value 0
        for (int e = 0; e < bs; ++e)
            sval[(slot * bs + e) * 32 + lane] = real ? v[(q0 + k) * nc + vm.m[e]] : 0.0;
    }
}

// Repack CSR (nc values per entry) into SELL-32 keeping bs values per entry,
// value e taken from component val_map[e] (identity if null).
void sell_from_csr(Ctx &c, const Csr &A, Sell &S, int bs, const int *val_map)
{
    S.nrows = A.n; S.bs = bs; S.ncols = A.m; S.nnz = A.nnz;
    S.nslices = (A.n + 31) / 32;
    ValMap vm;
    for (int e = 0; e < 16; ++e) vm.m[e] = e;
    if (val_map) for (int e = 0; e < bs; ++e) vm.m[e] = val_map[e];
    DBuf<int64_t> w; w.alloc(S.nslices + 1);
    S.off.alloc(S.nslices + 1);
    if (S.nslices) {
        k_sell_width<<<grid_for(S.nslices, 128), 128, 0, c.s>>>(A.n, A.rp, w);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, w.p, S.off.p, S.nslices + 1, c.s);
        void *t = scratch(c, tb);
        TSP_CUDA(cudaMemsetAsync(w.p + S.nslices, 0, sizeof(int64_t), c.s));
        cub::DeviceScan::ExclusiveSum(t, tb, w.p, S.off.p, S.nslices + 1, c.s);
        TSP_CUDA(cudaMemcpyAsync(&S.slots, S.off.p + S.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
    } else {
        S.slots = 0;
        S.off.zero(c.s);
    }
    S.col.alloc(S.slots * 32);
    S.val.alloc(S.slots * 32 * bs);
    if (A.n) k_sell_fill<<<grid_for(A.n, 256), 256, 0, c.s>>>(A.n, A.nc, bs, vm, A.rp, A.ci, A.v, S.off, S.col, S.val);
    TSP_CUDA(cudaGetLastError());
    c.launches += 2;
}

}  // namespace tsp

// gs.cu -- the paper's Gauss-Seidel AMG smoother ("one sweep of hybrid forward l1-Gauss-Seidel for the
// down cycle and one sweep of hybrid backward l1-Gauss-Seidel for the up cycle"), tsp_options.amg_smoother = 1,
// in the GPU-native reading R-gs:
//  * level 0 of each hierarchy (the grid level): multicolour GS over the whole level with the parity colourings
//    (nodes: (x&1) + 2(y&1) + 4(z&1), 8 colours for the 27-point mechanics graph; cells: (x+y+z)&1, red-black for
//    the 7-point S_pp) -- one launch per colour over a colour-ordered SELL copy of the level operator,
//    x_i <- x_i + (b_i - (A x)_i) / a_ii, colours ascending (forward) or descending (backward);
//  * coarse levels: hybrid l1-GS (Baker, Falgout, Kolev, Yang 2011) with the "processor" = a block of gs_block
//    consecutive rows = one CTA: inside the block multicolour GS in the block's own first-fit colouring (priority
//    (fmix32(i), i), computed here by Jones-Plassmann rounds, which equal the oracle's sequential first fit), the
//    block's x in shared memory, couplings to other blocks at their sweep-start values with the l1 diagonal
//    d_i = a_ii + sign(a_ii) sum_{j outside the block} |a_ij|; one launch per sweep.
// Single GPU (the colourings and blocks are global-row based; the z-slab path keeps l1-Jacobi).
// Apply arithmetic is free (parity with the oracle <= 1e-10); the colourings are exactly the oracle's.
#include <cub/cub.cuh>

#include "tsp_internal.cuh"

namespace tsp {

__device__ __forceinline__ uint32_t gs_fmix32(uint32_t x)
{
    x ^= x >> 16; x *= 0x85ebca6bU; x ^= x >> 13; x *= 0xc2b2ae35U; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint64_t gs_prio(int i) { return ((uint64_t)gs_fmix32((uint32_t)i) << 32) | (uint64_t)(uint32_t)i; }

// ---------------------------------------------------------------- level 0: multicolour
// parity colour of row i of the node (kind 0) or cell (kind 1) grid with NX x NY points per plane
__global__ void k_geo_colour(int n, int kind, int NX, int NY, int32_t *__restrict__ key, int32_t *__restrict__ row,
                             unsigned *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = i % NX, y = (i / NX) % NY, z = i / (NX * NY);
    const int k = kind == 0 ? (x & 1) + 2 * (y & 1) + 4 * (z & 1) : ((x + y + z) & 1);
    key[i] = k;
    row[i] = i;
    atomicAdd(cnt + k, 1u);
}
// rows sorted by colour -> padded order: colour c occupies [pad_off[c], pad_off[c] + count[c]), then -1 up to a
// multiple of 32 (a SELL slice holds one colour)
__global__ void k_pad_perm(int n, int ncol, const int64_t *__restrict__ off, const int64_t *__restrict__ pad_off,
                           const int32_t *__restrict__ sorted, int32_t *__restrict__ perm)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= pad_off[ncol]) return;
    int c = 0;
    while (c + 1 < ncol && r >= pad_off[c + 1]) ++c;
    const int64_t k = r - pad_off[c];
    perm[r] = k < off[c + 1] - off[c] ? sorted[off[c] + k] : -1;
}
__global__ void k_diag(int n, int nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                       double *__restrict__ d)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int c = 0; c < nc; ++c) d[(int64_t)i * nc + c] = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
        if (ci[q] == i)
            for (int c = 0; c < nc; ++c) d[(int64_t)i * nc + c] = v[q * nc + c];
}
// one colour of the multicolour sweep: SELL rows [32 s0, 32 s1) of the colour-ordered copy, in place on x
template <int NC>
__global__ void __launch_bounds__(256) k_gs_mc(int64_t r0, int64_t r1, const int64_t *__restrict__ off,
                                               const int32_t *__restrict__ col, const double *__restrict__ val,
                                               const int32_t *__restrict__ perm, const double *__restrict__ diag,
                                               const double *__restrict__ b, double *__restrict__ x)
{
    const int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= r1) return;
    const int i = perm[r];
    if (i < 0) return;
    const int64_t s = r >> 5;
    const int lane = (int)(r & 31);
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
#pragma unroll 2
    for (int64_t slot = off[s]; slot < off[s + 1]; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(val + (slot * NC + c) * 32 + lane), x[(int64_t)j * NC + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int64_t t = (int64_t)i * NC + c;
        const double d = diag[t];
        if (d != 0.0) x[t] = x[t] + (b[t] - acc[c]) / d;
    }
}
// width of each slice of the permuted rows
__global__ void k_sellp_width(int64_t nrows, const int32_t *__restrict__ perm, const int32_t *__restrict__ rp, int64_t *__restrict__ w)
{
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nrows / 32) return;
    int mx = 0;
    for (int l = 0; l < 32; ++l) {
        const int i = perm[s * 32 + l];
        if (i >= 0) mx = max(mx, rp[i + 1] - rp[i]);
    }
    w[s] = mx;
}
__global__ void k_sellp_fill(int64_t nrows, int nc, const int32_t *__restrict__ perm, const int32_t *__restrict__ rp,
                             const int32_t *__restrict__ ci, const double *__restrict__ v, const int64_t *__restrict__ off,
                             int32_t *__restrict__ scol, double *__restrict__ sval)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int64_t s = r >> 5;
    const int lane = (int)(r & 31);
    const int i = perm[r];
    const int64_t q0 = i >= 0 ? rp[i] : 0, len = i >= 0 ? rp[i + 1] - q0 : 0;
    for (int64_t k = 0; k < off[s + 1] - off[s]; ++k) {
        const int64_t slot = off[s] + k;
        const bool real = k < len;
        scol[slot * 32 + lane] = real ? ci[q0 + k] : (len ? ci[q0 + len - 1] : 0);
        for (int e = 0; e < nc; ++e) sval[(slot * nc + e) * 32 + lane] = real ? v[(q0 + k) * nc + e] : 0.0;
    }
}

static void gs_setup_multicolour(Ctx &c, Level &L, int nc, int kind, int NX, int NY)
{
    const int n = L.n;
    const int ncol = kind == 0 ? 8 : 2;
    DBuf<int32_t> key, row, key_s, row_s;
    key.alloc(n); row.alloc(n); key_s.alloc(n); row_s.alloc(n);
    DBuf<unsigned> cnt; cnt.alloc(8); cnt.zero(c.s);
    k_geo_colour<<<grid_for(n, 256), 256, 0, c.s>>>(n, kind, NX, NY, key, row, cnt);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_s.p, row.p, row_s.p, n, 0, 4, c.s);   // stable
    void *t = scratch(c, tb);
    cub::DeviceRadixSort::SortPairs(t, tb, key.p, key_s.p, row.p, row_s.p, n, 0, 4, c.s);
    unsigned h[8];
    TSP_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    std::vector<int64_t> off(ncol + 1, 0), pad(ncol + 1, 0);
    int used = 0;
    for (int k = 0; k < ncol; ++k) {
        off[k + 1] = off[k] + h[k];
        pad[k + 1] = pad[k] + ((h[k] + 31) / 32) * 32;
        if (h[k]) used = k + 1;
    }
    L.ncolor = used;
    L.gs_block = 0;
    L.cslice.assign(pad.begin(), pad.begin() + used + 1);
    DBuf<int64_t> doff, dpad;
    doff.alloc(ncol + 1); dpad.alloc(ncol + 1);
    TSP_CUDA(cudaMemcpyAsync(doff, off.data(), sizeof(int64_t) * (ncol + 1), cudaMemcpyHostToDevice, c.s));
    TSP_CUDA(cudaMemcpyAsync(dpad, pad.data(), sizeof(int64_t) * (ncol + 1), cudaMemcpyHostToDevice, c.s));
    const int64_t nrows = pad[ncol];
    L.gperm.alloc(std::max<int64_t>(nrows, 1));
    if (nrows) k_pad_perm<<<grid_for(nrows, 256), 256, 0, c.s>>>(n, ncol, doff, dpad, row_s, L.gperm);
    // colour-ordered SELL copy of the level operator
    Sell &S = L.sAc;
    S.nrows = (int)nrows; S.bs = nc; S.ncols = L.A.m; S.nnz = L.A.nnz; S.nslices = (int)(nrows / 32);
    DBuf<int64_t> w; w.alloc(S.nslices + 1);
    S.off.alloc(S.nslices + 1);
    TSP_CUDA(cudaMemsetAsync(w.p + S.nslices, 0, sizeof(int64_t), c.s));
    if (S.nslices) k_sellp_width<<<grid_for(S.nslices, 128), 128, 0, c.s>>>(nrows, L.gperm, L.A.rp, w);
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, w.p, S.off.p, S.nslices + 1, c.s);
    t = scratch(c, tb);
    cub::DeviceScan::ExclusiveSum(t, tb, w.p, S.off.p, S.nslices + 1, c.s);
    TSP_CUDA(cudaMemcpyAsync(&S.slots, S.off.p + S.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    S.col.alloc(S.slots * 32); S.val.alloc(S.slots * 32 * nc);
    if (nrows) k_sellp_fill<<<grid_for(nrows, 256), 256, 0, c.s>>>(nrows, nc, L.gperm, L.A.rp, L.A.ci, L.A.v, S.off, S.col, S.val);
    L.diag.alloc((size_t)std::max(n, 1) * nc);
    if (n) k_diag<<<grid_for(n, 256), 256, 0, c.s>>>(n, nc, L.A.rp, L.A.ci, L.A.v, L.diag);
    TSP_CUDA(cudaGetLastError());
    c.launches += 8;
}

// ---------------------------------------------------------------- coarse levels: hybrid l1-GS
constexpr int kGsThreads = 256;
constexpr int kGsMaxBlock = 1024;
constexpr int kGsMaxColours = 256;

// first-fit colouring of each block's induced subgraph by descending priority, Jones-Plassmann rounds: a row
// is coloured once all its higher-priority in-block neighbours are, with the smallest colour none of them holds
// (= the sequential first fit in descending priority)
__global__ void __launch_bounds__(kGsThreads) k_gs_colour(int n, int B, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                                          int16_t *__restrict__ col, int *__restrict__ maxcol,
                                                          int32_t *__restrict__ coff, int32_t *__restrict__ order)
{
    __shared__ int16_t cs[kGsMaxBlock];
    const int b0 = blockIdx.x * B, b1 = min(n, b0 + B);
    for (int r = b0 + threadIdx.x; r < b1; r += blockDim.x) cs[r - b0] = -1;
    __syncthreads();
    constexpr int RPT = kGsMaxBlock / kGsThreads;
    for (;;) {
        int16_t nw[RPT];
        int left = 0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            nw[u] = -1;
            const int r = b0 + threadIdx.x + u * kGsThreads;
            if (r >= b1 || cs[r - b0] >= 0) continue;
            left = 1;
            const uint64_t pr = gs_prio(r);
            uint64_t used[kGsMaxColours / 64] = {0, 0, 0, 0};
            bool ready = true;
            for (int64_t q = rp[r]; q < rp[r + 1]; ++q) {
                const int j = ci[q];
                if (j == r || j < b0 || j >= b1 || gs_prio(j) < pr) continue;
                const int cj = cs[j - b0];
                if (cj < 0) { ready = false; break; }
                if (cj < kGsMaxColours) used[cj >> 6] |= 1ull << (cj & 63);
            }
            if (!ready) continue;
            int k = 0;
            while (k < kGsMaxColours && ((used[k >> 6] >> (k & 63)) & 1ull)) ++k;
            nw[u] = (int16_t)k;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
            const int r = b0 + threadIdx.x + u * kGsThreads;
            if (nw[u] >= 0) { cs[r - b0] = nw[u]; atomicMax(maxcol, (int)nw[u]); }
        }
        if (!__syncthreads_or(left)) break;
    }
    for (int r = b0 + threadIdx.x; r < b1; r += blockDim.x) col[r] = cs[r - b0];
    // rows of the block grouped by colour (the sweep's warps take a colour's rows from this list; the order
    // inside a colour is immaterial -- no two rows of a colour are coupled)
    __shared__ int cnt[kGsMaxColours + 1];
    for (int k = threadIdx.x; k <= kGsMaxColours; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    for (int r = b0 + threadIdx.x; r < b1; r += blockDim.x) {
        const int k = cs[r - b0];
        if (k < kGsMaxColours) atomicAdd(&cnt[k + 1], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < kGsMaxColours; ++k) cnt[k + 1] += cnt[k];
    __syncthreads();
    for (int k = threadIdx.x; k <= kGsMaxColours; k += blockDim.x) coff[(int64_t)blockIdx.x * (kGsMaxColours + 1) + k] = b0 + cnt[k];
    __syncthreads();
    for (int r = b0 + threadIdx.x; r < b1; r += blockDim.x) {
        const int k = cs[r - b0];
        if (k < kGsMaxColours) order[b0 + atomicAdd(&cnt[k], 1)] = r;
    }
}
// hybrid l1 diagonal d_i = a_ii + sign(a_ii) sum_{j outside i's block} |a_ij| per component
__global__ void k_gs_dh(int n, int nc, int B, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                        const double *__restrict__ v, double *__restrict__ dh)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * nc) return;
    const int i = (int)(t / nc), c = (int)(t % nc);
    const int b0 = (i / B) * B, b1 = min(n, b0 + B);
    double aii = 0.0, l1 = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        const int j = ci[q];
        if (j == i) aii = v[q * nc + c];
        else if (j < b0 || j >= b1) l1 += fabs(v[q * nc + c]);
    }
    dh[t] = aii < 0.0 ? aii - l1 : aii + l1;
}
// one hybrid sweep: block of B rows per CTA, xs = the block's x in shared memory; ZERO: from x = 0 (no xin).
// Per colour, a warp per row: the lanes stride the row's entries, a shuffle tree sums them, lane 0 updates.
constexpr int kGsSweepThreads = 1024;   // a warp per row of the current colour: 32 rows of a colour in flight
template <int NC, bool ZERO>
__global__ void __launch_bounds__(kGsSweepThreads) k_gs_hyb(int n, int B, int ncol, int backward, const int32_t *__restrict__ rp,
                                                       const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                       const double *__restrict__ dh, const int32_t *__restrict__ coff,
                                                       const int32_t *__restrict__ order, const double *__restrict__ b,
                                                       const double *__restrict__ xin, double *__restrict__ xout)
{
    __shared__ double xs[kGsMaxBlock * NC];
    const int b0 = blockIdx.x * B, b1 = min(n, b0 + B);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int t = threadIdx.x; t < (b1 - b0) * NC; t += blockDim.x) xs[t] = ZERO ? 0.0 : xin[(int64_t)b0 * NC + t];
    __syncthreads();
    const int32_t *co = coff + (int64_t)blockIdx.x * (kGsMaxColours + 1);
    for (int k = 0; k < ncol; ++k) {
        const int cl = backward ? ncol - 1 - k : k;
        const int o0 = co[cl], o1 = co[cl + 1];
        for (int o = o0 + warp; o < o1; o += nwarp) {
            const int r = order[o];
            double s[NC], d[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) { s[c] = 0.0; d[c] = 0.0; }
            const int64_t q1 = rp[r + 1];
#pragma unroll 2
            for (int64_t q = rp[r] + lane; q < q1; q += 32) {
                const int j = __ldg(ci + q);
                const bool inb = j >= b0 && j < b1;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double a = __ldg(v + q * NC + c);
                    if (j == r) d[c] = a;
                    else if (inb) s[c] = fma(a, xs[(j - b0) * NC + c], s[c]);
                    else if (!ZERO) s[c] = fma(a, __ldg(xin + (int64_t)j * NC + c), s[c]);
                }
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int off = 16; off; off >>= 1) {
                    s[c] += __shfl_xor_sync(0xffffffffu, s[c], off);
                    d[c] += __shfl_xor_sync(0xffffffffu, d[c], off);
                }
            if (lane == 0)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double dd = dh[(int64_t)r * NC + c];
                    double &xr = xs[(r - b0) * NC + c];
                    if (dd != 0.0) xr = xr + ((b[(int64_t)r * NC + c] - s[c]) - d[c] * xr) / dd;
                }
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < (b1 - b0) * NC; t += blockDim.x) xout[(int64_t)b0 * NC + t] = xs[t];
}

static void gs_setup_hybrid(Ctx &c, Level &L, int nc)
{
    const int n = L.n;
    const int B = c.o.amg_gs_block;
    L.gs_block = B;
    L.gsc.alloc(std::max(n, 1));
    L.dh.alloc((size_t)std::max(n, 1) * nc);
    DBuf<int> mx; mx.alloc(1); mx.zero(c.s);
    const int nb = (n + B - 1) / B;
    L.gcoff.alloc((size_t)std::max(nb, 1) * (kGsMaxColours + 1));
    L.gorder.alloc(std::max(n, 1));
    if (nb) k_gs_colour<<<nb, kGsThreads, 0, c.s>>>(n, B, L.A.rp, L.A.ci, L.gsc, mx, L.gcoff, L.gorder);
    if (n) k_gs_dh<<<grid_for((int64_t)n * nc, 256), 256, 0, c.s>>>(n, nc, B, L.A.rp, L.A.ci, L.A.v, L.dh);
    int m = -1;
    TSP_CUDA(cudaMemcpyAsync(&m, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    TSP_REQUIRE(m < kGsMaxColours, TSP_ERR_INVALID_ARG, "GS smoother: a block needs more than 256 colours");
    L.ncolor = m + 1;
    c.launches += 2;
}

void gs_setup(Ctx &c, Hier &H, int nc)
{
    if (H.smoother != 1) return;
    TSP_REQUIRE(c.nranks == 1, TSP_ERR_INVALID_ARG, "amg_smoother = 1 (Gauss-Seidel) is single-GPU only");
    TSP_REQUIRE(c.o.amg_gs_block >= 32 && c.o.amg_gs_block <= kGsMaxBlock, TSP_ERR_INVALID_ARG, "amg_gs_block must be in [32, 1024]");
    for (size_t l = 0; l < H.L.size(); ++l) {
        Level &L = H.L[l];
        if (L.coarsest) continue;
        if (l == 0) {
            if (nc == 3) gs_setup_multicolour(c, L, nc, 0, c.nx + 1, c.ny + 1);   // node grid (mechanics)
            else gs_setup_multicolour(c, L, nc, 1, c.nx, c.ny);                  // cell grid (pressure)
        } else gs_setup_hybrid(c, L, nc);
    }
}

// ---------------------------------------------------------------- sweeps (apply)
template <int NC>
void gs_sweep(Ctx &c, Level &L, bool backward, const double *b, const double *xin, double *xout)
{
    const int n = L.n;
    if (!n) return;
    if (L.gs_block == 0) {
        if (!xin) TSP_CUDA(cudaMemsetAsync(xout, 0, sizeof(double) * n * NC, c.s));
        else if (xin != xout) TSP_CUDA(cudaMemcpyAsync(xout, xin, sizeof(double) * n * NC, cudaMemcpyDeviceToDevice, c.s));
        for (int k = 0; k < L.ncolor; ++k) {
            const int cl = backward ? L.ncolor - 1 - k : k;
            const int64_t r0 = L.cslice[cl], r1 = L.cslice[cl + 1];
            if (r1 > r0)
                k_gs_mc<NC><<<grid_for(r1 - r0, 256), 256, 0, c.s>>>(r0, r1, L.sAc.off, L.sAc.col, L.sAc.val, L.gperm, L.diag, b, xout);
            c.launches++;
        }
    } else {
        const int nb = (n + L.gs_block - 1) / L.gs_block;
        if (!xin) k_gs_hyb<NC, true><<<nb, kGsSweepThreads, 0, c.s>>>(n, L.gs_block, L.ncolor, backward, L.A.rp, L.A.ci, L.A.v, L.dh,
                                                                 L.gcoff, L.gorder, b, nullptr, xout);
        else k_gs_hyb<NC, false><<<nb, kGsSweepThreads, 0, c.s>>>(n, L.gs_block, L.ncolor, backward, L.A.rp, L.A.ci, L.A.v, L.dh,
                                                             L.gcoff, L.gorder, b, xin, xout);
        c.launches++;
    }
    TSP_CUDA(cudaGetLastError());
}
template void gs_sweep<1>(Ctx &, Level &, bool, const double *, const double *, double *);
template void gs_sweep<3>(Ctx &, Level &, bool, const double *, const double *, double *);

// test hook: colour per row of a level (tsp_export_colour)
__global__ void k_unperm_colour(int64_t nrows, const int32_t *__restrict__ perm, const int64_t *__restrict__ cs, int ncol,
                                int32_t *__restrict__ out)
{
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows || perm[r] < 0) return;
    int c = 0;
    while (c + 1 < ncol && r >= cs[c + 1]) ++c;
    out[perm[r]] = c;
}
__global__ void k_widen_colour(int n, const int16_t *__restrict__ in, int32_t *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}
void gs_export_colour(Ctx &c, const Level &L, int32_t *host_out)
{
    DBuf<int32_t> d; d.alloc(std::max(L.n, 1));
    if (L.gs_block == 0) {
        DBuf<int64_t> cs; cs.alloc(L.cslice.size());
        TSP_CUDA(cudaMemcpyAsync(cs, L.cslice.data(), sizeof(int64_t) * L.cslice.size(), cudaMemcpyHostToDevice, c.s));
        if (L.sAc.nrows) k_unperm_colour<<<grid_for(L.sAc.nrows, 256), 256, 0, c.s>>>(L.sAc.nrows, L.gperm, cs, L.ncolor, d);
    } else if (L.n) k_widen_colour<<<grid_for(L.n, 256), 256, 0, c.s>>>(L.n, L.gsc, d);
    TSP_CUDA(cudaMemcpyAsync(host_out, d.p, sizeof(int32_t) * L.n, cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
}

// algorithmic bytes of one sweep (matrix once + b, x read, x written)
double gs_sweep_bytes(const Level &L, int nc)
{
    const double vec = 8.0 * nc * L.n;
    if (L.gs_block == 0) return (double)L.sAc.slots * 32 * (4.0 + 8.0 * nc) + 4.0 * L.sAc.nrows + 3 * vec;
    return (double)L.A.nnz * (4.0 + 8.0 * nc) + 2.0 * L.n + 4 * vec;
}

}  // namespace tsp

// halo.cu -- z-slab partition, halo plans / exchanges, and the fixed reduction
// chunks that make every dot product bitwise identical for any number of ranks.
#include <algorithm>

#include "tsp_internal.cuh"

namespace tsp {

void partition(int nx, int ny, int nz, int zblock, int rank, int nranks, int64_t out6[6])
{
    const int nzb = (nz + zblock - 1) / zblock;
    const int zlo = (int)((int64_t)rank * nzb / nranks), zhi = (int)((int64_t)(rank + 1) * nzb / nranks);
    const int k0 = zlo * zblock, k1 = std::min(zhi * zblock, nz);
    const int64_t NP = (int64_t)(nx + 1) * (ny + 1), CP = (int64_t)nx * ny;
    const int last = rank == nranks - 1;
    out6[0] = k0; out6[1] = k1;
    out6[2] = k0 * NP; out6[3] = (int64_t)(k1 - k0 + last) * NP;
    out6[4] = k0 * CP; out6[5] = (int64_t)(k1 - k0) * CP;
}

__global__ void k_shift_cols(int64_t nnz, const int32_t *__restrict__ g, int64_t off, int32_t *__restrict__ l)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) l[q] = (int32_t)(g[q] - off);
}
__device__ int lower_bound_dev(const int32_t *a, int n, int32_t v)
{
    int lo = 0, hi = n;
    while (lo < hi) { int m = (lo + hi) >> 1; if (a[m] < v) lo = m + 1; else hi = m; }
    return lo;
}
__global__ void k_remap_cols(int64_t nnz, const int32_t *__restrict__ g, int64_t off, int nown, const int32_t *__restrict__ lo,
                             int nlo, const int32_t *__restrict__ hi, int nhi, int32_t *__restrict__ l)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    const int32_t c = g[q];
    if (c >= off && c < off + nown) l[q] = (int32_t)(c - off);
    else if (c < off) l[q] = nown + lower_bound_dev(lo, nlo, c);
    else l[q] = nown + nlo + lower_bound_dev(hi, nhi, c);
}

void halo_build(Ctx &c, Halo &H, int nown, int64_t own_off, const int32_t *gcols, int64_t nnz, int32_t *lcols)
{
    H = Halo();
    H.nown = nown;
    if (!c.comm) {
        if (nnz) k_shift_cols<<<grid_for(nnz, 256), 256, 0, c.s>>>(nnz, gcols, own_off, lcols);
        return;
    }
    std::vector<int32_t> gh(nnz);
    if (nnz) TSP_CUDA(cudaMemcpyAsync(gh.data(), gcols, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    std::vector<int32_t> lo, hi;
    for (int64_t q = 0; q < nnz; ++q) {
        const int64_t v = gh[q];
        if (v < own_off) lo.push_back((int32_t)v);
        else if (v >= own_off + nown) hi.push_back((int32_t)v);
    }
    std::sort(lo.begin(), lo.end()); lo.erase(std::unique(lo.begin(), lo.end()), lo.end());
    std::sort(hi.begin(), hi.end()); hi.erase(std::unique(hi.begin(), hi.end()), hi.end());
    TSP_REQUIRE(c.rank > 0 || lo.empty(), TSP_ERR_INVALID_ARG, "rank 0 references rows below its slab");
    TSP_REQUIRE(c.rank < c.nranks - 1 || hi.empty(), TSP_ERR_INVALID_ARG, "last rank references rows above its slab");
    // 1) request counts
    DBuf<int64_t> sc, rc;
    sc.alloc(2); rc.alloc(2); rc.zero(c.s);
    int64_t mine[2] = {(int64_t)lo.size(), (int64_t)hi.size()};
    TSP_CUDA(cudaMemcpyAsync(sc, mine, sizeof(mine), cudaMemcpyHostToDevice, c.s));
    c.comm->neighbor_exchange(sc.p, sizeof(int64_t), rc.p, sizeof(int64_t), sc.p + 1, sizeof(int64_t), rc.p + 1, sizeof(int64_t), c.s);
    int64_t req[2];
    TSP_CUDA(cudaMemcpyAsync(req, rc, sizeof(req), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    if (c.rank == 0) req[0] = 0;
    if (c.rank == c.nranks - 1) req[1] = 0;
    // 2) request lists (global ids); what the neighbours need from me comes back
    DBuf<int32_t> slo, shi, rlo, rhi;
    slo.alloc(std::max<size_t>(lo.size(), 1)); shi.alloc(std::max<size_t>(hi.size(), 1));
    rlo.alloc(std::max<int64_t>(req[0], 1)); rhi.alloc(std::max<int64_t>(req[1], 1));
    if (!lo.empty()) TSP_CUDA(cudaMemcpyAsync(slo, lo.data(), sizeof(int32_t) * lo.size(), cudaMemcpyHostToDevice, c.s));
    if (!hi.empty()) TSP_CUDA(cudaMemcpyAsync(shi, hi.data(), sizeof(int32_t) * hi.size(), cudaMemcpyHostToDevice, c.s));
    c.comm->neighbor_exchange(slo.p, sizeof(int32_t) * lo.size(), rlo.p, sizeof(int32_t) * req[0], shi.p,
                              sizeof(int32_t) * hi.size(), rhi.p, sizeof(int32_t) * req[1], c.s);
    std::vector<int32_t> want((size_t)(req[0] + req[1]));
    if (req[0]) TSP_CUDA(cudaMemcpyAsync(want.data(), rlo, sizeof(int32_t) * req[0], cudaMemcpyDeviceToHost, c.s));
    if (req[1]) TSP_CUDA(cudaMemcpyAsync(want.data() + req[0], rhi, sizeof(int32_t) * req[1], cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    for (auto &w : want) {
        TSP_REQUIRE(w >= own_off && w < own_off + nown, TSP_ERR_INVALID_ARG, "halo request outside the owned range");
        w = (int32_t)(w - own_off);
    }
    H.nsend[0] = (int)req[0]; H.nsend[1] = (int)req[1];
    H.nrecv[0] = (int)lo.size(); H.nrecv[1] = (int)hi.size();
    H.sidx.alloc(std::max<size_t>(want.size(), 1));
    if (!want.empty()) TSP_CUDA(cudaMemcpyAsync(H.sidx, want.data(), sizeof(int32_t) * want.size(), cudaMemcpyHostToDevice, c.s));
    H.sbuf.alloc(std::max<size_t>(want.size(), 1) * 3);
    if (nnz) k_remap_cols<<<grid_for(nnz, 256), 256, 0, c.s>>>(nnz, gcols, own_off, nown, slo, (int)lo.size(), shi, (int)hi.size(), lcols);
    TSP_CUDA(cudaStreamSynchronize(c.s));
    H.glo = std::move(slo);
    H.ghi = std::move(shi);
    c.launches++;
}

void halo_remap(Ctx &c, const Halo &H, int64_t own_off, const int32_t *gcols, int64_t nnz, int32_t *lcols)
{
    if (!c.comm) {
        if (nnz) k_shift_cols<<<grid_for(nnz, 256), 256, 0, c.s>>>(nnz, gcols, own_off, lcols);
        return;
    }
    if (nnz) k_remap_cols<<<grid_for(nnz, 256), 256, 0, c.s>>>(nnz, gcols, own_off, H.nown, H.glo, H.nrecv[0], H.ghi, H.nrecv[1], lcols);
    c.launches++;
}

__global__ void k_pack(int n, int nc, const int32_t *__restrict__ idx, const double *__restrict__ x, double *__restrict__ out)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n * nc) return;
    const int r = k / nc, e = k - r * nc;
    out[k] = x[(int64_t)idx[r] * nc + e];
}

void halo_exchange(Ctx &c, Halo &H, int nc, const double *x_own, double *ghost, cudaStream_t s)
{
    if (!c.comm || !H.any()) return;
    const int ns = H.nsend[0] + H.nsend[1];
    if (ns) k_pack<<<grid_for((int64_t)ns * nc, 256), 256, 0, s>>>(ns, nc, H.sidx, x_own, H.sbuf);
    c.launches++;
    const size_t b = sizeof(double) * nc;
    c.comm->neighbor_exchange(H.sbuf.p, b * H.nsend[0], ghost, b * H.nrecv[0], H.sbuf.p + (size_t)H.nsend[0] * nc,
                              b * H.nsend[1], ghost + (size_t)H.nrecv[0] * nc, b * H.nrecv[1], s);
}
void halo_exchange(Ctx &c, Halo &H, int nc, const double *x_own, double *ghost) { halo_exchange(c, H, nc, x_own, ghost, c.s); }

// ------------------------------------------------------------------ reduction layout (R-reduce)
// The global vector [u | f] is cut into SEGMENTS: the u rows of each z-block's node
// planes, then the f rows of each z-block's cell planes (global order: u of z-block
// 0..nzb-1, then f of z-block 0..nzb-1).  A rank owns whole z-blocks, hence whole
// segments.  Each segment is cut into chunks of CH values from its start (one CTA
// each, fixed tree), the chunks of a segment are summed by a fixed tree, and the
// segment sums of all ranks are added in global segment order: the result does not
// depend on the number of ranks.
constexpr int64_t CH = kRedChunk;

void reduce_setup(Ctx &c)
{
    const int zb = c.o.zblock, nzb = (c.nz_glob + zb - 1) / zb;
    const int64_t NP = (int64_t)(c.nx + 1) * (c.ny + 1), CP = (int64_t)c.nx * c.ny;
    auto ulen = [&](int b) { const int p0 = b * zb, p1 = std::min((b + 1) * zb, c.nz_glob) + (b == nzb - 1 ? 1 : 0); return 3 * NP * (p1 - p0); };
    auto flen = [&](int b) { const int p0 = b * zb, p1 = std::min((b + 1) * zb, c.nz_glob); return 2 * CP * (p1 - p0); };
    const int zlo = c.k0 / zb, zhi = (c.k1 + zb - 1) / zb;
    std::vector<int64_t> be;            // [beg, end) per local chunk
    std::vector<int32_t> segc(1, 0);    // first chunk of each local segment
    std::vector<int64_t> gseg;          // global index of each local segment
    int64_t off = 0;
    for (int part = 0; part < 2; ++part)
        for (int b = zlo; b < zhi; ++b) {
            const int64_t len = part == 0 ? ulen(b) : flen(b);
            for (int64_t k = 0; k * CH < len; ++k) { be.push_back(off + k * CH); be.push_back(off + std::min((k + 1) * CH, len)); }
            off += len;
            segc.push_back((int32_t)(be.size() / 2));
            gseg.push_back(part == 0 ? b : nzb + b);
        }
    TSP_REQUIRE(off == c.n, TSP_ERR_INVALID_ARG, "reduction segments do not cover the owned rows");
    c.nchunk_loc = (int)(be.size() / 2);
    c.nseg_loc = (int)gseg.size();
    c.nseg_glob = 2 * nzb;
    c.chunk_beg.alloc(std::max<size_t>(be.size(), 2));
    if (!be.empty()) TSP_CUDA(cudaMemcpyAsync(c.chunk_beg, be.data(), sizeof(int64_t) * be.size(), cudaMemcpyHostToDevice, c.s));
    c.seg_chunk.alloc(segc.size());
    TSP_CUDA(cudaMemcpyAsync(c.seg_chunk, segc.data(), sizeof(int32_t) * segc.size(), cudaMemcpyHostToDevice, c.s));
    std::vector<int64_t> cnt = host_allgather<int64_t>(c, std::vector<int64_t>{(int64_t)c.nseg_loc});
    int64_t mx = 0;
    for (auto v : cnt) mx = std::max(mx, v);
    c.nseg_max = (int)mx;
    std::vector<int64_t> mine(c.nseg_max, -1);
    for (int k = 0; k < c.nseg_loc; ++k) mine[k] = gseg[k];
    std::vector<int64_t> all = host_allgather<int64_t>(c, mine);
    std::vector<int32_t> perm(c.nseg_glob, -1);
    for (int r = 0; r < (c.comm ? c.nranks : 1); ++r)
        for (int k = 0; k < c.nseg_max; ++k) {
            const int64_t g = all[(size_t)r * c.nseg_max + k];
            if (g >= 0) perm[g] = r * c.nseg_max + k;
        }
    for (auto p : perm) TSP_REQUIRE(p >= 0, TSP_ERR_INVALID_ARG, "reduction segments not covered by the ranks");
    c.seg_perm.alloc(perm.size());
    TSP_CUDA(cudaMemcpyAsync(c.seg_perm, perm.data(), sizeof(int32_t) * perm.size(), cudaMemcpyHostToDevice, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
}

}  // namespace tsp

extern "C" tsp_status tsp_partition(int nx, int ny, int nz, int zblock, int rank, int nranks, int64_t out6[6])
{
    if (!out6 || nx <= 0 || ny <= 0 || nz <= 0 || zblock <= 0 || nranks <= 0 || rank < 0 || rank >= nranks) {
        tsp::set_error("tsp_partition: bad arguments");
        return TSP_ERR_INVALID_ARG;
    }
    tsp::partition(nx, ny, nz, zblock, rank, nranks, out6);
    return TSP_OK;
}

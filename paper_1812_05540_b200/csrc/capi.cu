// capi.cu -- the C-ABI of include/tsp.h: validation, deep copy, phase split
// (P:519), profiling hooks, parity export.  Host orchestration only;
// every numerical step is a kernel in apply.cu / amg.cu / ilu.cu / krylov.cu.
#include <cstdio>
#include <cstring>
#include <list>
#include <map>
#include <mutex>

#include "tsp_internal.cuh"

namespace tsp {

static thread_local std::string g_err;
thread_local cudaStream_t g_alloc_stream = 0;
thread_local AllocState *g_alloc_state = nullptr;
void set_error(const std::string &m) { g_err = m; }
static bool dbg_on() { static const bool on = getenv("TSP_DEBUG") != nullptr; return on; }
double dbg_now()
{
    if (!dbg_on()) return 0.0;
    timespec t; clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}
// per-stream cache of released device blocks, exact size (see tsp_internal.cuh); bounded, LRU-evicted
namespace {
struct Cache {
    std::multimap<size_t, void *> free;
    std::list<std::pair<size_t, void *>> lru;   // insertion order, for eviction
    size_t bytes = 0;
};
std::mutex g_cache_mu;
std::map<cudaStream_t, Cache> g_cache;
constexpr size_t kCacheMax = size_t(48) << 30;
}  // namespace
void *dev_alloc(size_t bytes, cudaStream_t s, AllocState *as)
{
    if (as && as->al.alloc) {                      // the caller's allocator (tsp_desc.allocator)
        void *p = as->al.alloc(bytes, (void *)s, as->al.ctx);
        TSP_REQUIRE(p != nullptr, TSP_ERR_OOM, "tsp_desc.allocator returned NULL");
        as->n_cb++;
        as->bytes_live += (int64_t)bytes;
        return p;
    }
    if (as) { as->n_pool++; as->bytes_live += (int64_t)bytes; }
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto &C = g_cache[s];
        auto it = C.free.find(bytes);
        if (it != C.free.end()) {
            void *p = it->second;
            C.free.erase(it);
            for (auto l = C.lru.begin(); l != C.lru.end(); ++l)
                if (l->second == p) { C.lru.erase(l); break; }
            C.bytes -= bytes;
            return p;
        }
    }
    void *p = nullptr;
    const double t0 = dbg_now();
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e == cudaErrorMemoryAllocation) {          // give the cached blocks back and retry once
        (void)cudaGetLastError();
        dev_cache_flush(s);
        e = cudaMallocAsync(&p, bytes, s);
    }
    TSP_CUDA(e);
    dbg_alloc(t0, bytes);
    return p;
}
void dev_free(void *p, size_t bytes, cudaStream_t s, AllocState *as)
{
    if (as) as->bytes_live -= (int64_t)bytes;
    if (as && as->al.alloc) { as->al.free(p, bytes, (void *)s, as->al.ctx); return; }
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto &C = g_cache[s];
    C.free.emplace(bytes, p);
    C.lru.emplace_back(bytes, p);
    C.bytes += bytes;
    while (C.bytes > kCacheMax && !C.lru.empty()) {
        auto [b, q] = C.lru.front();
        C.lru.pop_front();
        auto range = C.free.equal_range(b);
        for (auto it = range.first; it != range.second; ++it)
            if (it->second == q) { C.free.erase(it); break; }
        C.bytes -= b;
        cudaFreeAsync(q, s);
    }
}
void dev_cache_flush(cudaStream_t s)
{
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(s);
    if (it == g_cache.end()) return;
    for (auto &kv : it->second.free) cudaFreeAsync(kv.second, s);
    g_cache.erase(it);
}

void dbg_alloc(double t0, size_t bytes)
{
    if (!dbg_on()) return;
    const double dt = dbg_now() - t0;
    if (dt > 2e-3) fprintf(stderr, "[tsp alloc] %.1f MB took %.1f ms\n", bytes / 1e6, dt * 1e3);
}

StreamScope::StreamScope(cudaStream_t s, AllocState *as) : prev_stream(g_alloc_stream), prev_state(g_alloc_state)
{
    g_alloc_stream = s;
    g_alloc_state = as;
    // per call (idempotent, thread-safe, ~1 us): the pool belongs to the current device
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}
StreamScope::~StreamScope() { g_alloc_stream = prev_stream; g_alloc_state = prev_state; }

void *scratch(Ctx &c, size_t bytes)
{
    if (bytes > c.scratch_bytes) {
        c.scratch.alloc(bytes);
        c.scratch_bytes = bytes;
    }
    return c.scratch.p;
}

static const char *kProfNames[PK_COUNT] = {
    "op_node", "op_cell", "step2", "step34", "ilu_steps678", "vc_pre_u", "vc_restr_u", "vc_prol_u", "vc_post_u",
    "vc_pre_p", "vc_restr_p", "vc_prol_p", "vc_post_p", "coarse", "mdot", "maxpy", "norm", "vec", "setup",
    "vc_pre_u_l0", "vc_restr_u_l0", "vc_prol_u_l0", "vc_post_u_l0", "vc_pre_p_l0", "vc_restr_p_l0", "vc_prol_p_l0",
    "vc_post_p_l0"};

// Every launch of a profiled class is bracketed by two events from a pool that
// grows on demand (up to 4M events); prof_end only closes a record that the
// matching prof_begin opened.
void prof_begin(Ctx &c, int cls)
{
    Prof &p = c.prof;
    p.open = false;
    if (!p.on || !((p.mask >> cls) & 1u)) return;
    if (p.next + 2 > (int)p.pool.size()) {
        if (p.pool.size() >= (1u << 22)) return;
        size_t old = p.pool.size();
        p.pool.resize(old ? 2 * old : 4096);
        for (size_t k = old; k < p.pool.size(); ++k)
            if (cudaEventCreate(&p.pool[k]) != cudaSuccess) { p.pool.resize(k); return; }
        if (p.next + 2 > (int)p.pool.size()) return;
    }
    p.recs.push_back({cls, p.next, p.next + 1, 0.0});
    cudaEventRecord(p.pool[p.next], c.s);
    p.next += 2;
    p.open = true;
}
void prof_end(Ctx &c, int cls, double bytes)
{
    Prof &p = c.prof;
    if (!p.on || !p.open) return;
    p.open = false;
    Prof::Rec &r = p.recs.back();
    if (r.cls != cls) return;
    r.bytes = bytes;
    cudaEventRecord(p.pool[r.e1], c.s);
}

// the halo-overlap stream and events of a sharded handle (created with its communicator in tsp_create)
static void comm_stream_free(Ctx &c)
{
    if (c.cs) cudaStreamSynchronize(c.cs);
    if (c.ev_x) cudaEventDestroy(c.ev_x);
    if (c.ev_h) cudaEventDestroy(c.ev_h);
    if (c.cs) cudaStreamDestroy(c.cs);
    c.cs = nullptr; c.ev_x = c.ev_h = nullptr;
}

}  // namespace tsp

using namespace tsp;


#define API_BEGIN try { StreamScope ss_(h ? h->s : (cudaStream_t)0, h ? &h->alloc : nullptr);
#define API_END                                                                                     \
    }                                                                                               \
    catch (const tsp::Error &e) {                                                                   \
        set_error(e.msg);                                                                           \
        return e.st;                                                                                \
    }                                                                                               \
    catch (const std::bad_alloc &) {                                                                \
        set_error("host allocation failed");                                                        \
        return TSP_ERR_OOM;                                                                         \
    }                                                                                               \
    catch (const std::exception &e) {                                                               \
        set_error(e.what());                                                                        \
        return TSP_ERR_CUDA;                                                                        \
    }                                                                                               \
    catch (...) {                                                                                   \
        set_error("unknown exception");                                                             \
        return TSP_ERR_CUDA;                                                                        \
    }                                                                                               \
    return TSP_OK;

// status of the exception in flight (inside a catch block): every exception is mapped, none escapes extern "C"
tsp_status tsp::status_of_current_exception()
{
    try { throw; }
    catch (const tsp::Error &e) { set_error(e.msg); return e.st; }
    catch (const std::bad_alloc &) { set_error("host allocation failed"); return TSP_ERR_OOM; }
    catch (const std::exception &e) { set_error(e.what()); return TSP_ERR_CUDA; }
    catch (...) { set_error("unknown exception"); return TSP_ERR_CUDA; }
}

extern "C" {

int tsp_abi_version(void) { return TSP_ABI_VERSION; }
const char *tsp_last_error(void) { return g_err.c_str(); }

tsp_status tsp_default_options(tsp_options *o)
{
    if (!o) { set_error("null options"); return TSP_ERR_INVALID_ARG; }
    memset(o, 0, sizeof(*o));
    o->amg_theta = 0.25; o->amg_coarse_max = 64; o->amg_max_levels = 12; o->zblock = 16;
    o->tile_x = o->tile_y = o->tile_z = 16;
    o->rsl_iters = 2; o->fs_modulus_scale = 1.0;
    o->second_stage = 0; o->local_sweeps = 1;
    o->amg_smoother = 0; o->amg_gs_block = 1024;
    o->amg_cheb_degree = 2; o->amg_cheb_lower = 0.3;
    o->amg_smoother_p = -1;
    return TSP_OK;
}

void tsp_default_solve_opts(tsp_solve_opts *o)
{
    if (!o) return;
    o->rtol = 1e-8; o->restart = 64; o->max_iters = 1000; o->x0_zero = 1; o->host_ptrs = 0;
}

tsp_status tsp_create(tsp_handle *out, const tsp_desc *d)
{
    if (!out || !d) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    *out = nullptr;
    tsp_ctx *c = nullptr;
    tsp_handle h = nullptr;
    API_BEGIN
    TSP_REQUIRE(d->nx > 0 && d->ny > 0 && d->nz > 0, TSP_ERR_INVALID_ARG, "grid dimensions must be positive");
    TSP_REQUIRE(d->nranks >= 1 && d->rank >= 0 && d->rank < d->nranks, TSP_ERR_INVALID_ARG, "bad rank / nranks");
    const tsp_bsr *bs[4] = {&d->A_uu, &d->A_uf, &d->A_fu, &d->A_ff};
    for (int k = 0; k < 4; ++k)
        TSP_REQUIRE(bs[k]->rowptr && bs[k]->col && bs[k]->val, TSP_ERR_INVALID_ARG, "null matrix pointer");
    TSP_REQUIRE(d->fs_diag, TSP_ERR_INVALID_ARG, "null fs_diag");
    c = new tsp_ctx();
    c->s = (cudaStream_t)d->stream;
    TSP_REQUIRE(!d->allocator.alloc == !d->allocator.free, TSP_ERR_INVALID_ARG, "allocator: alloc and free go together");
    c->alloc.al = d->allocator;
    StreamScope ss2_(c->s, &c->alloc);
    c->o = d->opts;
    if (c->o.amg_theta <= 0 || c->o.amg_coarse_max <= 0) { int rr = c->o.replicate_rows; tsp_default_options(&c->o); c->o.replicate_rows = rr; }
    if (c->o.zblock <= 0) c->o.zblock = 16;
    if (c->o.tile_x <= 0 || c->o.tile_y <= 0 || c->o.tile_z <= 0) c->o.tile_x = c->o.tile_y = c->o.tile_z = 16;
    if (c->o.replicate_rows <= 0) c->o.replicate_rows = 32768;
    if (c->o.rsl_iters <= 0) c->o.rsl_iters = 2;
    if (c->o.local_sweeps <= 0) c->o.local_sweeps = 1;
    TSP_REQUIRE(c->o.second_stage == 0 || c->o.second_stage == 1, TSP_ERR_INVALID_ARG, "second_stage must be 0 (ILU0) or 1 (BGS)");
    if (c->o.amg_gs_block <= 0) c->o.amg_gs_block = 1024;
    TSP_REQUIRE(c->o.amg_smoother >= 0 && c->o.amg_smoother <= 2, TSP_ERR_INVALID_ARG,
                "amg_smoother must be 0 (l1-Jacobi), 1 (GS) or 2 (Chebyshev)");
    TSP_REQUIRE(c->o.amg_smoother_p >= -1 && c->o.amg_smoother_p <= 2, TSP_ERR_INVALID_ARG,
                "amg_smoother_p must be -1 (as amg_smoother), 0, 1 or 2");
    if (c->o.amg_cheb_degree == 0) c->o.amg_cheb_degree = 2;
    if (c->o.amg_cheb_lower == 0.0) c->o.amg_cheb_lower = 0.3;
    TSP_REQUIRE(c->o.amg_cheb_degree >= 1 && c->o.amg_cheb_degree <= 8, TSP_ERR_INVALID_ARG, "amg_cheb_degree must be in [1, 8]");
    TSP_REQUIRE(c->o.amg_cheb_lower > 0.0 && c->o.amg_cheb_lower < 1.0, TSP_ERR_INVALID_ARG, "amg_cheb_lower must be in (0, 1)");
    if (!(c->o.fs_modulus_scale > 0)) c->o.fs_modulus_scale = 1.0;
    TSP_REQUIRE(c->o.cpr_mode == 0 || c->o.cpr_mode == 1, TSP_ERR_INVALID_ARG, "cpr_mode must be 0 (quasi) or 1 (true IMPES)");
    TSP_REQUIRE(c->o.aps_mode == 0 || c->o.aps_mode == 1, TSP_ERR_INVALID_ARG, "aps_mode must be 0 (full) or 1 (diagonal)");
    TSP_REQUIRE(c->o.fs_mode == 0 || c->o.fs_mode == 1, TSP_ERR_INVALID_ARG, "fs_mode must be 0 (given) or 1 (RSL)");
    // z-slab partition (include/tsp.h): local sizes in Nn, Nc, n, nz
    c->rank = d->rank; c->nranks = d->nranks;
    c->nx = d->nx; c->ny = d->ny; c->nz_glob = d->nz;
    const int nzb = (d->nz + c->o.zblock - 1) / c->o.zblock;
    TSP_REQUIRE(d->nranks <= nzb, TSP_ERR_INVALID_ARG, "more ranks than z-blocks");
    int64_t part[6];
    partition(d->nx, d->ny, d->nz, c->o.zblock, d->rank, d->nranks, part);
    c->k0 = (int)part[0]; c->k1 = (int)part[1];
    c->node_off = part[2]; c->Nn = (int)part[3]; c->cell_off = part[4]; c->Nc = (int)part[5];
    c->nz = c->k1 - c->k0;
    c->Nn_glob = (int64_t)(d->nx + 1) * (d->ny + 1) * (d->nz + 1);
    c->Nc_glob = (int64_t)d->nx * d->ny * d->nz;
    c->n = 3 * (int64_t)c->Nn + 2 * (int64_t)c->Nc;
    c->n_glob = 3 * c->Nn_glob + 2 * c->Nc_glob;
    if (d->nranks > 1) {
        TSP_REQUIRE(d->comm_kind == TSP_COMM_NCCL || d->comm_kind == TSP_COMM_LOCAL, TSP_ERR_INVALID_ARG,
                    "nranks > 1 needs a communicator (comm_kind)");
        c->comm = make_comm(d->comm_kind, (void *)d->comm_arg, d->rank, d->nranks);
        TSP_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));      // halo overlap (apply.cu)
        TSP_CUDA(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
        TSP_CUDA(cudaEventCreateWithFlags(&c->ev_h, cudaEventDisableTiming));
    }
    int dev = 0;
    TSP_CUDA(cudaGetDevice(&dev));
    TSP_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev));
    const bool on_dev = d->inputs_on_device != 0;
    csr_upload(*c, c->uu, c->Nn, (int)c->Nn_glob, 9, d->A_uu.rowptr, d->A_uu.col, d->A_uu.val, on_dev);
    csr_upload(*c, c->uf, c->Nn, (int)c->Nc_glob, 6, d->A_uf.rowptr, d->A_uf.col, d->A_uf.val, on_dev);
    csr_upload(*c, c->fu, c->Nc, (int)c->Nn_glob, 6, d->A_fu.rowptr, d->A_fu.col, d->A_fu.val, on_dev);
    csr_upload(*c, c->ff, c->Nc, (int)c->Nc_glob, 4, d->A_ff.rowptr, d->A_ff.col, d->A_ff.val, on_dev);
    check_csr(*c, c->uu, "A_uu"); check_csr(*c, c->uf, "A_uf"); check_csr(*c, c->fu, "A_fu"); check_csr(*c, c->ff, "A_ff");
    // global -> local column ids; halo plans of the node (u) and cell (f) spaces
    if (c->comm) {
        Csr *ms[4] = {&c->uu, &c->uf, &c->fu, &c->ff};
        for (Csr *A : ms) {
            A->gci.alloc(std::max<int64_t>(A->nnz, 1));
            if (A->nnz) TSP_CUDA(cudaMemcpyAsync(A->gci, A->ci, 4 * A->nnz, cudaMemcpyDeviceToDevice, c->s));
        }
        halo_build(*c, c->hu, c->Nn, c->node_off, c->uu.gci, c->uu.nnz, c->uu.ci);
        halo_remap(*c, c->hu, c->node_off, c->fu.gci, c->fu.nnz, c->fu.ci);
        halo_build(*c, c->hf, c->Nc, c->cell_off, c->ff.gci, c->ff.nnz, c->ff.ci);
        halo_remap(*c, c->hf, c->cell_off, c->uf.gci, c->uf.nnz, c->uf.ci);
        c->gh_u.alloc((size_t)std::max(c->hu.nghost(), 1) * 3);
        c->gh_f.alloc((size_t)std::max(c->hf.nghost(), 1) * 2);
        c->gh_f2.alloc((size_t)std::max(c->hf.nghost(), 1) * 2);
        c->gh_dss.alloc((size_t)std::max(c->hf.nghost(), 1));
    } else {
        c->hu.nown = c->Nn; c->hf.nown = c->Nc;
    }
    reduce_setup(*c);
    c->fs.alloc(2 * (size_t)std::max(c->Nc, 1));
    if (c->Nc) TSP_CUDA(cudaMemcpyAsync(c->fs, d->fs_diag, sizeof(double) * 2 * c->Nc, on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->s));
    TSP_REQUIRE(all_nonneg(*c, c->fs, 2 * (int64_t)c->Nc), TSP_ERR_INVALID_ARG, "negative fixed-stress diagonal (S:355)");
    // structured symmetric A_uu (sym.cu) when it applies, else the SELL copy of A_uu
    sym_build(*c);
    if (!c->sym_uu.ok) sell_from_csr(*c, c->uu, c->s_uu, 9);
    sell_from_csr(*c, c->uf, c->s_uf, 6);
    sell_from_csr(*c, c->fu, c->s_fu, 6);
    sell_from_csr(*c, c->ff, c->s_ff, 4);
    // keep only what the setup phases read: A_uu's pattern + SDC values (a2), A_ff in full (a1, a3, a5)
    extract_sdc(*c);
    c->uu.v.release();
    for (Csr *A : {&c->uf, &c->fu}) A->v.release();   // patterns stay (tsp_update_values checks them)
    c->w_yf.alloc(2 * (size_t)c->Nc); c->w_wp.alloc(c->Nc); c->w_zp.alloc(c->Nc); c->w_tmp.alloc(c->Nc);
    c->kx.alloc(c->n); c->kb.alloc(c->n);
    c->dcount.alloc(4);
    TSP_CUDA(cudaStreamSynchronize(c->s));
    *out = c;
    return TSP_OK;
    }
    catch (...) {
        const tsp_status st = status_of_current_exception();
        (void)h;
        if (c) { Comm *cm = c->comm; comm_stream_free(*c); delete c; delete cm; }
        return st;
    }
}

tsp_status tsp_setup(tsp_handle h, unsigned what)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    krylov_graphs_drop(*h);             // the graphs bake in the hierarchy's buffer addresses
    TSP_REQUIRE(!(what & TSP_SETUP_REFRESH) || (what & TSP_SETUP_FLOW), TSP_ERR_INVALID_ARG,
                "TSP_SETUP_REFRESH goes with TSP_SETUP_FLOW");
    if (what & TSP_SETUP_MECH) setup_mech(*h);
    if (what & TSP_SETUP_FLOW) setup_flow(*h, (what & TSP_SETUP_REFRESH) != 0);
    TSP_CUDA(cudaStreamSynchronize(h->s));
    API_END
}

// 1 if (rp, ci) of `a` and `b` differ anywhere (rows n, entries nnz)
__global__ void k_pattern_diff(int n, int64_t nnz, const int32_t *__restrict__ rpa, const int32_t *__restrict__ cia,
                               const int32_t *__restrict__ rpb, const int32_t *__restrict__ cib, unsigned *flag)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if ((t <= n && rpa[t] != rpb[t]) || (t < nnz && cia[t] != cib[t])) atomicOr(flag, 1u);
}

tsp_status tsp_update_values(tsp_handle h, const tsp_desc *d)
{
    if (!h || !d) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    Ctx &c = *h;
    TSP_REQUIRE(d->nx == c.nx && d->ny == c.ny && d->nz == c.nz_glob && d->rank == c.rank && d->nranks == c.nranks,
                TSP_ERR_INVALID_ARG, "update_values: grid or rank differs from tsp_create");
    const tsp_bsr *bs[4] = {&d->A_uu, &d->A_uf, &d->A_fu, &d->A_ff};
    for (int k = 0; k < 4; ++k)
        TSP_REQUIRE(bs[k]->rowptr && bs[k]->col && bs[k]->val, TSP_ERR_INVALID_ARG, "null matrix pointer");
    TSP_REQUIRE(d->fs_diag, TSP_ERR_INVALID_ARG, "null fs_diag");
    const bool on_dev = d->inputs_on_device != 0;
    Csr *cur[4] = {&c.uu, &c.uf, &c.fu, &c.ff};
    const int ncv[4] = {9, 6, 6, 4};
    const char *names[4] = {"A_uu", "A_uf", "A_fu", "A_ff"};
    Csr nw[4];
    DBuf<unsigned> flag; flag.alloc(1);
    for (int k = 0; k < 4; ++k) {             // upload + compare with the stored pattern (global column ids)
        const Csr &A = *cur[k];
        csr_upload(c, nw[k], A.n, A.m, ncv[k], bs[k]->rowptr, bs[k]->col, bs[k]->val, on_dev);
        TSP_REQUIRE(nw[k].nnz == A.nnz, TSP_ERR_INVALID_ARG, std::string("update_values: ") + names[k] + " pattern changed");
        flag.zero(c.s);
        k_pattern_diff<<<grid_for(std::max<int64_t>(A.nnz, A.n + 1), 256), 256, 0, c.s>>>(
            A.n, A.nnz, nw[k].rp, nw[k].ci, A.rp, A.gci.p ? A.gci.p : A.ci.p, flag);
        c.launches++;
        unsigned f = 0;
        TSP_CUDA(cudaMemcpyAsync(&f, flag.p, sizeof(f), cudaMemcpyDeviceToHost, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
        TSP_REQUIRE(!f, TSP_ERR_INVALID_ARG, std::string("update_values: ") + names[k] + " pattern changed");
    }
    DBuf<double> fs; fs.alloc(2 * (size_t)std::max(c.Nc, 1));
    if (c.Nc) TSP_CUDA(cudaMemcpyAsync(fs, d->fs_diag, sizeof(double) * 2 * c.Nc, on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.s));
    DBuf<double> vals[4];
    for (int k = 0; k < 4; ++k) vals[k] = std::move(nw[k].v);
    commit_values(c, vals, fs);
    API_END
}

}  // extern "C"

namespace tsp {
// 1 if (rp, ci) of a device block differ from the stored pattern of A (global column ids when distributed)
bool pattern_differs(Ctx &c, const Csr &A, const int32_t *rp, const int32_t *ci)
{
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    k_pattern_diff<<<grid_for(std::max<int64_t>(A.nnz, A.n + 1), 256), 256, 0, c.s>>>(A.n, A.nnz, rp, ci, A.rp,
                                                                                  A.gci.p ? A.gci.p : A.ci.p, flag);
    c.launches++;
    unsigned f = 0;
    TSP_CUDA(cudaMemcpyAsync(&f, flag.p, sizeof(f), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    return f != 0;
}
// new values (moved in: A_uu 9, A_uf 6, A_fu 6, A_ff 4 per block entry, on the stored patterns) and D_fs; the apply
// layouts are refilled, the flow phase must be redone (tsp_update_values)
void commit_values(Ctx &c, DBuf<double> vals[4], DBuf<double> &fs)
{
    TSP_REQUIRE(all_nonneg(c, fs, 2 * (int64_t)c.Nc), TSP_ERR_INVALID_ARG, "negative fixed-stress diagonal (S:355)");
    Csr *cur[4] = {&c.uu, &c.uf, &c.fu, &c.ff};
    krylov_graphs_drop(c);                    // the graphs bake in the SELL buffers' addresses
    c.fs = std::move(fs);
    for (int k = 0; k < 4; ++k) cur[k]->v = std::move(vals[k]);
    if (!sym_refill_uu(c)) sell_from_csr(c, c.uu, c.s_uu, 9);
    extract_sdc(c);                           // input of the next TSP_SETUP_MECH (a2)
    c.sdc_stale = true;
    sell_from_csr(c, c.uf, c.s_uf, 6);
    sell_from_csr(c, c.fu, c.s_fu, 6);
    sell_from_csr(c, c.ff, c.s_ff, 4);
    c.uu.v.release(); c.uf.v.release(); c.fu.v.release();
    c.flow_ready = false;                     // apply / solve wait for the flow phase on the new values
    TSP_CUDA(cudaStreamSynchronize(c.s));
}
}  // namespace tsp

extern "C" {

tsp_status tsp_apply_preconditioner(tsp_handle h, const double *v, double *z)
{
    if (!h || !v || !z) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    if (v == z) { set_error("v and z must not alias"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    prec_apply(*h, v, z);
    API_END
}

tsp_status tsp_apply_operator(tsp_handle h, const double *x, double *y)
{
    if (!h || !x || !y) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    if (x == y) { set_error("x and y must not alias"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    op_apply(*h, x, y);
    API_END
}

static tsp_status solve_entry(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info,
                              bool richardson);

tsp_status tsp_solve(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info)
{
    return solve_entry(h, b, x, o, info, false);
}

tsp_status tsp_richardson(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info)
{
    return solve_entry(h, b, x, o, info, true);
}

static tsp_status solve_entry(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info,
                              bool richardson)
{
    if (!h || !b || !x) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    tsp_solve_opts oo;
    tsp_default_solve_opts(&oo);
    if (o) oo = *o;
    tsp_solve_info inf;
    memset(&inf, 0, sizeof(inf));
    API_BEGIN
    TSP_REQUIRE(h->mech_ready && h->flow_ready, TSP_ERR_STATE, "solve before tsp_setup(MECH|FLOW)");
    TSP_REQUIRE(oo.rtol > 0 && oo.restart > 0 && oo.max_iters >= 0, TSP_ERR_INVALID_ARG, "bad solve options");
    const double *db = b;
    double *dx = x;
    if (oo.host_ptrs) {
        TSP_CUDA(cudaMemcpyAsync(h->kb, b, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->s));
        if (!oo.x0_zero) TSP_CUDA(cudaMemcpyAsync(h->kx, x, sizeof(double) * h->n, cudaMemcpyHostToDevice, h->s));
        db = h->kb; dx = h->kx;
    }
    if (richardson) richardson_solve(*h, db, dx, oo, inf);
    else krylov_solve(*h, db, dx, oo, inf);
    if (oo.host_ptrs) {
        TSP_CUDA(cudaMemcpyAsync(x, h->kx, sizeof(double) * h->n, cudaMemcpyDeviceToHost, h->s));
        TSP_CUDA(cudaStreamSynchronize(h->s));
    }
    if (info) *info = inf;
    return inf.status;
    }
    catch (...) {
        inf.status = status_of_current_exception();
        if (info) *info = inf;
        return inf.status;
    }
}

static tsp_status check_asm(const tsp_asm_params *p, int rank, int nranks, int zblock)
{
    if (!p) { set_error("null params"); return TSP_ERR_INVALID_ARG; }
    if (p->nx <= 0 || p->ny <= 0 || p->nz <= 0 || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("assembly: bad grid or rank");
        return TSP_ERR_INVALID_ARG;
    }
    const int zb = zblock > 0 ? zblock : 16;
    if (nranks > (p->nz + zb - 1) / zb) { set_error("more ranks than z-blocks"); return TSP_ERR_INVALID_ARG; }
    return TSP_OK;
}

tsp_status tsp_assembly_sizes(const tsp_asm_params *p, int rank, int nranks, int zblock, int64_t out6[6])
{
    if (tsp_status st = check_asm(p, rank, nranks, zblock)) return st;
    if (!out6) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        assembly_sizes(*p, rank, nranks, zblock, out6);
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

tsp_status tsp_assemble(const tsp_asm_params *p, int rank, int nranks, int zblock, const tsp_cell_fields *f,
                        tsp_bsr_out blocks[4], double *fs, double row_max[3], void *stream)
{
    if (tsp_status st = check_asm(p, rank, nranks, zblock)) return st;
    if (!f || !blocks || !row_max) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        StreamScope ss_((cudaStream_t)stream, nullptr);
        assemble((cudaStream_t)stream, *p, rank, nranks, zblock, *f, blocks, fs, row_max);
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

tsp_status tsp_assemble_scale(const tsp_asm_params *p, int rank, int nranks, int zblock, const double row_max[3],
                              tsp_bsr_out blocks[4], double *fs, double scales[3], void *stream)
{
    if (tsp_status st = check_asm(p, rank, nranks, zblock)) return st;
    if (!blocks || !row_max || !fs) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        StreamScope ss_((cudaStream_t)stream, nullptr);
        assemble_scale((cudaStream_t)stream, *p, rank, nranks, zblock, row_max, blocks, fs, scales);
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

tsp_status tsp_export_colour(tsp_handle h, int which, int lvl, int32_t *colour, int *block, int *ncolour)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    Hier &H = which ? h->pres : h->mech;
    TSP_REQUIRE(lvl >= 0 && lvl < (int)H.L.size(), TSP_ERR_INVALID_ARG, "no such level");
    const Level &L = H.L[lvl];
    TSP_REQUIRE(H.smoother == 1 && !L.coarsest, TSP_ERR_STATE, "no Gauss-Seidel colouring on this level");
    if (block) *block = L.gs_block;
    if (ncolour) *ncolour = L.ncolor;
    if (colour) gs_export_colour(*h, L, colour);
    API_END
}

tsp_status tsp_variant_counts(tsp_handle h, int64_t out[TSP_NVARIANTS])
{
    if (!h || !out) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    for (int k = 0; k < TSP_NVARIANTS; ++k) out[k] = h->variants[k];
    return TSP_OK;
}

tsp_status tsp_get_stats(tsp_handle h, tsp_stats *s)
{
    if (!h || !s) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    memset(s, 0, sizeof(*s));
    Hier *H[2] = {&h->mech, &h->pres};
    double apply_bytes = 0;
    for (int w = 0; w < 2; ++w) {
        s->levels[w] = (int)H[w]->L.size();
        for (size_t l = 0; l < H[w]->L.size() && l < 16; ++l) {
            const Level &L = H[w]->L[l];
            s->rows[w][l] = L.n; s->nnz[w][l] = L.A.nnz;
            const double nc = L.nc, vec = 8.0 * nc * L.n;
            if (L.coarsest) { apply_bytes += 8.0 * L.n * L.n * nc + 2 * vec; continue; }
            auto sb = [](const Sell &S) { return (double)S.slots * 32 * (4.0 + 8.0 * S.bs); };
            const double bA = (w == 0 && l == 0 && h->sym_sdc.ok) ? sym_bytes(*h, 3)
                            : (w == 1 && l == 0 && h->p7_ok) ? p7_bytes(*h) : sb(L.sA);
            apply_bytes += 2 * bA + sb(L.sR) + sb(L.sP) + 11 * vec;
        }
        s->skipped_dss = h->skipped_dss;
        s->perturbed_pivots = h->perturbed + h->mech.perturbed + h->pres.perturbed;
        s->coarsening_fallbacks = h->mech.fallbacks + h->pres.fallbacks;
    }
    s->allocs_callback = h->alloc.n_cb;
    s->allocs_pool = h->alloc.n_pool;
    s->bytes_live = h->alloc.bytes_live;
    auto sb = [](const Sell &S) { return (double)S.slots * 32 * (4.0 + 8.0 * S.bs); };
    const double Nn = h->Nn, Nc = h->Nc, n = (double)h->n;
    apply_bytes += sb(h->s_fu) + 24 * Nn + 32 * Nc;            // step 2
    apply_bytes += sb(h->s_aps) + 40 * Nc;                     // steps 3-4
    apply_bytes += (28.0 * 8 + 32 + 48) * Nc;                  // steps 6-8
    s->bytes_apply = apply_bytes;
    s->bytes_operator = (h->sym_uu.ok ? sym_bytes(*h, 9) : sb(h->s_uu)) + sb(h->s_uf) + sb(h->s_fu) + sb(h->s_ff) + 16 * n;
    // Gram-Schmidt depends on the Krylov index: counted exactly per solve (tsp_solve_info.bytes_krylov).  The
    // FGMRES operator reuses Algorithm 1's A_fu z_u (op_apply_after_prec): its cell rows stream A_ff only
    static const bool no_fuse = getenv("TSP_NO_OP_FUSE") != nullptr;
    const double op_iter = no_fuse ? s->bytes_operator : s->bytes_operator - sb(h->s_fu) - 24 * Nn + 32 * Nc;
    s->bytes_iter_base = s->bytes_apply + op_iter;
    s->bytes_per_krylov_vec = 8 * n;
    s->launches = h->launches;
    return TSP_OK;
}

tsp_status tsp_level_sizes(tsp_handle h, int which, int lvl, int64_t out6[6])
{
    if (!h || !out6) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    Hier &H = which ? h->pres : h->mech;
    if (lvl < 0 || lvl >= (int)H.L.size()) { set_error("level out of range"); return TSP_ERR_INVALID_ARG; }
    const Level &L = H.L[lvl];
    out6[0] = L.n; out6[1] = L.A.nnz; out6[2] = L.nagg; out6[3] = L.coarsest ? 0 : L.P.nnz; out6[4] = L.nc; out6[5] = L.coarsest;
    return TSP_OK;
}

tsp_status tsp_export_level(tsp_handle h, int which, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v, int32_t *agg,
                            int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    Hier &H = which ? h->pres : h->mech;
    if (lvl < 0 || lvl >= (int)H.L.size()) { set_error("level out of range"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    Level &L = H.L[lvl];
    cudaStream_t s = h->s;
    auto cp = [&](void *dst, const void *src, size_t bytes) {
        if (dst && bytes) TSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    cp(A_rp, L.A.rp, sizeof(int32_t) * (L.n + 1));
    cp(A_ci, L.A.gci.p ? L.A.gci.p : L.A.ci.p, sizeof(int32_t) * L.A.nnz);   // global column ids
    cp(A_v, L.A.v, sizeof(double) * L.A.nnz * L.nc);
    cp(dl1, L.dl1, sizeof(double) * L.n * L.nc);
    if (!L.coarsest) {
        cp(agg, L.agg, sizeof(int32_t) * L.n);
        cp(P_rp, L.P.rp, sizeof(int32_t) * (L.n + 1));
        cp(P_ci, L.P.ci, sizeof(int32_t) * L.P.nnz);
        cp(P_v, L.P.v, sizeof(double) * L.P.nnz * L.nc);
    }
    TSP_CUDA(cudaStreamSynchronize(s));
    if (!L.coarsest && L.coarse_off) {     // aggregate / coarse ids exported in global numbering
        if (agg) for (int i = 0; i < L.n; ++i) if (agg[i] >= 0) agg[i] += (int32_t)L.coarse_off;
        if (P_ci && L.next_dist) for (int64_t q = 0; q < L.P.nnz; ++q) P_ci[q] += (int32_t)L.coarse_off;
    }
    API_END
}

tsp_status tsp_level_dist(tsp_handle h, int which, int lvl, int64_t out3[3])
{
    if (!h || !out3) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    Hier &H = which ? h->pres : h->mech;
    if (lvl < 0 || lvl >= (int)H.L.size()) { set_error("level out of range"); return TSP_ERR_INVALID_ARG; }
    const Level &L = H.L[lvl];
    out3[0] = L.dist; out3[1] = L.dist ? L.nglob : L.n; out3[2] = L.dist ? L.row_off : 0;
    return TSP_OK;
}

tsp_status tsp_prof_enable(tsp_handle h, int on)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    Prof &p = h->prof;
    TSP_CUDA(cudaStreamSynchronize(h->s));
    p.recs.clear();
    p.next = 0;
    p.on = on != 0;
    h->launches = 0;
    API_END
}

tsp_status tsp_export_cpr(tsp_handle h, double *dss, double *dps, double *fs_eff)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    TSP_REQUIRE(h->flow_ready, TSP_ERR_STATE, "export_cpr before tsp_setup(FLOW)");
    if (dss && h->Nc) TSP_CUDA(cudaMemcpyAsync(dss, h->cpr_dss, sizeof(double) * h->Nc, cudaMemcpyDeviceToHost, h->s));
    if (dps && h->Nc) TSP_CUDA(cudaMemcpyAsync(dps, h->cpr_dps, sizeof(double) * h->Nc, cudaMemcpyDeviceToHost, h->s));
    if (fs_eff && h->Nc) TSP_CUDA(cudaMemcpyAsync(fs_eff, h->fs_eff, sizeof(double) * 2 * h->Nc, cudaMemcpyDeviceToHost, h->s));
    TSP_CUDA(cudaStreamSynchronize(h->s));
    API_END
}

tsp_status tsp_prof_classes(tsp_handle h, unsigned mask)
{
    if (!h) { set_error("null handle"); return TSP_ERR_INVALID_ARG; }
    h->prof.mask = mask;
    return TSP_OK;
}

tsp_status tsp_prof_read(tsp_handle h, tsp_prof *out)
{
    if (!h || !out) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    API_BEGIN
    memset(out, 0, sizeof(*out));
    TSP_CUDA(cudaStreamSynchronize(h->s));
    out->nclasses = PK_COUNT;
    for (int k = 0; k < PK_COUNT; ++k) snprintf(out->name[k], sizeof(out->name[k]), "%s", kProfNames[k]);
    for (auto &r : h->prof.recs) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, h->prof.pool[r.e0], h->prof.pool[r.e1]) != cudaSuccess) continue;
        out->launches[r.cls] += 1;
        out->ms[r.cls] += ms;
        out->bytes[r.cls] += r.bytes;
    }
    API_END
}

void tsp_destroy(tsp_handle h)
{
    if (!h) return;
    StreamScope ss_(h->s, &h->alloc);
    cudaStreamSynchronize(h->s);
    for (auto &e : h->prof.pool) cudaEventDestroy(e);
    krylov_graphs_drop(*h);
    if (h->kcol_host) cudaFreeHost(h->kcol_host);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    comm_stream_free(*h);
    Comm *cm = h->comm;
    cudaStream_t s = h->s;
    delete h;
    delete cm;
    dev_cache_flush(s);
    cudaStreamSynchronize(s);
}

}  // extern "C"

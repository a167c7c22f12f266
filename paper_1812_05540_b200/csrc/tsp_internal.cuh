// tsp_internal.cuh -- shared declarations of libtsp.so (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "tsp.h"

namespace tsp {

// rows per deterministic-reduction chunk (halo.cu reduce_setup; krylov.cu stages one chunk in shared memory)
constexpr int kRedChunk = 2048;

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
struct Error {
    tsp_status st;
    std::string msg;
};
#define TSP_CUDA(x)                                                                                 \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess)                                                                      \
            throw ::tsp::Error{e_ == cudaErrorMemoryAllocation ? TSP_ERR_OOM : TSP_ERR_CUDA,        \
                               std::string(#x) + ": " + cudaGetErrorString(e_)};                    \
    } while (0)
#define TSP_REQUIRE(cond, st, msg)                                                                  \
    do {                                                                                            \
        if (!(cond)) throw ::tsp::Error{st, msg};                                                   \
    } while (0)

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocation on the stream of the API call in progress, through a per-stream
// cache of released blocks keyed by exact size (capi.cu): a repeated tsp_setup requests the same
// sizes, so after the first one no allocation reaches the driver (the stream-ordered pool grew
// by a few hundred MB now and then under the interleaved lifetimes of the two hierarchies, and a
// growth step cost 0.1-0.6 s).  Reuse within one stream is safe in stream order.
// With a caller allocator (tsp_desc.allocator) every buffer goes through its callbacks instead.
struct AllocState {
    tsp_allocator al{};
    int64_t n_cb = 0, n_pool = 0, bytes_live = 0;
};
extern thread_local cudaStream_t g_alloc_stream;
extern thread_local AllocState *g_alloc_state;  // the handle whose API call is in progress on this thread
// binds the allocation stream / allocator of an API call (restores the enclosing call's on exit: API calls nest)
struct StreamScope {
    cudaStream_t prev_stream;
    AllocState *prev_state;
    explicit StreamScope(cudaStream_t s, AllocState *as = nullptr);
    ~StreamScope();
};
tsp_status status_of_current_exception();        // inside a catch block: the tsp_status of the exception
double dbg_now();                              // TSP_DEBUG: wall clock (0 when off)
void dbg_alloc(double t0, size_t bytes);       // TSP_DEBUG: report slow allocations
void *dev_alloc(size_t bytes, cudaStream_t s, AllocState *as);
void dev_free(void *p, size_t bytes, cudaStream_t s, AllocState *as);
void dev_cache_flush(cudaStream_t s);          // return the stream's cached blocks to the pool
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t st = 0;
    AllocState *as = nullptr;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), st(o.st), as(o.as) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept { release(); p = o.p; n = o.n; st = o.st; as = o.as; o.p = nullptr; o.n = 0; return *this; }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        st = g_alloc_stream;
        as = g_alloc_state;
        if (count) p = (T *)dev_alloc(sizeof(T) * count, st, as);
    }
    void zero(cudaStream_t s) { if (n) TSP_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s)); }
    void release() { if (p) dev_free(p, sizeof(T) * n, st, as); p = nullptr; n = 0; }
    operator T *() const { return p; }
};

// ------------------------------------------------------------------ sparse layouts
// CSR with nc values per entry, entry-major: v[q*nc + c].
struct Csr {
    int n = 0, m = 0, nc = 1;
    int64_t nnz = 0;
    DBuf<int32_t> rp, ci;
    DBuf<double> v;
    DBuf<int32_t> gci;            // global column ids (distributed matrices only)
};

// Sliced ELL, slice height 32, column-major inside a slice (R-layout):
//   entry (row i, slot k): index (off[i/32] + k) * 32 + i % 32
//   value e of that entry : ((off[i/32] + k) * bs + e) * 32 + i % 32
// Padding slots carry value 0 and a valid column (the row's last column, or 0).
struct Sell {
    int nrows = 0, nslices = 0, bs = 1, ncols = 0;
    int64_t slots = 0;            // total entries incl. padding
    int64_t nnz = 0;              // true entries
    DBuf<int64_t> off;            // nslices + 1
    DBuf<int32_t> col;            // slots * 32
    DBuf<double> val;             // slots * 32 * bs
};

// Structured storage of a 27-point node operator (sym.cu): no column indices (the neighbour follows
// from the grid); the block entries that are exactly symmetric over the whole matrix (B(i,j)[r][c] ==
// B(j,i)[c][r] for every pair, detected at create) are kept only for the diagonal block and the 13 "upper"
// neighbours -- a lower neighbour reads them, transposed, from that neighbour's upper slot -- and the
// other entries are kept for all 27 neighbours.  Rows whose lower z-plane belongs to rank-1 keep those
// 9 blocks' symmetric entries explicitly (gl).  Used when the pattern is the full clipped 27-point
// stencil (checked at create); the generic SELL path otherwise.
struct SymMap {
    int bs, ks, kf;               // values per block (9: A_uu, 3: SDC), symmetric / full entries
    int full[9], idx[9];          // per block entry: 1 = kept for all 27 neighbours; index in its array
    int tr[9];                    // transposed entry (bs = 9), identity for bs = 3
};
struct Sym27 {
    bool ok = false;
    SymMap m{};
    DBuf<double> val_s;           // [slice][14][ks][32]: diagonal + 13 upper blocks, symmetric entries
    DBuf<double> val_f;           // [slice][27][kf][32]: all neighbours, the other entries
    DBuf<double> gl;              // [slice of local node plane 0][9][ks][32]
};

// ------------------------------------------------------------------ multi-GPU (row e)
struct Ctx;
// Communicator of the z-slab decomposition: halos with rank-1 / rank+1, allgather.
struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() {}
    virtual void neighbor_exchange(const void *send_lo, size_t bytes_send_lo, void *recv_lo, size_t bytes_recv_lo,
                                   const void *send_hi, size_t bytes_send_hi, void *recv_hi, size_t bytes_recv_hi,
                                   cudaStream_t s) = 0;
    virtual void allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // true when every call only enqueues stream work (no host-side rendezvous), so a stream capture may hold it
    virtual bool capturable() const { return false; }
};
Comm *make_comm(int kind, void *arg, int rank, int nranks);
template <class T> std::vector<T> host_allgather(Ctx &c, const std::vector<T> &mine);

// Halo plan of a row-distributed vector (rows owned by this rank are [0, nown) locally,
// ghosts are appended: [lo neighbour's rows | hi neighbour's rows], each list ascending
// in global numbering).  nsend/nrecv index 0 = lo neighbour, 1 = hi neighbour.
struct Halo {
    int nown = 0;
    int nsend[2] = {0, 0}, nrecv[2] = {0, 0};
    DBuf<int32_t> sidx;           // owned rows to send, [lo list | hi list]
    DBuf<double> sbuf;            // pack buffer (3 values per row max)
    DBuf<int32_t> glo, ghi;       // global ids of the ghost rows (ascending), to remap other matrices
    int nghost() const { return nrecv[0] + nrecv[1]; }
    bool any() const { return nsend[0] + nsend[1] + nrecv[0] + nrecv[1] > 0; }
};
// thread -> row map of a launch over up to two row ranges (the halo overlap launches the interior rows, then
// the slab's boundary rows): t < na -> r0 + t, else r1 + (t - na)
struct Rows {
    int r0, na, r1;
};
inline Rows rows_all(int n) { return Rows{0, n, n}; }
__device__ __forceinline__ int row_of(const Rows &R, int t) { return t < R.na ? R.r0 + t : R.r1 + (t - R.na); }

// ghost-aware vector for kernels: row j < nown is own[j*nc..], else gh[(j-nown)*nc..]
struct GV {
    const double *own;
    const double *gh;
    int nown;
};
#define GVLD(g, j, c, nc) ((j) < (g).nown ? __ldg((g).own + (int64_t)(j) * (nc) + (c)) : __ldg((g).gh + (int64_t)((j) - (g).nown) * (nc) + (c)))
inline GV gv(const double *own, int nown, const double *gh = nullptr) { return GV{own, gh, nown}; }
// D = false (single rank / replicated level): no ghost test at all
template <bool D>
__device__ __forceinline__ double gvld(const GV &g, int64_t j, int c, int nc)
{
    if (D) return GVLD(g, j, c, nc);
    return __ldg(g.own + j * nc + c);
}

// Fused Chebyshev smoothing step (R-cheb; amg.cu cheb_run): the row epilogue shared by the SELL, vector-CSR and
// structured kernels.  PRE = the first two steps from zero in one product (the kernel gathers sc dinv_j b_j,
// i.e. A x_1 with x_1 = D^-1 b / theta):  x_1 = sc dinv_i b_i, d_1 = alpha x_1 + beta dinv_i (b_i - acc),
// xo = x_1 + d_1.  STEP = one step from x (the kernel gathers x_j): d = alpha dprev_i + beta dinv_i (b_i - acc)
// (dprev == nullptr: first step, d = beta dinv_i (b_i - acc)), xo = x_i + d.  dout (may be nullptr) keeps d.
struct ChebArgs {
    const double *dprev;
    double *dout;
    double alpha, beta, sc;
};
template <bool PRE>
__device__ __forceinline__ void cheb_epi(int64_t t, double acc, double bi, double di, double xi, const ChebArgs &a, double *xo)
{
    if (PRE) {
        const double x1 = a.sc * (di * bi);
        const double d = a.alpha * x1 + a.beta * (di * (bi - acc));
        if (a.dout) a.dout[t] = d;
        xo[t] = x1 + d;
    } else {
        const double d = (a.dprev ? a.alpha * a.dprev[t] : 0.0) + a.beta * (di * (bi - acc));
        if (a.dout) a.dout[t] = d;
        xo[t] = xi + d;
    }
}

// builds the plan from the GLOBAL column ids of a row-distributed CSR (own rows =
// global [own_off, own_off + nown)) and rewrites `lcols` with local ids
void halo_build(Ctx &c, Halo &H, int nown, int64_t own_off, const int32_t *gcols, int64_t nnz, int32_t *lcols);
// remap another matrix whose columns live in the same row space with an existing plan
void halo_remap(Ctx &c, const Halo &H, int64_t own_off, const int32_t *gcols, int64_t nnz, int32_t *lcols);
// exchange: ghost[(nrecv0+nrecv1)*nc] <- neighbours' rows of x_own (nc values per row)
void halo_exchange(Ctx &c, Halo &H, int nc, const double *x_own, double *ghost);
void halo_exchange(Ctx &c, Halo &H, int nc, const double *x_own, double *ghost, cudaStream_t s);

// One AMG level (setup products in CSR, apply operators in SELL).
struct Level {
    int n = 0, nc = 1, coarsest = 0, nagg = 0;
    // distribution: a level is either DISTRIBUTED (rows split over ranks like the fine
    // grid, halos with the neighbours) or REPLICATED (every rank holds all rows)
    bool dist = false;
    int64_t nglob = 0, row_off = 0;    // global rows and this rank's first row (dist)
    int64_t coarse_off = 0;            // first global id of this rank's aggregates
    bool next_dist = false;            // is level+1 distributed?
    int warpA = 0, warpR = 0;          // lanes per row of the vector-CSR kernels, 0 = sliced-ELL (chosen from
                                       // GLOBAL row lengths: the same on every rank)
    Halo halo;                         // of A's columns (dist, coarse levels)
    Halo *hp = nullptr;                // plan in use: &halo, or the fine-grid plan on level 0
    DBuf<double> dinv_gh;              // ghost copy of dinv (dist)
    DBuf<double> gh_b, gh_x;           // ghost buffers for b and x (dist)
    std::vector<int64_t> rep_counts, rep_offs;  // next level replicated: rows per rank (allgather)
    DBuf<int64_t> rep_offs_d;          // rep_offs on the device (uploaded once at setup)
    // Gauss-Seidel smoother (tsp_options.amg_smoother = 1, gs.cu): level 0 multicolour (gs_block = 0), coarse
    // levels hybrid l1-GS over blocks of gs_block rows
    int gs_block = 0, ncolor = 0;
    DBuf<int16_t> gsc;                 // hybrid: colour of each row inside its block
    DBuf<double> dh;                   // hybrid: l1 diagonal per (row, component)
    DBuf<int32_t> gcoff, gorder;       // hybrid: per block, first position of each colour in gorder (rows by colour)
    Sell sAc;                          // multicolour: colour-ordered SELL copy of A (a slice holds one colour)
    DBuf<int32_t> gperm;               // multicolour: SELL row -> level row (-1 = padding)
    std::vector<int64_t> cslice;       // multicolour: first SELL row of each colour (+ end)
    DBuf<double> diag;                 // multicolour: a_ii per (row, component)
    DBuf<double> rep_buf;              // padded allgather buffer
    Csr A;                        // level operator (local column ids if dist)
    DBuf<int32_t> zb;             // z-block per row
    DBuf<double> dl1;             // l1 row norms [n][nc]
    DBuf<double> dinv;            // 1 / dl1
    DBuf<int32_t> agg;            // aggregate per row (-1 = none)
    DBuf<uint8_t> E;              // symmetrised strength flag per entry of A (kept for the frozen refresh)
    int64_t nagg_glob = 0;        // aggregates over all ranks
    Csr P, R;
    Sell sA, sP, sR;
    DBuf<double> cinv;            // coarsest: dense inverse [nc][n][n]
    // apply work vectors [n][nc]
    DBuf<double> b, x, x2, r;
    DBuf<double> dcheb, xc;       // Chebyshev smoother (amg_smoother = 2): direction, ping-pong iterate
};

struct Hier {
    int nc = 1;
    int smoother = 0;                  // 0 l1-Jacobi, 1 Gauss-Seidel, 2 Chebyshev (options, per hierarchy)
    std::vector<Level> L;
    int64_t fallbacks = 0, perturbed = 0;
};

// ------------------------------------------------------------------ profiling
enum ProfClass {
    PK_OP_NODE, PK_OP_CELL, PK_STEP2, PK_STEP34, PK_ILU, PK_VC_PRE_U, PK_VC_RESTR_U, PK_VC_PROL_U, PK_VC_POST_U,
    PK_VC_PRE_P, PK_VC_RESTR_P, PK_VC_PROL_P, PK_VC_POST_P, PK_COARSE, PK_DOT, PK_AXPY, PK_NORM, PK_VEC, PK_SETUP,
    // the same eight V-cycle classes on level 0 alone (the bandwidth-bound launches; the classes above then hold
    // levels >= 1, which are latency-bound): same order, PK_VC_L0 apart
    PK_VC_PRE_U0, PK_VC_RESTR_U0, PK_VC_PROL_U0, PK_VC_POST_U0, PK_VC_PRE_P0, PK_VC_RESTR_P0, PK_VC_PROL_P0, PK_VC_POST_P0,
    PK_COUNT
};

constexpr int PK_VC_L0 = PK_VC_PRE_U0 - PK_VC_PRE_U;
static_assert(PK_COUNT <= TSP_PROF_MAX, "too many profile classes");

struct Prof {
    bool on = false;
    unsigned mask = ~0u;             // classes recorded while on (tsp_prof_classes)
    std::vector<cudaEvent_t> pool;
    struct Rec { int cls; int e0, e1; double bytes; };
    std::vector<Rec> recs;
    int next = 0;
    bool open = false;
};

// ------------------------------------------------------------------ the handle
struct Ctx {
    AllocState alloc;                  // FIRST member: outlives every buffer of the handle
    // Nn, Nc, n and nz are this rank's LOCAL (owned) sizes; *_glob the global ones
    int nx, ny, nz, Nn, Nc;
    int64_t n;
    int nz_glob = 0;
    int64_t Nn_glob = 0, Nc_glob = 0, n_glob = 0;
    int rank = 0, nranks = 1;
    Comm *comm = nullptr;
    // halo overlap (comm != nullptr): exchanges run on `cs` while the interior rows run on `s`
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_x = nullptr, ev_h = nullptr;
    int k0 = 0, k1 = 0;                // owned cell planes [k0, k1)
    int64_t node_off = 0, cell_off = 0;
    Halo hu, hf;                       // fine node / cell halos
    DBuf<int32_t> ff_gcol;             // A_ff global column ids (ILU fill geometry)
    DBuf<double> gh_u, gh_f, gh_f2, gh_dss;   // fine ghost buffers
    // deterministic reductions (DESIGN.md R-reduce): the global vector is cut into
    // segments (u and f rows of each z-block) and each segment into fixed chunks;
    // chunk partials -> per-segment fixed-tree sums -> allgather -> sum in global order
    int nchunk_loc = 0;
    DBuf<int64_t> chunk_beg;           // [beg, end) of each local chunk (local offsets)
    int nseg_loc = 0, nseg_max = 0, nseg_glob = 0;
    DBuf<int32_t> seg_chunk;           // first local chunk of each local segment (+ end)
    DBuf<int32_t> seg_perm;            // global segment g -> slot (rank * nseg_max + local segment)
    DBuf<double> seg_part;             // [nv][nseg_max] per-rank segment sums
    cudaStream_t s;
    tsp_options o;
    int sm_count = 148;
    // original blocks (CSR on device) for setup + SELL for apply
    Csr uu, uf, fu, ff;           // nc = values per block entry (9, 6, 6, 4); after create only the patterns of
                                  // uu and the full ff stay (A_uf, A_fu and A_uu's values live in the SELL copies)
    DBuf<double> uu_sdc;          // a2: SDC values of A_uu (3 per block), extracted at create
    Sell s_uu, s_uf, s_fu, s_ff;  // SELL copies (operator rows)
    Sym27 sym_uu, sym_sdc;        // structured symmetric A_uu (operator) and A_uu^SDC (level-0 smoother)
    bool p7_ok = false;           // structured 7-point pressure level 0 (p7.cu) in use
    DBuf<double> p7_val;          // its values [slice][7][32]
    unsigned sym_asym = 0;        // their mask of non-symmetric block entries
    DBuf<double> fs;              // 2 per cell, as given (tsp_desc.fs_diag)
    DBuf<double> fs_eff;          // 2 per cell: the D_fs a1 uses (given / fs_modulus_scale, or RSL)
    DBuf<double> cpr_dss, cpr_dps; // D_ss^(CPR), D_ps^(CPR) (a3)
    // flow setup products
    DBuf<double> dss_inv;         // 1/D_ss (0 if D_ss == 0)
    Sell s_aps;                   // A_ps values on A_ff's pattern (bs 1)
    DBuf<double> ilu_val;         // tile-level-major S_ff^FS blocks, 7 slots x 4 (R-ilu)
    DBuf<double> ilu_dinv;        // tile-level-major U_KK^-1, 4 per cell
    bool ilu_eis = true;          // slot 3 of ilu_val holds E = S_KK - U_KK (ilu.cu, Eisenstat form of steps 6-8)
    DBuf<int32_t> ilu_lvlptr;     // level pointers of the full-tile table
    DBuf<int32_t> ilu_cells;      // local (i,j,k) packed per table position
    DBuf<int32_t> ilu_posmap;     // local linear index -> table position
    int ilu_nlev = 0, ilu_tsize = 0, ntiles = 0, ntx = 0, nty = 0, ntz = 0;
    Hier mech, pres;
    bool mech_ready = false, flow_ready = false;
    bool flow_built = false;      // the last TSP_SETUP_FLOW completed (its hierarchy can be refreshed); flow_ready is
                                  // also cleared by tsp_update_values (apply / solve need the flow phase first)
    bool sdc_stale = false;       // tsp_update_values changed A_uu: sym_sdc is refilled by the next TSP_SETUP_MECH
    // work vectors
    DBuf<double> w_yf, w_wp, w_zp, w_zf2, w_tmp;
    // Krylov storage
    DBuf<double> V, Z, kw, kr, kx, kb, kh, kpart;
    int kcap = 0;
    // CUDA graphs of the FGMRES iteration body, one per Krylov index j (krylov.cu); dropped by every
    // tsp_setup and basis reallocation (they bake in buffer addresses)
    struct KGraph { cudaGraphExec_t exec = nullptr; bool seen = false, failed = false; int64_t launches = 0; double bytes = 0; };
    std::vector<KGraph> kgraph;
    double *kcol_host = nullptr;       // pinned: the iteration's dots / scalars, read by the host
    cudaStream_t cap_stream = nullptr; // private stream the graphs are captured on
    // counters
    int64_t launches = 0, skipped_dss = 0, perturbed = 0;
    int64_t variants[TSP_NVARIANTS] = {};   // kernel-variant choices of the setup (tsp_variant_counts)
    DBuf<unsigned long long> dcount;  // device counters scratch
    DBuf<uint8_t> scratch; size_t scratch_bytes = 0;
    Prof prof;
};

// ------------------------------------------------------------------ launch helpers
inline int grid_for(int64_t threads, int block) { return (int)((threads + block - 1) / block); }
void prof_begin(Ctx &c, int cls);
void dbg_mark(Ctx &c, const char *what, int lvl);   // TSP_DEBUG=1: phase wall times of the setup
void prof_end(Ctx &c, int cls, double bytes);
void *scratch(Ctx &c, size_t bytes);

// sparse.cu
void csr_upload(Ctx &c, Csr &A, int n, int m, int nc, const int32_t *rp, const int32_t *ci, const double *v, bool on_device);
void sell_from_csr(Ctx &c, const Csr &A, Sell &S, int bs, const int *val_map = nullptr);
void check_csr(Ctx &c, const Csr &A, const char *name);
bool all_nonneg(Ctx &c, const double *v, int64_t n);

// operator / Algorithm 1 pieces (apply.cu)
void op_apply(Ctx &c, const double *x, double *y);
void sym_build(Ctx &c);           // sym_uu / sym_sdc from the uploaded A_uu (tsp_create)
bool sym_refill_uu(Ctx &c);       // tsp_update_values: sym_uu from the new c.uu.v (false: generic SELL needed)
void sym_refill_sdc(Ctx &c);      // TSP_SETUP_MECH after an update: sym_sdc from c.uu_sdc
bool sym_op_node(Ctx &c, const GV &gu, const GV &gf, double *yu, Rows R, int cnt);                      // A_uu x_u + A_uf x_f, if sym_uu.ok
bool sym_vcycle_post(Ctx &c, int n, const double *dinv, const double *b, const GV &x, double *xo);
double sym_bytes(const Ctx &c, int bs);   // bytes of one stream over a Sym27 with bs values per block
void prec_apply(Ctx &c, const double *v, double *z);
void op_apply_after_prec(Ctx &c, const double *v, const double *z, double *y);   // A z right after z = M^-1 v

// p7.cu: structured 7-point pressure level 0 (mode 1 pre, 2 post, 3 residual, 4 / 5 Chebyshev PRE / STEP)
void p7_build(Ctx &c, const Csr &A);
double p7_bytes(const Ctx &c);
void p7_launch(Ctx &c, int mode, const GV &dinv, const GV &b, const GV &x, double *o1, double *o2, const ChebArgs &ca);

// setup (setup_flow.cu, amg_setup.cu, ilu.cu)
void extract_sdc(Ctx &c);
void setup_mech(Ctx &c);
void setup_flow(Ctx &c, bool refresh = false);
void amg_build(Ctx &c, Hier &H, Csr &A0, DBuf<int32_t> &zb0, int nc, Halo *fine_halo, int64_t row_off0, int64_t nglob0,
               bool refresh = false);   // refresh: frozen aggregation, values only (R-refresh)
void amg_vcycle(Ctx &c, Hier &H, const double *b, double *x, bool mech);
// gs.cu: Gauss-Seidel smoother (R-gs)
void gs_setup(Ctx &c, Hier &H, int nc);
template <int NC> void gs_sweep(Ctx &c, Level &L, bool backward, const double *b, const double *xin, double *xout);
double gs_sweep_bytes(const Level &L, int nc);
void gs_export_colour(Ctx &c, const Level &L, int32_t *host_out);
bool sym_vcycle_resid(Ctx &c, int n, const double *b, const GV &x, double *r);   // level-0 SDC r = b - A x, if sym_sdc.ok
// level-0 SDC fused Chebyshev step (cheb_epi), if sym_sdc.ok
bool sym_vcycle_cheb(Ctx &c, int n, bool pre, const GV &dinv, const GV &b, const GV &x, const ChebArgs &a, double *xo);
void ilu_setup(Ctx &c, const double *sff_vals);
void ilu_apply_fused(Ctx &c, const double *yf, const double *zs, const double *zp, double *zf_out);

// assemble.cu: GPU assembly of the linearised Jacobian (NEXT-f1)
void assembly_sizes(const tsp_asm_params &P, int rank, int nranks, int zblock, int64_t out[6]);
void assemble(cudaStream_t s, const tsp_asm_params &P, int rank, int nranks, int zblock, const tsp_cell_fields &f,
              tsp_bsr_out blk[4], double *fs, double row_max[3]);
void assemble_scale(cudaStream_t s, const tsp_asm_params &P, int rank, int nranks, int zblock, const double row_max[3],
                    tsp_bsr_out blk[4], double *fs, double scales[3]);

// capi.cu: value update on the stored patterns (tsp_update_values; the Newton step moves its assembled values in)
bool pattern_differs(Ctx &c, const Csr &A, const int32_t *rp, const int32_t *ci);
void commit_values(Ctx &c, DBuf<double> vals[4], DBuf<double> &fs);

// Appendix B.1 residual, state fields and masses at x (single rank; ref: E, perm, phi = phi_0, pres = p_ref, well)
// residual rows of `rank` (its [u_own | f_own]) from the GLOBAL state x; mprev: this rank's cells
void residual(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, double dt, const double *x, const double *mprev,
              double *r, int rank = 0, int nranks = 1, int zblock = 16);
void masses_local(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *xg, double *m_local, int rank,
                  int nranks, int zblock);
void state_fields(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *x, double *phi, double *sat,
                  double *pres);
void masses(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *x, double *m);

// partition of the z-slab decomposition (include/tsp.h)
void partition(int nx, int ny, int nz, int zblock, int rank, int nranks, int64_t out6[6]);
void reduce_setup(Ctx &c);

// ---- bulk-copy (TMA) staging primitives: mbarrier init / expect-tx / arrive / parity wait, 1-D global -> shared
// copies completing on an mbarrier by byte count (k_mdot2_tma).  Sizes and addresses: 16-B multiples.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t phase)
{
    uint32_t done;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(smem_addr(b)), "r"(phase) : "memory");
    } while (!done);
}


// Krylov (krylov.cu)
void krylov_graphs_drop(Ctx &c);
void krylov_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info);
void richardson_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info);

}  // namespace tsp

// the opaque handle of include/tsp.h
struct tsp_ctx : tsp::Ctx {};

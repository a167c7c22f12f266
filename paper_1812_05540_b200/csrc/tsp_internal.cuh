// tsp_internal.cuh -- shared declarations of libtsp.so (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "tsp.h"

namespace tsp {

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
// Stream-ordered allocation (cudaMallocAsync on the stream of the API call in
// progress, pool kept resident): setup allocates per level without device syncs.
extern thread_local cudaStream_t g_alloc_stream;
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; return *this; }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) TSP_CUDA(cudaMallocAsync((void **)&p, sizeof(T) * count, g_alloc_stream));
    }
    void zero(cudaStream_t s) { if (n) TSP_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s)); }
    void release() { if (p) cudaFreeAsync(p, g_alloc_stream); p = nullptr; n = 0; }
    operator T *() const { return p; }
};

// ------------------------------------------------------------------ sparse layouts
// CSR with nc values per entry, entry-major: v[q*nc + c].
struct Csr {
    int n = 0, m = 0, nc = 1;
    int64_t nnz = 0;
    DBuf<int32_t> rp, ci;
    DBuf<double> v;
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

// One AMG level (setup products in CSR, apply operators in SELL).
struct Level {
    int n = 0, nc = 1, coarsest = 0, nagg = 0;
    Csr A;                        // level operator
    DBuf<int32_t> zb;             // z-block per row
    DBuf<double> dl1;             // l1 row norms [n][nc]
    DBuf<double> dinv;            // 1 / dl1
    DBuf<int32_t> agg;            // aggregate per row (-1 = none)
    Csr P, R;
    Sell sA, sP, sR;
    DBuf<double> cinv;            // coarsest: dense inverse [nc][n][n]
    // apply work vectors [n][nc]
    DBuf<double> b, x, x2, r;
};

struct Hier {
    int nc = 1;
    std::vector<Level> L;
    int64_t fallbacks = 0, perturbed = 0;
};

// ------------------------------------------------------------------ profiling
enum ProfClass {
    PK_OP_NODE, PK_OP_CELL, PK_STEP2, PK_STEP34, PK_ILU, PK_VC_PRE_U, PK_VC_RESTR_U, PK_VC_PROL_U, PK_VC_POST_U,
    PK_VC_PRE_P, PK_VC_RESTR_P, PK_VC_PROL_P, PK_VC_POST_P, PK_COARSE, PK_DOT, PK_AXPY, PK_NORM, PK_VEC, PK_SETUP,
    PK_COUNT
};

struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    struct Rec { int cls; int e0, e1; double bytes; };
    std::vector<Rec> recs;
    int next = 0;
    bool open = false;
};

// ------------------------------------------------------------------ the handle
struct Ctx {
    int nx, ny, nz, Nn, Nc;
    int64_t n;
    cudaStream_t s;
    tsp_options o;
    int sm_count = 148;
    // original blocks (CSR on device) for setup + SELL for apply
    Csr uu, uf, fu, ff;           // nc = values per block entry (9, 6, 6, 4)
    Sell s_uu, s_uf, s_fu, s_ff;  // SELL copies (operator rows)
    DBuf<double> fs;              // 2 per cell
    // flow setup products
    DBuf<double> dss_inv;         // 1/D_ss (0 if D_ss == 0)
    Sell s_aps;                   // A_ps values on A_ff's pattern (bs 1)
    DBuf<double> ilu_val;         // tile-level-major S_ff^FS blocks, 7 slots x 4 (R-ilu)
    DBuf<double> ilu_dinv;        // tile-level-major U_KK^-1, 4 per cell
    DBuf<int32_t> ilu_lvlptr;     // level pointers of the full-tile table
    DBuf<int32_t> ilu_cells;      // local (i,j,k) packed per table position
    DBuf<int32_t> ilu_posmap;     // local linear index -> table position
    int ilu_nlev = 0, ilu_tsize = 0, ntiles = 0, ntx = 0, nty = 0, ntz = 0;
    Hier mech, pres;
    bool mech_ready = false, flow_ready = false;
    // work vectors
    DBuf<double> w_yf, w_wp, w_zp, w_zf2, w_tmp;
    // Krylov storage
    DBuf<double> V, Z, kw, kr, kx, kb, kh, kpart;
    int kcap = 0;
    // counters
    int64_t launches = 0, skipped_dss = 0, perturbed = 0;
    DBuf<unsigned long long> dcount;  // device counters scratch
    DBuf<uint8_t> scratch; size_t scratch_bytes = 0;
    Prof prof;
};

// ------------------------------------------------------------------ launch helpers
inline int grid_for(int64_t threads, int block) { return (int)((threads + block - 1) / block); }
void prof_begin(Ctx &c, int cls);
void prof_end(Ctx &c, int cls, double bytes);
void *scratch(Ctx &c, size_t bytes);

// sparse.cu
void csr_upload(Ctx &c, Csr &A, int n, int m, int nc, const int32_t *rp, const int32_t *ci, const double *v, bool on_device);
void sell_from_csr(Ctx &c, const Csr &A, Sell &S, int bs, const int *val_map = nullptr);
void check_csr(Ctx &c, const Csr &A, const char *name);

// operator / Algorithm 1 pieces (apply.cu)
void op_apply(Ctx &c, const double *x, double *y);
void prec_apply(Ctx &c, const double *v, double *z);

// setup (setup_flow.cu, amg_setup.cu, ilu.cu)
void setup_mech(Ctx &c);
void setup_flow(Ctx &c);
void amg_build(Ctx &c, Hier &H, Csr &A0, DBuf<int32_t> &zb0, int nc);
void amg_vcycle(Ctx &c, Hier &H, const double *b, double *x, bool mech);
void ilu_setup(Ctx &c, const double *sff_vals);
void ilu_apply_fused(Ctx &c, const double *yf, const double *zs, const double *zp, double *zf_out);

// Krylov (krylov.cu)
void krylov_solve(Ctx &c, const double *b, double *x, const tsp_solve_opts &o, tsp_solve_info &info);

}  // namespace tsp

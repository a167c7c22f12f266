/*
 * tsp.h -- C-ABI of the B200-native two-stage preconditioner library (libtsp.so).
 *
 * "tsp" = two-stage preconditioner of White, Castelletto, Klevtsov, Bui,
 * Osei-Kuffuor, Tchelepi, "A Two-Stage Preconditioner for Multiphase
 * Poromechanics in Reservoir Simulation", arXiv 1812.05540.  P:n below is
 * /root/reference/PAPER.md line n (the LaTeX source); R-xx is a reading listed
 * in DESIGN.md.
 *
 * The library applies M^-1 of eq:blk_tr_prec by Algorithm 1
 * (alg:apply_M_inv) inside right-preconditioned flexible GMRES
 * on the fully coupled Jacobian of eq:jac_system:
 *   M_uu^-1 = amg(A_uu^SDC)
 *   M_ff^-1 = M_G^-1 + M_L^-1 (I - S_ff^FS M_G^-1) (eq:mult_prec_op)
 *   S_ff^FS = A_ff + diag(D_sp, D_pp)             (eq:Schur_1_FS)
 *   M_G^-1 with quasi-IMPES S_pp and amg(S_pp)
 *   M_L^-1 = tile-local block ILU(0)              (R-ilu)
 * Every step runs in sm_100a CUDA kernels; there is no CPU fallback.
 *
 * Conventions (all functions):
 *  - Vectors are fp64 in the layout [ u : 3*N_n, node-major (x,y,z) | f : 2*N_c,
 *    cell-major interleaved (s, p) ], i.e. the permutation P of P:606 applied.
 *    Node (i,j,k) = i + (nx+1)(j + (ny+1)k); cell (i,j,k) = i + nx(j + ny k).
 *  - Matrices are BSR with int32 row pointers / block column indices (sorted,
 *    unique per row, structurally symmetric patterns for A_uu and A_ff) and fp64
 *    row-major blocks.  The caller passes the block-row-scaled Jacobian
 *    with Dirichlet DoF as identity rows (R-dirichlet).
 *  - Device pointers are CUDA global-memory pointers valid on the handle's
 *    device; "host" pointers are ordinary (preferably pinned) host memory.
 *  - The library never keeps a caller pointer beyond the call (tsp_create deep
 *    copies).  All device work is ordered on the handle's stream.
 *  - Errors: every call returns tsp_status; on failure tsp_last_error() gives a
 *    thread-local message.  A handle is not thread safe.
 */
#ifndef TSP_H
#define TSP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSP_ABI_VERSION 5

typedef int tsp_status;
enum {
    TSP_OK = 0,
    TSP_NOT_CONVERGED = 1,       /* solve: x holds the last iterate, info filled */
    TSP_ERR_INVALID_ARG = -1,    /* null pointer, bad sizes, unsorted/duplicate columns, negative fs */
    TSP_ERR_DIM_MISMATCH = -2,
    TSP_ERR_STATE = -3,          /* apply/solve before setup */
    TSP_ERR_CUDA = -4,
    TSP_ERR_NCCL = -5,
    TSP_ERR_OOM = -6,
    TSP_ERR_SINGULAR = -7,       /* coarsest AMG level exceeds the dense limit */
    TSP_ERR_NUMERIC = -8         /* NaN/Inf in an Arnoldi norm */
};

typedef struct tsp_ctx *tsp_handle;

typedef struct {
    double amg_theta;            /* strength threshold, 0.25 (R-strength) */
    int amg_coarse_max;          /* dense solve at <= this many rows, 64 */
    int amg_max_levels;          /* 12 */
    int zblock;                  /* cell planes per z-block for aggregation confinement, 16 (R-zblock) */
    int tile_x, tile_y, tile_z;  /* ILU(0) tile, 16^3 (R-ilu) */
    int replicate_rows;          /* multi-GPU: coarse levels with <= this many global rows are gathered on
                                    every rank (default 32768); no effect on the result */
    /* setup variants of the paper; the defaults are the paper's choices */
    int cpr_mode;                /* 0 quasi-IMPES: D_ss = diagm(A_ss), D_ps = diagm(A_ps);
                                    1 true-IMPES: column-sum lumping D = diag(A^T e) (eq:CPR_CSL) */
    int aps_mode;                /* 0 full A_ps in step 4; 1 its diagonal approximation D_ps^(CPR) */
    int fs_mode;                 /* 0 D_fs = tsp_desc.fs_diag / fs_modulus_scale (eq:FS_Dps_Dpp, remark P:443);
                                    1 algebraic row-sum lumping (eq:FS_RSL): needs TSP_SETUP_MECH first */
    int rsl_iters;               /* fs_mode 1: A_uu^-1 ~ this many M_uu-preconditioned Richardson steps, 2 */
    double fs_modulus_scale;     /* fs_mode 0: K_dr -> scale * K_dr, i.e. D_fs / scale (default 1) */
    /* second stage M_L */
    int second_stage;            /* 0 tile ILU(0) (the paper's option 2, SPE10); 1 hybrid block Gauss-Seidel with the
                                    16^3 tile as the "processor" (option 1, the staircase) */
    int local_sweeps;            /* Algorithm 1 steps 6-8 repeated this many times (default 1; the staircase used 3) */
    /* AMG smoother of both hierarchies */
    int amg_smoother;            /* 0 l1-Jacobi (north_star; R-cycle); 2 Chebyshev (below); 1 Gauss-Seidel, forward on the way down and backward
                                    on the way up (reading R-gs): multicolour GS on level 0 (parity colourings), hybrid
                                    l1-GS on the coarse levels with blocks of amg_gs_block rows as the "processors";
                                    single GPU only */
    int amg_gs_block;            /* rows per hybrid block (default 1024, range [32, 1024]) */
    /* amg_smoother = 2: Chebyshev polynomial smoother on D_l1^-1 A (north_star "Jacobi/Chebyshev"; SURVEY NEXT-f3;
       DESIGN.md R-cheb): amg_cheb_degree steps of the Chebyshev iteration per pre-/post-smoothing on the interval
       [amg_cheb_lower, 1] (1 = the l1 bound of the spectrum); multi-GPU capable */
    int amg_cheb_degree;         /* default 2, range [1, 8] */
    double amg_cheb_lower;       /* default 0.3, range (0, 1) */
    int amg_smoother_p;          /* smoother of the pressure hierarchy only: -1 (default) = amg_smoother, else 0/1/2 */
} tsp_options;

/* BSR block matrix given to tsp_create (nrows block rows). */
typedef struct {
    const int32_t *rowptr;       /* nrows+1 */
    const int32_t *col;          /* rowptr[nrows] block columns */
    const double *val;           /* rowptr[nrows] * bm * bn, row-major blocks */
} tsp_bsr;

/* Multi-GPU (row e): z-slab decomposition.  The grid's cell planes are grouped
 * into z-blocks of opts.zblock planes (nzb = ceil(nz/zblock)); rank r owns the
 * z-blocks [floor(r nzb / P), floor((r+1) nzb / P)), i.e. cell planes [k0, k1),
 * node planes [k0, k1) plus plane nz on the last rank.  Each rank passes ONLY its
 * owned block rows (in global natural order) with GLOBAL column indices; vectors
 * are the rank's owned part [u_own | f_own].  Results are bitwise identical for
 * every P (aggregation and ILU tiles never cross z-blocks, reductions are summed
 * per fixed chunk in global order).  Requires 1 <= P <= nzb. */
enum { TSP_COMM_NONE = 0, TSP_COMM_NCCL = 1, TSP_COMM_LOCAL = 2 };

/* Device-memory callbacks (BASELINE.json north_star: "PyTorch only for device memory").
 * When `alloc` is non-NULL EVERY device buffer of the handle (matrices, hierarchies, Krylov basis, work
 * vectors, CUB scratch) is obtained from alloc(bytes, stream, ctx) and returned through
 * free(ptr, bytes, stream, ctx), both on the handle's stream (stream-ordered: a block freed on the stream
 * may be reused by later work on the same stream).  alloc returns a device pointer on the handle's device,
 * aligned to 256 bytes, or NULL when out of memory (the call then fails with TSP_ERR_OOM).  The callbacks
 * are called only from inside this library's API calls on the calling host thread (tsp_destroy included),
 * and must stay valid until tsp_destroy returns.  alloc = NULL: the library's own stream-ordered pool. */
typedef struct {
    void *(*alloc)(size_t bytes, void *stream, void *ctx);
    void (*free)(void *ptr, size_t bytes, void *stream, void *ctx);
    void *ctx;
} tsp_allocator;

typedef struct {
    int nx, ny, nz;              /* GLOBAL grid in cells: N_n = (nx+1)(ny+1)(nz+1), N_c = nx ny nz */
    int rank, nranks;            /* this rank and the number of ranks (one per GPU) */
    int comm_kind;               /* TSP_COMM_NCCL: comm_arg = 128-byte ncclUniqueId (tsp_nccl_unique_id on rank 0,
                                    broadcast by the caller); TSP_COMM_LOCAL: comm_arg = tsp_local_world_create()
                                    (test backend: P handles in one process, one host thread each) */
    const void *comm_arg;
    void *stream;                /* cudaStream_t to order all work on (0 = legacy default) */
    int inputs_on_device;        /* 0: all pointers below are host; 1: device */
    tsp_bsr A_uu;                /* 3x3, N_n block rows, N_n block cols */
    tsp_bsr A_uf;                /* 3x2 [A_us | A_up], N_n x N_c */
    tsp_bsr A_fu;                /* 2x3 [A_su ; A_pu], N_c x N_n */
    tsp_bsr A_ff;                /* 2x2 [[A_ss, A_sp],[A_ps, A_pp]], N_c x N_c */
    const double *fs_diag;       /* 2*N_c: (D_sp, D_pp) per cell, eq:FS_Dps_Dpp P:435-436, row-scaled */
    tsp_options opts;
    tsp_allocator allocator;     /* device memory callbacks; zero-initialised = the library's pool */
} tsp_desc;

/* TSP_SETUP_REFRESH (with TSP_SETUP_FLOW, DESIGN.md R-refresh): the flow phase after
 * tsp_update_values -- every a1/a3/a5 product is recomputed from the new values, and the pressure AMG keeps the
 * strength flags, MIS(2) aggregates and every pattern of its last full build (frozen aggregation) while all of
 * its values are recomputed in the build's own order and arithmetic (bit-identical to a full build whenever
 * that build would choose the same aggregates).  TSP_ERR_STATE without a previous completed TSP_SETUP_FLOW. */
enum { TSP_SETUP_MECH = 1, TSP_SETUP_FLOW = 2, TSP_SETUP_REFRESH = 4 };

typedef struct {
    double rtol;                 /* ||b - A x|| <= rtol ||b||, default 1e-8 */
    int restart;                 /* FGMRES(m), default 64; clamped to [1, 120] */
    int max_iters;               /* preconditioner applications, default 1000; 0 = only the true residual of x0 */
    int x0_zero;                 /* 1: ignore x on input, start from 0 */
    int host_ptrs;               /* 1: b and x are host pointers (copies are on the stream) */
} tsp_solve_opts;

typedef struct {
    int iterations;              /* preconditioner applications inside Arnoldi */
    int restarts;
    int status;                  /* TSP_OK, TSP_NOT_CONVERGED or an error */
    double est_relres;           /* Arnoldi estimate |g_{j+1}| / ||b|| */
    double true_relres;          /* recomputed ||b - A x|| / ||b|| at exit */
    double t_solve_s;
    int reorth;                  /* basis vectors re-orthogonalised (DCGS2: every one, one step late) */
    double bytes_krylov;         /* algorithmic bytes of the Gram-Schmidt / normalisation / x-update kernels */
    int dcgs_fallbacks;          /* iterations whose Pythagorean DCGS2 norm lost > 6 digits to cancellation and took
                                    the explicit two-pass Gram-Schmidt instead (env TSP_DCGS2_FALLBACK: all of them) */
} tsp_solve_info;

typedef struct {
    int levels[2];               /* [0] mechanics SDC hierarchy, [1] pressure hierarchy */
    int64_t rows[2][16], nnz[2][16];
    int64_t launches;            /* kernels launched by this handle since the last reset */
    int64_t skipped_dss, perturbed_pivots, coarsening_fallbacks;
    double bytes_apply;          /* algorithmic bytes of one tsp_apply_preconditioner */
    double bytes_operator;       /* algorithmic bytes of one tsp_apply_operator */
    double bytes_iter_base;      /* per FGMRES iteration excluding Gram-Schmidt: apply + the operator as FGMRES applies it
                                    (its cell rows reuse Algorithm 1's A_fu z_u, so A_fu is not streamed twice) */
    double bytes_per_krylov_vec; /* bytes of one basis-vector pass (8 n); exact Krylov bytes: tsp_solve_info */
    int64_t allocs_callback;     /* device allocations made through tsp_desc.allocator since tsp_create */
    int64_t allocs_pool;         /* device allocations made from the library's own pool since tsp_create */
    int64_t bytes_live;          /* device bytes the handle holds right now */
} tsp_stats;

/* per-kernel-class timing (CUDA events on the handle's stream), for roofline */
#define TSP_PROF_MAX 32
typedef struct {
    int nclasses;
    char name[TSP_PROF_MAX][24];
    int64_t launches[TSP_PROF_MAX];
    double ms[TSP_PROF_MAX];       /* summed device time */
    double bytes[TSP_PROF_MAX];    /* summed algorithmic bytes */
} tsp_prof;

int tsp_abi_version(void);
const char *tsp_last_error(void);
tsp_status tsp_default_options(tsp_options *o);

/* NCCL bootstrap: rank 0 creates the id, the caller broadcasts it (e.g. through
 * torch.distributed) and every rank passes it in tsp_desc.comm_arg. */
tsp_status tsp_nccl_unique_id(char out[128]);
/* Test backend: a world of `nranks` handles inside one process (each rank's calls
 * must come from its own host thread; every collective call is matched). */
void *tsp_local_world_create(int nranks);
void tsp_local_world_destroy(void *world);
/* Owned ranges of `rank` (for callers slicing a global problem): out6 =
 * {k0, k1, first owned node, owned nodes, first owned cell, owned cells}. */
tsp_status tsp_partition(int nx, int ny, int nz, int zblock, int rank, int nranks, int64_t out6[6]);

/* Validates, deep-copies the blocks into library-owned device memory and
 * repacks them (sliced-ELL, R-layout).  The caller may free its inputs after
 * return.  Returns TSP_ERR_INVALID_ARG on null/unsorted/inconsistent input. */
tsp_status tsp_create(tsp_handle *out, const tsp_desc *d);

/* TSP_SETUP_MECH: rows a2 + a4 (SDC extraction, mechanics AMG), once per
 * simulation.  TSP_SETUP_FLOW: rows a1 + a3 + a4 (pressure) + a5
 * (fixed stress, quasi-IMPES, pressure AMG, tile ILU(0)), per Newton step
 * (P:519).  Synchronises the stream. */
tsp_status tsp_setup(tsp_handle h, unsigned what);

/* A Newton step's new Jacobian values on the SAME patterns (the flow setup is
 * redone every Newton step, the mechanics setup once per simulation).  Reads from `d` only nx, ny, nz, rank,
 * nranks (must equal the handle's), inputs_on_device, the four blocks and fs_diag; everything else is ignored.
 * Every rowptr / col array must equal the one given to tsp_create (else TSP_ERR_INVALID_ARG and the handle is
 * unchanged); a negative fs_diag entry is TSP_ERR_INVALID_ARG.  Afterwards tsp_apply_operator uses the
 * new values at once, and tsp_apply_preconditioner / tsp_solve return TSP_ERR_STATE until the flow phase has been
 * redone on them (tsp_setup(TSP_SETUP_FLOW | TSP_SETUP_REFRESH) for a Newton step).  The mechanics AMG stays as
 * built (once per simulation); TSP_SETUP_MECH rebuilds it from the new A_uu^SDC.  Collective over the
 * ranks; synchronises the stream. */
tsp_status tsp_update_values(tsp_handle h, const tsp_desc *d);

/* z = M^-1 v (Algorithm 1).  Device pointers, length n = 3 N_n + 2 N_c, must
 * not alias.  Asynchronous on the handle's stream. */
tsp_status tsp_apply_preconditioner(tsp_handle h, const double *v, double *z);

/* y = A x with the original Jacobian (row a12).  Device pointers, asynchronous. */
tsp_status tsp_apply_operator(tsp_handle h, const double *x, double *y);

/* Right-preconditioned FGMRES(m) with classical Gram-Schmidt applied twice, the second pass
 * delayed one iteration (DCGS2, DESIGN.md R-krylov).  b, x: device pointers of length n (host pointers if
 * o->host_ptrs; copies on the stream); x is x0 on input (zero if o->x0_zero) and the solution on output.
 * Converged when the TRUE residual ||b - A x|| <= rtol ||b|| (recomputed at the end of every cycle; b = 0
 * gives x = 0).  Returns TSP_OK, TSP_NOT_CONVERGED (x = last iterate, info->true_relres its residual) or an
 * error (TSP_ERR_NUMERIC on a non-finite Arnoldi coefficient).  Collective over the ranks; synchronises. */
tsp_status tsp_solve(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info);
void tsp_default_solve_opts(tsp_solve_opts *o);

/* The "sequential" embedding of Algorithm 1 (remark P:640-642; SURVEY NEXT-f4 iii): stationary Richardson iteration
 * x <- x + M^-1 (b - A x) from x0, stopped when the TRUE residual ||b - A x|| <= rtol ||b|| (TSP_OK), after
 * o->max_iters preconditioner applications (TSP_NOT_CONVERGED) or on a non-finite residual norm (TSP_ERR_NUMERIC;
 * the iteration is a contraction only when M^-1 A has its spectrum inside (0, 2), which one SDC V-cycle as the
 * mechanics stage does not guarantee -- DESIGN.md section 7).  Same arguments, pointer kinds and info fields as
 * tsp_solve (o->restart is not read; restarts = reorth = 0; est_relres = true_relres); iterations counts the
 * preconditioner applications.  Collective over the ranks; synchronises. */
tsp_status tsp_richardson(tsp_handle h, const double *b, double *x, const tsp_solve_opts *o, tsp_solve_info *info);

tsp_status tsp_get_stats(tsp_handle h, tsp_stats *s);

/* ---- GPU assembly of the linearised Jacobian (Appendix B) --------------------------
 * The four blocks of eq:jac_system and the fixed-stress diagonals (eq:FS_Dps_Dpp) of the
 * synthetic poromechanics problem, assembled on the device from per-cell fields at a linearisation state, in the
 * layout and units tsp_create consumes (pressure unit p_unit on the p columns, R-punit; block rows scaled by
 * 1 / max row l1 norm, R-scale; bottom nodes Dirichlet identity rows / zero columns, R-dirichlet).
 * Physics: Q1 elasticity with 2x2x2 Gauss and the gravity term, Biot coupling, two-phase TPFA with single-point
 * upwinding and phase-averaged densities, Peaceman wells, Corey n = 2. */
typedef struct {
    int nx, ny, nz;              /* GLOBAL grid (cells); cubic cells of side h = length / nx (R-geom) */
    double length;
    double nu, biot, gravity, dt;
    double rho_w0, rho_nw0, c_w, c_nw, mu_w, mu_nw, rho_s, p0;   /* fluids, solid density, reference pressure (Pa) */
    double swr, snwr;            /* residual saturations of the Corey curves */
    double well_dbhp, rw_over_h; /* BHP offset of injectors (+) and producers (-) from hydrostatic; r_w / h (R-wells) */
    double p_unit;               /* Pa per unit of the pressure unknown (R-punit) */
    int burden;                  /* seal layers at top and bottom: perforations stop above them (R-s10) */
    int dirichlet_bottom, row_scale;
} tsp_asm_params;

/* per-cell fields of the GLOBAL grid (device pointers, N_c entries each, cell (i,j,k) = i + nx (j + ny k)):
 * Young's modulus (Pa), permeability (m^2), porosity, water saturation, pressure (Pa) at the linearisation state,
 * the well perforation of the cell (0 none, 1 water injector, 2 producer; NULL = no wells), and the reference
 * porosity phi_0 of eq:linearized_porosity whose compressibility term (b - phi_0)(1 - b)/K_dr enters the
 * p-derivatives (NULL = phi: the state is the reference state) */
typedef struct {
    const double *E, *perm, *phi, *sat, *pres;
    const int8_t *well;
    const double *phi0;
} tsp_cell_fields;

/* a device BSR block the assembly writes (rowptr: rows + 1, col / val: sizes from tsp_assembly_sizes) */
typedef struct {
    int32_t *rowptr, *col;
    double *val;
} tsp_bsr_out;

/* this rank's rows (the z-slab of include/tsp.h with opts.zblock = `zblock`) and block counts:
 * out6 = {N_n local, N_c local, blocks of A_uu, A_uf, A_fu, A_ff}.  Host only. */
tsp_status tsp_assembly_sizes(const tsp_asm_params *p, int rank, int nranks, int zblock, int64_t out6[6]);
/* blocks = {A_uu, A_uf, A_fu, A_ff}: this rank's rows with GLOBAL column ids, fs: 2 per local cell.  Writes the
 * unscaled values (p_unit applied) and returns in row_max (host) this rank's maxima of the row l1 norms of
 * (A_uu rows, A_ss entries, A_pp entries); the caller takes the maximum over the ranks and passes it to
 * tsp_assemble_scale, which applies the block-row scaling and the Dirichlet rows (scales out: 1/max, host).
 * Ordered on `stream` (cudaStream_t; 0 = legacy default); both calls synchronise it.  Errors: TSP_ERR_INVALID_ARG
 * on null pointers or a bad grid, TSP_ERR_CUDA. */
tsp_status tsp_assemble(const tsp_asm_params *p, int rank, int nranks, int zblock, const tsp_cell_fields *f,
                        tsp_bsr_out blocks[4], double *fs, double row_max[3], void *stream);
tsp_status tsp_assemble_scale(const tsp_asm_params *p, int rank, int nranks, int zblock, const double row_max[3],
                              tsp_bsr_out blocks[4], double *fs, double scales[3], void *stream);

/* ---- the nonlinear step: residual of Appendix B.1 and Newton ----------------------
 * State x (device, n = 3 N_n + 2 N_c): [u node-major (m) | (s, p [Pa]) per cell] -- raw pressure, unlike the
 * linear system's unknown p / p_unit.  `ref` fields: E, perm, well as for tsp_assemble, phi = the REFERENCE
 * porosity phi_0 and pres = the reference pressure p_ref of eq:linearized_porosity (phi = phi_0 + b eps_v +
 * (b - phi_0)(1 - b)/K_dr (p - p_ref), eps_v averaged over the cell); sat is not read.  tsp_residual and
 * tsp_masses take GLOBAL vectors (one GPU); tsp_newton_residual / tsp_newton_step work on z-slab ranks. */
/* r = r(x) in raw units (N for momentum rows, kg for mass rows); mprev: (V m_w, V m_nw) per cell of the previous
 * step (tsp_masses); Dirichlet rows 0.  Synchronises `stream`. */
tsp_status tsp_residual(const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, const double *x, const double *mprev,
                        double *r, void *stream);
tsp_status tsp_masses(const tsp_asm_params *p, const tsp_cell_fields *ref, const double *x, double *m, void *stream);

typedef struct {
    double rtol;                 /* converged when ||S0 r|| <= rtol ||S0 r_0|| (S0: the step's first row scales), 1e-6 */
    double atol;                 /* or ||S0 r|| <= atol, default 0 */
    int max_newton;              /* 12 */
    double lin_rtol;             /* FGMRES tolerance of every Newton system, 1e-8 */
    int max_lin_iters;           /* 1000 */
    int refresh;                 /* 1: per-Newton flow setup with frozen pressure aggregation (TSP_SETUP_REFRESH) */
    int max_halvings;            /* backtracking line search: alpha halved at most this often, 5 */
} tsp_newton_opts;
typedef struct {
    int newton_iters, lin_iters, halvings, status;   /* status 0 converged, 1 not */
    double res0, res;            /* ||S0 r|| at the start and at exit */
    double res_hist[16];         /* per Newton iteration */
    int lin_hist[16];            /* FGMRES iterations per Newton iteration */
} tsp_newton_info;
void tsp_default_newton_opts(tsp_newton_opts *o);
/* this rank's residual rows r (its [u_own | f_own], raw units) at the rank-local state x (gathered over the ranks
 * of h); mprev (this rank's cells, or NULL: the masses at x).  Collective; synchronises. */
tsp_status tsp_newton_residual(tsp_handle h, const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, const double *x,
                               const double *mprev, double *r);
/* One implicit time step (dt) by Newton's method with backtracking line search on the handle `h` (created from a
 * Jacobian of the same grid, tsp_setup(MECH) done): per iteration the Jacobian is re-assembled at x on the device
 * (tsp_assemble), moved into h, the flow phase redone (TSP_SETUP_FLOW[|REFRESH]; the mechanics AMG stays)
 * and J dx = -S r solved by the two-stage preconditioned FGMRES; x += alpha dx with alpha halved until ||S0 r||
 * decreases (saturation kept in [0, 1]).  r_off (device, 3 N_n, may be NULL): a momentum residual
 * subtracted from every evaluation (the initial-state equilibrium, so that u measures the displacement since t0).
 * On z-slab ranks (handle with a communicator) x, mprev, r_off are the rank's parts ([u_own | f_own], its cells, its
 * 3 N_n momentum rows); the state is gathered over the ranks for the residual and the state fields, the norms are
 * taken over the gathered residual, so every rank takes the same decisions and the step is bitwise the one-rank
 * step.  mprev NULL: the masses at x (the start of the step).  x is updated in place.  Returns TSP_OK,
 * TSP_NOT_CONVERGED (info filled) or an error. */
tsp_status tsp_newton_step(tsp_handle h, const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, double *x,
                           const double *mprev, const double *r_off, const tsp_newton_opts *o, tsp_newton_info *info);

/* Test hook (row c.5 parity): copy level `lvl` of hierarchy `which` (0 mech, 1
 * pressure) to host buffers.  Sizes: out6 = {n, nnz(A), nagg, nnz(P), nc,
 * coarsest}.  Any buffer may be NULL; A_v/P_v/dl1 are [entry][nc]. */
tsp_status tsp_level_sizes(tsp_handle h, int which, int lvl, int64_t out6[6]);
tsp_status tsp_export_level(tsp_handle h, int which, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v,
                            int32_t *agg, int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1);

/* Test hook (amg_smoother = 1): the Gauss-Seidel colouring of level `lvl` -- colour per row (int32, n) --
 * and the level's gs_block (0: multicolour over the level; B: hybrid blocks of B rows) in *block.  Returns
 * TSP_ERR_STATE when the smoother is not GS or the level is the coarsest. */
tsp_status tsp_export_colour(tsp_handle h, int which, int lvl, int32_t *colour, int *block, int *ncolour);

/* multi-GPU layout of a level: out3 = {distributed (rows split over ranks), global rows,
 * first global row of this rank}.  Replicated levels are complete on every rank. */
tsp_status tsp_level_dist(tsp_handle h, int which, int lvl, int64_t out3[3]);

tsp_status tsp_prof_enable(tsp_handle h, int on);   /* also resets */
tsp_status tsp_prof_read(tsp_handle h, tsp_prof *p);  /* synchronises */
/* restrict recording to the classes in `mask` (bit k = class k of tsp_prof.name; default all):
 * two timing events per recorded launch cost ~2 % of an FGMRES iteration, so a timed run records
 * only the class whose roofline it reports */
tsp_status tsp_prof_classes(tsp_handle h, unsigned mask);
/* Test hook (after TSP_SETUP_FLOW): this rank's D_ss^(CPR), D_ps^(CPR) (N_c,local each) and the fixed-stress
 * diagonal actually used by a1, (D_sp, D_pp) per cell (2 N_c,local); host buffers, any may be NULL. */
tsp_status tsp_export_cpr(tsp_handle h, double *dss, double *dps, double *fs_eff);

/* Test hook (parity coverage): how often each kernel variant was chosen by the setups of this handle.
 * out[TSP_NVARIANTS], indexed by TSP_VAR_*: the Galerkin product's per-row hash table (64 / 128 / 512 / 4096
 * slots; 512 and 4096 are the overflow retries) and lanes per row (4 / 8 / 32), both counted per launch; the
 * vector-CSR lanes per row of each coarse level's smoother A (0 = sliced-ELL / 8 / 16 / 32) and of each
 * level's restriction R, counted per level.  Test knobs (environment, read by every setup):
 * TSP_SPGEMM_MIN_SLOTS=512|4096 starts the products at the overflow tables (bitwise the same hierarchy);
 * TSP_FORCE_LANES=0|8|16|32 forces one vector-CSR variant on every level. */
enum {
    TSP_VAR_SPGEMM_HS64 = 0, TSP_VAR_SPGEMM_HS128, TSP_VAR_SPGEMM_HS512, TSP_VAR_SPGEMM_HS4096,
    TSP_VAR_SPGEMM_G4, TSP_VAR_SPGEMM_G8, TSP_VAR_SPGEMM_G32,
    TSP_VAR_LANES_A0, TSP_VAR_LANES_A8, TSP_VAR_LANES_A16, TSP_VAR_LANES_A32,
    TSP_VAR_LANES_R0, TSP_VAR_LANES_R8, TSP_VAR_LANES_R16, TSP_VAR_LANES_R32,
    TSP_NVARIANTS
};
tsp_status tsp_variant_counts(tsp_handle h, int64_t out[TSP_NVARIANTS]);

void tsp_destroy(tsp_handle h);

#ifdef __cplusplus
}
#endif
#endif

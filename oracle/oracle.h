/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential CPU C implementation of the two-stage preconditioner
 * path (fixed-stress Schur complement + CPR inside flexible GMRES) of
 * White et al., arXiv 1812.05540.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code with the CUDA library (paper_1812_05540_b200/), and the product never
 * calls it.  Every function cites the PAPER.md line (P:n) or the DESIGN.md
 * reading (R-xx, mirroring SURVEY.md D1-D25) it follows.
 */
#ifndef TSP_ORACLE_H
#define TSP_ORACLE_H
#include <stdint.h>

typedef struct {
    int nx, ny, nz;               /* grid (cells) */
    const int32_t *uu_rowptr, *uu_col; const double *uu_val;   /* A_uu BSR 3x3 */
    const int32_t *uf_rowptr, *uf_col; const double *uf_val;   /* A_uf BSR 3x2 */
    const int32_t *fu_rowptr, *fu_col; const double *fu_val;   /* A_fu BSR 2x3 */
    const int32_t *ff_rowptr, *ff_col; const double *ff_val;   /* A_ff BSR 2x2 (s,p) interleaved */
    const double *fs;             /* (D_sp, D_pp) per cell */
} orc_desc;

typedef struct {
    double amg_theta;             /* 0.25 (R-strength) */
    int amg_coarse_max;           /* 64 */
    int amg_max_levels;           /* 12 */
    int zblock;                   /* 16 cell planes (R-zblock) */
    int tile_x, tile_y, tile_z;   /* 16,16,16 (R-ilu-tile) */
    int mech_mode;                /* 0: amg(A_uu^SDC) P:515; 1: exact dense A_uu^-1 (pins) */
    int pres_mode;                /* 0: amg(S_pp) P:599;    1: exact dense S_pp^-1 (pins) */
    int local_mode;               /* 0: tile ILU(0) P:612;  1: exact (S_ff^FS)^-1; 2: none */
    int ff_mode;                  /* 0: CPR two-stage (Alg.1 steps 3-8); 1: exact dense S_ff^-1 (eq:LU) */
    /* NEXT-f3 variants (setup only; defaults reproduce the paper's choices) */
    int cpr_mode;                 /* 0: quasi-IMPES diagm; 1: true-IMPES column sums (eq:CPR_CSL) */
    int aps_mode;                 /* 0: full A_ps in step 4; 1: its diagonal approximation D_ps^(CPR) */
    int fs_mode;                  /* 0: D_fs given (eq:FS_Dps_Dpp); 1: row-sum lumping RSL (eq:FS_RSL) */
    int rsl_iters;                /* RSL: A_uu^-1 ~ this many M_uu-preconditioned Richardson steps, default 2 */
    double fs_modulus_scale;      /* fs_mode 0: modulus K_dr -> scale K_dr, i.e. D_fs / scale (remark P:443), default 1 */
    /* NEXT-f2: the second stage M_L */
    int second_stage;             /* 0: tile ILU(0) (option 2); 1: hybrid block Gauss-Seidel, tile = processor (option 1) */
    int local_sweeps;             /* steps 6-8 repeated this many times ("several sweeps"; 3 for the staircase) */
    /* AMG smoother of both hierarchies (NEXT-f2/f3) */
    int amg_smoother;             /* 0: l1-Jacobi (R-cycle, north_star); 1: Gauss-Seidel forward on the way down, backward on
                                     the way up (R-gs): multicolour on level 0, hybrid l1-GS on the coarse levels */
    int amg_gs_block;             /* R-gs hybrid levels: rows per "processor" block (1024) */
    /* amg_smoother 2: Chebyshev polynomial smoother (north_star "Jacobi/Chebyshev"; reading R-cheb) */
    int amg_cheb_degree;          /* polynomial degree per smoothing step (2) */
    double amg_cheb_lower;        /* interval [lower, 1] of D_l1^-1 A (the l1 bound makes 1 the upper end), 0.3 */
    int amg_smoother_p;           /* smoother of the pressure hierarchy only (-1: amg_smoother) */
} orc_opts;

typedef struct {
    int iterations, restarts, status;   /* status 0 converged, 1 max iters, 2 breakdown */
    double est_relres, true_relres;
    double t_setup, t_solve;
} orc_info;

typedef struct orc orc;

void orc_default_opts(orc_opts *o);
orc *orc_create(const orc_desc *d, const orc_opts *o);
void orc_destroy(orc *h);
int orc_setup(orc *h);                                    /* rows a1-a5 */
int orc_setup_flow(orc *h, int refresh);                  /* rows a1, a3, a4 (pressure), a5; refresh: frozen aggregation */
int orc_update_values(orc *h, const orc_desc *d);          /* new values, same patterns (Newton step); -1 on a pattern change */
int orc_apply(orc *h, const double *v, double *z);        /* Algorithm 1 */
void orc_apply_operator(orc *h, const double *x, double *y);   /* eq:jac_system */
int orc_solve(orc *h, const double *b, double *x, double rtol, int m, int maxit, orc_info *info);
int orc_richardson(orc *h, const double *b, double *x, double rtol, int maxit, orc_info *info);   /* remark P:640-642 */
/* diagnostics / parity hooks */
int orc_num_levels(orc *h, int which);                    /* which: 0 mechanics SDC, 1 pressure */
void orc_level_sizes(orc *h, int which, int lvl, int64_t out[6]); /* n, nnz(A), nagg, nnz(P), nc, coarsest */
void orc_level_export(orc *h, int which, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v,
                      int32_t *agg, int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1);
void orc_counters(orc *h, int64_t out[4]);                /* skipped D_ss, perturbed pivots, fallbacks, - */
void orc_get_spp(orc *h, double *Dss, int32_t *rp, int32_t *ci, double *v);   /* CPR products (a3) */
void orc_get_cpr(orc *h, double *Dss, double *Dps, double *fs_eff);  /* D^(CPR) and the D_fs actually used (a1) */

/* standalone primitives for pins (tests only) */
int orc_mis2(int n, const int32_t *rp, const int32_t *ci, const uint32_t *hash, int rounds_variant,
             int32_t *state_out, int *nrounds);
void *orc_amg_build(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb,
                    const orc_opts *o);
void orc_amg_vcycle(void *hier, const double *b, double *x);    /* nc interleaved components */
int orc_amg_levels(void *hier);
void orc_amg_level_sizes(void *hier, int lvl, int64_t out[6]);
void orc_amg_level_export(void *hier, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v,
                          int32_t *agg, int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1);
void orc_amg_free(void *hier);
int orc_amg_level_detail(void *hier, int lvl, int32_t *st, int32_t *ph1, double *omega);
int orc_amg_level_colour(void *hier, int lvl, int32_t *colour);
int orc_amg_level_gs(void *hier, int lvl, double *dh);     /* gs_block of the level (0: multicolour), hybrid l1 diagonal */
void *orc_amg_build_coloured(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb,
                             const int32_t *colour0, const orc_opts *o);
int orc_level_colour(orc *h, int which, int lvl, int32_t *colour);
int orc_strength(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb,
                 double theta, uint8_t *E);
void *orc_ilu_build(int nx, int ny, int nz, int tx, int ty, int tz, const int32_t *rp, const int32_t *ci,
                    const double *v);
void orc_ilu_apply(void *ilu, const double *w, double *dz);
void orc_ilu_free(void *ilu);
void *orc_bgs_build(int nx, int ny, int nz, int tx, int ty, int tz, const int32_t *rp, const int32_t *ci, const double *v);
void orc_bgs_apply(void *bgs, const double *w, double *dz);     /* one hbgs sweep from zero: tile (L+D)^-1 w */
/* R-cheb: `degree` Chebyshev steps on D_l1^-1 A (scalar CSR, the oracle's l1 rule) from x0 (NULL = 0) */
int orc_cheb_smooth(int n, const int32_t *rp, const int32_t *ci, const double *v, int degree, double lower,
                    const double *b, const double *x0, double *x);
/* ---- residual.c: the nonlinear residual of Appendix B.1 (raw units, p in Pa) ---- */
typedef struct {
    int nx, ny, nz;
    double length, nu, biot, gravity;
    double rho_w0, rho_nw0, c_w, c_nw, mu_w, mu_nw, rho_s, p0, swr, snwr;
    double well_dbhp, rw_over_h;
    int burden, dirichlet_bottom;
} orc_phys;
/* R = r(x) with x = [u node-major | (s, p [Pa]) per cell]; mprev = (V m_w, V m_nw) per cell of the previous step */
int orc_residual(const orc_phys *P, double dt, const double *E, const double *perm, const double *phi0, const double *pref,
                 const int8_t *well, const double *x, const double *mprev, double *R);
void orc_masses(const orc_phys *P, const double *E, const double *phi0, const double *pref, const double *x, double *m);
void orc_porosity(const orc_phys *P, const double *E, const double *phi0, const double *pref, const double *x, double *phi);
#endif

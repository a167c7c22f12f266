/*
 * synth.c -- seeded synthetic input generator (shared by the oracle tests and
 * the CUDA path; holds NONE of the preconditioner / Krylov arithmetic).
 *
 * Builds ONE linearised Jacobian of the paper's coupled problem at a synthetic
 * state, in the block layout the C-ABI consumes:
 *
 *   A_uu  BSR 3x3  node rows x node cols   (Q1 elasticity + gravity term)
 *   A_uf  BSR 3x2  node rows x cell cols   [A_us | A_up]
 *   A_fu  BSR 2x3  cell rows x node cols   [A_su ; A_pu]
 *   A_ff  BSR 2x2  cell rows x cell cols   [[A_ss, A_sp],[A_ps, A_pp]]  (interleaved, P of P:606 applied)
 *   fs    2 doubles per cell: (D_sp, D_pp) of eq:FS_Dps_Dpp, row-scaled
 *   x_rand U(-1,1); b = A x_rand
 *
 * Physics, with PAPER.md line citations (P:n):
 *   element blocks   Appendix B.2, expansions P:1024-1095
 *   face blocks      TPFA + SPU, eq:num_flux_approx P:207-216, eq:avg_density P:218-227,
 *                    eq:jac_f_int P:1104-1137, expansions P:1147-1156 (sign: SURVEY D24)
 *   wells            eq:peaceman P:240-245, eq:peaceman2 P:249, eq:well_index P:254-257 (r_w: D15)
 *   transmissibility eq:trans / eq:half_trans P:905-918
 *   fluids, rel-perm P:714-721; porosity eq:linearized_porosity P:141
 *   row scaling      P:318-320 (D12); Dirichlet identity rows (D11)
 *
 * Plain C11 + OpenMP over independent rows (each row is gathered by one
 * thread in a fixed order, so the output is identical for any thread count).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int nx, ny, nz;
    int recipe;            /* 1..5: field recipe of BASELINE.json configs[0..4] (D17) */
    uint64_t seed;
    double E_median, E_sigma;
    double perm_median, perm_sigma;
    double nu, biot, gravity, dt;
    double rho_w0, rho_nw0, c_w, c_nw, mu_w, mu_nw, rho_s, p0;
    double swr, snwr;
    double well_dbhp, rw_over_h, state_dp, p_unit, length;
    int wells;             /* 1: vertical injector in column (0,0), producer in (nx-1,ny-1) */
    int dirichlet_bottom;  /* 1: all 3 displacement components fixed at z = 0 */
    int row_scale;         /* 1: block-row scaling (D12) */
    int burden;            /* SPE10-shaped workload (R-s10): this many seal layers at the top and at the bottom */
    int well_pattern;      /* 0: the corner pair above; 1: injector in the centre column, producers in the 4
                              corner columns, perforated through the reservoir layers only */
    int pad2_;
    double burden_perm, burden_phi;   /* seal units: 0.01 mD, 1 % */
} synth_params;

typedef struct {
    int32_t *uu_rowptr, *uu_col; double *uu_val;
    int32_t *uf_rowptr, *uf_col; double *uf_val;
    int32_t *fu_rowptr, *fu_col; double *fu_val;
    int32_t *ff_rowptr, *ff_col; double *ff_val;
    double *fs;            /* 2 per cell */
    double *x_rand, *b;    /* n = 3 N_n + 2 N_c */
    double *E, *perm, *phi, *sat, *pres;   /* per cell diagnostics */
    double *scales;        /* 3: s_u, s_s, s_p */
} synth_out;

/* ------------------------------------------------------------------ sizes */
static int64_t ipow3(int n) { return (int64_t)(3 * n + 1); }

void synth_sizes(const synth_params *P, int64_t out[8])
{
    int64_t nx = P->nx, ny = P->ny, nz = P->nz;
    int64_t Nn = (nx + 1) * (ny + 1) * (nz + 1);
    int64_t Nc = nx * ny * nz;
    int64_t Buu = ipow3(P->nx) * ipow3(P->ny) * ipow3(P->nz);
    int64_t faces = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1);
    out[0] = Nn; out[1] = Nc; out[2] = Buu; out[3] = 8 * Nc; out[4] = 8 * Nc;
    out[5] = Nc + 2 * faces; out[6] = 3 * Nn + 2 * Nc; out[7] = faces;
}

/* ------------------------------------------------------------------ RNG (D18) */
static uint64_t sm64(uint64_t *s)
{
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static double unif(uint64_t *s) { return (double)(sm64(s) >> 11) * (1.0 / 9007199254740992.0); }
static void normals(uint64_t *s, double *out, int64_t n)
{
    for (int64_t i = 0; i < n; i += 2) {
        double u1 = unif(s), u2 = unif(s);
        double r = sqrt(-2.0 * log(1.0 - u1));
        out[i] = r * cos(2.0 * M_PI * u2);
        if (i + 1 < n) out[i + 1] = r * sin(2.0 * M_PI * u2);
    }
}
static uint64_t stream_seed(uint64_t seed, int field) { return seed * 0x100ULL + (uint64_t)field; }

/* Gaussian-filtered, standardised noise (D17, recipes 4/5). */
static void correlated_field(const synth_params *P, double *g)
{
    const int R = 12; const double sd = 4.0;
    int nx = P->nx, ny = P->ny, nz = P->nz;
    int px = nx + 2 * R, py = ny + 2 * R, pz = nz + 2 * R;
    int64_t np = (int64_t)px * py * pz;
    double *a = (double *)malloc(sizeof(double) * np);
    double *t = (double *)malloc(sizeof(double) * np);
    uint64_t st = stream_seed(P->seed, 2);
    normals(&st, a, np);
    double w[25], ws = 0;
    for (int k = -R; k <= R; ++k) { w[k + R] = exp(-0.5 * k * k / (sd * sd)); ws += w[k + R]; }
    for (int k = 0; k < 2 * R + 1; ++k) w[k] /= ws;
    /* x pass: a -> t (valid where the stencil fits, else 0; only the interior is used) */
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < (int64_t)py * pz; ++q) {
        int64_t base = q * px;
        for (int i = 0; i < px; ++i) {
            double s = 0;
            if (i >= R && i < px - R)
                for (int k = -R; k <= R; ++k) s += w[k + R] * a[base + i + k];
            t[base + i] = s;
        }
    }
    /* y pass: t -> a */
#pragma omp parallel for schedule(static)
    for (int kz = 0; kz < pz; ++kz)
        for (int j = 0; j < py; ++j)
            for (int i = 0; i < px; ++i) {
                double s = 0;
                if (j >= R && j < py - R)
                    for (int k = -R; k <= R; ++k) s += w[k + R] * t[((int64_t)kz * py + j + k) * px + i];
                a[((int64_t)kz * py + j) * px + i] = s;
            }
    /* z pass: a -> cropped g */
#pragma omp parallel for schedule(static)
    for (int kz = 0; kz < nz; ++kz)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                double s = 0;
                for (int k = -R; k <= R; ++k)
                    s += w[k + R] * a[((int64_t)(kz + R + k) * py + (j + R)) * px + (i + R)];
                g[((int64_t)kz * ny + j) * nx + i] = s;
            }
    free(a); free(t);
    int64_t nc = (int64_t)nx * ny * nz;
    double m = 0; for (int64_t c = 0; c < nc; ++c) m += g[c]; m /= (double)nc;
    double v = 0; for (int64_t c = 0; c < nc; ++c) v += (g[c] - m) * (g[c] - m); v /= (double)nc;
    double isd = v > 0 ? 1.0 / sqrt(v) : 1.0;
    for (int64_t c = 0; c < nc; ++c) g[c] = (g[c] - m) * isd;
}

/* Staircase benchmark geometry (R-stair; the paper gives it only as a figure): a channel of
 * width 1/8 of the side winds once around the domain at an inset of 1/8 in four straight legs, each leg one
 * quarter of the height lower than the previous one -- a descending square spiral "staircase".  Leg 0 runs
 * along +x near y = 1/8 in the top quarter, leg 1 along +y near x = 7/8, leg 2 along -x near y = 7/8, leg 3
 * along -y near x = 1/8 in the bottom quarter; at each corner the channel spans both legs' z-bands.
 * Normalised cell-centre coordinates u, v, w in [0, 1). */
static int stair_channel(double u, double v, double w)
{
    const double a = 0.125, b = 0.25, c = 0.75, d = 0.875;
    int q = (int)(4.0 * (1.0 - w)); if (q > 3) q = 3;          /* z band: 0 = top quarter ... 3 = bottom */
    const int in_s = (v >= a && v < b), in_e = (u >= c && u < d), in_n = (v >= c && v < d), in_w = (u >= a && u < b);
    const int ux = (u >= a && u < d), vy = (v >= a && v < d);
    if ((q == 0 || q == 1) && in_s && ux && (q == 0 || in_e)) return 1;   /* leg 0 (+ its corner step into leg 1) */
    if ((q == 1 || q == 2) && in_e && vy && (q == 1 || in_n)) return 1;   /* leg 1 */
    if ((q == 2 || q == 3) && in_n && ux && (q == 2 || in_w)) return 1;   /* leg 2 */
    if (q == 3 && in_w && vy) return 1;                                    /* leg 3 */
    return 0;
}

static void make_fields(const synth_params *P, double *E, double *perm, double *phi, double *sat)
{
    int64_t nx = P->nx, ny = P->ny, nz = P->nz, nc = nx * ny * nz;
    uint64_t st;
    if (P->recipe == 3) {
        /* layered: per z-layer (D17) */
        double *nl = (double *)malloc(sizeof(double) * (nz + 1));
        st = stream_seed(P->seed, 2); normals(&st, nl, nz);
        st = stream_seed(P->seed, 1);
        for (int64_t k = 0; k < nz; ++k) {
            double lk = P->perm_sigma * nl[k];
            double cl = log(1e3);
            if (lk > cl) lk = cl;
            if (lk < -cl) lk = -cl;
            double Ek = pow(10.0, 8.0 + 2.0 * unif(&st));
            for (int64_t q = 0; q < nx * ny; ++q) {
                perm[k * nx * ny + q] = P->perm_median * exp(lk);
                E[k * nx * ny + q] = Ek;
            }
        }
        free(nl);
    } else {
        double *z = (double *)malloc(sizeof(double) * (nc + 1));
        st = stream_seed(P->seed, 1); normals(&st, z, nc);
        for (int64_t c = 0; c < nc; ++c) E[c] = P->E_median * exp(P->E_sigma * z[c]);
        if (P->recipe >= 4) correlated_field(P, z);
        else { st = stream_seed(P->seed, 2); normals(&st, z, nc); }
        for (int64_t c = 0; c < nc; ++c) perm[c] = P->perm_median * exp(P->perm_sigma * z[c]);
        free(z);
    }
    st = stream_seed(P->seed, 3);
    for (int64_t c = 0; c < nc; ++c) phi[c] = 0.15 + 0.10 * unif(&st);
    if (P->recipe == 6)                                  /* staircase: 1000 mD / 0.20 channel in 1 mD / 0.05 seal (Table 1) */
        for (int64_t c = 0; c < nc; ++c) {
            const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
            const int ch = stair_channel((i + 0.5) / nx, (j + 0.5) / ny, (k + 0.5) / nz);
            perm[c] = ch ? 1000 * 9.869233e-16 : 9.869233e-16;
            phi[c] = ch ? 0.20 : 0.05;
        }
    if (P->burden > 0)                                   /* over- and underburden seal layers */
        for (int64_t c = 0; c < nc; ++c) {
            int64_t k = c / (nx * ny);
            if (k < P->burden || k >= nz - P->burden) { perm[c] = P->burden_perm; phi[c] = P->burden_phi; }
        }
    st = stream_seed(P->seed, 4);
    for (int64_t c = 0; c < nc; ++c) sat[c] = 0.2 + 0.6 * unif(&st);
}

/* ------------------------------------------------------------------ Q1 reference integrals */
/* local node a = ai + 2 aj + 4 ak, N_a = prod (1 +- xi)/2 on [-1,1]^3 */
typedef struct { double I1[8][8][3][3]; double I2[8][8][3]; double I0[8]; double Id[8][3]; } q1_t;

static void q1_integrals(double h, q1_t *Q)
{
    memset(Q, 0, sizeof(*Q));
    const double gp[2] = {-1.0 / sqrt(3.0), 1.0 / sqrt(3.0)};
    const double J = h / 2.0, detJ = J * J * J;
    for (int gx = 0; gx < 2; ++gx) for (int gy = 0; gy < 2; ++gy) for (int gz = 0; gz < 2; ++gz) {
        double xi[3] = {gp[gx], gp[gy], gp[gz]};
        double N[8], dN[8][3];
        for (int a = 0; a < 8; ++a) {
            int s[3] = {(a & 1) ? 1 : -1, (a & 2) ? 1 : -1, (a & 4) ? 1 : -1};
            double f[3], df[3];
            for (int d = 0; d < 3; ++d) { f[d] = 0.5 * (1 + s[d] * xi[d]); df[d] = 0.5 * s[d] / J; }
            N[a] = f[0] * f[1] * f[2];
            dN[a][0] = df[0] * f[1] * f[2];
            dN[a][1] = f[0] * df[1] * f[2];
            dN[a][2] = f[0] * f[1] * df[2];
        }
        for (int a = 0; a < 8; ++a) {
            Q->I0[a] += N[a] * detJ;
            for (int d = 0; d < 3; ++d) Q->Id[a][d] += dN[a][d] * detJ;
            for (int b = 0; b < 8; ++b)
                for (int d = 0; d < 3; ++d) {
                    Q->I2[a][b][d] += N[a] * dN[b][d] * detJ;
                    for (int e = 0; e < 3; ++e) Q->I1[a][b][d][e] += dN[a][d] * dN[b][e] * detJ;
                }
        }
    }
}

/* ------------------------------------------------------------------ per-cell state */
typedef struct {
    double lam, mu, Kdr, phi, s, p, z;
    double rw, rnw, drw, drnw;           /* densities and d/dp */
    double krw, krnw, dkrw, dkrnw;       /* rel perms and d/ds */
    double drho_deps, drho_ds, drho_dp, dphi_dp, dphi_deps;
} cell_t;

/* phi: porosity at the state; phi0: the reference porosity of eq:linearized_porosity (its compressibility term) */
static void cell_state(const synth_params *P, double E, double phi, double phi0, double s, double p, double z, cell_t *C)
{
    double nu = P->nu, b = P->biot;
    C->lam = E * nu / ((1 + nu) * (1 - 2 * nu));
    C->mu = E / (2 * (1 + nu));
    C->Kdr = E / (3 * (1 - 2 * nu));
    C->phi = phi; C->s = s; C->p = p; C->z = z;
    C->rw = P->rho_w0 * (1 + P->c_w * (p - P->p0));
    C->rnw = P->rho_nw0 * (1 + P->c_nw * (p - P->p0));
    C->drw = P->rho_w0 * P->c_w;
    C->drnw = P->rho_nw0 * P->c_nw;
    double span = 1.0 - P->swr - P->snwr;
    double sh = (s - P->swr) / span, dsh = 1.0 / span;
    if (sh <= 0) { sh = 0; dsh = 0; }
    if (sh >= 1) { sh = 1; dsh = 0; }
    C->krw = sh * sh; C->dkrw = 2 * sh * dsh;
    C->krnw = (1 - sh) * (1 - sh); C->dkrnw = -2 * (1 - sh) * dsh;
    C->dphi_deps = b;                                   /* eq:linearized_porosity */
    C->dphi_dp = (b - phi0) * (1 - b) / C->Kdr;
    double bracket = -P->rho_s + s * C->rw + (1 - s) * C->rnw;
    C->drho_deps = bracket * C->dphi_deps;
    C->drho_ds = phi * (C->rw - C->rnw);
    C->drho_dp = bracket * C->dphi_dp + s * phi * C->drw + (1 - s) * phi * C->drnw; /* P:1030, drho_s/dp = 0 */
}

/* well placement (R-wells, R-s10, R-stair): 0 none, 1 injector, 2 producer perforation in cell (i, j, k) */
static int well_type(const synth_params *P, int i, int j, int k)
{
    const int nx = P->nx, ny = P->ny, nz = P->nz;
    const int kw0 = P->burden > 0 ? P->burden : 0, kw1 = P->burden > 0 ? nz - P->burden : nz;   /* perforated layers */
    int inj = (i == 0 && j == 0), prod = (i == nx - 1 && j == ny - 1);
    if (P->well_pattern == 1) {
        inj = (i == nx / 2 && j == ny / 2);
        prod = (i == 0 || i == nx - 1) && (j == 0 || j == ny - 1);
    }
    if (P->well_pattern == 2) {                  /* staircase: channel ends, channel cells only */
        const int ci0 = (int)(0.1875 * nx), cj0 = (int)(0.1875 * ny);
        inj = (i == (int)(0.5 * nx) && j == cj0);
        prod = (i == ci0 && j == (int)(0.5 * ny));
        if (!stair_channel((i + 0.5) / nx, (j + 0.5) / ny, (k + 0.5) / nz)) inj = prod = 0;
    }
    if (k < kw0 || k >= kw1) inj = prod = 0;
    return inj ? 1 : prod ? 2 : 0;
}

/* ------------------------------------------------------------------ state only */
/* The per-cell fields (E, perm, phi, sat) and linearisation pressure of synth_generate, and x_rand, without
 * assembling the Jacobian: the input of a GPU assembly.  Same streams, same values. */
static void state_pressure(const synth_params *P, double *pres)
{
    const int nx = P->nx, ny = P->ny, nz = P->nz;
    const int64_t Nc = (int64_t)nx * ny * nz;
    const double h = (P->length > 0 ? P->length : 1.0) / nx, g = P->gravity, ztop = nz * h;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) {
        int64_t k = c / ((int64_t)nx * ny);
        double zc = (k + 0.5) * h;
        int64_t ci = c % nx, cj = (c / nx) % ny;
        double xy = ((ci + 0.5) + (cj + 0.5)) / (double)(nx + ny);
        pres[c] = P->p0 + P->rho_w0 * g * (ztop - zc) + P->state_dp * (1.0 - 2.0 * xy);
    }
}
static void draw_x_rand(const synth_params *P, double *x, int64_t n)
{
    uint64_t st = stream_seed(P->seed, 0);
    for (int64_t q = 0; q < n; ++q) x[q] = -1.0 + 2.0 * unif(&st);
}
int synth_fields(const synth_params *P, double *E, double *perm, double *phi, double *sat, double *pres, double *x_rand,
                 int8_t *well)
{
    if (P->nx < 1 || P->ny < 1 || P->nz < 1) return -1;
    int64_t sz[8]; synth_sizes(P, sz);
    make_fields(P, E, perm, phi, sat);
    state_pressure(P, pres);
    if (well)
        for (int64_t c = 0; c < sz[1]; ++c)
            well[c] = (int8_t)(P->wells ? well_type(P, (int)(c % P->nx), (int)((c / P->nx) % P->ny), (int)(c / ((int64_t)P->nx * P->ny))) : 0);
    if (x_rand) draw_x_rand(P, x_rand, sz[6]);
    return 0;
}

/* ------------------------------------------------------------------ generator */
/* the Jacobian blocks at the state given by the cell fields (phi0 = NULL: phi is also the reference porosity) */
static void assemble_at(const synth_params *P, const double *E, const double *perm, const double *phi, const double *phi0,
                        const double *sat, const double *pres, synth_out *O)
{
    const int nx = P->nx, ny = P->ny, nz = P->nz;
    int64_t sz[8]; synth_sizes(P, sz);
    const int64_t Nn = sz[0], Nc = sz[1];
    const int NX = nx + 1, NY = ny + 1;
    const double h = (P->length > 0 ? P->length : 1.0) / nx, V = h * h * h, g = P->gravity, b = P->biot, dt = P->dt;
    const double ztop = nz * h;
    cell_t *C = (cell_t *)malloc(sizeof(cell_t) * Nc);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) {
        int64_t k = c / ((int64_t)nx * ny);
        double zc = (k + 0.5) * h;
        cell_state(P, E[c], phi[c], phi0 ? phi0[c] : phi[c], sat[c], pres[c], zc, &C[c]);
    }
    q1_t Q; q1_integrals(h, &Q);

    /* ---------------- A_uu, A_uf : node rows (gather over the <= 8 adjacent elements) */
    {
        int32_t *rp = O->uu_rowptr, *rpf = O->uf_rowptr;
        rp[0] = 0; rpf[0] = 0;
        for (int64_t n = 0; n < Nn; ++n) {
            int i = n % NX, j = (n / NX) % NY, k = n / ((int64_t)NX * NY);
            int cx = 1 + (i > 0) + (i < nx), cy = 1 + (j > 0) + (j < ny), cz = 1 + (k > 0) + (k < nz);
            int ex = (i > 0) + (i < nx), ey = (j > 0) + (j < ny), ez = (k > 0) + (k < nz);
            rp[n + 1] = rp[n] + cx * cy * cz;
            rpf[n + 1] = rpf[n] + ex * ey * ez;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < Nn; ++n) {
        int i = n % NX, j = (n / NX) % NY, k = n / ((int64_t)NX * NY);
        int pos27[27];
        int64_t p0 = O->uu_rowptr[n], q = p0;
        for (int dk = -1; dk <= 1; ++dk) for (int dj = -1; dj <= 1; ++dj) for (int di = -1; di <= 1; ++di) {
            int code = (dk + 1) * 9 + (dj + 1) * 3 + (di + 1);
            int ii = i + di, jj = j + dj, kk = k + dk;
            if (ii < 0 || ii > nx || jj < 0 || jj > ny || kk < 0 || kk > nz) { pos27[code] = -1; continue; }
            pos27[code] = (int)(q - p0);
            O->uu_col[q] = (int32_t)(ii + (int64_t)NX * (jj + (int64_t)NY * kk));
            memset(&O->uu_val[9 * q], 0, 9 * sizeof(double));
            ++q;
        }
        int64_t f0 = O->uf_rowptr[n], fq = f0;
        int posc[8];
        for (int ek = -1; ek <= 0; ++ek) for (int ej = -1; ej <= 0; ++ej) for (int ei = -1; ei <= 0; ++ei) {
            int code = (ek + 1) * 4 + (ej + 1) * 2 + (ei + 1);
            int ci = i + ei, cj = j + ej, ck = k + ek;
            if (ci < 0 || ci >= nx || cj < 0 || cj >= ny || ck < 0 || ck >= nz) { posc[code] = -1; continue; }
            posc[code] = (int)(fq - f0);
            O->uf_col[fq] = (int32_t)(ci + (int64_t)nx * (cj + (int64_t)ny * ck));
            memset(&O->uf_val[6 * fq], 0, 6 * sizeof(double));
            ++fq;
        }
        for (int code = 0; code < 8; ++code) {
            if (posc[code] < 0) continue;
            int ei = (code & 1) - 1, ej = ((code >> 1) & 1) - 1, ek = ((code >> 2) & 1) - 1;
            int64_t c = (i + ei) + (int64_t)nx * ((j + ej) + (int64_t)ny * (k + ek));
            const cell_t *cc = &C[c];
            int a = (-ei) + 2 * (-ej) + 4 * (-ek);      /* local index of node n in element c */
            for (int bl = 0; bl < 8; ++bl) {
                int bi = bl & 1, bj = (bl >> 1) & 1, bk = (bl >> 2) & 1;
                int di = ei + bi, dj = ej + bj, dk = ek + bk;   /* offset node m - node n */
                int pcode = (dk + 1) * 9 + (dj + 1) * 3 + (di + 1);
                double *blk = &O->uu_val[9 * (p0 + pos27[pcode])];
                double trace = Q.I1[a][bl][0][0] + Q.I1[a][bl][1][1] + Q.I1[a][bl][2][2];
                for (int d = 0; d < 3; ++d)
                    for (int e = 0; e < 3; ++e) {
                        double v = cc->lam * Q.I1[a][bl][d][e] + cc->mu * Q.I1[a][bl][e][d];
                        if (d == e) v += cc->mu * trace;
                        if (d == 2) v += g * cc->drho_deps * Q.I2[a][bl][e];   /* P:971 gravity term */
                        blk[3 * d + e] += v;
                    }
            }
            double *bf = &O->uf_val[6 * (f0 + posc[code])];
            for (int d = 0; d < 3; ++d) {
                bf[2 * d + 0] += (d == 2) ? g * cc->drho_ds * Q.I0[a] : 0.0;                 /* A_us P:975 */
                bf[2 * d + 1] += -b * Q.Id[a][d] + ((d == 2) ? g * cc->drho_dp * Q.I0[a] : 0.0); /* A_up P:978 */
            }
        }
    }

    /* ---------------- A_fu : cell rows, 8 nodes each (ascending node id) */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c <= Nc; ++c) O->fu_rowptr[c] = (int32_t)(8 * c);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) {
        int i = c % nx, j = (c / nx) % ny, k = c / ((int64_t)nx * ny);
        const cell_t *cc = &C[c];
        for (int a = 0; a < 8; ++a) {
            int ai = a & 1, aj = (a >> 1) & 1, ak = (a >> 2) & 1;
            int64_t q = 8 * c + a;
            O->fu_col[q] = (int32_t)((i + ai) + (int64_t)NX * ((j + aj) + (int64_t)NY * (k + ak)));
            for (int d = 0; d < 3; ++d) {
                O->fu_val[6 * q + d] = cc->s * cc->rw * cc->dphi_deps * Q.Id[a][d];           /* A_su P:984 */
                O->fu_val[6 * q + 3 + d] = (1 - cc->s) * cc->rnw * cc->dphi_deps * Q.Id[a][d]; /* A_pu P:1001 */
            }
        }
    }

    /* ---------------- A_ff : cell rows, 7-point TPFA + accumulation + wells */
    {
        int32_t *rp = O->ff_rowptr; rp[0] = 0;
        for (int64_t c = 0; c < Nc; ++c) {
            int i = c % nx, j = (c / nx) % ny, k = c / ((int64_t)nx * ny);
            rp[c + 1] = rp[c] + 1 + (i > 0) + (i < nx - 1) + (j > 0) + (j < ny - 1) + (k > 0) + (k < nz - 1);
        }
    }
    /* well geometry (D15): WI of eq:well_index with r_w = rw_over_h * h, s_k = 0 */
    const double rpe = 0.28 * sqrt(h * h + h * h) / 2.0;
    const double lnr = log(rpe / (P->rw_over_h * h));
    const int kw1 = P->burden > 0 ? nz - P->burden : nz;   /* bottom of the perforated layers */
    const double zbh = (kw1 - 0.5) * h;
    const double pbh_ref = P->p0 + P->rho_w0 * g * (ztop - zbh);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) {
        int i = c % nx, j = (c / nx) % ny, k = c / ((int64_t)nx * ny);
        const cell_t *K = &C[c];
        int64_t r0 = O->ff_rowptr[c], q = r0, diag = -1;
        int64_t nb[7]; int64_t np = 0;
        const int64_t sx = 1, sy = nx, sz = (int64_t)nx * ny;
        if (k > 0) nb[np++] = c - sz;
        if (j > 0) nb[np++] = c - sy;
        if (i > 0) nb[np++] = c - sx;
        nb[np++] = c;
        if (i < nx - 1) nb[np++] = c + sx;
        if (j < ny - 1) nb[np++] = c + sy;
        if (k < nz - 1) nb[np++] = c + sz;
        for (int64_t t = 0; t < np; ++t) {
            O->ff_col[q + t] = (int32_t)nb[t];
            memset(&O->ff_val[4 * (q + t)], 0, 4 * sizeof(double));
            if (nb[t] == c) diag = q + t;
        }
        double *D = &O->ff_val[4 * diag];
        /* accumulation (element part, P:989-1014 with expansions P:1036-1079) */
        D[0] += V * K->phi * K->rw;                                   /* dm_w/ds  */
        D[1] += V * (K->s * K->rw * K->dphi_dp + K->phi * K->s * K->drw);  /* dm_w/dp  */
        D[2] += V * (-K->phi * K->rnw);                               /* dm_nw/ds */
        D[3] += V * ((1 - K->s) * K->rnw * K->dphi_dp + K->phi * (1 - K->s) * K->drnw);
        /* faces (eq:jac_f_int): this cell is K (lower) or L (upper) of each face */
        for (int64_t t = 0; t < np; ++t) {
            int64_t o = nb[t];
            if (o == c) continue;
            int64_t cK = c < o ? c : o, cL = c < o ? o : c;
            const cell_t *A = &C[cK], *B = &C[cL];
            /* half transmissibilities eq:half_trans: |f| (x_f-x_K).k.n_f / |x_f-x_K|^2 = h^2 k (h/2)/(h/2)^2 */
            double tK = h * h * perm[cK] * (h / 2) / ((h / 2) * (h / 2));
            double tL = h * h * perm[cL] * (h / 2) / ((h / 2) * (h / 2));
            double Ups = (tK + tL) > 0 ? tK * tL / (tK + tL) : 0.0;   /* eq:trans */
            double dz = B->z - A->z;
            double sgn = (c == cK) ? -1.0 : 1.0;                     /* [[psi_c]]_f : -1 for K, +1 for L */
            for (int ph = 0; ph < 2; ++ph) {
                double rK = ph ? A->rnw : A->rw, rL = ph ? B->rnw : B->rw;
                double dK = ph ? A->drnw : A->drw, dL = ph ? B->drnw : B->drw;
                double krK = ph ? A->krnw : A->krw, krL = ph ? B->krnw : B->krw;
                double dkK = ph ? A->dkrnw : A->dkrw, dkL = ph ? B->dkrnw : B->dkrw;
                double mu = ph ? P->mu_nw : P->mu_w;
                int presK = krK > 0, presL = krL > 0;               /* "phase appears" = lambda > 0 (SPEC) */
                double vr, dvrK, dvrL;
                if (presK && presL) { vr = 0.5 * (rK + rL); dvrK = 0.5 * dK; dvrL = 0.5 * dL; }
                else if (presK) { vr = rK; dvrK = dK; dvrL = 0; }
                else if (presL) { vr = rL; dvrK = 0; dvrL = dL; }
                else { vr = 0; dvrK = 0; dvrL = 0; }
                double Phi = Ups * ((B->p - A->p) + vr * g * dz);
                int upL = Phi > 0;                                    /* tie -> K */
                double rup = upL ? rL : rK, drup = upL ? dL : dK;
                double lup = (upL ? krL : krK) / mu, dkup = upL ? dkL : dkK;
                /* dF/ds_j (upstream only), dF/dp_K, dF/dp_L */
                double dFds = rup / mu * Phi * dkup;
                double dFdpK = (upL ? 0.0 : drup * lup) * Phi + rup * lup * Ups * (-1.0 + dvrK * g * dz);
                double dFdpL = (upL ? drup * lup : 0.0) * Phi + rup * lup * Ups * (1.0 + dvrL * g * dz);
                double coef = sgn * dt;
                int row = ph;   /* w -> s-row (0), nw -> p-row (1) */
                /* locate blocks for K and L in this row */
                int64_t posK = -1, posL = -1;
                for (int64_t u = 0; u < np; ++u) { if (nb[u] == cK) posK = r0 + u; if (nb[u] == cL) posL = r0 + u; }
                int64_t posUp = upL ? posL : posK;
                O->ff_val[4 * posUp + 2 * row + 0] += coef * dFds;
                O->ff_val[4 * posK + 2 * row + 1] += coef * dFdpK;
                O->ff_val[4 * posL + 2 * row + 1] += coef * dFdpL;
            }
        }
        /* wells (eq:peaceman, eq:peaceman2; derivatives P:1042-1095; residual sign P:941) */
        if (P->wells) {
            const int wt = well_type(P, i, j, k);
            const int inj = wt == 1, prod = wt == 2;
            if (inj || prod) {
                double WI = 2 * M_PI * h * perm[c] / lnr;
                double pbh = pbh_ref + (inj ? P->well_dbhp : -P->well_dbhp);
                double lw = K->krw / P->mu_w, lnw = K->krnw / P->mu_nw;
                for (int ph = 0; ph < 2; ++ph) {
                    double r = ph ? K->rnw : K->rw, dr = ph ? K->drnw : K->drw;
                    double Phi = WI * ((pbh + r * g * zbh) - (K->p + r * g * K->z));
                    double dPhi = WI * (-1.0 + dr * g * (zbh - K->z));
                    double dqds = 0, dqdp = 0;   /* d(q^I - q^P)/ds, /dp */
                    if (inj) {
                        if (ph == 0 && Phi > 0) {   /* water injector: q^I_w = rho_w (l_w + l_nw) Phi_w */
                            dqds = r * (K->dkrw / P->mu_w + K->dkrnw / P->mu_nw) * Phi;
                            dqdp = dr * (lw + lnw) * Phi + r * (lw + lnw) * dPhi;
                        }
                    } else if (Phi < 0) {          /* producer: q^P_l = -rho_l l_l Phi_l */
                        double l = ph ? lnw : lw, dk = ph ? K->dkrnw : K->dkrw, mu = ph ? P->mu_nw : P->mu_w;
                        dqds = -(-r * dk / mu * Phi);
                        dqdp = -(-dr * l * Phi - r * l * dPhi);
                    }
                    D[2 * ph + 0] += -dt * dqds;
                    D[2 * ph + 1] += -dt * dqdp;
                }
            }
        }
    }

    /* ---------------- fixed-stress diagonals (eq:FS_Dps_Dpp) */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) {
        O->fs[2 * c + 0] = V * b * b / C[c].Kdr * C[c].s * C[c].rw;
        O->fs[2 * c + 1] = V * b * b / C[c].Kdr * (1 - C[c].s) * C[c].rnw;
    }

    /* ---------------- units of the pressure unknown ("dimensionally consistent units";
     * Table 1 quotes pressures in MPa): p columns (A_up, A_sp, A_pp and the FS diagonals,
     * which sit in p columns) are multiplied by p_unit [Pa per unit of the unknown]. */
    if (P->p_unit != 1.0 && P->p_unit > 0) {
        const double pu = P->p_unit;
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < sz[3]; ++q) for (int d = 0; d < 3; ++d) O->uf_val[6 * q + 2 * d + 1] *= pu;
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < sz[5]; ++q) { O->ff_val[4 * q + 1] *= pu; O->ff_val[4 * q + 3] *= pu; }
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < Nc; ++c) { O->fs[2 * c] *= pu; O->fs[2 * c + 1] *= pu; }
    }

    /* ---------------- block-row scaling (D12) */
    double su = 1, ss = 1, sp = 1;
    if (P->row_scale) {
        double mu_ = 0, ms = 0, mp = 0;
        for (int64_t n = 0; n < 3 * Nn; ++n) {
            int64_t node = n / 3; int d = n % 3; double s = 0;
            for (int64_t q = O->uu_rowptr[node]; q < O->uu_rowptr[node + 1]; ++q)
                for (int e = 0; e < 3; ++e) s += fabs(O->uu_val[9 * q + 3 * d + e]);
            if (s > mu_) mu_ = s;
        }
        for (int64_t c = 0; c < Nc; ++c) {
            double s0 = 0, s1 = 0;
            for (int64_t q = O->ff_rowptr[c]; q < O->ff_rowptr[c + 1]; ++q) {
                s0 += fabs(O->ff_val[4 * q + 0]);
                s1 += fabs(O->ff_val[4 * q + 3]);
            }
            if (s0 > ms) ms = s0;
            if (s1 > mp) mp = s1;
        }
        su = mu_ > 0 ? 1.0 / mu_ : 1.0; ss = ms > 0 ? 1.0 / ms : 1.0; sp = mp > 0 ? 1.0 / mp : 1.0;
    }
    O->scales[0] = su; O->scales[1] = ss; O->scales[2] = sp;
    const int64_t Buu = sz[2], Buf = sz[3], Bff = sz[5];
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 9 * Buu; ++q) O->uu_val[q] *= su;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < 6 * Buf; ++q) O->uf_val[q] *= su;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < Buf; ++q)
        for (int d = 0; d < 3; ++d) { O->fu_val[6 * q + d] *= ss; O->fu_val[6 * q + 3 + d] *= sp; }
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < Bff; ++q) {
        O->ff_val[4 * q + 0] *= ss; O->ff_val[4 * q + 1] *= ss;
        O->ff_val[4 * q + 2] *= sp; O->ff_val[4 * q + 3] *= sp;
    }
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < Nc; ++c) { O->fs[2 * c] *= ss; O->fs[2 * c + 1] *= sp; }

    /* ---------------- Dirichlet identity rows / zero columns at z = 0 (D11) */
    if (P->dirichlet_bottom) {
        const int64_t nbot = (int64_t)NX * NY;
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < Nn; ++n) {
            int fixed_row = n < nbot;
            for (int64_t q = O->uu_rowptr[n]; q < O->uu_rowptr[n + 1]; ++q) {
                int fixed_col = O->uu_col[q] < nbot;
                if (fixed_row || fixed_col) {
                    memset(&O->uu_val[9 * q], 0, 9 * sizeof(double));
                    if (fixed_row && O->uu_col[q] == n) {
                        O->uu_val[9 * q + 0] = 1; O->uu_val[9 * q + 4] = 1; O->uu_val[9 * q + 8] = 1;
                    }
                }
            }
            if (fixed_row)
                for (int64_t q = O->uf_rowptr[n]; q < O->uf_rowptr[n + 1]; ++q) memset(&O->uf_val[6 * q], 0, 6 * sizeof(double));
        }
#pragma omp parallel for schedule(static)
        for (int64_t q = 0; q < Buf; ++q)
            if (O->fu_col[q] < nbot) memset(&O->fu_val[6 * q], 0, 6 * sizeof(double));
    }

    free(C);
}

int synth_generate(const synth_params *P, synth_out *O)
{
    if (P->nx < 1 || P->ny < 1 || P->nz < 1) return -1;
    int64_t sz[8]; synth_sizes(P, sz);
    const int64_t Nn = sz[0], Nc = sz[1];
    make_fields(P, O->E, O->perm, O->phi, O->sat);
    /* linearisation state (DESIGN.md R-state): hydrostatic + a linear injector->producer drawdown of
       +-state_dp along the (x+y) diagonal, so every face carries flow and SPU upwinding is exercised */
    state_pressure(P, O->pres);
    assemble_at(P, O->E, O->perm, O->phi, NULL, O->sat, O->pres, O);

    /* ---------------- x_rand (seed stream 0) and b = A x_rand */
    draw_x_rand(P, O->x_rand, sz[6]);
    const double *xu = O->x_rand, *xf = O->x_rand + 3 * Nn;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < Nn; ++r) {
        double y[3] = {0, 0, 0};
        for (int64_t q = O->uu_rowptr[r]; q < O->uu_rowptr[r + 1]; ++q)
            for (int d = 0; d < 3; ++d) for (int e = 0; e < 3; ++e) y[d] += O->uu_val[9 * q + 3 * d + e] * xu[3 * (int64_t)O->uu_col[q] + e];
        for (int64_t q = O->uf_rowptr[r]; q < O->uf_rowptr[r + 1]; ++q)
            for (int d = 0; d < 3; ++d) for (int e = 0; e < 2; ++e) y[d] += O->uf_val[6 * q + 2 * d + e] * xf[2 * (int64_t)O->uf_col[q] + e];
        for (int d = 0; d < 3; ++d) O->b[3 * r + d] = y[d];
    }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < Nc; ++r) {
        double y[2] = {0, 0};
        for (int64_t q = O->fu_rowptr[r]; q < O->fu_rowptr[r + 1]; ++q)
            for (int d = 0; d < 2; ++d) for (int e = 0; e < 3; ++e) y[d] += O->fu_val[6 * q + 3 * d + e] * xu[3 * (int64_t)O->fu_col[q] + e];
        for (int64_t q = O->ff_rowptr[r]; q < O->ff_rowptr[r + 1]; ++q)
            for (int d = 0; d < 2; ++d) for (int e = 0; e < 2; ++e) y[d] += O->ff_val[4 * q + 2 * d + e] * xf[2 * (int64_t)O->ff_col[q] + e];
        O->b[3 * Nn + 2 * r] = y[0]; O->b[3 * Nn + 2 * r + 1] = y[1];
    }
    (void)Nc;
    return 0;
}

/* the Jacobian at a given state (the CPU reference of the GPU assembly inside a Newton loop):
 * fields E, perm, phi (porosity at the state), phi0 (reference porosity, NULL = phi), sat, pres (Pa); the
 * generator's fields, x_rand and b of `O` are not touched */
int synth_assemble_state(const synth_params *P, const double *E, const double *perm, const double *phi, const double *phi0,
                         const double *sat, const double *pres, synth_out *O)
{
    if (P->nx < 1 || P->ny < 1 || P->nz < 1) return -1;
    assemble_at(P, E, perm, phi, phi0, sat, pres, O);
    return 0;
}

/*
 * residual.c -- TEST INFRASTRUCTURE ONLY (the oracle of SURVEY NEXT-f1, the nonlinear step around the hot path).
 *
 * The discrete residual of the coupled multiphase poromechanics problem, Appendix B.1, in raw units
 * (N for the momentum rows, kg for the mass rows), written out element by element and face by face:
 *   r_u  = int grad^s(eta) : sigma'  -  int div(eta) b p  -  int eta . rho g
 *   r_w  = int psi (m_w - m_w,prev)  -  dt int psi (q^I_w - q^P_w)  -  dt sum_f [[psi]]_f F^f_w
 *   r_nw = the same for the non-wetting phase
 * with sigma' = C_dr : grad^s u, rho = (1 - phi) rho_s + phi (s rho_w + (1 - s) rho_nw),
 * m_w = phi rho_w s, m_nw = phi rho_nw (1 - s), the porosity law eq:linearized_porosity
 *   phi = phi_0 + b eps_v + (b - phi_0)(1 - b)/K_dr (p - p_ref)   (cell average of eps_v over the hexahedron),
 * TPFA fluxes with single-point upwinding and the phase-averaged density of eq:num_flux_approx / eq:avg_density
 * (P:207-227), Peaceman wells (eq:peaceman P:240-249; water-only injection with the total mobility, R-wells),
 * Q1 elements with 2 x 2 x 2 Gauss points.  The gravity term integrates rho pointwise: its porosity carries
 * eps_v(x) of the Gauss point, its phase densities and saturation are the cell's.  Dirichlet rows (bottom nodes,
 * R-dirichlet) are zero.  Plain sequential C, fp64, no contraction.  Only tests/ may call it.
 *
 * Its derivative at u = 0 is the Jacobian synth/ assembles (pinned by tests/test_oracle_newton.py with finite
 * differences); at u != 0 the Jacobian drops terms of order eps_v (the u-dependence of the cell densities inside
 * the gravity term), which the Newton loop tolerates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef struct { double K[8][8][3][3], NB[8][8][3], N0[8], D[8][3]; } q1int;

/* int_K of the Q1 shape products on a cube of side h (local node a: bit d set = upper end along axis d) */
static void q1int_build(double h, q1int *q)
{
    memset(q, 0, sizeof(*q));
    const double gp = 1.0 / sqrt(3.0), half = 0.5 * h, w = half * half * half;
    for (int gz = -1; gz <= 1; gz += 2)
        for (int gy = -1; gy <= 1; gy += 2)
            for (int gx = -1; gx <= 1; gx += 2) {
                const double xi[3] = {gx * gp, gy * gp, gz * gp};
                double N[8], dN[8][3];
                for (int a = 0; a < 8; ++a) {
                    double f[3], df[3];
                    for (int d = 0; d < 3; ++d) {
                        const double sgn = (a >> d) & 1 ? 1.0 : -1.0;
                        f[d] = 0.5 * (1.0 + sgn * xi[d]);
                        df[d] = 0.5 * sgn / half;
                    }
                    N[a] = f[0] * f[1] * f[2];
                    dN[a][0] = df[0] * f[1] * f[2];
                    dN[a][1] = f[0] * df[1] * f[2];
                    dN[a][2] = f[0] * f[1] * df[2];
                }
                for (int a = 0; a < 8; ++a) {
                    q->N0[a] += N[a] * w;
                    for (int d = 0; d < 3; ++d) q->D[a][d] += dN[a][d] * w;
                    for (int b = 0; b < 8; ++b)
                        for (int d = 0; d < 3; ++d) {
                            q->NB[a][b][d] += N[a] * dN[b][d] * w;
                            for (int e = 0; e < 3; ++e) q->K[a][b][d][e] += dN[a][d] * dN[b][e] * w;
                        }
                }
            }
}

typedef struct {
    double lam, mu, Kdr, s, p, z, phi, phi_e0, rw, rn, drw, drn, krw, krn;
} ocell;

static int64_t node_of(const orc_phys *P, int64_t c, int a)
{
    const int64_t nx = P->nx, ny = P->ny, NX = nx + 1, NY = ny + 1;
    const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    return (i + (a & 1)) + NX * ((j + ((a >> 1) & 1)) + NY * (k + ((a >> 2) & 1)));
}

/* cell K's state at x (u node-major, f = (s, p [Pa]) interleaved) */
static void ocell_at(const orc_phys *P, const q1int *q, double h, int64_t c, const double *E, const double *phi0,
                     const double *pref, const double *x, int64_t Nn, ocell *C)
{
    const double nu = P->nu, b = P->biot, V = h * h * h;
    C->lam = E[c] * nu / ((1 + nu) * (1 - 2 * nu));
    C->mu = E[c] / (2 * (1 + nu));
    C->Kdr = E[c] / (3 * (1 - 2 * nu));
    C->s = x[3 * Nn + 2 * c];
    C->p = x[3 * Nn + 2 * c + 1];
    C->z = ((double)(c / ((int64_t)P->nx * P->ny)) + 0.5) * h;
    double ev = 0.0;                                        /* V eps_v = int div u */
    for (int a = 0; a < 8; ++a) {
        const int64_t n = node_of(P, c, a);
        for (int d = 0; d < 3; ++d) ev = ev + q->D[a][d] * x[3 * n + d];
    }
    ev = ev / V;
    C->phi_e0 = phi0[c] + (b - phi0[c]) * (1 - b) / C->Kdr * (C->p - pref[c]);   /* porosity without the strain */
    C->phi = C->phi_e0 + b * ev;                                               /* eq:linearized_porosity */
    C->rw = P->rho_w0 * (1 + P->c_w * (C->p - P->p0));
    C->rn = P->rho_nw0 * (1 + P->c_nw * (C->p - P->p0));
    C->drw = P->rho_w0 * P->c_w;
    C->drn = P->rho_nw0 * P->c_nw;
    const double span = 1.0 - P->swr - P->snwr;
    double se = (C->s - P->swr) / span;
    if (se < 0) se = 0;
    if (se > 1) se = 1;
    C->krw = se * se;
    C->krn = (1 - se) * (1 - se);
}

void orc_porosity(const orc_phys *P, const double *E, const double *phi0, const double *pref, const double *x, double *phi)
{
    const double h = (P->length > 0 ? P->length : 1.0) / P->nx;
    const int64_t Nc = (int64_t)P->nx * P->ny * P->nz, Nn = (int64_t)(P->nx + 1) * (P->ny + 1) * (P->nz + 1);
    q1int q; q1int_build(h, &q);
    for (int64_t c = 0; c < Nc; ++c) { ocell C; ocell_at(P, &q, h, c, E, phi0, pref, x, Nn, &C); phi[c] = C.phi; }
}

void orc_masses(const orc_phys *P, const double *E, const double *phi0, const double *pref, const double *x, double *m)
{
    const double h = (P->length > 0 ? P->length : 1.0) / P->nx, V = h * h * h;
    const int64_t Nc = (int64_t)P->nx * P->ny * P->nz, Nn = (int64_t)(P->nx + 1) * (P->ny + 1) * (P->nz + 1);
    q1int q; q1int_build(h, &q);
    for (int64_t c = 0; c < Nc; ++c) {
        ocell C; ocell_at(P, &q, h, c, E, phi0, pref, x, Nn, &C);
        m[2 * c] = V * C.phi * C.rw * C.s;
        m[2 * c + 1] = V * C.phi * C.rn * (1 - C.s);
    }
}

int orc_residual(const orc_phys *P, double dt, const double *E, const double *perm, const double *phi0, const double *pref,
                 const int8_t *well, const double *x, const double *mprev, double *R)
{
    const int nx = P->nx, ny = P->ny, nz = P->nz;
    if (nx < 1 || ny < 1 || nz < 1) return -1;
    const int64_t Nc = (int64_t)nx * ny * nz, Nn = (int64_t)(nx + 1) * (ny + 1) * (nz + 1), P2 = (int64_t)nx * ny;
    const double h = (P->length > 0 ? P->length : 1.0) / nx, V = h * h * h, g = P->gravity, b = P->biot;
    q1int q; q1int_build(h, &q);
    memset(R, 0, sizeof(double) * (3 * Nn + 2 * Nc));
    ocell *C = (ocell *)malloc(sizeof(ocell) * Nc);
    for (int64_t c = 0; c < Nc; ++c) ocell_at(P, &q, h, c, E, phi0, pref, x, Nn, &C[c]);
    /* momentum: element contributions */
    for (int64_t c = 0; c < Nc; ++c) {
        const ocell *K = &C[c];
        const double bracket = -P->rho_s + K->s * K->rw + (1 - K->s) * K->rn;
        const double rho0 = P->rho_s + K->phi_e0 * bracket;      /* mixture density without the strain part */
        int64_t nd[8];
        for (int a = 0; a < 8; ++a) nd[a] = node_of(P, c, a);
        for (int a = 0; a < 8; ++a)
            for (int d = 0; d < 3; ++d) {
                double r = 0.0;
                for (int bb = 0; bb < 8; ++bb) {
                    const double tr = q.K[a][bb][0][0] + q.K[a][bb][1][1] + q.K[a][bb][2][2];
                    for (int e = 0; e < 3; ++e) {
                        double k = K->lam * q.K[a][bb][d][e] + K->mu * q.K[a][bb][e][d];
                        if (d == e) k = k + K->mu * tr;
                        r = r + k * x[3 * nd[bb] + e];
                        if (d == 2) r = r + g * bracket * b * q.NB[a][bb][e] * x[3 * nd[bb] + e];   /* rho's strain part */
                    }
                }
                r = r - b * K->p * q.D[a][d];                   /* - int div(eta) b p */
                if (d == 2) r = r + g * rho0 * q.N0[a];         /* - int eta . rho g, g = -g e_z */
                R[3 * nd[a] + d] += r;
            }
    }
    /* mass: accumulation */
    for (int64_t c = 0; c < Nc; ++c) {
        R[3 * Nn + 2 * c] = V * C[c].phi * C[c].rw * C[c].s - mprev[2 * c];
        R[3 * Nn + 2 * c + 1] = V * C[c].phi * C[c].rn * (1 - C[c].s) - mprev[2 * c + 1];
    }
    /* mass: faces (each face once, K = lower id, L = upper id; r_K -= dt F, r_L += dt F) */
    for (int64_t c = 0; c < Nc; ++c) {
        const int64_t i = c % nx, j = (c / nx) % ny, k = c / P2;
        const int64_t up[3] = {i + 1 < nx ? c + 1 : -1, j + 1 < ny ? c + nx : -1, k + 1 < nz ? c + P2 : -1};
        for (int t = 0; t < 3; ++t) {
            const int64_t L = up[t];
            if (L < 0) continue;
            const ocell *A = &C[c], *B = &C[L];
            const double tK = h * h * perm[c] * (h / 2) / ((h / 2) * (h / 2)), tL = h * h * perm[L] * (h / 2) / ((h / 2) * (h / 2));
            const double T = (tK + tL) > 0 ? tK * tL / (tK + tL) : 0.0;
            const double dz = B->z - A->z;
            for (int ph = 0; ph < 2; ++ph) {
                const double rK = ph ? A->rn : A->rw, rL = ph ? B->rn : B->rw;
                const double kK = ph ? A->krn : A->krw, kL = ph ? B->krn : B->krw, mu = ph ? P->mu_nw : P->mu_w;
                double ravg;
                if (kK > 0 && kL > 0) ravg = 0.5 * (rK + rL);
                else if (kK > 0) ravg = rK;
                else if (kL > 0) ravg = rL;
                else ravg = 0.0;
                const double Phi = T * ((B->p - A->p) + ravg * g * dz);
                const int fromL = Phi > 0;
                const double F = (fromL ? rL : rK) * (fromL ? kL : kK) / mu * Phi;
                R[3 * Nn + 2 * c + ph] -= dt * F;
                R[3 * Nn + 2 * L + ph] += dt * F;
            }
        }
    }
    /* mass: wells */
    const int kw1 = P->burden > 0 ? nz - P->burden : nz;
    const double zbh = (kw1 - 0.5) * h, ztop = nz * h;
    const double re = 0.28 * sqrt(h * h + h * h) / 2.0, lnr = log(re / (P->rw_over_h * h));
    for (int64_t c = 0; well && c < Nc; ++c) {
        if (!well[c]) continue;
        const ocell *K = &C[c];
        const double WI = 2 * M_PI * h * perm[c] / lnr;
        const double pbh = P->p0 + P->rho_w0 * g * (ztop - zbh) + (well[c] == 1 ? P->well_dbhp : -P->well_dbhp);
        const double lw = K->krw / P->mu_w, ln = K->krn / P->mu_nw;
        for (int ph = 0; ph < 2; ++ph) {
            const double r = ph ? K->rn : K->rw;
            const double Phi = WI * ((pbh + r * g * zbh) - (K->p + r * g * K->z));
            double src = 0.0;                                   /* q^I - q^P */
            if (well[c] == 1) { if (ph == 0 && Phi > 0) src = r * (lw + ln) * Phi; }
            else if (Phi < 0) src = r * (ph ? ln : lw) * Phi;
            R[3 * Nn + 2 * c + ph] -= dt * src;
        }
    }
    /* Dirichlet rows */
    if (P->dirichlet_bottom)
        for (int64_t n = 0; n < (int64_t)(nx + 1) * (ny + 1); ++n) R[3 * n] = R[3 * n + 1] = R[3 * n + 2] = 0.0;
    free(C);
    return 0;
}

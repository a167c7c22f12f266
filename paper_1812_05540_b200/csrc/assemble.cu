// assemble.cu -- GPU assembly of the linearised coupled Jacobian ("GPU assembly of the Appendix B
// Jacobian"): the four blocks of eq:jac_system and the fixed-stress diagonals (eq:FS_Dps_Dpp)
// from per-cell fields, in exactly the layout tsp_create consumes, directly in device memory -- the host never holds
// the 27 GB of a C5 Jacobian.  The synthetic generator (synth/synth.c) assembles the same matrices on the CPU and is
// the oracle of this step (tests/test_gpu_assemble.py); the two share no code.
//
// Physics (P:n = PAPER.md lines):
//   Q1 elasticity, 2x2x2 Gauss: A_uu = int grad(N_a)^T C grad(N_b) + the gravity term g d(rho)/d(eps_v)
//   Biot coupling:  A_us = g drho/ds int N_a e_z;  A_up = -b int dN_a/dx_d + g drho/dp int N_a e_z
//   A_su, A_pu:     s rho_w b int dN_a/dx_d, (1-s) rho_nw b int dN_a/dx_d
//   A_ff:           accumulation + TPFA two-phase fluxes with single-point upwinding and
//                   phase-averaged densities (eq:num_flux_approx P:207-216, eq:avg_density P:218-227,
//                   eq:jac_f_int P:1104-1137; sign convention SURVEY D24) + Peaceman wells (eq:peaceman P:240-257)
//   fluids / rel-perm: P:714-721; porosity: eq:linearized_porosity P:141
//   units of p (R-punit), block-row scaling 1/max row l1 (R-scale), bottom Dirichlet rows (R-dirichlet)
// One thread per row gathers every contribution of the row in a fixed order (no atomics on values).  A z-slab rank
// assembles its owned rows with global column ids; the row scaling needs the global row maxima, so the assembly is
// split: tsp_assemble (values + this rank's maxima) and tsp_assemble_scale (global scales + Dirichlet rows).
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <vector>

#include "tsp_internal.cuh"

namespace tsp {

// Gauss integrals of the Q1 shape functions on a cube of side h (local node a = ax + 2 ay + 4 az):
//   KK[a][b][d][e] = int dN_a/dx_d dN_b/dx_e,  NB[a][b][e] = int N_a dN_b/dx_e,  NI[a] = int N_a,  DN[a][d] = int dN_a/dx_d
struct Q1 {
    double KK[8][8][3][3], NB[8][8][3], NI[8], DN[8][3];
};

static void q1_tables(double h, Q1 &q)
{
    memset(&q, 0, sizeof(q));
    const double xg[2] = {-1.0 / std::sqrt(3.0), 1.0 / std::sqrt(3.0)};
    const double jac = 0.5 * h, wdet = jac * jac * jac;   // unit Gauss weights, |J| = (h/2)^3
    for (int p = 0; p < 8; ++p) {
        const double xi[3] = {xg[p & 1], xg[(p >> 1) & 1], xg[(p >> 2) & 1]};
        double N[8], G[8][3];
        for (int a = 0; a < 8; ++a) {
            double f[3], df[3];
            for (int d = 0; d < 3; ++d) {
                const double sgn = ((a >> d) & 1) ? 1.0 : -1.0;
                f[d] = 0.5 * (1.0 + sgn * xi[d]);
                df[d] = 0.5 * sgn / jac;
            }
            N[a] = f[0] * f[1] * f[2];
            G[a][0] = df[0] * f[1] * f[2];
            G[a][1] = f[0] * df[1] * f[2];
            G[a][2] = f[0] * f[1] * df[2];
        }
        for (int a = 0; a < 8; ++a) {
            q.NI[a] += N[a] * wdet;
            for (int d = 0; d < 3; ++d) q.DN[a][d] += G[a][d] * wdet;
            for (int b = 0; b < 8; ++b)
                for (int d = 0; d < 3; ++d) {
                    q.NB[a][b][d] += N[a] * G[b][d] * wdet;
                    for (int e = 0; e < 3; ++e) q.KK[a][b][d][e] += G[a][d] * G[b][e] * wdet;
                }
        }
    }
}

struct AsmGeo {
    int nx, ny, nz;
    int64_t node0, cell0;   // first owned node / cell (global)
    int nn, ncl;            // owned nodes / cells
    double h;
};

// state of one cell at the linearisation point (Lame constants, densities, relative permeabilities and the
// derivatives the blocks need)
struct CellSt {
    double lam, mu, Kdr, phi, s, p, z;
    double rw, rn, drw, drn, krw, krn, dkrw, dkrn;
    double drho_de, drho_ds, drho_dp, dphi_dp;
};

__device__ __forceinline__ CellSt cell_st(const tsp_asm_params &P, const AsmGeo &g, int64_t c, const double *__restrict__ E,
                                          const double *__restrict__ phi, const double *__restrict__ sat,
                                          const double *__restrict__ pres, const double *__restrict__ phi0 = nullptr)
{
    CellSt C;
    const double nu = P.nu, b = P.biot, e = E[c];
    C.lam = e * nu / ((1 + nu) * (1 - 2 * nu));
    C.mu = e / (2 * (1 + nu));
    C.Kdr = e / (3 * (1 - 2 * nu));
    C.phi = phi[c]; C.s = sat[c]; C.p = pres[c];
    C.z = (c / ((int64_t)g.nx * g.ny) + 0.5) * g.h;
    C.rw = P.rho_w0 * (1 + P.c_w * (C.p - P.p0));
    C.rn = P.rho_nw0 * (1 + P.c_nw * (C.p - P.p0));
    C.drw = P.rho_w0 * P.c_w;
    C.drn = P.rho_nw0 * P.c_nw;
    const double span = 1.0 - P.swr - P.snwr;
    double se = (C.s - P.swr) / span, dse = 1.0 / span;
    if (se <= 0) { se = 0; dse = 0; }
    if (se >= 1) { se = 1; dse = 0; }
    C.krw = se * se; C.dkrw = 2 * se * dse;                  // Corey n = 2
    C.krn = (1 - se) * (1 - se); C.dkrn = -2 * (1 - se) * dse;
    C.dphi_dp = (b - (phi0 ? phi0[c] : C.phi)) * (1 - b) / C.Kdr;   // eq:linearized_porosity; d phi / d eps_v = b
    const double bracket = -P.rho_s + C.s * C.rw + (1 - C.s) * C.rn;
    C.drho_de = bracket * b;
    C.drho_ds = C.phi * (C.rw - C.rn);
    C.drho_dp = bracket * C.dphi_dp + C.s * C.phi * C.drw + (1 - C.s) * C.phi * C.drn;
    return C;
}

// ---------------------------------------------------------------- row lengths
__global__ void k_asm_counts(AsmGeo g, int32_t *cuu, int32_t *cuf, int32_t *cff)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int NX = g.nx + 1, NY = g.ny + 1;
    if (t < g.nn) {
        const int64_t n = g.node0 + t;
        const int i = n % NX, j = (n / NX) % NY, k = n / ((int64_t)NX * NY);
        const int ex = (i > 0) + (i < g.nx), ey = (j > 0) + (j < g.ny), ez = (k > 0) + (k < g.nz);
        cuu[t] = (1 + ex) * (1 + ey) * (1 + ez);
        cuf[t] = ex * ey * ez;
    }
    if (t < g.ncl) {
        const int64_t c = g.cell0 + t;
        const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / ((int64_t)g.nx * g.ny);
        cff[t] = 1 + (i > 0) + (i < g.nx - 1) + (j > 0) + (j < g.ny - 1) + (k > 0) + (k < g.nz - 1);
    }
}

// ---------------------------------------------------------------- node rows: A_uu, A_uf
// One thread per node row.  The row's <= 8 elements are summarised first (Lame constants, g d(rho)/d(eps_v), the
// node's local index a); then each of the <= 27 blocks is summed in registers over the elements shared with that
// neighbour, in ascending element order, and written once (no read-modify-write of global memory).
__global__ void __launch_bounds__(128) k_asm_node(tsp_asm_params P, AsmGeo g, const Q1 *q,
                                                  const double *__restrict__ E, const double *__restrict__ phi,
                                                  const double *__restrict__ sat, const double *__restrict__ pres,
                                                  const double *__restrict__ phi0,
                                                  const int32_t *__restrict__ rpu, int32_t *__restrict__ cu, double *__restrict__ vu,
                                                  const int32_t *__restrict__ rpf, int32_t *__restrict__ cf, double *__restrict__ vf,
                                                  unsigned long long *mx)
{
    __shared__ Q1 qs;                                   // the Gauss tables, read ~4500 times per row
    for (int e = threadIdx.x; e < (int)(sizeof(Q1) / sizeof(double)); e += blockDim.x)
        ((double *)&qs)[e] = ((const double *)q)[e];
    __syncthreads();
    q = &qs;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double rowmax = 0.0;                                // max over d of the row's l1 norm (R-scale), fused
    if (t < g.nn) {
    const int NX = g.nx + 1, NY = g.ny + 1;
    const int64_t n = g.node0 + t;
    const int i = n % NX, j = (n / NX) % NY, k = n / ((int64_t)NX * NY);
    const double gr = P.gravity, b = P.biot;
    // the adjacent elements o = (i-1+ox, j-1+oy, k-1+oz): presence, Lame constants, g d(rho)/d(eps_v); A_uf entries
    double lam[8], mu[8], gde[8];
    unsigned present = 0;
    int64_t qf = rpf[t];
    for (int o = 0; o < 8; ++o) {
        const int ci = i - 1 + (o & 1), cj = j - 1 + ((o >> 1) & 1), ck = k - 1 + ((o >> 2) & 1);
        lam[o] = mu[o] = gde[o] = 0.0;
        if (ci < 0 || ci >= g.nx || cj < 0 || cj >= g.ny || ck < 0 || ck >= g.nz) continue;
        present |= 1u << o;
        const int64_t c = ci + (int64_t)g.nx * (cj + (int64_t)g.ny * ck);
        const CellSt C = cell_st(P, g, c, E, phi, sat, pres, phi0);
        lam[o] = C.lam; mu[o] = C.mu; gde[o] = gr * C.drho_de;
        const int a = (1 - (o & 1)) + 2 * (1 - ((o >> 1) & 1)) + 4 * (1 - ((o >> 2) & 1));   // node n inside element o
        cf[qf] = (int32_t)c;
        double *F = vf + 6 * qf;
        for (int d = 0; d < 3; ++d) {
            F[2 * d] = d == 2 ? gr * C.drho_ds * q->NI[a] : 0.0;
            F[2 * d + 1] = (-b * q->DN[a][d] + (d == 2 ? gr * C.drho_dp * q->NI[a] : 0.0)) * P.p_unit;
        }
        ++qf;
    }
    // the clipped 27 neighbours m = n + (dx, dy, dz), ascending id; block (n, m) sums the elements holding both
    int64_t qu = rpu[t];
    double rs[3] = {0.0, 0.0, 0.0};
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int ii = i + dx, jj = j + dy, kk = k + dz;
                if (ii < 0 || ii > g.nx || jj < 0 || jj > g.ny || kk < 0 || kk > g.nz) continue;
                double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
                for (int o = 0; o < 8; ++o) {
                    if (!((present >> o) & 1u)) continue;
                    // element o spans nodes i-1+ox .. i+ox (per axis): it holds m iff each offset lies in its span
                    const int ox = o & 1, oy = (o >> 1) & 1, oz = (o >> 2) & 1;
                    const int bx = dx + 1 - ox, by = dy + 1 - oy, bz = dz + 1 - oz;   // m's local coordinates
                    if (bx < 0 || bx > 1 || by < 0 || by > 1 || bz < 0 || bz > 1) continue;
                    const int a = (1 - ox) + 2 * (1 - oy) + 4 * (1 - oz), bl = bx + 2 * by + 4 * bz;
                    const double tr = q->KK[a][bl][0][0] + q->KK[a][bl][1][1] + q->KK[a][bl][2][2];
                    for (int d = 0; d < 3; ++d)
                        for (int e = 0; e < 3; ++e) {
                            double v = lam[o] * q->KK[a][bl][d][e] + mu[o] * q->KK[a][bl][e][d];
                            if (d == e) v += mu[o] * tr;
                            if (d == 2) v += gde[o] * q->NB[a][bl][e];
                            B[3 * d + e] += v;
                        }
                }
                cu[qu] = (int32_t)(ii + (int64_t)NX * (jj + (int64_t)NY * kk));
                for (int e = 0; e < 9; ++e) vu[9 * qu + e] = B[e];
                for (int d = 0; d < 3; ++d)
                    for (int e = 0; e < 3; ++e) rs[d] += fabs(B[3 * d + e]);
                ++qu;
            }
    rowmax = fmax(rs[0], fmax(rs[1], rs[2]));
    }
    // values >= 0: their bit patterns order like the values; one atomic per warp
    for (int o = 16; o; o >>= 1) rowmax = fmax(rowmax, __shfl_xor_sync(0xffffffffu, rowmax, o));
    if ((threadIdx.x & 31) == 0 && rowmax > 0) atomicMax(mx, (unsigned long long)__double_as_longlong(rowmax));
}

__global__ void k_asm_fu_rowptr(int ncl, int32_t *rp)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c <= ncl) rp[c] = 8 * c;
}

// ---------------------------------------------------------------- cell rows: A_fu, A_ff, wells, D_fs
__global__ void __launch_bounds__(128) k_asm_cell(tsp_asm_params P, AsmGeo g, const Q1 *__restrict__ q,
                                                  const double *__restrict__ E, const double *__restrict__ perm,
                                                  const double *__restrict__ phi, const double *__restrict__ sat,
                                                  const double *__restrict__ pres, const int8_t *__restrict__ well,
                                                  const double *__restrict__ phi0, int32_t *__restrict__ cfu, double *__restrict__ vfu,
                                                  const int32_t *__restrict__ rpf, int32_t *__restrict__ cff, double *__restrict__ vff,
                                                  double *__restrict__ fs, unsigned long long *mx)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double ms = 0.0, mp = 0.0;                          // the row's l1 norms of A_ss and A_pp entries (R-scale), fused
    if (t < g.ncl) {
    const int NX = g.nx + 1, NY = g.ny + 1;
    const int64_t c = g.cell0 + t, P2 = (int64_t)g.nx * g.ny;
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / P2;
    const double h = g.h, V = h * h * h, gr = P.gravity, b = P.biot, dt = P.dt, pu = P.p_unit;
    const CellSt K = cell_st(P, g, c, E, phi, sat, pres, phi0);
    // A_fu: the 8 corner nodes of the cell
    for (int a = 0; a < 8; ++a) {
        const int64_t qq = 8 * (int64_t)t + a;
        cfu[qq] = (int32_t)((i + (a & 1)) + (int64_t)NX * ((j + ((a >> 1) & 1)) + (int64_t)NY * (k + ((a >> 2) & 1))));
        for (int d = 0; d < 3; ++d) {
            vfu[6 * qq + d] = K.s * K.rw * b * q->DN[a][d];
            vfu[6 * qq + 3 + d] = (1 - K.s) * K.rn * b * q->DN[a][d];
        }
    }
    // A_ff: 7-point pattern in ascending column order
    int64_t nb[7];
    int np = 0;
    if (k > 0) nb[np++] = c - P2;
    if (j > 0) nb[np++] = c - g.nx;
    if (i > 0) nb[np++] = c - 1;
    nb[np++] = c;
    if (i < g.nx - 1) nb[np++] = c + 1;
    if (j < g.ny - 1) nb[np++] = c + g.nx;
    if (k < g.nz - 1) nb[np++] = c + P2;
    const int64_t r0 = rpf[t];
    int dpos = 0;
    for (int u = 0; u < np; ++u) {
        cff[r0 + u] = (int32_t)nb[u];
        for (int e = 0; e < 4; ++e) vff[4 * (r0 + u) + e] = 0.0;
        if (nb[u] == c) dpos = u;
    }
    double *D = vff + 4 * (r0 + dpos);
    // accumulation: d(phi rho_alpha s_alpha V)/d(s, p)
    D[0] += V * K.phi * K.rw;
    D[1] += V * (K.s * K.rw * K.dphi_dp + K.phi * K.s * K.drw);
    D[2] += V * (-K.phi * K.rn);
    D[3] += V * ((1 - K.s) * K.rn * K.dphi_dp + K.phi * (1 - K.s) * K.drn);
    // faces
    for (int u = 0; u < np; ++u) {
        const int64_t o = nb[u];
        if (o == c) continue;
        const int64_t cK = c < o ? c : o, cL = c < o ? o : c;
        const CellSt A = (cK == c) ? K : cell_st(P, g, cK, E, phi, sat, pres, phi0);
        const CellSt B = (cL == c) ? K : cell_st(P, g, cL, E, phi, sat, pres, phi0);
        const double tK = h * h * perm[cK] * (h / 2) / ((h / 2) * (h / 2));     // eq:half_trans
        const double tL = h * h * perm[cL] * (h / 2) / ((h / 2) * (h / 2));
        const double T = (tK + tL) > 0 ? tK * tL / (tK + tL) : 0.0;           // eq:trans
        const double dz = B.z - A.z, sgn = (c == cK) ? -1.0 : 1.0;
        const int posK = (cK == c) ? dpos : u, posL = (cL == c) ? dpos : u;
        for (int ph = 0; ph < 2; ++ph) {
            const double rK = ph ? A.rn : A.rw, rL = ph ? B.rn : B.rw, dK = ph ? A.drn : A.drw, dL = ph ? B.drn : B.drw;
            const double krK = ph ? A.krn : A.krw, krL = ph ? B.krn : B.krw, dkK = ph ? A.dkrn : A.dkrw, dkL = ph ? B.dkrn : B.dkrw;
            const double mu = ph ? P.mu_nw : P.mu_w;
            const bool inK = krK > 0, inL = krL > 0;
            double vr = 0, dvK = 0, dvL = 0;                          // eq:avg_density over the phases present
            if (inK && inL) { vr = 0.5 * (rK + rL); dvK = 0.5 * dK; dvL = 0.5 * dL; }
            else if (inK) { vr = rK; dvK = dK; }
            else if (inL) { vr = rL; dvL = dL; }
            const double Phi = T * ((B.p - A.p) + vr * gr * dz);
            const bool upL = Phi > 0;                                  // ties upstream = K
            const double rup = upL ? rL : rK, drup = upL ? dL : dK, lup = (upL ? krL : krK) / mu, dkup = upL ? dkL : dkK;
            const double dFds = rup / mu * Phi * dkup;
            const double dFdpK = (upL ? 0.0 : drup * lup) * Phi + rup * lup * T * (-1.0 + dvK * gr * dz);
            const double dFdpL = (upL ? drup * lup : 0.0) * Phi + rup * lup * T * (1.0 + dvL * gr * dz);
            const double cf = sgn * dt;
            vff[4 * (r0 + (upL ? posL : posK)) + 2 * ph] += cf * dFds;
            vff[4 * (r0 + posK) + 2 * ph + 1] += cf * dFdpK;
            vff[4 * (r0 + posL) + 2 * ph + 1] += cf * dFdpL;
        }
    }
    // Peaceman wells: water injector at BHP + dbhp, producers at BHP - dbhp (per-cell perforation flags)
    const int wt = well ? well[c] : 0;
    if (wt) {
        const int kw1 = P.burden > 0 ? g.nz - P.burden : g.nz;
        const double zbh = (kw1 - 0.5) * h, ztop = g.nz * h;
        const double pbh = P.p0 + P.rho_w0 * gr * (ztop - zbh) + (wt == 1 ? P.well_dbhp : -P.well_dbhp);
        const double re = 0.28 * sqrt(h * h + h * h) / 2.0;
        const double WI = 2 * M_PI * h * perm[c] / log(re / (P.rw_over_h * h));
        const double lw = K.krw / P.mu_w, ln = K.krn / P.mu_nw;
        for (int ph = 0; ph < 2; ++ph) {
            const double r = ph ? K.rn : K.rw, dr = ph ? K.drn : K.drw;
            const double Phi = WI * ((pbh + r * gr * zbh) - (K.p + r * gr * K.z));
            const double dPhi = WI * (-1.0 + dr * gr * (zbh - K.z));
            double dqs = 0, dqp = 0;
            if (wt == 1) {
                if (ph == 0 && Phi > 0) {                              // water-only injection with the total mobility
                    dqs = r * (K.dkrw / P.mu_w + K.dkrn / P.mu_nw) * Phi;
                    dqp = dr * (lw + ln) * Phi + r * (lw + ln) * dPhi;
                }
            } else if (Phi < 0) {                                      // production of each phase
                const double l = ph ? ln : lw, dk = ph ? K.dkrn : K.dkrw, mu = ph ? P.mu_nw : P.mu_w;
                dqs = r * dk / mu * Phi;
                dqp = dr * l * Phi + r * l * dPhi;
            }
            D[2 * ph] += -dt * dqs;
            D[2 * ph + 1] += -dt * dqp;
        }
    }
    // pressure unit on the p columns (R-punit)
    for (int u = 0; u < np; ++u) { vff[4 * (r0 + u) + 1] *= pu; vff[4 * (r0 + u) + 3] *= pu; }
    // fixed-stress diagonals (eq:FS_Dps_Dpp), in p-column units
    fs[2 * t] = V * b * b / K.Kdr * K.s * K.rw * pu;
    fs[2 * t + 1] = V * b * b / K.Kdr * (1 - K.s) * K.rn * pu;
    for (int u = 0; u < np; ++u) { ms += fabs(vff[4 * (r0 + u)]); mp += fabs(vff[4 * (r0 + u) + 3]); }
    }
    for (int o = 16; o; o >>= 1) {
        ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
        mp = fmax(mp, __shfl_xor_sync(0xffffffffu, mp, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (ms > 0) atomicMax(mx + 1, (unsigned long long)__double_as_longlong(ms));
        if (mp > 0) atomicMax(mx + 2, (unsigned long long)__double_as_longlong(mp));
    }
}

// ---------------------------------------------------------------- scaling + Dirichlet rows (R-scale, R-dirichlet)
// elementwise over the value arrays (coalesced); `qfix`: the entries of the rank's fixed (bottom) rows, [0, rp[nfix])
__global__ void k_scale_uu(int64_t nv, double su, int dirichlet, int64_t nbot, const int32_t *__restrict__ rpu, int nfix,
                           const int32_t *__restrict__ cu, double *__restrict__ vu)
{
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= nv) return;
    const int64_t q = idx / 9;
    const bool fixed = dirichlet && (q < rpu[nfix] || cu[q] < nbot);
    vu[idx] = fixed ? 0.0 : vu[idx] * su;
}
__global__ void k_fix_diag(int nfix, int64_t node0, const int32_t *__restrict__ rpu, const int32_t *__restrict__ cu, double *__restrict__ vu)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nfix) return;
    for (int64_t q = rpu[t]; q < rpu[t + 1]; ++q)
        if (cu[q] == node0 + t) { vu[9 * q] = 1.0; vu[9 * q + 4] = 1.0; vu[9 * q + 8] = 1.0; }
}
__global__ void k_scale_uf(int64_t nv, double su, const int32_t *__restrict__ rpf, int nfix, double *__restrict__ vf)
{
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= nv) return;
    vf[idx] = idx / 6 < rpf[nfix] ? 0.0 : vf[idx] * su;
}
__global__ void k_scale_fu(int64_t nv, double ss, double sp, int dirichlet, int64_t nbot, const int32_t *__restrict__ cfu,
                           double *__restrict__ v)
{
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= nv) return;
    const int64_t q = idx / 6;
    v[idx] = (dirichlet && cfu[q] < nbot) ? 0.0 : v[idx] * ((idx % 6) < 3 ? ss : sp);
}
__global__ void k_scale_ff(int64_t nv, double ss, double sp, double *__restrict__ v, int64_t nfs, double *__restrict__ fs)
{
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx < nv) v[idx] *= (idx & 3) < 2 ? ss : sp;
    if (idx < nfs) fs[idx] *= (idx & 1) ? sp : ss;
}

// ---------------------------------------------------------------- residual of Appendix B.1, raw units
// x = [u node-major | (s, p [Pa]) per cell]; porosity phi = phi_0 + b eps_v + (b - phi_0)(1 - b)/K_dr (p - p_ref)
// with eps_v the cell average (eq:linearized_porosity); the gravity term integrates the mixture density pointwise
// (its porosity carries the Gauss point's eps_v).  Its CPU reference is residual.c of the test oracle.
struct ResSt {
    double lam, mu, Kdr, s, p, z, phi, phi_e0, rw, rn, krw, krn;
};
__device__ __forceinline__ int64_t cell_node(const AsmGeo &g, int64_t c, int a)
{
    const int64_t NX = g.nx + 1, NY = g.ny + 1;
    const int64_t i = c % g.nx, j = (c / g.nx) % g.ny, k = c / ((int64_t)g.nx * g.ny);
    return (i + (a & 1)) + NX * ((j + ((a >> 1) & 1)) + NY * (k + ((a >> 2) & 1)));
}
__device__ ResSt res_st(const tsp_asm_params &P, const AsmGeo &g, const Q1 *__restrict__ q, int64_t c, const double *__restrict__ E,
                        const double *__restrict__ phi0, const double *__restrict__ pref, const double *__restrict__ x,
                        int64_t Nn, bool strain)
{
    ResSt C;
    const double nu = P.nu, b = P.biot, V = g.h * g.h * g.h;
    C.lam = E[c] * nu / ((1 + nu) * (1 - 2 * nu));
    C.mu = E[c] / (2 * (1 + nu));
    C.Kdr = E[c] / (3 * (1 - 2 * nu));
    C.s = x[3 * Nn + 2 * c];
    C.p = x[3 * Nn + 2 * c + 1];
    C.z = (c / ((int64_t)g.nx * g.ny) + 0.5) * g.h;
    double ev = 0.0;
    if (strain)
        for (int a = 0; a < 8; ++a) {
            const int64_t n = cell_node(g, c, a);
            for (int d = 0; d < 3; ++d) ev += q->DN[a][d] * x[3 * n + d];
        }
    C.phi_e0 = phi0[c] + (b - phi0[c]) * (1 - b) / C.Kdr * (C.p - pref[c]);
    C.phi = C.phi_e0 + b * ev / V;
    C.rw = P.rho_w0 * (1 + P.c_w * (C.p - P.p0));
    C.rn = P.rho_nw0 * (1 + P.c_nw * (C.p - P.p0));
    const double span = 1.0 - P.swr - P.snwr;
    double se = (C.s - P.swr) / span;
    se = se < 0 ? 0 : se > 1 ? 1 : se;
    C.krw = se * se;
    C.krn = (1 - se) * (1 - se);
    return C;
}

// x: the GLOBAL state (NnG nodes); r: this rank's rows [u_own | f_own] (g.nn, g.ncl)
__global__ void __launch_bounds__(128) k_res_node(tsp_asm_params P, AsmGeo g, const Q1 *__restrict__ q, const double *__restrict__ E,
                                                  const double *__restrict__ phi0, const double *__restrict__ pref,
                                                  const double *__restrict__ x, int64_t Nn, double *__restrict__ r)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.nn) return;
    const int NX = g.nx + 1, NY = g.ny + 1;
    const int64_t n = g.node0 + t;
    const int i = n % NX, j = (n / NX) % NY, k = n / ((int64_t)NX * NY);
    const double gr = P.gravity, b = P.biot;
    double R[3] = {0.0, 0.0, 0.0};
    if (!(P.dirichlet_bottom && n < (int64_t)NX * NY))
        for (int o = 0; o < 8; ++o) {
            const int ci = i - 1 + (o & 1), cj = j - 1 + ((o >> 1) & 1), ck = k - 1 + ((o >> 2) & 1);
            if (ci < 0 || ci >= g.nx || cj < 0 || cj >= g.ny || ck < 0 || ck >= g.nz) continue;
            const int64_t c = ci + (int64_t)g.nx * (cj + (int64_t)g.ny * ck);
            const ResSt C = res_st(P, g, q, c, E, phi0, pref, x, Nn, false);
            const double bracket = -P.rho_s + C.s * C.rw + (1 - C.s) * C.rn;
            const double rho0 = P.rho_s + C.phi_e0 * bracket;
            const int a = (1 - (o & 1)) + 2 * (1 - ((o >> 1) & 1)) + 4 * (1 - ((o >> 2) & 1));
            double u[8][3];
            for (int bb = 0; bb < 8; ++bb) {
                const int64_t m = cell_node(g, c, bb);
                for (int e = 0; e < 3; ++e) u[bb][e] = x[3 * m + e];
            }
            for (int d = 0; d < 3; ++d) {
                double v = 0.0;
                for (int bb = 0; bb < 8; ++bb) {
                    const double tr = q->KK[a][bb][0][0] + q->KK[a][bb][1][1] + q->KK[a][bb][2][2];
                    for (int e = 0; e < 3; ++e) {
                        double kk = C.lam * q->KK[a][bb][d][e] + C.mu * q->KK[a][bb][e][d];
                        if (d == e) kk += C.mu * tr;
                        v += kk * u[bb][e];
                        if (d == 2) v += gr * bracket * b * q->NB[a][bb][e] * u[bb][e];
                    }
                }
                v -= b * C.p * q->DN[a][d];
                if (d == 2) v += gr * rho0 * q->NI[a];
                R[d] += v;
            }
        }
    for (int d = 0; d < 3; ++d) r[3 * (int64_t)t + d] = R[d];
}

__global__ void __launch_bounds__(128) k_res_cell(tsp_asm_params P, AsmGeo g, const Q1 *__restrict__ q, const double *__restrict__ E,
                                                  const double *__restrict__ perm, const double *__restrict__ phi0,
                                                  const double *__restrict__ pref, const int8_t *__restrict__ well,
                                                  const double *__restrict__ x, int64_t Nn, const double *__restrict__ mprev,
                                                  double dt, double *__restrict__ r)
{
    // mprev: this rank's cells; r: this rank's rows (the cell part starts after its 3 g.nn node rows)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.ncl) return;
    const int64_t c = g.cell0 + t, P2 = (int64_t)g.nx * g.ny;
    const int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / P2;
    const double h = g.h, V = h * h * h, gr = P.gravity;
    const ResSt K = res_st(P, g, q, c, E, phi0, pref, x, Nn, true);
    double rw = V * K.phi * K.rw * K.s - mprev[2 * t];
    double rn = V * K.phi * K.rn * (1 - K.s) - mprev[2 * t + 1];
    int64_t nb[6];
    int np = 0;
    if (k > 0) nb[np++] = c - P2;
    if (j > 0) nb[np++] = c - g.nx;
    if (i > 0) nb[np++] = c - 1;
    if (i < g.nx - 1) nb[np++] = c + 1;
    if (j < g.ny - 1) nb[np++] = c + g.nx;
    if (k < g.nz - 1) nb[np++] = c + P2;
    for (int u = 0; u < np; ++u) {
        const int64_t o = nb[u], cK = c < o ? c : o, cL = c < o ? o : c;
        const ResSt O = res_st(P, g, q, o, E, phi0, pref, x, Nn, false);
        const ResSt &A = (cK == c) ? K : O, &B = (cL == c) ? K : O;
        const double tK = h * h * perm[cK] * (h / 2) / ((h / 2) * (h / 2)), tL = h * h * perm[cL] * (h / 2) / ((h / 2) * (h / 2));
        const double T = (tK + tL) > 0 ? tK * tL / (tK + tL) : 0.0;
        const double dz = B.z - A.z, sgn = (c == cK) ? -1.0 : 1.0;
        for (int ph = 0; ph < 2; ++ph) {
            const double rK = ph ? A.rn : A.rw, rL = ph ? B.rn : B.rw, kK = ph ? A.krn : A.krw, kL = ph ? B.krn : B.krw;
            const double mu = ph ? P.mu_nw : P.mu_w;
            const double ravg = (kK > 0 && kL > 0) ? 0.5 * (rK + rL) : kK > 0 ? rK : kL > 0 ? rL : 0.0;
            const double Phi = T * ((B.p - A.p) + ravg * gr * dz);
            const bool fromL = Phi > 0;
            const double F = (fromL ? rL : rK) * (fromL ? kL : kK) / mu * Phi;
            (ph ? rn : rw) += sgn * dt * F;
        }
    }
    const int wt = well ? well[c] : 0;
    if (wt) {
        const int kw1 = P.burden > 0 ? g.nz - P.burden : g.nz;
        const double zbh = (kw1 - 0.5) * h, ztop = g.nz * h;
        const double pbh = P.p0 + P.rho_w0 * gr * (ztop - zbh) + (wt == 1 ? P.well_dbhp : -P.well_dbhp);
        const double re = 0.28 * sqrt(h * h + h * h) / 2.0;
        const double WI = 2 * M_PI * h * perm[c] / log(re / (P.rw_over_h * h));
        const double lw = K.krw / P.mu_w, ln = K.krn / P.mu_nw;
        for (int ph = 0; ph < 2; ++ph) {
            const double rr = ph ? K.rn : K.rw;
            const double Phi = WI * ((pbh + rr * gr * zbh) - (K.p + rr * gr * K.z));
            double src = 0.0;
            if (wt == 1) { if (ph == 0 && Phi > 0) src = rr * (lw + ln) * Phi; }
            else if (Phi < 0) src = rr * (ph ? ln : lw) * Phi;
            (ph ? rn : rw) -= dt * src;
        }
    }
    r[3 * (int64_t)g.nn + 2 * (int64_t)t] = rw;
    r[3 * (int64_t)g.nn + 2 * (int64_t)t + 1] = rn;
}

// current porosity, saturation and pressure of every cell at x (the fields of the Jacobian at the state)
__global__ void k_state_fields(tsp_asm_params P, AsmGeo g, const Q1 *__restrict__ q, const double *__restrict__ E,
                               const double *__restrict__ phi0, const double *__restrict__ pref, const double *__restrict__ x,
                               int64_t Nn, double *__restrict__ phi, double *__restrict__ sat, double *__restrict__ pres)
{
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)g.nx * g.ny * g.nz) return;
    const ResSt C = res_st(P, g, q, c, E, phi0, pref, x, Nn, true);
    phi[c] = C.phi; sat[c] = C.s; pres[c] = C.p;
}
__global__ void k_masses(tsp_asm_params P, AsmGeo g, const Q1 *__restrict__ q, const double *__restrict__ E,
                         const double *__restrict__ phi0, const double *__restrict__ pref, const double *__restrict__ x,
                         int64_t Nn, double *__restrict__ m)
{
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)g.nx * g.ny * g.nz) return;
    const ResSt C = res_st(P, g, q, c, E, phi0, pref, x, Nn, true);
    const double V = g.h * g.h * g.h;
    m[2 * c] = V * C.phi * C.rw * C.s;
    m[2 * c + 1] = V * C.phi * C.rn * (1 - C.s);
}

static AsmGeo asm_geo(const tsp_asm_params &P, int rank, int nranks, int zblock);

struct Q1Dev {
    DBuf<Q1> q;
    explicit Q1Dev(cudaStream_t s, double h)
    {
        Q1 t;
        q1_tables(h, t);
        q.alloc(1);
        TSP_CUDA(cudaMemcpyAsync(q.p, &t, sizeof(Q1), cudaMemcpyHostToDevice, s));
        TSP_CUDA(cudaStreamSynchronize(s));
    }
};

void residual(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, double dt, const double *x, const double *mprev,
              double *r, int rank, int nranks, int zblock)
{
    TSP_REQUIRE(ref.E && ref.perm && ref.phi && ref.pres && x && mprev && r, TSP_ERR_INVALID_ARG, "residual: null pointer");
    const AsmGeo g = asm_geo(P, rank, nranks, zblock);
    Q1Dev q(s, g.h);
    const int64_t Nn = (int64_t)(P.nx + 1) * (P.ny + 1) * (P.nz + 1);   // x is the global state
    if (g.nn) k_res_node<<<grid_for(g.nn, 128), 128, 0, s>>>(P, g, q.q.p, ref.E, ref.phi, ref.pres, x, Nn, r);
    if (g.ncl) k_res_cell<<<grid_for(g.ncl, 128), 128, 0, s>>>(P, g, q.q.p, ref.E, ref.perm, ref.phi, ref.pres, ref.well, x, Nn,
                                                              mprev, dt, r);
    TSP_CUDA(cudaGetLastError());
}
void state_fields(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *x, double *phi, double *sat,
                  double *pres)
{
    const AsmGeo g = asm_geo(P, 0, 1, 16);
    Q1Dev q(s, g.h);
    if (g.ncl) k_state_fields<<<grid_for(g.ncl, 128), 128, 0, s>>>(P, g, q.q.p, ref.E, ref.phi, ref.pres, x, g.nn, phi, sat, pres);
    TSP_CUDA(cudaGetLastError());
}
void masses(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *x, double *m)
{
    const AsmGeo g = asm_geo(P, 0, 1, 16);
    Q1Dev q(s, g.h);
    if (g.ncl) k_masses<<<grid_for(g.ncl, 128), 128, 0, s>>>(P, g, q.q.p, ref.E, ref.phi, ref.pres, x, g.nn, m);
    TSP_CUDA(cudaGetLastError());
}
// this rank's cells of a global per-cell array pair (V m_w, V m_nw)
void masses_local(cudaStream_t s, const tsp_asm_params &P, const tsp_cell_fields &ref, const double *xg, double *m_local, int rank,
                  int nranks, int zblock)
{
    const AsmGeo gl = asm_geo(P, rank, nranks, zblock);
    DBuf<double> mg; mg.alloc((size_t)std::max<int64_t>(2 * (int64_t)P.nx * P.ny * P.nz, 1));
    masses(s, P, ref, xg, mg);
    if (gl.ncl) TSP_CUDA(cudaMemcpyAsync(m_local, mg.p + 2 * gl.cell0, sizeof(double) * 2 * gl.ncl, cudaMemcpyDeviceToDevice, s));
}

static AsmGeo asm_geo(const tsp_asm_params &P, int rank, int nranks, int zblock)
{
    int64_t part[6];
    partition(P.nx, P.ny, P.nz, zblock > 0 ? zblock : 16, rank, nranks, part);
    AsmGeo g;
    g.nx = P.nx; g.ny = P.ny; g.nz = P.nz;
    g.node0 = part[2]; g.nn = (int)part[3]; g.cell0 = part[4]; g.ncl = (int)part[5];
    g.h = (P.length > 0 ? P.length : 1.0) / P.nx;
    return g;
}

// block counts of this rank's rows: the per-node and per-cell counts factor over the axes, so the sums do too
void assembly_sizes(const tsp_asm_params &P, int rank, int nranks, int zblock, int64_t out[6])
{
    const AsmGeo g = asm_geo(P, rank, nranks, zblock);
    const int NX = P.nx + 1, NY = P.ny + 1;
    auto e1 = [](int i, int n) { return (int64_t)((i > 0) + (i < n)); };          // adjacent cells along an axis
    int64_t sx1 = 0, sx0 = 0, sy1 = 0, sy0 = 0, sz1 = 0, sz0 = 0;
    for (int i = 0; i < NX; ++i) { sx1 += 1 + e1(i, P.nx); sx0 += e1(i, P.nx); }
    for (int j = 0; j < NY; ++j) { sy1 += 1 + e1(j, P.ny); sy0 += e1(j, P.ny); }
    const int64_t kn0 = g.node0 / ((int64_t)NX * NY), kn1 = kn0 + g.nn / ((int64_t)NX * NY);
    for (int64_t k = kn0; k < kn1; ++k) { sz1 += 1 + e1((int)k, P.nz); sz0 += e1((int)k, P.nz); }
    const int64_t buu = sx1 * sy1 * sz1, buf = sx0 * sy0 * sz0;
    // cells: 1 + neighbours along x, y, z
    const int64_t P2 = (int64_t)P.nx * P.ny, kc0 = g.cell0 / P2, nzl = g.ncl / P2;
    auto nb = [](int64_t i, int64_t n) { return (int64_t)((i > 0) + (i < n - 1)); };
    int64_t fx = 0, fy = 0, fz = 0;
    for (int i = 0; i < P.nx; ++i) fx += nb(i, P.nx);
    for (int j = 0; j < P.ny; ++j) fy += nb(j, P.ny);
    for (int64_t k = kc0; k < kc0 + nzl; ++k) fz += nb(k, P.nz);
    const int64_t bff = g.ncl + fx * P.ny * nzl + fy * P.nx * nzl + fz * P2;
    out[0] = g.nn; out[1] = g.ncl; out[2] = buu; out[3] = buf; out[4] = 8 * (int64_t)g.ncl; out[5] = bff;
}

void assemble(cudaStream_t s, const tsp_asm_params &P, int rank, int nranks, int zblock, const tsp_cell_fields &f,
              tsp_bsr_out blk[4], double *fs, double row_max[3])
{
    TSP_REQUIRE(P.nx > 0 && P.ny > 0 && P.nz > 0, TSP_ERR_INVALID_ARG, "assemble: grid dimensions must be positive");
    TSP_REQUIRE(f.E && f.perm && f.phi && f.sat && f.pres, TSP_ERR_INVALID_ARG, "assemble: null field");
    for (int k = 0; k < 4; ++k)
        TSP_REQUIRE(blk[k].rowptr && blk[k].col && blk[k].val, TSP_ERR_INVALID_ARG, "assemble: null output block");
    TSP_REQUIRE(fs, TSP_ERR_INVALID_ARG, "assemble: null fs");
    const AsmGeo g = asm_geo(P, rank, nranks, zblock);
    Q1 q;
    q1_tables(g.h, q);
    DBuf<Q1> dq; dq.alloc(1);
    DBuf<int32_t> cnt; cnt.alloc((size_t)3 * (std::max(g.nn, g.ncl) + 1));
    int32_t *cuu = cnt.p, *cuf = cnt.p + std::max(g.nn, g.ncl) + 1, *cff = cuf + std::max(g.nn, g.ncl) + 1;
    TSP_CUDA(cudaMemcpyAsync(dq.p, &q, sizeof(Q1), cudaMemcpyHostToDevice, s));
    const int m = std::max(g.nn, g.ncl);
    if (m) k_asm_counts<<<grid_for(m, 256), 256, 0, s>>>(g, cuu, cuf, cff);
    auto scan = [&](int32_t *c, int len, int32_t *rp) {
        TSP_CUDA(cudaMemsetAsync(c + len, 0, sizeof(int32_t), s));
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, c, rp, len + 1, s);
        DBuf<uint8_t> tmp; tmp.alloc(std::max<size_t>(tb, 1));
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, c, rp, len + 1, s);
    };
    scan(cuu, g.nn, blk[0].rowptr);
    scan(cuf, g.nn, blk[1].rowptr);
    scan(cff, g.ncl, blk[3].rowptr);
    k_asm_fu_rowptr<<<grid_for(g.ncl + 1, 256), 256, 0, s>>>(g.ncl, blk[2].rowptr);   // A_fu: 8 nodes per cell
    DBuf<unsigned long long> mx; mx.alloc(3); mx.zero(s);
    if (g.nn) k_asm_node<<<grid_for(g.nn, 128), 128, 0, s>>>(P, g, dq.p, f.E, f.phi, f.sat, f.pres, f.phi0, blk[0].rowptr, blk[0].col,
                                                            blk[0].val, blk[1].rowptr, blk[1].col, blk[1].val, mx.p);
    if (g.ncl) k_asm_cell<<<grid_for(g.ncl, 128), 128, 0, s>>>(P, g, dq.p, f.E, f.perm, f.phi, f.sat, f.pres, f.well, f.phi0, blk[2].col,
                                                              blk[2].val, blk[3].rowptr, blk[3].col, blk[3].val, fs, mx.p);
    TSP_CUDA(cudaGetLastError());
    unsigned long long hb[3];
    TSP_CUDA(cudaMemcpyAsync(hb, mx.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    TSP_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < 3; ++k) memcpy(&row_max[k], &hb[k], sizeof(double));
}

void assemble_scale(cudaStream_t s, const tsp_asm_params &P, int rank, int nranks, int zblock, const double row_max[3],
                    tsp_bsr_out blk[4], double *fs, double scales[3])
{
    const AsmGeo g = asm_geo(P, rank, nranks, zblock);
    double sc[3] = {1.0, 1.0, 1.0};
    if (P.row_scale)
        for (int k = 0; k < 3; ++k) sc[k] = row_max[k] > 0 ? 1.0 / row_max[k] : 1.0;
    int64_t sz[6];
    assembly_sizes(P, rank, nranks, zblock, sz);
    const int64_t nbot = (int64_t)(P.nx + 1) * (P.ny + 1);
    const int nfix = P.dirichlet_bottom ? (int)std::max<int64_t>(0, std::min<int64_t>(nbot - g.node0, g.nn)) : 0;
    const int64_t vuu = 9 * sz[2], vuf = 6 * sz[3], vfu = 6 * sz[4], vff = 4 * sz[5], nfs = 2 * (int64_t)g.ncl;
    if (vuu) k_scale_uu<<<grid_for(vuu, 256), 256, 0, s>>>(vuu, sc[0], P.dirichlet_bottom, nbot, blk[0].rowptr, nfix, blk[0].col, blk[0].val);
    if (nfix) k_fix_diag<<<grid_for(nfix, 128), 128, 0, s>>>(nfix, g.node0, blk[0].rowptr, blk[0].col, blk[0].val);
    if (vuf) k_scale_uf<<<grid_for(vuf, 256), 256, 0, s>>>(vuf, sc[0], blk[1].rowptr, nfix, blk[1].val);
    if (vfu) k_scale_fu<<<grid_for(vfu, 256), 256, 0, s>>>(vfu, sc[1], sc[2], P.dirichlet_bottom, nbot, blk[2].col, blk[2].val);
    if (std::max(vff, nfs)) k_scale_ff<<<grid_for(std::max(vff, nfs), 256), 256, 0, s>>>(vff, sc[1], sc[2], blk[3].val, nfs, fs);
    TSP_CUDA(cudaGetLastError());
    TSP_CUDA(cudaStreamSynchronize(s));
    if (scales) for (int k = 0; k < 3; ++k) scales[k] = sc[k];
}

}  // namespace tsp

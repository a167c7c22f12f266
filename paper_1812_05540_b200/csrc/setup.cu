// setup.cu -- rows a1-a3 on the GPU and the MECH / FLOW setup phases of P:519,
// P:638 (mechanics once per simulation, flow per Newton step).
#include "tsp_internal.cuh"

namespace tsp {

// a2: SDC: keep the (x,x), (y,y), (z,z) entries of every 3x3 block (run by tsp_create)
__global__ void k_sdc(int64_t nnzb, const double *__restrict__ uu, double *__restrict__ sdc)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnzb) return;
    sdc[3 * q + 0] = uu[9 * q + 0];
    sdc[3 * q + 1] = uu[9 * q + 4];
    sdc[3 * q + 2] = uu[9 * q + 8];
}

// z-block of every owned row; k0 = first owned cell plane (global)
__global__ void k_zb_nodes(int Nn, int nx, int ny, int nz_glob, int k0, int zblock, int32_t *zb)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nn) return;
    int k = k0 + i / ((nx + 1) * (ny + 1));
    int kc = k < nz_glob ? k : nz_glob - 1;        // node plane k belongs to cell plane min(k, nz-1) (R-zblock)
    zb[i] = kc / zblock;
}
__global__ void k_zb_cells(int Nc, int nx, int ny, int k0, int zblock, int32_t *zb)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < Nc) zb[i] = (k0 + i / (nx * ny)) / zblock;
}

// a3 diagonals D_ss^(CPR), D_ps^(CPR) (`ci` local ids: the diagonal of row i is column i; ghosts >= Nc)
//   mode 0 quasi-IMPES: entries (0,0) and (1,0) of the diagonal block;
//   mode 1 true-IMPES (eq:CPR_CSL): column sums over the rows k of column i, in the order of
//   row i's columns (the pattern is structurally symmetric); A[k][i] of a ghost row k comes from the
//   neighbour rank: `gh_up` (ghost below: its coupling to the plane above) / `gh_dn` (ghost above).
__global__ void k_cpr_diag(int Nc, int mode, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const double *__restrict__ gh_up, const double *__restrict__ gh_dn,
                           int nlo, double *__restrict__ dss, double *__restrict__ dps)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc) return;
    double ss = 0.0, ps = 0.0;
    if (mode == 0) {
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
            if (ci[q] == i) { ss = v[q * 4 + 0]; ps = v[q * 4 + 2]; break; }
    } else {
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
            const int k = ci[q];
            double a = 0.0, b = 0.0;
            if (k < Nc) {
                for (int64_t p = rp[k]; p < rp[k + 1]; ++p)
                    if (ci[p] == i) { a = v[p * 4 + 0]; b = v[p * 4 + 2]; break; }
            } else {
                const int g = k - Nc;
                const double *src = g < nlo ? gh_up : gh_dn;
                a = src[2 * g]; b = src[2 * g + 1];
            }
            ss = __dadd_rn(ss, a);
            ps = __dadd_rn(ps, b);
        }
    }
    dss[i] = ss;
    dps[i] = ps;
}
// multi-GPU true-IMPES: (A_ss, A_ps)[k][k +- P] of every owned row k (P = cells per plane), by global column
__global__ void k_zcouple(int Nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ gci, const double *__restrict__ v,
                          int64_t cell_off, int64_t P, double *__restrict__ up, double *__restrict__ dn)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= Nc) return;
    const int64_t K = cell_off + k;
    double u0 = 0, u1 = 0, d0 = 0, d1 = 0;
    for (int64_t q = rp[k]; q < rp[k + 1]; ++q) {
        if (gci[q] == K + P) { u0 = v[q * 4 + 0]; u1 = v[q * 4 + 2]; }
        if (gci[q] == K - P) { d0 = v[q * 4 + 0]; d1 = v[q * 4 + 2]; }
    }
    up[2 * k] = u0; up[2 * k + 1] = u1;
    dn[2 * k] = d0; dn[2 * k + 1] = d1;
}

// a1 + a3: fixed stress (eq:Schur_1_FS) and the CPR reduction:
//   A_sp^FS = A_sp + D_sp, A_pp^FS = A_pp + D_pp on the diagonal;
//   S_pp = A_pp^FS - (D_ps / D_ss) A_sp^FS  (same pattern).
// Bit-identical to the oracle (IEEE intrinsics, same expression order).
__global__ void k_fs_qimpes(int Nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                            const double *__restrict__ fs, const double *__restrict__ dssv, const double *__restrict__ dpsv,
                            double *__restrict__ spp, double *__restrict__ dssinv, unsigned long long *skipped)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc) return;
    int64_t qd = -1;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) if (ci[q] == i) { qd = q; break; }
    const double dss = dssv[i], dps = dpsv[i];
    double cfac = 0.0;
    if (dss != 0.0) cfac = __ddiv_rn(dps, dss);
    else atomicAdd(skipped, 1ULL);                         // skip the correction, count it
    dssinv[i] = dss != 0.0 ? 1.0 / dss : 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        double app = v[q * 4 + 3], asp = v[q * 4 + 1];
        if (q == qd) { app = __dadd_rn(app, fs[2 * i + 1]); asp = __dadd_rn(asp, fs[2 * i]); }
        spp[q] = __dsub_rn(app, __dmul_rn(cfac, asp));
    }
}

// D_fs / fs_modulus_scale (remark P:443)
__global__ void k_fs_scale(int64_t n, const double *__restrict__ fs, double scale, double *__restrict__ out)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = __ddiv_rn(fs[k], scale);
}
// RSL helpers: x = [0_u | (0, 1) per cell]; y_u = a - b; out_f = -t_f
__global__ void k_rsl_e(int64_t nu, int Nc, double *x)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < nu) x[k] = 0.0;
    else if (k < nu + 2 * (int64_t)Nc) x[k] = ((k - nu) & 1) ? 1.0 : 0.0;
}
__global__ void k_sub(int64_t n, const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ y)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) y[k] = a[k] - b[k];
}
__global__ void k_axpy1(int64_t n, const double *__restrict__ a, double *__restrict__ y)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) y[k] = y[k] + a[k];
}
__global__ void k_neg(int64_t n, const double *__restrict__ a, double *__restrict__ y)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) y[k] = -a[k];
}
__global__ void k_diag_csr(int n, const double *__restrict__ d, int32_t *rp, int32_t *ci, double *v)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { rp[i] = i; ci[i] = i; v[i] = d[i]; }
    if (i == n) rp[n] = n;
}

// copy the pattern (local + global column ids) of a device CSR
static void copy_pattern(Ctx &c, const Csr &src, Csr &dst, int nc)
{
    dst.n = src.n; dst.m = src.m; dst.nc = nc; dst.nnz = src.nnz;
    dst.rp.alloc(src.n + 1); dst.ci.alloc(std::max<int64_t>(src.nnz, 1)); dst.v.alloc(std::max<int64_t>(src.nnz, 1) * nc);
    TSP_CUDA(cudaMemcpyAsync(dst.rp, src.rp, sizeof(int32_t) * (src.n + 1), cudaMemcpyDeviceToDevice, c.s));
    if (src.nnz) TSP_CUDA(cudaMemcpyAsync(dst.ci, src.ci, sizeof(int32_t) * src.nnz, cudaMemcpyDeviceToDevice, c.s));
    if (src.gci.p) {
        dst.gci.alloc(std::max<int64_t>(src.nnz, 1));
        if (src.nnz) TSP_CUDA(cudaMemcpyAsync(dst.gci, src.gci, sizeof(int32_t) * src.nnz, cudaMemcpyDeviceToDevice, c.s));
    }
}

void extract_sdc(Ctx &c)
{
    c.uu_sdc.alloc(3 * (size_t)std::max<int64_t>(c.uu.nnz, 1));
    if (c.uu.nnz) k_sdc<<<grid_for(c.uu.nnz, 256), 256, 0, c.s>>>(c.uu.nnz, c.uu.v, c.uu_sdc);
    c.launches++;
}

void setup_mech(Ctx &c)
{
    c.mech_ready = false;
    dbg_mark(c, "mech begin", -1);
    c.mech.L.clear();                     // free the previous hierarchy first: its memory is reused below
    if (c.sdc_stale) { sym_refill_sdc(c); c.sdc_stale = false; }   // A_uu changed since create (tsp_update_values)
    Csr A;
    copy_pattern(c, c.uu, A, 3);
    prof_begin(c, PK_SETUP);
    if (c.uu.nnz) TSP_CUDA(cudaMemcpyAsync(A.v, c.uu_sdc, sizeof(double) * 3 * c.uu.nnz, cudaMemcpyDeviceToDevice, c.s));
    DBuf<int32_t> zb; zb.alloc(std::max(c.Nn, 1));
    if (c.Nn) k_zb_nodes<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(c.Nn, c.nx, c.ny, c.nz_glob, c.k0, c.o.zblock, zb);
    prof_end(c, PK_SETUP, 0);
    c.launches += 2;
    dbg_mark(c, "mech sdc", -2);
    amg_build(c, c.mech, A, zb, 3, &c.hu, c.node_off, c.Nn_glob);   // a4 (mechanics): M_uu^-1 = amg(A_uu^SDC)
    c.mech_ready = true;
}

// eq:FS_RSL: D_sp = -diag(A_su A_uu^-1 A_up e), D_pp = -diag(A_pu A_uu^-1 A_up e), A_uu^-1
// approximated by the available preconditioner: rsl_iters steps of Richardson iteration
// y <- y + M_uu^-1 (g - A_uu y), y_0 = 0, g = A_up e.  Every product is the operator apply (row a12) with
// one block of the input zero, so the folds are those of the operator.
static void rsl_diag(Ctx &c)
{
    TSP_REQUIRE(c.mech_ready, TSP_ERR_STATE, "fs_mode RSL applies M_uu: run tsp_setup(MECH) before FLOW");
    const int64_t nu = 3 * (int64_t)c.Nn, n = c.n;
    DBuf<double> x, t, g, y, r, dy;
    x.alloc(std::max<int64_t>(n, 1)); t.alloc(std::max<int64_t>(n, 1));
    g.alloc(std::max<int64_t>(nu, 1)); y.alloc(std::max<int64_t>(nu, 1)); r.alloc(std::max<int64_t>(nu, 1));
    dy.alloc(std::max<int64_t>(nu, 1));
    if (n) k_rsl_e<<<grid_for(n, 256), 256, 0, c.s>>>(nu, c.Nc, x);
    op_apply(c, x, t);                                       // t_u = A_uu 0 + A_uf [0; e] = A_up e
    if (nu) TSP_CUDA(cudaMemcpyAsync(g, t, sizeof(double) * nu, cudaMemcpyDeviceToDevice, c.s));
    y.zero(c.s);
    if (n) TSP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c.s));
    for (int it = 0; it < c.o.rsl_iters; ++it) {
        if (nu) TSP_CUDA(cudaMemcpyAsync(x, y, sizeof(double) * nu, cudaMemcpyDeviceToDevice, c.s));
        op_apply(c, x, t);                                   // t_u = A_uu y
        if (nu) k_sub<<<grid_for(nu, 256), 256, 0, c.s>>>(nu, g, t, r);
        amg_vcycle(c, c.mech, r, dy, true);
        if (nu) k_axpy1<<<grid_for(nu, 256), 256, 0, c.s>>>(nu, dy, y);
        c.launches += 2;
    }
    if (nu) TSP_CUDA(cudaMemcpyAsync(x, y, sizeof(double) * nu, cudaMemcpyDeviceToDevice, c.s));
    op_apply(c, x, t);                                       // t_f = A_fu y + A_ff 0 = (A_su y, A_pu y)
    if (c.Nc) k_neg<<<grid_for(2 * (int64_t)c.Nc, 256), 256, 0, c.s>>>(2 * (int64_t)c.Nc, t.p + nu, c.fs_eff);
    c.launches += 3;
}

// refresh (NEXT-f1, R-refresh): the values of A_ff / A_fu / D_fs changed since the last flow setup
// (tsp_update_values), the patterns did not: every a1/a3/a5 product is recomputed and the pressure hierarchy
// keeps its strength flags, aggregates and patterns (amg_build refresh, the oracle's amg_refresh)
void setup_flow(Ctx &c, bool refresh)
{
    TSP_REQUIRE(!refresh || c.flow_built, TSP_ERR_STATE, "TSP_SETUP_REFRESH needs a completed TSP_SETUP_FLOW on this handle");
    c.flow_ready = c.flow_built = false;
    dbg_mark(c, "flow begin", -1);
    if (!refresh) c.pres.L.clear();
    // a1 input: the fixed-stress diagonal (given / scale, or RSL)
    c.fs_eff.alloc(2 * (size_t)std::max(c.Nc, 1));
    if (c.o.fs_mode == 1) rsl_diag(c);
    else if (c.Nc) {
        k_fs_scale<<<grid_for(2 * (int64_t)c.Nc, 256), 256, 0, c.s>>>(2 * (int64_t)c.Nc, c.fs, c.o.fs_modulus_scale, c.fs_eff);
        c.launches++;
    }
    // a3 diagonals (true-IMPES needs the ghost rows' couplings into this slab)
    c.cpr_dss.alloc(std::max(c.Nc, 1)); c.cpr_dps.alloc(std::max(c.Nc, 1));
    DBuf<double> up, dn, gup, gdn;
    const int ng = c.hf.nghost();
    if (c.o.cpr_mode == 1 && c.comm) {
        up.alloc(2 * (size_t)std::max(c.Nc, 1)); dn.alloc(2 * (size_t)std::max(c.Nc, 1));
        gup.alloc(2 * (size_t)std::max(ng, 1)); gdn.alloc(2 * (size_t)std::max(ng, 1));
        if (c.Nc) k_zcouple<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.ff.rp, c.ff.gci, c.ff.v, c.cell_off,
                                                                  (int64_t)c.nx * c.ny, up, dn);
        halo_exchange(c, c.hf, 2, up, gup);
        halo_exchange(c, c.hf, 2, dn, gdn);
        c.launches++;
    }
    if (c.Nc) k_cpr_diag<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.o.cpr_mode, c.ff.rp, c.ff.ci, c.ff.v, gup.p, gdn.p,
                                                               c.hf.nrecv[0], c.cpr_dss, c.cpr_dps);
    Csr S;
    copy_pattern(c, c.ff, S, 1);
    c.dss_inv.alloc(std::max(c.Nc, 1));
    c.dcount.zero(c.s);
    if (c.Nc) k_fs_qimpes<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.ff.rp, c.ff.ci, c.ff.v, c.fs_eff, c.cpr_dss, c.cpr_dps,
                                                                S.v, c.dss_inv, c.dcount);
    unsigned long long sk = 0;
    TSP_CUDA(cudaMemcpyAsync(&sk, c.dcount, sizeof(sk), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.skipped_dss = (int64_t)sk;
    halo_exchange(c, c.hf, 1, c.dss_inv, c.gh_dss);  // D_ss^-1 of the ghost cells (steps 3-4)
    if (c.o.aps_mode == 1) {                          // step 4 with D_ps^(CPR): a one-entry-per-row operator
        Csr D;
        D.n = c.Nc; D.m = c.Nc; D.nc = 1; D.nnz = c.Nc;
        D.rp.alloc(c.Nc + 1); D.ci.alloc(std::max(c.Nc, 1)); D.v.alloc(std::max(c.Nc, 1));
        k_diag_csr<<<grid_for(c.Nc + 1, 256), 256, 0, c.s>>>(c.Nc, c.cpr_dps, D.rp, D.ci, D.v);
        sell_from_csr(c, D, c.s_aps, 1);
        c.launches++;
    } else {
        const int map_aps[1] = {2};       // A_ps = entry (1,0) of every 2x2 block (full A_ps)
        sell_from_csr(c, c.ff, c.s_aps, 1, map_aps);
    }
    DBuf<int32_t> zb; zb.alloc(std::max(c.Nc, 1));
    if (c.Nc) k_zb_cells<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.nx, c.ny, c.k0, c.o.zblock, zb);
    c.launches += 3;
    dbg_mark(c, "flow qimpes", -2);
    amg_build(c, c.pres, S, zb, 1, &c.hf, c.cell_off, c.Nc_glob, refresh);   // a4 (pressure): M_pp^-1 = amg(S_pp)
    ilu_setup(c, nullptr);                // a5: tile ILU(0) of P S_ff^FS P^T
    dbg_mark(c, "ilu", -2);
    c.flow_ready = c.flow_built = true;
}

}  // namespace tsp

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

// a1 + a3: fixed stress (eq:Schur_1_FS) and quasi-IMPES:
//   A_sp^FS = A_sp + D_sp, A_pp^FS = A_pp + D_pp on the diagonal;
//   D_ss = diagm(A_ss), D_ps = diagm(A_ps);  S_pp = A_pp^FS - (D_ps / D_ss) A_sp^FS  (same pattern).
// Bit-identical to the oracle (IEEE intrinsics, same expression order).  `ci` are
// local ids: the diagonal of row i is column i.
__global__ void k_fs_qimpes(int Nc, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci, const double *__restrict__ v,
                            const double *__restrict__ fs, double *__restrict__ spp, double *__restrict__ dssinv,
                            unsigned long long *skipped)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc) return;
    int64_t qd = -1;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) if (ci[q] == i) { qd = q; break; }
    double dss = qd >= 0 ? v[qd * 4 + 0] : 0.0, dps = qd >= 0 ? v[qd * 4 + 2] : 0.0;
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

void setup_flow(Ctx &c)
{
    c.flow_ready = false;
    dbg_mark(c, "flow begin", -1);
    c.pres.L.clear();
    Csr S;
    copy_pattern(c, c.ff, S, 1);
    c.dss_inv.alloc(std::max(c.Nc, 1));
    c.dcount.zero(c.s);
    if (c.Nc) k_fs_qimpes<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.ff.rp, c.ff.ci, c.ff.v, c.fs, S.v, c.dss_inv, c.dcount);
    unsigned long long sk = 0;
    TSP_CUDA(cudaMemcpyAsync(&sk, c.dcount, sizeof(sk), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.skipped_dss = (int64_t)sk;
    halo_exchange(c, c.hf, 1, c.dss_inv, c.gh_dss);  // D_ss^-1 of the ghost cells (steps 3-4)
    const int map_aps[1] = {2};           // A_ps = entry (1,0) of every 2x2 block (full A_ps)
    sell_from_csr(c, c.ff, c.s_aps, 1, map_aps);
    DBuf<int32_t> zb; zb.alloc(std::max(c.Nc, 1));
    if (c.Nc) k_zb_cells<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, c.nx, c.ny, c.k0, c.o.zblock, zb);
    c.launches += 2;
    dbg_mark(c, "flow qimpes", -2);
    amg_build(c, c.pres, S, zb, 1, &c.hf, c.cell_off, c.Nc_glob);   // a4 (pressure): M_pp^-1 = amg(S_pp)
    ilu_setup(c, nullptr);                // a5: tile ILU(0) of P S_ff^FS P^T
    dbg_mark(c, "ilu", -2);
    c.flow_ready = true;
}

}  // namespace tsp

// apply.cu -- operator apply (row a12) and Algorithm 1 (alg:apply_M_inv,
// P:616-636) orchestration: steps 1 (mechanics V-cycle), 2,
// 3-4, 5 (pressure V-cycle), 6-8 fused with the tile ILU
// (P:629-634).  All matrices are SELL-32 (thread per block row, coalesced
// slot-major values, streaming loads for the matrix, cached loads for x).
// On a z-slab (multi-GPU) every x-gather is ghost-aware (GV): columns >= the
// owned count read the halo received from rank-1 / rank+1 just before.
#include "tsp_internal.cuh"

namespace tsp {

// ------------------------------------------------------------------ operator, node rows:
// y_u = A_uu x_u + A_uf x_f
template <bool D>
__global__ void __launch_bounds__(256) k_op_node(int cnt, Rows R, const int64_t *__restrict__ off_uu, const int32_t *__restrict__ col_uu,
                                                 const double *__restrict__ val_uu, const int64_t *__restrict__ off_uf,
                                                 const int32_t *__restrict__ col_uf, const double *__restrict__ val_uf,
                                                 GV xu, GV xf, double *__restrict__ yu)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int i = row_of(R, t);
    const int s = i >> 5, lane = i & 31;
    double a0 = 0, a1 = 0, a2 = 0;
    {
        const int64_t b0 = off_uu[s], b1 = off_uu[s + 1];
#pragma unroll 3
        for (int64_t slot = b0; slot < b1; ++slot) {
            const int cidx = __ldcs(col_uu + slot * 32 + lane);
            const double *v = val_uu + slot * (9 * 32) + lane;
            const double x0 = gvld<D>(xu, cidx, 0, 3), x1 = gvld<D>(xu, cidx, 1, 3), x2 = gvld<D>(xu, cidx, 2, 3);
            a0 = fma(__ldcs(v + 0 * 32), x0, a0); a0 = fma(__ldcs(v + 1 * 32), x1, a0); a0 = fma(__ldcs(v + 2 * 32), x2, a0);
            a1 = fma(__ldcs(v + 3 * 32), x0, a1); a1 = fma(__ldcs(v + 4 * 32), x1, a1); a1 = fma(__ldcs(v + 5 * 32), x2, a1);
            a2 = fma(__ldcs(v + 6 * 32), x0, a2); a2 = fma(__ldcs(v + 7 * 32), x1, a2); a2 = fma(__ldcs(v + 8 * 32), x2, a2);
        }
    }
    {
        const int64_t b0 = off_uf[s], b1 = off_uf[s + 1];
#pragma unroll 2
        for (int64_t slot = b0; slot < b1; ++slot) {
            const int cidx = __ldcs(col_uf + slot * 32 + lane);
            const double *v = val_uf + slot * (6 * 32) + lane;
            const double x0 = gvld<D>(xf, cidx, 0, 2), x1 = gvld<D>(xf, cidx, 1, 2);
            a0 = fma(__ldcs(v + 0 * 32), x0, a0); a0 = fma(__ldcs(v + 1 * 32), x1, a0);
            a1 = fma(__ldcs(v + 2 * 32), x0, a1); a1 = fma(__ldcs(v + 3 * 32), x1, a1);
            a2 = fma(__ldcs(v + 4 * 32), x0, a2); a2 = fma(__ldcs(v + 5 * 32), x1, a2);
        }
    }
    yu[3 * (int64_t)i] = a0; yu[3 * (int64_t)i + 1] = a1; yu[3 * (int64_t)i + 2] = a2;
}

// cell rows: y_f = [vf -] (A_fu x_u [+ A_ff x_f]);  mode 0: operator; mode 1: step 2, y_f = v_f - A_fu z_u;
// mode 2: the operator right after Algorithm 1 on the same vector -- its step 2 left y2 = v_f - A_fu z_u, so
// A_fu z_u = v_f - y2 and only A_ff is streamed: y_f = (v_f - y2) + A_ff x_f (y2 passed in `y2`)
template <int MODE, bool D>
__global__ void __launch_bounds__(256) k_op_cell(int cnt, Rows R, const int64_t *__restrict__ off_fu, const int32_t *__restrict__ col_fu,
                                                 const double *__restrict__ val_fu, const int64_t *__restrict__ off_ff,
                                                 const int32_t *__restrict__ col_ff, const double *__restrict__ val_ff,
                                                 GV xu, GV xf, const double *__restrict__ vf, double *__restrict__ yf,
                                                 const double *__restrict__ y2)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int i = row_of(R, t);
    const int s = i >> 5, lane = i & 31;
    double a0 = 0, a1 = 0;
    if (MODE == 2) {
        a0 = vf[2 * (int64_t)i] - y2[2 * (int64_t)i];
        a1 = vf[2 * (int64_t)i + 1] - y2[2 * (int64_t)i + 1];
    } else {
        const int64_t b0 = off_fu[s], b1 = off_fu[s + 1];
#pragma unroll 2
        for (int64_t slot = b0; slot < b1; ++slot) {
            const int cidx = __ldcs(col_fu + slot * 32 + lane);
            const double *v = val_fu + slot * (6 * 32) + lane;
            const double x0 = gvld<D>(xu, cidx, 0, 3), x1 = gvld<D>(xu, cidx, 1, 3), x2 = gvld<D>(xu, cidx, 2, 3);
            a0 = fma(__ldcs(v + 0 * 32), x0, a0); a0 = fma(__ldcs(v + 1 * 32), x1, a0); a0 = fma(__ldcs(v + 2 * 32), x2, a0);
            a1 = fma(__ldcs(v + 3 * 32), x0, a1); a1 = fma(__ldcs(v + 4 * 32), x1, a1); a1 = fma(__ldcs(v + 5 * 32), x2, a1);
        }
    }
    if (MODE == 0 || MODE == 2) {
        const int64_t b0 = off_ff[s], b1 = off_ff[s + 1];
#pragma unroll 2
        for (int64_t slot = b0; slot < b1; ++slot) {
            const int cidx = __ldcs(col_ff + slot * 32 + lane);
            const double *v = val_ff + slot * (4 * 32) + lane;
            const double x0 = gvld<D>(xf, cidx, 0, 2), x1 = gvld<D>(xf, cidx, 1, 2);
            a0 = fma(__ldcs(v + 0 * 32), x0, a0); a0 = fma(__ldcs(v + 1 * 32), x1, a0);
            a1 = fma(__ldcs(v + 2 * 32), x0, a1); a1 = fma(__ldcs(v + 3 * 32), x1, a1);
        }
        yf[2 * (int64_t)i] = a0; yf[2 * (int64_t)i + 1] = a1;
    } else {
        yf[2 * (int64_t)i] = vf[2 * (int64_t)i] - a0;
        yf[2 * (int64_t)i + 1] = vf[2 * (int64_t)i + 1] - a1;
    }
}

// steps 3-4: z_s = D_ss^-1 y_s ; w_p = y_p - A_ps z_s with the full A_ps;
// z_s of the neighbours is recomputed from y_s instead of re-read.
template <bool D>
__global__ void __launch_bounds__(256) k_step34(int Nc, const int64_t *__restrict__ off, const int32_t *__restrict__ col,
                                                const double *__restrict__ aps, GV dssinv, GV yf, double *__restrict__ zs,
                                                double *__restrict__ wp)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc) return;
    const int s = i >> 5, lane = i & 31;
    double acc = 0;
    const int64_t b0 = off[s], b1 = off[s + 1];
#pragma unroll 4
    for (int64_t slot = b0; slot < b1; ++slot) {
        const int j = __ldcs(col + slot * 32 + lane);
        acc = fma(__ldcs(aps + slot * 32 + lane), gvld<D>(yf, j, 0, 2) * gvld<D>(dssinv, j, 0, 1), acc);
    }
    zs[i] = yf.own[2 * (int64_t)i] * dssinv.own[i];
    wp[i] = yf.own[2 * (int64_t)i + 1] - acc;
}

// z_f (interleaved) -> (z_s, z_p) for the next second-stage sweep
__global__ void k_split_f(int Nc, const double *__restrict__ zf, double *__restrict__ zs, double *__restrict__ zp)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < Nc) { zs[i] = zf[2 * (int64_t)i]; zp[i] = zf[2 * (int64_t)i + 1]; }
}

static double sell_bytes(const Sell &S) { return (double)S.slots * 32 * (4.0 + 8.0 * S.bs); }

// ---- halo overlap on a z-slab (multi-GPU): the rows whose stencils reach a neighbour's planes are the first
// node / cell plane (rank > 0) and the last one (rank < P - 1); everything else is computed on the main stream
// while the halo exchange runs on the comm stream, then the boundary rows.  Same kernels and per-row arithmetic
// as one launch over all rows: bitwise the same result (TSP_NO_OVERLAP: exchange first, one launch per kernel).
struct Split {
    bool on = false;
    Rows in_n, bd_n, in_c, bd_c;
    int cin_n = 0, cbd_n = 0, cin_c = 0, cbd_c = 0;
};
static Split slab_split(const Ctx &c)
{
    Split sp;
    if (!c.comm || !c.cs || getenv("TSP_NO_OVERLAP")) return sp;
    const int NXY = (c.nx + 1) * (c.ny + 1), CP = c.nx * c.ny;
    const int lo = c.rank > 0, hi = c.rank < c.nranks - 1;
    const int nlo = lo * NXY, nhi = hi * NXY, clo = lo * CP, chi = hi * CP;
    if (c.Nn < nlo + nhi + NXY || c.Nc < clo + chi + CP) return sp;     // slab too thin to have interior planes
    sp.on = true;
    sp.in_n = Rows{nlo, c.Nn - nlo - nhi, c.Nn}; sp.cin_n = c.Nn - nlo - nhi;
    sp.bd_n = Rows{0, nlo, c.Nn - nhi}; sp.cbd_n = nlo + nhi;
    sp.in_c = Rows{clo, c.Nc - clo - chi, c.Nc}; sp.cin_c = c.Nc - clo - chi;
    sp.bd_c = Rows{0, clo, c.Nc - chi}; sp.cbd_c = clo + chi;
    return sp;
}
// the exchanges of `xchg` on the comm stream after everything already on the main stream; `interior` launched
// first (so a host-blocking backend does not delay it), the main stream then waits for the halos
template <class FI, class FX>
static void overlapped(Ctx &c, FI interior, FX xchg)
{
    TSP_CUDA(cudaEventRecord(c.ev_x, c.s));
    interior();
    TSP_CUDA(cudaStreamWaitEvent(c.cs, c.ev_x, 0));
    xchg(c.cs);
    TSP_CUDA(cudaEventRecord(c.ev_h, c.cs));
    TSP_CUDA(cudaStreamWaitEvent(c.s, c.ev_h, 0));
}

static void op_node_rows(Ctx &c, const GV &gu, const GV &gf, double *yu, Rows R, int cnt, double frac)
{
    prof_begin(c, PK_OP_NODE);
    if (!sym_op_node(c, gu, gf, yu, R, cnt) && cnt)
        (c.comm ? k_op_node<true> : k_op_node<false>)<<<grid_for(cnt, 256), 256, 0, c.s>>>(
            cnt, R, c.s_uu.off, c.s_uu.col, c.s_uu.val, c.s_uf.off, c.s_uf.col, c.s_uf.val, gu, gf, yu);
    prof_end(c, PK_OP_NODE, frac * ((c.sym_uu.ok ? sym_bytes(c, 9) : sell_bytes(c.s_uu)) + sell_bytes(c.s_uf) + 48.0 * c.Nn + 16.0 * c.Nc));
    c.launches++;
}
// MODE 0: y_f = A_fu x_u + A_ff x_f; MODE 2: y_f = (v_f - y2) + A_ff x_f (see k_op_cell)
template <int MODE>
static void op_cell_rows(Ctx &c, const GV &gu, const GV &gf, const double *vf, double *yf, Rows R, int cnt, double frac)
{
    prof_begin(c, PK_OP_CELL);
    if (cnt) {
        if (MODE == 0)
            (c.comm ? k_op_cell<0, true> : k_op_cell<0, false>)<<<grid_for(cnt, 256), 256, 0, c.s>>>(
                cnt, R, c.s_fu.off, c.s_fu.col, c.s_fu.val, c.s_ff.off, c.s_ff.col, c.s_ff.val, gu, gf, nullptr, yf, nullptr);
        else
            (c.comm ? k_op_cell<2, true> : k_op_cell<2, false>)<<<grid_for(cnt, 256), 256, 0, c.s>>>(
                cnt, R, nullptr, nullptr, nullptr, c.s_ff.off, c.s_ff.col, c.s_ff.val, gu, gf, vf, yf, c.w_yf);
    }
    prof_end(c, PK_OP_CELL, frac * (MODE == 0 ? sell_bytes(c.s_fu) + sell_bytes(c.s_ff) + 24.0 * c.Nn + 32.0 * c.Nc
                                              : sell_bytes(c.s_ff) + 64.0 * c.Nc));   // MODE 2: + v_f, y2, x_f read, y_f written
    c.launches++;
}

template <int MODE>
static void op_common(Ctx &c, const double *x, const double *vf, double *y)
{
    const double *xu = x, *xf = x + 3 * (int64_t)c.Nn;
    double *yu = y, *yf = y + 3 * (int64_t)c.Nn;
    const GV gu = gv(xu, c.Nn, c.gh_u.p), gf = gv(xf, c.Nc, c.gh_f.p);
    const Split sp = slab_split(c);
    if (!sp.on) {
        halo_exchange(c, c.hu, 3, xu, c.gh_u);
        halo_exchange(c, c.hf, 2, xf, c.gh_f);
        op_node_rows(c, gu, gf, yu, rows_all(c.Nn), c.Nn, 1.0);
        op_cell_rows<MODE>(c, gu, gf, vf, yf, rows_all(c.Nc), c.Nc, 1.0);
    } else {
        const double fn = c.Nn ? (double)sp.cin_n / c.Nn : 0.0, fc = c.Nc ? (double)sp.cin_c / c.Nc : 0.0;
        overlapped(c, [&] {
            op_node_rows(c, gu, gf, yu, sp.in_n, sp.cin_n, fn);
            op_cell_rows<MODE>(c, gu, gf, vf, yf, sp.in_c, sp.cin_c, fc);
        }, [&](cudaStream_t s) {
            halo_exchange(c, c.hu, 3, xu, c.gh_u, s);
            halo_exchange(c, c.hf, 2, xf, c.gh_f, s);
        });
        op_node_rows(c, gu, gf, yu, sp.bd_n, sp.cbd_n, 1.0 - fn);
        op_cell_rows<MODE>(c, gu, gf, vf, yf, sp.bd_c, sp.cbd_c, 1.0 - fc);
    }
    TSP_CUDA(cudaGetLastError());
}

void op_apply(Ctx &c, const double *x, double *y) { op_common<0>(c, x, nullptr, y); }

// y = A z right after z = M^-1 v (the FGMRES body): the cell rows reuse step 2's A_fu z_u (k_op_cell<2>), so A_fu
// is streamed once per iteration instead of twice (SELL(A_fu) x 52 B = 3.5 GB at C5)
void op_apply_after_prec(Ctx &c, const double *v, const double *z, double *y) { op_common<2>(c, z, v + 3 * (int64_t)c.Nn, y); }

void prec_apply(Ctx &c, const double *v, double *z)
{
    TSP_REQUIRE(c.mech_ready && c.flow_ready, TSP_ERR_STATE, "apply before tsp_setup(MECH|FLOW)");
    const int64_t nu = 3 * (int64_t)c.Nn;
    const double *vu = v, *vf = v + nu;
    double *zu = z, *zf = z + nu;
    // step 1: z_u = M_uu^-1 v_u
    amg_vcycle(c, c.mech, vu, zu, true);
    // step 2: y_f = v_f - A_fu z_u; on a slab the last cell plane (rank < P - 1) needs the node
    // plane above, so it waits for the halo while the other planes run
    {
        const GV gz = gv(zu, c.Nn, c.gh_u.p);
        auto step2 = [&](Rows R, int cnt, double frac) {
            prof_begin(c, PK_STEP2);
            if (cnt) (c.comm ? k_op_cell<1, true> : k_op_cell<1, false>)<<<grid_for(cnt, 256), 256, 0, c.s>>>(
                cnt, R, c.s_fu.off, c.s_fu.col, c.s_fu.val, nullptr, nullptr, nullptr, gz, gv(nullptr, 0), vf, c.w_yf, nullptr);
            prof_end(c, PK_STEP2, frac * (sell_bytes(c.s_fu) + 24.0 * c.Nn + 32.0 * c.Nc));
            c.launches++;
        };
        const Split sp = slab_split(c);
        if (!sp.on) {
            halo_exchange(c, c.hu, 3, zu, c.gh_u);
            step2(rows_all(c.Nc), c.Nc, 1.0);
        } else {
            const double fc = c.Nc ? (double)sp.cin_c / c.Nc : 0.0;
            overlapped(c, [&] { step2(sp.in_c, sp.cin_c, fc); }, [&](cudaStream_t s) { halo_exchange(c, c.hu, 3, zu, c.gh_u, s); });
            step2(sp.bd_c, sp.cbd_c, 1.0 - fc);
        }
    }
    // steps 3-4
    halo_exchange(c, c.hf, 2, c.w_yf, c.gh_f);
    prof_begin(c, PK_STEP34);
    if (c.Nc) (c.comm ? k_step34<true> : k_step34<false>)<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(
        c.Nc, c.s_aps.off, c.s_aps.col, c.s_aps.val, gv(c.dss_inv, c.Nc, c.gh_dss.p), gv(c.w_yf, c.Nc, c.gh_f.p), c.w_tmp, c.w_wp);
    prof_end(c, PK_STEP34, sell_bytes(c.s_aps) + 40.0 * c.Nc);
    // step 5: z_p = M_pp^-1 w_p
    amg_vcycle(c, c.pres, c.w_wp, c.w_zp, false);
    // steps 6-8: w_f = y_f - S_ff^FS z_f ; z_f += P^T M_L^-1 P w_f
    // repeated local_sweeps times ("several sweeps"): the next sweep's z = this sweep's z_f
    const int ng = c.hf.nghost();
    for (int sw = 0; sw < c.o.local_sweeps; ++sw) {
        if (sw > 0) {
            if (c.Nc) k_split_f<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(c.Nc, zf, c.w_tmp, c.w_zp);
            c.launches++;
        }
        halo_exchange(c, c.hf, 1, c.w_tmp, c.gh_f2);
        halo_exchange(c, c.hf, 1, c.w_zp, c.gh_f2.p + ng);
        ilu_apply_fused(c, c.w_yf, c.w_tmp, c.w_zp, zf);
    }
    c.launches += 1;                                 // steps 3-4
    TSP_CUDA(cudaGetLastError());
}

}  // namespace tsp

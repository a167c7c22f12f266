// newton.cu -- the nonlinear step around the hot path: one implicit time step of the coupled
// problem by Newton's method with a backtracking line search, entirely on the device.  Per Newton iteration:
//   state fields at x (porosity with the strain, s, p)  ->  tsp_assemble / tsp_assemble_scale (the Jacobian,
//   assemble.cu)  ->  tsp_update_values + tsp_setup(FLOW | REFRESH) (the per-Newton flow setup on frozen
//   aggregates; the mechanics AMG stays as built)  ->  residual (Appendix B.1, assemble.cu)  ->
//   FGMRES with the two-stage preconditioner  ->  x += alpha dx, alpha halved until the scaled residual norm drops.
// The residual norm is measured with the row scales of the step's first Jacobian (fixed within the step); the
// linear system of iteration k uses its own scales S_k:  J_k y = -S_k r,  dx = (y_u, y_s, p_unit y_p).
// Its CPU reference (the same algorithm on the test oracle's pieces) is newton.py of the oracle package.
#include <cmath>
#include <cstring>
#include <vector>

#include "tsp_internal.cuh"

namespace tsp {

constexpr int kNT = 256;

// per-block partial sums of (w_i r_i)^2 (w = su on u rows, ss / sp on the interleaved (s, p) rows; fixed order)
__global__ void __launch_bounds__(kNT) k_wnorm_part(int64_t nu, int64_t n, const double *__restrict__ r, double su, double ss,
                                                     double sp, double *__restrict__ part)
{
    __shared__ double red[kNT];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const double w = i < nu ? su : (((i - nu) & 1) ? sp : ss);
        const double v = w * r[i];
        acc = fma(v, v, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = kNT / 2; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_sum_parts(int np, const double *__restrict__ part, double *__restrict__ out)
{
    if (threadIdx.x || blockIdx.x) return;
    double s = 0.0;
    for (int k = 0; k < np; ++k) s += part[k];
    *out = sqrt(s);
}
// rhs = -S (r - r_off) on the rows (r_off: the momentum offset of the initial state, u rows only; may be null)
__global__ void k_newton_rhs(int64_t nu, int64_t n, const double *__restrict__ r, const double *__restrict__ r_off, double su,
                             double ss, double sp, double *__restrict__ rhs, double *__restrict__ rc)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = r[i] - (r_off && i < nu ? r_off[i] : 0.0);
    rc[i] = v;
    const double w = i < nu ? su : (((i - nu) & 1) ? sp : ss);
    rhs[i] = -w * v;
}
// x_new = x + alpha (y_u, y_s, p_unit y_p), saturation kept in [0, 1]
__global__ void k_newton_update(int64_t nu, int64_t n, const double *__restrict__ x, const double *__restrict__ y, double alpha,
                                double p_unit, double *__restrict__ xn)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (i < nu) { xn[i] = x[i] + alpha * y[i]; return; }
    if (((i - nu) & 1) == 0) { const double s = x[i] + alpha * y[i]; xn[i] = s < 0.0 ? 0.0 : s > 1.0 ? 1.0 : s; }
    else xn[i] = x[i] + alpha * p_unit * y[i];
}

struct NewtonWork {
    int64_t nn, nc, n, b[4];            // this rank's rows
    int64_t NnG, NcG, NG;               // global sizes
    DBuf<int32_t> rp[4], ci[4];
    DBuf<double> val[4], fs, phi, sat, pres, r, rc, rhs, y, xt, xg, rg, part, nrm, mp, sbuf, rbuf;
    void alloc(const tsp_asm_params &P, int rank, int nranks, int zblock)
    {
        int64_t sz[6];
        assembly_sizes(P, rank, nranks, zblock, sz);
        nn = sz[0]; nc = sz[1]; n = 3 * nn + 2 * nc;
        NnG = (int64_t)(P.nx + 1) * (P.ny + 1) * (P.nz + 1); NcG = (int64_t)P.nx * P.ny * P.nz; NG = 3 * NnG + 2 * NcG;
        const int64_t rows[4] = {nn, nn, nc, nc};
        for (int k = 0; k < 4; ++k) {
            b[k] = sz[2 + k];
            rp[k].alloc(rows[k] + 1); ci[k].alloc(std::max<int64_t>(b[k], 1));
        }
        realloc_values();
        phi.alloc(std::max<int64_t>(NcG, 1)); sat.alloc(std::max<int64_t>(NcG, 1)); pres.alloc(std::max<int64_t>(NcG, 1));
        r.alloc(n); rc.alloc(n); rhs.alloc(n); y.alloc(n); xt.alloc(n); xg.alloc(NG); rg.alloc(NG);
        part.alloc(1024); nrm.alloc(1); mp.alloc(std::max<int64_t>(2 * nc, 1));
    }
    void realloc_values()   // (again) after commit_values took the assembled values
    {
        const int64_t bs[4] = {9, 6, 6, 4};
        for (int k = 0; k < 4; ++k) val[k].alloc(std::max<int64_t>(b[k], 1) * bs[k]);
        fs.alloc(std::max<int64_t>(2 * nc, 1));
    }
};

// the ranks' [u_own | f_own] gathered into the global [u | f] (identical on every rank; a copy on one rank)
static void gather_state(Ctx &c, NewtonWork &W, const double *xl, double *xg)
{
    const cudaStream_t s = c.s;
    if (!c.comm) { TSP_CUDA(cudaMemcpyAsync(xg, xl, sizeof(double) * W.n, cudaMemcpyDeviceToDevice, s)); return; }
    const int P = c.nranks;
    std::vector<int64_t> parts(6 * (size_t)P);
    int64_t mu = 1, mf = 1;
    for (int r = 0; r < P; ++r) {
        partition(c.nx, c.ny, c.nz_glob, c.o.zblock, r, P, &parts[6 * r]);
        mu = std::max(mu, 3 * parts[6 * r + 3]); mf = std::max(mf, 2 * parts[6 * r + 5]);
    }
    const int64_t blk = mu + mf;
    if (W.sbuf.n < (size_t)blk) W.sbuf.alloc(blk);
    if (W.rbuf.n < (size_t)blk * P) W.rbuf.alloc(blk * P);
    TSP_CUDA(cudaMemcpyAsync(W.sbuf.p, xl, sizeof(double) * 3 * W.nn, cudaMemcpyDeviceToDevice, s));
    TSP_CUDA(cudaMemcpyAsync(W.sbuf.p + mu, xl + 3 * W.nn, sizeof(double) * 2 * W.nc, cudaMemcpyDeviceToDevice, s));
    c.comm->allgather(W.sbuf.p, W.rbuf.p, sizeof(double) * blk, s);
    for (int r = 0; r < P; ++r) {
        const int64_t *q = &parts[6 * r];
        if (q[3]) TSP_CUDA(cudaMemcpyAsync(xg + 3 * q[2], W.rbuf.p + r * blk, sizeof(double) * 3 * q[3], cudaMemcpyDeviceToDevice, s));
        if (q[5]) TSP_CUDA(cudaMemcpyAsync(xg + 3 * W.NnG + 2 * q[4], W.rbuf.p + r * blk + mu, sizeof(double) * 2 * q[5],
                                           cudaMemcpyDeviceToDevice, s));
    }
}

// ||S0 r|| over the GLOBAL residual (gathered): every rank computes the same number, equal to the one-rank value
static double wnorm(Ctx &c, NewtonWork &W, const double *rl, const double sc[3])
{
    const cudaStream_t s = c.s;
    gather_state(c, W, rl, W.rg);
    const int nb = (int)std::min<int64_t>(1024, (W.NG + kNT - 1) / kNT);
    if (W.NG) k_wnorm_part<<<nb, kNT, 0, s>>>(3 * W.NnG, W.NG, W.rg, sc[0], sc[1], sc[2], W.part);
    k_sum_parts<<<1, 1, 0, s>>>(nb, W.part, W.nrm);
    double v = 0.0;
    TSP_CUDA(cudaMemcpyAsync(&v, W.nrm.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    TSP_CUDA(cudaStreamSynchronize(s));
    return v;
}

}  // namespace tsp

using namespace tsp;

extern "C" {

tsp_status tsp_residual(const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, const double *x, const double *mprev,
                        double *r, void *stream)
{
    if (!p || !ref) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        StreamScope ss_((cudaStream_t)stream, nullptr);
        residual((cudaStream_t)stream, *p, *ref, dt, x, mprev, r);
        TSP_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

tsp_status tsp_masses(const tsp_asm_params *p, const tsp_cell_fields *ref, const double *x, double *m, void *stream)
{
    if (!p || !ref || !x || !m) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        StreamScope ss_((cudaStream_t)stream, nullptr);
        masses((cudaStream_t)stream, *p, *ref, x, m);
        TSP_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

void tsp_default_newton_opts(tsp_newton_opts *o)
{
    if (!o) return;
    o->rtol = 1e-6; o->atol = 0.0; o->max_newton = 12; o->lin_rtol = 1e-8; o->max_lin_iters = 1000; o->refresh = 1;
    o->max_halvings = 5;
}

tsp_status tsp_newton_step(tsp_handle h, const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, double *x,
                           const double *mprev, const double *r_off, const tsp_newton_opts *opts, tsp_newton_info *info)
{
    if (!h || !p || !ref || !x || !info) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    tsp_newton_opts o;
    tsp_default_newton_opts(&o);
    if (opts) o = *opts;
    memset(info, 0, sizeof(*info));
    try {
        Ctx &c = *h;
        StreamScope ss_(c.s, &c.alloc);
        TSP_REQUIRE(c.mech_ready, TSP_ERR_STATE, "tsp_newton_step: run tsp_setup(TSP_SETUP_MECH) first");
        TSP_REQUIRE(p->nx == c.nx && p->ny == c.ny && p->nz == c.nz_glob, TSP_ERR_INVALID_ARG, "tsp_newton_step: grid differs");
        const cudaStream_t s = c.s;
        const int rank = c.rank, P = c.nranks, zb = c.o.zblock;
        tsp_asm_params Pd = *p;
        Pd.dt = dt;                                           // the Jacobian of this step's time step
        p = &Pd;
        NewtonWork W;
        W.alloc(*p, rank, P, zb);
        TSP_REQUIRE(W.n == c.n, TSP_ERR_INVALID_ARG, "tsp_newton_step: the handle's rows are not this rank's slab");
        const int64_t nu = 3 * W.nn, n = W.n;
        // masses of the state at the start of the step (unless given)
        const double *mp = mprev;
        if (!mp) {
            gather_state(c, W, x, W.xg);
            masses_local(s, *p, *ref, W.xg, W.mp, rank, P, zb);
            mp = W.mp;
        }
        auto eval = [&](const double *xl, double *rl) {       // this rank's residual rows at the local state xl
            gather_state(c, W, xl, W.xg);
            residual(s, *p, *ref, dt, W.xg, mp, rl, rank, P, zb);
        };
        double S0[3] = {1, 1, 1};
        double norm0 = 0.0;
        info->status = 1;
        for (int it = 0;; ++it) {
            // the Jacobian at x (this rank's slab, the state fields of the whole grid) and its row scales
            tsp_bsr_out blk[4];
            for (int k = 0; k < 4; ++k) blk[k] = tsp_bsr_out{W.rp[k].p, W.ci[k].p, W.val[k].p};
            gather_state(c, W, x, W.xg);
            state_fields(s, *p, *ref, W.xg, W.phi, W.sat, W.pres);
            const tsp_cell_fields at{ref->E, ref->perm, W.phi.p, W.sat.p, W.pres.p, ref->well, ref->phi};
            double rmax[3], sc[3];
            assemble(s, *p, rank, P, zb, at, blk, W.fs, rmax);
            if (c.comm) {                                     // the row maxima over the ranks (exact)
                std::vector<double> all = host_allgather<double>(c, std::vector<double>(rmax, rmax + 3));
                for (int r = 0; r < P; ++r) for (int k = 0; k < 3; ++k) rmax[k] = std::max(rmax[k], all[3 * r + k]);
            }
            assemble_scale(s, *p, rank, P, zb, rmax, blk, W.fs, sc);
            if (it == 0) memcpy(S0, sc, sizeof(S0));
            // residual (minus the initial-state momentum offset)
            eval(x, W.r);
            if (n) k_newton_rhs<<<grid_for(n, 256), 256, 0, s>>>(nu, n, W.r, r_off, sc[0], sc[1], sc[2], W.rhs, W.rc);
            const double nrm = wnorm(c, W, W.rc, S0);
            if (it == 0) { norm0 = nrm; info->res0 = nrm; }
            info->res = nrm;
            if (it < 16) info->res_hist[it] = nrm;
            if (nrm <= o.atol || nrm <= o.rtol * norm0 || norm0 == 0.0) { info->status = 0; break; }
            if (it >= o.max_newton) break;
            // the linear system of this iteration: the assembled values move into the handle (same patterns, checked
            // once), per-Newton flow setup, FGMRES
            if (it == 0) {
                const Csr *cur[4] = {&c.uu, &c.uf, &c.fu, &c.ff};
                for (int k = 0; k < 4; ++k)
                    TSP_REQUIRE(cur[k]->nnz == W.b[k] && !pattern_differs(c, *cur[k], W.rp[k], W.ci[k]), TSP_ERR_INVALID_ARG,
                                "tsp_newton_step: the handle's patterns are not this grid's");
            }
            commit_values(c, W.val, W.fs);
            W.realloc_values();
            tsp_status st = tsp_setup(h, TSP_SETUP_FLOW | (o.refresh && c.flow_built ? TSP_SETUP_REFRESH : 0));
            if (st != TSP_OK) return st;
            tsp_solve_opts so;
            tsp_default_solve_opts(&so);
            so.rtol = o.lin_rtol; so.max_iters = o.max_lin_iters; so.x0_zero = 1;
            tsp_solve_info si;
            st = tsp_solve(h, W.rhs, W.y, &so, &si);
            if (st != TSP_OK && st != TSP_NOT_CONVERGED) return st;
            info->lin_iters += si.iterations;
            if (it < 16) info->lin_hist[it] = si.iterations;
            // backtracking line search on the S0-scaled residual norm (the same decisions on every rank)
            double alpha = 1.0, nt = 0.0;
            for (int hv = 0;; ++hv) {
                if (n) k_newton_update<<<grid_for(n, 256), 256, 0, s>>>(nu, n, x, W.y, alpha, p->p_unit, W.xt);
                eval(W.xt, W.r);
                if (n) k_newton_rhs<<<grid_for(n, 256), 256, 0, s>>>(nu, n, W.r, r_off, 1.0, 1.0, 1.0, W.rhs, W.rc);
                nt = wnorm(c, W, W.rc, S0);
                if (nt <= (1.0 - 1e-4 * alpha) * nrm || hv >= o.max_halvings) break;
                alpha *= 0.5;
                info->halvings++;
            }
            TSP_CUDA(cudaMemcpyAsync(x, W.xt.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
            info->newton_iters = it + 1;
            c.launches += 8;
        }
        TSP_CUDA(cudaStreamSynchronize(s));
        return info->status == 0 ? TSP_OK : TSP_NOT_CONVERGED;
    } catch (...) {
        return status_of_current_exception();
    }
}

tsp_status tsp_newton_residual(tsp_handle h, const tsp_asm_params *p, const tsp_cell_fields *ref, double dt, const double *x,
                               const double *mprev, double *r)
{
    if (!h || !p || !ref || !x || !r) { set_error("null argument"); return TSP_ERR_INVALID_ARG; }
    try {
        Ctx &c = *h;
        StreamScope ss_(c.s, &c.alloc);
        NewtonWork W;
        W.alloc(*p, c.rank, c.nranks, c.o.zblock);
        TSP_REQUIRE(W.n == c.n, TSP_ERR_INVALID_ARG, "tsp_newton_residual: the handle's rows are not this rank's slab");
        gather_state(c, W, x, W.xg);
        const double *mp = mprev;
        if (!mp) { masses_local(c.s, *p, *ref, W.xg, W.mp, c.rank, c.nranks, c.o.zblock); mp = W.mp; }
        residual(c.s, *p, *ref, dt, W.xg, mp, r, c.rank, c.nranks, c.o.zblock);
        TSP_CUDA(cudaStreamSynchronize(c.s));
        return TSP_OK;
    } catch (...) {
        return status_of_current_exception();
    }
}

}  // extern "C"

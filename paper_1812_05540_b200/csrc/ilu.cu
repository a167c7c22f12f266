// ilu.cu -- row a5 (factorisation) and rows a10-a11 (steps 6-8 of Algorithm 1,
// P:629-634) as one fused kernel: the second-stage local preconditioner M_L of
// P:606-612 read as tile-local 2x2-block ILU(0) of the interleaved S_ff^FS
// (DESIGN.md R-ilu: block Jacobi over fixed 16^3 tiles, natural order inside).
//
// On the 7-point TPFA pattern ILU(0) produces no update of off-diagonal blocks
// (a lower neighbour's upper neighbours are never neighbours of the row), so
//   U_KJ = A_KJ (J > K),  L_KJ = A_KJ U_JJ^-1 (J < K),
//   U_KK = A_KK - sum_{J < K, same tile} A_KJ U_JJ^-1 A_JK,
// and the solve needs only A and D^-1 = U_KK^-1:
//   forward   yhat_K = D_K^-1 (w_K - sum_{J<K} A_KJ yhat_J)
//   backward  x_K    = yhat_K - D_K^-1 sum_{J>K} A_KJ x_J
// One CTA per tile walks the i+j+k wavefronts (46 levels for 16^3) with the tile
// vector in shared memory.  The oracle instead runs textbook IKJ block ILU(0).
#include <algorithm>

#include "tsp_internal.cuh"

namespace tsp {

// slot order: 0 -z, 1 -y, 2 -x, 3 self, 4 +x, 5 +y, 6 +z  (lower = 0..2, upper = 4..6)
__constant__ int c_dx[7] = {0, 0, -1, 0, 1, 0, 0};
__constant__ int c_dy[7] = {0, -1, 0, 0, 0, 1, 0};
__constant__ int c_dz[7] = {-1, 0, 0, 0, 0, 0, 1};

struct TileGeo {
    int nx, ny, nz, tx, ty, tz, ntx, nty, ntz, T, Tpad;
};

__device__ __forceinline__ int64_t ival_idx(const TileGeo &g, int64_t t, int p, int k, int e)
{
    return ((((t * (g.Tpad >> 5) + (p >> 5)) * 7 + k) * 4 + e) << 5) + (p & 31);
}
__device__ __forceinline__ int64_t idinv_idx(const TileGeo &g, int64_t t, int p, int e)
{
    return (((t * (g.Tpad >> 5) + (p >> 5)) * 4 + e) << 5) + (p & 31);
}

// fill the tile-ordered S_ff^FS = A_ff + diag(D_sp, D_pp) blocks (a1 folded in)
__global__ void k_ilu_fill(TileGeo g, const int32_t *__restrict__ rp, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const double *__restrict__ fs, const int32_t *__restrict__ posmap,
                           double *__restrict__ ival)
{
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)g.nx * g.ny * g.nz) return;
    int i = c % g.nx, j = (c / g.nx) % g.ny, k = c / ((int64_t)g.nx * g.ny);
    int TI = i / g.tx, TJ = j / g.ty, TK = k / g.tz;
    int64_t t = ((int64_t)TK * g.nty + TJ) * g.ntx + TI;
    int li = i - TI * g.tx, lj = j - TJ * g.ty, lk = k - TK * g.tz;
    int p = posmap[(lk * g.ty + lj) * g.tx + li];
    for (int s = 0; s < 7; ++s)
        for (int e = 0; e < 4; ++e) ival[ival_idx(g, t, p, s, e)] = 0.0;
    for (int64_t q = rp[c]; q < rp[c + 1]; ++q) {
        int64_t d = ci[q];
        int di = (int)(d % g.nx) - i, dj = (int)((d / g.nx) % g.ny) - j, dk = (int)(d / ((int64_t)g.nx * g.ny)) - k;
        int s = -1;
        for (int u = 0; u < 7; ++u) if (c_dx[u] == di && c_dy[u] == dj && c_dz[u] == dk) s = u;
        if (s < 0) continue;   // not a 7-point neighbour (never happens for TPFA input)
        for (int e = 0; e < 4; ++e) {
            double a = v[q * 4 + e];
            if (s == 3 && e == 1) a += fs[2 * c];      // A_sp^FS = A_sp + D_sp
            if (s == 3 && e == 3) a += fs[2 * c + 1];  // A_pp^FS = A_pp + D_pp
            ival[ival_idx(g, t, p, s, e)] = a;
        }
    }
}

__device__ __forceinline__ void ld4(const double *__restrict__ a, const TileGeo &g, int64_t t, int p, int s, double r[4])
{
    for (int e = 0; e < 4; ++e) r[e] = a[ival_idx(g, t, p, s, e)];
}

// a5: U_KK = A_KK - sum_{J<K in tile} A_KJ U_JJ^-1 A_JK ; store U_KK^-1 (perturbed if singular)
__global__ void __launch_bounds__(256) k_ilu_factor(TileGeo g, const int32_t *__restrict__ lvlptr, int nlev,
                                                    const int32_t *__restrict__ cells, const int32_t *__restrict__ posmap,
                                                    const double *__restrict__ ival, double *__restrict__ dinv,
                                                    unsigned long long *__restrict__ npert)
{
    const int64_t t = blockIdx.x;
    const int TI = t % g.ntx, TJ = (t / g.ntx) % g.nty, TK = t / ((int64_t)g.ntx * g.nty);
    for (int l = 0; l < nlev; ++l) {
        for (int idx = lvlptr[l] + threadIdx.x; idx < lvlptr[l + 1]; idx += blockDim.x) {
            int pk = cells[idx];
            int li = pk & 255, lj = (pk >> 8) & 255, lk = pk >> 16;
            if (TI * g.tx + li >= g.nx || TJ * g.ty + lj >= g.ny || TK * g.tz + lk >= g.nz) continue;
            int p = idx;
            double U[4];
            ld4(ival, g, t, p, 3, U);
            for (int s = 0; s < 3; ++s) {
                int ni = li + c_dx[s], nj = lj + c_dy[s], nk = lk + c_dz[s];
                if (ni < 0 || nj < 0 || nk < 0) continue;   // outside the tile (or domain): dropped
                int pn = posmap[(nk * g.ty + nj) * g.tx + ni];
                double A[4], B[4], D[4];
                ld4(ival, g, t, p, s, A);          // A_KJ
                ld4(ival, g, t, pn, 6 - s, B);     // A_JK (J's block toward K)
                for (int e = 0; e < 4; ++e) D[e] = dinv[idinv_idx(g, t, pn, e)];
                double L0 = A[0] * D[0] + A[1] * D[2], L1 = A[0] * D[1] + A[1] * D[3];
                double L2 = A[2] * D[0] + A[3] * D[2], L3 = A[2] * D[1] + A[3] * D[3];
                U[0] -= L0 * B[0] + L1 * B[2]; U[1] -= L0 * B[1] + L1 * B[3];
                U[2] -= L2 * B[0] + L3 * B[2]; U[3] -= L2 * B[1] + L3 * B[3];
            }
            double sc = fmax(fmax(fabs(U[0]), fabs(U[1])), fmax(fabs(U[2]), fabs(U[3])));
            double det = U[0] * U[3] - U[1] * U[2];
            if (sc == 0.0 || fabs(det) <= 1e-14 * sc * sc) {
                double dl = 1e-12 * (sc > 0.0 ? sc : 1.0);
                U[0] += dl; U[3] += dl;
                det = U[0] * U[3] - U[1] * U[2];
                atomicAdd(npert, 1ULL);
            }
            dinv[idinv_idx(g, t, p, 0)] = U[3] / det;
            dinv[idinv_idx(g, t, p, 1)] = -U[1] / det;
            dinv[idinv_idx(g, t, p, 2)] = -U[2] / det;
            dinv[idinv_idx(g, t, p, 3)] = U[0] / det;
        }
        __syncthreads();
    }
}

// steps 6-8 fused: w = y - S^FS z (all neighbours, global z), forward/backward
// tile solve, z_out = z + dz (interleaved)
__global__ void __launch_bounds__(256) k_ilu_apply(TileGeo g, const int32_t *__restrict__ lvlptr, int nlev,
                                                   const int32_t *__restrict__ cells, const int32_t *__restrict__ posmap,
                                                   const double *__restrict__ ival, const double *__restrict__ dinv,
                                                   const double *__restrict__ yf, const double *__restrict__ zs,
                                                   const double *__restrict__ zp, double *__restrict__ zout)
{
    extern __shared__ double sm[];   // [Tpad][2]
    const int64_t t = blockIdx.x;
    const int TI = t % g.ntx, TJ = (t / g.ntx) % g.nty, TK = t / ((int64_t)g.ntx * g.nty);
    const int64_t sx = 1, sy = g.nx, sz = (int64_t)g.nx * g.ny;
    for (int l = 0; l < nlev; ++l) {
        for (int idx = lvlptr[l] + threadIdx.x; idx < lvlptr[l + 1]; idx += blockDim.x) {
            int pk = cells[idx];
            int li = pk & 255, lj = (pk >> 8) & 255, lk = pk >> 16;
            int gi = TI * g.tx + li, gj = TJ * g.ty + lj, gk = TK * g.tz + lk;
            if (gi >= g.nx || gj >= g.ny || gk >= g.nz) continue;
            int64_t gc = gi + sy * gj + sz * gk;
            double r0 = yf[2 * gc], r1 = yf[2 * gc + 1];
            // step 6: w = y - S^FS z over all 7 neighbours
#pragma unroll
            for (int s = 0; s < 7; ++s) {
                int ni = gi + c_dx[s], nj = gj + c_dy[s], nk = gk + c_dz[s];
                if (ni < 0 || nj < 0 || nk < 0 || ni >= g.nx || nj >= g.ny || nk >= g.nz) continue;
                int64_t gn = gc + c_dx[s] * sx + c_dy[s] * sy + c_dz[s] * sz;
                double a0 = ival[ival_idx(g, t, idx, s, 0)], a1 = ival[ival_idx(g, t, idx, s, 1)];
                double a2 = ival[ival_idx(g, t, idx, s, 2)], a3 = ival[ival_idx(g, t, idx, s, 3)];
                double z0 = zs[gn], z1 = zp[gn];
                r0 -= a0 * z0 + a1 * z1;
                r1 -= a2 * z0 + a3 * z1;
            }
            // forward: r -= sum_{lower in tile} A_KJ yhat_J
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                int ni = li + c_dx[s], nj = lj + c_dy[s], nk = lk + c_dz[s];
                if (ni < 0 || nj < 0 || nk < 0) continue;
                int pn = posmap[(nk * g.ty + nj) * g.tx + ni];
                double a0 = ival[ival_idx(g, t, idx, s, 0)], a1 = ival[ival_idx(g, t, idx, s, 1)];
                double a2 = ival[ival_idx(g, t, idx, s, 2)], a3 = ival[ival_idx(g, t, idx, s, 3)];
                double y0 = sm[2 * pn], y1 = sm[2 * pn + 1];
                r0 -= a0 * y0 + a1 * y1;
                r1 -= a2 * y0 + a3 * y1;
            }
            double d0 = dinv[idinv_idx(g, t, idx, 0)], d1 = dinv[idinv_idx(g, t, idx, 1)];
            double d2 = dinv[idinv_idx(g, t, idx, 2)], d3 = dinv[idinv_idx(g, t, idx, 3)];
            sm[2 * idx] = d0 * r0 + d1 * r1;
            sm[2 * idx + 1] = d2 * r0 + d3 * r1;
        }
        __syncthreads();
    }
    for (int l = nlev - 1; l >= 0; --l) {
        for (int idx = lvlptr[l] + threadIdx.x; idx < lvlptr[l + 1]; idx += blockDim.x) {
            int pk = cells[idx];
            int li = pk & 255, lj = (pk >> 8) & 255, lk = pk >> 16;
            int gi = TI * g.tx + li, gj = TJ * g.ty + lj, gk = TK * g.tz + lk;
            if (gi >= g.nx || gj >= g.ny || gk >= g.nz) continue;
            double t0 = 0, t1 = 0;
#pragma unroll
            for (int s = 4; s < 7; ++s) {
                int ni = li + c_dx[s], nj = lj + c_dy[s], nk = lk + c_dz[s];
                if (ni >= g.tx || nj >= g.ty || nk >= g.tz || gi + c_dx[s] >= g.nx || gj + c_dy[s] >= g.ny || gk + c_dz[s] >= g.nz) continue;
                int pn = posmap[(nk * g.ty + nj) * g.tx + ni];
                double a0 = ival[ival_idx(g, t, idx, s, 0)], a1 = ival[ival_idx(g, t, idx, s, 1)];
                double a2 = ival[ival_idx(g, t, idx, s, 2)], a3 = ival[ival_idx(g, t, idx, s, 3)];
                double x0 = sm[2 * pn], x1 = sm[2 * pn + 1];
                t0 += a0 * x0 + a1 * x1;
                t1 += a2 * x0 + a3 * x1;
            }
            double d0 = dinv[idinv_idx(g, t, idx, 0)], d1 = dinv[idinv_idx(g, t, idx, 1)];
            double d2 = dinv[idinv_idx(g, t, idx, 2)], d3 = dinv[idinv_idx(g, t, idx, 3)];
            double x0 = sm[2 * idx] - (d0 * t0 + d1 * t1);
            double x1 = sm[2 * idx + 1] - (d2 * t0 + d3 * t1);
            sm[2 * idx] = x0; sm[2 * idx + 1] = x1;
            int64_t gc = gi + sy * gj + sz * gk;
            zout[2 * gc] = zs[gc] + x0;        // step 8
            zout[2 * gc + 1] = zp[gc] + x1;
        }
        __syncthreads();
    }
}

static TileGeo geo(const Ctx &c)
{
    TileGeo g;
    g.nx = c.nx; g.ny = c.ny; g.nz = c.nz;
    g.tx = std::min(c.o.tile_x, c.nx); g.ty = std::min(c.o.tile_y, c.ny); g.tz = std::min(c.o.tile_z, c.nz);
    g.ntx = (c.nx + g.tx - 1) / g.tx; g.nty = (c.ny + g.ty - 1) / g.ty; g.ntz = (c.nz + g.tz - 1) / g.tz;
    g.T = g.tx * g.ty * g.tz; g.Tpad = (g.T + 31) / 32 * 32;
    return g;
}

void ilu_setup(Ctx &c, const double *)
{
    TileGeo g = geo(c);
    TSP_REQUIRE(g.tx <= 255 && g.ty <= 255 && g.tz <= 255, TSP_ERR_INVALID_ARG, "ILU tile edge must be <= 255");
    // level-major table of the full tile (same for every tile; clipped tiles skip cells)
    if (c.ilu_tsize != g.T) {
        std::vector<int32_t> cells, lvlptr, posmap(g.T);
        int nlev = g.tx + g.ty + g.tz - 2;
        for (int l = 0; l < nlev; ++l) {
            lvlptr.push_back((int32_t)cells.size());
            for (int k = 0; k < g.tz; ++k)
                for (int j = 0; j < g.ty; ++j)
                    for (int i = 0; i < g.tx; ++i)
                        if (i + j + k == l) {
                            posmap[(k * g.ty + j) * g.tx + i] = (int32_t)cells.size();
                            cells.push_back(i | (j << 8) | (k << 16));
                        }
        }
        lvlptr.push_back((int32_t)cells.size());
        c.ilu_nlev = nlev; c.ilu_tsize = g.T;
        c.ilu_cells.alloc(cells.size()); c.ilu_lvlptr.alloc(lvlptr.size());
        DBuf<int32_t> pm; pm.alloc(posmap.size());
        TSP_CUDA(cudaMemcpyAsync(c.ilu_cells, cells.data(), sizeof(int32_t) * cells.size(), cudaMemcpyHostToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(c.ilu_lvlptr, lvlptr.data(), sizeof(int32_t) * lvlptr.size(), cudaMemcpyHostToDevice, c.s));
        TSP_CUDA(cudaMemcpyAsync(pm, posmap.data(), sizeof(int32_t) * posmap.size(), cudaMemcpyHostToDevice, c.s));
        TSP_CUDA(cudaStreamSynchronize(c.s));
        c.ilu_posmap = std::move(pm);
    }
    c.ntx = g.ntx; c.nty = g.nty; c.ntz = g.ntz;
    c.ntiles = g.ntx * g.nty * g.ntz;
    c.ilu_val.alloc((size_t)c.ntiles * g.Tpad * 28);
    c.ilu_dinv.alloc((size_t)c.ntiles * g.Tpad * 4);
    c.ilu_val.zero(c.s);
    c.ilu_dinv.zero(c.s);
    k_ilu_fill<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(g, c.ff.rp, c.ff.ci, c.ff.v, c.fs, c.ilu_posmap, c.ilu_val);
    c.dcount.zero(c.s);
    k_ilu_factor<<<c.ntiles, 256, 0, c.s>>>(g, c.ilu_lvlptr, c.ilu_nlev, c.ilu_cells, c.ilu_posmap, c.ilu_val, c.ilu_dinv,
                                            c.dcount);
    TSP_CUDA(cudaGetLastError());
    unsigned long long np = 0;
    TSP_CUDA(cudaMemcpyAsync(&np, c.dcount, sizeof(np), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    c.perturbed += (int64_t)np;
    c.launches += 2;
}

void ilu_apply_fused(Ctx &c, const double *yf, const double *zs, const double *zp, double *zf_out)
{
    TileGeo g = geo(c);
    size_t smem = sizeof(double) * 2 * g.Tpad;
    static bool attr_set = false;
    if (!attr_set) {
        TSP_CUDA(cudaFuncSetAttribute(k_ilu_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    prof_begin(c, PK_ILU);
    k_ilu_apply<<<c.ntiles, 256, smem, c.s>>>(g, c.ilu_lvlptr, c.ilu_nlev, c.ilu_cells, c.ilu_posmap, c.ilu_val,
                                              c.ilu_dinv, yf, zs, zp, zf_out);
    prof_end(c, PK_ILU, (28.0 * 8 + 32 + 16 + 16 + 16) * c.Nc);
    c.launches += 1;
    TSP_CUDA(cudaGetLastError());
}

}  // namespace tsp

// p7.cu -- structured storage of the pressure AMG's level 0 (S_pp = A_pp^FS - D_ps D_ss^-1 A_sp^FS):
// on the 7-point TPFA cell stencil the neighbour of every entry follows from the grid, so the level-0 smoother
// kernels of the pressure V-cycle (row a9) read 7 values per row and no column indices (56 B instead of the
// sliced-ELL 7 x 12 B + padding).  Layout [slice of 32 rows][slot 0..6][32], slots in ascending-column order
// (-z, -y, -x, self, +x, +y, +z); absent neighbours (grid boundary) hold 0 and are skipped.  Used when every
// stored entry of the level is one of those 7 neighbours (checked at setup; the generic SELL path otherwise).
// A z-slab's ghost planes come from the fine cell halo (full planes in natural order: rank-1's last plane, then
// rank+1's first plane), read through the GV ghost convention like every other level-0 kernel.
// Summation order = the sliced-ELL kernels' (ascending columns), so results match the generic path bitwise.
#include "tsp_internal.cuh"

namespace tsp {

struct P7Geo {
    int nx, ny, nzl, n, nlo, nhi;   // local slab grid (cells), rows, ghost rows below / above
    int64_t off;                    // first global cell of the slab
    int kz0, nzg;                   // first global plane, global planes
};

__device__ __forceinline__ int64_t p7idx(int i, int s) { return ((int64_t)(i >> 5) * 7 + s) * 32 + (i & 31); }

// neighbour of local row i in slot s: local index, a GV ghost index (>= n), or -1 (outside the domain)
__device__ __forceinline__ int p7_nbr(const P7Geo &g, int i, int s)
{
    const int x = i % g.nx, y = (i / g.nx) % g.ny, z = i / (g.nx * g.ny);
    const int P = g.nx * g.ny;
    switch (s) {
    case 0: if (z > 0) return i - P; return g.kz0 > 0 && g.nlo ? g.n + (i % P) : -1;
    case 1: return y > 0 ? i - g.nx : -1;
    case 2: return x > 0 ? i - 1 : -1;
    case 3: return i;
    case 4: return x + 1 < g.nx ? i + 1 : -1;
    case 5: return y + 1 < g.ny ? i + g.nx : -1;
    default: if (z + 1 < g.nzl) return i + P; return g.kz0 + g.nzl < g.nzg && g.nhi ? g.n + g.nlo + (i % P) : -1;
    }
}

// fill from the level's CSR (global column ids `gcol`); flag bit 0: an entry outside the 7-point stencil
__global__ void k_p7_fill(P7Geo g, const int32_t *__restrict__ rp, const int32_t *__restrict__ gcol, const int32_t *__restrict__ lcol,
                          const double *__restrict__ v, double *__restrict__ val, unsigned *flag)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const int64_t P = (int64_t)g.nx * g.ny, me = g.off + i;
    const int x = i % g.nx, y = (i / g.nx) % g.ny, zg = g.kz0 + i / (g.nx * g.ny);
    const int64_t offs[7] = {-P, -(int64_t)g.nx, -1, 0, 1, g.nx, P};
    const bool in[7] = {zg > 0, y > 0, x > 0, true, x + 1 < g.nx, y + 1 < g.ny, zg + 1 < g.nzg};
    for (int s = 0; s < 7; ++s) val[p7idx(i, s)] = 0.0;
    for (int64_t q = rp[i]; q < rp[i + 1]; ++q) {
        const int64_t d = (gcol ? (int64_t)gcol[q] : (int64_t)lcol[q] + g.off) - me;
        int slot = -1;
        for (int s = 0; s < 7 && slot < 0; ++s) if (in[s] && offs[s] == d) slot = s;   // degenerate grids: the one inside
        if (slot < 0) { atomicOr(flag, 1u); continue; }
        val[p7idx(i, slot)] = v[q];
    }
}

// MODE 1 pre: x = D^-1 b, r = b - A D^-1 b; MODE 2 post: xo = x + D^-1 (b - A x); MODE 3 residual b - A x;
// MODE 4 / 5 fused Chebyshev PRE / STEP (cheb_epi)
template <int MODE, bool D>
__global__ void __launch_bounds__(256) k_p7(P7Geo g, const double *__restrict__ val, GV dinv, GV b, GV x,
                                            double *__restrict__ out1, double *__restrict__ out2, ChebArgs ca)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < 7; ++s) {
        const int j = p7_nbr(g, i, s);
        if (j < 0) continue;
        const double xv = MODE == 1 ? gvld<D>(b, j, 0, 1) * gvld<D>(dinv, j, 0, 1)
                        : MODE == 4 ? ca.sc * (gvld<D>(dinv, j, 0, 1) * gvld<D>(b, j, 0, 1)) : gvld<D>(x, j, 0, 1);
        acc = fma(__ldcs(val + p7idx(i, s)), xv, acc);
    }
    if (MODE == 1) { const double bi = b.own[i]; out1[i] = bi * dinv.own[i]; out2[i] = bi - acc; }
    else if (MODE == 3) out1[i] = b.own[i] - acc;
    else if (MODE == 4 || MODE == 5) cheb_epi<MODE == 4>(i, acc, b.own[i], dinv.own[i], MODE == 5 ? x.own[i] : 0.0, ca, out1);
    else out1[i] = x.own[i] + dinv.own[i] * (b.own[i] - acc);
}

static P7Geo p7_geo(const Ctx &c)
{
    P7Geo g;
    g.nx = c.nx; g.ny = c.ny; g.nzl = c.nz; g.n = c.Nc;
    g.nlo = c.hf.nrecv[0]; g.nhi = c.hf.nrecv[1];
    g.off = c.cell_off; g.kz0 = c.k0; g.nzg = c.nz_glob;
    return g;
}

void p7_build(Ctx &c, const Csr &A)
{
    c.p7_ok = false;
    c.p7_val.release();
    if (getenv("TSP_NO_P7") || A.n != c.Nc) return;
    const P7Geo g = p7_geo(c);
    const int P = c.nx * c.ny;
    unsigned f = 0;
    if (c.comm && !((g.nlo == 0 || g.nlo == P) && (g.nhi == 0 || g.nhi == P))) f = 1u;   // ghosts must be whole planes
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    c.p7_val.alloc((size_t)std::max((c.Nc + 31) / 32, 1) * 7 * 32);
    c.p7_val.zero(c.s);
    if (c.Nc) k_p7_fill<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(g, A.rp, A.gci.p, A.ci, A.v, c.p7_val, flag);
    c.launches += 2;
    unsigned fd = 0;
    TSP_CUDA(cudaMemcpyAsync(&fd, flag.p, sizeof(fd), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    f |= fd;
    if (c.comm) {                                            // one layout on every rank
        std::vector<int64_t> all = host_allgather<int64_t>(c, std::vector<int64_t>{(int64_t)f});
        for (auto a : all) f |= (unsigned)a;
    }
    if (f) { c.p7_val.release(); return; }
    c.p7_ok = true;
}

double p7_bytes(const Ctx &c) { return (double)((c.Nc + 31) / 32) * 32 * 7 * 8; }

// launchers: mode 1 pre, 2 post, 3 residual, 4 / 5 Chebyshev
void p7_launch(Ctx &c, int mode, const GV &dinv, const GV &b, const GV &x, double *o1, double *o2, const ChebArgs &ca)
{
    if (!c.Nc) return;
    const P7Geo g = p7_geo(c);
    const bool D = c.comm != nullptr;
#define P7L(M)                                                                                                    \
    (D ? k_p7<M, true> : k_p7<M, false>)<<<grid_for(c.Nc, 256), 256, 0, c.s>>>(g, c.p7_val, dinv, b, x, o1, o2, ca)
    switch (mode) {
    case 1: P7L(1); break;
    case 2: P7L(2); break;
    case 3: P7L(3); break;
    case 4: P7L(4); break;
    default: P7L(5); break;
    }
#undef P7L
    c.launches++;
}

}  // namespace tsp

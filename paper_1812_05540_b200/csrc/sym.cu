// sym.cu -- structured storage of the 27-point node operators (R-sym): the mechanics block
// A_uu of the operator (row a12, k_op_node) and its SDC part for the level-0 smoother of the mechanics
// V-cycle (row a6).  On the clipped 27-point node stencil the neighbour of every block follows from the
// grid (no column indices), and the block entries that are exactly symmetric over the whole matrix
// (B(i,j)[r][c] == B(j,i)[c][r] for every pair -- for the Q1 elasticity part all of them; the gravity
// term of the momentum balance, d(rho g)/d eps_v, breaks it in the z row and column) are stored for the
// diagonal block and the 13 "upper" neighbours only: a lower neighbour j reads B(i,j) = B(j,i)^T from
// row j's upper slot.  The other entries are stored for all 27 neighbours.  A row sums its own entries first
// (diagonal, then the 13 upper neighbours) and the 13 mirrored lower blocks after them: with the generic
// ascending-column order every mirror load was issued before (or with) the load of the row that owns the
// entry and both missed L2 -- ncu at C5: 22.7 GB of L2 requests, 20.1 GB of DRAM reads for 17.07 GB of
// algorithmic bytes; own-entries-first: 18.1 GB of DRAM reads, 2.87 -> 2.61 ms (level-0 SDC smoother
// 0.97/0.91 -> 0.92/0.79 ms).  L2 eviction-priority hints (evict-last on the own +z entries, evict-first on
// their mirrors, with or without a persisting-L2 carve-out) did not help further (measured).  The sums are
// the generic path's up to the summation order (tests/test_gpu_parity.py).
//
// Local node n of a z-slab: x = n % NX, y = (n / NX) % NY, plane zl = n / (NX NY); global plane
// zg = zn0 + zl.  A neighbour outside [0, Nn) is a ghost: below the slab (rank-1's last node plane,
// ghost index n' + NXY) or above (rank+1's first plane, ghost index nlo + n' - Nn).  Rows of local
// plane 0 whose lower z-plane is a ghost keep the symmetric entries of those 9 blocks explicitly (gl).
#include "tsp_internal.cuh"

namespace tsp {

struct SymGeo {
    int NX, NY, NXY, Nn, nlo, zn0, NZ;   // NZ = global node planes
};

__device__ __forceinline__ int64_t sidx_s(int n, int s, int e, int ks) { return (((int64_t)(n >> 5) * 14 + s) * ks + e) * 32 + (n & 31); }
__device__ __forceinline__ int64_t sidx_f(int n, int c, int e, int kf) { return (((int64_t)(n >> 5) * 27 + c) * kf + e) * 32 + (n & 31); }
__device__ __forceinline__ int64_t sidx_g(int n, int c, int e, int ks) { return (((int64_t)(n >> 5) * 9 + c) * ks + e) * 32 + (n & 31); }

__device__ __forceinline__ bool sym_inside(const SymGeo &g, int x, int y, int zg, int c)
{
    const int dz = c / 9 - 1, dy = (c / 3) % 3 - 1, dx = c % 3 - 1;
    return x + dx >= 0 && x + dx < g.NX && y + dy >= 0 && y + dy < g.NY && zg + dz >= 0 && zg + dz < g.NZ;
}
__device__ __forceinline__ int sym_off(const SymGeo &g, int c) { return (c % 3 - 1) + ((c / 3) % 3 - 1) * g.NX + (c / 9 - 1) * g.NXY; }

// pattern check (bit 31: not the clipped 27-point stencil in ascending order) and the 9-bit mask of block
// entries (r,c) with B(i,j)[r][c] != B(j,i)[c][r] for some owned pair
// bs = 9: the 3x3 blocks of A_uu; bs = 3: SDC values (x,x), (y,y), (z,z) of each block (bit 4e for value e)
__global__ void k_sym_check(SymGeo g, int64_t node_off, const int32_t *__restrict__ rp, const int32_t *__restrict__ gci,
                            const double *__restrict__ v, int bs, unsigned *flag)
{
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= g.Nn) return;
    const int x = n % g.NX, y = (n / g.NX) % g.NY, zg = g.zn0 + n / g.NXY;
    const int64_t gid = node_off + n;
    int64_t q = rp[n];
    const int64_t q1 = rp[n + 1];
    unsigned f = 0;
    for (int c = 0; c < 27; ++c) {
        if (!sym_inside(g, x, y, zg, c)) continue;
        const int64_t col = gid + sym_off(g, c);
        if (q >= q1 || gci[q] != col) { f |= 1u << 31; break; }
        if (c > 13) {                                        // owned upper neighbour: its row holds the mirror
            const int64_t n2 = n + sym_off(g, c);
            if (n2 < g.Nn) {
                bool found = false;
                for (int64_t p = rp[n2]; p < rp[n2 + 1]; ++p)
                    if (gci[p] == gid) {
                        found = true;
                        if (bs == 9) {
                            for (int r = 0; r < 3; ++r)
                                for (int cc = 0; cc < 3; ++cc)
                                    if (v[q * 9 + r * 3 + cc] != v[p * 9 + cc * 3 + r]) f |= 1u << (r * 3 + cc);
                        } else {
                            for (int e = 0; e < 3; ++e)
                                if (v[q * 3 + e] != v[p * 3 + e]) f |= 1u << (4 * e);
                        }
                        break;
                    }
                if (!found) f |= 1u << 31;
            }
        }
        ++q;
    }
    if (q != q1) f |= 1u << 31;
    if (f) atomicOr(flag, f);
}

// fill from `v` (`stride` values per block entry; `src[e]`: the offset of stored value e in an entry)
__global__ void k_sym_fill(SymGeo g, SymMap m, const int32_t *__restrict__ rp, const double *__restrict__ v, int stride, int s0, int s1, int s2,
                           int s3, int s4, int s5, int s6, int s7, int s8, double *__restrict__ vs, double *__restrict__ vf,
                           double *__restrict__ gl)
{
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= g.Nn) return;
    const int src[9] = {s0, s1, s2, s3, s4, s5, s6, s7, s8};
    const int x = n % g.NX, y = (n / g.NX) % g.NY, zg = g.zn0 + n / g.NXY;
    int64_t q = rp[n];
    for (int c = 0; c < 27; ++c) {
        if (!sym_inside(g, x, y, zg, c)) continue;
        const bool ghost_lower = c < 9 && n + sym_off(g, c) < 0;
        for (int e = 0; e < m.bs; ++e) {
            const double val = v[q * stride + src[e]];
            if (m.full[e]) vf[sidx_f(n, c, m.idx[e], m.kf)] = val;
            else if (c >= 13) vs[sidx_s(n, c - 13, m.idx[e], m.ks)] = val;
            else if (ghost_lower) gl[sidx_g(n, c, m.idx[e], m.ks)] = val;
        }
        ++q;
    }
}

// compile-time layout for a mask of non-symmetric 3x3-block entries (ASYM, closed under transposition):
// stored value e of a BS-valued block is block entry be(e); symmetric ones live in val_s, the rest in val_f
template <int ASYM, int BS>
struct SM {
    static constexpr int be(int e) { return BS == 9 ? e : 4 * e; }
    static constexpr bool full(int e) { return (ASYM >> be(e)) & 1; }
    static constexpr int idx(int e)
    {
        int k = 0;
        for (int t = 0; t < e; ++t) k += full(t) == full(e);
        return k;
    }
    static constexpr int ks()
    {
        int k = 0;
        for (int t = 0; t < BS; ++t) k += !full(t);
        return k;
    }
    static constexpr int kf() { return BS - ks(); }
    static constexpr int tr(int e) { return BS == 9 ? (e % 3) * 3 + e / 3 : e; }
};

// block entries of stencil position c of row n (n2 = the neighbour's local index)
template <int ASYM, int BS, int E = 0>
__device__ __forceinline__ void sym_block(const double *__restrict__ vs, const double *__restrict__ vf, const double *__restrict__ gl,
                                          int n, int n2, int c, bool ghost_lower, double (&B)[BS])
{
    if constexpr (E < BS) {
        using M = SM<ASYM, BS>;
        if constexpr (M::full(E)) B[E] = __ldcs(vf + sidx_f(n, c, M::idx(E), M::kf()));
        else if (c >= 13) B[E] = __ldg(vs + sidx_s(n, c - 13, M::idx(E), M::ks()));
        else if (ghost_lower) B[E] = __ldcs(gl + sidx_g(n, c, M::idx(E), M::ks()));
        else B[E] = __ldcs(vs + sidx_s(n2, 13 - c, M::idx(M::tr(E)), M::ks()));   // mirror: upper slot 26 - c, transposed
        sym_block<ASYM, BS, E + 1>(vs, vf, gl, n, n2, c, ghost_lower, B);
    }
}

__device__ __forceinline__ int sym_xidx(const SymGeo &g, int n2)
{
    if (n2 >= 0 && n2 < g.Nn) return n2;
    return n2 < 0 ? g.Nn + n2 + g.NXY : g.Nn + g.nlo + (n2 - g.Nn);
}

// operator node rows: y_u = A_uu x_u (structured) + A_uf x_f (SELL)
template <int ASYM, bool D>
__global__ void __launch_bounds__(256) k_op_node_sym(SymGeo g, const double *__restrict__ vs, const double *__restrict__ vf,
                                                     const double *__restrict__ gl, const int64_t *__restrict__ off_uf,
                                                     const int32_t *__restrict__ col_uf, const double *__restrict__ val_uf, GV xu,
                                                     GV xf, double *__restrict__ yu, Rows R, int cnt)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int n = row_of(R, t);
    const int x = n % g.NX, y = (n / g.NX) % g.NY, zg = g.zn0 + n / g.NXY;
    double a0 = 0, a1 = 0, a2 = 0;
    // the diagonal and the 13 upper blocks (the row's own stored entries) first, then the 13 lower ones, whose
    // symmetric entries are read back from the neighbours' upper slots -- after those rows read them themselves
#pragma unroll
    for (int cc = 0; cc < 27; ++cc) {
        const int c = cc < 14 ? 13 + cc : 26 - cc;
        if (!sym_inside(g, x, y, zg, c)) continue;
        const int n2 = n + sym_off(g, c);
        double B[9];
        sym_block<ASYM, 9>(vs, vf, gl, n, n2, c, c < 9 && n2 < 0, B);
        const int j = sym_xidx(g, n2);
        const double x0 = gvld<D>(xu, j, 0, 3), x1 = gvld<D>(xu, j, 1, 3), x2 = gvld<D>(xu, j, 2, 3);
        a0 = fma(B[0], x0, a0); a0 = fma(B[1], x1, a0); a0 = fma(B[2], x2, a0);
        a1 = fma(B[3], x0, a1); a1 = fma(B[4], x1, a1); a1 = fma(B[5], x2, a1);
        a2 = fma(B[6], x0, a2); a2 = fma(B[7], x1, a2); a2 = fma(B[8], x2, a2);
    }
    const int s = n >> 5, lane = n & 31;
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
    yu[3 * (int64_t)n] = a0; yu[3 * (int64_t)n + 1] = a1; yu[3 * (int64_t)n + 2] = a2;
}

// level-0 SDC smoother (3 scalar components on one node graph; pre-smoothing from zero = amg.cu k_dscale +
// MODE 3), MODE 2 post: xo = x + D^-1 (b - A x); MODE 3 residual (Gauss-Seidel smoother): out1 = b - A x
template <int ASYM, int MODE, bool D>
__global__ void __launch_bounds__(256) k_vc_sym(SymGeo g, const double *__restrict__ vs, const double *__restrict__ vf,
                                                const double *__restrict__ gl, GV dinv, GV b, GV xin, double *__restrict__ out1,
                                                double *__restrict__ out2, ChebArgs ca)
{
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= g.Nn) return;
    const int x = n % g.NX, y = (n / g.NX) % g.NY, zg = g.zn0 + n / g.NXY;
    double acc[3] = {0, 0, 0};
#pragma unroll
    for (int ck = 0; ck < 27; ++ck) {
        const int c = ck < 14 ? 13 + ck : 26 - ck;   // own entries first (see k_op_node_sym)
        if (!sym_inside(g, x, y, zg, c)) continue;
        const int n2 = n + sym_off(g, c);
        double B[3];
        sym_block<ASYM, 3>(vs, vf, gl, n, n2, c, c < 9 && n2 < 0, B);
        const int j = sym_xidx(g, n2);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            const double xv = MODE == 4 ? ca.sc * (gvld<D>(dinv, j, cc, 3) * gvld<D>(b, j, cc, 3)) : gvld<D>(xin, j, cc, 3);
            acc[cc] = fma(B[cc], xv, acc[cc]);
        }
    }
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const int64_t t = 3 * (int64_t)n + cc;
        if (MODE == 3) {
            out1[t] = b.own[t] - acc[cc];
        } else if (MODE == 4 || MODE == 5) {
            cheb_epi<MODE == 4>(t, acc[cc], b.own[t], dinv.own[t], MODE == 5 ? xin.own[t] : 0.0, ca, out1);
        } else {
            out1[t] = xin.own[t] + dinv.own[t] * (b.own[t] - acc[cc]);
        }
    }
}

// layouts instantiated: a fully symmetric block, and the poromechanics one (z row and column not symmetric)
constexpr unsigned kAsymZ = (1u << 2) | (1u << 5) | (1u << 6) | (1u << 7) | (1u << 8);
static bool sym_supported(unsigned asym) { return asym == 0 || asym == kAsymZ; }

static SymGeo sym_geo(const Ctx &c)
{
    SymGeo g;
    g.NX = c.nx + 1; g.NY = c.ny + 1; g.NXY = g.NX * g.NY; g.Nn = c.Nn;
    g.nlo = c.hu.nrecv[0];
    g.zn0 = (int)(c.node_off / g.NXY);
    g.NZ = c.nz_glob + 1;
    return g;
}

// `src[e]`: the 3x3-block entry behind stored value e; `asym`: 9-bit mask of the non-symmetric block entries;
// values read from `v` (`stride` per block entry, stored value e at offset rd[e]; default: A_uu's blocks)
static void sym_fill_one(Ctx &c, const SymGeo &g, int bs, const int *src, unsigned asym, Sym27 &S,
                         const double *v = nullptr, int stride = 9, const int *rd = nullptr)
{
    SymMap &m = S.m;
    m.bs = bs; m.ks = m.kf = 0;
    for (int e = 0; e < bs; ++e) {
        const int be = src[e], r = be / 3, cc = be % 3;
        m.full[e] = (asym >> be) & 1u;
        m.idx[e] = m.full[e] ? m.kf++ : m.ks++;
        m.tr[e] = e;
        if (bs == 9) m.tr[e] = cc * 3 + r;
    }
    const int nsl = (c.Nn + 31) / 32, nsl0 = g.nlo ? (g.NXY + 31) / 32 : 0;
    S.val_s.alloc((size_t)std::max(nsl, 1) * 14 * std::max(m.ks, 1) * 32); S.val_s.zero(c.s);
    S.val_f.alloc((size_t)std::max(nsl, 1) * 27 * std::max(m.kf, 1) * 32); S.val_f.zero(c.s);
    S.gl.alloc((size_t)std::max(nsl0, 1) * 9 * std::max(m.ks, 1) * 32); S.gl.zero(c.s);
    int s9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int e = 0; e < bs; ++e) s9[e] = rd ? rd[e] : src[e];
    if (!v) v = c.uu.v;
    if (c.Nn) k_sym_fill<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(g, m, c.uu.rp, v, stride, s9[0], s9[1], s9[2], s9[3], s9[4], s9[5], s9[6],
                                                              s9[7], s9[8], S.val_s, S.val_f, S.gl);
    c.launches++;
    S.ok = true;
}

void sym_build(Ctx &c)
{
    c.sym_uu.ok = c.sym_sdc.ok = false;
    if (getenv("TSP_NO_SYM")) return;                        // generic SELL path (tests compare both)
    const SymGeo g = sym_geo(c);
    // the halo of a slab must be whole node planes (the clipped 27-point stencil guarantees it)
    unsigned f = 0;
    if (c.comm && !((g.nlo == 0 || g.nlo == g.NXY) && (c.hu.nrecv[1] == 0 || c.hu.nrecv[1] == g.NXY))) f = 1u << 31;
    const int32_t *gci = c.uu.gci.p ? c.uu.gci.p : c.uu.ci.p;
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    if (c.Nn) k_sym_check<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(g, c.node_off, c.uu.rp, gci, c.uu.v, 9, flag);
    c.launches++;
    unsigned fd = 0;
    TSP_CUDA(cudaMemcpyAsync(&fd, flag.p, sizeof(fd), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    f |= fd;
    if (c.comm) {                                            // every rank takes the same path and layout (P-invariance)
        std::vector<int64_t> all = host_allgather<int64_t>(c, std::vector<int64_t>{(int64_t)f});
        for (auto a : all) f |= (unsigned)a;
    }
    if (f >> 31) return;
    // close the mask under transposition: a lower block's entry (r,c) is read from the mirror's (c,r)
    unsigned asym = f & 0x1ffu;
    for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc)
            if ((asym >> (r * 3 + cc)) & 1u) asym |= 1u << (cc * 3 + r);
    const int id9[9] = {0, 1, 2, 3, 4, 5, 6, 7, 8}, sdc[3] = {0, 4, 8};
    if (!sym_supported(asym)) return;
    c.sym_asym = asym;
    sym_fill_one(c, g, 9, id9, asym, c.sym_uu);
    sym_fill_one(c, g, 3, sdc, asym, c.sym_sdc);
}

// mask of non-symmetric entries of `v` (bs 9: A_uu blocks, bs 3: SDC values), bit 31 = not the 27-point
// stencil; the same on every rank
static unsigned sym_mask(Ctx &c, const SymGeo &g, const double *v, int bs)
{
    const int32_t *gci = c.uu.gci.p ? c.uu.gci.p : c.uu.ci.p;
    DBuf<unsigned> flag; flag.alloc(1); flag.zero(c.s);
    if (c.Nn) k_sym_check<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(g, c.node_off, c.uu.rp, gci, v, bs, flag);
    c.launches++;
    unsigned f = 0;
    TSP_CUDA(cudaMemcpyAsync(&f, flag.p, sizeof(f), cudaMemcpyDeviceToHost, c.s));
    TSP_CUDA(cudaStreamSynchronize(c.s));
    if (c.comm) {
        std::vector<int64_t> all = host_allgather<int64_t>(c, std::vector<int64_t>{(int64_t)f});
        for (auto a : all) f |= (unsigned)a;
    }
    return f;
}

// tsp_update_values: new A_uu values (c.uu.v) on the same pattern.  The structured operator keeps its layout
// when the new values are symmetric wherever the layout assumes it (their mask is inside sym_asym); otherwise
// the operator falls back to the generic SELL copy.  Returns whether the structured copy is in use.
bool sym_refill_uu(Ctx &c)
{
    if (!c.sym_uu.ok) return false;
    const SymGeo g = sym_geo(c);
    const unsigned f = sym_mask(c, g, c.uu.v, 9);
    if ((f >> 31) || (f & 0x1ffu & ~c.sym_asym)) {
        c.sym_uu.ok = false;
        c.sym_uu.val_s.release(); c.sym_uu.val_f.release(); c.sym_uu.gl.release();
        return false;
    }
    const int id9[9] = {0, 1, 2, 3, 4, 5, 6, 7, 8};
    sym_fill_one(c, g, 9, id9, c.sym_asym, c.sym_uu);
    return true;
}

// TSP_SETUP_MECH after tsp_update_values: the level-0 SDC smoother copy from the new SDC values (c.uu_sdc)
void sym_refill_sdc(Ctx &c)
{
    if (!c.sym_sdc.ok) return;
    const SymGeo g = sym_geo(c);
    const unsigned f = sym_mask(c, g, c.uu_sdc, 3);
    if ((f >> 31) || (f & 0x1ffu & ~c.sym_asym)) {
        c.sym_sdc.ok = false;
        c.sym_sdc.val_s.release(); c.sym_sdc.val_f.release(); c.sym_sdc.gl.release();
        return;
    }
    const int sdc[3] = {0, 4, 8}, rd[3] = {0, 1, 2};
    sym_fill_one(c, g, 3, sdc, c.sym_asym, c.sym_sdc, c.uu_sdc, 3, rd);
}

// ---- launchers used by apply.cu (operator) and amg.cu (level-0 mechanics smoother); the layouts are
// instantiated for a fully symmetric block and for the poromechanics one (z row and column not symmetric)

bool sym_op_node(Ctx &c, const GV &gu, const GV &gf, double *yu, Rows R, int cnt)
{
    if (!c.sym_uu.ok) return false;
    const SymGeo g = sym_geo(c);
    const Sym27 &S = c.sym_uu;
#define OPS(A)                                                                                                    \
    (c.comm ? k_op_node_sym<A, true> : k_op_node_sym<A, false>)<<<grid_for(cnt, 256), 256, 0, c.s>>>(                      \
        g, S.val_s, S.val_f, S.gl, c.s_uf.off, c.s_uf.col, c.s_uf.val, gu, gf, yu, R, cnt)
    if (cnt) {
        if (c.sym_asym == 0) OPS(0u);
        else OPS(kAsymZ);
    }
#undef OPS
    return true;
}
bool sym_vcycle_post(Ctx &c, int n, const double *dinv, const double *b, const GV &x, double *xo)
{
    if (!c.sym_sdc.ok || n != c.Nn) return false;
    const SymGeo g = sym_geo(c);
    const Sym27 &S = c.sym_sdc;
#define VCS(A)                                                                                                    \
    (c.comm ? k_vc_sym<A, 2, true> : k_vc_sym<A, 2, false>)<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(                        \
        g, S.val_s, S.val_f, S.gl, gv(dinv, n), gv(b, n), x, xo, nullptr, ChebArgs{})
    if (n) {
        if (c.sym_asym == 0) VCS(0u);
        else VCS(kAsymZ);
    }
#undef VCS
    return true;
}
bool sym_vcycle_cheb(Ctx &c, int n, bool pre, const GV &dinv, const GV &b, const GV &x, const ChebArgs &a, double *xo)
{
    if (!c.sym_sdc.ok || n != c.Nn) return false;
    const SymGeo g = sym_geo(c);
    const Sym27 &S = c.sym_sdc;
#define VCS(A, M)                                                                                                 \
    (c.comm ? k_vc_sym<A, M, true> : k_vc_sym<A, M, false>)<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(                        \
        g, S.val_s, S.val_f, S.gl, dinv, b, x, xo, nullptr, a)
    if (n) {
        if (c.sym_asym == 0) { if (pre) VCS(0u, 4); else VCS(0u, 5); }
        else { if (pre) VCS(kAsymZ, 4); else VCS(kAsymZ, 5); }
    }
#undef VCS
    return true;
}
bool sym_vcycle_resid(Ctx &c, int n, const double *b, const GV &x, double *r)
{
    if (!c.sym_sdc.ok || n != c.Nn) return false;
    const SymGeo g = sym_geo(c);
    const Sym27 &S = c.sym_sdc;
#define VCS(A)                                                                                                    \
    (c.comm ? k_vc_sym<A, 3, true> : k_vc_sym<A, 3, false>)<<<grid_for(c.Nn, 256), 256, 0, c.s>>>(                        \
        g, S.val_s, S.val_f, S.gl, gv(nullptr, 0), gv(b, n), x, r, nullptr, ChebArgs{})
    if (n) {
        if (c.sym_asym == 0) VCS(0u);
        else VCS(kAsymZ);
    }
#undef VCS
    return true;
}
// algorithmic bytes of one stream over the structure (each stored value once)
double sym_bytes(const Ctx &c, int bs)
{
    const Sym27 &S = bs == 9 ? c.sym_uu : c.sym_sdc;
    const double nsl = (c.Nn + 31) / 32;
    return nsl * 32 * 8.0 * (14.0 * S.m.ks + 27.0 * S.m.kf);
}

}  // namespace tsp

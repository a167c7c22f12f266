/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Parity pinned by
 * tests/test_oracle_*.py; functions without a pin say so in DESIGN.md.
 *
 * Plain sequential C, -ffp-contract=off, IEEE double (OMP_ROWS below: an optional
 * timing-only build runs row-independent loops on all host cores).  Written in the paper's
 * order and notation:
 *   a1 fixed stress          eq:Schur_1_FS P:406-417, eq:FS_Dps_Dpp P:418-437
 *   a2 SDC
 *   a3 quasi-IMPES / S_pp
 *   a4 AMG setup             P:513-519, P:599 (method: DESIGN.md R-amg*)
 *   a5 tile ILU(0)           P:606-612 (R-ilu)
 *   a6-a11 Algorithm 1       alg:apply_M_inv
 *   a12 operator             eq:jac_system P:283-298
 *   a14 FGMRES(m), MGS       P:302-307 (R-krylov, SURVEY O-4)
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* OMP_ROWS marks loops whose iterations are independent rows (nothing is summed across them).  The plain
 * liboracle.so ignores it; liboracle_omp.so (-fopenmp, Makefile; loaded when ORACLE_OMP=1, the timing-only
 * "oracle-omp" row of tools/config_sweep.py) runs those loops on all host cores with bitwise the same
 * results: every dot product, Gauss-Seidel / ILU sweep and setup step stays sequential. */
#ifdef _OPENMP
#define OMP_ROWS _Pragma("omp parallel for schedule(static)")
#else
#define OMP_ROWS
#endif

static void *xmalloc(size_t n) { void *p = malloc(n ? n : 1); if (!p) { fprintf(stderr, "oracle: OOM\n"); abort(); } return p; }
static void *xcalloc(size_t n, size_t s) { void *p = calloc(n ? n : 1, s ? s : 1); if (!p) { fprintf(stderr, "oracle: OOM\n"); abort(); } return p; }
static double now_s(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }

/* ======================================================================
 * multi-component scalar CSR: nc value sets sharing one pattern
 * (nc = 3 for the SDC mechanics hierarchy: A_xx, A_yy, A_zz)
 * ==================================================================== */
typedef struct { int n, m, nc; int32_t *rp, *ci; double *v[3]; } mcsr;

static void mcsr_alloc(mcsr *A, int n, int m, int nc, int64_t nnz)
{
    A->n = n; A->m = m; A->nc = nc;
    A->rp = (int32_t *)xcalloc(n + 1, sizeof(int32_t));
    A->ci = (int32_t *)xmalloc(sizeof(int32_t) * nnz);
    for (int c = 0; c < 3; ++c) A->v[c] = c < nc ? (double *)xcalloc(nnz, sizeof(double)) : NULL;
}
static void mcsr_free(mcsr *A)
{
    free(A->rp); free(A->ci);
    for (int c = 0; c < 3; ++c) free(A->v[c]);
    memset(A, 0, sizeof(*A));
}
static int64_t mnnz(const mcsr *A) { return A->rp[A->n]; }

/* y = A_c x (one component) */
static void spmv(const mcsr *A, int c, const double *x, double *y)
{
    OMP_ROWS
    for (int i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) s += A->v[c][q] * x[A->ci[q]];
        y[i] = s;
    }
}
/* y = y - A_c x */
static void spmv_sub(const mcsr *A, int c, const double *x, double *y)
{
    OMP_ROWS
    for (int i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) s += A->v[c][q] * x[A->ci[q]];
        y[i] -= s;
    }
}
static int64_t find_col(const mcsr *A, int i, int j)
{
    for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) if (A->ci[q] == j) return q;
    return -1;
}

/* ======================================================================
 * dense LU with partial pivoting (textbook; pivot = first maximal |a| in the
 * column, i.e. lowest row index on ties -- R-coarse).  Row-major n x n.
 * ==================================================================== */
static int dense_lu(int n, double *a, int *piv, int64_t *npert)
{
    double scale = 0.0;
    for (int64_t q = 0; q < (int64_t)n * n; ++q) if (fabs(a[q]) > scale) scale = fabs(a[q]);
    if (scale == 0.0) scale = 1.0;
    for (int k = 0; k < n; ++k) {
        int p = k; double best = fabs(a[(int64_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) if (fabs(a[(int64_t)i * n + k]) > best) { best = fabs(a[(int64_t)i * n + k]); p = i; }
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) { double t = a[(int64_t)k * n + j]; a[(int64_t)k * n + j] = a[(int64_t)p * n + j]; a[(int64_t)p * n + j] = t; }
        if (a[(int64_t)k * n + k] == 0.0) { a[(int64_t)k * n + k] = 1e-12 * scale; if (npert) ++*npert; }
        double d = a[(int64_t)k * n + k];
        for (int i = k + 1; i < n; ++i) {
            double l = a[(int64_t)i * n + k] / d;
            a[(int64_t)i * n + k] = l;
            if (l != 0.0)
                for (int j = k + 1; j < n; ++j) a[(int64_t)i * n + j] -= l * a[(int64_t)k * n + j];
        }
    }
    return 0;
}
static void dense_lu_solve(int n, const double *lu, const int *piv, const double *b, double *x)
{
    double *y = (double *)xmalloc(sizeof(double) * n);
    memcpy(y, b, sizeof(double) * n);
    for (int k = 0; k < n; ++k) if (piv[k] != k) { double t = y[k]; y[k] = y[piv[k]]; y[piv[k]] = t; }
    for (int i = 0; i < n; ++i) { double s = y[i]; for (int j = 0; j < i; ++j) s -= lu[(int64_t)i * n + j] * y[j]; y[i] = s; }
    for (int i = n - 1; i >= 0; --i) { double s = y[i]; for (int j = i + 1; j < n; ++j) s -= lu[(int64_t)i * n + j] * y[j]; y[i] = s / lu[(int64_t)i * n + i]; }
    memcpy(x, y, sizeof(double) * n);
    free(y);
}

/* ======================================================================
 * a4: aggregation AMG (R-amg: smoothed aggregation, Galerkin R = P^T, one
 * V(1,1) l1-Jacobi cycle; substitutes the paper's Hypre BoomerAMG, P:711,
 * per BASELINE.json north_star "deterministic aggregation plus Galerkin RAP")
 * ==================================================================== */
enum { ST_ISOLATED = -1, ST_UNDECIDED = 0, ST_ROOT = 1, ST_OUT = 2 };

typedef struct {
    mcsr A; int32_t *zb; double *dl1[3];
    int coarsest;
    int nagg; int32_t *agg;       /* aggregate id per row, -1 = not aggregated */
    int32_t *st, *ph1;            /* MIS(2) state and phase-1 aggregate per row (kept for the pins) */
    mcsr P, R;
    double *lu[3]; int *piv[3];
    double omega[3];
    int32_t *color; int ncolor;   /* GS smoother (R-gs): colour of each row, number of colours (max over blocks) */
    int gs_block;                 /* 0: multicolour over the level (given colouring); B: hybrid, blocks of B rows */
    uint8_t *E;                   /* symmetrised strength flags per stored entry (kept for the frozen refresh) */
    double *dh[3];                /* hybrid l1 diagonal per component */
} olevel;

typedef struct {
    int nl, nc;
    olevel L[16];
    int64_t fallbacks, perturbed;
    orc_opts o;
} ohier;

/* MurmurHash3 fmix32 finaliser: the fixed priority hash of R-mis2 */
static uint32_t fmix32(uint32_t x)
{
    x ^= x >> 16; x *= 0x85ebca6bU; x ^= x >> 13; x *= 0xc2b2ae35U; x ^= x >> 16;
    return x;
}

/* strength measure of entry q: sum_c |a^c_q|, c ascending (R-strength) */
static double meas(const mcsr *A, int64_t q)
{
    double s = 0.0;
    for (int c = 0; c < A->nc; ++c) s = s + fabs(A->v[c][q]);
    return s;
}

/* Strength (R-strength): S_ij iff j != i, zb(i) == zb(j), m_i > 0 and
 * meas(i,j) >= theta * m_i with m_i = max_{k != i} meas(i,k).  Symmetrised:
 * edge(i,j) iff S_ij or S_ji.  Requires a structurally symmetric pattern. */
static int strength(const mcsr *A, const int32_t *zb, double theta, uint8_t *E)
{
    int n = A->n;
    uint8_t *S = (uint8_t *)xcalloc(mnnz(A) + 1, 1);
    for (int i = 0; i < n; ++i) {
        double m = 0.0;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) if (A->ci[q] != i) { double t = meas(A, q); if (t > m) m = t; }
        double thr = theta * m;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
            int j = A->ci[q];
            S[q] = (j != i && m > 0.0 && zb[i] == zb[j] && meas(A, q) >= thr) ? 1 : 0;
        }
    }
    for (int i = 0; i < n; ++i)
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
            int j = A->ci[q];
            if (j == i) { E[q] = 0; continue; }
            int64_t qt = find_col(A, j, i);
            if (qt < 0) { free(S); return -1; }   /* pattern not structurally symmetric */
            E[q] = (S[q] || S[qt]) ? 1 : 0;
        }
    free(S);
    return 0;
}

/* adjacency lists of the symmetrised strength graph */
static void graph_from_E(const mcsr *A, const uint8_t *E, int32_t **grp, int32_t **gci)
{
    int n = A->n;
    int32_t *rp = (int32_t *)xcalloc(n + 1, sizeof(int32_t));
    for (int i = 0; i < n; ++i) { int c = 0; for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) c += E[q]; rp[i + 1] = rp[i] + c; }
    int32_t *ci = (int32_t *)xmalloc(sizeof(int32_t) * (rp[n] + 1));
    for (int i = 0; i < n; ++i) { int64_t t = rp[i]; for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) if (E[q]) ci[t++] = A->ci[q]; }
    *grp = rp; *gci = ci;
}

typedef struct { uint32_t h; int32_t i; } prio_t;
static int prio_desc(const void *a, const void *b)
{
    const prio_t *x = (const prio_t *)a, *y = (const prio_t *)b;
    if (x->h != y->h) return x->h < y->h ? 1 : -1;
    if (x->i != y->i) return x->i < y->i ? 1 : -1;
    return 0;
}

/* MIS(2) = maximal independent set of the distance-2 graph (R-mis2).
 * Definition used by the oracle: sequential greedy in descending priority
 * pi(i) = (hash(i), i).  Nodes with no edge are ISOLATED. */
static void mis2_greedy(int n, const int32_t *rp, const int32_t *ci, const uint32_t *hash, int32_t *st)
{
    prio_t *p = (prio_t *)xmalloc(sizeof(prio_t) * (n + 1));
    int np = 0;
    for (int i = 0; i < n; ++i) {
        st[i] = (rp[i + 1] > rp[i]) ? ST_UNDECIDED : ST_ISOLATED;
        if (st[i] == ST_UNDECIDED) { p[np].h = hash[i]; p[np].i = i; ++np; }
    }
    qsort(p, np, sizeof(prio_t), prio_desc);
    for (int t = 0; t < np; ++t) {
        int v = p[t].i;
        if (st[v] != ST_UNDECIDED) continue;
        st[v] = ST_ROOT;
        for (int64_t q = rp[v]; q < rp[v + 1]; ++q) {
            int u = ci[q];
            if (st[u] == ST_UNDECIDED) st[u] = ST_OUT;
            for (int64_t q2 = rp[u]; q2 < rp[u + 1]; ++q2) if (st[ci[q2]] == ST_UNDECIDED) st[ci[q2]] = ST_OUT;
        }
    }
    free(p);
}

/* Independent second implementation (R-mis2): rounds of
 * "undecided v is a root iff its priority is the maximum over the undecided
 * nodes of its closed distance-2 neighbourhood", then every undecided node
 * within distance 2 of a new root is OUT.  Used only to pin the greedy. */
static int mis2_rounds(int n, const int32_t *rp, const int32_t *ci, const uint32_t *hash, int32_t *st)
{
    uint64_t *t1 = (uint64_t *)xmalloc(sizeof(uint64_t) * (n + 1));
    uint8_t *newr = (uint8_t *)xmalloc(n + 1), *near1 = (uint8_t *)xmalloc(n + 1);
    for (int i = 0; i < n; ++i) st[i] = (rp[i + 1] > rp[i]) ? ST_UNDECIDED : ST_ISOLATED;
#define PRIO(i) ((((uint64_t)hash[i]) << 32) | (uint64_t)(uint32_t)(i))
    int rounds = 0;
    for (;;) {
        int any = 0;
        for (int i = 0; i < n; ++i) if (st[i] == ST_UNDECIDED) { any = 1; break; }
        if (!any) break;
        ++rounds;
        for (int x = 0; x < n; ++x) {
            uint64_t m = 0; int has = 0;
            if (st[x] == ST_UNDECIDED) { m = PRIO(x); has = 1; }
            for (int64_t q = rp[x]; q < rp[x + 1]; ++q) { int u = ci[q]; if (st[u] == ST_UNDECIDED && (!has || PRIO(u) > m)) { m = PRIO(u); has = 1; } }
            t1[x] = has ? m + 1 : 0;   /* +1 so that 0 means "none" */
        }
        for (int v = 0; v < n; ++v) {
            newr[v] = 0;
            if (st[v] != ST_UNDECIDED) continue;
            uint64_t m = t1[v];
            for (int64_t q = rp[v]; q < rp[v + 1]; ++q) if (t1[ci[q]] > m) m = t1[ci[q]];
            if (m == PRIO(v) + 1) newr[v] = 1;
        }
        for (int v = 0; v < n; ++v) if (newr[v]) st[v] = ST_ROOT;
        for (int x = 0; x < n; ++x) {
            near1[x] = newr[x];
            for (int64_t q = rp[x]; q < rp[x + 1]; ++q) if (newr[ci[q]]) near1[x] = 1;
        }
        for (int v = 0; v < n; ++v) {
            if (st[v] != ST_UNDECIDED) continue;
            int hit = near1[v];
            for (int64_t q = rp[v]; q < rp[v + 1] && !hit; ++q) if (near1[ci[q]]) hit = 1;
            if (hit) st[v] = ST_OUT;
        }
    }
#undef PRIO
    free(t1); free(newr); free(near1);
    return rounds;
}

int orc_mis2(int n, const int32_t *rp, const int32_t *ci, const uint32_t *hash, int rounds_variant,
             int32_t *state_out, int *nrounds)
{
    if (rounds_variant) { int r = mis2_rounds(n, rp, ci, hash, state_out); if (nrounds) *nrounds = r; }
    else { mis2_greedy(n, rp, ci, hash, state_out); if (nrounds) *nrounds = 0; }
    return 0;
}

/* Aggregates (R-agg): roots numbered by ascending node id; phase 1 = root and
 * its strong neighbours; phase 2 = each remaining non-isolated node joins the
 * phase-1 aggregate of its strong neighbour of maximal measure, ties to the
 * smallest aggregate id. */
static int aggregate(const mcsr *A, const uint8_t *E, const int32_t *st, int32_t *agg, int32_t *ph1_out)
{
    int n = A->n, nagg = 0;
    int32_t *rid = (int32_t *)xmalloc(sizeof(int32_t) * (n + 1));
    for (int i = 0; i < n; ++i) { rid[i] = (st[i] == ST_ROOT) ? nagg++ : -1; agg[i] = -1; }
    for (int r = 0; r < n; ++r) {
        if (st[r] != ST_ROOT) continue;
        agg[r] = rid[r];
        for (int64_t q = A->rp[r]; q < A->rp[r + 1]; ++q) if (E[q]) agg[A->ci[q]] = rid[r];
    }
    int32_t *ph1 = (int32_t *)xmalloc(sizeof(int32_t) * (n + 1));
    memcpy(ph1, agg, sizeof(int32_t) * n);
    for (int v = 0; v < n; ++v) {
        if (st[v] == ST_ISOLATED || ph1[v] >= 0) continue;
        int best = -1; double bw = 0.0;
        for (int64_t q = A->rp[v]; q < A->rp[v + 1]; ++q) {
            if (!E[q]) continue;
            int a = ph1[A->ci[q]];
            if (a < 0) continue;
            double w = meas(A, q);
            if (best < 0 || w > bw || (w == bw && a < best)) { best = a; bw = w; }
        }
        agg[v] = best;
    }
    if (ph1_out) memcpy(ph1_out, ph1, sizeof(int32_t) * n);
    free(rid); free(ph1);
    return nagg;
}

static int cmp_i32(const void *a, const void *b) { int32_t x = *(const int32_t *)a, y = *(const int32_t *)b; return (x > y) - (x < y); }

/* Smoothed prolongator (R-prolong), per component c:
 *   filtered A^F: strong entries kept, weak entries lumped into the diagonal
 *     d_i = a_ii + sum_{weak j, ascending} a_ij
 *   rho_c = max_i (sum_j |a^F_ij|) / |d_i|,  omega_c = 4 / (3 rho_c)
 *   P_iJ = [J == agg(i)] - (omega_c / d_i) * sum_{j in {i} U strong(i), agg(j) = J, ascending} a^F_ij
 * (unnormalised tentative prolongator with unit entries). */
static void build_P(olevel *L, const uint8_t *E)
{
    const mcsr *A = &L->A;
    int n = A->n, nc = A->nc;
    double *d[3];
    for (int c = 0; c < nc; ++c) {
        d[c] = (double *)xmalloc(sizeof(double) * (n + 1));
        double rho = 0.0;
        for (int i = 0; i < n; ++i) {
            int64_t qd = find_col(A, i, i);
            double di = qd >= 0 ? A->v[c][qd] : 0.0;
            for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q)
                if (A->ci[q] != i && !E[q]) di = di + A->v[c][q];
            d[c][i] = di;
            if (di == 0.0) continue;
            double s = 0.0;
            for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                double a = (A->ci[q] == i) ? di : (E[q] ? A->v[c][q] : 0.0);
                s = s + fabs(a);
            }
            double r = s / fabs(di);
            if (r > rho) rho = r;
        }
        L->omega[c] = rho > 0.0 ? 4.0 / (3.0 * rho) : 0.0;
    }
    /* pattern: sorted unique aggregates of {i} U strong(i) */
    int32_t *rp = (int32_t *)xcalloc(n + 1, sizeof(int32_t));
    int32_t *tmp = (int32_t *)xmalloc(sizeof(int32_t) * 4096);
    int64_t cap = 16 * (int64_t)n + 16, nz = 0;
    int32_t *ci = (int32_t *)xmalloc(sizeof(int32_t) * cap);
    for (int i = 0; i < n; ++i) {
        int cnt = 0;
        if (L->agg[i] >= 0)
            for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                int j = A->ci[q];
                if ((j == i || E[q]) && L->agg[j] >= 0) tmp[cnt++] = L->agg[j];
            }
        qsort(tmp, cnt, sizeof(int32_t), cmp_i32);
        int u = 0;
        for (int t = 0; t < cnt; ++t) if (u == 0 || tmp[t] != tmp[u - 1]) tmp[u++] = tmp[t];
        if (nz + u > cap) { cap = 2 * (nz + u); ci = (int32_t *)realloc(ci, sizeof(int32_t) * cap); }
        memcpy(ci + nz, tmp, sizeof(int32_t) * u);
        nz += u; rp[i + 1] = (int32_t)nz;
    }
    mcsr *P = &L->P;
    mcsr_alloc(P, n, L->nagg, nc, nz);
    memcpy(P->rp, rp, sizeof(int32_t) * (n + 1));
    memcpy(P->ci, ci, sizeof(int32_t) * (nz ? nz : 1));
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < n; ++i) {
            double di = d[c][i];
            double w = (di != 0.0) ? L->omega[c] / di : 0.0;
            for (int64_t p = P->rp[i]; p < P->rp[i + 1]; ++p) {
                int J = P->ci[p];
                double s = 0.0;
                for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                    int j = A->ci[q];
                    if (!((j == i) || E[q]) || L->agg[j] != J) continue;
                    double a = (j == i) ? di : A->v[c][q];
                    s = s + a;
                }
                double delta = (J == L->agg[i]) ? 1.0 : 0.0;
                P->v[c][p] = delta - w * s;
            }
        }
    for (int c = 0; c < nc; ++c) free(d[c]);
    free(rp); free(tmp); free(ci);
}

/* R = P^T, entries of each row in ascending fine index */
static void transpose(const mcsr *P, mcsr *R)
{
    int n = P->n, m = P->m, nc = P->nc;
    int64_t nz = mnnz(P);
    mcsr_alloc(R, m, n, nc, nz);
    for (int64_t q = 0; q < nz; ++q) R->rp[P->ci[q] + 1]++;
    for (int J = 0; J < m; ++J) R->rp[J + 1] += R->rp[J];
    int32_t *fill = (int32_t *)xmalloc(sizeof(int32_t) * (m + 1));
    memcpy(fill, R->rp, sizeof(int32_t) * m);
    for (int i = 0; i < n; ++i)
        for (int64_t q = P->rp[i]; q < P->rp[i + 1]; ++q) {
            int64_t t = fill[P->ci[q]]++;
            R->ci[t] = i;
            for (int c = 0; c < nc; ++c) R->v[c][t] = P->v[c][q];
        }
    free(fill);
}

/* C = A B with canonical summation (R-rap): C_ik is the left fold,
 * starting from 0.0, over the entries of A's row i in ascending column order
 * of a_ij * b_jk.  Pattern: union, ascending. */
static void spgemm(const mcsr *A, const mcsr *B, mcsr *Cm)
{
    int n = A->n, m = B->m, nc = A->nc;
    int32_t *mark = (int32_t *)xmalloc(sizeof(int32_t) * (m + 1));
    for (int k = 0; k < m; ++k) mark[k] = -1;
    int32_t *rp = (int32_t *)xcalloc(n + 1, sizeof(int32_t));
    for (int i = 0; i < n; ++i) {
        int cnt = 0;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
            int j = A->ci[q];
            for (int64_t p = B->rp[j]; p < B->rp[j + 1]; ++p)
                if (mark[B->ci[p]] != i) { mark[B->ci[p]] = i; ++cnt; }
        }
        rp[i + 1] = rp[i] + cnt;
    }
    mcsr_alloc(Cm, n, m, nc, rp[n]);
    memcpy(Cm->rp, rp, sizeof(int32_t) * (n + 1));
    for (int k = 0; k < m; ++k) mark[k] = -1;
    double *acc[3];
    for (int c = 0; c < nc; ++c) acc[c] = (double *)xcalloc(m + 1, sizeof(double));
    for (int i = 0; i < n; ++i) {
        int64_t t = Cm->rp[i];
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
            int j = A->ci[q];
            for (int64_t p = B->rp[j]; p < B->rp[j + 1]; ++p) {
                int k = B->ci[p];
                if (mark[k] != i) { mark[k] = i; Cm->ci[t++] = k; for (int c = 0; c < nc; ++c) acc[c][k] = 0.0; }
                for (int c = 0; c < nc; ++c) acc[c][k] = acc[c][k] + A->v[c][q] * B->v[c][p];
            }
        }
        qsort(Cm->ci + Cm->rp[i], Cm->rp[i + 1] - Cm->rp[i], sizeof(int32_t), cmp_i32);
        for (int64_t u = Cm->rp[i]; u < Cm->rp[i + 1]; ++u)
            for (int c = 0; c < nc; ++c) Cm->v[c][u] = acc[c][Cm->ci[u]];
    }
    for (int c = 0; c < nc; ++c) free(acc[c]);
    free(mark); free(rp);
}

/* l1 row norms d_i = sign(a_ii) sum_j |a_ij| (R-smoother: l1-Jacobi; R-l1: a row whose diagonal
 * is negative keeps that sign, so the smoother's correction points the way Jacobi's would) */
static void l1_diag(olevel *L)
{
    const mcsr *A = &L->A;
    for (int c = 0; c < A->nc; ++c) {
        L->dl1[c] = (double *)xmalloc(sizeof(double) * (A->n + 1));
        for (int i = 0; i < A->n; ++i) {
            double s = 0.0, aii = 0.0;
            for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                s = s + fabs(A->v[c][q]);
                if (A->ci[q] == i) aii = A->v[c][q];
            }
            L->dl1[c][i] = aii < 0.0 ? -s : s;
        }
    }
}

static int make_coarsest(ohier *H, olevel *L)
{
    int n = L->A.n;
    if (n > 4096) return -1;
    L->coarsest = 1;
    for (int c = 0; c < L->A.nc; ++c) {
        L->lu[c] = (double *)xcalloc((int64_t)n * n + 1, sizeof(double));
        L->piv[c] = (int *)xmalloc(sizeof(int) * (n + 1));
        for (int i = 0; i < n; ++i)
            for (int64_t q = L->A.rp[i]; q < L->A.rp[i + 1]; ++q) L->lu[c][(int64_t)i * n + L->A.ci[q]] = L->A.v[c][q];
        dense_lu(n, L->lu[c], L->piv[c], &H->perturbed);
    }
    return 0;
}

/* a4: build the hierarchy (level 0 = a deep copy of the input operator) */
static void hybrid_setup(olevel *L, int B);
static int make_coarsest(ohier *H, olevel *L);
static ohier *amg_build(const mcsr *A0, const int32_t *zb0, const int32_t *colour0, const orc_opts *o)
{
    ohier *H = (ohier *)xcalloc(1, sizeof(ohier));
    H->nc = A0->nc; H->o = *o;
    olevel *L = &H->L[0];
    mcsr_alloc(&L->A, A0->n, A0->m, A0->nc, mnnz(A0));
    memcpy(L->A.rp, A0->rp, sizeof(int32_t) * (A0->n + 1));
    memcpy(L->A.ci, A0->ci, sizeof(int32_t) * mnnz(A0));
    for (int c = 0; c < A0->nc; ++c) memcpy(L->A.v[c], A0->v[c], sizeof(double) * mnnz(A0));
    L->zb = (int32_t *)xmalloc(sizeof(int32_t) * (A0->n + 1));
    memcpy(L->zb, zb0, sizeof(int32_t) * A0->n);
    int lvl = 0;
    for (;;) {
        L = &H->L[lvl];
        l1_diag(L);
        if (o->amg_smoother == 1) {            /* R-gs: level 0 comes with a geometric colouring, the rest is hybrid */
            L->color = (int32_t *)xmalloc(sizeof(int32_t) * (L->A.n + 1));
            if (lvl == 0 && colour0) {
                memcpy(L->color, colour0, sizeof(int32_t) * L->A.n);
                L->ncolor = 0;
                for (int i = 0; i < L->A.n; ++i) if (L->color[i] + 1 > L->ncolor) L->ncolor = L->color[i] + 1;
            } else hybrid_setup(L, o->amg_gs_block > 0 ? o->amg_gs_block : 1024);
        }
        int n = L->A.n;
        if (n <= o->amg_coarse_max || lvl == o->amg_max_levels - 1) {
            if (make_coarsest(H, L)) goto fail;
            break;
        }
        uint8_t *E = (uint8_t *)xcalloc(mnnz(&L->A) + 1, 1);
        if (strength(&L->A, L->zb, o->amg_theta, E)) { free(E); goto fail; }
        int32_t *grp, *gci;
        graph_from_E(&L->A, E, &grp, &gci);
        uint32_t *hs = (uint32_t *)xmalloc(sizeof(uint32_t) * (n + 1));
        for (int i = 0; i < n; ++i) hs[i] = fmix32((uint32_t)i);
        int32_t *st = (int32_t *)xmalloc(sizeof(int32_t) * (n + 1));
        mis2_greedy(n, grp, gci, hs, st);
        L->agg = (int32_t *)xmalloc(sizeof(int32_t) * (n + 1));
        L->ph1 = (int32_t *)xmalloc(sizeof(int32_t) * (n + 1));
        L->nagg = aggregate(&L->A, E, st, L->agg, L->ph1);
        if (L->nagg == 0 || (double)L->nagg > 0.8 * (double)n) {
            /* coarsening stagnation: direct solve at this level */
            H->fallbacks++;
            free(E); free(grp); free(gci); free(hs); free(st);
            free(L->agg); L->agg = NULL; L->nagg = 0;
            free(L->ph1); L->ph1 = NULL;
            if (make_coarsest(H, L)) goto fail;
            break;
        }
        build_P(L, E);
        transpose(&L->P, &L->R);
        mcsr AP; spgemm(&L->A, &L->P, &AP);
        olevel *Lc = &H->L[lvl + 1];
        spgemm(&L->R, &AP, &Lc->A);
        mcsr_free(&AP);
        Lc->zb = (int32_t *)xmalloc(sizeof(int32_t) * (L->nagg + 1));
        for (int i = 0; i < n; ++i) if (st[i] == ST_ROOT) Lc->zb[L->agg[i]] = L->zb[i];
        L->st = st;
        L->E = E;
        free(grp); free(gci); free(hs);
        ++lvl;
    }
    H->nl = lvl + 1;
    return H;
fail:
    H->nl = lvl + 1;
    return NULL;
}

static void amg_free(ohier *H)
{
    if (!H) return;
    for (int l = 0; l < 16; ++l) {
        olevel *L = &H->L[l];
        mcsr_free(&L->A); mcsr_free(&L->P); mcsr_free(&L->R);
        free(L->zb); free(L->agg); free(L->st); free(L->ph1); free(L->color); free(L->E);
        for (int c = 0; c < 3; ++c) { free(L->dl1[c]); free(L->lu[c]); free(L->piv[c]); free(L->dh[c]); }
    }
    free(H);
}

/* One Gauss-Seidel sweep on component c (R-gs), forward (colours ascending) or backward (descending).
 * Level with a given (geometric) colouring -- level 0 of the coupled problem: multicolour GS over the whole
 * level, x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii with the current x (a_ii = 0 leaves x_i).
 * Other levels: hybrid l1-Gauss-Seidel (Baker, Falgout, Kolev, Yang 2011) with the "processor" a block
 * of gs_block consecutive rows: inside the block multicolour GS in the block's own colouring, couplings to
 * other blocks use the values from before the sweep and enter the l1 diagonal
 *   d_i = a_ii + sign(a_ii) sum_{j outside the block} |a_ij|,   x_i <- x_i + (b_i - sum_j a_ij x~_j) / d_i
 * (x~ = current in-block values, sweep-start values outside; R-l1 sign convention).  Rows of one colour are
 * never coupled, so the order inside a colour is immaterial. */
static void gs_sweep(const olevel *L, int c, const double *b, double *x, int backward)
{
    const mcsr *A = &L->A;
    const int n = A->n;
    if (!L->gs_block) {
        for (int t = 0; t < L->ncolor; ++t) {
            int col = backward ? L->ncolor - 1 - t : t;
            for (int i = 0; i < n; ++i) {
                if (L->color[i] != col) continue;
                double s = b[i], d = 0.0;
                for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                    if (A->ci[q] == i) d = A->v[c][q];
                    else s = s - A->v[c][q] * x[A->ci[q]];
                }
                if (d != 0.0) x[i] = s / d;
            }
        }
        return;
    }
    const int B = L->gs_block;
    double *xo = (double *)xmalloc(sizeof(double) * (n + 1));
    memcpy(xo, x, sizeof(double) * n);
    for (int b0 = 0; b0 < n; b0 += B) {
        const int b1 = b0 + B < n ? b0 + B : n;
        for (int t = 0; t < L->ncolor; ++t) {
            int col = backward ? L->ncolor - 1 - t : t;
            for (int i = b0; i < b1; ++i) {
                if (L->color[i] != col) continue;
                double s = b[i], d = 0.0;
                for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                    int j = A->ci[q];
                    if (j == i) d = A->v[c][q];
                    else s = s - A->v[c][q] * ((j >= b0 && j < b1) ? x[j] : xo[j]);
                }
                if (L->dh[c][i] != 0.0) x[i] = x[i] + (s - d * x[i]) / L->dh[c][i];
            }
        }
    }
    free(xo);
}

/* colouring of a hybrid level: each block of B rows coloured on its own, first fit in descending priority
 * (fmix32(i), i) over the block's induced subgraph (row v takes the smallest colour none of its in-block
 * neighbours coloured before it holds), and the l1 diagonal of the off-block couplings */
static void hybrid_setup(olevel *L, int B)
{
    const mcsr *A = &L->A;
    int n = A->n;
    L->gs_block = B;
    L->ncolor = 0;
    prio_t *p = (prio_t *)xmalloc(sizeof(prio_t) * (B + 1));
    uint8_t *used = (uint8_t *)xmalloc(4096);
    for (int b0 = 0; b0 < n; b0 += B) {
        const int b1 = b0 + B < n ? b0 + B : n, m = b1 - b0;
        for (int i = 0; i < m; ++i) { p[i].h = fmix32((uint32_t)(b0 + i)); p[i].i = b0 + i; L->color[b0 + i] = -1; }
        qsort(p, m, sizeof(prio_t), prio_desc);
        for (int t = 0; t < m; ++t) {
            int v = p[t].i;
            memset(used, 0, 4096);
            for (int64_t q = A->rp[v]; q < A->rp[v + 1]; ++q) {
                int u = A->ci[q];
                if (u != v && u >= b0 && u < b1 && L->color[u] >= 0 && L->color[u] < 4096) used[L->color[u]] = 1;
            }
            int cc = 0;
            while (used[cc]) ++cc;
            L->color[v] = cc;
            if (cc + 1 > L->ncolor) L->ncolor = cc + 1;
        }
    }
    free(p); free(used);
    for (int c = 0; c < A->nc; ++c) {
        L->dh[c] = (double *)xmalloc(sizeof(double) * (n + 1));
        for (int i = 0; i < n; ++i) {
            const int b0 = (i / B) * B, b1 = b0 + B < n ? b0 + B : n;
            double aii = 0.0, l1 = 0.0;
            for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) {
                int j = A->ci[q];
                if (j == i) aii = A->v[c][q];
                else if (j < b0 || j >= b1) l1 = l1 + fabs(A->v[c][q]);
            }
            L->dh[c][i] = aii < 0.0 ? aii - l1 : aii + l1;
        }
    }
}

/* Frozen-aggregation refresh (NEXT-f1, reading R-refresh): the values of A_0 changed, its pattern did not.
 * Strength graphs, MIS(2), aggregates, the P / R / A_c patterns and the GS colourings of the previous build are
 * kept; recomputed in the build's own order and arithmetic: l1 norms, the filtered diagonal with the KEPT strength
 * flags, rho and omega, P's values, R = P^T, A_c = R (A P), the hybrid l1 diagonals and the coarsest LU. */
static int amg_refresh(ohier *H, const mcsr *A0)
{
    olevel *L0 = &H->L[0];
    if (A0->n != L0->A.n || mnnz(A0) != mnnz(&L0->A)) return -1;
    for (int64_t q = 0; q < mnnz(A0); ++q) if (A0->ci[q] != L0->A.ci[q]) return -1;
    for (int c = 0; c < A0->nc; ++c) memcpy(L0->A.v[c], A0->v[c], sizeof(double) * mnnz(A0));
    H->perturbed = 0;
    for (int lvl = 0; lvl < H->nl; ++lvl) {
        olevel *L = &H->L[lvl];
        for (int c = 0; c < 3; ++c) { free(L->dl1[c]); L->dl1[c] = NULL; free(L->dh[c]); L->dh[c] = NULL; }
        l1_diag(L);
        if (L->gs_block) hybrid_setup(L, L->gs_block);
        if (L->coarsest) {
            for (int c = 0; c < 3; ++c) { free(L->lu[c]); L->lu[c] = NULL; free(L->piv[c]); L->piv[c] = NULL; }
            if (make_coarsest(H, L)) return -2;
            break;
        }
        mcsr_free(&L->P); mcsr_free(&L->R);
        build_P(L, L->E);
        transpose(&L->P, &L->R);
        mcsr AP; spgemm(&L->A, &L->P, &AP);
        mcsr Ac; spgemm(&L->R, &AP, &Ac);
        mcsr_free(&AP);
        olevel *Lc = &H->L[lvl + 1];
        if (Ac.n != Lc->A.n || mnnz(&Ac) != mnnz(&Lc->A)) { mcsr_free(&Ac); return -3; }
        mcsr_free(&Lc->A);
        Lc->A = Ac;
    }
    return 0;
}

/* Chebyshev smoother (reading R-cheb; north_star "fused Jacobi/Chebyshev ... AMG smoothers"): `degree` steps of
 * the Chebyshev iteration (Saad, Iterative Methods for Sparse Linear Systems, Alg. 12.1) for D^-1 A x = D^-1 b with
 * D the signed l1 diagonal (R-l1), on the interval [a, b] = [lower, 1] -- b = 1 because D_l1 >= A (Gershgorin on the
 * rows of D_l1^-1 A), a = lower * b (hypre's default fraction 0.3):
 *   theta = (b + a)/2, delta = (b - a)/2, sigma = theta/delta, rho_0 = 1/sigma
 *   r_0 = D^-1 (b - A x_0), d_0 = r_0 / theta, x_1 = x_0 + d_0
 *   for k = 1 .. degree-1:  rho_k = 1/(2 sigma - rho_{k-1}),  r_k = D^-1 (b - A x_k),
 *                           d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) r_k,  x_{k+1} = x_k + d_k
 * dl1 == 0 rows take r = 0 (as l1-Jacobi). from_zero: x_0 = 0 (then r_0 = D^-1 b without a product). */
static void cheb_smooth(const mcsr *A, int c, const double *dl1, int degree, double lower, const double *b, double *x,
                        int from_zero)
{
    const int n = A->n;
    const double bb = 1.0, aa = lower * bb;
    const double theta = 0.5 * (bb + aa), delta = 0.5 * (bb - aa), sigma = theta / delta;
    double *r = (double *)xmalloc(sizeof(double) * (n + 1)), *d = (double *)xmalloc(sizeof(double) * (n + 1));
    double rho = 1.0 / sigma;
    for (int k = 0; k < degree; ++k) {
        /* r_k = D^-1 (b - A x_k) */
        OMP_ROWS
        for (int i = 0; i < n; ++i) {
            double s = b[i];
            if (!(k == 0 && from_zero))
                for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) s -= A->v[c][q] * x[A->ci[q]];
            r[i] = dl1[i] != 0.0 ? s / dl1[i] : 0.0;
        }
        if (k == 0) {
            OMP_ROWS
            for (int i = 0; i < n; ++i) { d[i] = r[i] / theta; x[i] = (from_zero ? 0.0 : x[i]) + d[i]; }
        } else {
            const double rho_new = 1.0 / (2.0 * sigma - rho);
            OMP_ROWS
            for (int i = 0; i < n; ++i) { d[i] = rho_new * rho * d[i] + (2.0 * rho_new / delta) * r[i]; x[i] = x[i] + d[i]; }
            rho = rho_new;
        }
    }
    free(r); free(d);
}

int orc_cheb_smooth(int n, const int32_t *rp, const int32_t *ci, const double *v, int degree, double lower,
                    const double *b, const double *x0, double *x)
{
    if (degree < 1 || !(lower > 0.0 && lower < 1.0)) return -1;
    olevel L; memset(&L, 0, sizeof(L));
    mcsr_alloc(&L.A, n, n, 1, rp[n]);
    memcpy(L.A.rp, rp, sizeof(int32_t) * (n + 1)); memcpy(L.A.ci, ci, sizeof(int32_t) * rp[n]);
    memcpy(L.A.v[0], v, sizeof(double) * rp[n]);
    l1_diag(&L);
    for (int i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
    cheb_smooth(&L.A, 0, L.dl1[0], degree, lower, b, x, x0 == NULL);
    free(L.dl1[0]); mcsr_free(&L.A);
    return 0;
}

/* V(1,1)-cycle with l1-Jacobi, zero initial guess (R-cycle), component c:
 *   x = D^-1 b; r = b - A x; b_c = R r; x_c = cycle(b_c); x += P x_c; x += D^-1 (b - A x)
 * amg_smoother 1 (R-gs): x = forward GS sweep from 0; ... ; backward GS sweep on x */
static void vcycle(const ohier *H, int lvl, int c, const double *b, double *x)
{
    const olevel *L = &H->L[lvl];
    int n = L->A.n;
    if (L->coarsest) { dense_lu_solve(n, L->lu[c], L->piv[c], b, x); return; }
    static int lvmax = -2; if (lvmax == -2) { const char *e = getenv("ORC_GS_MAXLVL"); lvmax = e ? atoi(e) : 99; }
    const int gs = H->o.amg_smoother == 1 && lvl <= lvmax;
    const int cheb = H->o.amg_smoother == 2;
    if (gs) { for (int i = 0; i < n; ++i) x[i] = 0.0; gs_sweep(L, c, b, x, 0); }       /* forward GS from zero */
    else if (cheb) cheb_smooth(&L->A, c, L->dl1[c], H->o.amg_cheb_degree, H->o.amg_cheb_lower, b, x, 1);
    else {
        OMP_ROWS
        for (int i = 0; i < n; ++i) x[i] = L->dl1[c][i] != 0.0 ? b[i] / L->dl1[c][i] : 0.0;
    }
    double *r = (double *)xmalloc(sizeof(double) * (n + 1));
    memcpy(r, b, sizeof(double) * n);
    spmv_sub(&L->A, c, x, r);
    int m = L->nagg;
    double *bc = (double *)xmalloc(sizeof(double) * (m + 1)), *xc = (double *)xcalloc(m + 1, sizeof(double));
    spmv(&L->R, c, r, bc);
    vcycle(H, lvl + 1, c, bc, xc);
    OMP_ROWS
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t q = L->P.rp[i]; q < L->P.rp[i + 1]; ++q) s += L->P.v[c][q] * xc[L->P.ci[q]];
        x[i] += s;
    }
    if (gs) gs_sweep(L, c, b, x, 1);                                                       /* backward GS */
    else if (cheb) cheb_smooth(&L->A, c, L->dl1[c], H->o.amg_cheb_degree, H->o.amg_cheb_lower, b, x, 0);
    else {
        memcpy(r, b, sizeof(double) * n);
        spmv_sub(&L->A, c, x, r);
        OMP_ROWS
        for (int i = 0; i < n; ++i) if (L->dl1[c][i] != 0.0) x[i] += r[i] / L->dl1[c][i];
    }
    free(r); free(bc); free(xc);
}

/* ======================================================================
 * a5: tile-local 2x2-block ILU(0) of P S_ff^FS P^T (R-ilu):
 * block Jacobi over fixed tiles; inside a tile, textbook IKJ block ILU(0) in
 * natural order on the tile's sub-pattern (couplings between tiles dropped).
 * ==================================================================== */
typedef struct {
    int nc; int nx, ny, nz, tx, ty, tz;
    int32_t *rp, *ci; double *F;   /* F: L (strict lower) and U (upper incl. diag), 2x2 row-major */
    double *Uinv;                  /* 4 per cell */
    int64_t perturbed;
} oilu;

static int same_tile(const oilu *I, int a, int b)
{
    int ai = a % I->nx, aj = (a / I->nx) % I->ny, ak = a / (I->nx * I->ny);
    int bi = b % I->nx, bj = (b / I->nx) % I->ny, bk = b / (I->nx * I->ny);
    return ai / I->tx == bi / I->tx && aj / I->ty == bj / I->ty && ak / I->tz == bk / I->tz;
}
static void inv2(const double *a, double *r) { double det = a[0] * a[3] - a[1] * a[2]; r[0] = a[3] / det; r[1] = -a[1] / det; r[2] = -a[2] / det; r[3] = a[0] / det; }
static void mul2(const double *a, const double *b, double *r)
{
    r[0] = a[0] * b[0] + a[1] * b[2]; r[1] = a[0] * b[1] + a[1] * b[3];
    r[2] = a[2] * b[0] + a[3] * b[2]; r[3] = a[2] * b[1] + a[3] * b[3];
}

void *orc_ilu_build(int nx, int ny, int nz, int tx, int ty, int tz, const int32_t *rp, const int32_t *ci, const double *v)
{
    oilu *I = (oilu *)xcalloc(1, sizeof(oilu));
    int nc = nx * ny * nz;
    I->nc = nc; I->nx = nx; I->ny = ny; I->nz = nz; I->tx = tx; I->ty = ty; I->tz = tz;
    I->rp = (int32_t *)xcalloc(nc + 1, sizeof(int32_t));
    for (int i = 0; i < nc; ++i) { int c = 0; for (int64_t q = rp[i]; q < rp[i + 1]; ++q) c += same_tile(I, i, ci[q]); I->rp[i + 1] = I->rp[i] + c; }
    I->ci = (int32_t *)xmalloc(sizeof(int32_t) * (I->rp[nc] + 1));
    I->F = (double *)xmalloc(sizeof(double) * 4 * (I->rp[nc] + 1));
    for (int i = 0; i < nc; ++i) {
        int64_t t = I->rp[i];
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
            if (same_tile(I, i, ci[q])) { I->ci[t] = ci[q]; memcpy(&I->F[4 * t], &v[4 * q], 4 * sizeof(double)); ++t; }
    }
    I->Uinv = (double *)xmalloc(sizeof(double) * 4 * (nc + 1));
    for (int i = 0; i < nc; ++i) {
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) {
            int k = I->ci[q];
            if (k >= i) continue;
            double L[4];
            mul2(&I->F[4 * q], &I->Uinv[4 * k], L);          /* L_ik = A_ik U_kk^-1 */
            memcpy(&I->F[4 * q], L, sizeof(L));
            for (int64_t q2 = I->rp[i]; q2 < I->rp[i + 1]; ++q2) {
                int j = I->ci[q2];
                if (j <= k) continue;
                for (int64_t q3 = I->rp[k]; q3 < I->rp[k + 1]; ++q3)
                    if (I->ci[q3] == j) {                    /* A_ij -= L_ik U_kj (on the pattern only) */
                        double t[4]; mul2(L, &I->F[4 * q3], t);
                        for (int e = 0; e < 4; ++e) I->F[4 * q2 + e] -= t[e];
                    }
            }
        }
        int64_t qd = -1;
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) if (I->ci[q] == i) qd = q;
        double *D = &I->F[4 * qd];
        double s = fmax(fmax(fabs(D[0]), fabs(D[1])), fmax(fabs(D[2]), fabs(D[3])));
        double det = D[0] * D[3] - D[1] * D[2];
        if (s == 0.0 || fabs(det) <= 1e-14 * s * s) {     /* singular pivot: perturb */
            double dl = 1e-12 * (s > 0.0 ? s : 1.0);
            D[0] += dl; D[3] += dl; I->perturbed++;
        }
        inv2(D, &I->Uinv[4 * i]);
    }
    return I;
}

void orc_ilu_apply(void *ilu, const double *w, double *dz)
{
    oilu *I = (oilu *)ilu;
    int nc = I->nc;
    double *y = (double *)xmalloc(sizeof(double) * 2 * (nc + 1));
    for (int i = 0; i < nc; ++i) {           /* forward: unit block-lower L */
        double a = w[2 * i], b = w[2 * i + 1];
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) {
            int k = I->ci[q]; if (k >= i) continue;
            const double *L = &I->F[4 * q];
            a -= L[0] * y[2 * k] + L[1] * y[2 * k + 1];
            b -= L[2] * y[2 * k] + L[3] * y[2 * k + 1];
        }
        y[2 * i] = a; y[2 * i + 1] = b;
    }
    for (int i = nc - 1; i >= 0; --i) {      /* backward: U */
        double a = y[2 * i], b = y[2 * i + 1];
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) {
            int j = I->ci[q]; if (j <= i) continue;
            const double *U = &I->F[4 * q];
            a -= U[0] * dz[2 * j] + U[1] * dz[2 * j + 1];
            b -= U[2] * dz[2 * j] + U[3] * dz[2 * j + 1];
        }
        const double *Ui = &I->Uinv[4 * i];
        dz[2 * i] = Ui[0] * a + Ui[1] * b;
        dz[2 * i + 1] = Ui[2] * a + Ui[3] * b;
    }
    free(y);
}
void orc_ilu_free(void *ilu) { oilu *I = (oilu *)ilu; if (!I) return; free(I->rp); free(I->ci); free(I->F); free(I->Uinv); free(I); }

/* ---------------- option 1 of the second stage: hybrid block Gauss-Seidel (hbgs) ----------------
 * One sweep from zero = the block forward substitution (L + D)^-1 of the tile-local lower triangle of
 * P S_ff^FS P^T in natural order (x fastest), D = the 2x2 diagonal blocks (inverted exactly; singular ones
 * perturbed as the ILU's); couplings leaving the tile are the "hybrid" (Jacobi) part and enter
 * only through the residual of the next sweep (R-hbgs). */
void *orc_bgs_build(int nx, int ny, int nz, int tx, int ty, int tz, const int32_t *rp, const int32_t *ci, const double *v)
{
    oilu *I = (oilu *)xcalloc(1, sizeof(oilu));
    int nc = nx * ny * nz;
    I->nc = nc; I->nx = nx; I->ny = ny; I->nz = nz; I->tx = tx; I->ty = ty; I->tz = tz;
    I->rp = (int32_t *)xcalloc(nc + 1, sizeof(int32_t));
    for (int i = 0; i < nc; ++i) { int c = 0; for (int64_t q = rp[i]; q < rp[i + 1]; ++q) c += same_tile(I, i, ci[q]); I->rp[i + 1] = I->rp[i] + c; }
    I->ci = (int32_t *)xmalloc(sizeof(int32_t) * (I->rp[nc] + 1));
    I->F = (double *)xmalloc(sizeof(double) * 4 * (I->rp[nc] + 1));
    I->Uinv = (double *)xmalloc(sizeof(double) * 4 * (nc + 1));
    for (int i = 0; i < nc; ++i) {
        int64_t t = I->rp[i];
        for (int64_t q = rp[i]; q < rp[i + 1]; ++q)
            if (same_tile(I, i, ci[q])) { I->ci[t] = ci[q]; memcpy(&I->F[4 * t], &v[4 * q], 4 * sizeof(double)); ++t; }
        double D[4] = {0, 0, 0, 0};
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) if (I->ci[q] == i) memcpy(D, &I->F[4 * q], sizeof(D));
        double sc = fmax(fmax(fabs(D[0]), fabs(D[1])), fmax(fabs(D[2]), fabs(D[3])));
        double det = D[0] * D[3] - D[1] * D[2];
        if (sc == 0.0 || fabs(det) <= 1e-14 * sc * sc) {
            double dl = 1e-12 * (sc > 0.0 ? sc : 1.0);
            D[0] += dl; D[3] += dl; I->perturbed++;
        }
        inv2(D, &I->Uinv[4 * i]);
    }
    return I;
}
void orc_bgs_apply(void *bgs, const double *w, double *dz)
{
    oilu *I = (oilu *)bgs;
    for (int i = 0; i < I->nc; ++i) {
        double a = w[2 * i], b = w[2 * i + 1];
        for (int64_t q = I->rp[i]; q < I->rp[i + 1]; ++q) {
            int k = I->ci[q]; if (k >= i) continue;
            const double *A = &I->F[4 * q];
            a -= A[0] * dz[2 * k] + A[1] * dz[2 * k + 1];
            b -= A[2] * dz[2 * k] + A[3] * dz[2 * k + 1];
        }
        const double *Di = &I->Uinv[4 * i];
        dz[2 * i] = Di[0] * a + Di[1] * b;
        dz[2 * i + 1] = Di[2] * a + Di[3] * b;
    }
}

/* ======================================================================
 * the handle: inputs, setup products (a1-a5), Algorithm 1, operator, FGMRES
 * ==================================================================== */
typedef struct { int nr, ncol, bm, bn; int32_t *rp, *ci; double *v; } obsr;

struct orc {
    int nx, ny, nz, Nn, Nc, n;
    orc_opts o;
    obsr uu, uf, fu, ff; double *fs;
    /* a1/a3 products (partitioned scalar blocks) */
    mcsr Ass, Asp, Aps, App, Asp_fs, App_fs, Asu, Apu, Spp;
    double *Dss, *Dps;            /* D_ss^(CPR), D_ps^(CPR) (P:568-575 / eq:CPR_CSL) */
    double *fs_eff;               /* (D_sp, D_pp) used by a1: given / scale, or RSL */
    obsr Sff;                     /* interleaved S_ff^FS for M_L */
    ohier *mech, *pres;
    oilu *ilu;
    double *dense_uu, *dense_pp, *dense_ff, *dense_schur; int *piv_uu, *piv_pp, *piv_ff, *piv_schur;
    int64_t skipped_dss, perturbed;
    int setup_done;
};

static void bsr_copy(obsr *B, int nr, int ncol, int bm, int bn, const int32_t *rp, const int32_t *ci, const double *v)
{
    B->nr = nr; B->ncol = ncol; B->bm = bm; B->bn = bn;
    int64_t nb = rp[nr];
    B->rp = (int32_t *)xmalloc(sizeof(int32_t) * (nr + 1)); memcpy(B->rp, rp, sizeof(int32_t) * (nr + 1));
    B->ci = (int32_t *)xmalloc(sizeof(int32_t) * (nb + 1)); memcpy(B->ci, ci, sizeof(int32_t) * nb);
    B->v = (double *)xmalloc(sizeof(double) * bm * bn * (nb + 1)); memcpy(B->v, v, sizeof(double) * bm * bn * nb);
}
static void bsr_free(obsr *B) { free(B->rp); free(B->ci); free(B->v); memset(B, 0, sizeof(*B)); }

/* scalar CSR of entry (r, s) of every block of a BSR matrix (same block pattern) */
static void bsr_entry(const obsr *B, int r, int s, mcsr *A)
{
    int64_t nb = B->rp[B->nr];
    mcsr_alloc(A, B->nr, B->ncol, 1, nb);
    memcpy(A->rp, B->rp, sizeof(int32_t) * (B->nr + 1));
    memcpy(A->ci, B->ci, sizeof(int32_t) * nb);
    for (int64_t q = 0; q < nb; ++q) A->v[0][q] = B->v[(int64_t)B->bm * B->bn * q + r * B->bn + s];
}
/* scalar CSR of row r of each block row, all bn columns of each block: (nr x ncol*bn) */
static void bsr_rowslice(const obsr *B, int r, mcsr *A)
{
    int64_t nb = B->rp[B->nr];
    mcsr_alloc(A, B->nr, B->ncol * B->bn, 1, nb * B->bn);
    for (int i = 0; i < B->nr; ++i) A->rp[i + 1] = (int32_t)(B->rp[i + 1] * (int64_t)B->bn);
    for (int64_t q = 0; q < nb; ++q)
        for (int e = 0; e < B->bn; ++e) {
            A->ci[q * B->bn + e] = B->ci[q] * B->bn + e;
            A->v[0][q * B->bn + e] = B->v[(int64_t)B->bm * B->bn * q + r * B->bn + e];
        }
}

void orc_default_opts(orc_opts *o)
{
    memset(o, 0, sizeof(*o));
    o->amg_theta = 0.25; o->amg_coarse_max = 64; o->amg_max_levels = 12;
    o->zblock = 16; o->tile_x = 16; o->tile_y = 16; o->tile_z = 16;
    o->rsl_iters = 2; o->fs_modulus_scale = 1.0;
    o->second_stage = 0; o->local_sweeps = 1;
    o->amg_smoother = 0; o->amg_gs_block = 1024;
    o->amg_cheb_degree = 2; o->amg_cheb_lower = 0.3;
    o->amg_smoother_p = -1;
}

orc *orc_create(const orc_desc *d, const orc_opts *o)
{
    orc *h = (orc *)xcalloc(1, sizeof(orc));
    h->nx = d->nx; h->ny = d->ny; h->nz = d->nz;
    h->Nn = (d->nx + 1) * (d->ny + 1) * (d->nz + 1);
    h->Nc = d->nx * d->ny * d->nz;
    h->n = 3 * h->Nn + 2 * h->Nc;
    if (o) h->o = *o; else orc_default_opts(&h->o);
    bsr_copy(&h->uu, h->Nn, h->Nn, 3, 3, d->uu_rowptr, d->uu_col, d->uu_val);
    bsr_copy(&h->uf, h->Nn, h->Nc, 3, 2, d->uf_rowptr, d->uf_col, d->uf_val);
    bsr_copy(&h->fu, h->Nc, h->Nn, 2, 3, d->fu_rowptr, d->fu_col, d->fu_val);
    bsr_copy(&h->ff, h->Nc, h->Nc, 2, 2, d->ff_rowptr, d->ff_col, d->ff_val);
    h->fs = (double *)xmalloc(sizeof(double) * 2 * h->Nc);
    memcpy(h->fs, d->fs, sizeof(double) * 2 * h->Nc);
    return h;
}

static void dense_from_bsr(const obsr *B, double *D, int ld)
{
    for (int i = 0; i < B->nr; ++i)
        for (int64_t q = B->rp[i]; q < B->rp[i + 1]; ++q)
            for (int r = 0; r < B->bm; ++r)
                for (int s = 0; s < B->bn; ++s)
                    D[(int64_t)(i * B->bm + r) * ld + B->ci[q] * B->bn + s] = B->v[(int64_t)B->bm * B->bn * q + r * B->bn + s];
}

/* step 1 of Algorithm 1: z_u = M_uu^-1 v_u, one SDC V-cycle per displacement component
 * (P:513-517), or the exact dense solve (pins) */
static void mech_apply(orc *h, const double *vu, double *zu)
{
    int Nn = h->Nn;
    if (h->o.mech_mode == 0) {
        double *bc = (double *)xmalloc(sizeof(double) * Nn), *xc = (double *)xmalloc(sizeof(double) * Nn);
        for (int c = 0; c < 3; ++c) {
            for (int i = 0; i < Nn; ++i) bc[i] = vu[3 * i + c];
            vcycle(h->mech, 0, c, bc, xc);
            for (int i = 0; i < Nn; ++i) zu[3 * i + c] = xc[i];
        }
        free(bc); free(xc);
    } else {
        dense_lu_solve(3 * Nn, h->dense_uu, h->piv_uu, vu, zu);
    }
}

/* y = A_uu x, 3x3 blocks (eq:jac_system) */
static void uu_matvec(const orc *h, const double *x, double *y)
{
    OMP_ROWS
    for (int i = 0; i < h->Nn; ++i)
        for (int r = 0; r < 3; ++r) {
            double s = 0.0;
            for (int64_t q = h->uu.rp[i]; q < h->uu.rp[i + 1]; ++q)
                for (int c = 0; c < 3; ++c) s = s + h->uu.v[9 * q + 3 * r + c] * x[3 * (int64_t)h->uu.ci[q] + c];
            y[3 * (int64_t)i + r] = s;
        }
}

/* eq:FS_RSL: D_sp = -diag(A_su A_uu^-1 A_up e), D_pp = -diag(A_pu A_uu^-1 A_up e).  A_uu^-1 is
 * approximated with the available preconditioner: rsl_iters steps of Richardson iteration
 * y_{t+1} = y_t + M_uu^-1 (g - A_uu y_t), y_0 = 0, g = A_up e.  out = (D_sp, D_pp) per cell. */
static void rsl_diag(orc *h, double *out)
{
    int Nn = h->Nn, Nc = h->Nc, N = 3 * Nn;
    double *g = (double *)xcalloc(N, sizeof(double)), *y = (double *)xcalloc(N, sizeof(double));
    double *r = (double *)xmalloc(sizeof(double) * N), *t = (double *)xmalloc(sizeof(double) * N);
    double *dy = (double *)xmalloc(sizeof(double) * N);
    for (int i = 0; i < Nn; ++i)                         /* g = A_up e: the p column of every 3x2 block of A_uf */
        for (int64_t q = h->uf.rp[i]; q < h->uf.rp[i + 1]; ++q)
            for (int rr = 0; rr < 3; ++rr) g[3 * (int64_t)i + rr] = g[3 * (int64_t)i + rr] + h->uf.v[6 * q + 2 * rr + 1];
    int iters = h->o.rsl_iters > 0 ? h->o.rsl_iters : 1;
    for (int it = 0; it < iters; ++it) {
        uu_matvec(h, y, t);
        for (int k = 0; k < N; ++k) r[k] = g[k] - t[k];
        mech_apply(h, r, dy);
        for (int k = 0; k < N; ++k) y[k] = y[k] + dy[k];
    }
    for (int K = 0; K < Nc; ++K) {                       /* A_su y, A_pu y: rows s and p of the 2x3 blocks */
        double ss = 0.0, sp = 0.0;
        for (int64_t q = h->fu.rp[K]; q < h->fu.rp[K + 1]; ++q)
            for (int c = 0; c < 3; ++c) {
                ss = ss + h->fu.v[6 * q + c] * y[3 * (int64_t)h->fu.ci[q] + c];
                sp = sp + h->fu.v[6 * q + 3 + c] * y[3 * (int64_t)h->fu.ci[q] + c];
            }
        out[2 * K] = -ss;
        out[2 * K + 1] = -sp;
    }
    free(g); free(y); free(r); free(t); free(dy);
}

int orc_setup(orc *h)
{
    double t0 = now_s();
    int Nn = h->Nn;
    /* ---- a2 + a4 (mechanics): M_uu^-1 = amg(A_uu^SDC), three components on one
     *      node graph */
    if (h->o.mech_mode == 0) {
        mcsr Asdc;
        int64_t nb = h->uu.rp[Nn];
        mcsr_alloc(&Asdc, Nn, Nn, 3, nb);
        memcpy(Asdc.rp, h->uu.rp, sizeof(int32_t) * (Nn + 1));
        memcpy(Asdc.ci, h->uu.ci, sizeof(int32_t) * nb);
        for (int64_t q = 0; q < nb; ++q)
            for (int c = 0; c < 3; ++c) Asdc.v[c][q] = h->uu.v[9 * q + 4 * c];   /* (x,x), (y,y), (z,z) */
        int32_t *zb = (int32_t *)xmalloc(sizeof(int32_t) * Nn);
        for (int n = 0; n < Nn; ++n) {
            int k = n / ((h->nx + 1) * (h->ny + 1));
            int kc = k < h->nz ? k : h->nz - 1;               /* node plane k -> cell plane min(k, nz-1) (R-zblock) */
            zb[n] = kc / h->o.zblock;
        }
        /* R-gs: level-0 node colour = parity of (x, y, z), 8 colours (no two 27-point neighbours share one) */
        int32_t *col0 = (int32_t *)xmalloc(sizeof(int32_t) * Nn);
        for (int n = 0; n < Nn; ++n) {
            int x = n % (h->nx + 1), y = (n / (h->nx + 1)) % (h->ny + 1), z = n / ((h->nx + 1) * (h->ny + 1));
            col0[n] = (x & 1) + 2 * (y & 1) + 4 * (z & 1);
        }
        h->mech = amg_build(&Asdc, zb, col0, &h->o);
        mcsr_free(&Asdc); free(zb); free(col0);
        if (!h->mech) return -2;
    } else {
        int N = 3 * Nn;
        h->dense_uu = (double *)xcalloc((int64_t)N * N, sizeof(double));
        h->piv_uu = (int *)xmalloc(sizeof(int) * N);
        dense_from_bsr(&h->uu, h->dense_uu, N);
        dense_lu(N, h->dense_uu, h->piv_uu, &h->perturbed);
    }
    (void)t0;
    return orc_setup_flow(h, 0);
}

/* the flow phase (rows a1, a3, a4 pressure, a5; redone per Newton step).  refresh = 1: the values
 * changed since the last flow setup, the patterns did not; the pressure hierarchy keeps its structure (frozen
 * aggregation, amg_refresh) and only its values are recomputed (NEXT-f1, reading R-refresh). */
int orc_setup_flow(orc *h, int refresh)
{
    int Nc = h->Nc, Nn = h->Nn;
    if (refresh && (!h->pres || h->o.pres_mode != 0)) return -4;
    /* products of a previous flow phase */
    mcsr *m[] = {&h->Ass, &h->Asp, &h->Aps, &h->App, &h->Asp_fs, &h->App_fs, &h->Asu, &h->Apu, &h->Spp};
    for (size_t k = 0; k < sizeof(m) / sizeof(m[0]); ++k) mcsr_free(m[k]);
    bsr_free(&h->Sff);
    free(h->Dss); free(h->Dps); free(h->fs_eff); h->Dss = h->Dps = h->fs_eff = NULL;
    orc_ilu_free(h->ilu); h->ilu = NULL;
    free(h->dense_pp); free(h->piv_pp); free(h->dense_ff); free(h->piv_ff); free(h->dense_schur); free(h->piv_schur);
    h->dense_pp = h->dense_ff = h->dense_schur = NULL; h->piv_pp = h->piv_ff = h->piv_schur = NULL;
    if (!refresh) { amg_free(h->pres); h->pres = NULL; }
    h->skipped_dss = 0;
    /* ---- a1 input: the fixed-stress diagonal D_fs -- given (eq:FS_Dps_Dpp), divided by
     *      fs_modulus_scale (remark P:443), or by row-sum lumping (eq:FS_RSL) */
    bsr_rowslice(&h->fu, 0, &h->Asu); bsr_rowslice(&h->fu, 1, &h->Apu);
    h->fs_eff = (double *)xmalloc(sizeof(double) * 2 * Nc);
    if (h->o.fs_mode == 1) rsl_diag(h, h->fs_eff);
    else for (int k = 0; k < 2 * Nc; ++k) h->fs_eff[k] = h->fs[k] / h->o.fs_modulus_scale;
    /* ---- a1: fixed-stress augmentation, eq:Schur_1_FS:
     *      A_sp^FS = A_sp + D_sp, A_pp^FS = A_pp + D_pp, D diagonal; A_us ~ 0 */
    bsr_entry(&h->ff, 0, 0, &h->Ass); bsr_entry(&h->ff, 0, 1, &h->Asp);
    bsr_entry(&h->ff, 1, 0, &h->Aps); bsr_entry(&h->ff, 1, 1, &h->App);
    bsr_entry(&h->ff, 0, 1, &h->Asp_fs); bsr_entry(&h->ff, 1, 1, &h->App_fs);
    for (int i = 0; i < Nc; ++i) {
        int64_t q = find_col(&h->Asp_fs, i, i);
        if (q < 0) return -1;
        h->Asp_fs.v[0][q] = h->Asp_fs.v[0][q] + h->fs_eff[2 * i];
        h->App_fs.v[0][q] = h->App_fs.v[0][q] + h->fs_eff[2 * i + 1];
    }
    /* interleaved S_ff^FS for the local stage */
    bsr_copy(&h->Sff, Nc, Nc, 2, 2, h->ff.rp, h->ff.ci, h->ff.v);
    for (int i = 0; i < Nc; ++i)
        for (int64_t q = h->Sff.rp[i]; q < h->Sff.rp[i + 1]; ++q)
            if (h->Sff.ci[q] == i) { h->Sff.v[4 * q + 1] = h->Sff.v[4 * q + 1] + h->fs_eff[2 * i]; h->Sff.v[4 * q + 3] = h->Sff.v[4 * q + 3] + h->fs_eff[2 * i + 1]; }

    /* ---- a3: CPR reduction.  quasi-IMPES: D_ss = diagm(A_ss), D_ps = diagm(A_ps);
     *      true-IMPES (eq:CPR_CSL): D_ss = diag(A_ss^T e), D_ps = diag(A_ps^T e), the column
     *      sums taken over the rows k of column i in ascending order.
     *      S_pp = A_pp^FS - D_ps D_ss^-1 A_sp^FS, same pattern */
    h->Dss = (double *)xmalloc(sizeof(double) * Nc);
    h->Dps = (double *)xmalloc(sizeof(double) * Nc);
    for (int i = 0; i < Nc; ++i) {
        if (h->o.cpr_mode == 1) {
            double dss = 0.0, dps = 0.0;
            for (int64_t q = h->Ass.rp[i]; q < h->Ass.rp[i + 1]; ++q) {   /* symmetric pattern: rows k of column i */
                int k = h->Ass.ci[q];
                int64_t qk = find_col(&h->Ass, k, i);
                if (qk < 0) return -1;
                dss = dss + h->Ass.v[0][qk];
                dps = dps + h->Aps.v[0][qk];
            }
            h->Dss[i] = dss; h->Dps[i] = dps;
        } else {
            int64_t qd = find_col(&h->Ass, i, i);
            h->Dss[i] = h->Ass.v[0][qd]; h->Dps[i] = h->Aps.v[0][qd];
        }
    }
    mcsr_alloc(&h->Spp, Nc, Nc, 1, mnnz(&h->App_fs));
    memcpy(h->Spp.rp, h->App_fs.rp, sizeof(int32_t) * (Nc + 1));
    memcpy(h->Spp.ci, h->App_fs.ci, sizeof(int32_t) * mnnz(&h->App_fs));
    for (int i = 0; i < Nc; ++i) {
        double dss = h->Dss[i], dps = h->Dps[i];
        double ci = 0.0;
        if (dss != 0.0) ci = dps / dss; else h->skipped_dss++;
        for (int64_t q = h->Spp.rp[i]; q < h->Spp.rp[i + 1]; ++q)
            h->Spp.v[0][q] = h->App_fs.v[0][q] - ci * h->Asp_fs.v[0][q];
    }

    /* ---- a4 (pressure): M_pp^-1 = amg(S_pp^(CPR-FS)) */
    if (refresh) {
        if (amg_refresh(h->pres, &h->Spp)) return -5;
    } else if (h->o.pres_mode == 0) {
        int32_t *zb = (int32_t *)xmalloc(sizeof(int32_t) * Nc);
        for (int c = 0; c < Nc; ++c) zb[c] = (c / (h->nx * h->ny)) / h->o.zblock;
        /* R-gs: level-0 cell colour = parity of x + y + z (red-black on the 7-point pattern of S_pp) */
        int32_t *col0 = (int32_t *)xmalloc(sizeof(int32_t) * Nc);
        for (int c = 0; c < Nc; ++c) col0[c] = (c % h->nx + (c / h->nx) % h->ny + c / (h->nx * h->ny)) & 1;
        orc_opts po = h->o;                   /* the pressure hierarchy's own smoother (amg_smoother_p) */
        if (po.amg_smoother_p >= 0) po.amg_smoother = po.amg_smoother_p;
        h->pres = amg_build(&h->Spp, zb, col0, &po);
        free(zb); free(col0);
        if (!h->pres) return -3;
    } else {
        h->dense_pp = (double *)xcalloc((int64_t)Nc * Nc, sizeof(double));
        h->piv_pp = (int *)xmalloc(sizeof(int) * Nc);
        for (int i = 0; i < Nc; ++i) for (int64_t q = h->Spp.rp[i]; q < h->Spp.rp[i + 1]; ++q) h->dense_pp[(int64_t)i * Nc + h->Spp.ci[q]] = h->Spp.v[0][q];
        dense_lu(Nc, h->dense_pp, h->piv_pp, &h->perturbed);
    }
    /* ---- a5: local stage M_L on P S_ff^FS P^T */
    if (h->o.local_mode == 0) {
        h->ilu = (oilu *)(h->o.second_stage == 1 ? orc_bgs_build : orc_ilu_build)(h->nx, h->ny, h->nz, h->o.tile_x, h->o.tile_y,
                                                                                h->o.tile_z, h->Sff.rp, h->Sff.ci, h->Sff.v);
    } else if (h->o.local_mode == 1) {
        int N = 2 * Nc;
        h->dense_ff = (double *)xcalloc((int64_t)N * N, sizeof(double));
        h->piv_ff = (int *)xmalloc(sizeof(int) * N);
        dense_from_bsr(&h->Sff, h->dense_ff, N);
        dense_lu(N, h->dense_ff, h->piv_ff, &h->perturbed);
    }
    /* ---- exact first-level Schur complement S_ff = A_ff - A_fu A_uu^-1 A_uf (eq:LU), pins only */
    if (h->o.ff_mode == 1) {
        int N = 3 * Nn, M = 2 * Nc;
        double *Auu = (double *)xcalloc((int64_t)N * N, sizeof(double)); int *pv = (int *)xmalloc(sizeof(int) * N);
        dense_from_bsr(&h->uu, Auu, N);
        dense_lu(N, Auu, pv, NULL);
        double *Auf = (double *)xcalloc((int64_t)N * M, sizeof(double)), *Afu = (double *)xcalloc((int64_t)M * N, sizeof(double));
        dense_from_bsr(&h->uf, Auf, M); dense_from_bsr(&h->fu, Afu, N);
        h->dense_schur = (double *)xcalloc((int64_t)M * M, sizeof(double));
        dense_from_bsr(&h->ff, h->dense_schur, M);
        double *col = (double *)xmalloc(sizeof(double) * N), *sol = (double *)xmalloc(sizeof(double) * N);
        for (int j = 0; j < M; ++j) {
            for (int i = 0; i < N; ++i) col[i] = Auf[(int64_t)i * M + j];
            dense_lu_solve(N, Auu, pv, col, sol);
            for (int i = 0; i < M; ++i) { double s = 0; for (int k = 0; k < N; ++k) s += Afu[(int64_t)i * N + k] * sol[k]; h->dense_schur[(int64_t)i * M + j] -= s; }
        }
        h->piv_schur = (int *)xmalloc(sizeof(int) * M);
        dense_lu(M, h->dense_schur, h->piv_schur, NULL);
        free(Auu); free(pv); free(Auf); free(Afu); free(col); free(sol);
    }
    h->setup_done = 1;
    return 0;
}

/* ---------------- Algorithm 1 (alg:apply_M_inv) ----------------
 * v, z in library layout [u (node-major x,y,z) | f (interleaved s,p)]; the
 * permutation P of P:606 is applied explicitly to work on partitioned (s; p). */
int orc_apply(orc *h, const double *v, double *z)
{
    if (!h->setup_done) return -3;
    int Nn = h->Nn, Nc = h->Nc;
    const double *vu = v, *vf = v + 3 * Nn;
    double *zu = z, *zf = z + 3 * Nn;
    double *vs = (double *)xmalloc(sizeof(double) * Nc), *vp = (double *)xmalloc(sizeof(double) * Nc);
    for (int K = 0; K < Nc; ++K) { vs[K] = vf[2 * K]; vp[K] = vf[2 * K + 1]; }   /* P^T */
    /* step 1: z_u = M_uu^-1 v_u */
    mech_apply(h, vu, zu);
    /* step 2: [y_s; y_p] = [v_s; v_p] - [A_su; A_pu] z_u */
    double *ys = (double *)xmalloc(sizeof(double) * Nc), *yp = (double *)xmalloc(sizeof(double) * Nc);
    memcpy(ys, vs, sizeof(double) * Nc); memcpy(yp, vp, sizeof(double) * Nc);
    spmv_sub(&h->Asu, 0, zu, ys);
    spmv_sub(&h->Apu, 0, zu, yp);
    if (h->o.ff_mode == 1) {   /* exact M_ff = S_ff^-1 (pins) */
        double *yf = (double *)xmalloc(sizeof(double) * 2 * Nc);
        for (int K = 0; K < Nc; ++K) { yf[2 * K] = ys[K]; yf[2 * K + 1] = yp[K]; }
        dense_lu_solve(2 * Nc, h->dense_schur, h->piv_schur, yf, zf);
        free(yf); free(vs); free(vp); free(ys); free(yp);
        return 0;
    }
    /* step 3: z_s = (D_ss^(CPR))^-1 y_s */
    double *zs = (double *)xmalloc(sizeof(double) * Nc), *zp = (double *)xmalloc(sizeof(double) * Nc);
    for (int K = 0; K < Nc; ++K) zs[K] = h->Dss[K] != 0.0 ? ys[K] / h->Dss[K] : 0.0;
    /* step 4: w_p = y_p - A_ps z_s, full A_ps, or its diagonal D_ps^(CPR) */
    double *wp = (double *)xmalloc(sizeof(double) * Nc);
    memcpy(wp, yp, sizeof(double) * Nc);
    if (h->o.aps_mode == 1) for (int K = 0; K < Nc; ++K) wp[K] = wp[K] - h->Dps[K] * zs[K];
    else spmv_sub(&h->Aps, 0, zs, wp);
    /* step 5: z_p = M_pp^-1 w_p */
    if (h->o.pres_mode == 0) vcycle(h->pres, 0, 0, wp, zp);
    else dense_lu_solve(Nc, h->dense_pp, h->piv_pp, wp, zp);
    if (h->o.local_mode != 2) {
        /* steps 6-8, repeated local_sweeps times (R-sweeps: "several sweeps") */
        double *ws = (double *)xmalloc(sizeof(double) * Nc), *wp2 = (double *)xmalloc(sizeof(double) * Nc);
        double *wf = (double *)xmalloc(sizeof(double) * 2 * Nc), *dzf = (double *)xmalloc(sizeof(double) * 2 * Nc);
        int sweeps = h->o.local_sweeps > 0 ? h->o.local_sweeps : 1;
        for (int sw = 0; sw < sweeps; ++sw) {
            /* step 6: [w_s; w_p] = [y_s; y_p] - [[A_ss, A_sp^FS],[A_ps, A_pp^FS]] [z_s; z_p] */
            memcpy(ws, ys, sizeof(double) * Nc); memcpy(wp2, yp, sizeof(double) * Nc);
            spmv_sub(&h->Ass, 0, zs, ws); spmv_sub(&h->Asp_fs, 0, zp, ws);
            spmv_sub(&h->Aps, 0, zs, wp2); spmv_sub(&h->App_fs, 0, zp, wp2);
            /* step 7: [dz_s; dz_p] = P^T M_L^-1 P [w_s; w_p]; M_L = ILU(0) or hbgs */
            for (int K = 0; K < Nc; ++K) { wf[2 * K] = ws[K]; wf[2 * K + 1] = wp2[K]; }
            if (h->o.local_mode == 0) (h->o.second_stage == 1 ? orc_bgs_apply : orc_ilu_apply)(h->ilu, wf, dzf);
            else dense_lu_solve(2 * Nc, h->dense_ff, h->piv_ff, wf, dzf);
            /* step 8: z += dz */
            for (int K = 0; K < Nc; ++K) { zs[K] += dzf[2 * K]; zp[K] += dzf[2 * K + 1]; }
        }
        free(ws); free(wp2); free(wf); free(dzf);
    }
    for (int K = 0; K < Nc; ++K) { zf[2 * K] = zs[K]; zf[2 * K + 1] = zp[K]; }   /* P */
    free(vs); free(vp); free(ys); free(yp); free(zs); free(zp); free(wp);
    return 0;
}

/* ---------------- operator y = A x, eq:jac_system ---------------- */
static void bsr_mv_add(const obsr *B, const double *x, double *y)
{
    OMP_ROWS
    for (int i = 0; i < B->nr; ++i)
        for (int r = 0; r < B->bm; ++r) {
            double s = 0.0;
            for (int64_t q = B->rp[i]; q < B->rp[i + 1]; ++q)
                for (int e = 0; e < B->bn; ++e) s += B->v[(int64_t)B->bm * B->bn * q + r * B->bn + e] * x[(int64_t)B->ci[q] * B->bn + e];
            y[(int64_t)i * B->bm + r] += s;
        }
}
void orc_apply_operator(orc *h, const double *x, double *y)
{
    memset(y, 0, sizeof(double) * h->n);
    const double *xu = x, *xf = x + 3 * h->Nn;
    double *yu = y, *yf = y + 3 * h->Nn;
    bsr_mv_add(&h->uu, xu, yu); bsr_mv_add(&h->uf, xf, yu);
    bsr_mv_add(&h->fu, xu, yf); bsr_mv_add(&h->ff, xf, yf);
}

/* ---------------- FGMRES(m) with modified Gram-Schmidt (R-krylov, SURVEY O-4) ----------------
 * right-preconditioned, flexible form: Z keeps M^-1 v_j. */
static double dot(const double *a, const double *b, int n) { double s = 0.0; for (int i = 0; i < n; ++i) s += a[i] * b[i]; return s; }

/* the "sequential" embedding of the remark at P:640-642: Richardson iteration x <- x + M^-1 (b - A x),
 * x0 = 0, stopped when ||b - A x|| <= rtol ||b||; iterations = preconditioner applications */
int orc_richardson(orc *h, const double *b, double *x, double rtol, int maxit, orc_info *info)
{
    double t0 = now_s();
    int n = h->n;
    memset(info, 0, sizeof(*info));
    double *r = (double *)xmalloc(sizeof(double) * n), *z = (double *)xmalloc(sizeof(double) * n);
    double bn = sqrt(dot(b, b, n));
    int it = 0, status = 1;
    memset(x, 0, sizeof(double) * n);
    for (;;) {
        orc_apply_operator(h, x, r);
        for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
        double rn = sqrt(dot(r, r, n));
        info->true_relres = bn > 0.0 ? rn / bn : 0.0;
        info->est_relres = info->true_relres;
        if (rn <= rtol * bn) { status = 0; break; }
        if (!isfinite(rn)) { status = 2; break; }
        if (it >= maxit) { status = 1; break; }
        orc_apply(h, r, z);
        for (int i = 0; i < n; ++i) x[i] = x[i] + z[i];
        ++it;
    }
    free(r); free(z);
    info->iterations = it;
    info->status = status;
    info->t_solve = now_s() - t0;
    return status;
}

int orc_solve(orc *h, const double *b, double *x, double rtol, int m, int maxit, orc_info *info)
{
    double t0 = now_s();
    int n = h->n;
    memset(info, 0, sizeof(*info));
    double **V = (double **)xmalloc(sizeof(double *) * (m + 1)), **Z = (double **)xmalloc(sizeof(double *) * m);
    for (int j = 0; j <= m; ++j) V[j] = (double *)xmalloc(sizeof(double) * n);
    for (int j = 0; j < m; ++j) Z[j] = (double *)xmalloc(sizeof(double) * n);
    double *H = (double *)xcalloc((size_t)(m + 1) * m, sizeof(double));
    double *cs = (double *)xmalloc(sizeof(double) * m), *sn = (double *)xmalloc(sizeof(double) * m);
    double *g = (double *)xmalloc(sizeof(double) * (m + 1)), *yv = (double *)xmalloc(sizeof(double) * m);
    double *r = (double *)xmalloc(sizeof(double) * n), *w = (double *)xmalloc(sizeof(double) * n);
    double bn = sqrt(dot(b, b, n));
    int it = 0, status = 1;
    memset(x, 0, sizeof(double) * n);
    if (bn == 0.0) { status = 0; goto done; }
    for (;;) {
        orc_apply_operator(h, x, r);
        for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
        double beta = sqrt(dot(r, r, n));
        info->true_relres = beta / bn;
        if (beta <= rtol * bn) { status = 0; break; }
        if (it >= maxit) { status = 1; break; }
        if (it > 0) info->restarts++;
        for (int i = 0; i < n; ++i) V[0][i] = r[i] / beta;
        memset(g, 0, sizeof(double) * (m + 1)); g[0] = beta;
        int k = 0, breakdown = 0;
        for (int j = 0; j < m; ++j) {
            orc_apply(h, V[j], Z[j]);
            orc_apply_operator(h, Z[j], w);
            for (int i = 0; i <= j; ++i) {                 /* MGS */
                double hij = dot(w, V[i], n);
                H[(size_t)j * (m + 1) + i] = hij;
                OMP_ROWS
                for (int t = 0; t < n; ++t) w[t] -= hij * V[i][t];
            }
            double hn = sqrt(dot(w, w, n));
            H[(size_t)j * (m + 1) + j + 1] = hn;
            if (hn != 0.0) {
                OMP_ROWS
                for (int t = 0; t < n; ++t) V[j + 1][t] = w[t] / hn;
            }
            else breakdown = 1;
            for (int i = 0; i < j; ++i) {                  /* apply previous Givens rotations */
                double a = H[(size_t)j * (m + 1) + i], c = H[(size_t)j * (m + 1) + i + 1];
                H[(size_t)j * (m + 1) + i] = cs[i] * a + sn[i] * c;
                H[(size_t)j * (m + 1) + i + 1] = -sn[i] * a + cs[i] * c;
            }
            double a = H[(size_t)j * (m + 1) + j], c = H[(size_t)j * (m + 1) + j + 1];
            double rho = hypot(a, c);
            cs[j] = a / rho; sn[j] = c / rho;
            H[(size_t)j * (m + 1) + j] = rho; H[(size_t)j * (m + 1) + j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j]; g[j] = cs[j] * g[j];
            ++it; k = j + 1;
            info->est_relres = fabs(g[j + 1]) / bn;
            if (!isfinite(hn)) { status = 2; breakdown = 1; }
            if (fabs(g[j + 1]) <= rtol * bn || it >= maxit || breakdown) break;
        }
        for (int i = k - 1; i >= 0; --i) {                 /* H y = g */
            double s = g[i];
            for (int t = i + 1; t < k; ++t) s -= H[(size_t)t * (m + 1) + i] * yv[t];
            yv[i] = s / H[(size_t)i * (m + 1) + i];
        }
        for (int i = 0; i < k; ++i) {
            OMP_ROWS
            for (int t = 0; t < n; ++t) x[t] += yv[i] * Z[i][t];
        }
        if (status == 2) break;
        if (breakdown && k == 0) break;
    }
done:
    info->iterations = it; info->status = status;
    info->t_solve = now_s() - t0;
    for (int j = 0; j <= m; ++j) free(V[j]);
    for (int j = 0; j < m; ++j) free(Z[j]);
    free(V); free(Z); free(H); free(cs); free(sn); free(g); free(yv); free(r); free(w);
    return status;
}

/* ---------------- diagnostics / parity hooks ---------------- */
int orc_num_levels(orc *h, int which) { ohier *H = which ? h->pres : h->mech; return H ? H->nl : 0; }

static void level_sizes(ohier *H, int lvl, int64_t out[6])
{
    olevel *L = &H->L[lvl];
    out[0] = L->A.n; out[1] = mnnz(&L->A); out[2] = L->nagg; out[3] = L->P.rp ? mnnz(&L->P) : 0; out[4] = H->nc; out[5] = L->coarsest;
}
static void level_export(ohier *H, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v, int32_t *agg,
                         int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1)
{
    olevel *L = &H->L[lvl];
    int n = L->A.n, nc = H->nc; int64_t nz = mnnz(&L->A);
    if (A_rp) memcpy(A_rp, L->A.rp, sizeof(int32_t) * (n + 1));
    if (A_ci) memcpy(A_ci, L->A.ci, sizeof(int32_t) * nz);
    if (A_v) for (int64_t q = 0; q < nz; ++q) for (int c = 0; c < nc; ++c) A_v[q * nc + c] = L->A.v[c][q];
    if (dl1) for (int i = 0; i < n; ++i) for (int c = 0; c < nc; ++c) dl1[(int64_t)i * nc + c] = L->dl1[c][i];
    if (L->coarsest || !L->agg) return;
    if (agg) memcpy(agg, L->agg, sizeof(int32_t) * n);
    int64_t pz = mnnz(&L->P);
    if (P_rp) memcpy(P_rp, L->P.rp, sizeof(int32_t) * (n + 1));
    if (P_ci) memcpy(P_ci, L->P.ci, sizeof(int32_t) * pz);
    if (P_v) for (int64_t q = 0; q < pz; ++q) for (int c = 0; c < nc; ++c) P_v[q * nc + c] = L->P.v[c][q];
}
void orc_level_sizes(orc *h, int which, int lvl, int64_t out[6]) { level_sizes(which ? h->pres : h->mech, lvl, out); }
int orc_level_colour(orc *h, int which, int lvl, int32_t *colour) { return orc_amg_level_colour(which ? h->pres : h->mech, lvl, colour); }
void orc_level_export(orc *h, int which, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v,
                      int32_t *agg, int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1)
{ level_export(which ? h->pres : h->mech, lvl, A_rp, A_ci, A_v, agg, P_rp, P_ci, P_v, dl1); }

void orc_counters(orc *h, int64_t out[4])
{
    out[0] = h->skipped_dss;
    out[1] = h->perturbed + (h->ilu ? h->ilu->perturbed : 0) + (h->mech ? h->mech->perturbed : 0) + (h->pres ? h->pres->perturbed : 0);
    out[2] = (h->mech ? h->mech->fallbacks : 0) + (h->pres ? h->pres->fallbacks : 0);
    out[3] = 0;
}
void orc_get_spp(orc *h, double *Dss, int32_t *rp, int32_t *ci, double *v)
{
    if (Dss) memcpy(Dss, h->Dss, sizeof(double) * h->Nc);
    if (rp) memcpy(rp, h->Spp.rp, sizeof(int32_t) * (h->Nc + 1));
    if (ci) memcpy(ci, h->Spp.ci, sizeof(int32_t) * mnnz(&h->Spp));
    if (v) memcpy(v, h->Spp.v[0], sizeof(double) * mnnz(&h->Spp));
}

void orc_get_cpr(orc *h, double *Dss, double *Dps, double *fs_eff)
{
    if (Dss) memcpy(Dss, h->Dss, sizeof(double) * h->Nc);
    if (Dps) memcpy(Dps, h->Dps, sizeof(double) * h->Nc);
    if (fs_eff) memcpy(fs_eff, h->fs_eff, sizeof(double) * 2 * h->Nc);
}

static int bsr_same_pattern(const obsr *B, const int32_t *rp, const int32_t *ci)
{
    for (int i = 0; i <= B->nr; ++i) if (B->rp[i] != rp[i]) return 0;
    for (int64_t q = 0; q < B->rp[B->nr]; ++q) if (B->ci[q] != ci[q]) return 0;
    return 1;
}
/* a Newton step's new Jacobian values on the same patterns (NEXT-f1): the operator uses them at once; the flow
 * setup products follow with orc_setup_flow, the mechanics hierarchy stays as built */
int orc_update_values(orc *h, const orc_desc *d)
{
    obsr *B[4] = {&h->uu, &h->uf, &h->fu, &h->ff};
    const int32_t *rp[4] = {d->uu_rowptr, d->uf_rowptr, d->fu_rowptr, d->ff_rowptr};
    const int32_t *ci[4] = {d->uu_col, d->uf_col, d->fu_col, d->ff_col};
    const double *v[4] = {d->uu_val, d->uf_val, d->fu_val, d->ff_val};
    for (int k = 0; k < 4; ++k) if (!bsr_same_pattern(B[k], rp[k], ci[k])) return -1;
    for (int k = 0; k < 4; ++k) memcpy(B[k]->v, v[k], sizeof(double) * B[k]->bm * B[k]->bn * B[k]->rp[B[k]->nr]);
    memcpy(h->fs, d->fs, sizeof(double) * 2 * h->Nc);
    return 0;
}

void orc_destroy(orc *h)
{
    if (!h) return;
    bsr_free(&h->uu); bsr_free(&h->uf); bsr_free(&h->fu); bsr_free(&h->ff); bsr_free(&h->Sff);
    free(h->fs);
    mcsr *m[] = {&h->Ass, &h->Asp, &h->Aps, &h->App, &h->Asp_fs, &h->App_fs, &h->Asu, &h->Apu, &h->Spp};
    for (size_t i = 0; i < sizeof(m) / sizeof(m[0]); ++i) mcsr_free(m[i]);
    free(h->Dss); free(h->Dps); free(h->fs_eff);
    amg_free(h->mech); amg_free(h->pres); orc_ilu_free(h->ilu);
    free(h->dense_uu); free(h->dense_pp); free(h->dense_ff); free(h->dense_schur);
    free(h->piv_uu); free(h->piv_pp); free(h->piv_ff); free(h->piv_schur);
    free(h);
}

/* ---------------- standalone AMG (pins) ---------------- */
void *orc_amg_build(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb, const orc_opts *o)
{
    mcsr A; mcsr_alloc(&A, n, n, nc, rp[n]);
    memcpy(A.rp, rp, sizeof(int32_t) * (n + 1)); memcpy(A.ci, ci, sizeof(int32_t) * rp[n]);
    for (int64_t q = 0; q < rp[n]; ++q) for (int c = 0; c < nc; ++c) A.v[c][q] = v[q * nc + c];
    orc_opts dflt; if (!o) { orc_default_opts(&dflt); o = &dflt; }
    ohier *H = amg_build(&A, zb, NULL, o);
    mcsr_free(&A);
    return H;
}
void *orc_amg_build_coloured(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb,
                             const int32_t *colour0, const orc_opts *o)
{
    mcsr A; mcsr_alloc(&A, n, n, nc, rp[n]);
    memcpy(A.rp, rp, sizeof(int32_t) * (n + 1)); memcpy(A.ci, ci, sizeof(int32_t) * rp[n]);
    for (int64_t q = 0; q < rp[n]; ++q) for (int c = 0; c < nc; ++c) A.v[c][q] = v[q * nc + c];
    orc_opts dflt; if (!o) { orc_default_opts(&dflt); o = &dflt; }
    ohier *H = amg_build(&A, zb, colour0, o);
    mcsr_free(&A);
    return H;
}
void orc_amg_vcycle(void *hier, const double *b, double *x)
{
    ohier *H = (ohier *)hier; int n = H->L[0].A.n;
    double *bc = (double *)xmalloc(sizeof(double) * n), *xc = (double *)xmalloc(sizeof(double) * n);
    for (int c = 0; c < H->nc; ++c) {
        for (int i = 0; i < n; ++i) bc[i] = b[(int64_t)i * H->nc + c];
        vcycle(H, 0, c, bc, xc);
        for (int i = 0; i < n; ++i) x[(int64_t)i * H->nc + c] = xc[i];
    }
    free(bc); free(xc);
}
int orc_amg_levels(void *hier) { return ((ohier *)hier)->nl; }
void orc_amg_level_sizes(void *hier, int lvl, int64_t out[6]) { level_sizes((ohier *)hier, lvl, out); }
void orc_amg_level_export(void *hier, int lvl, int32_t *A_rp, int32_t *A_ci, double *A_v,
                          int32_t *agg, int32_t *P_rp, int32_t *P_ci, double *P_v, double *dl1)
{ level_export((ohier *)hier, lvl, A_rp, A_ci, A_v, agg, P_rp, P_ci, P_v, dl1); }
void orc_amg_free(void *hier) { amg_free((ohier *)hier); }
/* pins: the GS colouring of a level (returns the number of colours; 0 when the smoother is not GS) and the
 * hybrid l1 diagonal (NULL ok) */
int orc_amg_level_colour(void *hier, int lvl, int32_t *colour)
{
    ohier *H = (ohier *)hier;
    olevel *L = &H->L[lvl];
    if (lvl >= H->nl || !L->color) return 0;
    if (colour) memcpy(colour, L->color, sizeof(int32_t) * L->A.n);
    return L->ncolor;
}
int orc_amg_level_gs(void *hier, int lvl, double *dh)
{
    ohier *H = (ohier *)hier;
    olevel *L = &H->L[lvl];
    if (lvl >= H->nl || !L->color) return -1;
    if (dh && L->gs_block) for (int i = 0; i < L->A.n; ++i) for (int c = 0; c < H->nc; ++c) dh[(int64_t)i * H->nc + c] = L->dh[c][i];
    return L->gs_block;
}
/* pins: the MIS(2) state, the phase-1 aggregates and omega_c of a non-coarsest level (returns -1 otherwise) */
int orc_amg_level_detail(void *hier, int lvl, int32_t *st, int32_t *ph1, double *omega)
{
    ohier *H = (ohier *)hier;
    olevel *L = &H->L[lvl];
    if (lvl >= H->nl || L->coarsest || !L->st) return -1;
    if (st) memcpy(st, L->st, sizeof(int32_t) * L->A.n);
    if (ph1) memcpy(ph1, L->ph1, sizeof(int32_t) * L->A.n);
    if (omega) for (int c = 0; c < H->nc; ++c) omega[c] = L->omega[c];
    return 0;
}
/* pins: the symmetrised strength graph E (one byte per stored entry) of R-strength */
int orc_strength(int n, int nc, const int32_t *rp, const int32_t *ci, const double *v, const int32_t *zb,
                 double theta, uint8_t *E)
{
    mcsr A; mcsr_alloc(&A, n, n, nc, rp[n]);
    memcpy(A.rp, rp, sizeof(int32_t) * (n + 1)); memcpy(A.ci, ci, sizeof(int32_t) * rp[n]);
    for (int64_t q = 0; q < rp[n]; ++q) for (int c = 0; c < nc; ++c) A.v[c][q] = v[q * nc + c];
    int rc = strength(&A, zb, theta, E);
    mcsr_free(&A);
    return rc;
}

/*
 * meshfree_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `meshfree` hot path, used as the parity
 * checker for the CUDA kernels and as the CPU baseline arm of bench.py.
 * Nothing in the product path (paper_1912_13282_b200/) links or calls this.
 *
 * Every routine cites the reference function it restates
 * (paths relative to the reference checkout, pkg/src/meshfree/...).
 *
 * Arithmetic contract: compiled with -ffp-contract=off (no FMA), IEEE division
 * and sqrt, and glibc `pow` called with run-time exponents, which is exactly
 * what the numba-compiled reference kernel does (LLVM, no FMA, libm pow).
 * The restatement is therefore bit-identical to the reference on the same
 * host; tests/test_oracle_pins.py checks that against golden vectors produced
 * by the live reference (tests/golden/, oracle/gen_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXD 3

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* numba integer power of a float base (numba/cpython/numbers.py int_power):
 * r = 1; while exp: if exp & 1: r *= a; exp >>= 1; a *= a; invert if b < 0. */
static double numba_int_power(double a, int64_t b) {
    double r = 1.0;
    int invert = b < 0;
    uint64_t e = (uint64_t)(invert ? -b : b);
    if (e > 0x10000) return pow(a, (double)b);
    while (e != 0) {
        if (e & 1) r *= a;
        e >>= 1;
        a *= a;
    }
    return invert ? 1.0 / r : r;
}

/* ------------------------------------------------------------------------ */
/* _solve_multi (_phs_batch.py:142-184): row-pivoted elimination, solution   */
/* left in b.  a is s x s row-major, b is s x nr row-major.                  */
/* ------------------------------------------------------------------------ */
static int solve_multi(double* a, double* b, int s, int nr) {
    for (int col = 0; col < s; ++col) {
        int piv = col;
        double big = fabs(a[(size_t)col * s + col]);
        for (int r = col + 1; r < s; ++r) {
            double v = fabs(a[(size_t)r * s + col]);
            if (v > big) { big = v; piv = r; }
        }
        if (big == 0.0 || !isfinite(big)) return 0;
        if (piv != col) {
            for (int cc = col; cc < s; ++cc) {
                double t = a[(size_t)col * s + cc];
                a[(size_t)col * s + cc] = a[(size_t)piv * s + cc];
                a[(size_t)piv * s + cc] = t;
            }
            for (int cc = 0; cc < nr; ++cc) {
                double t = b[(size_t)col * nr + cc];
                b[(size_t)col * nr + cc] = b[(size_t)piv * nr + cc];
                b[(size_t)piv * nr + cc] = t;
            }
        }
        double inv = 1.0 / a[(size_t)col * s + col];
        for (int r = col + 1; r < s; ++r) {
            double fac = a[(size_t)r * s + col] * inv;
            if (fac != 0.0) {
                for (int cc = col + 1; cc < s; ++cc)
                    a[(size_t)r * s + cc] -= fac * a[(size_t)col * s + cc];
                for (int cc = 0; cc < nr; ++cc)
                    b[(size_t)r * nr + cc] -= fac * b[(size_t)col * nr + cc];
            }
        }
    }
    for (int col = s - 1; col >= 0; --col) {
        double inv = 1.0 / a[(size_t)col * s + col];
        for (int cc = 0; cc < nr; ++cc) {
            double acc = b[(size_t)col * nr + cc];
            for (int r = col + 1; r < s; ++r) acc -= a[(size_t)col * s + r] * b[(size_t)r * nr + cc];
            b[(size_t)col * nr + cc] = acc * inv;
        }
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* _batch_numba (_phs_batch.py:186-302).                                     */
/*   pts (N,d) f64; rows (m) i64; stencils (m,n) i64; expos (l,d) i64;       */
/*   base_bot (nf,l) f64; kinds/ax_a/ax_b/orders (nf) i64.                   */
/*   out (m,nf,n) f64; fail (m) i8 (0 ok, 1 singular/non-finite, 2 scale).   */
/* ------------------------------------------------------------------------ */
int oracle_phs_weights(const double* pts, int64_t N, int d,
                       const int64_t* rows, const int64_t* stencils, int64_t m, int n,
                       int64_t k, int even, const int64_t* expos, int l,
                       const double* base_bot, const int64_t* kinds, const int64_t* ax_a,
                       const int64_t* ax_b, const int64_t* orders, int nf, int scale_code,
                       double* out, int8_t* fail, int threads) {
    (void)N;
    if (d < 1 || d > MAXD) return -1;
    set_threads(threads);
    const int size = n + l;
    int64_t idx;
#pragma omp parallel for schedule(dynamic, 64)
    for (idx = 0; idx < m; ++idx) {
        double* local = (double*)malloc(sizeof(double) * (size_t)n * d);
        double* sys = (double*)malloc(sizeof(double) * (size_t)size * size);
        double* rhs = (double*)malloc(sizeof(double) * (size_t)size * (nf > 0 ? nf : 1));
        int status = 0;
        const double* center = pts + rows[idx] * d;
        for (int j = 0; j < n; ++j)
            for (int a = 0; a < d; ++a)
                local[j * d + a] = pts[stencils[idx * n + j] * d + a] - center[a];

        double s = 1.0;
        if (scale_code != 0) {
            double best = -1.0;
            for (int j = 0; j < n; ++j) {
                double r2 = 0.0;
                for (int a = 0; a < d; ++a) r2 += local[j * d + a] * local[j * d + a];
                double r = sqrt(r2);
                if (scale_code == 1) {
                    if (r > 0.0 && (best < 0.0 || r < best)) best = r;
                } else {
                    if (r > best) best = r;
                }
            }
            if (best <= 0.0) status = 2;
            else s = best;
        }

        if (status == 0) {
            for (int j = 0; j < n; ++j)
                for (int a = 0; a < d; ++a) local[j * d + a] /= s;

            memset(sys, 0, sizeof(double) * (size_t)size * size);
            const double kf = (double)k;
            for (int i = 0; i < n; ++i) {
                for (int j = 0; j < n; ++j) {
                    double r2 = 0.0;
                    for (int a = 0; a < d; ++a) {
                        double diff = local[i * d + a] - local[j * d + a];
                        r2 += diff * diff;
                    }
                    double r = sqrt(r2);
                    if (even)
                        sys[(size_t)i * size + j] = r > 0.0 ? numba_int_power(r, k) * log(r) : 0.0;
                    else
                        sys[(size_t)i * size + j] = pow(r, kf);
                }
            }
            for (int j = 0; j < l; ++j) {
                for (int i = 0; i < n; ++i) {
                    double q = 1.0;
                    for (int a = 0; a < d; ++a)
                        if (expos[j * d + a]) q *= numba_int_power(local[i * d + a], expos[j * d + a]);
                    sys[(size_t)i * size + n + j] = q;
                    sys[(size_t)(n + j) * size + i] = q;
                }
            }

            memset(rhs, 0, sizeof(double) * (size_t)size * nf);
            for (int j = 0; j < n; ++j) {
                double r2 = 0.0;
                for (int a = 0; a < d; ++a) r2 += local[j * d + a] * local[j * d + a];
                double r = sqrt(r2);
                double val, d1r, d2v;
                if (r > 0.0) {
                    if (even) {
                        double lg = log(r);
                        val = numba_int_power(r, k) * lg;
                        d1r = pow(r, kf - 2.0) * (kf * lg + 1.0);
                        d2v = pow(r, kf - 2.0) * ((double)(k * k - k) * lg + 2.0 * kf - 1.0);
                    } else {
                        val = pow(r, kf);
                        d1r = kf * pow(r, kf - 2.0);
                        d2v = kf * (kf - 1.0) * pow(r, kf - 2.0);
                    }
                } else {
                    val = 0.0; d1r = 0.0; d2v = 0.0;
                }
                for (int f = 0; f < nf; ++f) {
                    int64_t kind = kinds[f];
                    double top;
                    if (kind == 0) {
                        top = val;
                    } else if (kind == 1) {
                        top = d1r * (-local[j * d + ax_a[f]]);
                    } else if (kind == 2) {
                        double ee = r > 0.0 ? local[j * d + ax_a[f]] * local[j * d + ax_b[f]] / r2 : 0.0;
                        double delta = ax_a[f] == ax_b[f] ? 1.0 : 0.0;
                        top = d2v * ee + d1r * (delta - ee);
                    } else {
                        top = d2v + (double)(d - 1) * d1r;
                    }
                    rhs[(size_t)j * nf + f] = top;
                }
            }
            for (int f = 0; f < nf; ++f) {
                double fac = pow(s, -(double)orders[f]);
                for (int j = 0; j < n; ++j) rhs[(size_t)j * nf + f] *= fac;
                for (int j = 0; j < l; ++j) rhs[(size_t)(n + j) * nf + f] = base_bot[f * l + j] * fac;
            }

            if (solve_multi(sys, rhs, size, nf)) {
                for (int f = 0; f < nf; ++f)
                    for (int j = 0; j < n; ++j) {
                        double v = rhs[(size_t)j * nf + f];
                        if (!isfinite(v)) status = 1;
                        out[(idx * nf + f) * n + j] = v;
                    }
            } else {
                status = 1;
            }
        }
        fail[idx] = (int8_t)status;
        free(local); free(sys); free(rhs);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* find_closest_stencils (geometry/stencils.py:19-93), exact restatement.    */
/*                                                                           */
/* The reference queries a kd-tree for k = min(n+8, P) candidates, re-sorts  */
/* them by (d2_E, index) where d2_E is numpy einsum's rounding order, and    */
/* falls back to a ball query ordered by (d2_S, index) when the k-th and     */
/* n-th candidates tie to 1e-12 (the "straddle" rows).  Because the final    */
/* order is an exact function of the keys, the result equals: top-n of the   */
/* pool under (d2_E, index), or under (d2_S, index) for straddle rows,       */
/* followed by the self-first fix.  This restatement finds the exact top-k   */
/* with a uniform cell grid instead of a kd-tree.                            */
/* ------------------------------------------------------------------------ */

/* numpy.einsum("tkd,tkd->tk") summation order on this numpy build
 * (probed: 1D x0; 2D x0+x1; 3D (x0+x2)+x1). */
static inline double d2_einsum(const double* dd, int d) {
    if (d == 1) return dd[0] * dd[0];
    if (d == 2) return dd[0] * dd[0] + dd[1] * dd[1];
    return (dd[0] * dd[0] + dd[2] * dd[2]) + dd[1] * dd[1];
}
/* np.sum(diff ** 2, axis=1): sequential over axes. */
static inline double d2_seqsum(const double* dd, int d) {
    double s = dd[0] * dd[0];
    for (int a = 1; a < d; ++a) s = s + dd[a] * dd[a];
    return s;
}

typedef struct { double d2; int64_t idx; int64_t ppos; } cand_t;

static inline int cand_lt(const cand_t* x, const cand_t* y) {
    if (x->d2 != y->d2) return x->d2 < y->d2;
    if (x->idx != y->idx) return x->idx < y->idx;
    return x->ppos < y->ppos;
}

/* keep the K smallest of buf[0..cnt) in sorted order at buf[0..K) */
static void top_k(cand_t* buf, int64_t cnt, int64_t K) {
    /* insertion into a sorted prefix: fine for the small K used here */
    int64_t have = 0;
    for (int64_t i = 0; i < cnt; ++i) {
        cand_t c = buf[i];
        if (have == K && !cand_lt(&c, &buf[K - 1])) continue;
        int64_t p = have < K ? have : K - 1;
        while (p > 0 && cand_lt(&c, &buf[p - 1])) { buf[p] = buf[p - 1]; --p; }
        buf[p] = c;
        if (have < K) ++have;
    }
}

typedef struct {
    int d;
    double lo[MAXD], cw[MAXD], inv[MAXD];
    int64_t G[MAXD];
    int64_t ncell;
    int64_t* start;   /* ncell + 1 */
    int64_t* item;    /* P: pool positions sorted by cell */
} grid_t;

static int64_t cell_coord(const grid_t* g, int a, double x) {
    double t = (x - g->lo[a]) * g->inv[a];
    if (!(t >= 0.0)) return 0;
    if (t >= (double)g->G[a]) return g->G[a] - 1;
    int64_t c = (int64_t)t;
    return c < g->G[a] ? c : g->G[a] - 1;
}

static void grid_build(grid_t* g, const double* pos, int d, const int64_t* pool, int64_t P) {
    g->d = d;
    double lo[MAXD], hi[MAXD];
    for (int a = 0; a < d; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
    for (int64_t i = 0; i < P; ++i)
        for (int a = 0; a < d; ++a) {
            double x = pos[pool[i] * d + a];
            if (x < lo[a]) lo[a] = x;
            if (x > hi[a]) hi[a] = x;
        }
    double vol = 1.0; int nd = 0;
    for (int a = 0; a < d; ++a) if (hi[a] > lo[a]) { vol *= hi[a] - lo[a]; ++nd; }
    double w = nd ? pow(vol * 2.0 / (double)P, 1.0 / nd) : 1.0;
    g->ncell = 1;
    for (int a = 0; a < d; ++a) {
        double ext = hi[a] - lo[a];
        int64_t G = 1;
        if (ext > 0.0 && w > 0.0) {
            double gg = floor(ext / w);
            if (gg < 1.0) gg = 1.0;
            if (gg > 4096.0) gg = 4096.0;
            G = (int64_t)gg;
        }
        g->G[a] = G;
        g->lo[a] = lo[a];
        g->cw[a] = ext > 0.0 ? ext / (double)G : 0.0;
        g->inv[a] = ext > 0.0 ? (double)G / ext : 0.0;
        g->ncell *= G;
    }
    g->start = (int64_t*)calloc((size_t)g->ncell + 1, sizeof(int64_t));
    g->item = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    int64_t* cid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    for (int64_t i = 0; i < P; ++i) {
        int64_t c = 0;
        for (int a = 0; a < d; ++a) c = c * g->G[a] + cell_coord(g, a, pos[pool[i] * d + a]);
        cid[i] = c;
        g->start[c + 1]++;
    }
    for (int64_t c = 0; c < g->ncell; ++c) g->start[c + 1] += g->start[c];
    int64_t* fillp = (int64_t*)malloc(sizeof(int64_t) * (size_t)g->ncell);
    for (int64_t c = 0; c < g->ncell; ++c) fillp[c] = g->start[c];
    for (int64_t i = 0; i < P; ++i) g->item[fillp[cid[i]]++] = i;
    free(fillp); free(cid);
}

/* gather all pool points of the cell box [clo, chi] with their d2_E keys */
static int64_t gather_box(const grid_t* g, const double* pos, const int64_t* pool,
                          const double* p, const int64_t* clo, const int64_t* chi,
                          cand_t** buf, int64_t* cap) {
    int d = g->d;
    int64_t cnt = 0;
    int64_t c[MAXD];
    for (int a = 0; a < d; ++a) c[a] = clo[a];
    for (;;) {
        int64_t cell = 0;
        for (int a = 0; a < d; ++a) cell = cell * g->G[a] + c[a];
        for (int64_t q = g->start[cell]; q < g->start[cell + 1]; ++q) {
            int64_t pp = g->item[q];
            int64_t id = pool[pp];
            double dd[MAXD];
            for (int a = 0; a < d; ++a) dd[a] = pos[id * d + a] - p[a];
            if (cnt == *cap) { *cap *= 2; *buf = (cand_t*)realloc(*buf, sizeof(cand_t) * (size_t)*cap); }
            (*buf)[cnt].d2 = d2_einsum(dd, d);
            (*buf)[cnt].idx = id;
            (*buf)[cnt].ppos = pp;
            ++cnt;
        }
        int a = d - 1;
        while (a >= 0 && c[a] == chi[a]) { c[a] = clo[a]; --a; }
        if (a < 0) break;
        ++c[a];
    }
    return cnt;
}

int oracle_knn(const double* pos, int64_t N, int d, const int64_t* targets, int64_t T,
               const int64_t* pool, int64_t P, int n, int64_t* out, int64_t* n_straddle,
               int threads) {
    if (d < 1 || d > MAXD || n < 1 || n > P) return -1;
    set_threads(threads);
    grid_t g;
    grid_build(&g, pos, d, pool, P);
    uint8_t* in_pool = (uint8_t*)calloc((size_t)N, 1);
    for (int64_t i = 0; i < P; ++i) in_pool[pool[i]] = 1;
    const int64_t K = (int64_t)n + 8 < P ? (int64_t)n + 8 : P;
    int64_t straddles = 0;
    int64_t t;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : straddles)
    for (t = 0; t < T; ++t) {
        int64_t cap = 1024;
        cand_t* buf = (cand_t*)malloc(sizeof(cand_t) * (size_t)cap);
        const double* p = pos + targets[t] * d;
        int64_t home[MAXD];
        for (int a = 0; a < d; ++a) home[a] = cell_coord(&g, a, p[a]);
        int64_t rho = 1;
        int64_t cnt;
        for (;;) {
            int64_t clo[MAXD], chi[MAXD];
            double inner = INFINITY;
            for (int a = 0; a < d; ++a) {
                clo[a] = home[a] - rho < 0 ? 0 : home[a] - rho;
                chi[a] = home[a] + rho > g.G[a] - 1 ? g.G[a] - 1 : home[a] + rho;
                if (clo[a] > 0) {
                    double face = g.lo[a] + (double)clo[a] * g.cw[a];
                    double dist = p[a] - face;
                    if (dist < inner) inner = dist < 0.0 ? 0.0 : dist;
                }
                if (chi[a] < g.G[a] - 1) {
                    double face = g.lo[a] + (double)(chi[a] + 1) * g.cw[a];
                    double dist = face - p[a];
                    if (dist < inner) inner = dist < 0.0 ? 0.0 : dist;
                }
            }
            cnt = gather_box(&g, pos, pool, p, clo, chi, &buf, &cap);
            if (cnt >= K) {
                top_k(buf, cnt, K);
                if (inner == INFINITY || buf[K - 1].d2 < inner * inner * (1.0 - 1e-12)) break;
            }
            ++rho;
        }
        int64_t* row = out + t * n;
        for (int j = 0; j < n; ++j) row[j] = buf[j].idx;
        if (K > n) {
            double edge = buf[n - 1].d2;
            if (fabs(buf[K - 1].d2 - edge) <= 1e-18 + 1e-12 * edge) {
                /* straddle: order the whole pool by (np.sum d2, index); the
                 * reference's ball query contains this top-n (stencils.py:67-75) */
                ++straddles;
                int64_t need = P;
                if (need > cap) { cap = need; buf = (cand_t*)realloc(buf, sizeof(cand_t) * (size_t)cap); }
                for (int64_t i = 0; i < P; ++i) {
                    double dd[MAXD];
                    int64_t id = pool[i];
                    for (int a = 0; a < d; ++a) dd[a] = pos[id * d + a] - p[a];
                    buf[i].d2 = d2_seqsum(dd, d);
                    buf[i].idx = id;
                    buf[i].ppos = i;
                }
                top_k(buf, P, n);
                for (int j = 0; j < n; ++j) row[j] = buf[j].idx;
            }
        }
        /* self-first fix (stencils.py:77-91) */
        int64_t tg = targets[t];
        if (in_pool[tg] && row[0] != tg) {
            int hit = -1;
            for (int j = 0; j < n; ++j) if (row[j] == tg) { hit = j; break; }
            if (hit >= 0) {
                for (int j = hit; j > 0; --j) row[j] = row[j - 1];
            } else {
                for (int j = n - 1; j > 0; --j) row[j] = row[j - 1];
            }
            row[0] = tg;
        }
        free(buf);
    }
    if (n_straddle) *n_straddle = straddles;
    free(in_pool); free(g.start); free(g.item);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* WeightStore.matrix (storage.py:156-170): canonical CSR, rows ascending,   */
/* columns ascending (stable lexsort), rows only for stored nodes.           */
/* rows (m) i64, stencils (m,n) i64, w (m,n) f64 -> indptr (N+1) i64,        */
/* indices (m*n) i64, data (m*n) f64.                                        */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t col; int64_t pos; } colpos_t;
static int colpos_cmp(const void* a, const void* b) {
    const colpos_t* x = (const colpos_t*)a;
    const colpos_t* y = (const colpos_t*)b;
    if (x->col != y->col) return x->col < y->col ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

int oracle_csr_canonical(const int64_t* rows, const int64_t* stencils, const double* w,
                         int64_t m, int n, int64_t N, int64_t* indptr, int64_t* indices,
                         double* data) {
    int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    for (int64_t i = 0; i < N; ++i) slot[i] = -1;
    for (int64_t r = 0; r < m; ++r) {
        if (rows[r] < 0 || rows[r] >= N || slot[rows[r]] >= 0) { free(slot); return -1; }
        slot[rows[r]] = r;
    }
    indptr[0] = 0;
    for (int64_t i = 0; i < N; ++i) indptr[i + 1] = indptr[i] + (slot[i] >= 0 ? n : 0);
    colpos_t* tmp = (colpos_t*)malloc(sizeof(colpos_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < N; ++i) {
        int64_t r = slot[i];
        if (r < 0) continue;
        for (int j = 0; j < n; ++j) { tmp[j].col = stencils[r * n + j]; tmp[j].pos = j; }
        qsort(tmp, (size_t)n, sizeof(colpos_t), colpos_cmp);
        for (int j = 0; j < n; ++j) {
            indices[indptr[i] + j] = tmp[j].col;
            data[indptr[i] + j] = w[r * n + tmp[j].pos];
        }
    }
    free(tmp); free(slot);
    return 0;
}

/* scipy csr_matvec as used by WeightStore.apply_all (storage.py:186-188):   */
/* y_i = sum over the row in storage order, sequential from 0.0, no FMA.    */
int oracle_apply(const int64_t* indptr, const int64_t* indices, const double* data,
                 const double* u, double* y, int64_t N, int threads) {
    set_threads(threads);
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < N; ++i) {
        double acc = 0.0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) acc = acc + data[p] * u[indices[p]];
        y[i] = acc;
    }
    return 0;
}

/* run_heat_explicit step loop (drivers.py:87-110) for step-invariant data:  */
/* interior mask, Dirichlet mask + values, optional per-node source f.       */
/* Returns 0, or the 1-based step at which max|u| > 1e12 / non-finite, with  */
/* the peak written to *peak_out.  u is updated in place.                    */
int64_t oracle_heat_steps(const int64_t* indptr, const int64_t* indices, const double* data,
                          int64_t N, const uint8_t* interior, const uint8_t* dirichlet,
                          const double* g_dir, const double* source, double dt, double D,
                          int64_t steps, double* u, double* peak_out, int threads) {
    set_threads(threads);
    double* un = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    /* Dirichlet data is applied to the initial field (drivers.py:84-85) */
    for (int64_t i = 0; i < N; ++i) if (dirichlet[i]) u[i] = g_dir[i];
    for (int64_t step = 0; step < steps; ++step) {
        double peak = 0.0;
        int nan_seen = 0;
        int64_t i;
#pragma omp parallel for schedule(static) reduction(max : peak) reduction(| : nan_seen)
        for (i = 0; i < N; ++i) {
            double v = u[i];
            if (interior[i]) {
                double acc = 0.0;
                for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) acc = acc + data[p] * u[indices[p]];
                double f = source ? source[i] : 0.0;
                v = u[i] + dt * (D * acc + f);
            }
            if (dirichlet[i]) v = g_dir[i];
            un[i] = v;
            double av = fabs(v);
            if (av != av) nan_seen = 1;
            else if (av > peak) peak = av;
        }
        memcpy(u, un, sizeof(double) * (size_t)N);
        if (nan_seen || !isfinite(peak) || peak > 1e12) {
            if (peak_out) *peak_out = nan_seen ? NAN : peak;
            free(un);
            return step + 1;
        }
    }
    free(un);
    return 0;
}

// Stencil selection: uniform-grid cell-list kNN with warp-level exact top-k.
//
// Replaces find_closest_stencils (geometry/stencils.py:19-93).  The reference
// takes a kd-tree window of k = min(n+8, P) candidates, re-orders them by
// (d2, node index) with d2 in numpy einsum's rounding order, re-selects
// "straddle" rows (k-th and n-th candidates equal to 1e-12) from a ball query
// ordered by (np.sum d2, index), and moves the target to slot 0.  The final
// order is an exact function of those keys, so this kernel computes the same
// mathematical object directly:
//
//   1. pool points are counting-sorted into a uniform grid (~2 per cell);
//   2. one warp per target (targets processed in cell order for locality)
//      gathers the points of a cube of cells around the target, whose inner
//      radius bounds every point left outside;
//   3. the K smallest keys are found exactly: bisection on d2 shrinks the
//      candidate set to a window just above K, and every survivor's rank by
//      (d2, index) is counted against the packed survivor keys in shared
//      memory; the cube grows until the K-th key is provably inside it;
//   4. straddle rows are re-run with the sequential-sum metric (K = n);
//   5. the self-first rule is applied before the row is written.
#include <cstdio>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <mutex>

#include "common.cuh"

namespace mf {

constexpr double KNN_OCC = 2.0;   // mean pool points per grid cell (wide stencils take a coarser grid: GridParams::occ)
constexpr int KNN_WARPS = 4;      // warps per block
constexpr int KNN_SCAP = 256;     // survivor capacity per warp (shared memory)
constexpr int KNN_RMAX = 255;     // cell-row ranges per cube held in shared memory
constexpr int KNN_WIN = 16;       // kernel-variant choice: K + WIN > 64 takes 32 candidate rounds

struct GridParams {
    double lo[3], cw[3], inv[3];
    double occ;  // mean pool points per cell the grid was sized for (>= KNN_OCC)
    int G[3];
    int ncell;
};

struct KnnArgs {
    const double* pos;
    int d;
    const int64_t* targets;
    const GridParams* gp;
    const int32_t* start;  // ncell + 1
    const double* spos;    // pool points sorted by cell, AoS d doubles
    const int32_t* sidx;   // node index of each sorted point
    const uint8_t* in_pool;
    int n;
    int K;
    int32_t* out;
    int32_t* straddle_list;
    unsigned long long* straddle_count;
};

// numpy.einsum("tkd,tkd->tk") order on this numpy build (probed):
// 1D x0; 2D x0 + x1; 3D (x0 + x2) + x1.  np.sum order (straddle path): sequential.
template <bool SEQ>
__device__ __forceinline__ double metric(const double* q, const double* p, int d) {
    double dx = __dsub_rn(q[0], p[0]);
    double s = __dmul_rn(dx, dx);
    if (d == 1) return s;
    double dy = __dsub_rn(q[1], p[1]);
    if (d == 2) return __dadd_rn(s, __dmul_rn(dy, dy));
    double dz = __dsub_rn(q[2], p[2]);
    if (SEQ) return __dadd_rn(__dadd_rn(s, __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return __dadd_rn(__dadd_rn(s, __dmul_rn(dz, dz)), __dmul_rn(dy, dy));
}

__device__ __forceinline__ int cell_coord(const GridParams& g, int a, double x) {
    double t = (x - g.lo[a]) * g.inv[a];
    if (!(t >= 0.0)) return 0;
    if (t >= (double)g.G[a]) return g.G[a] - 1;
    int c = (int)t;
    return c < g.G[a] ? c : g.G[a] - 1;
}

__device__ __forceinline__ int cell_of(const GridParams& g, const double* x, int d) {
    int c = 0;
    for (int a = 0; a < d; ++a) c = c * g.G[a] + cell_coord(g, a, x[a]);
    return c;
}

// key order: (d2, node index, candidate id) -- the candidate id only separates
// repeated pool entries, which carry the same node index
__device__ __forceinline__ bool key_lt(double d1, int i1, int c1, double d2, int i2, int c2) {
    // branch-free: predicates combined with bitwise ops (no divergent short-circuit)
    const bool dl = d1 < d2, de = d1 == d2;
    const bool il = i1 < i2, ie = i1 == i2;
    return dl | (de & (il | (ie & (c1 < c2))));
}

__device__ __forceinline__ bool key_lt2(double d1, int i1, double d2, int i2) {
    return (d1 < d2) | ((d1 == d2) & (i1 < i2));
}

struct Box {
    int clo[3], chi[3];
    double limit;  // K-th key must be <= limit to be provably inside
    bool all;
};

__device__ __forceinline__ Box make_box(const GridParams& g, const double* p, const int* home, int rho, int d) {
    Box b;
    double inner = INFINITY;
    b.all = true;
    for (int a = 0; a < 3; ++a) {
        b.clo[a] = 0;
        b.chi[a] = 0;
    }
    for (int a = 0; a < d; ++a) {
        b.clo[a] = max(home[a] - rho, 0);
        b.chi[a] = min(home[a] + rho, g.G[a] - 1);
        if (b.clo[a] > 0) {
            b.all = false;
            double dist = p[a] - (g.lo[a] + (double)b.clo[a] * g.cw[a]);
            inner = fmin(inner, fmax(dist, 0.0));
        }
        if (b.chi[a] < g.G[a] - 1) {
            b.all = false;
            double dist = (g.lo[a] + (double)(b.chi[a] + 1) * g.cw[a]) - p[a];
            inner = fmin(inner, fmax(dist, 0.0));
        }
    }
    b.limit = b.all ? INFINITY : inner * inner * (1.0 - 1e-12);
    return b;
}

// range r of the cube: the cells along the last axis at fixed leading coordinates
__device__ __forceinline__ void range_bounds(const GridParams& g, const Box& b, int d, int r, const int32_t* start,
                                             int& lo, int& hi) {
    int lead = 0;
    int rem = r;
    int coords[2] = {0, 0};
    for (int a = d - 2; a >= 0; --a) {
        int span = b.chi[a] - b.clo[a] + 1;
        coords[a] = b.clo[a] + rem % span;
        rem /= span;
    }
    for (int a = 0; a < d - 1; ++a) lead = lead * g.G[a] + coords[a];
    int c_lo = lead * g.G[d - 1] + b.clo[d - 1];
    int c_hi = lead * g.G[d - 1] + b.chi[d - 1];
    lo = start[c_lo];
    hi = start[c_hi + 1];
}

// range r clipped to the ball of squared radius R2 around p (R2 = inf: the whole
// row): rows whose cells all lie farther than R from p are empty, the others keep
// the cells along the last axis that the ball reaches.  Monotone cell_coord makes
// every point within R of p fall in a kept cell (the radius carries a relative
// margin for the floor in cell_coord).
__device__ __forceinline__ void range_bounds_ball(const GridParams& g, const Box& b, int d, int r,
                                                  const int32_t* start, const double* p, double R2, int& lo,
                                                  int& hi) {
    int rem = r;
    int coords[2] = {0, 0};
    for (int a = d - 2; a >= 0; --a) {
        const int span = b.chi[a] - b.clo[a] + 1;
        coords[a] = b.clo[a] + rem % span;
        rem /= span;
    }
    int zl = b.clo[d - 1], zh = b.chi[d - 1];
    if (R2 < INFINITY) {
        double t2 = 0.0;
        for (int a = 0; a < d - 1; ++a) {
            const double e0 = g.lo[a] + (double)coords[a] * g.cw[a];
            const double dd = fmax(fmax(e0 - p[a], p[a] - (e0 + g.cw[a])), 0.0);
            t2 += dd * dd;
        }
        if (t2 > R2) {
            lo = hi = 0;
            return;
        }
        const double h = sqrt(R2 - t2);
        zl = max(zl, cell_coord(g, d - 1, p[d - 1] - h));
        zh = min(zh, cell_coord(g, d - 1, p[d - 1] + h));
        if (zl > zh) {
            lo = hi = 0;
            return;
        }
    }
    int lead = 0;
    for (int a = 0; a < d - 1; ++a) lead = lead * g.G[a] + coords[a];
    lo = start[lead * g.G[d - 1] + zl];
    hi = start[lead * g.G[d - 1] + zh + 1];
}

__device__ __forceinline__ int box_ranges(const Box& b, int d) {
    int R = 1;
    for (int a = 0; a < d - 1; ++a) R *= b.chi[a] - b.clo[a] + 1;
    return R;
}

constexpr int KNN_CQ = 32 * 32;  // candidate table capacity (32 * the largest MAXIT)

// survivor key, 16 bytes: one shared load per comparison
struct __align__(16) KnnKey {
    double d2;
    unsigned long long ic;  // (node index << 32) | candidate id
};

struct WarpSmem {
    int32_t roff[KNN_RMAX + 1];  // candidate offset of each range (prefix)
    int32_t rlo[KNN_RMAX];       // first item of each range
    int32_t cq[KNN_CQ];          // sorted-pool position of each candidate
    KnnKey skey[KNN_SCAP];
    double sd2[KNN_SCAP + 2];    // survivor d2 alone, padded to an even count
    int32_t sel[KNN_SCAP];
    double seld2[KNN_SCAP];
};

// Exact K smallest keys by repeated arg-min over the cube (any size, any ties).
// Writes sel/seld2[0..K) and returns the K-th d2.
template <bool SEQ, int DD>
__device__ double extract_topk(const KnnArgs& a, const Box& b, const double* p, int K, WarpSmem& sm, int lane) {
    const GridParams& g = *a.gp;
    constexpr int d = DD;
    const int R = box_ranges(b, d);
    double pd = -INFINITY;
    int pi = -1, pc = -1;
    for (int k = 0; k < K; ++k) {
        double bd = INFINITY;
        int bi = 0x7fffffff, bc = 0x7fffffff;
        int cid = 0;
        for (int r = 0; r < R; ++r) {
            int lo, hi;
            range_bounds(g, b, d, r, a.start, lo, hi);
            for (int q = lo + lane; q < hi; q += 32) {
                double d2 = metric<SEQ>(a.spos + (size_t)q * d, p, d);
                int id = a.sidx[q];
                int c = cid + (q - lo);
                if (key_lt(pd, pi, pc, d2, id, c) && key_lt(d2, id, c, bd, bi, bc)) {
                    bd = d2;
                    bi = id;
                    bc = c;
                }
            }
            cid += hi - lo;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double od = __shfl_xor_sync(FULL, bd, o);
            int oi = __shfl_xor_sync(FULL, bi, o);
            int oc = __shfl_xor_sync(FULL, bc, o);
            if (key_lt(od, oi, oc, bd, bi, bc)) {
                bd = od;
                bi = oi;
                bc = oc;
            }
        }
        if (lane == 0 && k < KNN_SCAP) {
            sm.sel[k] = bi;
            sm.seld2[k] = bd;
        }
        pd = bd;
        pi = bi;
        pc = bc;
    }
    __syncwarp();
    return pd;
}

template <bool SEQ, int DD, int MAXIT>
__global__ void __launch_bounds__(KNN_WARPS * 32, 3) knn_kernel(KnnArgs a, const int32_t* __restrict__ order,
                                                            int64_t count, const unsigned long long* count_dev,
                                                            int K) {
    extern __shared__ __align__(16) unsigned char knn_smem[];  // KNN_WARPS x WarpSmem
    WarpSmem* smem = reinterpret_cast<WarpSmem*>(knn_smem);
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem& sm = smem[wib];
    const GridParams g = *a.gp;
    constexpr int d = DD;
    const int n = a.n;
    if (count_dev) count = (int64_t)*count_dev;
    // first cube: half-width ~ the K-th neighbour radius at the grid density
    // (in cells), so the inner-radius proof usually succeeds on the first pass
    const double cdim0 = d == 1 ? 2.0 : (d == 2 ? 3.141592653589793 : 4.1887902047863905);
    int rho0 = (int)floor(pow((double)K / (g.occ * cdim0), 1.0 / d) + 0.5);
    if (rho0 < 1) rho0 = 1;
    // bisection stops at <= K + win survivors: as wide as keeps the rank pass
    // within one 64-survivor round (fewer bisection counts), 8..24; windows that
    // need several rounds anyway keep 16
    const int win = 64 - K >= 8 ? min(24, 64 - K) : 16;

    for (int64_t w = (int64_t)blockIdx.x * KNN_WARPS + wib; w < count; w += (int64_t)gridDim.x * KNN_WARPS) {
        const int trow = order[w];
        const int64_t tnode = a.targets[trow];
        double p[3] = {0.0, 0.0, 0.0};
        for (int ax = 0; ax < d; ++ax) p[ax] = a.pos[tnode * d + ax];
        int home[3] = {0, 0, 0};
        for (int ax = 0; ax < d; ++ax) home[ax] = cell_coord(g, ax, p[ax]);

        double dK = 0.0;
        for (int rho = rho0;; ++rho) {
            Box b = make_box(g, p, home, rho, d);
            const int R = box_ranges(b, d);
            // candidate count and range prefix offsets
            int M = 0;
            bool small = R <= KNN_RMAX;
            if (small) {
                for (int r0 = 0; r0 < R; r0 += 32) {
                    int r = r0 + lane;
                    int lo = 0, hi = 0;
                    if (r < R) range_bounds(g, b, d, r, a.start, lo, hi);
                    int len = hi - lo;
                    int incl = len;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        int v = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += v;
                    }
                    if (r < R) {
                        const int off = M + incl - len;
                        sm.roff[r] = off;
                        sm.rlo[r] = lo;
                        const int lim = min(len, KNN_CQ - off);
                        for (int t = 0; t < lim; ++t) sm.cq[off + t] = lo + t;
                    }
                    M += __shfl_sync(FULL, incl, 31);
                }
                if (lane == 0) sm.roff[R] = M;
                __syncwarp();
            } else {
                for (int r = lane; r < R; r += 32) {
                    int lo, hi;
                    range_bounds(g, b, d, r, a.start, lo, hi);
                    M += hi - lo;
                }
                M = warp_sum(M);
            }
            if (M < K) continue;

            bool done = false;
            if (small && M <= 32 * MAXIT) {
                // ---- register path: candidates c = it*32 + lane
                double cd[MAXIT];
                int ci[MAXIT];
#pragma unroll
                for (int it = 0; it < MAXIT; ++it) {
                    int c = it * 32 + lane;
                    cd[it] = INFINITY;
                    ci[it] = 0x7fffffff;
                    if (it * 32 < M && c < M) {
                        const int q = sm.cq[c];
                        cd[it] = metric<SEQ>(a.spos + (size_t)q * d, p, d);
                        ci[it] = a.sidx[q];
                    }
                }
                auto count_le = [&](double t) {
                    int c = 0;
#pragma unroll
                    for (int it = 0; it < MAXIT; ++it)
                        if (it * 32 < M) c += __popc(__ballot_sync(FULL, cd[it] <= t));
                    return c;
                };
                const double L = b.limit;
                int cL = count_le(L);
                if (cL < K && !b.all) continue;  // K-th key not provably inside: grow
                double hi = L, lo = -1.0;
                int chi = cL;
                if (hi == INFINITY) {
                    double mx = 0.0;
#pragma unroll
                    for (int it = 0; it < MAXIT; ++it)
                        if (cd[it] != INFINITY) mx = fmax(mx, cd[it]);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
                    hi = mx;
                    chi = count_le(hi);
                }
                // first guess from the local density of the cube: K' = K + WIN/2 points
                // lie within r with M/vol * c_d r^d = K'
                if (chi > K + win) {
                    double vol = 1.0;
                    for (int ax = 0; ax < d; ++ax) vol *= (double)(b.chi[ax] - b.clo[ax] + 1) * g.cw[ax];
                    const double cdim = d == 1 ? 2.0 : (d == 2 ? 3.141592653589793 : 4.1887902047863905);
                    const double want = (double)K + 0.5 * win;
                    double rg = pow(want * vol / ((double)M * cdim), 1.0 / d);
                    double tg = rg * rg;
                    if (tg > 0.0 && tg < hi) {
                        int c = count_le(tg);
                        if (c >= K) {
                            hi = tg;
                            chi = c;
                        } else {
                            lo = tg;
                        }
                    }
                }
                for (int iter = 0; iter < 80 && chi > K + win; ++iter) {
                    // interpolate in r^d (count ~ r^d), fall back to bisection
                    double mid;
                    if (lo >= 0.0) {
                        mid = lo + 0.5 * (hi - lo);
                    } else {
                        const double scale = pow(((double)K + 0.5 * win) / (double)chi, 2.0 / d);
                        mid = hi * fmin(fmax(scale, 0.25), 0.95);
                    }
                    if (!(mid < hi) || (lo >= 0.0 && !(mid > lo))) break;
                    int c = count_le(mid);
                    if (c >= K) {
                        hi = mid;
                        chi = c;
                    } else {
                        lo = mid;
                    }
                }
                if (chi >= K && chi <= KNN_SCAP) {
                    // compact the survivors (d2 <= hi) as packed keys, in candidate order
                    int base = 0;
#pragma unroll
                    for (int it = 0; it < MAXIT; ++it) {
                        if (it * 32 < M) {
                            bool keep = cd[it] <= hi;
                            unsigned bal = __ballot_sync(FULL, keep);
                            if (keep) {
                                int at = base + __popc(bal & ((1u << lane) - 1u));
                                KnnKey kk;
                                kk.d2 = cd[it];
                                kk.ic = ((unsigned long long)(unsigned)ci[it] << 32) | (unsigned)(it * 32 + lane);
                                sm.skey[at] = kk;
                                sm.sd2[at] = cd[it];
                            }
                            base += __popc(bal);
                        }
                    }
                    __syncwarp();
                    // rank of each survivor = number of survivors with a smaller
                    // (d2, node index, candidate id).  Count on d2 alone, two keys per
                    // 16-byte load, two survivors per lane per pass; a d2 shared by two
                    // survivors (rare) shows up as a rank collision and re-counts every
                    // rank on the full key.
                    const int S = base;
                    if (lane == 0) sm.sd2[S] = INFINITY;  // pad to an even count
                    __syncwarp();
                    int32_t* slot = sm.cq;              // the candidate table is free by now
                    int32_t* srank = sm.cq + KNN_SCAP;
                    for (int e0 = 0; e0 < S; e0 += 64) {
                        const int ea = e0 + lane, eb = ea + 32;
                        const double da = ea < S ? sm.sd2[ea] : INFINITY;
                        const double db = eb < S ? sm.sd2[eb] : INFINITY;
                        int ra = 0, rb = 0;
#pragma unroll 4
                        for (int f = 0; f < S; f += 2) {
                            const double2 v = *reinterpret_cast<const double2*>(sm.sd2 + f);
                            ra += (v.x < da) + (v.y < da);
                            rb += (v.x < db) + (v.y < db);
                        }
                        if (ea < S) srank[ea] = ra;
                        if (eb < S) srank[eb] = rb;
                    }
                    __syncwarp();
                    // survivors sharing a d2 get the same count: claim slot[rank], read it back
                    for (int e = lane; e < S; e += 32) slot[srank[e]] = e;
                    __syncwarp();
                    bool clash = false;
                    for (int e = lane; e < S; e += 32) clash |= slot[srank[e]] != e;
                    __syncwarp();
                    if (__any_sync(FULL, clash)) {
                        for (int e = lane; e < S; e += 32) {
                            const KnnKey ke = sm.skey[e];
                            int r = 0;
                            for (int f = 0; f < S; ++f) {
                                const KnnKey kf = sm.skey[f];
                                r += (kf.d2 < ke.d2) | ((kf.d2 == ke.d2) & (kf.ic < ke.ic));
                            }
                            srank[e] = r;
                        }
                        __syncwarp();
                    }
                    for (int e = lane; e < S; e += 32) {
                        const int r = srank[e];
                        if (r < K) {
                            sm.sel[r] = (int)(sm.skey[e].ic >> 32);
                            sm.seld2[r] = sm.skey[e].d2;
                        }
                    }
                    __syncwarp();
                    dK = sm.seld2[K - 1];
                    done = true;
                }
            }
            if (!done) {
                dK = extract_topk<SEQ, DD>(a, b, p, K, sm, lane);
                if (!b.all && !(dK <= b.limit)) continue;
            }
            break;
        }

        // straddle rows: the (K-1)-th and (n-1)-th keys tie to 1e-12 (stencils.py:61-65)
        if (!SEQ && K > n) {
            double edge = sm.seld2[n - 1];
            if (fabs(dK - edge) <= 1e-18 + 1e-12 * edge) {
                if (lane == 0) {
                    unsigned long long slot = atomicAdd(a.straddle_count, 1ull);
                    a.straddle_list[slot] = trow;
                }
            }
        }
        // self-first (stencils.py:77-91)
        if (a.in_pool[tnode]) {
            int first = sm.sel[0];
            if (first != (int)tnode) {
                int hit = 0x7fffffff;
                for (int j = lane; j < n; j += 32)
                    if (sm.sel[j] == (int)tnode) hit = min(hit, j);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) hit = min(hit, __shfl_xor_sync(FULL, hit, o));
                int last = hit == 0x7fffffff ? n - 1 : hit;
                // shift sel[0..last) right by one; serial but tiny (rare rows)
                if (lane == 0) {
                    for (int j = last; j > 0; --j) sm.sel[j] = sm.sel[j - 1];
                    sm.sel[0] = (int)tnode;
                }
                __syncwarp();
            }
        }
        int32_t* row = a.out + (int64_t)trow * n;
        for (int j = lane; j < n; j += 32) row[j] = sm.sel[j];
        __syncwarp();
    }
}

// ---- fast path ------------------------------------------------------------------
// The common case (d = 2 or 3, K <= 56, one cube of half-width rho around the home
// cell, at most 32 * SLOTS candidates) with a fixed register layout: candidate c
// of the cube sits in slot c / 32 of lane c % 32.  The threshold search starts
// from the previous target's final threshold (targets run in cell order, so the
// local density barely changes), the survivors are ranked exactly as in the
// general kernel, and every row the fast path cannot prove (too many candidates,
// the K-th key outside the cube's inner ball, more than KF_SCAP survivors) goes
// to a list that the general kernel re-solves from scratch.  Results are the
// same object either way: the K smallest (d2, node, candidate) keys.
constexpr int KF_WARPS = 4;
constexpr int KF_SCAP = 64;  // survivors ranked by the fast path (K <= 56); wide stencils (K <= 112) rank 128

template <int SLOTS, int SCAP>
struct FastSmem {
    int32_t cq[32 * SLOTS];  // sorted-pool position of each candidate
    KnnKey skey[SCAP];
    uint32_t sk32[SCAP + 4];  // high words of the survivor d2 (monotone in d2), padded to 4
    int32_t srank[SCAP];
    int32_t slot[SCAP];
    int32_t sel[SCAP];
    double seld2[SCAP];
};

template <int DD, int SLOTS, bool TPOS, int SCAP = KF_SCAP>
__global__ void __launch_bounds__(KF_WARPS * 32, SLOTS <= 5 ? 8 : (SLOTS <= 10 ? 6 : (SLOTS <= 16 ? 4 : 2)))
    knn_fast(KnnArgs a, const int32_t* __restrict__ order, int64_t count, const unsigned long long* count_dev, int K,
             int rho, int32_t* __restrict__ fb_list, unsigned long long* __restrict__ fb_count,
             const double* __restrict__ tpos, const uint32_t* __restrict__ tinfo, int win_max) {
    extern __shared__ __align__(16) unsigned char kf_smem[];
    const int lane = threadIdx.x & 31;
    FastSmem<SLOTS, SCAP>& sm = reinterpret_cast<FastSmem<SLOTS, SCAP>*>(kf_smem)[threadIdx.x >> 5];
    const GridParams g = *a.gp;
    constexpr int d = DD;
    const int n = a.n;
    const int win = min(SCAP - K, win_max);
    if (count_dev) count = (int64_t)*count_dev;
    // first threshold: the d2 of the (K + win/2)-th neighbour at the nominal grid
    // density (KNN_OCC points per cell); afterwards the previous target's
    double cellvol = 1.0;
    for (int ax = 0; ax < d; ++ax) cellvol *= g.cw[ax];
    const double cdim = d == 2 ? 3.141592653589793 : 4.1887902047863905;
    double tguess = pow(((double)K + 0.5 * win) * cellvol / (g.occ * cdim), 2.0 / d);

    // tpos / tinfo (first pass): target positions and (node | in-pool << 31)
    // gathered in processing order, so the next target's data are independent
    // coalesced loads issued a target ahead (not a chain order -> targets -> in_pool)
    const int64_t wstride = (int64_t)gridDim.x * KF_WARPS;
    int64_t w = (int64_t)blockIdx.x * KF_WARPS + (threadIdx.x >> 5);
    double pn[3] = {0.0, 0.0, 0.0};
    int trn = 0;
    int64_t tnn = 0;
    bool inp = false;
    auto fetch = [&](int64_t ww) {
        if (ww < count) {
            trn = order[ww];
            if constexpr (TPOS) {
                const uint32_t ti = tinfo[ww];
                tnn = (int64_t)(ti & 0x7fffffffu);
                inp = (ti >> 31) != 0u;
#pragma unroll
                for (int ax = 0; ax < d; ++ax) pn[ax] = tpos[ww * d + ax];
            }
        }
    };
    fetch(w);
    for (; w < count; w += wstride) {
        const int trow = trn;
        int64_t tnode;
        bool in_pool;
        double p[3] = {0.0, 0.0, 0.0};
        if constexpr (TPOS) {
            tnode = tnn;
            in_pool = inp;
#pragma unroll
            for (int ax = 0; ax < d; ++ax) p[ax] = pn[ax];
        } else {
            tnode = a.targets[trow];
            in_pool = a.in_pool[tnode] != 0;
#pragma unroll
            for (int ax = 0; ax < d; ++ax) p[ax] = a.pos[tnode * d + ax];
        }
        fetch(w + wstride);
        int home[3] = {0, 0, 0};
#pragma unroll
        for (int ax = 0; ax < d; ++ax) home[ax] = cell_coord(g, ax, p[ax]);
        const Box b = make_box(g, p, home, rho, d);
        const int R = box_ranges(b, d);
        // candidates: the cube's cells that reach the ball the proof covers
        const double R2 = (d == 2 || b.all) ? INFINITY : b.limit * (1.0 + 1e-6);  // (2D rows are few: no clipping)
        int M = 0;
        for (int r0 = 0; r0 < R; r0 += 32) {
            int lo = 0, hi = 0;
            if (r0 + lane < R) range_bounds_ball(g, b, d, r0 + lane, a.start, p, R2, lo, hi);
            const int len = hi - lo;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            const int off = M + incl - len;
            const int lim = min(len, 32 * SLOTS - off);
            for (int t = 0; t < lim; ++t) sm.cq[off + t] = lo + t;
            M += __shfl_sync(FULL, incl, 31);
        }
        bool fail = M > 32 * SLOTS || M < K;
        __syncwarp();
        double cd[SLOTS];
        int ci[SLOTS];
#pragma unroll
        for (int it = 0; it < SLOTS; ++it) {
            const int c = it * 32 + lane;
            cd[it] = INFINITY;
            ci[it] = 0x7fffffff;
            if (!fail && c < M) {
                const int q = sm.cq[c];
                cd[it] = metric<false>(a.spos + (size_t)q * d, p, d);
                ci[it] = a.sidx[q];
            }
        }
        auto count_le = [&](double t) {
            int c = 0;
#pragma unroll
            for (int it = 0; it < SLOTS; ++it) c += __popc(__ballot_sync(FULL, cd[it] <= t));
            return c;
        };
        // threshold t with K <= count(d2 <= t) <= K + win
        double t = tguess, tlo = 0.0, thi = INFINITY;
        int ct = 0;
        if (!fail) {
            int iter = 0;
            for (; iter < 40; ++iter) {
                ct = count_le(t);
                if (ct < K) {
                    tlo = t;
                    t = thi < INFINITY ? tlo + 0.5 * (thi - tlo) : t * 1.5;
                } else if (ct > K + win) {
                    thi = t;
                    if (tlo > 0.0) {
                        t = tlo + 0.5 * (thi - tlo);
                    } else {
                        // count ~ t^(d/2): aim at K + win/2
                        const float x = (float)((double)K + 0.5 * win) / (float)ct;
                        t = thi * (double)__powf(x, 2.0f / d);
                    }
                } else {
                    break;
                }
                if (!(t > tlo && t < thi)) break;  // exhausted the d2 resolution (heavy ties)
            }
            fail = ct < K || ct > K + win;
        }
        if (!fail) {
            // aim the next target's first threshold at K + win/2 points
            const float x = (float)((double)K + 0.5 * win) / (float)ct;
            tguess = t * (double)__powf(x, 2.0f / d);
            // compact the survivors as packed keys, in candidate order
            int base = 0;
#pragma unroll
            for (int it = 0; it < SLOTS; ++it) {
                const bool keep = cd[it] <= t;
                const unsigned bal = __ballot_sync(FULL, keep);
                if (keep) {
                    const int at = base + __popc(bal & ((1u << lane) - 1u));
                    KnnKey kk;
                    kk.d2 = cd[it];
                    kk.ic = ((unsigned long long)(unsigned)ci[it] << 32) | (unsigned)(it * 32 + lane);
                    sm.skey[at] = kk;
                    sm.sk32[at] = (uint32_t)((unsigned long long)__double_as_longlong(cd[it]) >> 32);
                }
                base += __popc(bal);
            }
            const int S = base;
            if (lane < 4) sm.sk32[S + lane] = 0x7fffffffu;  // pad to a multiple of 4
            __syncwarp();
            // ranks on the high word of d2 (monotone in d2: four keys per 16-byte load,
            // two survivors per lane); equal high words collide in `slot` and fall back
            // to the full key.  d2 is finite and >= +0, so every key (and the pad) is
            // below 2^31 and [v < d] is the sign bit of v - d: one IADD + one LEA.HI
            // per comparison instead of ISETP + IADD + a predicated move
            {
                // SCAP / 32 survivors per lane, two accumulators each
                constexpr int NS = SCAP / 32;
                uint32_t dv[NS], r0[NS], r1[NS];
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    const int e = lane + 32 * q;
                    dv[q] = e < S ? sm.sk32[e] : 0u;
                    r0[q] = r1[q] = 0u;
                }
#pragma unroll 4
                for (int f = 0; f < S; f += 4) {
                    const uint4 v = *reinterpret_cast<const uint4*>(sm.sk32 + f);
#pragma unroll
                    for (int q = 0; q < NS; ++q) {
                        r0[q] += ((v.x - dv[q]) >> 31) + ((v.y - dv[q]) >> 31);
                        r1[q] += ((v.z - dv[q]) >> 31) + ((v.w - dv[q]) >> 31);
                    }
                }
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    const int e = lane + 32 * q;
                    if (e < S) sm.srank[e] = (int)(r0[q] + r1[q]);
                }
            }
            __syncwarp();
            for (int e = lane; e < S; e += 32) sm.slot[sm.srank[e]] = e;
            __syncwarp();
            bool clash = false;
            for (int e = lane; e < S; e += 32) clash |= sm.slot[sm.srank[e]] != e;
            __syncwarp();
            if (__any_sync(FULL, clash)) {
                for (int e = lane; e < S; e += 32) {
                    const KnnKey ke = sm.skey[e];
                    int r = 0;
                    for (int f = 0; f < S; ++f) {
                        const KnnKey kf = sm.skey[f];
                        r += (kf.d2 < ke.d2) | ((kf.d2 == ke.d2) & (kf.ic < ke.ic));
                    }
                    sm.srank[e] = r;
                }
                __syncwarp();
            }
            for (int e = lane; e < S; e += 32) {
                const int r = sm.srank[e];
                if (r < K) {
                    sm.sel[r] = (int)(sm.skey[e].ic >> 32);
                    sm.seld2[r] = sm.skey[e].d2;
                }
            }
            __syncwarp();
            // the K-th key must be provably inside the cube's inner ball
            const double dK = sm.seld2[K - 1];
            fail = !b.all && !(dK <= b.limit);
            if (!fail) {
                // straddle rows: the (K-1)-th and (n-1)-th keys tie to 1e-12 (stencils.py:61-65)
                if (K > n) {
                    const double edge = sm.seld2[n - 1];
                    if (fabs(dK - edge) <= 1e-18 + 1e-12 * edge && lane == 0) {
                        const unsigned long long sl = atomicAdd(a.straddle_count, 1ull);
                        a.straddle_list[sl] = trow;
                    }
                }
                // self-first (stencils.py:77-91)
                if (in_pool && sm.sel[0] != (int)tnode) {
                    int hitv = 0x7fffffff;
                    for (int j = lane; j < n; j += 32)
                        if (sm.sel[j] == (int)tnode) hitv = min(hitv, j);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) hitv = min(hitv, __shfl_xor_sync(FULL, hitv, o));
                    const int last = hitv == 0x7fffffff ? n - 1 : hitv;
                    if (lane == 0) {
                        for (int j = last; j > 0; --j) sm.sel[j] = sm.sel[j - 1];
                        sm.sel[0] = (int)tnode;
                    }
                    __syncwarp();
                }
                int32_t* row = a.out + (int64_t)trow * n;
                for (int j = lane; j < n; j += 32) row[j] = sm.sel[j];
            }
        }
        if (fail && lane == 0) {
            const unsigned long long sl = atomicAdd(fb_count, 1ull);
            fb_list[sl] = trow;
        }
        __syncwarp();
    }
}

// ---- grid construction ------------------------------------------------------
__global__ void knn_bbox(const double* __restrict__ pos, int d, const int64_t* __restrict__ pool, int64_t P,
                         unsigned long long* bb) {
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = pool[i];
        for (int a = 0; a < d; ++a) {
            double x = pos[node * d + a];
            mn[a] = fmin(mn[a], x);
            mx[a] = fmax(mx[a], x);
        }
    }
    block_bbox_commit(mn, mx, d, bb);
}

// grid over the pool's bounding box with `occ_grid` points per cell of the BOX;
// `occ_true` is the density the kernels assume inside the occupied cells
__device__ void grid_from_bbox(const unsigned long long* bb, int d, int64_t P, double occ_grid, double occ_true,
                               GridParams* gp) {
    GridParams g;
    g.occ = occ_true;
    double lo[3], hi[3];
    double vol = 1.0;
    int nd = 0;
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = 0.0;
        g.cw[a] = 0.0;
        g.inv[a] = 0.0;
        g.G[a] = 1;
    }
    for (int a = 0; a < d; ++a) {
        lo[a] = from_ordered_bits(bb[a]);
        hi[a] = from_ordered_bits(bb[3 + a]);
        if (hi[a] > lo[a]) {
            vol *= hi[a] - lo[a];
            ++nd;
        }
    }
    double w = nd ? pow(vol * occ_grid / (double)P, 1.0 / nd) : 1.0;
    double ncell = 1.0;
    for (int a = 0; a < d; ++a) {
        double ext = hi[a] - lo[a];
        double G = 1.0;
        if (ext > 0.0 && w > 0.0) G = fmin(fmax(floor(ext / w), 1.0), 2097152.0);
        // keep the total within the workspace bound P/occ + 1 (occ >= KNN_OCC, which sizes the workspace)
        if (ncell * G > (double)P / occ_grid + 1.0) G = fmax(1.0, floor(((double)P / occ_grid + 1.0) / ncell));
        ncell *= G;
        g.G[a] = (int)G;
        g.lo[a] = lo[a];
        g.cw[a] = ext > 0.0 ? ext / G : 0.0;
        g.inv[a] = ext > 0.0 ? G / ext : 0.0;
    }
    g.ncell = (int)ncell;
    *gp = g;
}

__global__ void knn_params(const unsigned long long* bb, int d, int64_t P, double occ, GridParams* gp) {
    grid_from_bbox(bb, d, P, occ, occ, gp);
}

// Wide stencils: the pool may fill only part of its bounding box (a ball fills
// 52% of it), which makes the occupied cells denser than the box average and
// overflows the fast pass's candidate slots.  The cells of a first grid are
// counted, and the grid is rebuilt so that the OCCUPIED cells hold `occ` points
// on average (never finer than KNN_OCC per box cell: the workspace bound).
__global__ void knn_count_occupied(const int32_t* __restrict__ cnt, const GridParams* __restrict__ gp,
                                   unsigned long long* __restrict__ occupied) {
    const int nc = gp->ncell;
    int mine = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) mine += cnt[i] > 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(FULL, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(occupied, (unsigned long long)mine);
}
__global__ void knn_params_refit(const unsigned long long* bb, int d, int64_t P, double occ,
                                 const unsigned long long* occupied, GridParams* gp) {
    const double fill = fmin(1.0, fmax((double)*occupied / (double)gp->ncell, 1e-3));
    const double occ_grid = fmax(KNN_OCC, occ * fill);
    grid_from_bbox(bb, d, P, occ_grid, occ_grid / fill, gp);
}

__global__ void knn_cells(const double* __restrict__ pos, int d, const int64_t* __restrict__ pool, int64_t P,
                          const GridParams* __restrict__ gp, int32_t* __restrict__ cell, int32_t* __restrict__ cnt,
                          uint8_t* __restrict__ in_pool) {
    const GridParams g = *gp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = pool[i];
        int c = cell_of(g, pos + node * d, d);
        cell[i] = c;
        atomicAdd(&cnt[c], 1);
        in_pool[node] = 1;
    }
}

__global__ void knn_scatter(const double* __restrict__ pos, int d, const int64_t* __restrict__ pool, int64_t P,
                            const int32_t* __restrict__ cell, int32_t* __restrict__ cursor, double* __restrict__ spos,
                            int32_t* __restrict__ sidx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = pool[i];
        int at = atomicAdd(&cursor[cell[i]], 1);
        for (int a = 0; a < d; ++a) spos[(size_t)at * d + a] = pos[node * d + a];
        sidx[at] = (int32_t)node;
    }
}

__global__ void knn_target_keys(const double* __restrict__ pos, int d, const int64_t* __restrict__ targets, int64_t T,
                                const GridParams* __restrict__ gp, int32_t* __restrict__ key, int32_t* __restrict__ val) {
    const GridParams g = *gp;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        key[t] = cell_of(g, pos + targets[t] * d, d);
        val[t] = (int32_t)t;
    }
}

__global__ void knn_target_gather(const double* __restrict__ pos, int d, const int64_t* __restrict__ targets,
                                  const int32_t* __restrict__ order, const uint8_t* __restrict__ in_pool, int64_t T,
                                  double* __restrict__ tpos, uint32_t* __restrict__ tinfo) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < T; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = targets[order[w]];
        for (int a = 0; a < d; ++a) tpos[w * d + a] = pos[node * d + a];
        tinfo[w] = (uint32_t)node | (in_pool[node] ? 0x80000000u : 0u);  // (N < 2^31, checked by mf_knn)
    }
}
inline int grid_for(int64_t work, int threads, int per_sm = 8) { return grid_cap(work, threads, per_sm); }

struct KnnLayout {
    GridParams* gp;
    unsigned long long* bb;
    unsigned long long* straddle_count;
    int32_t* cnt;     // ncell_max + 1 (counts, then starts)
    int32_t* cursor;  // ncell_max
    int32_t* cell;    // P
    double* spos;     // P * d
    int32_t* sidx;    // P
    uint8_t* in_pool; // N
    int32_t* tkey[2];
    int32_t* tval[2];
    int32_t* straddle_list;  // T
    double* tpos;            // T * d: target positions in processing (cell) order
    int32_t* fb_list[2];     // T each: rows a fast pass hands to the next pass
    unsigned long long* fb_count;  // 2
    char* cub_tmp;    // scan temporary storage
    size_t cub_bytes;
    char* sort_tmp;   // sort temporary storage (separate: scan and sort may overlap)
    size_t sort_bytes;
};

inline int64_t ncell_max(int64_t P) { return (int64_t)((double)P / KNN_OCC) + 2; }

inline size_t knn_cub_bytes(int64_t P, int64_t T) {
    size_t a = 0, b = 0;
    int64_t nc = ncell_max(P);
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nc + 1));
    cub::DoubleBuffer<int32_t> k(nullptr, nullptr), v(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, b, k, v, (int)(T > 0 ? T : 1));
    return a > b ? a : b;
}

inline KnnLayout knn_layout(Arena& ar, int64_t N, int d, int64_t T, int64_t P) {
    KnnLayout L;
    int64_t nc = ncell_max(P);
    L.gp = ar.take<GridParams>(1);
    L.bb = ar.take<unsigned long long>(8);  // bounding box (6), occupied-cell count
    L.straddle_count = ar.take<unsigned long long>(1);
    L.cnt = ar.take<int32_t>(nc + 1);
    L.cursor = ar.take<int32_t>(nc + 1);
    L.cell = ar.take<int32_t>(P);
    L.spos = ar.take<double>((size_t)P * d);
    L.sidx = ar.take<int32_t>(P);
    L.in_pool = ar.take<uint8_t>(N);
    for (int i = 0; i < 2; ++i) {
        L.tkey[i] = ar.take<int32_t>(T);
        L.tval[i] = ar.take<int32_t>(T);
    }
    L.straddle_list = ar.take<int32_t>(T);
    L.tpos = ar.take<double>((size_t)T * d);
    L.fb_list[0] = ar.take<int32_t>(T);
    L.fb_list[1] = ar.take<int32_t>(T);
    L.fb_count = ar.take<unsigned long long>(2);
    L.cub_bytes = knn_cub_bytes(P, T);
    L.cub_tmp = ar.take<char>(L.cub_bytes);
    L.sort_bytes = L.cub_bytes;
    L.sort_tmp = ar.take<char>(L.sort_bytes);
    return L;
}

}  // namespace mf

using namespace mf;

namespace {
// Fork / join for the target-side preparation (keys + sort), which depends only on
// the grid parameters and runs beside the pool-side binning (cells, scan, scatter).
// One non-blocking side stream and two timing-free events per device, created on
// first use; the pattern is a plain fork-join, so it is capturable in a CUDA graph.
struct KnnSide {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    bool ok = false;
    std::mutex mu;  // one fork .. join enqueue at a time per device (the events are shared)
};
KnnSide* knn_side() {
    static KnnSide side[16];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    KnnSide& s = side[dev];
    std::lock_guard<std::mutex> init(s.mu);
    if (!s.ok) {
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        s.ok = true;
    }
    return &s;
}
}  // namespace

extern "C" int mf_knn_workspace_size(int64_t N, int32_t d, int64_t T, int64_t P, int32_t n, size_t* bytes) {
    (void)n;
    if (!bytes || N < 0 || T < 0 || P < 1 || d < 1 || d > MF_MAX_DIM) {
        set_error("mf_knn_workspace_size: bad arguments");
        return MF_ERR_ARG;
    }
    Arena ar{nullptr, 0, 0, true};
    knn_layout(ar, N, d, T, P);
    *bytes = ar.off;
    return MF_OK;
}

extern "C" int mf_knn(const double* pos, int64_t N, int32_t d, const int64_t* targets, int64_t T,
                      const int64_t* pool, int64_t P, int32_t n, int32_t* out_idx, int64_t* n_straddle, void* ws,
                      size_t ws_bytes, void* stream) {
    MF_REQUIRE(d >= 1 && d <= MF_MAX_DIM, "mf_knn: dimension %d not in 1..3", d);
    MF_REQUIRE(n >= 1 && n <= P, "mf_knn: stencil size %d vs pool %lld", n, (long long)P);
    MF_REQUIRE(N < 2147483647 && P < 2147483647 && T < 2147483647, "mf_knn: sizes exceed int32 indexing");
    MF_REQUIRE(n + 8 <= KNN_SCAP, "mf_knn: stencil size %d above the kernel limit %d", n, KNN_SCAP - 8);
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char*)ws, ws_bytes, 0, false};
    KnnLayout L = knn_layout(ar, N, d, T, P);
    if (!ws || !ar.ok()) {
        set_error("mf_knn: workspace too small (%zu < %zu)", ws_bytes, ar.off);
        return MF_ERR_WORKSPACE;
    }
    if (n_straddle) MF_CUDA_CHECK(cudaMemsetAsync(n_straddle, 0, sizeof(int64_t), st));
    if (T == 0) return MF_OK;
    const int64_t nc = ncell_max(P);
    const int K = (int)(n + 8 < P ? n + 8 : P);
    // wide 3D stencils (56 < K <= 112) take a coarser grid, sized so that the
    // rho = 2 cube's inner ball (33.5 cells) holds ~1.6 K points: the first fast
    // pass then proves most rows, as it does at KNN_OCC for K <= 56
    const bool wide = d == 3 && K > 56 && K + 16 <= 128;
    const double occ = wide ? fmax(KNN_OCC, 1.6 * (double)K / 33.51) : KNN_OCC;
    MF_CUDA_CHECK(cudaMemsetAsync(L.bb, 0xff, 3 * sizeof(unsigned long long), st));
    MF_CUDA_CHECK(cudaMemsetAsync(L.bb + 3, 0, 3 * sizeof(unsigned long long), st));
    MF_CUDA_CHECK(cudaMemsetAsync(L.straddle_count, 0, sizeof(unsigned long long), st));
    MF_CUDA_CHECK(cudaMemsetAsync(L.fb_count, 0, 2 * sizeof(unsigned long long), st));
    MF_CUDA_CHECK(cudaMemsetAsync(L.cnt, 0, sizeof(int32_t) * (nc + 1), st));
    MF_CUDA_CHECK(cudaMemsetAsync(L.in_pool, 0, (size_t)N, st));
    knn_bbox<<<grid_for(P, 256, 4), 256, 0, st>>>(pos, d, pool, P, L.bb);
    MF_LAUNCH_CHECK();
    knn_params<<<1, 1, 0, st>>>(L.bb, d, P, occ, L.gp);
    MF_LAUNCH_CHECK();
    // target side on the side stream from here: keys by home cell, sorted (the grid is
    // final at this point unless the wide path refits it below)
    KnnSide* side = wide ? nullptr : knn_side();
    cudaStream_t ts = side ? side->stream : st;
    std::unique_lock<std::mutex> side_lock;
    if (side) side_lock = std::unique_lock<std::mutex>(side->mu);
    if (side) {
        MF_CUDA_CHECK(cudaEventRecord(side->fork, st));
        MF_CUDA_CHECK(cudaStreamWaitEvent(ts, side->fork, 0));
    }
    cub::DoubleBuffer<int32_t> kb(L.tkey[0], L.tkey[1]), vb(L.tval[0], L.tval[1]);
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < nc) ++bits;
    auto sort_targets = [&]() -> int {
        knn_target_keys<<<grid_for(T, 256), 256, 0, ts>>>(pos, d, targets, T, L.gp, L.tkey[0], L.tval[0]);
        MF_LAUNCH_CHECK();
        size_t sb = L.sort_bytes;
        MF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(L.sort_tmp, sb, kb, vb, (int)T, 0, bits, ts));
        return MF_OK;
    };
    if (side) {
        const int rc = sort_targets();
        if (rc != MF_OK) return rc;
        MF_CUDA_CHECK(cudaEventRecord(side->join, ts));
    }
    knn_cells<<<grid_for(P, 256), 256, 0, st>>>(pos, d, pool, P, L.gp, L.cell, L.cnt, L.in_pool);
    MF_LAUNCH_CHECK();
    if (wide) {
        // refit the grid to the occupied part of the bounding box and bin again
        MF_CUDA_CHECK(cudaMemsetAsync(L.bb + 6, 0, sizeof(unsigned long long), st));
        knn_count_occupied<<<grid_for(nc, 256), 256, 0, st>>>(L.cnt, L.gp, L.bb + 6);
        MF_LAUNCH_CHECK();
        knn_params_refit<<<1, 1, 0, st>>>(L.bb, d, P, occ, L.bb + 6, L.gp);
        MF_LAUNCH_CHECK();
        MF_CUDA_CHECK(cudaMemsetAsync(L.cnt, 0, sizeof(int32_t) * (nc + 1), st));
        knn_cells<<<grid_for(P, 256), 256, 0, st>>>(pos, d, pool, P, L.gp, L.cell, L.cnt, L.in_pool);
        MF_LAUNCH_CHECK();
    }
    size_t cb = L.cub_bytes;
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.cnt, L.cnt, (int)(nc + 1), st));
    MF_CUDA_CHECK(cudaMemcpyAsync(L.cursor, L.cnt, sizeof(int32_t) * (nc + 1), cudaMemcpyDeviceToDevice, st));
    knn_scatter<<<grid_for(P, 256), 256, 0, st>>>(pos, d, pool, P, L.cell, L.cursor, L.spos, L.sidx);
    MF_LAUNCH_CHECK();
    if (side) {
        MF_CUDA_CHECK(cudaStreamWaitEvent(st, side->join, 0));
        side_lock.unlock();
    } else {
        const int rc = sort_targets();
        if (rc != MF_OK) return rc;
    }
    const int32_t* order = vb.Current();

    KnnArgs a{pos, d, targets, L.gp, L.cnt, L.spos, L.sidx, L.in_pool, n, K, out_idx, L.straddle_list, L.straddle_count};
    // candidates per warp (32 * MAXIT) sized by K
    const bool big = K + KNN_WIN > 64;
    auto main_k = big ? (d == 1 ? knn_kernel<false, 1, 32> : (d == 2 ? knn_kernel<false, 2, 32> : knn_kernel<false, 3, 32>))
                      : (d == 1 ? knn_kernel<false, 1, 16> : (d == 2 ? knn_kernel<false, 2, 16> : knn_kernel<false, 3, 16>));
    auto strd_k = big ? (d == 1 ? knn_kernel<true, 1, 32> : (d == 2 ? knn_kernel<true, 2, 32> : knn_kernel<true, 3, 32>))
                      : (d == 1 ? knn_kernel<true, 1, 16> : (d == 2 ? knn_kernel<true, 2, 16> : knn_kernel<true, 3, 16>));
    constexpr int smem_bytes = KNN_WARPS * (int)sizeof(WarpSmem);
    MF_CUDA_CHECK(ensure_smem(main_k, smem_bytes));
    MF_CUDA_CHECK(ensure_smem(strd_k, smem_bytes));
    // fast passes where they apply: a cube that usually proves the K-th key
    // (2D: rho0 + 1; 3D: rho0), then the rows it hands back with one more cell of
    // half-width, then the general kernel for whatever is left
    const double cdim0 = d == 1 ? 2.0 : (d == 2 ? 3.141592653589793 : 4.1887902047863905);
    int rho0 = (int)floor(pow((double)K / (occ * cdim0), 1.0 / d) + 0.5);
    if (rho0 < 1) rho0 = 1;
    auto fits = [&](int rho, int slots) {
        return occ * pow(2.0 * rho + 1.0, (double)d) <= 0.8 * 32 * slots;
    };
    const int rho1 = d == 2 ? rho0 + 1 : rho0, rho2 = rho1 + 1;
    const bool fast = K <= 56 &&
                      ((d == 3 && fits(rho1, 10) && fits(rho2, 28)) || (d == 2 && fits(rho1, 5) && fits(rho2, 8)));
    // (the first pass keeps only the cells that reach the proof's ball: ~0.7 of the
    // cube, so 8 slots hold it in 3D)
    constexpr int kf_win = 16;  // first-pass survivor window (bisection stops at K..K+16)
    if (fast || wide) {
        // K <= 56: 8 / 28 candidate slots (3D), 5 / 8 (2D), 64 ranked survivors;
        // wide 3D: 16 / 32 slots on the coarser grid, 128 ranked survivors
        auto f1 = wide ? knn_fast<3, 16, true, 128> : (d == 3 ? knn_fast<3, 8, true> : knn_fast<2, 5, true>);
        auto f2 = wide ? knn_fast<3, 32, false, 128> : (d == 3 ? knn_fast<3, 28, false> : knn_fast<2, 8, false>);
        const int sm1 = KF_WARPS * (wide ? (int)sizeof(FastSmem<16, 128>)
                                         : (d == 3 ? (int)sizeof(FastSmem<8, KF_SCAP>) : (int)sizeof(FastSmem<5, KF_SCAP>)));
        const int sm2 = KF_WARPS * (wide ? (int)sizeof(FastSmem<32, 128>)
                                         : (d == 3 ? (int)sizeof(FastSmem<28, KF_SCAP>) : (int)sizeof(FastSmem<8, KF_SCAP>)));
        MF_CUDA_CHECK(ensure_smem(f1, sm1));
        MF_CUDA_CHECK(ensure_smem(f2, sm2));
        // (the sort's spare key buffer is free now: it takes the packed target info)
        uint32_t* tinfo = reinterpret_cast<uint32_t*>(kb.Alternate());
        knn_target_gather<<<grid_for(T, 256), 256, 0, st>>>(pos, d, targets, order, L.in_pool, T, L.tpos, tinfo);
        MF_LAUNCH_CHECK();
        f1<<<grid_for(T, KF_WARPS, 64), KF_WARPS * 32, sm1, st>>>(a, order, T, nullptr, K, rho1, L.fb_list[0],
                                                                  L.fb_count, L.tpos, tinfo, kf_win);
        MF_LAUNCH_CHECK();
        f2<<<grid_for(T, KF_WARPS, 4), KF_WARPS * 32, sm2, st>>>(a, L.fb_list[0], T, L.fb_count, K, rho2,
                                                                 L.fb_list[1], L.fb_count + 1, nullptr, nullptr, 16);
        MF_LAUNCH_CHECK();
        main_k<<<grid_for(T, KNN_WARPS, 4), KNN_WARPS * 32, smem_bytes, st>>>(a, L.fb_list[1], T, L.fb_count + 1, K);
        MF_LAUNCH_CHECK();
    } else {
        main_k<<<grid_for(T, KNN_WARPS, 64), KNN_WARPS * 32, smem_bytes, st>>>(a, order, T, nullptr, K);
        MF_LAUNCH_CHECK();
    }
    if (K > n) {
        // straddle rows: top-n by the sequential-sum metric (stencils.py:67-75)
        strd_k<<<grid_for(T, KNN_WARPS, 4), KNN_WARPS * 32, smem_bytes, st>>>(a, L.straddle_list, T, L.straddle_count,
                                                                            n);
        MF_LAUNCH_CHECK();
    }
    if (n_straddle)
        MF_CUDA_CHECK(cudaMemcpyAsync(n_straddle, L.straddle_count, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    return MF_OK;
}

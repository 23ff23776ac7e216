// General weight engines, batched (sm_100a): the configurations the reference
// sends through its per-node loop (storage.py:325-339) instead of
// batch_phs_weights -- RbfFd with the qr / svd solvers or a non-polyharmonic
// kernel (Gaussian, multiquadric, inverse multiquadric, r^k with k <= 2),
// WeightedLeastSquares (approx/engines.py:102-145), and composite operators
// (ScaledOperator / OperatorSum / Directional, approx/operators.py).
//
// One warp per stencil, the local system in shared memory (column-major, odd
// pitch so a warp's column-parallel accesses are bank-conflict free):
//   RbfFd   [Phi Q; Q^T 0] (n+l)^2, right-hand sides per family
//           (engines.py:168-201)
//   WLS     (W B)^T (l x n); l <= n is stored transposed as W B (n x l) and
//           solved for the minimum-norm solution (engines.py:129-138)
// and solved by
//   lu      partial pivoting (LAPACK getrf's pivot rule: first max |a|)
//   qr      Householder QR: least squares for tall / square systems, minimum
//           norm through the QR of the transpose for wide ones (gelsy's answer
//           for full-rank systems)
//   svd     one-sided Jacobi SVD, singular values below 1e-13 of the largest
//           dropped (engines.py:84-88)
// Every family is solved from the same factorisation (the reference calls the
// engine once per family with the same matrix).  Per (stencil, family) status
// codes reproduce the engine's exceptions; the host maps the lowest failing row
// and its first failing family to the reference's WeightError text.
#include <cfloat>

#include "common.cuh"

namespace mf {

namespace {

constexpr int EW = 2;  // warps per block

struct EngArgs {
    const double* pos;
    const int64_t* rows;
    const int32_t* stencils;
    int64_t m;
    int n;
    double* out;
    int8_t* status;
    unsigned long long* first_fail;
    mf_engine_t E;
    // derived sizes
    int p, q, nr;  // stored matrix p x q (p >= q except lu / square), right-hand side rows
    int wide;      // stored matrix is the transpose of the system (minimum-norm solve)
    int ld;        // column pitch
    int warp_dbl;  // doubles of shared memory per warp
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ double warp_maxd(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// ---- radial kernels (basis.py:93-228): value, phi'(r)/r, phi''(r) ----------
__device__ double ipow(double x, int k) {  // x^k, k >= 0, binary powering
    double r = 1.0, b = x;
    while (k) {
        if (k & 1) r *= b;
        b *= b;
        k >>= 1;
    }
    return r;
}
__device__ double rbf_value(const mf_engine_t& E, double r) {
    switch (E.rbf) {
        case MF_RBF_PHS:
            if (!(E.k & 1)) return r > 0.0 ? pow(r, (double)E.k) * log(r) : 0.0;
            return pow(r, (double)E.k);
        case MF_RBF_GAUSSIAN: return exp(-(r * r) / (E.sigma * E.sigma));
        case MF_RBF_MQ: {
            const double u = r / E.sigma;
            return sqrt(1.0 + u * u);
        }
        default: {
            const double u = r / E.sigma;
            return 1.0 / sqrt(1.0 + u * u);
        }
    }
}
__device__ double rbf_d1r(const mf_engine_t& E, double r) {
    const double s2 = E.sigma * E.sigma;
    switch (E.rbf) {
        case MF_RBF_PHS: {
            const int k = E.k;
            if (k & 1) return k * pow(r, k - 2.0);
            return r > 0.0 ? pow(r, (double)(k - 2)) * (k * log(r) + 1.0) : 0.0;
        }
        case MF_RBF_GAUSSIAN: return -2.0 / s2 * exp(-(r * r) / s2);
        case MF_RBF_MQ: {
            const double u = r / E.sigma;
            return 1.0 / (s2 * sqrt(1.0 + u * u));
        }
        default: {
            const double u = r / E.sigma;
            const double g = 1.0 / sqrt(1.0 + u * u);
            return -(g * g * g) / s2;
        }
    }
}
__device__ double rbf_d2(const mf_engine_t& E, double r) {
    const double s2 = E.sigma * E.sigma;
    switch (E.rbf) {
        case MF_RBF_PHS: {
            const int k = E.k;
            if (k & 1) return k * (k - 1.0) * pow(r, k - 2.0);
            return r > 0.0 ? pow(r, (double)(k - 2)) * ((double)(k * k - k) * log(r) + 2.0 * k - 1.0) : 0.0;
        }
        case MF_RBF_GAUSSIAN: return (4.0 * r * r / (s2 * s2) - 2.0 / s2) * exp(-(r * r) / s2);
        case MF_RBF_MQ: {
            const double u = r / E.sigma;
            const double f = sqrt(1.0 + u * u);
            return 1.0 / (s2 * f) - r * r / (s2 * s2 * (f * f * f));
        }
        default: {
            const double u = r / E.sigma;
            const double g = 1.0 / sqrt(1.0 + u * u);
            const double g3 = g * g * g;
            return -g3 / s2 + 3.0 * r * r * (g3 * g * g) / (s2 * s2);
        }
    }
}

// (L_t phi(|x - c|)) at the centre for a node at local offset loc: diff = -loc
// (operators.py:99-214).  *sing is set when a polyharmonic kernel with k <= 2
// would be differentiated at r = 0 (basis.py:180-186).
__device__ double term_rbf(const mf_engine_t& E, int t, const double* loc, int d, bool* sing) {
    double diff[MF_MAX_DIM], r2 = 0.0;
    for (int a = 0; a < d; ++a) {
        diff[a] = -loc[a];
        r2 += diff[a] * diff[a];
    }
    const double r = sqrt(r2);
    const int kind = E.term_kind[t];
    const bool low_phs = E.rbf == MF_RBF_PHS && E.k <= 2;
    switch (kind) {
        case MF_TERM_IDENTITY: return rbf_value(E, r);
        case MF_TERM_D1:
            return r > 0.0 ? rbf_d1r(E, r) * diff[E.term_a[t]] : 0.0;
        case MF_TERM_DIRECTIONAL: {
            if (!(r > 0.0)) return 0.0;
            double dv = 0.0;
            for (int a = 0; a < d; ++a) dv += diff[a] * E.term_vec[t * MF_MAX_DIM + a];
            return rbf_d1r(E, r) * dv;
        }
        case MF_TERM_D2: {
            if (low_phs && r == 0.0) *sing = true;
            const int ta = E.term_a[t], tb = E.term_b[t];
            const double d2v = rbf_d2(E, r), d1r = rbf_d1r(E, r);
            const double ee = r > 0.0 ? diff[ta] * diff[tb] / (r * r) : 0.0;
            return d2v * ee + d1r * ((ta == tb ? 1.0 : 0.0) - ee);
        }
        default:  // Laplacian
            if (low_phs && r == 0.0) *sing = true;
            return rbf_d2(E, r) + (d - 1) * rbf_d1r(E, r);
    }
}

// (L_t x^e)(0) (operators.py:57-76 evaluated at the origin)
__device__ double term_mono0(const mf_engine_t& E, int t, int j, int d) {
    const int* e = E.expos + j * MF_MAX_DIM;
    int tot = 0;
    for (int a = 0; a < d; ++a) tot += e[a];
    const int kind = E.term_kind[t], ta = E.term_a[t], tb = E.term_b[t];
    switch (kind) {
        case MF_TERM_IDENTITY: return tot == 0 ? 1.0 : 0.0;
        case MF_TERM_D1: return (tot == 1 && e[ta] == 1) ? 1.0 : 0.0;
        case MF_TERM_DIRECTIONAL: {
            if (tot != 1) return 0.0;
            double v = 0.0;
            for (int a = 0; a < d; ++a)
                if (e[a] == 1) v = E.term_vec[t * MF_MAX_DIM + a];
            return v;
        }
        case MF_TERM_D2:
            if (tot != 2) return 0.0;
            if (ta == tb) return e[ta] == 2 ? 2.0 : 0.0;
            return (e[ta] == 1 && e[tb] == 1) ? 1.0 : 0.0;
        default: {
            if (tot != 2) return 0.0;
            for (int a = 0; a < d; ++a)
                if (e[a] == 2) return 2.0;
            return 0.0;
        }
    }
}

__device__ __forceinline__ double monomial(const mf_engine_t& E, int j, const double* x, int d) {
    const int* e = E.expos + j * MF_MAX_DIM;
    double v = 1.0;
    for (int a = 0; a < d; ++a)
        if (e[a]) v *= ipow(x[a], e[a]);
    return v;
}

// ---- warp-level dense solvers on column-major shared matrices ---------------

// LU with partial pivoting of A (p x p) and the solve for B (p x nr) in place.
__device__ void warp_lu(double* A, double* B, int p, int nr, int ld, int lane) {
    for (int k = 0; k < p; ++k) {
        // pivot: first row of max |a| (LAPACK idamax)
        double best = -1.0;
        int bi = p;
        for (int i = k + lane; i < p; i += 32) {
            const double v = fabs(A[k * ld + i]);
            if (v > best || (v == best && i < bi) || (v != v && best == -1.0)) {
                best = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(FULL, best, o);
            const int oi = __shfl_xor_sync(FULL, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if (bi >= p) bi = k;
        if (bi != k) {
            for (int c = lane; c < p; c += 32) {
                const double t = A[c * ld + k];
                A[c * ld + k] = A[c * ld + bi];
                A[c * ld + bi] = t;
            }
            for (int c = lane; c < nr; c += 32) {
                const double t = B[c * ld + k];
                B[c * ld + k] = B[c * ld + bi];
                B[c * ld + bi] = t;
            }
        }
        __syncwarp();
        const double inv = 1.0 / A[k * ld + k];
        for (int i = k + 1 + lane; i < p; i += 32) A[k * ld + i] *= inv;
        __syncwarp();
        // trailing update, one column per lane
        for (int c = k + 1 + lane; c < p + nr; c += 32) {
            double* col = c < p ? A + c * ld : B + (c - p) * ld;
            const double akc = col[k];
            if (akc != 0.0)
                for (int i = k + 1; i < p; ++i) col[i] = fma(-A[k * ld + i], akc, col[i]);
        }
        __syncwarp();
    }
    // back substitution U x = y, column-oriented, right-hand sides per lane
    for (int k = p - 1; k >= 0; --k) {
        for (int c = lane; c < nr; c += 32) {
            double* b = B + c * ld;
            const double xk = b[k] / A[k * ld + k];
            b[k] = xk;
            for (int i = 0; i < k; ++i) b[i] = fma(-A[k * ld + i], xk, b[i]);
        }
    }
    __syncwarp();
}

// Householder QR of A (p x q, p >= q) in place: v below the diagonal (v_k = 1
// implicit), R on and above, tau[k].  Columns of B (p x nr, may be null) are
// transformed by Q^T as they go.  With piv (q ints, nullable) the columns are
// pivoted as in LAPACK dgeqp3 (largest remaining column norm first, first one
// on ties; cn = q doubles of scratch): the reference's gelsy starts from that
// factorisation, and it keeps badly scaled systems (monomial columns against
// kernel columns under "nearest" scaling) accurate.
__device__ void warp_householder(double* A, double* B, double* tau, int p, int q, int nr, int ld, int lane,
                                 int* piv = nullptr, double* cn = nullptr) {
    if (piv) {
        for (int c = lane; c < q; c += 32) {
            double s2 = 0.0;
            for (int i = 0; i < p; ++i) s2 = fma(A[c * ld + i], A[c * ld + i], s2);
            cn[c] = s2;
            piv[c] = c;
        }
        __syncwarp();
    }
    for (int k = 0; k < q; ++k) {
        if (piv) {
            double best = -1.0;
            int bj = q;
            for (int c = k + lane; c < q; c += 32)
                if (cn[c] > best) {
                    best = cn[c];
                    bj = c;
                }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(FULL, best, o);
                const int oj = __shfl_xor_sync(FULL, bj, o);
                if (ob > best || (ob == best && oj < bj)) {
                    best = ob;
                    bj = oj;
                }
            }
            if (bj < q && bj != k) {
                for (int i = lane; i < p; i += 32) {
                    const double t = A[k * ld + i];
                    A[k * ld + i] = A[bj * ld + i];
                    A[bj * ld + i] = t;
                }
                __syncwarp();
                if (lane == 0) {
                    const int t = piv[k];
                    piv[k] = piv[bj];
                    piv[bj] = t;
                    const double tc = cn[k];
                    cn[k] = cn[bj];
                    cn[bj] = tc;
                }
            }
            __syncwarp();
        }
        double* a = A + k * ld;
        double s = 0.0;
        for (int i = k + 1 + lane; i < p; i += 32) s += a[i] * a[i];
        s = warp_sum(s);
        const double x0 = a[k];
        double t = 0.0, beta = x0, scal = 0.0;
        if (s > 0.0) {
            const double nrm = sqrt(x0 * x0 + s);
            beta = x0 >= 0.0 ? -nrm : nrm;
            t = (beta - x0) / beta;
            scal = 1.0 / (x0 - beta);
        }
        __syncwarp();
        if (t != 0.0)
            for (int i = k + 1 + lane; i < p; i += 32) a[i] *= scal;
        if (lane == 0) {
            a[k] = beta;
            tau[k] = t;
        }
        __syncwarp();
        for (int c = k + 1 + lane; c < q + nr; c += 32) {
            double* col = c < q ? A + c * ld : B + (c - q) * ld;
            if (t != 0.0) {
                double dot = col[k];
                for (int i = k + 1; i < p; ++i) dot = fma(a[i], col[i], dot);
                dot *= t;
                col[k] -= dot;
                for (int i = k + 1; i < p; ++i) col[i] = fma(-dot, a[i], col[i]);
            }
            if (piv && c < q) {  // remaining norm below row k (recomputed: no cancellation)
                double s2 = 0.0;
                for (int i = k + 1; i < p; ++i) s2 = fma(col[i], col[i], s2);
                cn[c] = s2;
            }
        }
        __syncwarp();
    }
}

// x = R^-1 y for the upper-triangular q x q R (in A), right-hand sides in the
// first q rows of B's columns
__device__ void warp_rsolve(const double* A, double* B, int q, int nr, int ld, int lane) {
    for (int k = q - 1; k >= 0; --k) {
        for (int c = lane; c < nr; c += 32) {
            double* b = B + c * ld;
            const double xk = b[k] / A[k * ld + k];
            b[k] = xk;
            for (int i = 0; i < k; ++i) b[i] = fma(-A[k * ld + i], xk, b[i]);
        }
    }
    __syncwarp();
}

// minimum-norm solution of C^T x = b for C (p x q, p >= q) factored by
// warp_householder: R^T z = b (forward), x = Q [z; 0].  b: first q rows of
// B's columns; x overwrites the first p rows.
__device__ void warp_minnorm(const double* A, const double* tau, double* B, int p, int q, int nr, int ld,
                             int lane) {
    for (int c = lane; c < nr; c += 32) {
        double* b = B + c * ld;
        for (int k = 0; k < q; ++k) {
            double acc = b[k];
            for (int i = 0; i < k; ++i) acc = fma(-A[k * ld + i], b[i], acc);  // R[i][k] = A[k*ld+i]
            b[k] = acc / A[k * ld + k];
        }
        for (int i = q; i < p; ++i) b[i] = 0.0;
        for (int k = q - 1; k >= 0; --k) {
            const double* v = A + k * ld;
            double dot = b[k];
            for (int i = k + 1; i < p; ++i) dot = fma(v[i], b[i], dot);
            dot *= tau[k];
            b[k] -= dot;
            for (int i = k + 1; i < p; ++i) b[i] = fma(-dot, v[i], b[i]);
        }
    }
    __syncwarp();
}

// One-sided Jacobi SVD of T (p x q, p >= q): T's columns become U Sigma, V
// (q x q) accumulates the rotations.  Round-robin pair order, one pair per lane.
__device__ void warp_jacobi(double* T, double* V, int* perm, int p, int q, int ld, int ldv, int lane) {
    for (int c = lane; c < q; c += 32)
        for (int i = 0; i < q; ++i) V[c * ldv + i] = i == c ? 1.0 : 0.0;
    const int qq = q + (q & 1);  // even player count (a dummy column when q is odd)
    for (int i = lane; i < qq; i += 32) perm[i] = i;
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rot = 0;
        for (int round = 0; round < qq - 1; ++round) {
            for (int pr = lane; pr < qq / 2; pr += 32) {
                int ci = perm[pr], cj = perm[qq - 1 - pr];
                if (ci >= q || cj >= q) continue;
                if (ci > cj) {
                    const int t = ci;
                    ci = cj;
                    cj = t;
                }
                double* ti = T + ci * ld;
                double* tj = T + cj * ld;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = 0; r < p; ++r) {
                    al = fma(ti[r], ti[r], al);
                    be = fma(tj[r], tj[r], be);
                    ga = fma(ti[r], tj[r], ga);
                }
                if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                    for (int r = 0; r < p; ++r) {
                        const double a = ti[r], b = tj[r];
                        ti[r] = cs * a - sn * b;
                        tj[r] = sn * a + cs * b;
                    }
                    double* vi = V + ci * ldv;
                    double* vj = V + cj * ldv;
                    for (int r = 0; r < q; ++r) {
                        const double a = vi[r], b = vj[r];
                        vi[r] = cs * a - sn * b;
                        vj[r] = sn * a + cs * b;
                    }
                    rot = 1;
                }
            }
            __syncwarp();
            // rotate the schedule: player 0 stays, the others shift by one
            int nxt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = lane + 32 * u;
                nxt[u] = i < qq ? (i == 0 ? perm[0] : perm[i == 1 ? qq - 1 : i - 1]) : 0;
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (lane + 32 * u < qq) perm[lane + 32 * u] = nxt[u];
            __syncwarp();
        }
        if (!__any_sync(FULL, rot)) break;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(EW * 32) engine_k(EngArgs a) {
    extern __shared__ double esm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const mf_engine_t& E = a.E;
    const int n = a.n, d = E.d, l = E.l, nf = E.nf, ld = a.ld;
    const bool wls = E.engine == MF_ENGINE_WLS;
    double* X = esm + (size_t)wib * a.warp_dbl;       // n x d local coordinates (scaled)
    double* WD = X + ((n * d + 1) & ~1);              // n WLS weights
    double* A = WD + ((n + 1) & ~1);                  // ld x q
    double* B = A + (size_t)ld * a.q;                 // ld x nf
    double* TAU = B + (size_t)ld * nf;                // q
    double* V = TAU + ((a.q + 1) & ~1);               // (svd) q x (q | 1)
    double* SCR = V + (E.solver == MF_SOLVER_SVD ? (size_t)a.q * (a.q | 1) : 0);  // svd: coefficients, solution; qr: column norms
    int* PERM = reinterpret_cast<int*>(SCR + ((a.q + a.p + 1) & ~1));  // (svd) pair schedule
    const int s_sys = wls ? 0 : n + l;

    for (int64_t idx = (int64_t)blockIdx.x * EW + wib; idx < a.m; idx += (int64_t)gridDim.x * EW) {
        const int64_t row = a.rows[idx];
        const int32_t* st = a.stencils + idx * n;
        // local offsets and the scale (engines.py:42-59)
        for (int e = lane; e < n * d; e += 32) {
            const int j = e / d, ax = e - j * d;
            X[e] = a.pos[(int64_t)st[j] * d + ax] - a.pos[row * d + ax];
        }
        __syncwarp();
        double sc = 1.0;
        int stat_all = 0;
        if (E.scale_code != MF_SCALE_NONE) {
            const bool nearest = E.scale_code == MF_SCALE_NEAREST;
            double best = nearest ? INFINITY : 0.0;
            for (int j = lane; j < n; j += 32) {
                double r2 = 0.0;
                for (int ax = 0; ax < d; ++ax) r2 += X[j * d + ax] * X[j * d + ax];
                const double r = sqrt(r2);
                if (nearest) {
                    if (r > 0.0) best = fmin(best, r);
                } else {
                    best = fmax(best, r);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(FULL, best, o);
                best = nearest ? fmin(best, ob) : fmax(best, ob);
            }
            if (nearest ? !(best < INFINITY) : !(best > 0.0)) stat_all = 2;
            sc = best;
        }
        unsigned sing_mask = 0;  // families whose polyharmonic derivative is singular at the centre
        bool wbad = false;
        if (stat_all == 0) {
            for (int e = lane; e < n * d; e += 32) X[e] = X[e] / sc;
            __syncwarp();
            // family scale factors s^-order per term
            if (!wls) {
                // system [Phi Q; Q^T 0], column-major (engines.py:183-196)
                const int s = s_sys;
                for (int c = lane; c < s; c += 32) {
                    double* col = A + (size_t)c * ld;
                    for (int i = 0; i < s; ++i) {
                        double v;
                        if (i < n && c < n) {
                            double r2 = 0.0;
                            for (int ax = 0; ax < d; ++ax) {
                                const double df = X[i * d + ax] - X[c * d + ax];
                                r2 += df * df;
                            }
                            v = rbf_value(E, sqrt(r2));
                        } else if (i < n) {
                            v = monomial(E, c - n, X + i * d, d);
                        } else if (c < n) {
                            v = monomial(E, i - n, X + c * d, d);
                        } else {
                            v = 0.0;
                        }
                        col[i] = v;
                    }
                }
                // right-hand sides: top (L phi)(0 - x_j), bottom (L b_j)(0), each
                // term times coeff * s^-order, summed term by term (engines.py:92-99)
                for (int e = lane; e < s * nf; e += 32) {
                    const int f = e / s, i = e - f * s;
                    double acc = 0.0;
                    bool sing = false;
                    for (int t = E.term0[f]; t < E.term0[f + 1]; ++t) {
                        const double fac = E.term_coeff[t] * pow(sc, (double)-E.term_order[t]);
                        const double v = i < n ? term_rbf(E, t, X + i * d, d, &sing) : term_mono0(E, t, i - n, d);
                        acc = t == E.term0[f] ? fac * v : acc + fac * v;
                    }
                    B[(size_t)f * ld + i] = acc;
                    if (sing) sing_mask |= 1u << f;
                }
            } else {
                // WLS: w_j = weight(local_j) > 0, C = W B (n x l): the system is C^T
                for (int j = lane; j < n; j += 32) {
                    double w = 1.0;
                    if (E.weight == MF_WEIGHT_GAUSSIAN) {
                        double r2 = 0.0;
                        for (int ax = 0; ax < d; ++ax) r2 += X[j * d + ax] * X[j * d + ax];
                        w = exp(-r2 / (E.weight_sigma * E.weight_sigma));
                    }
                    WD[j] = w;
                    if (!(w > 0.0)) wbad = true;
                }
                wbad = __any_sync(FULL, wbad);
                __syncwarp();
                if (a.wide) {
                    for (int c = lane; c < l; c += 32)
                        for (int j = 0; j < n; ++j) A[(size_t)c * ld + j] = WD[j] * monomial(E, c, X + j * d, d);
                } else {
                    for (int c = lane; c < n; c += 32)
                        for (int i = 0; i < l; ++i) A[(size_t)c * ld + i] = WD[c] * monomial(E, i, X + c * d, d);
                }
                for (int e = lane; e < l * nf; e += 32) {
                    const int f = e / l, i = e - f * l;
                    double acc = 0.0;
                    for (int t = E.term0[f]; t < E.term0[f + 1]; ++t) {
                        const double fac = E.term_coeff[t] * pow(sc, (double)-E.term_order[t]);
                        const double v = term_mono0(E, t, i, d);
                        acc = t == E.term0[f] ? fac * v : acc + fac * v;
                    }
                    B[(size_t)f * ld + i] = acc;
                }
            }
        }
        // union of lanes' singular flags
#pragma unroll
        for (int o = 16; o; o >>= 1) sing_mask |= __shfl_xor_sync(FULL, sing_mask, o);
        __syncwarp();
        const bool solve = stat_all == 0 && !wbad;
        if (solve) {
            const int p = a.p, q = a.q;
            if (E.solver == MF_SOLVER_LU) {
                warp_lu(A, B, p, nf, ld, lane);
            } else if (E.solver == MF_SOLVER_QR) {
                if (a.wide) {
                    warp_householder(A, nullptr, TAU, p, q, 0, ld, lane);
                    warp_minnorm(A, TAU, B, p, q, nf, ld, lane);
                } else {
                    // column-pivoted: x[piv[j]] = (R^-1 Q^T b)[j]
                    warp_householder(A, B, TAU, p, q, nf, ld, lane, PERM, SCR);
                    warp_rsolve(A, B, q, nf, ld, lane);
                    for (int f = 0; f < nf; ++f) {
                        double* b = B + (size_t)f * ld;
                        double v[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = lane + 32 * u;
                            v[u] = j < q ? b[j] : 0.0;
                        }
                        __syncwarp();
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int j = lane + 32 * u;
                            if (j < q) b[PERM[j]] = v[u];
                        }
                        __syncwarp();
                    }
                }
            } else {
                const int ldv = q | 1;
                warp_jacobi(A, V, PERM, p, q, ld, ldv, lane);
                // sigma_j = |t_j|; cutoff 1e-13 sigma_max (engines.py:84-88)
                double smax = 0.0;
                for (int c = lane; c < q; c += 32) {
                    double s2 = 0.0;
                    for (int r = 0; r < p; ++r) s2 = fma(A[(size_t)c * ld + r], A[(size_t)c * ld + r], s2);
                    TAU[c] = s2;
                    smax = fmax(smax, sqrt(s2));
                }
                smax = warp_maxd(smax);
                __syncwarp();
                const double cut = 1e-13 * smax;
                // per family: c_j = (t_j . b) / s_j^2 (tall) or (v_j . b) / s_j^2 (wide),
                // then x = sum_j c_j v_j (tall) or sum_j c_j t_j (wide)
                const int nout = a.wide ? p : q;
                for (int f = 0; f < nf; ++f) {
                    double* b = B + (size_t)f * ld;
                    for (int c = lane; c < q; c += 32) {
                        const double s2 = TAU[c];
                        double cj = 0.0;
                        if (sqrt(s2) > cut) {
                            double dot = 0.0;
                            if (!a.wide)
                                for (int r = 0; r < p; ++r) dot = fma(A[(size_t)c * ld + r], b[r], dot);
                            else
                                for (int r = 0; r < q; ++r) dot = fma(V[(size_t)c * ldv + r], b[r], dot);
                            cj = dot / s2;
                        }
                        SCR[c] = cj;
                    }
                    __syncwarp();
                    for (int r = lane; r < nout; r += 32) {
                        double x = 0.0;
                        for (int c = 0; c < q; ++c)
                            x = fma(a.wide ? A[(size_t)c * ld + r] : V[(size_t)c * ldv + r], SCR[c], x);
                        SCR[q + r] = x;
                    }
                    __syncwarp();
                    for (int r = lane; r < nout; r += 32) b[r] = SCR[q + r];
                    __syncwarp();
                }
            }
        }
        // outputs: RbfFd w = x[:n]; WLS w = W y (engines.py:138, 197-201)
        for (int e = lane; e < nf * n; e += 32) {
            const int f = e / n, j = e - f * n;
            double w = 0.0;
            if (solve) {
                w = B[(size_t)f * ld + j];
                if (wls) w = WD[j] * w;
            }
            a.out[((size_t)idx * nf + f) * n + j] = w;
        }
        unsigned nonfin = 0;
        if (solve)
            for (int e = lane; e < nf * n; e += 32) {
                const int f = e / n;
                if (!isfinite(a.out[((size_t)idx * nf + f) * n + (e - f * n)])) nonfin |= 1u << f;
            }
#pragma unroll
        for (int o = 16; o; o >>= 1) nonfin |= __shfl_xor_sync(FULL, nonfin, o);
        bool any = false;
        for (int f = lane; f < nf; f += 32) {
            int8_t code = 0;
            if (stat_all) code = (int8_t)stat_all;
            else if (sing_mask & (1u << f)) code = 3;
            else if (wbad) code = 4;
            else if (nonfin & (1u << f)) code = 1;
            a.status[idx * nf + f] = code;
            any |= code != 0;
        }
        if (__any_sync(FULL, any) && lane == 0) atomicMin(a.first_fail, (unsigned long long)idx);
        __syncwarp();
    }
}

}  // namespace

int engine_sizes(const mf_engine_t& E, int n, int& p, int& q, int& wide, int& ld, int& warp_dbl) {
    const int d = E.d, l = E.l, nf = E.nf;
    wide = 0;
    if (E.engine == MF_ENGINE_RBFFD) {
        p = q = n + l;
    } else {
        // system (W B)^T: l equations, n unknowns
        if (E.solver == MF_SOLVER_LU) {
            if (l != n) return MF_ERR_ARG;
            p = l;
            q = n;
        } else if (l <= n) {
            wide = 1;  // stored as W B (n x l)
            p = n;
            q = l;
        } else {
            p = l;
            q = n;
        }
    }
    // rows of the stored matrix and of the right-hand sides (l equations for WLS)
    const int rows = E.engine == MF_ENGINE_RBFFD ? n + l : (p > l ? p : l);
    ld = rows | 1;
    size_t v = (size_t)((n * d + 1) & ~1) + ((n + 1) & ~1) + (size_t)ld * q + (size_t)ld * nf + ((q + 1) & ~1);
    if (E.solver == MF_SOLVER_SVD) {
        if (q > 128) return MF_ERR_UNSUPPORTED;
        v += (size_t)q * (q | 1) + ((q + p + 1) & ~1) + (q + 2) / 2 + 1;  // V, SCR, PERM
    } else if (E.solver == MF_SOLVER_QR) {
        if (q > 256) return MF_ERR_UNSUPPORTED;
        v += ((q + p + 1) & ~1) + (q + 2) / 2 + 1;  // SCR (column norms), PERM (pivots)
    }
    warp_dbl = (int)((v + 1) & ~(size_t)1);
    return MF_OK;
}

}  // namespace mf

extern "C" int mf_engine_weights(const double* pos, int64_t N, const int64_t* rows, const int32_t* stencils,
                                 int64_t m, int32_t n, const mf_engine_t* eng, double* out, int8_t* status,
                                 int64_t* first_fail, void* stream) {
    using namespace mf;
    MF_REQUIRE(eng != nullptr, "mf_engine_weights: null engine descriptor");
    const mf_engine_t& E = *eng;
    MF_REQUIRE(E.d >= 1 && E.d <= MF_MAX_DIM, "mf_engine_weights: bad dimension %d", E.d);
    MF_REQUIRE(E.nf >= 1 && E.nf <= MF_MAX_FAMILIES, "mf_engine_weights: bad family count %d", E.nf);
    MF_REQUIRE(E.l >= 0 && E.l <= MF_MAX_MONOMIALS, "mf_engine_weights: bad monomial count %d", E.l);
    MF_REQUIRE(E.term0[0] == 0 && E.term0[E.nf] <= MF_MAX_ENGINE_TERMS, "mf_engine_weights: bad term table");
    for (int f = 0; f < E.nf; ++f)
        MF_REQUIRE(E.term0[f + 1] > E.term0[f], "mf_engine_weights: family %d has no terms", f);
    for (int t = 0; t < E.term0[E.nf]; ++t)
        MF_REQUIRE(E.term_kind[t] >= MF_TERM_IDENTITY && E.term_kind[t] <= MF_TERM_DIRECTIONAL &&
                       E.term_a[t] >= 0 && E.term_a[t] < E.d && E.term_b[t] >= 0 && E.term_b[t] < E.d,
                   "mf_engine_weights: bad term %d", t);
    MF_REQUIRE(E.engine == MF_ENGINE_RBFFD || E.engine == MF_ENGINE_WLS, "mf_engine_weights: bad engine");
    MF_REQUIRE(E.solver >= MF_SOLVER_LU && E.solver <= MF_SOLVER_SVD, "mf_engine_weights: bad solver");
    MF_REQUIRE(E.rbf >= MF_RBF_PHS && E.rbf <= MF_RBF_IMQ, "mf_engine_weights: bad kernel");
    MF_REQUIRE(E.scale_code >= MF_SCALE_NONE && E.scale_code <= MF_SCALE_SUPPORT, "mf_engine_weights: bad scale");
    MF_REQUIRE(n >= 1 && m >= 0, "mf_engine_weights: bad sizes");
    MF_REQUIRE(E.engine == MF_ENGINE_WLS ? E.l >= 1 : true, "mf_engine_weights: empty least-squares basis");
    MF_REQUIRE(E.engine == MF_ENGINE_WLS || E.rbf != MF_RBF_PHS || E.k >= 1, "mf_engine_weights: bad exponent");
    MF_REQUIRE(E.engine == MF_ENGINE_WLS || E.rbf == MF_RBF_PHS || E.sigma > 0.0, "mf_engine_weights: bad shape parameter");
    EngArgs a{};
    a.pos = pos;
    a.rows = rows;
    a.stencils = stencils;
    a.m = m;
    a.n = n;
    a.out = out;
    a.status = status;
    a.first_fail = reinterpret_cast<unsigned long long*>(first_fail);
    a.E = E;
    const int rc = engine_sizes(E, n, a.p, a.q, a.wide, a.ld, a.warp_dbl);
    if (rc != MF_OK) {
        set_error(rc == MF_ERR_ARG ? "mf_engine_weights: lu needs a square local system"
                                   : "mf_engine_weights: local system too large for the svd (128) / qr (256) solver");
        return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    MF_CUDA_CHECK(cudaMemsetAsync(first_fail, 0x7f, sizeof(int64_t), st));
    if (m == 0) return MF_OK;
    const size_t smem = (size_t)EW * a.warp_dbl * sizeof(double);
    MF_REQUIRE(smem <= (size_t)dev_max_smem_optin(), "mf_engine_weights: local system too large (%zu bytes)", smem);
    MF_CUDA_CHECK(ensure_smem(engine_k, (int)smem));
    const int per_sm = occupancy(engine_k, EW * 32, smem);
    int64_t blocks = (m + EW - 1) / EW;
    const int64_t cap = (int64_t)dev_sms() * (per_sm > 0 ? per_sm : 1) * 4;
    if (blocks > cap) blocks = cap;
    engine_k<<<(unsigned)blocks, EW * 32, smem, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

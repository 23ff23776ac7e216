// CTA-per-stencil shape solve for large or unusual stencil shapes (sm_100a).
//
// One thread block (W warps) per stencil; the augmented system [A | B] lives
// in shared memory (s x (s + nrhs) doubles: 92 KB for C5's s = 105, so two
// blocks per SM).  The W warps split every elimination step: the pivot search
// is a block-wide argmax over (|a|, position) (warp REDUX-free reduction +
// shared scratch), the row swap and rank-1 update are distributed rows-over-
// warps / columns-over-lanes with the pivot row cached in registers.
// REPLAY follows _solve_multi (_phs_batch.py:142-184) op for op; FAST uses FMA
// and carries the +-1 probe right-hand side for the HYBRID criterion, exactly
// as the warp kernels do.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "phs_params.cuh"
#include "phs_reg.cuh"  // fast_rcp, fast_rsqrt
#include "phs_nullspace.cuh"  // dmma_f64, monomials_reg

namespace mf {

constexpr int CTA_WARPS = 8;
constexpr int CTA_THREADS = CTA_WARPS * 32;
constexpr int CTA_MAXCOLS = 128;  // s + nrhs: pivot-row cache of 4 values per lane

__host__ __device__ inline size_t cta_doubles(int n, int d, int s, int nrhs) {
    size_t v = (size_t)n * d + (size_t)s * (s + nrhs) + (size_t)nrhs * s + 4 * CTA_WARPS + 8;
    return (v + 1) & ~(size_t)1;
}

// block-wide argmax of (value, -pos), NaN never wins; returns via shared scratch
__device__ __forceinline__ void block_argmax(double v, int pos, double* sv, int* sp, double& best, int& bpos) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(FULL, v, o);
        int op = __shfl_xor_sync(FULL, pos, o);
        if (ov > v || (ov == v && op < pos)) {
            v = ov;
            pos = op;
        }
    }
    if (lane == 0) {
        sv[w] = v;
        sp[w] = pos;
    }
    __syncthreads();
    // every warp reduces the CTA_WARPS candidates in its first lanes (3 shuffle steps)
    v = lane < CTA_WARPS ? sv[lane] : -INFINITY;
    pos = lane < CTA_WARPS ? sp[lane] : 0x7fffffff;
#pragma unroll
    for (int o = CTA_WARPS / 2; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(FULL, v, o);
        int op = __shfl_xor_sync(FULL, pos, o);
        if (ov > v || (ov == v && op < pos)) {
            v = ov;
            pos = op;
        }
    }
    best = __shfl_sync(FULL, v, 0);
    bpos = __shfl_sync(FULL, pos, 0);
    __syncthreads();
}

__device__ __forceinline__ double block_reduce_max(double v, double* sv) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    if (lane == 0) sv[w] = v;
    __syncthreads();
    double r = sv[0];
    for (int k = 1; k < CTA_WARPS; ++k) r = fmax(r, sv[k]);
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_reduce_min(double v, double* sv) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    if (lane == 0) sv[w] = v;
    __syncthreads();
    double r = sv[0];
    for (int k = 1; k < CTA_WARPS; ++k) r = fmin(r, sv[k]);
    __syncthreads();
    return r;
}

template <bool REPLAY>
__global__ void __launch_bounds__(CTA_THREADS) phs_cta(PhsArgs a, const int64_t* __restrict__ list,
                                                       const int64_t* __restrict__ list_count) {
    extern __shared__ double smem_c[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = a.n, d = a.P.d, l = a.P.l, nf = a.P.nf;
    const int s = n + l;
    constexpr bool PROBE = !REPLAY;
    const int nrhs = nf + (PROBE ? 1 : 0);
    const int lda = s + nrhs;
    double* loc = smem_c;
    double* A = loc + n * d;
    double* scr = A + (size_t)s * lda;
    double* red = scr + (size_t)nrhs * s;
    int* redi = reinterpret_cast<int*>(red + 2 * CTA_WARPS);
    const int64_t count = list ? *list_count : a.m;
    const bool want_flag = PROBE && a.flag_list != nullptr;
    const bool want_est = PROBE && (a.flag_list != nullptr || a.kappa != nullptr);
    const PhsParams& P = a.P;

    for (int64_t it = blockIdx.x; it < count; it += gridDim.x) {
        const int64_t idx = list ? list[it] : it;
        const int64_t row = a.rows[idx];
        const int32_t* sti = a.stencils + idx * n;
        // 1. local coordinates (_phs_batch.py:198-202)
        for (int e = tid; e < n * d; e += CTA_THREADS) {
            int j = e / d, ax = e - j * d;
            loc[e] = __dsub_rn(a.pos[(int64_t)sti[j] * d + ax], a.pos[row * d + ax]);
        }
        __syncthreads();
        // 2. scale (_phs_batch.py:204-221)
        int stat = 0;
        double sc = 1.0;
        if (P.scale_code != MF_SCALE_NONE) {
            const bool nearest = P.scale_code == MF_SCALE_NEAREST;
            double best = nearest ? INFINITY : -1.0;
            for (int j = tid; j < n; j += CTA_THREADS) {
                double r2 = 0.0;
                for (int ax = 0; ax < d; ++ax) r2 = __dadd_rn(r2, __dmul_rn(loc[j * d + ax], loc[j * d + ax]));
                double r = __dsqrt_rn(r2);
                if (nearest) {
                    if (r > 0.0 && r < best) best = r;
                } else if (r > best) {
                    best = r;
                }
            }
            best = nearest ? block_reduce_min(best, red) : block_reduce_max(best, red);
            if (nearest ? (best == INFINITY) : !(best > 0.0)) stat = 2;
            else sc = best;
        }
        double anorm = 0.0, r2min = INFINITY, rc2max = 0.0;
        if (stat == 0) {
            for (int e = tid; e < n * d; e += CTA_THREADS) loc[e] = __ddiv_rn(loc[e], sc);
            __syncthreads();
            // 3. system (_phs_batch.py:228-290); PHS block symmetric, one evaluation per pair
            for (int e = tid; e < n * n; e += CTA_THREADS) {
                int i = e / n, j = e - i * n;
                if (j < i) continue;
                double v = 0.0;
                if (j > i) {
                    double r2 = 0.0;
                    for (int ax = 0; ax < d; ++ax) {
                        double df = __dsub_rn(loc[i * d + ax], loc[j * d + ax]);
                        r2 = __dadd_rn(r2, __dmul_rn(df, df));
                    }
                    r2min = fmin(r2min, r2);
                    v = phs_phi(__dsqrt_rn(r2), P.k, P.even);
                }
                A[(size_t)i * lda + j] = v;
                A[(size_t)j * lda + i] = v;
            }
            for (int e = tid; e < n * l; e += CTA_THREADS) {
                int jm = e / n, i = e - jm * n;
                double q = phs_monomial(loc + i * d, P.expos + jm * d, d);
                A[(size_t)i * lda + n + jm] = q;
                A[(size_t)(n + jm) * lda + i] = q;
            }
            for (int e = tid; e < l * l; e += CTA_THREADS) {
                int i = e / l, j = e - i * l;
                A[(size_t)(n + i) * lda + n + j] = 0.0;
            }
            for (int j = tid; j < n; j += CTA_THREADS) {
                double top[MF_MAX_FAMILIES];
                phs_rhs_top(loc + j * d, d, P, top);
                for (int f = 0; f < nf; ++f) A[(size_t)j * lda + s + f] = __dmul_rn(top[f], pow_cr_int(sc, -P.orders[f]));
                double rc2 = 0.0;
                for (int ax = 0; ax < d; ++ax) rc2 = fma(loc[j * d + ax], loc[j * d + ax], rc2);
                rc2max = fmax(rc2max, rc2);
            }
            for (int e = tid; e < l * nf; e += CTA_THREADS) {
                int f = e / l, j = e - f * l;
                A[(size_t)(n + j) * lda + s + f] = __dmul_rn(P.base_bot[f * MF_MAX_MONOMIALS + j], pow_cr_int(sc, -P.orders[f]));
            }
            if (PROBE)
                for (int r = tid; r < s; r += CTA_THREADS) A[(size_t)r * lda + s + nf] = probe_sign(idx, r);
            __syncthreads();
            if (want_est) {
                double mx = 0.0;
                for (int r = tid; r < s; r += CTA_THREADS) {
                    double acc = 0.0;
                    for (int c = 0; c < s; ++c) acc += fabs(A[(size_t)r * lda + c]);
                    mx = fmax(mx, acc);
                }
                anorm = block_reduce_max(mx, red);
            }
            // 4. elimination with row partial pivoting (_phs_batch.py:150-176)
            for (int col = 0; col < s; ++col) {
                double best = -1.0;
                int piv = 0x7fffffff;
                for (int r = col + tid; r < s; r += CTA_THREADS) {
                    double v = fabs(A[(size_t)r * lda + col]);
                    if (v > best) {
                        best = v;
                        piv = r;
                    }
                }
                const double a00 = fabs(A[(size_t)col * lda + col]);
                block_argmax(best, piv, red, redi, best, piv);
                if (isnan(a00) || best == 0.0 || !isfinite(best) || piv == 0x7fffffff) {
                    stat = 1;
                    break;
                }
                if (piv != col) {
                    for (int cc = col + tid; cc < lda; cc += CTA_THREADS) {
                        double t = A[(size_t)col * lda + cc];
                        A[(size_t)col * lda + cc] = A[(size_t)piv * lda + cc];
                        A[(size_t)piv * lda + cc] = t;
                    }
                    __syncthreads();
                }
                const double inv = __drcp_rn(A[(size_t)col * lda + col]);
                const double* prow = A + (size_t)col * lda;
                double pv[CTA_MAXCOLS / 32];
#pragma unroll
                for (int q = 0; q < CTA_MAXCOLS / 32; ++q) {
                    const int cc = col + 1 + lane + 32 * q;
                    pv[q] = cc < lda ? prow[cc] : 0.0;
                }
                for (int r = col + 1 + w; r < s; r += CTA_WARPS) {
                    double* arow = A + (size_t)r * lda;
                    const double fac = REPLAY ? __dmul_rn(arow[col], inv) : arow[col] * inv;
                    if (!REPLAY || fac != 0.0) {  // the reference skips zero multipliers
#pragma unroll
                        for (int q = 0; q < CTA_MAXCOLS / 32; ++q) {
                            const int cc = col + 1 + lane + 32 * q;
                            if (cc < lda) {
                                if (REPLAY) arow[cc] = __dsub_rn(arow[cc], __dmul_rn(fac, pv[q]));
                                else arow[cc] = fma(-fac, pv[q], arow[cc]);
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
        if (stat == 0) {
            // 5. back-substitution (_phs_batch.py:177-183)
            if (REPLAY) {
                for (int col = s - 1; col >= 0; --col) {
                    const int len = s - col - 1;
                    for (int e = tid; e < len * nf; e += CTA_THREADS) {
                        int f = e / len, r = col + 1 + (e - f * len);
                        scr[f * s + r] = __dmul_rn(A[(size_t)col * lda + r], A[(size_t)r * lda + s + f]);
                    }
                    __syncthreads();
                    if (tid < nf) {
                        double acc = A[(size_t)col * lda + s + tid];
                        for (int r = col + 1; r < s; ++r) acc = __dsub_rn(acc, scr[tid * s + r]);
                        A[(size_t)col * lda + s + tid] = __dmul_rn(acc, __drcp_rn(A[(size_t)col * lda + col]));
                    }
                    __syncthreads();
                }
            } else {
                for (int col = s - 1; col >= 0; --col) {
                    if (tid < nrhs) A[(size_t)col * lda + s + tid] *= __drcp_rn(A[(size_t)col * lda + col]);
                    __syncthreads();
                    for (int r = tid; r < col; r += CTA_THREADS) {
                        double* arow = A + (size_t)r * lda;
                        const double u = arow[col];
                        for (int f = 0; f < nrhs; ++f) arow[s + f] = fma(-u, A[(size_t)col * lda + s + f], arow[s + f]);
                    }
                    __syncthreads();
                }
            }
            // 6. outputs, non-finite check (_phs_batch.py:293-298)
            double badv = 0.0;
            for (int e = tid; e < n * nf; e += CTA_THREADS) {
                int f = e / n, j = e - f * n;
                double v = A[(size_t)j * lda + s + f];
                if (!isfinite(v)) badv = 1.0;
                a.out[((size_t)idx * nf + f) * n + j] = v;
            }
            if (block_reduce_max(badv, red) > 0.0) stat = 1;
            if (want_est && stat == 0) {
                double zw = 0.0, za = 0.0;
                for (int r = tid; r < s; r += CTA_THREADS) {
                    double v = fabs(A[(size_t)r * lda + s + nf]);
                    za = fmax(za, v);
                    if (r < n) zw = fmax(zw, v);
                }
                zw = block_reduce_max(zw, red);
                za = block_reduce_max(za, red);
                double ratio = 0.0;
                for (int f = 0; f < nf; ++f) {
                    double xa = 0.0, xw = 0.0;
                    for (int r = tid; r < s; r += CTA_THREADS) {
                        double v = fabs(A[(size_t)r * lda + s + f]);
                        xa = fmax(xa, v);
                        if (r < n) xw = fmax(xw, v);
                    }
                    xa = block_reduce_max(xa, red);
                    xw = block_reduce_max(xw, red);
                    ratio = fmax(ratio, xa / xw);
                }
                r2min = block_reduce_min(r2min, red);
                rc2max = block_reduce_max(rc2max, red);
                const double est = anorm * zw * ratio;
                const bool close = r2min < a.min_sep2 * rc2max;
                if (tid == 0 && a.kappa) {
                    a.kappa[4 * idx + 0] = anorm;
                    a.kappa[4 * idx + 1] = zw;
                    a.kappa[4 * idx + 2] = za;
                    a.kappa[4 * idx + 3] = ratio;
                }
                if (want_flag && tid == 0 && (close || !(est <= a.hybrid_thresh))) {
                    unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                    a.flag_list[slot] = idx;
                }
            }
        }
        if (want_flag && stat != 0) {
            if (tid == 0) {
                unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                a.flag_list[slot] = idx;
            }
            stat = 0;
        }
        if (tid == 0) {
            a.status[idx] = (int8_t)stat;
            if (stat && a.first_fail) atomicMin((unsigned long long*)a.first_fail, (unsigned long long)idx);
        }
        __syncthreads();
    }
}

template <bool REPLAY>
int launch_cta_t(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count, cudaStream_t st,
                 int sms) {
    const int s = a.n + a.P.l;
    const int nrhs = a.P.nf + (REPLAY ? 0 : 1);
    if (s + nrhs > CTA_MAXCOLS) return MF_ERR_UNSUPPORTED;
    const size_t bytes = cta_doubles(a.n, a.P.d, s, nrhs) * sizeof(double);
    if (bytes > (size_t)dev_max_smem_optin()) return MF_ERR_UNSUPPORTED;
    MF_CUDA_CHECK(ensure_smem(phs_cta<REPLAY>, (int)bytes));
    int per_sm = occupancy(phs_cta<REPLAY>, CTA_THREADS, bytes);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = max_count;
    int64_t cap = (int64_t)sms * per_sm * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    phs_cta<REPLAY><<<(unsigned)blocks, CTA_THREADS, bytes, st>>>(a, list, list_count);
    MF_LAUNCH_CHECK();
    return MF_OK;
}


// ---------------------------------------------------------------------------
// Nullspace solve for large stencils (HYBRID first pass, r^3, degree >= 1):
// the CTA counterpart of phs_ns.cuh.  Gauss-Jordan column elimination with
// partial pivoting over the nodes runs on the stacked matrix [Q; g^T]
// ((n + nrhs) x l): after l steps the
// free node rows hold W = Q2 Q1^-1 and the g rows the particular solutions
// w1p = Q1^-T g; the recorded column operations give Q1^-1 s for lambda.  The reduced system K v = Z^T (f - Phi w_p) (K = Z^T Phi Z,
// (n-l)^2, definite) is solved by pivot-free Gauss-Jordan on [K | b].  Every
// phase is a parallel sweep over a shared-memory array between barriers.
// ---------------------------------------------------------------------------
struct NsCtaLayout {
    int n, d, l, nrhs, M, RG, GP, KP;
    size_t loc, E, G, ops, F, Y, K, prow, colk, red, ints, total;
};

__host__ __device__ inline NsCtaLayout ns_cta_layout(int n, int d, int l, int nrhs) {
    NsCtaLayout L;
    L.n = n;
    L.d = d;
    L.l = l;
    L.nrhs = nrhs;
    L.M = n - l;
    L.RG = n + nrhs;  // node rows, then one row per right-hand side
    L.GP = l | 1;  // odd pitch: column sweeps hit distinct banks
    L.KP = (L.M + nrhs) | 1;
    size_t o = 0;
    auto take = [&](size_t c) { size_t at = o; o += (c + 1) & ~(size_t)1; return at; };
    L.loc = take((size_t)n * d);
    L.E = take((size_t)n * n);
    L.G = take((size_t)L.RG * L.GP);
    L.ops = take((size_t)l * L.GP + l);  // per step: pivot-row snapshot, then 1 / pivot
    L.F = take((size_t)n * nrhs);
    L.Y = take((size_t)l * L.M);
    L.K = take((size_t)L.M * L.KP);
    L.prow = take((size_t)(l > L.KP ? l : L.KP));
    const int lnf = l * (nrhs - 1);  // lambda right-hand sides
    L.colk = take((size_t)(L.RG > lnf ? L.RG : lnf));  // RG >= M
    L.red = take(4 * CTA_WARPS + 8);
    L.ints = take(((size_t)n + l + L.M + 1) / 2 + 1);  // isp[n], piv[l], nonpiv[M]
    L.total = o;
    return L;
}

// NN > 0: sizes fixed at compile time (every index split and loop bound folds);
// NN = 0: sizes from the call (any shape the launcher accepts)
template <int NN, int DD, int LL, int NF>
__global__ void __launch_bounds__(CTA_THREADS) phs_ns_cta(PhsArgs a) {
    extern __shared__ __align__(16) double smem_n[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const PhsParams& P = a.P;
    const int n = NN ? NN : a.n, d = NN ? DD : P.d, l = NN ? LL : P.l, nf = NN ? NF : P.nf, nrhs = nf + 1;
    const NsCtaLayout L = ns_cta_layout(n, d, l, nrhs);
    const int M = L.M, RG = L.RG, GP = L.GP, KP = L.KP;
    double* loc = smem_n + L.loc;
    double* E = smem_n + L.E;
    double* G = smem_n + L.G;
    double* F = smem_n + L.F;
    double* Y = smem_n + L.Y;
    double* K = smem_n + L.K;
    double* prow = smem_n + L.prow;
    double* colk = smem_n + L.colk;
    double* red = smem_n + L.red;
    int* redi = reinterpret_cast<int*>(red + 2 * CTA_WARPS);
    double* ops = smem_n + L.ops;
    double* invs = ops + (size_t)l * GP;
    int* isp = reinterpret_cast<int*>(smem_n + L.ints);
    int* piv = isp + n;
    int* nonpiv = piv + l;

    for (int64_t idx = blockIdx.x; idx < a.m; idx += gridDim.x) {
        const int64_t row = a.rows[idx];
        const int32_t* sti = a.stencils + idx * n;
        // ---- local coordinates, scale (max r^2, one root), family factors
        for (int e = tid; e < n * d; e += CTA_THREADS) {
            const int j = e / d, ax = e - j * d;
            loc[e] = a.pos[(int64_t)sti[j] * d + ax] - a.pos[row * d + ax];
        }
        __syncthreads();
        int stat = 0;
        double sc = 1.0;
        if (P.scale_code != MF_SCALE_NONE) {
            const bool nearest = P.scale_code == MF_SCALE_NEAREST;
            double best = nearest ? INFINITY : -1.0;
            for (int j = tid; j < n; j += CTA_THREADS) {
                double r2 = 0.0;
                for (int ax = 0; ax < d; ++ax) r2 = __dadd_rn(r2, __dmul_rn(loc[j * d + ax], loc[j * d + ax]));
                if (nearest) {
                    if (r2 > 0.0 && r2 < best) best = r2;
                } else if (r2 > best) {
                    best = r2;
                }
            }
            best = nearest ? block_reduce_min(best, red) : block_reduce_max(best, red);
            if (nearest ? (best == INFINITY) : !(best > 0.0)) stat = 2;
            else sc = __dsqrt_rn(best);
        }
        double facs[MF_MAX_FAMILIES];
        for (int f = 0; f < nf; ++f) facs[f] = pow_cr_int(sc, -P.orders[f]);
        const double rs = fast_rcp(sc);
        for (int e = tid; e < n * d; e += CTA_THREADS) loc[e] *= rs;
        for (int i = tid; i < n; i += CTA_THREADS) isp[i] = 0;
        __syncthreads();

        // ---- Phi (zero diagonal), [Q; g; I], node right-hand sides
        double r2min = INFINITY, rc2max = 0.0;
        for (int e = tid; e < n * n; e += CTA_THREADS) {
            const int i = e / n, j = e - i * n;
            if (j < i) continue;
            double v = 0.0;
            if (j > i) {
                double df = loc[i * d] - loc[j * d];
                double r2 = df * df;
                for (int ax = 1; ax < d; ++ax) {
                    df = loc[i * d + ax] - loc[j * d + ax];
                    r2 = fma(df, df, r2);
                }
                r2min = r2 < r2min ? r2 : r2min;
                v = r2 * (r2 * fast_rsqrt(fmax(r2, 1e-300)));
            }
            E[i * n + j] = v;
            E[j * n + i] = v;
        }
        for (int e = tid; e < n * l; e += CTA_THREADS) {
            const int i = e / l, m = e - i * l;
            G[i * GP + m] = phs_monomial(loc + i * d, P.expos + m * d, d);
        }
        for (int e = tid; e < nrhs * l; e += CTA_THREADS) {
            const int f = e / l, m = e - f * l;
            G[(n + f) * GP + m] = f < nf ? __dmul_rn(P.base_bot[f * MF_MAX_MONOMIALS + m], facs[f]) : probe_sign(idx, n + m);
        }
        for (int i = tid; i < n; i += CTA_THREADS) {
            double top[MF_MAX_FAMILIES];
            phs_rhs_top_k3(loc + i * d, d, P, top);
            for (int f = 0; f < nf; ++f) F[i * nrhs + f] = __dmul_rn(top[f], facs[f]);
            F[i * nrhs + nf] = probe_sign(idx, i);
            double rc2 = 0.0;
            for (int ax = 0; ax < d; ++ax) rc2 = fma(loc[i * d + ax], loc[i * d + ax], rc2);
            rc2max = fmax(rc2max, rc2);
        }
        __syncthreads();
        r2min = block_reduce_min(r2min, red);
        rc2max = block_reduce_max(rc2max, red);
        // ||A||_inf of the saddle-point matrix (estimate only)
        double anorm = 0.0;
        for (int r = tid; r < n + l; r += CTA_THREADS) {
            double acc = 0.0;
            if (r < n) {
                for (int j = 0; j < n; ++j) acc += E[r * n + j];  // r^3 >= 0
                for (int m = 0; m < l; ++m) acc += fabs(G[r * GP + m]);
            } else {
                for (int i = 0; i < n; ++i) acc += fabs(G[i * GP + (r - n)]);
            }
            anorm = fmax(anorm, acc);
        }
        anorm = block_reduce_max(anorm, red);

        // ---- Gauss-Jordan column elimination of [Q; g; I] with node pivoting
        bool ok = stat == 0;
        for (int k = 0; k < l && ok; ++k) {
            double best = -1.0;
            int pr = 0x7fffffff;
            for (int r = tid; r < n; r += CTA_THREADS) {
                const double v = isp[r] ? -1.0 : fabs(G[r * GP + k]);
                if (v > best) {
                    best = v;
                    pr = r;
                }
            }
            block_argmax(best, pr, red, redi, best, pr);
            if (!(best > 0.0) || !isfinite(best) || pr == 0x7fffffff) {
                ok = false;
                break;
            }
            {
                const double inv = fast_rcp(G[pr * GP + k]);
                for (int j = tid; j < l; j += CTA_THREADS) {
                    const double v = G[pr * GP + j];
                    prow[j] = v;
                    ops[k * GP + j] = v;  // kept for lambda (the column operations, replayed backwards)
                }
                for (int r = tid; r < RG; r += CTA_THREADS) colk[r] = G[r * GP + k] * inv;  // scaled column k
                if (tid == 0) {
                    isp[pr] = 1;
                    piv[k] = pr;
                    invs[k] = inv;
                }
            }
            __syncthreads();
            {
                // each thread owns one column jj and strides over the rows (pivot rows
                // keep being swept harmlessly: they are never read again)
                const int jj = tid % l, r0 = tid / l, rstep = CTA_THREADS / l;
                if (r0 < rstep) {
                    const double pj = prow[jj];
                    for (int r = r0; r < RG; r += rstep) {
                        const double cr = colk[r];
                        G[r * GP + jj] = jj == k ? cr : fma(-pj, cr, G[r * GP + jj]);
                    }
                }
            }
            __syncthreads();
        }
        // free (non-pivot) nodes in node order
        if (w == 0) {
            int base = 0;
            for (int c0 = 0; c0 < n; c0 += 32) {
                const int i = c0 + lane;
                const bool fr = i < n && !isp[i];
                const unsigned bal = __ballot_sync(FULL, fr);
                const int at = base + __popc(bal & ((1u << lane) - 1u));
                if (fr && at < M) nonpiv[at] = i;
                base += __popc(bal);
            }
            if (lane == 0) redi[CTA_WARPS] = base;
        }
        __syncthreads();
        ok = ok && redi[CTA_WARPS] == M;

        bool definite = true;
        if (ok) {
            // ---- r = f - Phi[:, piv] w1p (in place in F);  Y = Phi12 - Phi11 W^T
            for (int e = tid; e < n * nrhs; e += CTA_THREADS) {
                const int i = e / nrhs, f = e - i * nrhs;
                double r = F[e];
                for (int k = 0; k < l; ++k) r = fma(-E[i * n + piv[k]], G[(n + f) * GP + k], r);
                F[e] = r;
            }
            for (int e = tid; e < l * M; e += CTA_THREADS) {
                const int k = e / M, c = e - k * M;
                const int pk = piv[k], qc = nonpiv[c];
                double y = E[pk * n + qc];
                for (int k2 = 0; k2 < l; ++k2) y = fma(-E[pk * n + piv[k2]], G[qc * GP + k2], y);
                Y[k * M + c] = y;
            }
            __syncthreads();
            // ---- [K | b]: K = Phi22 - H W^T - W Y,  b = r_free - W r_piv
            for (int e = tid; e < M * M; e += CTA_THREADS) {
                const int c = e / M, c2 = e - c * M;
                const int qc = nonpiv[c], qc2 = nonpiv[c2];
                double v = E[qc * n + qc2];
                for (int k = 0; k < l; ++k) {
                    v = fma(-E[qc * n + piv[k]], G[qc2 * GP + k], v);
                    v = fma(-G[qc * GP + k], Y[k * M + c2], v);
                }
                K[c * KP + c2] = v;
            }
            for (int e = tid; e < M * nrhs; e += CTA_THREADS) {
                const int c = e / nrhs, f = e - c * nrhs;
                const int qc = nonpiv[c];
                double b = F[qc * nrhs + f];
                for (int k = 0; k < l; ++k) b = fma(-G[qc * GP + k], F[piv[k] * nrhs + f], b);
                K[c * KP + M + f] = b;
            }
            __syncthreads();
            // ---- pivot-free Gauss-Jordan on [K | b] (K definite)
            const double d0 = K[0];
            for (int k = 0; k < M; ++k) {
                const double dk = K[k * KP + k];
                definite = definite && dk * d0 > 0.0;
                const double inv = fast_rcp(dk);
                for (int j = tid; j < M + nrhs; j += CTA_THREADS) prow[j] = K[k * KP + j];
                for (int r = tid; r < M; r += CTA_THREADS) colk[r] = K[r * KP + k] * inv;
                __syncthreads();
                {
                    const int wk = M + nrhs - k - 1;  // columns right of the pivot
                    const int jj = k + 1 + tid % wk, r0 = tid / wk, rstep = CTA_THREADS / wk;
                    if (r0 < rstep) {
                        const double pj = prow[jj];
                        for (int r = r0; r < M; r += rstep)
                            K[r * KP + jj] = r == k ? pj * inv : fma(-pj, colk[r], K[r * KP + jj]);
                    }
                }
                __syncthreads();
            }
        }
        ok = ok && definite;

        // ---- outputs: free weights v, pivot weights w1p - W^T v; estimate
        bool bad = !ok;
        double zw = 0.0, xw[MF_MAX_FAMILIES], la[MF_MAX_FAMILIES];
        for (int f = 0; f < nf; ++f) xw[f] = la[f] = 0.0;
        if (ok) {
            for (int e = tid; e < M * nrhs; e += CTA_THREADS) {
                const int c = e / nrhs, f = e - c * nrhs;
                const double v = K[c * KP + M + f];
                if (f < nf) {
                    bad |= !isfinite(v);
                    a.out[((size_t)idx * nf + f) * n + nonpiv[c]] = v;
                    xw[f] = fmax(xw[f], fabs(v));
                } else {
                    zw = fmax(zw, fabs(v));
                }
            }
            for (int e = tid; e < l * nrhs; e += CTA_THREADS) {
                const int k = e / nrhs, f = e - k * nrhs;
                double wv = G[(n + f) * GP + k];
                for (int c = 0; c < M; ++c) wv = fma(-G[nonpiv[c] * GP + k], K[c * KP + M + f], wv);
                if (f < nf) {
                    bad |= !isfinite(wv);
                    a.out[((size_t)idx * nf + f) * n + piv[k]] = wv;
                    xw[f] = fmax(xw[f], fabs(wv));
                } else {
                    zw = fmax(zw, fabs(wv));
                }
            }
            // lambda_f = Q1^-1 (r_piv - Y v)   (family columns): Q1^-1 is the product
            // of the sweep's column operations, applied to s last step first
            for (int e = tid; e < l * nf; e += CTA_THREADS) {
                const int k = e / nf, f = e - k * nf;
                double sv = F[piv[k] * nrhs + f];
                for (int c = 0; c < M; ++c) sv = fma(-Y[k * M + c], K[c * KP + M + f], sv);
                colk[k * nf + f] = sv;
            }
            __syncthreads();
            for (int f = w; f < nf; f += CTA_WARPS) {
                for (int k = l - 1; k >= 0; --k) {
                    double part = 0.0;
                    for (int j = lane; j < l; j += 32)
                        if (j != k) part = fma(ops[k * GP + j], colk[j * nf + f], part);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
                    if (lane == 0) colk[k * nf + f] = invs[k] * (colk[k * nf + f] - part);
                    __syncwarp();
                }
                double mx = 0.0;
                for (int j = lane; j < l; j += 32) mx = fmax(mx, fabs(colk[j * nf + f]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
                la[f] = mx;
            }
        }
        bad = __syncthreads_or(bad) != 0;
        if (bad && stat == 0) stat = 1;
        zw = block_reduce_max(zw, red);
        double ratio = 0.0;
        for (int f = 0; f < nf; ++f) {
            const double xwf = block_reduce_max(xw[f], red);
            const double laf = block_reduce_max(la[f], red);
            ratio = fmax(ratio, fmax(xwf, laf) / xwf);
        }
        if (tid == 0) {
            const double est = anorm * zw * ratio;
            const bool close = r2min < a.min_sep2 * rc2max;
            if (stat != 0 || close || !(est <= a.hybrid_thresh)) {
                const unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                a.flag_list[slot] = idx;
            }
            a.status[idx] = 0;  // failures are re-derived in reference order by the re-solve
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------------------
// Nullspace pass for one large stencil shape with compile-time sizes (the C5
// shape: n = 70, degree 4 in 3D, 35 monomials, four families), same mathematics
// as phs_ns_cta with the data held where the work is:
//   * the Gauss-Jordan sweep over [Q; g] keeps every element in a register of
//     the thread that owns its column (rows strided over the row groups); per
//     step only the pivot row and the pivot column go through shared memory
//     (double-buffered: two barriers per step, no read-modify-write of the
//     matrix in shared memory);
//   * Y = Phi12 - Phi11 W^T and [K | b] = [Phi22 | f] - [H W][W^T w1p; Y r_piv]
//     are tensor-core products (mma.sync.m8n8k4.f64), 8 x 8 tiles spread over
//     the warps, the particular solution's residuals riding as extra columns;
//   * the pivot-free Gauss-Jordan on [K | b] is register-resident the same way.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cta_cp_async4(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cta_cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cta_cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cta_cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// barrier over the first `count` threads of the block (ids 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// a warp's share of a tile grid: NA row tiles x NB column tiles, bit ia * NB + ib of
// MASK set for the tiles it owns
template <int NA, int NB, unsigned MASK>
struct TileRole {
    static constexpr int na = NA, nb = NB;
    static constexpr unsigned mask = MASK;
};

template <int NN, int DD, int DEG, int NF>
struct Cta2Cfg {
    static constexpr int LL = binom(DEG + DD, DD);
    static constexpr int M = NN - LL;
    static constexpr int NR = NF + 1;        // families + probe
    static constexpr int MR = M + NR;        // columns of [K | b]
    static constexpr int RG = NN + NR;       // rows of [Q; g]
    // Phi pitch, even: the pair walk stores E[i][i + q] and its mirror from lane pairs
    // i = pp, pp + 1, ..: the lane stride is EP + 1 doubles, which must be odd for the
    // 16 pairs of a warp to hit distinct banks (EP = 71 put them on two)
    static constexpr int EP = (NN + 1) & ~1;
    static constexpr int GP = LL | 1;        // [Q; g] pitch
    static constexpr int WP = ((LL + 3) / 8) * 8 + 4;  // pitch of the swept rows (W, particular solutions), 4 mod 8
    static constexpr int YP = ((LL + 3) / 8) * 8 + 4;  // Y column pitch, 4 mod 8 (conflict-free fragments)
    static constexpr int KP = MR | 1;
    // sweeps with rows in lanes: a lane pair per row, one column half each
    static constexpr int QH = (LL + 1) / 2;              // [Q; g] columns per lane (halves)
    static constexpr int QWARPS = (RG + 15) / 16;        // warps of the [Q; g] sweep
    static constexpr int KH = (MR + 1) / 2;              // [K | b] columns per lane (interleaved)
    static constexpr int KWARPS = (MR + 15) / 16;        // warps of the [K | b] elimination
    static constexpr int UPB = 2 * MR + 2;               // block slot: column pairs, 1 / det
    static constexpr int RT = (LL + 7) / 8, CT = (MR + 7) / 8, MT = (M + 7) / 8;
    // shared layout (doubles)
    static constexpr int LOC = 0;
    // Phi in full (both triangles, node order): two stencils per SM (the register
    // budget's limit) fit in shared memory; [K | b] and the elimination's pivot
    // rows reuse the region once Phi is consumed
    static constexpr int EFULL = NN * EP;
    static constexpr int E = LOC + ((NN * DD + 1) & ~1);
    static constexpr int G = E + ((EFULL + 1) & ~1);
    static constexpr int F = G + ((RG * GP + 1) & ~1);
    static constexpr int Y = F + NN * NR;
    static constexpr int K = E;
    static constexpr int OPS = Y + ((MR * YP + 1) & ~1);  // pivot rows per step, then 1 / pivot
    static constexpr int V = OPS + ((LL * GP + LL + 1) & ~1);
    static constexpr int PROW = V + M * NR;              // 2 x 64
    static constexpr int COLK = PROW + 128;              // 2 x 80
    static constexpr int RED = COLK + 160;               // reductions / candidates
    static constexpr int INTS = RED + 4 * CTA_WARPS + 16;  // isp[NN], piv[LL], nonpiv[M] (ints)
    static constexpr int AUX = INTS + (NN + LL + M + 16) / 2 + 2;  // partial maxima, flags, pivot keys
    static constexpr int AXP = 8 + QWARPS + 1;           // aux slots of the published prologue scalars (2)
    static constexpr int SIDX = AUX + AXP + 2;            // staged next-stencil indices (ints), row
    static constexpr int SROW = 2 * ((NN + 1) / 2);       // int offset of the row (8-byte aligned)
    static constexpr int SPOS = SIDX + SROW / 2 + 1;      // staged next-stencil positions, centre
    static constexpr int TOTAL = SPOS + NN * DD + DD + 1;
    static_assert(NN * DD + DD <= CTA_THREADS, "one staged position per thread");
    static_assert(QWARPS < CTA_WARPS && CTA_WARPS - QWARPS <= 3 && KWARPS <= CTA_WARPS, "sweep layouts");
    static_assert(NN % 2 == 0 && NN < 128, "Phi row pairing / pivot keys");
    static_assert((M / 2 + 1) * UPB <= EFULL && UPB % 2 == 0, "block slots fit the Phi region");
    static_assert(MR <= 64 && RG <= 80 && M <= 80, "pivot buffers");
    static_assert(M * KP <= EFULL, "[K | b] fits the Phi region");
};

template <int NN, int DD, int DEG, int NF>
__global__ void __launch_bounds__(CTA_THREADS, 2) phs_ns_cta2(PhsArgs a) {
    using C = Cta2Cfg<NN, DD, DEG, NF>;
    constexpr int LL = C::LL, M = C::M, NR = C::NR, MR = C::MR, RG = C::RG, GP = C::GP, YP = C::YP,
                  KP = C::KP, EP = C::EP, WP = C::WP;
    static_assert(MR * WP <= RG * GP, "the swept rows fit the [Q; g] region");
    extern __shared__ __align__(16) double sm2[];
    double* loc = sm2 + C::LOC;
    double* E = sm2 + C::E;
    double* G = sm2 + C::G;
    double* F = sm2 + C::F;
    double* Y = sm2 + C::Y;
    double* K = sm2 + C::K;
    double* ops = sm2 + C::OPS;
    double* invs = ops + LL * GP;
    double* V = sm2 + C::V;
    double* prow = sm2 + C::PROW;
    double* colk = sm2 + C::COLK;
    double* red = sm2 + C::RED;
    int* redi = reinterpret_cast<int*>(red + 2 * CTA_WARPS);
    int* isp = reinterpret_cast<int*>(sm2 + C::INTS);
    int* piv = isp + NN;
    int* nonpiv = piv + LL;
    double* aux = sm2 + C::AUX;
#ifdef MF_CTA_TIMING
    long long ts_[12] = {};
#define MF_TS(i) if (tid == 0) ts_[i] = clock64()
#else
#define MF_TS(i)
#endif
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    const PhsParams& P = a.P;

    // The next stencil's node positions are staged by cp.async while the current
    // one is solved: its node indices (and row) right after the coordinates are
    // read, its positions once the sweep has joined (two dependent global loads
    // off the chain)
    int* sidx = reinterpret_cast<int*>(sm2 + C::SIDX);  // NN node indices, then the row (int64)
    double* spos = sm2 + C::SPOS;                        // NN * DD positions, then the centre
    auto stage_idx = [&](int64_t id) {
        if (id < a.m) {
            if (tid < NN) cta_cp_async4(sidx + tid, a.stencils + id * NN + tid);
            else if (tid == NN) cta_cp_async8(sidx + C::SROW, a.rows + id);
        }
        cta_cp_async_commit();
    };
    auto stage_pos = [&](int64_t id) {
        if (id < a.m) {
            if (tid < NN * DD) {
                const int j = tid / DD, ax = tid - j * DD;
                cta_cp_async8(spos + tid, a.pos + (int64_t)sidx[j] * DD + ax);
            } else if (tid < NN * DD + DD) {
                const int64_t rw = *reinterpret_cast<const int64_t*>(sidx + C::SROW);
                cta_cp_async8(spos + tid, a.pos + rw * DD + (tid - NN * DD));
            }
        }
        cta_cp_async_commit();
    };
    // Prologue of one stencil, run by warps 4..7 (threads pt = tid - 128) while warps 0..3
    // finish the previous stencil's multipliers: thread pt < NN owns node pt from the staged
    // position to its row of [Q; g] and its right-hand sides (no shared-memory round trip
    // of the coordinates in between); one fused reduction over the four warps gives the
    // scale and the radius.  Publishes stat and (radius / scale)^2 in aux[AXP..AXP + 1].
    constexpr int PW0 = CTA_WARPS / 2, PTH = (CTA_WARPS - PW0) * 32;
    static_assert(NN <= PTH - 32, "node threads and one helper warp");
    auto prologue = [&](int64_t idx) {
        const int pt = tid - PW0 * 32, pw = w - PW0;
        const bool mine = pt < NN;
        double xr[DD], r2 = 0.0;
#pragma unroll
        for (int ax = 0; ax < DD; ++ax) {
            xr[ax] = mine ? spos[pt * DD + ax] - spos[NN * DD + ax] : 0.0;
            r2 = __dadd_rn(r2, __dmul_rn(xr[ax], xr[ax]));
        }
        int stat = 0;
        double sc = 1.0, r2max;
        {
            // max r^2 (radius; the support scale) and min positive r^2 (nearest scale)
            double vmax = mine ? r2 : 0.0, vmin = (mine && r2 > 0.0) ? r2 : INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                vmax = fmax(vmax, __shfl_xor_sync(FULL, vmax, o));
                vmin = fmin(vmin, __shfl_xor_sync(FULL, vmin, o));
            }
            if (lane == 0) {
                red[pw] = vmax;
                red[CTA_WARPS + pw] = vmin;
            }
            named_bar(3, PTH);
            r2max = red[0];
            double r2min_pos = red[CTA_WARPS];
#pragma unroll
            for (int k = 1; k < CTA_WARPS - PW0; ++k) {
                r2max = fmax(r2max, red[k]);
                r2min_pos = fmin(r2min_pos, red[CTA_WARPS + k]);
            }
            if (P.scale_code == MF_SCALE_SUPPORT) {
                if (r2max > 0.0) sc = __dsqrt_rn(r2max);
                else stat = 2;
            } else if (P.scale_code == MF_SCALE_NEAREST) {
                if (r2min_pos < INFINITY) sc = __dsqrt_rn(r2min_pos);
                else stat = 2;
            }
        }
        const double rs = fast_rcp(sc);
        double facs[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int o = P.orders[f];
            facs[f] = o == 0 ? 1.0 : (o == 1 ? rs : rs * rs);
        }
        if (pt == 0) {
            aux[C::AXP] = (double)stat;
            aux[C::AXP + 1] = r2max * rs * rs;
        }
        if (mine) {
            double x[DD], q[LL];
#pragma unroll
            for (int ax = 0; ax < DD; ++ax) {
                x[ax] = xr[ax] * rs;
                loc[pt * DD + ax] = x[ax];
            }
            monomials_reg<DD, DEG, 0, LL>(q, x);
#pragma unroll
            for (int m = 0; m < LL; ++m) G[pt * GP + m] = q[m];
            // k = 3 right-hand sides with a refined reciprocal root (no IEEE sqrt / divide)
            double rr2 = x[0] * x[0];
#pragma unroll
            for (int ax = 1; ax < DD; ++ax) rr2 = fma(x[ax], x[ax], rr2);
            const double rsq = rr2 > 0.0 ? fast_rsqrt(rr2) : 0.0;
            const double r = rr2 * rsq, ir2 = rsq * rsq;
            const double d1r = 3.0 * r, d2v = 6.0 * r;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int kind = P.kinds[f];
                double t;
                if (kind == MF_KIND_IDENTITY) {
                    t = rr2 * r;
                } else if (kind == MF_KIND_D1) {
                    t = -d1r * x[P.ax_a[f]];
                } else if (kind == MF_KIND_D2) {
                    const double ee = x[P.ax_a[f]] * x[P.ax_b[f]] * ir2;
                    const double delta = P.ax_a[f] == P.ax_b[f] ? 1.0 : 0.0;
                    t = fma(d2v, ee, d1r * (delta - ee));
                } else {
                    t = fma((double)(DD - 1), d1r, d2v);
                }
                F[pt * NR + f] = t * facs[f];
            }
            F[pt * NR + NF] = probe_sign(idx, pt);
        } else if (pt >= PTH - 32) {
            // the last warp: constraint right-hand sides, pivot marks
            for (int e = pt - (PTH - 32); e < NR * LL; e += 32) {
                const int f = e / LL, m = e - f * LL;
                G[(NN + f) * GP + m] = f < NF ? P.base_bot[f * MF_MAX_MONOMIALS + m] * facs[f] : probe_sign(idx, NN + m);
            }
            for (int i = pt - (PTH - 32); i < NN; i += 32) isp[i] = 0;
        }
    };

    stage_idx(blockIdx.x);
    cta_cp_async_wait_all();
    __syncthreads();
    stage_pos(blockIdx.x);
    cta_cp_async_wait_all();
    __syncthreads();  // the first stencil's positions are visible
    stage_idx((int64_t)blockIdx.x + gridDim.x);
    if (w >= PW0 && blockIdx.x < a.m) prologue(blockIdx.x);
    __syncthreads();  // [Q; g], the right-hand sides and the coordinates are published

    for (int64_t idx = blockIdx.x; idx < a.m; idx += gridDim.x) {
        MF_TS(0);
        MF_TS(1);
        int stat = (int)aux[C::AXP];
        const double rc2max = aux[C::AXP + 1];
        unsigned* qkw = reinterpret_cast<unsigned*>(aux + 8);  // [2][QWARPS] pivot keys
        MF_TS(2);

        bool ok = stat == 0;
        // the sweep's row registers stay live until G is written back after the join
        double gq[C::QH];
        const int qr = w * 16 + (lane >> 1), qh = lane & 1;  // row, column half (sweep warps)
        if (w < C::QWARPS) {
            // ---- Gauss-Jordan column sweep of [Q; g] with node pivoting, rows in lanes:
            //      lane pair (2 r, 2 r + 1) of the first QWARPS warps owns row r, one
            //      column half each.  Per step the pivot row (two threads) goes through
            //      shared memory and every lane folds it into its own row: one broadcast
            //      load and one FMA per element, the column-k factor from the partner
            //      lane by one shuffle.  Pivot search: one 32-bit key per candidate row
            //      (float bits of |v|, low 7 bits = 127 - row), warp REDUX into a per-warp
            //      slot (double-buffered), every thread merges the QWARPS slots; column
            //      k+1 is updated first so its keys and the reciprocals of the candidate
            //      pivots leave early (the winner publishes its own: no reciprocal on
            //      the step's chain).  Two barriers per step over the sweep warps only
            //      (publishing every warp's candidate row to save one measured slower).
            const bool qrow = qr < RG;
#pragma unroll
            for (int j = 0; j < C::QH; ++j) {
                const int c = qh * C::QH + j;
                gq[j] = (qrow && c < LL) ? G[qr * GP + c] : 0.0;
            }
            auto key_of = [](double v, int r) -> unsigned {
                const float f = __double2float_ru(fabs(v));
                return (__float_as_uint(f) & ~127u) | (unsigned)(127 - r);
            };
            bool isp_row = false;
            double myinv = fast_rcp(gq[0]);
            {
                const unsigned kb = (ok && qh == 0 && qr < NN) ? key_of(gq[0], qr) : 0u;
                const unsigned km = __reduce_max_sync(FULL, kb);
                if (lane == 0) qkw[w] = km;
            }
#pragma unroll
            for (int k = 0; k < LL; ++k) {
                constexpr int QH = C::QH;
                const int hk = k / QH, kk = k - hk * QH;
                named_bar(1, C::QWARPS * 32);  // keys of column k complete
                if (!ok) break;
                unsigned key = qkw[(k & 1) * C::QWARPS];
#pragma unroll
                for (int q = 1; q < C::QWARPS; ++q) key = max(key, qkw[(k & 1) * C::QWARPS + q]);
                const int pr = 127 - (int)(key & 127u);
                const float best = __uint_as_float(key & ~127u);
                if (key == 0u || !(best > 0.0f) || !isfinite(best) || pr >= NN) {
                    ok = false;  // uniform: every thread read the same key
                    break;
                }
                if (tid == 0) {
                    isp[pr] = 1;
                    piv[k] = pr;
                }
                if (qr == pr) {
                    // the raw pivot row (kept for the lambda back substitution) and 1 / pivot
#pragma unroll
                    for (int j = 0; j < QH; ++j)
                        if (qh == 0 || j < LL - QH) ops[k * GP + qh * QH + j] = gq[j];
                    if (qh == hk) invs[k] = myinv;
                    isp_row = true;
                }
                named_bar(1, C::QWARPS * 32);  // pivot row and 1 / pivot published
                const double inv = invs[k];
                const double tk = __shfl_sync(FULL, gq[kk], (lane & ~1) | hk);
                const double s = tk * inv;
                const double* prw = ops + k * GP + qh * QH;
                if (k + 1 < LL) {
                    // column k + 1 first: its pivot keys and reciprocals
                    const int h1 = (k + 1) / QH, k1 = (k + 1) - h1 * QH;
                    if (qh == h1) gq[k1] = fma(-s, prw[k1], gq[k1]);
                    const unsigned kb = (qh == h1 && qr < NN && !isp_row) ? key_of(gq[k1], qr) : 0u;
                    const unsigned km = __reduce_max_sync(FULL, kb);
                    if (lane == 0) qkw[((k + 1) & 1) * C::QWARPS + w] = km;
                    myinv = fast_rcp(gq[k1]);
                }
#pragma unroll
                for (int j = 0; j < QH; ++j) {
                    const int h1 = (k + 1) / QH, k1 = (k + 1) - h1 * QH;
                    if (k + 1 < LL && j == k1) {
                        if (qh != h1) gq[j] = fma(-s, prw[j], gq[j]);
                    } else if (j == kk) {
                        gq[j] = qh == hk ? s : fma(-s, prw[j], gq[j]);
                    } else {
                        gq[j] = fma(-s, prw[j], gq[j]);
                    }
                }
            }
            if (tid == 0) aux[6] = ok ? 1.0 : 0.0;
        } else {
            // ---- Phi (both triangles, zero diagonal) and ||A||_inf while the
            //      sweep runs: rows i and NN-1-i pair up to NN+1 entries, split in two
            const int pt = tid - C::QWARPS * 32;
            constexpr int PT = (CTA_WARPS - C::QWARPS) * 32;
            constexpr int UNIT = (NN + 1 + 1) / 2;
            double r2min = INFINITY;
            for (int u = pt; u < NN; u += PT) {  // NN/2 row pairs x 2 halves
                const int pp = u >> 1, half = u & 1;
                const int q0 = half * UNIT, q1 = half ? NN + 1 : UNIT;
                for (int q = q0; q < q1; ++q) {
                    const bool first = q < NN - pp;
                    const int i = first ? pp : NN - 1 - pp;
                    const int j = first ? pp + q : i + (q - (NN - pp));
                    double v = 0.0;
                    if (j > i) {
                        double df = loc[i * DD] - loc[j * DD];
                        double r2 = df * df;
#pragma unroll
                        for (int ax = 1; ax < DD; ++ax) {
                            df = loc[i * DD + ax] - loc[j * DD + ax];
                            r2 = fma(df, df, r2);
                        }
                        r2min = r2 < r2min ? r2 : r2min;
                        v = r2 * (r2 * fast_rsqrt(fmax(r2, 1e-300)));
                    }
                    E[i * EP + j] = v;
                    E[j * EP + i] = v;
                }
            }
            named_bar(2, PT);
            double an = 0.0;
            for (int r = pt; r < NN + LL; r += PT) {
                double acc = 0.0;
                if (r < NN) {
                    for (int j = 0; j < NN; ++j) acc += E[j * EP + r];  // r^3 >= 0; column r == row r, lanes adjacent
                    for (int m = 0; m < LL; ++m) acc += fabs(G[r * GP + m]);
                } else {
                    for (int i = 0; i < NN; ++i) acc += fabs(G[i * GP + (r - NN)]);
                }
                an = fmax(an, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                an = fmax(an, __shfl_xor_sync(FULL, an, o));
                r2min = fmin(r2min, __shfl_xor_sync(FULL, r2min, o));
            }
            if (lane == 0) {
                aux[w - C::QWARPS] = r2min;
                aux[3 + w - C::QWARPS] = an;
            }
        }
        cta_cp_async_wait_all();  // the next stencil's indices
        __syncthreads();  // join: sweep done, Phi and the estimates' inputs ready
        stage_pos(idx + gridDim.x);
        MF_TS(3);
        ok = aux[6] != 0.0;
        double r2min = aux[0], anorm = aux[3];
#pragma unroll
        for (int q = 1; q < CTA_WARPS - C::QWARPS; ++q) {
            r2min = fmin(r2min, aux[q]);
            anorm = fmax(anorm, aux[3 + q]);
        }
        // free (non-pivot) nodes in node order; isp[i] becomes the free index of node
        // i (-1 for the pivots)
        if (ok && w == 0) {
            int base = 0;
            for (int c0 = 0; c0 < NN; c0 += 32) {
                const int i = c0 + lane;
                const bool fr = i < NN && !isp[i];
                const unsigned bal = __ballot_sync(FULL, fr);
                const int at = base + __popc(bal & ((1u << lane) - 1u));
                if (fr && at < M) nonpiv[at] = i;
                if (i < NN) isp[i] = (fr && at < M) ? at : -1;
                base += __popc(bal);
            }
            if (lane == 0) redi[CTA_WARPS] = base;
        }
        __syncthreads();
        ok = ok && redi[CTA_WARPS] == M;
        // the swept rows leave the registers in the order the products read them:
        // W row c (free index) at c * WP, the particular solutions at (M + f) * WP;
        // pitch 4 mod 8, so the tensor-core fragment loads (8 rows x 4 columns) hit
        // distinct banks (the node-order rows behind a gather collided)
        if (ok && w < C::QWARPS && qr < RG) {
            const int row = qr < NN ? isp[qr] : M + (qr - NN);
            if (row >= 0) {
#pragma unroll
                for (int j = 0; j < C::QH; ++j) {
                    const int c = qh * C::QH + j;
                    if (c < LL) G[row * WP + c] = gq[j];
                }
            }
        }
        __syncthreads();

        bool definite = true;
        if (ok) {
            // ---- Y (l x [M | NR]) on the tensor cores, then [K | b]: 8 x 8 tiles spread
            //      over the warps, each warp's tiles advanced together (k-step outer,
            //      tiles inner: independent accumulator chains); the row and column
            //      offsets of every fragment are resolved once per tile
            MF_TS(4);
            // Tile ownership: the 5 x 5 tile grid is cut into four 2 x 2 blocks (warps
            // 0..3), a row strip, a corner and a column strip (warps 4..6), so a warp's
            // tiles share their operand fragments: 4 fragment loads per k-step feed 4
            // (3) tensor-core products instead of 8 loads for 4 scattered tiles
            static_assert(C::RT == 5 && C::CT == 5 && C::MT == 5 && CTA_WARPS == 8, "tile ownership below");
            // Y = Phi12 - Phi11 [W^T | w1p]
            auto y_tiles = [&](auto role, const int* at, const int* bt) {
                constexpr int NA = decltype(role)::na, NB = decltype(role)::nb;
                constexpr unsigned MASK = decltype(role)::mask;
                double acc[NA][NB][2];
                int arow[NA], brow[NB], pka[NA];
#pragma unroll
                for (int ia = 0; ia < NA; ++ia) {
                    const int kr = at[ia] * 8 + g8;
                    pka[ia] = piv[kr < LL ? kr : 0];
                    arow[ia] = kr < LL ? pka[ia] * EP : -1;
                }
#pragma unroll
                for (int ib = 0; ib < NB; ++ib) {
                    const int cb = bt[ib] * 8 + g8;
                    brow[ib] = cb < MR ? cb * WP : -1;
                }
#pragma unroll
                for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) {
                        if (!((MASK >> (ia * NB + ib)) & 1u)) continue;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c = bt[ib] * 8 + 2 * t4 + h;
                            double v = 0.0;
                            if (arow[ia] >= 0 && c < M) v = E[arow[ia] + nonpiv[c]];
                            else if (arow[ia] >= 0 && c < MR) v = F[pka[ia] * NR + (c - M)];
                            acc[ia][ib][h] = v;
                        }
                    }
#pragma unroll
                for (int ks = 0; ks < (LL + 3) / 4; ++ks) {
                    const int k2 = ks * 4 + t4;
                    const bool kin = k2 < LL;
                    const int pv = piv[kin ? k2 : 0];
                    double av[NA], bv[NB];
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia) av[ia] = (kin && arow[ia] >= 0) ? -E[arow[ia] + pv] : 0.0;
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) bv[ib] = (kin && brow[ib] >= 0) ? G[brow[ib] + k2] : 0.0;
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                        for (int ib = 0; ib < NB; ++ib)
                            if ((MASK >> (ia * NB + ib)) & 1u) dmma_f64(acc[ia][ib][0], acc[ia][ib][1], av[ia], bv[ib]);
                }
#pragma unroll
                for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) {
                        if (!((MASK >> (ia * NB + ib)) & 1u)) continue;
                        const int kr = at[ia] * 8 + g8;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c = bt[ib] * 8 + 2 * t4 + h;
                            if (kr < LL && c < MR) Y[c * YP + kr] = acc[ia][ib][h];
                        }
                    }
            };
            // [K | b] = [Phi22 | f] - H [W^T | w1p] - W [Y | r_piv]; the accumulators
            // cross the barrier after which [K | b] takes Phi's place
            auto k_tiles = [&](auto role, const int* at, const int* bt) {
                constexpr int NA = decltype(role)::na, NB = decltype(role)::nb;
                constexpr unsigned MASK = decltype(role)::mask;
                double acc[NA][NB][2];
                int arE[NA], arW[NA], brW[NB], brY[NB], qca[NA];
#pragma unroll
                for (int ia = 0; ia < NA; ++ia) {
                    const int c = at[ia] * 8 + g8;
                    qca[ia] = nonpiv[c < M ? c : 0];
                    arE[ia] = c < M ? qca[ia] * EP : -1;
                    arW[ia] = c < M ? c * WP : -1;
                }
#pragma unroll
                for (int ib = 0; ib < NB; ++ib) {
                    const int cb = bt[ib] * 8 + g8;
                    brW[ib] = cb < MR ? cb * WP : -1;
                    brY[ib] = cb < MR ? cb * YP : -1;
                }
#pragma unroll
                for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) {
                        if (!((MASK >> (ia * NB + ib)) & 1u)) continue;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c2 = bt[ib] * 8 + 2 * t4 + h;
                            double v = 0.0;
                            if (arE[ia] >= 0 && c2 < M) v = E[arE[ia] + nonpiv[c2]];
                            else if (arE[ia] >= 0 && c2 < MR) v = F[qca[ia] * NR + (c2 - M)];
                            acc[ia][ib][h] = v;
                        }
                    }
#pragma unroll
                for (int ks = 0; ks < (LL + 3) / 4; ++ks) {
                    const int kk = ks * 4 + t4;
                    const bool kin = kk < LL;
                    const int pv = piv[kin ? kk : 0];
                    double av[NA], bv[NB];
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia) av[ia] = (kin && arE[ia] >= 0) ? -E[arE[ia] + pv] : 0.0;
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) bv[ib] = (kin && brW[ib] >= 0) ? G[brW[ib] + kk] : 0.0;
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                        for (int ib = 0; ib < NB; ++ib)
                            if ((MASK >> (ia * NB + ib)) & 1u) dmma_f64(acc[ia][ib][0], acc[ia][ib][1], av[ia], bv[ib]);
                }
#pragma unroll
                for (int ks = 0; ks < (LL + 3) / 4; ++ks) {
                    const int kw = ks * 4 + t4;
                    const bool kin = kw < LL;
                    double av[NA], bv[NB];
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia) av[ia] = (kin && arW[ia] >= 0) ? -G[arW[ia] + kw] : 0.0;
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) bv[ib] = (kin && brY[ib] >= 0) ? Y[brY[ib] + kw] : 0.0;
#pragma unroll
                    for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                        for (int ib = 0; ib < NB; ++ib)
                            if ((MASK >> (ia * NB + ib)) & 1u) dmma_f64(acc[ia][ib][0], acc[ia][ib][1], av[ia], bv[ib]);
                }
                __syncthreads();  // Phi is consumed: [K | b] takes its place
#pragma unroll
                for (int ia = 0; ia < NA; ++ia)
#pragma unroll
                    for (int ib = 0; ib < NB; ++ib) {
                        if (!((MASK >> (ia * NB + ib)) & 1u)) continue;
                        const int c = at[ia] * 8 + g8;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c2 = bt[ib] * 8 + 2 * t4 + h;
                            if (c < M && c2 < MR) K[c * KP + c2] = acc[ia][ib][h];
                        }
                    }
            };
            // (warp-uniform dispatch: every warp runs exactly one role per product)
            auto for_role = [&](auto&& fn) {
                if (w < 4) {
                    const int at[2] = {2 * (w >> 1), 2 * (w >> 1) + 1}, bt[2] = {2 * (w & 1), 2 * (w & 1) + 1};
                    fn(TileRole<2, 2, 0xFu>{}, at, bt);
                } else if (w == 4) {
                    const int at[1] = {4}, bt[3] = {0, 1, 2};
                    fn(TileRole<1, 3, 0x7u>{}, at, bt);
                } else if (w == 5) {
                    const int at[2] = {4, 3}, bt[2] = {3, 4};  // (4,3) (4,4) (3,4)
                    fn(TileRole<2, 2, 0xBu>{}, at, bt);
                } else if (w == 6) {
                    const int at[3] = {0, 1, 2}, bt[1] = {4};
                    fn(TileRole<3, 1, 0x7u>{}, at, bt);
                } else {
                    fn(TileRole<1, 1, 0x0u>{}, nullptr, nullptr);
                }
            };
            for_role(y_tiles);
            __syncthreads();
            MF_TS(5);
            for_role(k_tiles);
            __syncthreads();
            // ---- pivot-free block Gauss-Jordan on [K | b] with 2 x 2 pivots, rows in
            //      lanes: lane pair (2 c, 2 c + 1) of the first KWARPS warps owns row c,
            //      columns interleaved (col = 2 j + half), so both columns of block p sit
            //      at register j = p of the pair.  Rows M .. M+NR-1 carry b^T: the two
            //      block columns of the symmetric [K b; b^T .] -- stored by every lane in
            //      ONE instruction, pairs adjacent -- are the two pivot rows including
            //      b; each row reads a pivot-row pair with one 16-byte load.  The block's
            //      lane quad forms 1 / det of the next block as soon as its entries are
            //      final (off the chain).  One barrier per TWO columns (each block has
            //      its own slot in the free Phi region) over the elimination warps.
            if (w < C::KWARPS) {
                constexpr int KH = C::KH, NB = M / 2, UB = C::UPB;
                const int kc = w * 16 + (lane >> 1), kh = lane & 1;
                double kv[KH];
#pragma unroll
                for (int j = 0; j < KH; ++j) {
                    const int col = 2 * j + kh;
                    double v = 0.0;
                    if (kc < M && col < MR) v = K[kc * KP + col];
                    else if (kc < MR && col < M) v = K[col * KP + kc];  // b^T rows
                    kv[j] = v;
                }
                named_bar(1, C::KWARPS * 32);  // [K | b] read: the slots may overwrite it
                MF_TS(6);
                double* U = K;  // block p's two columns at p * UB (pairs), 1 / det at p * UB + 2 MR
                // 1 / det of the 2 x 2 block whose entries sit at register j in this quad
                auto quad_rdet = [&](int j) {
                    const int base = lane & ~3;
                    const double d00 = __shfl_sync(FULL, kv[j], base), d01 = __shfl_sync(FULL, kv[j], base + 1);
                    const double d10 = __shfl_sync(FULL, kv[j], base + 2), d11 = __shfl_sync(FULL, kv[j], base + 3);
                    return fast_rcp(fma(d00, d11, -d01 * d10));
                };
                double rdet = NB > 0 ? quad_rdet(0) : 0.0;
                bool def = true;
                double s0 = 0.0;
#pragma unroll
                for (int p = 0; p < NB; ++p) {
                    const int k0 = 2 * p, k1 = 2 * p + 1;
                    double* Up = U + p * UB;
                    const double own = kv[p], oth = __shfl_xor_sync(FULL, kv[p], 1);
                    if (kc < MR) Up[2 * kc + kh] = own;
                    if (kc == k0 && kh == 0) Up[2 * MR] = rdet;
                    named_bar(1, C::KWARPS * 32);
                    const double2 r0 = *reinterpret_cast<const double2*>(Up + 2 * k0);  // D00 D01
                    const double2 r1 = *reinterpret_cast<const double2*>(Up + 2 * k1);  // D10 D11
                    const double rd = Up[2 * MR];
                    if (p == 0) s0 = r0.x;
                    def = def && r0.x * s0 > 0.0 && rd > 0.0;
                    const double t0 = kh == 0 ? own : oth, t1 = kh == 0 ? oth : own;  // K(c, k0), K(c, k1)
                    const bool piv_row = kc == k0 || kc == k1;
                    const double fa = piv_row ? 0.0 : rd * fma(t0, r1.y, -t1 * r1.x);
                    const double fb = piv_row ? 0.0 : rd * fma(t1, r0.x, -t0 * r0.y);
                    // the next block's columns first, then its 1 / det
                    if (p + 1 < KH) {
                        const int col = 2 * (p + 1) + kh;
                        if (col < MR) {
                            const double2 u = *reinterpret_cast<const double2*>(Up + 2 * col);
                            kv[p + 1] = fma(-fa, u.x, fma(-fb, u.y, kv[p + 1]));
                        }
                        if (p + 1 < NB) rdet = quad_rdet(p + 1);
                    }
#pragma unroll
                    for (int j = p + 2; j < KH; ++j) {
                        const int col = 2 * j + kh;
                        if (col < MR) {
                            const double2 u = *reinterpret_cast<const double2*>(Up + 2 * col);
                            kv[j] = fma(-fa, u.x, fma(-fb, u.y, kv[j]));
                        }
                    }
                }
                double rlast = 0.0;
                if constexpr (M % 2 == 1) {
                    // the last column alone: 1 / d from its owner, one more barrier
                    constexpr int kl = M - 1, jl = kl / 2;
                    double* Ul = U + NB * UB;
                    const double rn = fast_rcp(kv[jl]);
                    if (kc < MR && kh == 0) Ul[kc] = kc == kl ? rn : kv[jl];
                    named_bar(1, C::KWARPS * 32);
                    rlast = Ul[kl];
                    def = def && (NB == 0 || rlast * s0 > 0.0);
                    const double tk = __shfl_sync(FULL, kv[jl], lane & ~1);
                    const double fac = kc != kl ? tk * rlast : 0.0;
#pragma unroll
                    for (int j = jl; j < KH; ++j) {
                        const int col = 2 * j + kh;
                        if (col > kl && col < MR) kv[j] = fma(-fac, Ul[col], kv[j]);
                    }
                }
                // the solution columns: 2 x 2 block solves (the partner row sits two
                // lanes away), the odd last row by its reciprocal
#pragma unroll
                for (int j = 0; j < KH; ++j) {
                    const int col = 2 * j + kh;
                    if (2 * j + 1 < M) continue;  // (compile-time: only the b columns)
                    const double ob = __shfl_xor_sync(FULL, kv[j], 2);
                    if (kc < M && col >= M && col < MR) {
                        double x;
                        if (kc < 2 * NB) {
                            const int p = kc >> 1;
                            const double* Up = U + p * UB;
                            const double2 r0 = *reinterpret_cast<const double2*>(Up + 4 * p);
                            const double2 r1 = *reinterpret_cast<const double2*>(Up + 4 * p + 2);
                            const double rd = Up[2 * MR];
                            x = (kc & 1) == 0 ? rd * fma(r1.y, kv[j], -r0.y * ob) : rd * fma(r0.x, kv[j], -r1.x * ob);
                        } else {
                            x = kv[j] * rlast;
                        }
                        V[kc * NR + (col - M)] = x;
                    }
                }
                if (tid == 0) aux[7] = def ? 1.0 : 0.0;
            }
            __syncthreads();
            definite = aux[7] != 0.0;
        }
        ok = ok && definite;

        // ---- outputs: free weights v, pivot weights w1p - W^T v; estimate
        MF_TS(7);
        bool bad = !ok;
        double zw = 0.0, xw[NF], la[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) xw[f] = la[f] = 0.0;
        if (ok) {
            for (int e = tid; e < M * NR; e += CTA_THREADS) {
                const int c = e / NR, f = e - c * NR;
                const double v = V[e];
                if (f < NF) {
                    bad |= !isfinite(v);
                    a.out[((size_t)idx * NF + f) * NN + nonpiv[c]] = v;
                    xw[f] = fmax(xw[f], fabs(v));
                } else {
                    zw = fmax(zw, fabs(v));
                }
            }
            // pivot weights w1p - W^T v (rows k < LL) and the multipliers' right-hand
            // side r_piv - Y v (rows LL + k) as one tensor-core product over the free
            // columns c: A(r, c) = W(c, r) | Y(c, r - LL), B(c, f) = v(c, f)
            {
                constexpr int R2 = (2 * LL + 7) / 8, TPW = (R2 + CTA_WARPS - 1) / CTA_WARPS;
                double acc[TPW][2];
#pragma unroll
                for (int ti = 0; ti < TPW; ++ti) acc[ti][0] = acc[ti][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < (M + 3) / 4; ++ks) {
                    const int c = ks * 4 + t4;
                    const bool cin = c < M;
                    const int cr = cin ? c : 0;
                    const int wrow = cr * WP;
                    const double bv = (cin && g8 < NR) ? V[cr * NR + (g8 < NR ? g8 : 0)] : 0.0;
#pragma unroll
                    for (int ti = 0; ti < TPW; ++ti) {
                        const int rt = w + ti * CTA_WARPS;
                        if (rt >= R2) continue;  // warp-uniform
                        const int r = rt * 8 + g8;
                        double av = 0.0;
                        if (cin && r < 2 * LL) av = r < LL ? G[wrow + r] : Y[cr * YP + (r - LL)];
                        dmma_f64(acc[ti][0], acc[ti][1], av, bv);
                    }
                }
#pragma unroll
                for (int ti = 0; ti < TPW; ++ti) {
                    const int rt = w + ti * CTA_WARPS;
                    if (rt >= R2) continue;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = rt * 8 + g8, f = 2 * t4 + h;
                        if (r < LL && f < NR) {
                            const double wv = G[(M + f) * WP + r] - acc[ti][h];
                            if (f < NF) {
                                bad |= !isfinite(wv);
                                a.out[((size_t)idx * NF + f) * NN + piv[r]] = wv;
#pragma unroll
                                for (int ff = 0; ff < NF; ++ff)
                                    if (ff == f) xw[ff] = fmax(xw[ff], fabs(wv));
                            } else {
                                zw = fmax(zw, fabs(wv));
                            }
                        } else if (r >= LL && r < 2 * LL && f < NF) {
                            colk[(r - LL) * NF + f] = Y[(M + f) * YP + (r - LL)] - acc[ti][h];
                        }
                    }
                }
            }
            MF_TS(9);
        }
        // The multipliers of this stencil (warps 0..3, one family each) and the prologue of
        // the next one (warps 4..7) run side by side; the barrier publishes the products'
        // right-hand side for the former and the staged positions for the latter.
        static_assert(NF <= PW0, "one multiplier warp per family");
        cta_cp_async_wait_all();
        __syncthreads();
        MF_TS(10);
        const int64_t nxt = idx + gridDim.x;
        stage_idx(nxt + gridDim.x);  // (sidx was consumed by this stencil's position staging)
        if (w >= PW0) {
            if (nxt < a.m) prologue(nxt);
        } else if (ok) {
            // lambda_f = Q1^-1 (r_piv - Y v): the recorded column operations, last
            // first.  Step k needs the finished x_j (j > k) and the untouched s_j
            // (j < k): the j < k part is one parallel product up front, the rest a
            // column-oriented back substitution (x_k broadcast by one shuffle, the
            // lanes j < k fold it in) -- a 35-step chain of shuffle + FMA instead
            // of a warp reduction per step.  Only the estimate uses lambda.
            constexpr int LS = (LL + 31) / 32;
            for (int f = w; f < NF; f += CTA_WARPS) {
                double acc[LS];
#pragma unroll
                for (int q = 0; q < LS; ++q) {
                    const int jr = lane + 32 * q;
                    const int jc = jr < LL ? jr : 0;
                    // two interleaved partial sums halve the FMA chain
                    double a0 = jr < LL ? colk[jc * NF + f] : 0.0, a1 = 0.0;
#pragma unroll
                    for (int i2 = 0; i2 < LL - 1; ++i2) {
                        if (i2 < 32 * q + 31 && i2 < jr) {
                            if (i2 & 1) a1 = fma(-ops[jc * GP + i2], colk[i2 * NF + f], a1);
                            else a0 = fma(-ops[jc * GP + i2], colk[i2 * NF + f], a0);
                        }
                    }
                    acc[q] = a0 + a1;
                }
                double mx = 0.0;
#pragma unroll
                for (int k = LL - 1; k >= 0; --k) {
                    const double xk = __shfl_sync(FULL, acc[k >> 5], k & 31) * invs[k];
                    mx = fmax(mx, fabs(xk));
#pragma unroll
                    for (int q = 0; q < LS; ++q) {
                        if (32 * q >= k) continue;
                        const int jr = lane + 32 * q;
                        if (jr < k) acc[q] = fma(-ops[jr * GP + k], xk, acc[q]);
                    }
                }
                la[f] = mx;  // uniform over the warp
            }
        }
        MF_TS(11);
        // one fused reduction of the failure flag and the 1 + 2 NF maxima (all
        // >= 0); only thread 0 consumes them
        {
            constexpr int NV = 2 + 2 * NF;
            double rv[NV];
            rv[0] = bad ? 1.0 : 0.0;
            rv[1] = zw;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                rv[2 + f] = xw[f];
                rv[2 + NF + f] = la[f];
            }
            // warp maxima by two REDUX on the IEEE bits (non-negative doubles order
            // like their bit patterns), then lane v of warp 0 merges value v
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const unsigned long long b = (unsigned long long)__double_as_longlong(rv[v]);
                const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
                const unsigned mh = __reduce_max_sync(FULL, hi);
                const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
                rv[v] = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
            }
            if (lane == 0) {
#pragma unroll
                for (int v = 0; v < NV; ++v) prow[v * CTA_WARPS + w] = rv[v];
            }
            __syncthreads();
            if (w == 0) {
                double m = 0.0;
                if (lane < NV) {
                    m = prow[lane * CTA_WARPS];
#pragma unroll
                    for (int q = 1; q < CTA_WARPS; ++q) m = fmax(m, prow[lane * CTA_WARPS + q]);
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) rv[v] = __shfl_sync(FULL, m, v);
                bad = rv[0] != 0.0;
                zw = rv[1];
            }
            if (bad && stat == 0) stat = 1;
            double ratio = 0.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) ratio = fmax(ratio, fmax(rv[2 + f], rv[2 + NF + f]) / rv[2 + f]);
            xw[0] = ratio;  // thread 0's
        }
        if (tid == 0) {
            const double ratio = xw[0];
            const double est = anorm * zw * ratio;
            const bool close = r2min < a.min_sep2 * rc2max;
            if (stat != 0 || close || !(est <= a.hybrid_thresh)) {
                const unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                a.flag_list[slot] = idx;
            }
            a.status[idx] = 0;  // failures are re-derived in reference order by the re-solve
            MF_TS(8);
#ifdef MF_CTA_TIMING
            if (blockIdx.x == 0 && idx < 4 * (int64_t)gridDim.x)
                printf("cta2 %lld: coords %lld qg %lld sweep %lld joinY %lld Y %lld Kprod %lld elim %lld out %lld [dmma %lld bar %lld lam %lld red %lld]\n", (long long)idx,
                       ts_[1] - ts_[0], ts_[2] - ts_[1], ts_[3] - ts_[2], ts_[4] - ts_[3], ts_[5] - ts_[4], ts_[6] - ts_[5], ts_[7] - ts_[6], ts_[8] - ts_[7],
                       ts_[9] - ts_[7], ts_[10] - ts_[9], ts_[11] - ts_[10], ts_[8] - ts_[11]);
#endif
        }
        // (no barrier here: the reduction's barrier above published the next stencil's
        // prologue, and nothing the flag decision reads is written before the next one)
    }
    cta_cp_async_wait_all();
}

template <int NN, int DD, int DEG, int NF>
int launch_ns_cta2(const PhsArgs& a, cudaStream_t st, int sms) {
    using C = Cta2Cfg<NN, DD, DEG, NF>;
    constexpr GradedLex<DD, DEG> gl{};
    for (int m = 0; m < C::LL; ++m)
        for (int ax = 0; ax < DD; ++ax)
            if (a.P.expos[m * DD + ax] != gl.e[m][ax]) return MF_ERR_UNSUPPORTED;
    const size_t bytes = (size_t)C::TOTAL * sizeof(double);
    auto kern = phs_ns_cta2<NN, DD, DEG, NF>;
    MF_CUDA_CHECK(ensure_smem(kern, (int)bytes));
    int per_sm = occupancy(kern, CTA_THREADS, bytes);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = a.m;
    const int64_t cap = (int64_t)sms * per_sm * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, CTA_THREADS, bytes, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

int launch_phs_ns_cta(const PhsArgs& a, cudaStream_t st, int sms) {
    const int n = a.n, l = a.P.l, nf = a.P.nf;
    // HYBRID only (rows that fail or lose definiteness are re-solved); r^3 with
    // degree >= 1 (constant and linear monomials present: l >= d + 1)
    if (!a.flag_list || a.kappa || a.P.k != 3 || a.P.even || l < a.P.d + 1 || n - l < 1) return MF_ERR_UNSUPPORTED;
    if (n == 70 && l == 35 && a.P.d == 3 && nf == 4) {
        const int rc = launch_ns_cta2<70, 3, 4, 4>(a, st, sms);
        if (rc != MF_ERR_UNSUPPORTED) return rc;
    }
    const NsCtaLayout L = ns_cta_layout(n, a.P.d, l, nf + 1);
    const size_t bytes = L.total * sizeof(double);
    if (bytes > (size_t)dev_max_smem_optin()) return MF_ERR_UNSUPPORTED;
    auto kern = phs_ns_cta<0, 0, 0, 0>;
    MF_CUDA_CHECK(ensure_smem(kern, (int)bytes));
    int per_sm = occupancy(kern, CTA_THREADS, bytes);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = a.m;
    const int64_t cap = (int64_t)sms * per_sm * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, CTA_THREADS, bytes, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

int launch_phs_cta(const PhsArgs& a, bool replay, const int64_t* list, const int64_t* list_count,
                   int64_t max_count, cudaStream_t st, int sms) {
    return replay ? launch_cta_t<true>(a, list, list_count, max_count, st, sms)
                  : launch_cta_t<false>(a, list, list_count, max_count, st, sms);
}

}  // namespace mf

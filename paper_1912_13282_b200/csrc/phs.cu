// Batched polyharmonic RBF-FD shape computation (sm_100a).
//
// Replaces the reference's batch_phs_weights (_phs_batch.py:305-324) whose
// numba kernel _batch_numba (_phs_batch.py:186-302) builds, per stencil, the
// scaled (n+l)x(n+l) augmented collocation system and solves it with
// _solve_multi (_phs_batch.py:142-184).
//
// Kernels
//   phs_generic<REPLAY>   one warp per stencil, augmented system [A | B] in
//                         shared memory.  REPLAY=true follows the reference
//                         rounding sequence op for op (no FMA, same pivot
//                         rule, sequential ascending back-substitution);
//                         REPLAY=false uses FMA and a parallel back-substitution
//                         and carries one extra right-hand side z (+-1 probe)
//                         whose solution gives a conditioning estimate used by
//                         HYBRID mode to re-solve ill-conditioned stencils in
//                         REPLAY order.
//   phs_reg<S, NR, ...>   (phs_reg.cuh) register-resident fast path for the
//                         hot sizes.
#include <cfloat>
#include <cstdarg>

#include "common.cuh"
#include "phs_params.cuh"

namespace mf {

// Conditioning threshold for HYBRID re-solves: kappa_est = ||A||_inf *
// ||A^-1 z||_inf above this re-runs the stencil in REPLAY order.
__device__ __forceinline__ bool hybrid_flag(double kappa, double thresh) {
    return !(kappa <= thresh);  // NaN flags too
}

// per-warp shared-memory footprint of phs_generic, in doubles
__host__ __device__ inline int generic_lda(int s, int nf, bool probe) { return s + nf + (probe ? 1 : 0); }
__host__ __device__ inline size_t generic_warp_doubles(int n, int d, int s, int nf, bool probe) {
    int lda = generic_lda(s, nf, probe);
    size_t v = (size_t)n * d + (size_t)s * lda + (size_t)(nf + 1) * s + 8;
    return (v + 1) & ~(size_t)1;  // keep 16-byte alignment per warp
}

template <bool REPLAY>
__global__ void __launch_bounds__(256) phs_generic(PhsArgs a, const int64_t* __restrict__ list,
                                                   const int64_t* __restrict__ list_count) {
    extern __shared__ double smem_g[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int n = a.n, d = a.P.d, l = a.P.l, nf = a.P.nf;
    const int s = n + l;
    constexpr bool PROBE = !REPLAY;
    const int nrhs = nf + (PROBE ? 1 : 0);
    const int lda = s + nrhs;
    double* loc = smem_g + (size_t)wib * generic_warp_doubles(n, d, s, nf, PROBE);
    double* A = loc + n * d;
    double* scr = A + (size_t)s * lda;

    const int64_t count = list ? *list_count : a.m;
    const bool want_flag = PROBE && a.flag_list != nullptr;
    const bool want_est = PROBE && (a.flag_list != nullptr || a.kappa != nullptr);

    for (int64_t it = (int64_t)blockIdx.x * wpb + wib; it < count; it += (int64_t)gridDim.x * wpb) {
        const int64_t idx = list ? list[it] : it;
        const int64_t row = a.rows[idx];
        const int32_t* sti = a.stencils + idx * n;
        // 1. local coordinates (_phs_batch.py:198-202)
        for (int e = lane; e < n * d; e += 32) {
            int j = e / d, ax = e - j * d;
            loc[e] = __dsub_rn(a.pos[(int64_t)sti[j] * d + ax], a.pos[row * d + ax]);
        }
        __syncwarp();
        // 2. scale (_phs_batch.py:204-221)
        int stat = 0;
        double sc = 1.0;
        double anorm = 0.0;
        double r2min = INFINITY, rc2max = 0.0;
        if (a.P.scale_code != MF_SCALE_NONE) {
            const bool nearest = a.P.scale_code == MF_SCALE_NEAREST;
            double best = nearest ? INFINITY : -1.0;
            for (int j = lane; j < n; j += 32) {
                double r2 = 0.0;
                for (int ax = 0; ax < d; ++ax) r2 = __dadd_rn(r2, __dmul_rn(loc[j * d + ax], loc[j * d + ax]));
                double r = __dsqrt_rn(r2);
                if (nearest) {
                    if (r > 0.0 && r < best) best = r;
                } else if (r > best) {
                    best = r;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(FULL, best, o);
                best = nearest ? fmin(best, ob) : fmax(best, ob);
            }
            if (nearest ? (best == INFINITY) : !(best > 0.0)) stat = 2;
            else sc = best;
        }
        if (stat == 0) {
            // 3. local /= s
            for (int e = lane; e < n * d; e += 32) loc[e] = __ddiv_rn(loc[e], sc);
            __syncwarp();
            // 4. system: PHS block (symmetric, bitwise: (a-b)^2 == (b-a)^2)
            for (int e = lane; e < n * n; e += 32) {
                int i = e / n, j = e - i * n;
                if (j < i) continue;
                double v = 0.0;
                if (j > i) {
                    double r2 = 0.0;
                    for (int ax = 0; ax < d; ++ax) {
                        double df = __dsub_rn(loc[i * d + ax], loc[j * d + ax]);
                        r2 = __dadd_rn(r2, __dmul_rn(df, df));
                    }
                    v = phs_phi(__dsqrt_rn(r2), a.P.k, a.P.even);
                    r2min = fmin(r2min, r2);
                }
                A[(size_t)i * lda + j] = v;
                A[(size_t)j * lda + i] = v;
            }
            // monomial blocks Q, Q^T (_phs_batch.py:240-247) and zero corner
            for (int e = lane; e < n * l; e += 32) {
                int jm = e / n, i = e - jm * n;
                double q = phs_monomial(loc + i * d, a.P.expos + jm * d, d);
                A[(size_t)i * lda + n + jm] = q;
                A[(size_t)(n + jm) * lda + i] = q;
            }
            for (int e = lane; e < l * l; e += 32) {
                int i = e / l, j = e - i * l;
                A[(size_t)(n + i) * lda + n + j] = 0.0;
            }
            // right-hand sides (_phs_batch.py:249-290)
            for (int j = lane; j < n; j += 32) {
                double top[MF_MAX_FAMILIES];
                phs_rhs_top(loc + j * d, d, a.P, top);
                for (int f = 0; f < nf; ++f)
                    A[(size_t)j * lda + s + f] = __dmul_rn(top[f], pow_cr_int(sc, -a.P.orders[f]));
            }
            for (int e = lane; e < l * nf; e += 32) {
                int f = e / l, j = e - f * l;
                A[(size_t)(n + j) * lda + s + f] =
                    __dmul_rn(a.P.base_bot[f * MF_MAX_MONOMIALS + j], pow_cr_int(sc, -a.P.orders[f]));
            }
            if (PROBE) {
                for (int r = lane; r < s; r += 32) A[(size_t)r * lda + s + nf] = probe_sign(idx, r);
            }
            __syncwarp();
            if (PROBE) {
                for (int r = lane; r < s; r += 32) {
                    double acc = 0.0;
                    for (int c = 0; c < s; ++c) acc += fabs(A[(size_t)r * lda + c]);
                    anorm = fmax(anorm, acc);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) anorm = fmax(anorm, __shfl_xor_sync(FULL, anorm, o));
            }

            // 5. elimination with row partial pivoting (_phs_batch.py:150-176)
            for (int col = 0; col < s; ++col) {
                double a00 = fabs(A[(size_t)col * lda + col]);
                double best = -1.0;
                int piv = s;
                for (int r = col + lane; r < s; r += 32) {
                    double v = fabs(A[(size_t)r * lda + col]);
                    if (v > best) { best = v; piv = r; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    double ob = __shfl_xor_sync(FULL, best, o);
                    int op = __shfl_xor_sync(FULL, piv, o);
                    if (ob > best || (ob == best && op < piv)) { best = ob; piv = op; }
                }
                if (isnan(a00) || best == 0.0 || !isfinite(best)) { stat = 1; break; }
                if (piv != col) {
                    for (int cc = col + lane; cc < lda; cc += 32) {
                        double t = A[(size_t)col * lda + cc];
                        A[(size_t)col * lda + cc] = A[(size_t)piv * lda + cc];
                        A[(size_t)piv * lda + cc] = t;
                    }
                    __syncwarp();
                }
                const double inv = __drcp_rn(A[(size_t)col * lda + col]);
                const double* prow = A + (size_t)col * lda;
                for (int r = col + 1; r < s; ++r) {
                    double* arow = A + (size_t)r * lda;
                    double fac = __dmul_rn(arow[col], inv);
                    if (fac != 0.0) {
                        for (int cc = col + 1 + lane; cc < lda; cc += 32) {
                            if (REPLAY) arow[cc] = __dsub_rn(arow[cc], __dmul_rn(fac, prow[cc]));
                            else arow[cc] = fma(-fac, prow[cc], arow[cc]);
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (stat == 0) {
            // 6. back-substitution (_phs_batch.py:177-183)
            if (REPLAY) {
                for (int col = s - 1; col >= 0; --col) {
                    const double inv = __drcp_rn(A[(size_t)col * lda + col]);
                    const int len = s - col - 1;
                    for (int e = lane; e < len * nf; e += 32) {
                        int f = e / len, rr = e - f * len;
                        int r = col + 1 + rr;
                        scr[f * s + r] = __dmul_rn(A[(size_t)col * lda + r], A[(size_t)r * lda + s + f]);
                    }
                    __syncwarp();
                    if (lane < nf) {
                        double acc = A[(size_t)col * lda + s + lane];
                        for (int r = col + 1; r < s; ++r) acc = __dsub_rn(acc, scr[lane * s + r]);
                        A[(size_t)col * lda + s + lane] = __dmul_rn(acc, inv);
                    }
                    __syncwarp();
                }
            } else {
                for (int col = s - 1; col >= 0; --col) {
                    const double inv = __drcp_rn(A[(size_t)col * lda + col]);
                    if (lane < nrhs) A[(size_t)col * lda + s + lane] *= inv;
                    __syncwarp();
                    for (int e = lane; e < col * nrhs; e += 32) {
                        int f = e / col, r = e - f * col;
                        A[(size_t)r * lda + s + f] =
                            fma(-A[(size_t)r * lda + col], A[(size_t)col * lda + s + f], A[(size_t)r * lda + s + f]);
                    }
                    __syncwarp();
                }
            }
            // 7. outputs, non-finite check (_phs_batch.py:293-298)
            bool bad = false;
            for (int e = lane; e < n * nf; e += 32) {
                int f = e / n, j = e - f * n;
                double v = A[(size_t)j * lda + s + f];
                bad |= !isfinite(v);
                a.out[((size_t)idx * nf + f) * n + j] = v;
            }
            if (__any_sync(FULL, bad)) stat = 1;
            if (want_est && stat == 0) {
                // same estimate as phs_reg.cuh
                double zw = 0.0, za = 0.0, ratio = 0.0;
                for (int r = lane; r < s; r += 32) {
                    const double v = fabs(A[(size_t)r * lda + s + nf]);
                    za = fmax(za, v);
                    if (r < n) zw = fmax(zw, v);
                }
                for (int f = 0; f < nf; ++f) {
                    double xa = 0.0, xw = 0.0;
                    for (int r = lane; r < s; r += 32) {
                        const double v = fabs(A[(size_t)r * lda + s + f]);
                        xa = fmax(xa, v);
                        if (r < n) xw = fmax(xw, v);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        xa = fmax(xa, __shfl_xor_sync(FULL, xa, o));
                        xw = fmax(xw, __shfl_xor_sync(FULL, xw, o));
                    }
                    ratio = fmax(ratio, xa / xw);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    zw = fmax(zw, __shfl_xor_sync(FULL, zw, o));
                    za = fmax(za, __shfl_xor_sync(FULL, za, o));
                }
                for (int j = lane; j < n; j += 32) {
                    double rc2 = 0.0;
                    for (int ax = 0; ax < d; ++ax) rc2 = fma(loc[j * d + ax], loc[j * d + ax], rc2);
                    rc2max = fmax(rc2max, rc2);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    r2min = fmin(r2min, __shfl_xor_sync(FULL, r2min, o));
                    rc2max = fmax(rc2max, __shfl_xor_sync(FULL, rc2max, o));
                }
                const double est = anorm * zw * ratio;
                const bool close = r2min < a.min_sep2 * rc2max;
                if (lane == 0 && a.kappa) {
                    a.kappa[4 * idx + 0] = anorm;
                    a.kappa[4 * idx + 1] = zw;
                    a.kappa[4 * idx + 2] = za;
                    a.kappa[4 * idx + 3] = ratio;
                }
                if (want_flag && lane == 0 && (close || hybrid_flag(est, a.hybrid_thresh))) {
                    unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                    a.flag_list[slot] = idx;
                }
            }
        }
        if (PROBE && want_flag && stat != 0 && lane == 0) {
            // failures are re-derived in reference order so the status matches
            unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
            a.flag_list[slot] = idx;
            stat = 0;
        }
        if (lane == 0) {
            a.status[idx] = (int8_t)stat;
            if (stat && a.first_fail) atomicMin((unsigned long long*)a.first_fail, (unsigned long long)idx);
        }
        __syncwarp();
    }
}

}  // namespace mf

using namespace mf;

namespace {

int sm_count() { return dev_sms(); }

template <bool REPLAY>
int launch_generic(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count,
                   cudaStream_t st) {
    const int s = a.n + a.P.l;
    size_t per_warp = generic_warp_doubles(a.n, a.P.d, s, a.P.nf, !REPLAY) * sizeof(double);
    const int max_smem = dev_max_smem_optin();
    int wpb = (int)((size_t)(max_smem / 2) / per_warp);
    if (wpb > 4) wpb = 4;
    if (wpb < 1) wpb = per_warp <= (size_t)max_smem ? 1 : 0;
    MF_REQUIRE(wpb >= 1, "stencil system of size %d needs %zu bytes of shared memory (max %d)", s,
               per_warp, max_smem);
    size_t bytes = per_warp * wpb;
    MF_CUDA_CHECK(ensure_smem(phs_generic<REPLAY>, (int)bytes));
    int64_t blocks = (max_count + wpb - 1) / wpb;
    int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    phs_generic<REPLAY><<<(unsigned)blocks, 32 * wpb, bytes, st>>>(a, list, list_count);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

}  // namespace

extern "C" int mf_phs_workspace_size(int64_t m, size_t* bytes) {
    if (!bytes || m < 0) {
        set_error("mf_phs_workspace_size: bad arguments");
        return MF_ERR_ARG;
    }
    Arena ar{nullptr, 0, 0, true};
    ar.take<int64_t>(1);
    ar.take<int64_t>((size_t)m + 1);
    ar.take<int>((size_t)m + 1);  // flag marks (family chunks)
    *bytes = ar.off;
    return MF_OK;
}

extern "C" int mf_phs_weights(const double* pos, int64_t N, int32_t d, const int64_t* rows,
                              const int32_t* stencils, int64_t m, int32_t n, int32_t k, int32_t even,
                              const int32_t* expos, int32_t l, const double* base_bot,
                              const int32_t* kinds, const int32_t* ax_a, const int32_t* ax_b,
                              const int32_t* orders, int32_t nf, int32_t scale_code, int32_t mode,
                              double* out, int8_t* status, int64_t* first_fail, int64_t* n_replayed,
                              const mf_phs_options_t* opts, void* ws, size_t ws_bytes, void* stream) {
    (void)N;
    MF_REQUIRE(d >= 1 && d <= MF_MAX_DIM, "mf_phs_weights: dimension %d not in 1..%d", d, MF_MAX_DIM);
    MF_REQUIRE(nf >= 1 && nf <= MF_MAX_FAMILIES, "mf_phs_weights: %d families (max %d)", nf, MF_MAX_FAMILIES);
    MF_REQUIRE(l >= 0 && l <= MF_MAX_MONOMIALS, "mf_phs_weights: %d monomials (max %d)", l, MF_MAX_MONOMIALS);
    MF_REQUIRE(n >= 1 && m >= 0, "mf_phs_weights: bad stencil shape");
    MF_REQUIRE(k >= 1 && k <= 64, "mf_phs_weights: exponent %d out of range", k);
    MF_REQUIRE(mode >= MF_PHS_REPLAY && mode <= MF_PHS_HYBRID, "mf_phs_weights: bad mode %d", mode);
    cudaStream_t st = (cudaStream_t)stream;
    if (first_fail) MF_CUDA_CHECK(cudaMemsetAsync(first_fail, 0x7f, sizeof(int64_t), st));
    if (n_replayed) MF_CUDA_CHECK(cudaMemsetAsync(n_replayed, 0, sizeof(int64_t), st));
    if (m == 0) return MF_OK;

    PhsArgs a{};
    a.pos = pos;
    a.rows = rows;
    a.stencils = stencils;
    a.m = m;
    a.n = n;
    a.out = out;
    a.status = status;
    a.first_fail = first_fail;
    a.hybrid_thresh = (opts && opts->hybrid_threshold > 0.0) ? opts->hybrid_threshold : MF_PHS_DEFAULT_THRESHOLD;
    a.kappa = opts ? opts->kappa : nullptr;
    {
        const double sep = (opts && opts->min_separation > 0.0) ? opts->min_separation : MF_PHS_DEFAULT_MIN_SEPARATION;
        a.min_sep2 = sep * sep;
    }
    a.out_nf = nf;
    a.out_f0 = 0;
    a.flag_mark = nullptr;
    int rc = fill_phs_params(a.P, d, k, even, expos, l, base_bot, kinds, ax_a, ax_b, orders, nf, scale_code);
    if (rc != MF_OK) return rc;

    const bool big = n + l > 48;  // CTA-per-stencil kernel for large systems
    if (mode == MF_PHS_REPLAY) {
        rc = launch_phs_replay_reg(a, nullptr, nullptr, m, st, sm_count());
        if (rc == MF_ERR_UNSUPPORTED && big) rc = launch_phs_cta(a, true, nullptr, nullptr, m, st, sm_count());
        if (rc == MF_ERR_UNSUPPORTED) rc = launch_generic<true>(a, nullptr, nullptr, m, st);
        return rc;
    }

    int64_t* flag_count = nullptr;
    int64_t* flag_list = nullptr;
    if (mode == MF_PHS_HYBRID) {
        Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
        flag_count = ar.take<int64_t>(1);
        flag_list = ar.take<int64_t>((size_t)m + 1);
        int* flag_mark = ar.take<int>((size_t)m + 1);
        if (ws == nullptr || !ar.ok()) {
            set_error("mf_phs_weights: HYBRID mode needs a workspace of mf_phs_workspace_size bytes");
            return MF_ERR_WORKSPACE;
        }
        MF_CUDA_CHECK(cudaMemsetAsync(flag_count, 0, sizeof(int64_t), st));
        a.flag_list = flag_list;
        a.flag_count = flag_count;
        a.flag_mark = flag_mark;  // used (and zeroed) only when the first pass runs in family chunks
    }
    rc = launch_phs_fast(a, st, sm_count());
    if (rc == MF_ERR_UNSUPPORTED && big) rc = launch_phs_ns_cta(a, st, sm_count());
    if (rc == MF_ERR_UNSUPPORTED && big) rc = launch_phs_cta(a, false, nullptr, nullptr, m, st, sm_count());
    if (rc == MF_ERR_UNSUPPORTED) rc = launch_generic<false>(a, nullptr, nullptr, m, st);
    if (rc != MF_OK) return rc;
    if (mode == MF_PHS_HYBRID) {
        rc = launch_phs_replay_reg(a, flag_list, flag_count, m, st, sm_count());
        if (rc == MF_ERR_UNSUPPORTED && big) rc = launch_phs_cta(a, true, flag_list, flag_count, m, st, sm_count());
        if (rc == MF_ERR_UNSUPPORTED) rc = launch_generic<true>(a, flag_list, flag_count, m, st);
        if (rc != MF_OK) return rc;
        if (n_replayed) MF_CUDA_CHECK(cudaMemcpyAsync(n_replayed, flag_count, sizeof(int64_t),
                                                      cudaMemcpyDeviceToDevice, st));
    }
    return MF_OK;
}

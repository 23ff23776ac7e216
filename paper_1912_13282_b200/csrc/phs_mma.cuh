// Blocked shape solve on the fp64 tensor cores (sm_100a, FAST mode).
//
// One warp per stencil.  The augmented system [A Q | B ; Q^T 0 | B'] (S rows,
// C = S + NR columns) lives in registers in the accumulator layout of the
// fp64 MMA (mma.sync m8n8k4 .f64): tile (ti, tj) covers rows 8ti.. and
// columns 8tj..; lane (g = lane/4, t = lane%4) holds rows 8ti+g and columns
// 8tj+2t, 8tj+2t+1.  LU with row partial pivoting runs in panels of four
// columns (right-looking, LAPACK getrf order):
//
//   1. panel factorisation, column by column: pivot search (one REDUX, a
//      ballot, the winner lane's speculative reciprocal), the owner quad
//      writes the pivot row to U in shared memory, every quad forms its
//      multipliers, and the rest of the panel gets the rank-1 update;
//   2. U12 = L11^-1 A12 on the four new U rows in shared memory;
//   3. A22 -= L21 U12 as m8n8k4 DMMAs: L21 is the A operand (each lane holds
//      the multiplier of its row for panel column t), U12 the B operand.
//
// Rows never move: pivoted rows retire (live flag) and keep receiving
// harmless updates.  The trailing update -- two thirds of the flops -- runs on
// the tensor pipe at 256 FMAs per instruction, which is what lifts the solve
// off the instruction-issue limit of the rank-1 DFMA formulation (phs_reg.cuh).
// Back-substitution, outputs and the HYBRID criterion follow phs_reg.cuh.
#pragma once

#include "phs_reg.cuh"

namespace mf {

template <int NN, int DEG, int DD, int NF>
struct MmaCfg {
    static constexpr int LL = binom(DEG + DD, DD);
    static constexpr int S = NN + LL;
    static constexpr int NR = NF + 1;  // + probe
    static constexpr int C = S + NR;
    static constexpr int TR = (S + 7) / 8;
    static constexpr int TC = (C + 7) / 8;
    // U row stride: >= 8*TC (B-fragment loads read 8 columns past a panel) and
    // == 4 (mod 16) doubles so the four U12 rows of a B load hit disjoint banks
    static constexpr int CP = ((8 * TC - 4 + 15) / 16) * 16 + 4;
    static constexpr int R = (S + 31) / 32;  // back-substitution: rows per lane
    static constexpr int NP = (S + 3) / 4;   // panels
    static constexpr int WARPS = 4;
    static constexpr int U_DBL = S * CP;
    static constexpr int LOC_DBL = ((NN * DD + 1) & ~1);
    static constexpr int RHS_DBL = ((S * NR + 1) & ~1);
    static constexpr int L11_DBL = 16;
    static constexpr int WARP_DBL = U_DBL + LOC_DBL + RHS_DBL + L11_DBL;
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DBL * sizeof(double);
    static_assert(S * NN <= U_DBL, "staging matrix must fit in U");
    static_assert(CP >= C, "row stride");
};

__device__ __forceinline__ void dmma_neg(double& d0, double& d1, double a, double b) {
    // D = (-a) x b + D  on the fp64 tensor core (m8n8k4, row.col)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(-a), "d"(b));
}

// owner quad writes pivot row (tile row TI) columns >= 8*tj0 to U and retires it
// (pti is warp-uniform: one branch of the chain is taken by the whole warp)
template <int TI, int TR, int TC>
__device__ __forceinline__ void store_pivot_row(int pti, bool quad_owner, int t, int jj, int tj0,
                                                double (&acc)[TR][TC][2], const double (&Lf)[TR], double (&alive)[TR],
                                                double* urow, double* l11) {
    if constexpr (TI < TR) {
        if (pti == TI) {
#pragma unroll
            for (int tj = 0; tj < TC; ++tj)
                if (tj >= tj0) st_shared_v2_if(quad_owner, urow + 8 * tj + 2 * t, acc[TI][tj][0], acc[TI][tj][1]);
            if (quad_owner && t < jj) l11[jj * 4 + t] = Lf[TI];
            alive[TI] = quad_owner ? 0.0 : alive[TI];
        } else {
            store_pivot_row<TI + 1, TR, TC>(pti, quad_owner, t, jj, tj0, acc, Lf, alive, urow, l11);
        }
    }
}

template <int NN, int DEG, int DD, int NF>
__global__ void __launch_bounds__(128) phs_mma(PhsArgs a) {
    using Cfg = MmaCfg<NN, DEG, DD, NF>;
    constexpr int LL = Cfg::LL, S = Cfg::S, NR = Cfg::NR, C = Cfg::C, CP = Cfg::CP, R = Cfg::R;
    constexpr int TR = Cfg::TR, TC = Cfg::TC;
    extern __shared__ __align__(16) double smem_m[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* U = smem_m + (size_t)wib * Cfg::WARP_DBL;
    double* E = U;
    double* loc = U + Cfg::U_DBL;
    double* Rs = loc + Cfg::LOC_DBL;
    double* L11 = Rs + Cfg::RHS_DBL;
    const bool want_flag = a.flag_list != nullptr;
    const bool want_est = a.flag_list != nullptr || a.kappa != nullptr;
    const PhsParams& P = a.P;

    for (int64_t idx = (int64_t)blockIdx.x * Cfg::WARPS + wib; idx < a.m; idx += (int64_t)gridDim.x * Cfg::WARPS) {
        const int64_t row = a.rows[idx];
        const int32_t* sti = a.stencils + idx * NN;
        // ---- local coordinates and scale (_phs_batch.py:198-226)
        for (int e = lane; e < NN * DD; e += 32) {
            int j = e / DD, ax = e - j * DD;
            loc[e] = __dsub_rn(a.pos[(int64_t)sti[j] * DD + ax], a.pos[row * DD + ax]);
        }
        __syncwarp();
        int stat = 0;
        double sc = 1.0;
        if (P.scale_code != MF_SCALE_NONE) {
            const bool nearest = P.scale_code == MF_SCALE_NEAREST;
            double best = nearest ? INFINITY : -1.0;
            for (int j = lane; j < NN; j += 32) {
                double r2 = 0.0;
#pragma unroll
                for (int ax = 0; ax < DD; ++ax) r2 = __dadd_rn(r2, __dmul_rn(loc[j * DD + ax], loc[j * DD + ax]));
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
        double facs[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) facs[f] = pow_cr_int(sc, -P.orders[f]);

        // ---- staging: PHS block over unordered pairs, Q^T, right-hand sides
        double r2min = INFINITY, rc2max = 0.0;
        for (int e = lane; e < NN * DD; e += 32) loc[e] = __ddiv_rn(loc[e], sc);
        __syncwarp();
        for (int p = lane; p < NN * (NN - 1) / 2; p += 32) {
            int i, j;
            pair_of<NN>(p, i, j);
            double df = loc[i * DD] - loc[j * DD];
            double r2 = df * df;
#pragma unroll
            for (int ax = 1; ax < DD; ++ax) {
                df = loc[i * DD + ax] - loc[j * DD + ax];
                r2 = fma(df, df, r2);
            }
            const double v = (P.k == 3 && !P.even) ? r2 * sqrt(r2) : phs_phi(sqrt(r2), P.k, P.even);
            r2min = fmin(r2min, r2);
            E[i * NN + j] = v;
            E[j * NN + i] = v;
        }
        for (int i = lane; i < NN; i += 32) {
            E[i * NN + i] = 0.0;
            double rc2 = 0.0;
#pragma unroll
            for (int ax = 0; ax < DD; ++ax) rc2 = fma(loc[i * DD + ax], loc[i * DD + ax], rc2);
            rc2max = fmax(rc2max, rc2);
        }
        monomial_rows<DD, DEG, 0, LL>(E, loc, NN, lane);
        for (int r = lane; r < S; r += 32) {
            if (r < NN) {
                double top[MF_MAX_FAMILIES];
                phs_rhs_top(loc + r * DD, DD, P, top);
#pragma unroll
                for (int f = 0; f < NF; ++f) Rs[r * NR + f] = __dmul_rn(top[f], facs[f]);
            } else {
#pragma unroll
                for (int f = 0; f < NF; ++f) Rs[r * NR + f] = __dmul_rn(P.base_bot[f * MF_MAX_MONOMIALS + (r - NN)], facs[f]);
            }
            Rs[r * NR + NF] = probe_sign(idx, r);
        }
        __syncwarp();

        // ---- accumulator tiles
        double acc[TR][TC][2];
        double rowsum[TR];
#pragma unroll
        for (int ti = 0; ti < TR; ++ti) {
            const int r = 8 * ti + g;
            rowsum[ti] = 0.0;
#pragma unroll
            for (int tj = 0; tj < TC; ++tj) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * tj + 2 * t + e;
                    double v = 0.0;
                    if (r < S) {
                        if (c < NN) v = E[r * NN + c];
                        else if (c < S) v = r < NN ? E[c * NN + r] : 0.0;
                        else if (c < C) v = Rs[r * NR + (c - S)];
                    }
                    acc[ti][tj][e] = v;
                    if (c < S) rowsum[ti] += fabs(v);
                }
            }
        }
        __syncwarp();  // staging is dead; U takes its place
        double anorm = 0.0;
        if (want_est) {
#pragma unroll
            for (int ti = 0; ti < TR; ++ti) {
                double s = rowsum[ti];
                s += __shfl_xor_sync(FULL, s, 1);
                s += __shfl_xor_sync(FULL, s, 2);
                anorm = fmax(anorm, s);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) anorm = fmax(anorm, __shfl_xor_sync(FULL, anorm, o));
        }

        // ---- blocked LU with partial pivoting.  Runtime loop over the tile columns
        //      it = 0..; the register tiles rotate left by one tile column per
        //      iteration, so the active panels always sit in acc[.][0] and the loop
        //      body (two 4-column panels) is compiled once.
        bool ok = stat == 0;
        double alive[TR];  // 1.0 while the row is not yet a pivot row
        double Lf[TR];
#pragma unroll
        for (int ti = 0; ti < TR; ++ti) {
            alive[ti] = 8 * ti + g < S ? 1.0 : 0.0;
            Lf[ti] = 0.0;
        }
        constexpr int NIT = (S + 7) / 8;
#pragma unroll 1
        for (int it = 0; it < NIT; ++it) {
            const int cbase = 8 * it;  // absolute column of acc[.][0]
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j0 = cbase + 4 * h;
                if (j0 < S) {
                    const int jn = (S - j0) < 4 ? (S - j0) : 4;
                    const int pe = j0 + jn;
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        if (jj < jn) {
                            const int j = j0 + jj;
                            constexpr int dummy = 0;
                            (void)dummy;
                            const int jl = 4 * h + jj;  // column inside tile 0 (compile-time)
                            const int tcj = jl >> 1, ej = jl & 1;
                            // (a) pivot search over the live rows of column j
                            double best = -1.0, cval = 1.0;
                            int bti = 0;
#pragma unroll
                            for (int ti = 0; ti < TR; ++ti) {
                                const double v = acc[ti][0][ej];
                                const double av = fabs(v) * alive[ti];
                                const bool bt = av > best;
                                best = bt ? av : best;
                                cval = bt ? v : cval;
                                bti = bt ? ti : bti;
                            }
                            if (t != tcj) best = -1.0;
                            const double cinv = fast_rcp(cval);
                            const unsigned hk =
                                best >= 0.0 ? (unsigned)((unsigned long long)__double_as_longlong(best) >> 32) : 0u;
                            const unsigned mh = __reduce_max_sync(FULL, hk);
                            const unsigned ball = __ballot_sync(FULL, best >= 0.0 && hk == mh);
                            ok = ok && ball != 0u && mh != 0u;
                            const int wl = (__ffs(ball) - 1) & 31;
                            const double inv = __shfl_sync(FULL, cinv, wl);
                            const int pti = __shfl_sync(FULL, bti, wl);
                            const bool quad_owner = g == (wl >> 2) && ball != 0u;
                            // (b) pivot row -> U[j][cbase..], L11 entries of this row, retire it
                            store_pivot_row<0, TR, TC>(pti, quad_owner, t, jj, 0, acc, Lf, alive,
                                                       U + j * CP + cbase, L11);
                            // (c) multipliers of every row for column j (lane tcj of each quad holds it)
                            double l[TR];
#pragma unroll
                            for (int ti = 0; ti < TR; ++ti) {
                                l[ti] = __shfl_sync(FULL, acc[ti][0][ej], (lane & ~3) | tcj) * inv;
                                if (t == jj) Lf[ti] = l[ti];
                            }
                            __syncwarp();
                            // (d) rank-1 update of the remaining panel columns (tile 0)
                            if (jj + 1 < jn) {
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int cl = 2 * t + e;  // column inside tile 0
                                    if (cl > jl && cl < 4 * h + jn) {
                                        const double u = U[j * CP + cbase + cl];
#pragma unroll
                                        for (int ti = 0; ti < TR; ++ti) acc[ti][0][e] = fma(-l[ti], u, acc[ti][0][e]);
                                    }
                                }
                            }
                        }
                    }
                    // (2) U12 = L11^-1 A12 on rows j0.. (columns pe.., incl. right-hand sides)
                    __syncwarp();
#pragma unroll
                    for (int k = 1; k < 4; ++k) {
                        if (k < jn) {
                            for (int c = pe + lane; c < C; c += 32) {
                                double v = U[(j0 + k) * CP + c];
#pragma unroll
                                for (int i = 0; i < k; ++i) v = fma(-L11[k * 4 + i], U[(j0 + i) * CP + c], v);
                                U[(j0 + k) * CP + c] = v;
                            }
                            __syncwarp();
                        }
                    }
                    // (3) A22 -= L21 U12 on the tensor cores (live tile columns only)
#pragma unroll
                    for (int tj = h; tj < TC; ++tj) {
                        if (tj < TC - it) {
                            const int cb = cbase + 8 * tj + g;  // absolute column of B's n index
                            const double b = (cb >= pe && cb < C && t < jn) ? U[(j0 + t) * CP + cb] : 0.0;
#pragma unroll
                            for (int ti = 0; ti < TR; ++ti) dmma_neg(acc[ti][tj][0], acc[ti][tj][1], Lf[ti], b);
                        }
                    }
                }
            }
            // rotate the tiles: absolute tile column it+1 moves to acc[.][0]
#pragma unroll
            for (int ti = 0; ti < TR; ++ti) {
#pragma unroll
                for (int tj = 0; tj + 1 < TC; ++tj) {
                    acc[ti][tj][0] = acc[ti][tj + 1][0];
                    acc[ti][tj][1] = acc[ti][tj + 1][1];
                }
                acc[ti][TC - 1][0] = 0.0;
                acc[ti][TC - 1][1] = 0.0;
            }
        }
        __syncwarp();

        // ---- back-substitution on U (rows in pivot order), x in registers
        double bb[R][NR], dinv[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int r = lane + 32 * k;
            const int rr = r < S ? r : 0;
#pragma unroll
            for (int f = 0; f < NR; ++f) bb[k][f] = U[rr * CP + S + f];
            dinv[k] = fast_rcp(U[rr * CP + rr]);
        }
#pragma unroll
        for (int col = S - 1; col >= 0; --col) {
            const int kc = col >> 5, lc = col & 31;
            double xs[NR];
#pragma unroll
            for (int f = 0; f < NR; ++f) xs[f] = __shfl_sync(FULL, bb[kc][f] * dinv[kc], lc);
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (32 * k < col) {
                    const int r = lane + 32 * k;
                    const double ur = U[(r < S ? r : 0) * CP + col];
                    if (r < col) {
#pragma unroll
                        for (int f = 0; f < NR; ++f) bb[k][f] = fma(-ur, xs[f], bb[k][f]);
                    }
                }
            }
            if (lane == lc) {
#pragma unroll
                for (int f = 0; f < NR; ++f) bb[kc][f] = xs[f];
            }
        }
        // ---- outputs, non-finite check, HYBRID criterion (as phs_reg.cuh)
        bool bad = !ok;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int r = lane + 32 * k;
            if (r < NN) {
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    bad |= !isfinite(bb[k][f]);
                    a.out[((size_t)idx * NF + f) * NN + r] = bb[k][f];
                }
            }
        }
        if (__any_sync(FULL, bad) && stat == 0) stat = 1;
        if (want_est) {
            double zw = 0.0, za = 0.0, xa[NF], xw[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) xa[f] = xw[f] = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int r = lane + 32 * k;
                if (r < S) {
                    const double z = fabs(bb[k][NF]);
                    za = fmax(za, z);
                    if (r < NN) zw = fmax(zw, z);
#pragma unroll
                    for (int f = 0; f < NF; ++f) {
                        xa[f] = fmax(xa[f], fabs(bb[k][f]));
                        if (r < NN) xw[f] = fmax(xw[f], fabs(bb[k][f]));
                    }
                }
            }
            double sep2 = r2min;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                zw = fmax(zw, __shfl_xor_sync(FULL, zw, o));
                za = fmax(za, __shfl_xor_sync(FULL, za, o));
                sep2 = fmin(sep2, __shfl_xor_sync(FULL, sep2, o));
                rc2max = fmax(rc2max, __shfl_xor_sync(FULL, rc2max, o));
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    xa[f] = fmax(xa[f], __shfl_xor_sync(FULL, xa[f], o));
                    xw[f] = fmax(xw[f], __shfl_xor_sync(FULL, xw[f], o));
                }
            }
            double ratio = 0.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) ratio = fmax(ratio, xa[f] / xw[f]);
            const double est = anorm * zw * ratio;
            const bool close = sep2 < a.min_sep2 * rc2max;
            if (lane == 0 && a.kappa) {
                a.kappa[4 * idx + 0] = anorm;
                a.kappa[4 * idx + 1] = zw;
                a.kappa[4 * idx + 2] = za;
                a.kappa[4 * idx + 3] = ratio;
            }
            if (want_flag && stat == 0 && lane == 0 && (close || !(est <= a.hybrid_thresh))) {
                unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                a.flag_list[slot] = idx;
            }
        }
        if (want_flag && stat != 0) {
            if (lane == 0) {
                unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
                a.flag_list[slot] = idx;
            }
            stat = 0;
        }
        if (lane == 0) {
            a.status[idx] = (int8_t)stat;
            if (stat && a.first_fail) atomicMin((unsigned long long*)a.first_fail, (unsigned long long)idx);
        }
        __syncwarp();
    }
}

template <int NN, int DEG, int DD, int NF>
int launch_mma(const PhsArgs& a, cudaStream_t st, int sms) {
    using Cfg = MmaCfg<NN, DEG, DD, NF>;
    constexpr GradedLex<DD, DEG> gl{};
    if (a.P.l != Cfg::LL) return MF_ERR_UNSUPPORTED;
    for (int m = 0; m < Cfg::LL; ++m)
        for (int ax = 0; ax < DD; ++ax)
            if (a.P.expos[m * DD + ax] != gl.e[m][ax]) return MF_ERR_UNSUPPORTED;
    auto kern = phs_mma<NN, DEG, DD, NF>;
    MF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    int per_sm = 0;
    MF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::WARPS * 32, Cfg::SMEM));
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (a.m + Cfg::WARPS - 1) / Cfg::WARPS;
    int64_t cap = (int64_t)sms * per_sm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, Cfg::WARPS * 32, Cfg::SMEM, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

#define MF_INSTANTIATE_MMA(NN, DEG, DD, NF) \
    template int launch_mma<NN, DEG, DD, NF>(const PhsArgs&, cudaStream_t, int);

}  // namespace mf

// Register shape solve for 32 < S <= 64 (FAST mode): rows 0..31 one per lane,
// the E = S-32 extra rows split into column halves across lane pairs.
//
// phs_reg.cuh gives every lane R = 2 full row slots when S > 32, although only
// S-32 lanes have a second row: for C3 (S = 45) that is 94 doubles per lane
// and 8 warps per SM, and every step stores the pivot row from both slots.
// Here lane l holds row l (all C columns) and half h = l&1 of extra row
// 32 + l/2 (columns [hH, hH+H), H = ceil(C/2)).  The rank-1 update is still
// one FMA per lane per column (the extra-row FMA is predicated on the half),
// registers drop to C + H doubles (71 for C3), and the pivot row -- a lane row
// or an extra row held by a lane pair -- is stored once.  Everything else
// (staging build, pipelined pivot search, U in shared memory, register
// back-substitution, HYBRID criterion) follows phs_reg.cuh / phs_mma.cuh.
#pragma once

#include "phs_mma.cuh"

namespace mf {

template <int NN, int DEG, int DD, int NF>
struct SplitCfg {
    static constexpr int LL = binom(DEG + DD, DD);
    static constexpr int S = NN + LL;
    static constexpr int NR = NF + 1;  // + probe
    static constexpr int C = S + NR;
    static constexpr int CP = (C + 1) & ~1;
    static constexpr int H = (C + 1) / 2;  // columns per extra-row half
    static constexpr int EX = S - 32;      // extra rows
    static constexpr int R = 2;            // back-substitution rows per lane
    static constexpr int WARPS = 2;        // small blocks: 5 per SM at <= 204 registers
    static constexpr int U_DBL = S * CP;
    static constexpr int LOC_DBL = ((NN * DD + 1) & ~1);
    static constexpr int RHS_DBL = ((S * NR + 1) & ~1);
    static constexpr int WARP_DBL = U_DBL + LOC_DBL + RHS_DBL;
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DBL * sizeof(double);
    static_assert(S > 32 && S <= 64, "split kernel covers 32 < S <= 64");
    static_assert(S * NN <= U_DBL, "staging matrix must fit in U");
};

// A[r][c] of the staged system (E: PHS block + Q^T, Rs: right-hand sides)
template <int NN, int S, int NR, int C>
__device__ __forceinline__ double staged_entry(const double* E, const double* Rs, int r, int c) {
    if (r >= S || c >= C) return 0.0;
    if (c < NN) return E[r * NN + c];
    if (c < S) return r < NN ? E[c * NN + r] : 0.0;
    return Rs[r * NR + (c - S)];
}

template <int NN, int DEG, int DD, int NF>
__global__ void __maxnreg__(255) phs_split(PhsArgs a) {
    using Cfg = SplitCfg<NN, DEG, DD, NF>;
    constexpr int LL = Cfg::LL, S = Cfg::S, NR = Cfg::NR, C = Cfg::C, CP = Cfg::CP, H = Cfg::H, R = Cfg::R;
    extern __shared__ __align__(16) double smem_s[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int half = lane & 1;
    const int xrow = 32 + (lane >> 1);  // extra row held (in part) by this lane
    const bool has_x = xrow < S;
    double* U = smem_s + (size_t)wib * Cfg::WARP_DBL;
    double* E = U;
    double* loc = U + Cfg::U_DBL;
    double* Rs = loc + Cfg::LOC_DBL;
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

        // ---- lane row (all columns) and extra-row half (H columns)
        double A0[C], X[H];
        double rowsum0 = 0.0, rowsumx = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            A0[c] = staged_entry<NN, S, NR, C>(E, Rs, lane, c);
            if (c < S) rowsum0 += fabs(A0[c]);
        }
#pragma unroll
        for (int c = 0; c < H; ++c) {
            const int cc = half * H + c;
            X[c] = has_x ? staged_entry<NN, S, NR, C>(E, Rs, xrow, cc) : 0.0;
            if (cc < S) rowsumx += fabs(X[c]);
        }
        __syncwarp();  // staging is dead; U takes its place
        double anorm = 0.0;
        if (want_est) {
            rowsumx += __shfl_xor_sync(FULL, rowsumx, 1);
            anorm = fmax(rowsum0, rowsumx);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) anorm = fmax(anorm, __shfl_xor_sync(FULL, anorm, o));
        }

        // ---- pipelined elimination with partial pivoting
        bool ok = stat == 0;
        bool live0 = lane < S, livex = has_x;
        double fac0 = 0.0, facx = 0.0;
#pragma unroll
        for (int col = 0; col < S; ++col) {
            constexpr int dummy = 0;
            (void)dummy;
            // (1) candidates: this lane's row, and its extra row if it holds column col
            const bool xhold = (col < H) ? (half == 0) : (half == 1);
            const double vx = (col < H) ? X[col < H ? col : 0] : X[col >= H ? col - H : 0];
            const double v0 = A0[col];
            const double a0 = live0 ? fabs(v0) : -1.0;
            const double ax_ = (livex && xhold) ? fabs(vx) : -1.0;
            const bool takex = ax_ > a0;
            const double best = takex ? ax_ : a0;
            const double cval = takex ? vx : v0;
            const double cinv = fast_rcp(best >= 0.0 ? cval : 1.0);
            const unsigned hk = best >= 0.0 ? (unsigned)((unsigned long long)__double_as_longlong(best) >> 32) : 0u;
            const unsigned mh = __reduce_max_sync(FULL, hk);
            // (2) bulk rank-1 update of the previous step (columns col+1..), overlapping the search
            if (col > 0) {
                const double* up = U + (col - 1) * CP;
#pragma unroll
                for (int c2 = (col + 1) & ~1; c2 < CP; c2 += 2) {
                    const double2 u = *reinterpret_cast<const double2*>(up + c2);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int c = c2 + hh;
                        if (c > col && c < C) {
                            const double uc = hh ? u.y : u.x;
                            A0[c] = fma(-fac0, uc, A0[c]);
                            if (c < H) {
                                if (half == 0) X[c < H ? c : 0] = fma(-facx, uc, X[c < H ? c : 0]);
                            } else {
                                if (half == 1) X[c >= H ? c - H : 0] = fma(-facx, uc, X[c >= H ? c - H : 0]);
                            }
                        }
                    }
                }
            }
            // (3) finish the search
            const unsigned ball = __ballot_sync(FULL, best >= 0.0 && hk == mh);
            ok = ok && ball != 0u && mh != 0u;
            const int wl = (__ffs(ball) - 1) & 31;
            const double inv = __shfl_sync(FULL, cinv, wl);
            const bool px = __shfl_sync(FULL, takex, wl);  // pivot is an extra row
            // (4) pivot row -> U[col][col..]
            double* urow = U + col * CP;
            if (!px) {
                const bool owner = lane == wl && ball != 0u;
#pragma unroll
                for (int c = col & ~1; c < CP; c += 2)
                    st_shared_v2_if(owner, urow + c, c < C ? A0[c] : 0.0, c + 1 < C ? A0[c + 1] : 0.0);
                live0 = live0 && !owner;
            } else {
                const bool owner = (lane >> 1) == (wl >> 1) && ball != 0u;
                // half 0 holds [0, H), half 1 holds [H, C); H is even-aligned below
#pragma unroll
                for (int c = col & ~1; c < CP; c += 2) {
                    if (c + 1 < H) {
                        st_shared_v2_if(owner && half == 0, urow + c, X[c], X[c + 1]);
                    } else if (c >= H) {
                        st_shared_v2_if(owner && half == 1, urow + c, c - H < H ? X[c - H < H ? c - H : 0] : 0.0,
                                        c + 1 - H < H && c + 1 < C ? X[c + 1 - H < H ? c + 1 - H : 0] : 0.0);
                    } else {  // c == H - 1: columns H-1 (half 0) and H (half 1)
                        if (owner && half == 0) urow[c] = X[H - 1];
                        if (owner && half == 1) urow[c + 1] = X[0];
                    }
                }
                livex = livex && !owner;
            }
            // (5) multipliers; early update of column col+1 (next pivot column)
            fac0 = v0 * inv;
            const double fmine = vx * inv;
            const double fother = __shfl_xor_sync(FULL, fmine, 1);
            facx = xhold ? fmine : fother;
            __syncwarp();
            if (col + 1 < S) {
                const double u1 = urow[col + 1];
                A0[col + 1] = fma(-fac0, u1, A0[col + 1]);
                constexpr int dummy2 = 0;
                (void)dummy2;
                if (col + 1 < H) {
                    if (half == 0) X[col + 1 < H ? col + 1 : 0] = fma(-facx, u1, X[col + 1 < H ? col + 1 : 0]);
                } else {
                    if (half == 1) X[col + 1 >= H ? col + 1 - H : 0] = fma(-facx, u1, X[col + 1 >= H ? col + 1 - H : 0]);
                }
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
        // ---- outputs, non-finite check, HYBRID criterion
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
int launch_split(const PhsArgs& a, cudaStream_t st, int sms) {
    using Cfg = SplitCfg<NN, DEG, DD, NF>;
    constexpr GradedLex<DD, DEG> gl{};
    if (a.P.l != Cfg::LL) return MF_ERR_UNSUPPORTED;
    for (int m = 0; m < Cfg::LL; ++m)
        for (int ax = 0; ax < DD; ++ax)
            if (a.P.expos[m * DD + ax] != gl.e[m][ax]) return MF_ERR_UNSUPPORTED;
    auto kern = phs_split<NN, DEG, DD, NF>;
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

#define MF_INSTANTIATE_SPLIT(NN, DEG, DD, NF) \
    template int launch_split<NN, DEG, DD, NF>(const PhsArgs&, cudaStream_t, int);

}  // namespace mf

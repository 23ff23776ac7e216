// Nullspace shape solve: the HYBRID first pass for the hot stencil shapes (sm_100a).
//
// The saddle-point system [Phi Q; Q^T 0][w; lambda] = [f; g] of one stencil
// (_phs_batch.py:228-290) is solved on the nullspace of Q^T instead of by a
// pivoted LU of the whole (n+l)^2 matrix:
//   1. LU with partial pivoting of Q over the nodes picks l pivot nodes,
//      P Q = [L1; L2] U1 (l sequential steps of width l);
//   2. W = L2 L1^-1 maps the free (non-pivot) weights v to the pivot weights,
//      w_piv = w1p - W^T v with the particular solution w1p = L1^-T U1^-T g;
//   3. the reduced matrix K = Z^T Phi Z (Z = [-W^T; I], (n-l)^2) is symmetric
//      and definite for a polyharmonic kernel whose order the polynomial degree
//      covers (conditional positive definiteness), so it is factored by a
//      pivot-free Gauss-Jordan elimination: at step k every lane stores its
//      column-k entry once and reads the pivot row back as 16-byte broadcasts;
//   4. v solves K v = Z^T (f - Phi w_p), and w = w_p + Z v.
// One warp per stencil; lane c owns reduced row c (n - l <= 32) in registers
// and ends with its own unknown, v_c = b_c / d_c (no back-substitution).  The +-1 probe rides along
// as one more right-hand side, and the family multipliers lambda (for the
// sensitivity estimate) come from Q1 lambda = (f - Phi w)_piv.  Rounding differs from the reference's LU;
// HYBRID re-solves, in the reference's order, the rows the LU FAST kernel would
// flag (near-coincident nodes, sensitivity estimate) plus any row whose reduced
// pivots lose definiteness.
#pragma once

#include "phs_reg.cuh"

namespace mf {

__host__ __device__ constexpr int ns_even(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int ns_max(int a, int b) { return a > b ? a : b; }

template <int NN, int DEG, int DD, int NF>
struct NsCfg {
    static constexpr int LL = binom(DEG + DD, DD);
    static constexpr int LLP = ns_even(LL);  // row pitch of W / Y (16-byte aligned rows)
    static constexpr int M = NN - LL;        // reduced (nullspace) system size
    static constexpr int MP = ns_even(M);
    static constexpr int NR = NF + 1;        // families + probe
    static constexpr int RN = (NN + 31) / 32;
    static constexpr int RW = LL * NR + LL * NF;  // per-lane products reduced for w_piv and lambda
    static constexpr int WARPS = 4;
    // per-warp shared layout (doubles); E hosts Phi, then the elimination rows, then the reductions
    static constexpr int E_DBL = ns_even(ns_max(NN * NN, ns_max(M * MP + M * NR, M * RW + RW)));
    static constexpr int QU_DBL = ns_even(LL * LL);
    static constexpr int QL_DBL = ns_even(LL * LL);
    static constexpr int W_DBL = M * LLP;
    static constexpr int Y_DBL = M * LLP;
    static constexpr int F_DBL = ns_even(NN * NR);
    static constexpr int V_DBL = ns_even(2 * LL * NR + LL);  // + 1/U1[k][k]
    static constexpr int LOC_DBL = ns_even(NN * DD);
    static constexpr int IDX_DBL = ns_even((NN + 1) / 2);
    static constexpr int WARP_DBL = E_DBL + QU_DBL + QL_DBL + W_DBL + Y_DBL + F_DBL + V_DBL + LOC_DBL + IDX_DBL;
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DBL * sizeof(double);
    static_assert(M >= 1 && M <= 32, "the reduced system must fit one warp");
    static_assert(RN <= 2, "at most 64 stencil nodes");
};

// D = a x b + D on the fp64 tensor core (m8n8k4, row.col): lane holds A[g][t4],
// B[t4][g] and D[g][2 t4 .. 2 t4 + 1] with g = lane / 4, t4 = lane % 4
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

template <int DD, int DEG, int MM, int LL>
__device__ __forceinline__ void monomials_reg(double (&q)[LL], const double* x) {
    if constexpr (MM < LL) {
        q[MM] = monomial_ct<DD, DEG, MM>(x);
        monomials_reg<DD, DEG, MM + 1, LL>(q, x);
    }
}

template <int NN, int DEG, int DD, int NF>
__global__ void __launch_bounds__(128, 3) phs_ns(PhsArgs a) {
    using Cfg = NsCfg<NN, DEG, DD, NF>;
    constexpr int LL = Cfg::LL, LLP = Cfg::LLP, M = Cfg::M, MP = Cfg::MP, NR = Cfg::NR, RN = Cfg::RN,
                  RW = Cfg::RW;
    extern __shared__ __align__(16) double smem_n[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double* E = smem_n + (size_t)wib * Cfg::WARP_DBL;
    double* QU = E + Cfg::E_DBL;     // U1 row k at k*LL (entries k..)
    double* QL = QU + Cfg::QU_DBL;   // L1 row k at k*LL (entries ..k-1)
    double* Wm = QL + Cfg::QL_DBL;   // L2 rows, then W rows (row c at c*LLP)
    double* Ym = Wm + Cfg::W_DBL;    // Y column c at c*LLP: Y[k][c] = (Phi Z)[p_k][c]
    double* F = Ym + Cfg::Y_DBL;     // node rhs: F[i*NR + f]
    double* V = F + Cfg::F_DBL;      // w1p[k][f] at k*NR+f, r_piv at LL*NR + k*NR + f
    double* QD = V + 2 * LL * NR;    // 1/U1[k][k]
    double* loc = V + Cfg::V_DBL;
    int* IDX = reinterpret_cast<int*>(loc + Cfg::LOC_DBL);  // pivot nodes, then non-pivot nodes
    // HYBRID only (launch_ns): the flag list and the estimate are always wanted
    constexpr bool want_flag = true, want_est = true;
    const PhsParams& P = a.P;
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool act = lane < M;

    for (int t = lane; t < NN; t += 32) IDX[t] = 0;  // every table entry is a valid node from here on
    __syncwarp();

#pragma unroll 1
    for (int64_t idx = (int64_t)blockIdx.x * Cfg::WARPS + wib; idx < a.m; idx += (int64_t)gridDim.x * Cfg::WARPS) {
        const int64_t row = a.rows[idx];
        const int32_t* sti = a.stencils + idx * NN;
        int stat;
        bool k3;
        double facs[NF], r2min, rc2max;
        phs_stage<NN, DD, NF, false, true>(a, row, sti, lane, E, loc, stat, facs, r2min, rc2max, k3);

        // ---- own nodes: Q rows (monomials) and node right-hand sides
        double q[RN][LL];
        bool live[RN];
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int i = lane + 32 * s;
            live[s] = i < NN;
            const int ic = live[s] ? i : 0;
            monomials_reg<DD, DEG, 0, LL>(q[s], loc + ic * DD);
            if (live[s]) {
                double top[MF_MAX_FAMILIES];
                phs_rhs_top_k3(loc + ic * DD, DD, P, top);
#pragma unroll
                for (int f = 0; f < NF; ++f) F[ic * NR + f] = __dmul_rn(top[f], facs[f]);
                F[ic * NR + NF] = probe_sign(idx, ic);
            } else {
#pragma unroll
                for (int m = 0; m < LL; ++m) q[s][m] = 0.0;
            }
        }
        __syncwarp();

        // ---- ||A||_inf of the full saddle-point matrix (estimate only)
        double anorm = 0.0;
        if (want_est) {
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                if (live[s]) {
                    const int i = lane + 32 * s;
                    double acc = 0.0;
                    for (int j = 0; j < NN; ++j) acc += fabs(E[j * NN + i]);  // column i == row i
#pragma unroll
                    for (int m = 0; m < LL; ++m) acc += fabs(q[s][m]);
                    anorm = fmax(anorm, acc);
                }
            }
            if (P.scale_code == MF_SCALE_SUPPORT) {
                // constraint rows sum |Q_im| over the nodes: the constant column gives
                // exactly n and every other monomial of |x| <= 1 is at most 1
                anorm = fmax(anorm, (double)NN);
            } else {
#pragma unroll
                for (int m = 0; m < LL; ++m) {
                    double cs = 0.0;
#pragma unroll
                    for (int s = 0; s < RN; ++s) cs += fabs(q[s][m]);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(FULL, cs, o);
                    anorm = fmax(anorm, cs);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) anorm = fmax(anorm, __shfl_xor_sync(FULL, anorm, o));
        }

        // ---- (1) LU with partial pivoting of Q over the nodes
        bool ok = stat == 0;
#pragma unroll
        for (int k = 0; k < LL; ++k) {
            double best = -1.0, cval = 1.0;
            int bslot = 0;
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                const double v = live[s] ? fabs(q[s][k]) : -1.0;
                const bool t = v > best;
                best = t ? v : best;
                cval = t ? q[s][k] : cval;
                bslot = t ? s : bslot;
            }
            const unsigned hk = best >= 0.0 ? (unsigned)((unsigned long long)__double_as_longlong(best) >> 32) : 0u;
            const unsigned mh = __reduce_max_sync(FULL, hk);
            const unsigned ball = __ballot_sync(FULL, best >= 0.0 && hk == mh);
            ok = ok && ball != 0u && mh != 0u;
            const int wl = (__ffs(ball) - 1) & 31;
            const double inv = __shfl_sync(FULL, fast_rcp(cval), wl);
            QD[k] = inv;  // every lane stores the same value
            const int ps = __shfl_sync(FULL, bslot, wl);
            if (lane == wl) {
#pragma unroll
                for (int s = 0; s < RN; ++s) {
                    if (s == ps) {
#pragma unroll
                        for (int m = 0; m < LL; ++m) {
                            if (m < k) QL[k * LL + m] = q[s][m];
                            else QU[k * LL + m] = q[s][m];
                        }
                        live[s] = false;
                        IDX[k] = lane + 32 * s;
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                const double l = live[s] ? q[s][k] * inv : 0.0;
                q[s][k] = live[s] ? l : q[s][k];
#pragma unroll
                for (int m = k + 1; m < LL; ++m) q[s][m] = fma(-l, QU[k * LL + m], q[s][m]);
            }
        }
        // non-pivot nodes in lane order -> reduced index c; their L2 rows -> Wm
        {
            int base = 0;
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                const unsigned bm = __ballot_sync(FULL, live[s]);
                const int c = base + __popc(bm & lt_mask);
                if (live[s] && c < M) {
                    IDX[LL + c] = lane + 32 * s;
#pragma unroll
                    for (int m = 0; m < LL; ++m) Wm[c * LLP + m] = q[s][m];
                }
                base += __popc(bm);
            }
            ok = ok && base == M;
        }
        __syncwarp();

        // ---- (2) W row of lane c: x L1 = l  (L1 unit lower, L1[j][k] = QL[j*LL + k])
        const int cc = act ? lane : 0;
        const int qn = IDX[LL + cc];
        int pv[LL];
#pragma unroll
        for (int k = 0; k < LL; ++k) pv[k] = IDX[k];
        double wr[LL];
#pragma unroll
        for (int m = 0; m < LL; ++m) wr[m] = Wm[cc * LLP + m];
#pragma unroll
        for (int k = LL - 2; k >= 0; --k) {
#pragma unroll
            for (int j = k + 1; j < LL; ++j) wr[k] = fma(-wr[j], QL[j * LL + k], wr[k]);
        }
        double phq[LL];  // Phi[q_c][p_k]
#pragma unroll
        for (int k = 0; k < LL; ++k) phq[k] = E[qn * NN + pv[k]];
        __syncwarp();  // every L2 row is read before the W rows replace them
        if (act) {
#pragma unroll
            for (int m = 0; m < LL; ++m) Wm[lane * LLP + m] = wr[m];
        }

        // ---- particular solution w1p = L1^-T U1^-T g, per right-hand side (uniform)
        double w1p[LL][NR];
#pragma unroll
        for (int k = 0; k < LL; ++k) {
#pragma unroll
            for (int f = 0; f < NF; ++f) w1p[k][f] = __dmul_rn(P.base_bot[f * MF_MAX_MONOMIALS + k], facs[f]);
            w1p[k][NF] = probe_sign(idx, NN + k);
#pragma unroll
            for (int j = 0; j < k; ++j) {
                const double u = QU[j * LL + k];
#pragma unroll
                for (int f = 0; f < NR; ++f) w1p[k][f] = fma(-u, w1p[j][f], w1p[k][f]);
            }
            const double di = QD[k];
#pragma unroll
            for (int f = 0; f < NR; ++f) w1p[k][f] *= di;
        }
#pragma unroll
        for (int k = LL - 2; k >= 0; --k) {
#pragma unroll
            for (int j = k + 1; j < LL; ++j) {
                const double l = QL[j * LL + k];
#pragma unroll
                for (int f = 0; f < NR; ++f) w1p[k][f] = fma(-l, w1p[j][f], w1p[k][f]);
            }
        }

        // ---- (3) Y column of lane c and r_piv = (f - Phi w_p)_piv (uniform)
        double bb[NR];
#pragma unroll
        for (int f = 0; f < NR; ++f) {
            double r = F[qn * NR + f];
#pragma unroll
            for (int k = 0; k < LL; ++k) r = fma(-phq[k], w1p[k][f], r);
            bb[f] = r;  // r at the non-pivot node q_c
        }
        __syncwarp();  // W rows visible
        // Y = Phi12 - Phi11 W^T (l x m) on the fp64 tensor core; fragments straight
        // from Phi (through the pivot / free node table) and the W rows
        {
            constexpr int LT = (LL + 7) / 8, MT = (M + 7) / 8, KS = (LL + 3) / 4;
            const int g = lane >> 2, t4 = lane & 3;
            int pr[LT];
#pragma unroll
            for (int lt = 0; lt < LT; ++lt) pr[lt] = IDX[min(lt * 8 + g, LL - 1)];
            double acc[LT][MT][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int c = mt * 8 + 2 * t4 + h;
                    const int qc = IDX[LL + min(c, M - 1)];
#pragma unroll
                    for (int lt = 0; lt < LT; ++lt) {
                        const double v = E[pr[lt] * NN + qc];
                        acc[lt][mt][h] = (lt * 8 + g < LL && c < M) ? v : 0.0;
                    }
                }
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int k2 = ks * 4 + t4;
                const bool k2v = k2 < LL;
                const int pk2 = IDX[min(k2, LL - 1)];
                double af[LT], bf[MT];
#pragma unroll
                for (int lt = 0; lt < LT; ++lt) {
                    const double v = E[pr[lt] * NN + pk2];
                    af[lt] = (k2v && lt * 8 + g < LL) ? -v : 0.0;
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int c = mt * 8 + g;
                    const double v = Wm[min(c, M - 1) * LLP + min(k2, LL - 1)];
                    bf[mt] = (k2v && c < M) ? v : 0.0;
                }
#pragma unroll
                for (int lt = 0; lt < LT; ++lt)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) dmma_f64(acc[lt][mt][0], acc[lt][mt][1], af[lt], bf[mt]);
            }
#pragma unroll
            for (int lt = 0; lt < LT; ++lt) {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int k = lt * 8 + g, c = mt * 8 + 2 * t4 + h;
                        if (k < LL && c < M) Ym[c * LLP + k] = acc[lt][mt][h];
                    }
                }
            }
        }
        {
            // r_piv[k] = f(p_k) - Phi[p_k][piv] w1p, one pivot per lane
            const int kk = lane < LL ? lane : 0;
            const int pk = IDX[kk];
            double rr[NR];
#pragma unroll
            for (int f = 0; f < NR; ++f) rr[f] = F[pk * NR + f];
#pragma unroll
            for (int k2 = 0; k2 < LL; ++k2) {
                const double ph = E[pk * NN + pv[k2]];
#pragma unroll
                for (int f = 0; f < NR; ++f) rr[f] = fma(-ph, w1p[k2][f], rr[f]);
            }
            if (lane < LL) {
#pragma unroll
                for (int f = 0; f < NR; ++f) V[LL * NR + lane * NR + f] = rr[f];
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < LL; ++k)
#pragma unroll
                for (int f = 0; f < NR; ++f) V[k * NR + f] = w1p[k][f];
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < LL; ++k)
#pragma unroll
            for (int f = 0; f < NR; ++f) bb[f] = fma(-wr[k], V[LL * NR + k * NR + f], bb[f]);  // r_c - W r_piv

        // ---- (4) reduced matrix K = Phi22 - [H W] [W^T; Y] (H = Phi21) on the fp64
        //      tensor core, then one row per lane through shared memory
        __syncwarp();  // Y columns visible
        double K[M];
        {
            constexpr int MT = (M + 7) / 8, KS = (2 * LL + 3) / 4, KP = MP;
            const int g = lane >> 2, t4 = lane & 3;
            int qr[MT];
#pragma unroll
            for (int rt = 0; rt < MT; ++rt) qr[rt] = IDX[LL + min(rt * 8 + g, M - 1)];
            double acc[MT][MT][2];
#pragma unroll
            for (int ct = 0; ct < MT; ++ct) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int c2 = ct * 8 + 2 * t4 + h;
                    const int qc = IDX[LL + min(c2, M - 1)];
#pragma unroll
                    for (int rt = 0; rt < MT; ++rt) {
                        const double v = E[qr[rt] * NN + qc];
                        acc[rt][ct][h] = (rt * 8 + g < M && c2 < M) ? v : 0.0;
                    }
                }
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int kk = ks * 4 + t4;  // < LL: H column kk, else W / Y row kk - LL
                const bool hp = kk < LL, kv = kk < 2 * LL;
                const int kh = min(kk, LL - 1), kw = min(max(kk - LL, 0), LL - 1);
                const int pk = IDX[kh];
                double af[MT], bf[MT];
#pragma unroll
                for (int rt = 0; rt < MT; ++rt) {
                    const int c = rt * 8 + g;
                    const double vh = E[qr[rt] * NN + pk];
                    const double vw = Wm[min(c, M - 1) * LLP + kw];
                    af[rt] = (c < M && kv) ? -(hp ? vh : vw) : 0.0;
                }
#pragma unroll
                for (int ct = 0; ct < MT; ++ct) {
                    const int c2 = min(ct * 8 + g, M - 1);
                    const double vw = Wm[c2 * LLP + kh];
                    const double vy = Ym[c2 * LLP + kw];
                    bf[ct] = (ct * 8 + g < M && kv) ? (hp ? vw : vy) : 0.0;
                }
#pragma unroll
                for (int rt = 0; rt < MT; ++rt)
#pragma unroll
                    for (int ct = 0; ct < MT; ++ct) dmma_f64(acc[rt][ct][0], acc[rt][ct][1], af[rt], bf[ct]);
            }
            __syncwarp();  // every read of Phi is done: K takes its place
            double* Ks = E;
#pragma unroll
            for (int rt = 0; rt < MT; ++rt) {
#pragma unroll
                for (int ct = 0; ct < MT; ++ct) {
                    const int c = rt * 8 + g, c2 = ct * 8 + 2 * t4;
                    if (c < M && c2 < M) {
                        if (c2 + 1 < KP) {
                            *reinterpret_cast<double2*>(Ks + c * KP + c2) = make_double2(acc[rt][ct][0], acc[rt][ct][1]);
                        } else {
                            Ks[c * KP + c2] = acc[rt][ct][0];
                        }
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < M; ++j) K[j] = Ks[cc * KP + j];
        }
        __syncwarp();  // E (Phi) is dead from here on

        // ---- (5) pivot-free Gauss-Jordan on [K | b]; lane c keeps row c in registers
        double* Us = E;
        double* Bs = E + M * MP;
        double dinv_own = 0.0, d0 = 0.0;
        bool definite = true;
#pragma unroll
        for (int k = 0; k < M; ++k) {
            if (act) Us[k * MP + lane] = K[k];
            if (lane == k) {
#pragma unroll
                for (int f = 0; f < NR; ++f) Bs[k * NR + f] = bb[f];
            }
            __syncwarp();
            const double* urow = Us + k * MP;
            const double dk = urow[k];
            const double rk = fast_rcp(dk);
            if (k == 0) d0 = dk;
            dinv_own = lane == k ? rk : dinv_own;
            // Gauss-Jordan: rows above the pivot are eliminated too (those lanes issue
            // the FMAs anyway), so no back-substitution follows
            const double fac = lane != k ? K[k] * rk : 0.0;
#pragma unroll
            for (int j = k + 1; j < M; ++j) K[j] = fma(-fac, urow[j], K[j]);
#pragma unroll
            for (int f = 0; f < NR; ++f) bb[f] = fma(-fac, Bs[k * NR + f], bb[f]);
        }
#pragma unroll
        for (int f = 0; f < NR; ++f) bb[f] *= dinv_own;  // v_c = b_c / d_c
        __syncwarp();

        // ---- (6) outputs: free weights v (lanes c < M), pivot weights w1p - W^T v
        definite = __all_sync(FULL, !act || dinv_own * d0 > 0.0);
        bool bad = !ok || !definite;
        double* Red = E;
        if (act) {
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                bad |= !isfinite(bb[f]);
                a.out[((size_t)idx * NF + f) * NN + qn] = bb[f];
            }
#pragma unroll
            for (int k = 0; k < LL; ++k) {
                const double y = Ym[lane * LLP + k];
#pragma unroll
                for (int f = 0; f < NR; ++f) {
                    Red[lane * RW + k * NR + f] = wr[k] * bb[f];
                    if (f < NF) Red[lane * RW + LL * NR + k * NF + f] = y * bb[f];
                }
            }
        }
        __syncwarp();
        for (int t = lane; t < RW; t += 32) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < M; ++c) s += Red[c * RW + t];
            Red[M * RW + t] = s;
        }
        __syncwarp();
        const double* sums = Red + M * RW;
        double zw = 0.0, xw[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) xw[f] = act ? fabs(bb[f]) : 0.0;
        if (act) zw = fabs(bb[NF]);
        if (lane < LL) {
            const int pn = IDX[lane];
#pragma unroll
            for (int f = 0; f < NR; ++f) {
                const double w = V[lane * NR + f] - sums[lane * NR + f];
                if (f < NF) {
                    bad |= !isfinite(w);
                    a.out[((size_t)idx * NF + f) * NN + pn] = w;
                    xw[f] = fmax(xw[f], fabs(w));
                } else {
                    zw = fmax(zw, fabs(w));
                }
            }
        }
        if (__any_sync(FULL, bad) && stat == 0) stat = 1;

        if (want_est) {
            // lambda (family columns) from Q1 lambda = r_piv - Y v (L1 then U1, uniform)
            double lam[LL][NF];
#pragma unroll
            for (int k = 0; k < LL; ++k) {
#pragma unroll
                for (int f = 0; f < NF; ++f) lam[k][f] = V[LL * NR + k * NR + f] - sums[LL * NR + k * NF + f];
#pragma unroll
                for (int j = 0; j < k; ++j) {
                    const double l = QL[k * LL + j];
#pragma unroll
                    for (int f = 0; f < NF; ++f) lam[k][f] = fma(-l, lam[j][f], lam[k][f]);
                }
            }
            double la[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) la[f] = 0.0;
#pragma unroll
            for (int k = LL - 1; k >= 0; --k) {
#pragma unroll
                for (int j = k + 1; j < LL; ++j) {
                    const double u = QU[k * LL + j];
#pragma unroll
                    for (int f = 0; f < NF; ++f) lam[k][f] = fma(-u, lam[j][f], lam[k][f]);
                }
                const double di = QD[k];
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    lam[k][f] *= di;
                    la[f] = fmax(la[f], fabs(lam[k][f]));
                }
            }
            double sep2 = r2min;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                zw = fmax(zw, __shfl_xor_sync(FULL, zw, o));
                sep2 = fmin(sep2, __shfl_xor_sync(FULL, sep2, o));
                rc2max = fmax(rc2max, __shfl_xor_sync(FULL, rc2max, o));
#pragma unroll
                for (int f = 0; f < NF; ++f) xw[f] = fmax(xw[f], __shfl_xor_sync(FULL, xw[f], o));
            }
            double ratio = 0.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) ratio = fmax(ratio, fmax(xw[f], la[f]) / xw[f]);
            const double est = anorm * zw * ratio;
            const bool close = sep2 < a.min_sep2 * rc2max;
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

// HYBRID only (rows that lose definiteness are re-solved), and only where the
// kernel's order is covered by the polynomial degree.
template <int NN, int DEG, int DD, int NF>
int launch_ns(const PhsArgs& a, cudaStream_t st, int sms) {
    using Cfg = NsCfg<NN, DEG, DD, NF>;
    constexpr GradedLex<DD, DEG> g{};
    // (per-row kappa diagnostics come from the LU kernel)
    if (!a.flag_list || a.kappa || a.P.l != Cfg::LL || a.P.nf != NF) return MF_ERR_UNSUPPORTED;
    for (int m = 0; m < Cfg::LL; ++m)
        for (int ax = 0; ax < DD; ++ax)
            if (a.P.expos[m * DD + ax] != g.e[m][ax]) return MF_ERR_UNSUPPORTED;
    // r^3 (conditionally positive definite of order 2: the reduced matrix is
    // definite for degree >= 1); other kernels take the LU path
    if (a.P.k != 3 || a.P.even || DEG < 1) return MF_ERR_UNSUPPORTED;
    auto kern = phs_ns<NN, DEG, DD, NF>;
    MF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    int per_sm = 0;
    MF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::WARPS * 32, Cfg::SMEM));
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (a.m + Cfg::WARPS - 1) / Cfg::WARPS;
    const int64_t cap = (int64_t)sms * per_sm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, Cfg::WARPS * 32, Cfg::SMEM, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

#define MF_INSTANTIATE_NS(NN, DEG, DD, NF) template int launch_ns<NN, DEG, DD, NF>(const PhsArgs&, cudaStream_t, int);

}  // namespace mf

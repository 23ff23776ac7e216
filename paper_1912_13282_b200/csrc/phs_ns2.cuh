// Nullspace shape solve, pivots-first layout: the HYBRID first pass for the hot
// stencil shapes (sm_100a).  Mathematics in phs_nullspace.cuh (nullspace of
// Q^T, pivot-free Gauss-Jordan on the reduced definite system); one warp per
// stencil, and the work is ordered so that every phase has instruction-level
// parallelism and regular shared memory addressing:
//
//   0. the next stencil's node positions are staged with cp.async while the
//      current one is solved (the index -> position gather is two dependent
//      global loads; issuing them one stencil ahead takes them off the chain);
//   1. local coordinates, scale (warp max by two REDUX on the IEEE bits),
//      monomials and node right-hand sides in registers, one node per lane
//      (nodes 32.. ride in a second slot of lanes 0..);
//   2. LU with partial pivoting of Q over the lane-resident nodes (one REDUX
//      per step picks value and lane at once; nodes 32.. are never pivots, so
//      the pivot search is one compare per lane);
//   3. the PHS block Phi is evaluated AFTER the pivots are known, directly in
//      the order [pivot nodes; free nodes], so the blocks Phi11, Phi12, Phi22
//      are contiguous and the tensor-core fragments for Y = Phi12 - Phi11 W^T
//      and K = Phi22 - [H W][W^T; Y] are plain strided loads;
//   4. every triangular solve (W, the particular solution, lambda) runs in
//      right-looking order, whose dependency chain is one FMA per level;
//   5. W^T v and Y v (pivot weights and the estimate's multipliers) are one
//      small tensor-core product instead of a shared-memory reduction.
//
// Rounding differs from the reference's LU (phs_nullspace.cuh); the HYBRID flags (near-coincident nodes, sensitivity estimate, failed or
// indefinite reduction, non-finite weights) are the same.
#pragma once

#include "phs_nullspace.cuh"

namespace mf {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 1/x from the MUFU seed (high word, ~2^-22) by one cubically convergent step:
// r (1 + e + e^2), e = 1 - x r
__device__ __forceinline__ double rcp_c3(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}
// 1/sqrt(x), x > 0, likewise: y (1 + e/2 + 3 e^2 / 8), e = 1 - x y^2
__device__ __forceinline__ double rsqrt_c3(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

// warp max of a non-negative double (or +0 for lanes that do not take part):
// the IEEE bit pattern of non-negative doubles is ordered like the values
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_max_sync(FULL, hi);
    const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}
// warp min of a non-negative double (+inf for lanes that do not take part)
__device__ __forceinline__ double warp_min_nonneg(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_min_sync(FULL, hi);
    const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}

// smallest pitch >= x that is 4 mod 8 doubles: the tensor-core fragment loads
// (8 rows g x 4 columns t, or 4 rows x 8 columns) then hit 16 distinct 8-byte
// bank pairs per half warp
__host__ __device__ constexpr int ns_pitch(int x) { return x % 8 <= 4 ? x + (4 - x % 8) : x + (12 - x % 8); }

template <int NN, int DEG, int DD, int NF>
struct Ns2Cfg {
    static constexpr int LL = binom(DEG + DD, DD);
    static constexpr int M = NN - LL;           // reduced system size
    static constexpr int MP = ns_even(M);       // elimination row pitch
    static constexpr int NR = NF + 1;           // families + probe
    static constexpr int RN = (NN + 31) / 32;   // node slots per lane
    static constexpr int XN = NN - 32 > 0 ? NN - 32 : 0;  // nodes in slot 1
    static constexpr int NP = ns_even(NN);      // pitch of the coordinate arrays
    static constexpr int P = ns_pitch(NN + 1);  // Phi row pitch
    static constexpr int LP = ns_pitch(LL);     // W / Y row pitch
    static constexpr int WARPS = 4;
    // per-warp shared layout (doubles)
    static constexpr int UP = ns_even(M + 1);   // Gauss-Jordan column pitch
    static constexpr int KTP = (M + NR <= 16 && M <= 16) ? 20 : 36;  // [K | b] staging pitch (4 mod 16 doubles)
    static constexpr int PH_DBL = ns_even(ns_max(ns_max(NN * P, M * UP + M * (NR + 1)), M * KTP));
    static constexpr int XS_DBL = ns_even(DD * NP + DD);  // scaled coords (permuted), then the staged raw positions
    static constexpr int NC = NN + NR + LL;     // columns of [Q^T | g | I] in the Gauss-Jordan sweep
    static constexpr int CS = (NC + 31) / 32;   // column slots per lane
    static constexpr int QLU_DBL = ns_even(LL * LL + 2 * (LL + 1));  // rows of Q1^-1, then two pivot-column buffers
    static constexpr int W_DBL = M * LP;
    static constexpr int Y_DBL = (M + NR) * LP;  // Y columns, then the pivot residuals (rows M..)
    static constexpr int F_DBL = ns_even(NN * NR + NN);   // node rhs (permuted) + |Q| row sums
    static constexpr int V_DBL = ns_even(3 * LL * NR + M * NR);  // w1p, r_piv, lambda rhs, v
    static constexpr int IDX_DBL = ns_even((NN + 1) / 2);
    static constexpr int IB_ROW = 2 * ns_even((NN + 1) / 2);  // int offset of the staged row index (8-byte aligned)
    static constexpr int IB_DBL = IB_ROW / 2 + 2;
    static constexpr int WARP_DBL = PH_DBL + XS_DBL + QLU_DBL + W_DBL + Y_DBL + F_DBL + V_DBL + IDX_DBL + IB_DBL;
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DBL * sizeof(double);
    static_assert(M >= 1 && M <= 32, "the reduced system must fit one warp");
    static_assert(RN <= 2 && LL <= 32 && NR <= 8, "shape outside the kernel's layout");
};

// queue a row for the REPLAY re-solve (once, however many family chunks flag it)
__device__ __forceinline__ void flag_row(const PhsArgs& a, int64_t idx) {
    if (a.flag_mark && atomicExch(a.flag_mark + idx, 1) != 0) return;
    unsigned long long slot = atomicAdd((unsigned long long*)a.flag_count, 1ull);
    a.flag_list[slot] = idx;
}

template <int NN, int DEG, int DD, int NF>
__global__ void __launch_bounds__(128, NN <= 16 ? 8 : (NN <= 25 ? 5 : 3)) phs_ns2(PhsArgs a) {
    using Cfg = Ns2Cfg<NN, DEG, DD, NF>;
    constexpr int LL = Cfg::LL, M = Cfg::M, NR = Cfg::NR, RN = Cfg::RN, XN = Cfg::XN,
                  NP = Cfg::NP, P = Cfg::P, LP = Cfg::LP, NC = Cfg::NC, CS = Cfg::CS;
    extern __shared__ __align__(16) double smem_n2[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double* PH = smem_n2 + (size_t)wib * Cfg::WARP_DBL;  // Phi (permuted), then K / elimination rows
    double* XS = PH + Cfg::PH_DBL;     // scaled coords SoA [ax*NP + t]; staged raw positions (next stencil)
    double* QI = XS + Cfg::XS_DBL;     // row m of Q1^-1 at m*LL; pivot columns (double-buffered) at LL*LL
    double* PV = QI + LL * LL;
    double* Wm = QI + Cfg::QLU_DBL;    // W rows (reduced index c at c*LP)
    double* Ym = Wm + Cfg::W_DBL;      // Y column c at c*LP; r_piv[.][f] at (M + f)*LP
    double* FS = Ym + Cfg::Y_DBL;      // node rhs FS[t*NR + f] (permuted t); |Q| row sums at NN*NR + t
    double* VS = FS + Cfg::F_DBL;      // w1p[k*NR+f], lambda rhs at 2*LL*NR, v at 3*LL*NR
    int* IDX = reinterpret_cast<int*>(VS + Cfg::V_DBL);  // permuted index -> stencil node
    int* IB = IDX + 2 * Cfg::IDX_DBL;  // staged node indices of the next-but-one stencil, then its row
    const PhsParams& P_ = a.P;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int g8 = lane >> 2, t4 = lane & 3;  // tensor-core fragment coordinates

    const int64_t stride = (int64_t)gridDim.x * Cfg::WARPS;
    int64_t idx = (int64_t)blockIdx.x * Cfg::WARPS + wib;

    // Two-stage prefetch, all through cp.async (no register ever waits on a
    // global load): the node indices of stencil i+2 go to IB while the
    // positions of stencil i+1 (addressed by the indices staged one stencil
    // earlier) go to XS.
    auto stage_idx = [&](int64_t id) {
        if (id < a.m) {
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                const int j = lane + 32 * s;
                if (j < NN) cp_async4(IB + j, a.stencils + id * NN + j);
            }
            if (lane == 0) cp_async8(IB + Cfg::IB_ROW, a.rows + id);
        }
    };
    auto stage = [&](int64_t id) {
        if (id < a.m) {
            int nd[RN];
#pragma unroll
            for (int s = 0; s < RN; ++s) nd[s] = lane + 32 * s < NN ? IB[lane + 32 * s] : 0;
            const int64_t rw = *reinterpret_cast<const int64_t*>(IB + Cfg::IB_ROW);
            __syncwarp();  // IB is read: the next indices may land
#pragma unroll
            for (int s = 0; s < RN; ++s) {
                const int j = lane + 32 * s;
                if (j < NN) {
#pragma unroll
                    for (int ax = 0; ax < DD; ++ax) cp_async8(XS + ax * NP + j, a.pos + (int64_t)nd[s] * DD + ax);
                }
            }
            if (lane < DD) cp_async8(XS + DD * NP + lane, a.pos + rw * DD + lane);
        }
        stage_idx(id + stride);
        cp_async_commit();
    };
    stage_idx(idx);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    stage(idx);

#pragma unroll 1
    for (; idx < a.m; idx += stride) {
        cp_async_wait_all();
        __syncwarp();

        // ---- (1) local coordinates, scale, monomials, node right-hand sides
        double x[RN][DD], r2[RN];
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int j = lane + 32 * s;
            const bool in = j < NN;
#pragma unroll
            for (int ax = 0; ax < DD; ++ax) x[s][ax] = in ? XS[ax * NP + j] - XS[DD * NP + ax] : 0.0;
            r2[s] = x[s][0] * x[s][0];
#pragma unroll
            for (int ax = 1; ax < DD; ++ax) r2[s] = fma(x[s][ax], x[s][ax], r2[s]);
        }
        __syncwarp();  // staged positions consumed: XS is free for the scaled coordinates
        int stat = 0;
        double rs = 1.0, r2max;
        {
            double mx = r2[0];
            if (RN > 1) mx = fmax(mx, r2[RN - 1]);
            r2max = warp_max_nonneg(mx);
            const int sc_code = P_.scale_code;
            if (sc_code == MF_SCALE_SUPPORT) {
                if (r2max > 0.0) rs = rsqrt_c3(r2max);
                else stat = 2;
            } else if (sc_code == MF_SCALE_NEAREST) {
                double mn = INFINITY;
#pragma unroll
                for (int s = 0; s < RN; ++s)
                    if (r2[s] > 0.0) mn = fmin(mn, r2[s]);
                mn = warp_min_nonneg(mn);
                if (mn < INFINITY) rs = rsqrt_c3(mn);
                else stat = 2;
            }
        }
        const double rc2max = r2max * rs * rs;
        double facs[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int o = P_.orders[f];
            facs[f] = o == 0 ? 1.0 : (o == 1 ? rs : rs * rs);
        }
        // columns of [Q^T | g | I]: column j = lane + 32 s is node j (its monomials),
        // then the constraint right-hand sides (families, probe), then the identity
        double q[CS][LL], fr[RN][NF], qsum[RN];
#pragma unroll
        for (int s = 0; s < RN; ++s) {
#pragma unroll
            for (int ax = 0; ax < DD; ++ax) x[s][ax] *= rs;
            monomials_reg<DD, DEG, 0, LL>(q[s], x[s]);
            qsum[s] = 0.0;
#pragma unroll
            for (int m = 0; m < LL; ++m) qsum[s] += fabs(q[s][m]);
            // FAST k = 3 right-hand side (phs_rhs_top_k3 with reciprocal roots)
            double rr2 = x[s][0] * x[s][0];
#pragma unroll
            for (int ax = 1; ax < DD; ++ax) rr2 = fma(x[s][ax], x[s][ax], rr2);
            const double rsq = rr2 > 0.0 ? rsqrt_c3(rr2) : 0.0;
            const double r = rr2 * rsq, ir2 = rsq * rsq;
            const double d1r = 3.0 * r, d2v = 6.0 * r;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int kind = P_.kinds[f];
                double t;
                if (kind == MF_KIND_IDENTITY) {
                    t = rr2 * r;
                } else if (kind == MF_KIND_D1) {
                    t = -d1r * x[s][P_.ax_a[f]];
                } else if (kind == MF_KIND_D2) {
                    const double ee = x[s][P_.ax_a[f]] * x[s][P_.ax_b[f]] * ir2;
                    const double delta = P_.ax_a[f] == P_.ax_b[f] ? 1.0 : 0.0;
                    t = fma(d2v, ee, d1r * (delta - ee));
                } else {
                    t = fma((double)(DD - 1), d1r, d2v);
                }
                fr[s][f] = t * facs[f];
            }
        }
        // (branch-free: every lane forms the three candidates, selects are uniform
        // loads of the constraint rows plus per-lane selects)
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            if (32 * s + 31 < NN) continue;  // slot holds only node columns
            const int j = lane + 32 * s;
            const int f = j - NN, m = j - NN - NR;
#pragma unroll
            for (int k = 0; k < LL; ++k) {
                double vb = 0.0;
#pragma unroll
                for (int ff = 0; ff < NF; ++ff) vb = f == ff ? P_.base_bot[ff * MF_MAX_MONOMIALS + k] * facs[ff] : vb;
                const double vp = probe_sign(idx, NN + k);
                const double v = f < NF ? vb : (f == NF ? vp : (m == k ? 1.0 : 0.0));
                if (j >= NN) q[s][k] = v;
            }
        }

        // ---- (2) Gauss-Jordan on [Q^T | g | I] with node (column) pivoting over the
        //      lane-resident nodes: the row operations are Q1^-T, so the free node
        //      columns become W^T, the g columns the particular solution w1p and the
        //      identity columns the rows of Q1^-1
        bool ok = stat == 0;
        bool live = lane < NN;  // slot 0 is a pivot candidate until it wins
        int myk = 0;
#pragma unroll
        for (int k = 0; k < LL; ++k) {
            unsigned key = 0u;
            if (live) {
                const unsigned hi = (unsigned)((unsigned long long)__double_as_longlong(fabs(q[0][k])) >> 32);
                key = (hi & ~31u) | (unsigned)(31 - lane);
            }
            // the reciprocal of every candidate pivot is formed while the REDUX runs:
            // the winner publishes its own, so no reciprocal sits on the step's chain
            const double my_inv = rcp_c3(q[0][k]);
            const unsigned mk = __reduce_max_sync(FULL, key);
            const int wl = 31 - (int)(mk & 31u);
            ok = ok && (mk >> 5) != 0u;
            double* pc = PV + (k & 1) * (LL + 1);  // two buffers: the next step's winner never overwrites a column being read
            if (lane == wl && live) {
#pragma unroll
                for (int r = 0; r < LL; ++r) pc[r] = r == k ? my_inv : q[0][r];
                live = false;
                myk = k;
            }
            __syncwarp();
            double pv[LL];
#pragma unroll
            for (int r = 0; r < LL; ++r) pv[r] = pc[r];
            const double inv = pv[k];
#pragma unroll
            for (int s = 0; s < CS; ++s) {
                const double t = q[s][k] * inv;
#pragma unroll
                for (int r = 0; r < LL; ++r)
                    if (r != k) q[s][r] = fma(-t, pv[r], q[s][r]);
                q[s][k] = t;
            }
        }
        // free nodes: live slot-0 lanes in lane order, then the slot-1 nodes
        const unsigned fb = __ballot_sync(FULL, live);
        const int nfl = __popc(fb);
        ok = ok && nfl + XN == M;
        const int c0 = live ? LL + __popc(fb & lt_mask) : myk;  // permuted index of node `lane`
        if (lane < NN) {
            IDX[c0] = lane;
#pragma unroll
            for (int ax = 0; ax < DD; ++ax) XS[ax * NP + c0] = x[0][ax];
#pragma unroll
            for (int f = 0; f < NF; ++f) FS[c0 * NR + f] = fr[0][f];
            FS[c0 * NR + NF] = probe_sign(idx, lane);
            FS[NN * NR + c0] = qsum[0];
            if (live) {
#pragma unroll
                for (int m = 0; m < LL; ++m) Wm[(c0 - LL) * LP + m] = q[0][m];
            }
        }
        if (RN > 1 && lane < XN) {
            const int c1 = LL + nfl + lane;
            if (c1 < NN) {
                IDX[c1] = 32 + lane;
#pragma unroll
                for (int ax = 0; ax < DD; ++ax) XS[ax * NP + c1] = x[RN - 1][ax];
#pragma unroll
                for (int f = 0; f < NF; ++f) FS[c1 * NR + f] = fr[RN - 1][f];
                FS[c1 * NR + NF] = probe_sign(idx, 32 + lane);
                FS[NN * NR + c1] = qsum[RN - 1];
#pragma unroll
                for (int m = 0; m < LL; ++m) Wm[(c1 - LL) * LP + m] = q[RN - 1][m];
            }
        }
#pragma unroll
        for (int s = 0; s < CS; ++s) {
            const int j = lane + 32 * s;
            if (j >= NN && j < NN + NR) {
#pragma unroll
                for (int k = 0; k < LL; ++k) VS[k * NR + (j - NN)] = q[s][k];  // w1p
            } else if (j >= NN + NR && j < NC) {
#pragma unroll
                for (int r = 0; r < LL; ++r) QI[(j - NN - NR) * LL + r] = q[s][r];  // Q1^-1 row
            }
        }
        ok = __all_sync(FULL, ok);
        __syncwarp();

        // constraint rows of ||A||_inf: the constant column sums to n and every other
        // |monomial| <= 1 under the support scale; otherwise bound them by n * max |Q row|
        const double qbound = P_.scale_code == MF_SCALE_SUPPORT
                                  ? (double)NN
                                  : (double)NN * warp_max_nonneg(fmax(qsum[0], qsum[RN - 1]));
        const double close_thr = a.min_sep2 * rc2max;  // HYBRID: (min separation / radius)^2 threshold
        bool close = false;
        double anorm = 0.0;
        bool bad = !ok;
        if (ok) {
            // ---- (3) Phi in the permuted order [pivots; free]
            // pair walk: lane t owns node t and walks t+1 .. t+(NN-1)/2 (mod NN);
            // nodes 32.. take the tail
            {
                // pairs (t, t + s), s = 1 .. H: every unordered pair once for odd NN; for
                // even NN the antipodal pair is met from both ends (same value stored twice)
                constexpr int H = NN / 2;
                // loads of a chunk of pairs first, then the arithmetic, then the
                // stores: shared stores would otherwise order every pair's loads
                // behind the previous pair's stores and serialise the chains
                constexpr int CH = 6;
                if (lane < NN) {
                    double xi[DD];
#pragma unroll
                    for (int ax = 0; ax < DD; ++ax) xi[ax] = XS[ax * NP + lane];
#pragma unroll
                    for (int st0 = 1; st0 <= H; st0 += CH) {
                        int jc[CH];
                        double xj[CH][DD], v[CH];
                        bool cl = false;
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            if (st0 + u <= H) {
                                const int t = lane + st0 + u;
                                jc[u] = t >= NN ? t - NN : t;
#pragma unroll
                                for (int ax = 0; ax < DD; ++ax) xj[u][ax] = XS[ax * NP + jc[u]];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            if (st0 + u <= H) {
                                double df = xi[0] - xj[u][0];
                                double d2 = df * df;
#pragma unroll
                                for (int ax = 1; ax < DD; ++ax) {
                                    df = xi[ax] - xj[u][ax];
                                    d2 = fma(df, df, d2);
                                }
                                cl = cl | (d2 < close_thr);
                                // (+1e-300: coincident nodes give r^3 = 0 instead of 0 * inf)
                                v[u] = d2 * (d2 * rsqrt_c3(d2 + 1e-300));
                            }
                        }
                        close = close | cl;
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            if (st0 + u <= H) {
                                PH[lane * P + jc[u]] = v[u];
                                PH[jc[u] * P + lane] = v[u];
                            }
                        }
                    }
                    PH[lane * P + lane] = 0.0;
                }
                if constexpr (XN > 0) {
                    constexpr int REM = XN * H, RT = (REM + 31) / 32;
                    int ic[RT], jc[RT];
                    double xa[RT][DD], xb[RT][DD], v[RT];
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int p = lane + 32 * t < REM ? lane + 32 * t : 0;
                        ic[t] = 32 + p / H;
                        jc[t] = ic[t] + p % H + 1;
                        if (jc[t] >= NN) jc[t] -= NN;
#pragma unroll
                        for (int ax = 0; ax < DD; ++ax) {
                            xa[t][ax] = XS[ax * NP + ic[t]];
                            xb[t][ax] = XS[ax * NP + jc[t]];
                        }
                    }
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        double df = xa[t][0] - xb[t][0];
                        double d2 = df * df;
#pragma unroll
                        for (int ax = 1; ax < DD; ++ax) {
                            df = xa[t][ax] - xb[t][ax];
                            d2 = fma(df, df, d2);
                        }
                        close = close | (d2 < close_thr);
                        v[t] = d2 * (d2 * rsqrt_c3(d2 + 1e-300));
                    }
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        if (lane + 32 * t < REM) {
                            PH[ic[t] * P + jc[t]] = v[t];
                            PH[jc[t] * P + ic[t]] = v[t];
                        }
                    }
                    if (lane < XN) PH[(32 + lane) * P + 32 + lane] = 0.0;
                }
            }
            __syncwarp();
        }
        // the coordinates are consumed: stage the next stencil's positions into XS
        stage(idx + stride);
        if (ok) {
            // ||A||_inf of the saddle-point matrix (estimate only): the node rows of Phi
            // are summed from the tensor-core operands below (every entry of Phi is
            // loaded exactly once as a Y / K operand: Phi11, Phi12 in Y; H, Phi22 in K)
            double rs_y[(LL + 7) / 8] = {}, rs_k[(M + 7) / 8] = {};
            // ---- (4) Y = Phi12 - Phi11 W^T on the fp64 tensor core, with NR extra
            //      columns that carry the pivot residuals of the particular solution:
            //      C-init f(p_k), B column w1p  ->  r_piv[k] = f(p_k) - Phi11[k] w1p
            constexpr int MR = M + NR;  // columns of [K | b]
            {
                constexpr int LT = (LL + 7) / 8, YT = (MR + 7) / 8, KS = (LL + 3) / 4;
                double acc[LT][YT][2];
#pragma unroll
                for (int lt = 0; lt < LT; ++lt)
#pragma unroll
                    for (int mt = 0; mt < YT; ++mt)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int k = lt * 8 + g8, c = mt * 8 + 2 * t4 + h;
                            double v = 0.0;
                            if (k < LL && c < M) {
                                v = PH[k * P + LL + c];
                                rs_y[lt] += v;
                            } else if (k < LL && c < MR) {
                                v = FS[k * NR + (c - M)];
                            }
                            acc[lt][mt][h] = v;
                        }
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int k2 = ks * 4 + t4;
                    double af[LT], bf[YT];
#pragma unroll
                    for (int lt = 0; lt < LT; ++lt) {
                        const int k = lt * 8 + g8;
                        const double v = (k2 < LL && k < LL) ? PH[k2 * P + k] : 0.0;
                        rs_y[lt] += v;
                        af[lt] = -v;
                    }
#pragma unroll
                    for (int mt = 0; mt < YT; ++mt) {
                        const int c = mt * 8 + g8;
                        double v = 0.0;
                        if (k2 < LL && c < M) v = Wm[c * LP + k2];
                        else if (k2 < LL && c < MR) v = VS[k2 * NR + (c - M)];
                        bf[mt] = v;
                    }
#pragma unroll
                    for (int lt = 0; lt < LT; ++lt)
#pragma unroll
                        for (int mt = 0; mt < YT; ++mt) dmma_f64(acc[lt][mt][0], acc[lt][mt][1], af[lt], bf[mt]);
                }
#pragma unroll
                for (int lt = 0; lt < LT; ++lt)
#pragma unroll
                    for (int mt = 0; mt < YT; ++mt)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int k = lt * 8 + g8, c = mt * 8 + 2 * t4 + h;
                            if (k < LL && c < MR) Ym[c * LP + k] = acc[lt][mt][h];
                        }
            }
            __syncwarp();  // Y and r_piv (Y rows M..) visible

            // ---- (5) [K | b] = [Phi22 | f_free] - [H W] [W^T w1p; Y r_piv] on the fp64
            //      tensor core: b = Z^T (f - Phi w_p) comes out as NR extra columns
            constexpr int RT = (M + 7) / 8, CT = (MR + 7) / 8;
            static_assert(MR <= 32, "[K | b] must fit 32 columns");
            double acc[RT][CT][2];
            {
                constexpr int KS = (2 * LL + 3) / 4;
#pragma unroll
                for (int rt = 0; rt < RT; ++rt)
#pragma unroll
                    for (int ct = 0; ct < CT; ++ct)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int c = rt * 8 + g8, c2 = ct * 8 + 2 * t4 + h;
                            double v = 0.0;
                            if (c < M && c2 < M) {
                                v = PH[(LL + c) * P + LL + c2];
                                rs_k[rt] += v;
                            } else if (c < M && c2 < MR) {
                                v = FS[(LL + c) * NR + (c2 - M)];
                            }
                            acc[rt][ct][h] = v;
                        }
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int kk = ks * 4 + t4;  // < LL: H column kk, else W / Y row kk - LL
                    const bool hp = kk < LL, kv = kk < 2 * LL;
                    const int kh = hp ? kk : 0, kw = hp ? 0 : (kv ? kk - LL : 0);
                    double af[RT], bf[CT];
#pragma unroll
                    for (int rt = 0; rt < RT; ++rt) {
                        const int c = rt * 8 + g8;
                        const int cr = c < M ? c : 0;
                        const double v = hp ? PH[(LL + cr) * P + kh] : Wm[cr * LP + kw];
                        if (hp && c < M) rs_k[rt] += v;
                        af[rt] = (c < M && kv) ? -v : 0.0;
                    }
#pragma unroll
                    for (int ct = 0; ct < CT; ++ct) {
                        const int c2 = ct * 8 + g8;
                        double v = 0.0;
                        if (kv && c2 < MR) {
                            if (!hp) v = Ym[c2 * LP + kw];
                            else v = c2 < M ? Wm[c2 * LP + kh] : VS[kh * NR + (c2 - M)];
                        }
                        bf[ct] = v;
                    }
#pragma unroll
                    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
                        for (int ct = 0; ct < CT; ++ct) dmma_f64(acc[rt][ct][0], acc[rt][ct][1], af[rt], bf[ct]);
                }
            }
            {
                // row sums: each row's entries sit in the four lanes t4 = 0..3 of its g
#pragma unroll
                for (int lt = 0; lt < (LL + 7) / 8; ++lt) {
                    double v = rs_y[lt];
                    v += __shfl_xor_sync(FULL, v, 1);
                    v += __shfl_xor_sync(FULL, v, 2);
                    const int k = lt * 8 + g8;
                    if (k < LL) anorm = fmax(anorm, v + FS[NN * NR + k]);
                }
#pragma unroll
                for (int rt = 0; rt < RT; ++rt) {
                    double v = rs_k[rt];
                    v += __shfl_xor_sync(FULL, v, 1);
                    v += __shfl_xor_sync(FULL, v, 2);
                    const int c = rt * 8 + g8;
                    if (c < M) anorm = fmax(anorm, v + FS[NN * NR + LL + c]);
                }
                anorm = fmax(warp_max_nonneg(anorm), qbound);
            }
            __syncwarp();  // every read of Phi is done: the panel buffers take its place

            // ---- (6) [K | b] to one row per lane through shared memory: element (r, c)
            //      at r * 36 + (c ^ r), which keeps both the accumulator-fragment stores
            //      and the row reads free of bank conflicts
            constexpr int KTP = Cfg::KTP;
            static_assert(M * KTP <= Cfg::PH_DBL && MR <= 32, "[K | b] staging");
            const bool act = lane < M;
            const int cc = act ? lane : 0;
#pragma unroll
            for (int rt = 0; rt < RT; ++rt)
#pragma unroll
                for (int ct = 0; ct < CT; ++ct)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = rt * 8 + g8, c = ct * 8 + 2 * t4 + h;
                        if (r < M && c < MR) PH[r * KTP + (c ^ r)] = acc[rt][ct][h];
                    }
            __syncwarp();
            double K[M], bb[NR];
#pragma unroll
            for (int j = 0; j < M; ++j) K[j] = PH[cc * KTP + (j ^ cc)];
#pragma unroll
            for (int f = 0; f < NR; ++f) bb[f] = PH[cc * KTP + ((M + f) ^ cc)];
            __syncwarp();

            // ---- (7) pivot-free Gauss-Jordan on [K | b]; lane c keeps row c.  Column k
            //      (== row k of the symmetric trailing matrix) is stored with entry k+1
            //      on a 16-byte boundary, so the pivot row streams in pairs
            double* Us = PH;
            double* Bs = PH + M * Cfg::UP;
            // the pivot lane publishes 1 / d_k with its right-hand sides; every lane
            // forms the reciprocal of its next diagonal candidate as soon as that
            // entry is final (the first update of the step), off the broadcast chain
            double rnext = rcp_c3(K[0]);
#pragma unroll
            for (int k = 0; k < M; ++k) {
                double* urow = Us + k * Cfg::UP + ((k + 1) & 1);
                if (act) urow[lane] = K[k];
                if (lane == k) {
#pragma unroll
                    for (int f = 0; f < NR; ++f) Bs[k * (NR + 1) + f] = bb[f];
                    Bs[k * (NR + 1) + NR] = rnext;
                }
                __syncwarp();
                const double rk = Bs[k * (NR + 1) + NR];
                const double fac = lane != k ? K[k] * rk : 0.0;
                if (k + 1 < M) {
                    K[k + 1] = fma(-fac, urow[k + 1], K[k + 1]);
                    rnext = rcp_c3(K[k + 1]);
                }
#pragma unroll
                for (int j = k + 2; j < M; ++j) K[j] = fma(-fac, urow[j], K[j]);
#pragma unroll
                for (int f = 0; f < NR; ++f) bb[f] = fma(-fac, Bs[k * (NR + 1) + f], bb[f]);
            }
            // v_c = b_c / d_c with d_c the pivot lane c stored at its step
            {
                const double d0 = Us[1], dc = Us[cc * Cfg::UP + ((cc + 1) & 1) + cc];
                const double dinv_own = rcp_c3(dc);
#pragma unroll
                for (int f = 0; f < NR; ++f) bb[f] *= dinv_own;
                bad = bad || !__all_sync(FULL, !act || dc * d0 > 0.0);
            }

            // ---- (8) outputs: free weights; pivot weights w1p - W^T v and the
            //      multipliers' right-hand side r_piv - Y v as one tensor-core product
            double zw = 0.0, xw[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) xw[f] = 0.0;
            if (act) {
                const int node = IDX[LL + lane];
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    bad |= !isfinite(bb[f]);
                    a.out[((size_t)idx * a.out_nf + a.out_f0 + f) * NN + node] = bb[f];
                    xw[f] = fabs(bb[f]);
                }
                zw = fabs(bb[NF]);
#pragma unroll
                for (int f = 0; f < NR; ++f) VS[3 * LL * NR + lane * NR + f] = bb[f];
            }
            __syncwarp();
            {
                constexpr int R2 = (2 * LL + 7) / 8, CSN = (M + 3) / 4;
                double oacc[R2][2];
#pragma unroll
                for (int rt = 0; rt < R2; ++rt) oacc[rt][0] = oacc[rt][1] = 0.0;
#pragma unroll
                for (int cs = 0; cs < CSN; ++cs) {
                    const int c = cs * 4 + t4;
                    const int cr = c < M ? c : 0;
                    const double bv = (c < M && g8 < NR) ? VS[3 * LL * NR + cr * NR + (g8 < NR ? g8 : 0)] : 0.0;
#pragma unroll
                    for (int rt = 0; rt < R2; ++rt) {
                        const int r = rt * 8 + g8;
                        double av = 0.0;
                        if (c < M && r < 2 * LL) av = r < LL ? Wm[cr * LP + r] : Ym[cr * LP + (r - LL)];
                        dmma_f64(oacc[rt][0], oacc[rt][1], av, bv);
                    }
                }
#pragma unroll
                for (int rt = 0; rt < R2; ++rt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = rt * 8 + g8, f = 2 * t4 + h;
                        if (f < NR && r < LL) {
                            const double w = VS[r * NR + f] - oacc[rt][h];
                            if (f < NF) {
                                bad |= !isfinite(w);
                                a.out[((size_t)idx * a.out_nf + a.out_f0 + f) * NN + IDX[r]] = w;
                                xw[f] = fmax(xw[f], fabs(w));
                            } else {
                                zw = fmax(zw, fabs(w));
                            }
                        } else if (f < NF && r >= LL && r < 2 * LL) {
                            VS[2 * LL * NR + (r - LL) * NR + f] = Ym[(M + f) * LP + (r - LL)] - oacc[rt][h];
                        }
                    }
            }
            __syncwarp();
            // lambda = Q1^-1 (r_piv - Y v): lane m owns row m of Q1^-1
            double la[NF];
            {
                const int mm = lane < LL ? lane : 0;
                double lam[NF];
#pragma unroll
                for (int f = 0; f < NF; ++f) lam[f] = 0.0;
#pragma unroll
                for (int r = 0; r < LL; ++r) {
                    const double qi = QI[mm * LL + r];
#pragma unroll
                    for (int f = 0; f < NF; ++f) lam[f] = fma(qi, VS[2 * LL * NR + r * NR + f], lam[f]);
                }
#pragma unroll
                for (int f = 0; f < NF; ++f) la[f] = warp_max_nonneg(lane < LL ? fabs(lam[f]) : 0.0);
            }
            zw = warp_max_nonneg(zw);
#pragma unroll
            for (int f = 0; f < NF; ++f) xw[f] = warp_max_nonneg(xw[f]);
            double ratio = 0.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) ratio = fmax(ratio, fmax(xw[f], la[f]) / xw[f]);
            const double est = anorm * zw * ratio;
            close = __any_sync(FULL, close);
            bad = __any_sync(FULL, bad);
            if (!bad && lane == 0 && (close || !(est <= a.hybrid_thresh))) flag_row(a, idx);
        }
        // failed / indefinite / non-finite rows are re-solved in the reference's order
        if (bad && lane == 0) flag_row(a, idx);
        if (lane == 0) a.status[idx] = 0;
        __syncwarp();
    }
    cp_async_wait_all();
}

template <int NN, int DEG, int DD, int NF>
int launch_ns2(const PhsArgs& a, cudaStream_t st, int sms) {
    using Cfg = Ns2Cfg<NN, DEG, DD, NF>;
    constexpr GradedLex<DD, DEG> g{};
    if (!a.flag_list || a.kappa || a.P.l != Cfg::LL || a.P.nf != NF) return MF_ERR_UNSUPPORTED;
    for (int m = 0; m < Cfg::LL; ++m)
        for (int ax = 0; ax < DD; ++ax)
            if (a.P.expos[m * DD + ax] != g.e[m][ax]) return MF_ERR_UNSUPPORTED;
    if (a.P.k != 3 || a.P.even || DEG < 1) return MF_ERR_UNSUPPORTED;
    auto kern = phs_ns2<NN, DEG, DD, NF>;
    MF_CUDA_CHECK(ensure_smem(kern, (int)Cfg::SMEM));
    int per_sm = occupancy(kern, Cfg::WARPS * 32, Cfg::SMEM);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (a.m + Cfg::WARPS - 1) / Cfg::WARPS;
    const int64_t cap = (int64_t)sms * per_sm * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, Cfg::WARPS * 32, Cfg::SMEM, st>>>(a);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

#define MF_INSTANTIATE_NS2(NN, DEG, DD, NF) template int launch_ns2<NN, DEG, DD, NF>(const PhsArgs&, cudaStream_t, int);

}  // namespace mf

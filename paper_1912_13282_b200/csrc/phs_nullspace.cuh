// Helpers of the nullspace shape solve (phs_ns2.cuh, phs_cta.cu), and its mathematics:
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
// The +-1 probe rides along as one more right-hand side, and the family
// multipliers lambda (for the sensitivity estimate) come from
// Q1 lambda = (f - Phi w)_piv.  Rounding differs from the reference's LU;
// HYBRID re-solves, in the reference's order, the rows the LU FAST kernel would
// flag (near-coincident nodes, sensitivity estimate) plus any row whose reduced
// pivots lose definiteness.
#pragma once

#include "phs_reg.cuh"

namespace mf {

__host__ __device__ constexpr int ns_even(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int ns_max(int a, int b) { return a > b ? a : b; }

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

}  // namespace mf

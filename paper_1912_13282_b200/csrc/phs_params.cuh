// Per-call parameters and per-entry formulas of the PHS shape computation.
// Formulas follow _batch_numba (_phs_batch.py:228-290) operation for operation.
#pragma once

#include "common.cuh"

namespace mf {

struct PhsParams {
    int d, l, nf, k, even, scale_code;
    int kinds[MF_MAX_FAMILIES];
    int ax_a[MF_MAX_FAMILIES];
    int ax_b[MF_MAX_FAMILIES];
    int orders[MF_MAX_FAMILIES];
    int expos[MF_MAX_MONOMIALS * MF_MAX_DIM];
    double base_bot[MF_MAX_FAMILIES * MF_MAX_MONOMIALS];
};

struct PhsArgs {
    const double* pos;
    const int64_t* rows;
    const int32_t* stencils;
    int64_t m;
    int n;
    double* out;
    int8_t* status;
    int64_t* first_fail;
    int64_t* flag_list;   // HYBRID: rows to re-solve in REPLAY order
    int64_t* flag_count;
    double hybrid_thresh;
    double* kappa;        // optional per-row conditioning diagnostics (FAST/HYBRID)
    double min_sep2;      // HYBRID: (min node separation / stencil radius)^2 below which to re-solve
    // family chunks (nullspace first pass): the kernel solves P.nf families and
    // writes them as families out_f0 .. of an out_nf-family output; flag_mark
    // (m ints, zeroed, nullable) keeps a row flagged by several chunks listed once
    int out_nf, out_f0;
    int* flag_mark;
    PhsParams P;
};

inline int fill_phs_params(PhsParams& P, int d, int k, int even, const int32_t* expos, int l,
                           const double* base_bot, const int32_t* kinds, const int32_t* ax_a,
                           const int32_t* ax_b, const int32_t* orders, int nf, int scale_code) {
    P.d = d;
    P.l = l;
    P.nf = nf;
    P.k = k;
    P.even = even ? 1 : 0;
    P.scale_code = scale_code;
    if (scale_code < MF_SCALE_NONE || scale_code > MF_SCALE_SUPPORT) {
        set_error("mf_phs_weights: bad scale code %d", scale_code);
        return MF_ERR_ARG;
    }
    for (int f = 0; f < nf; ++f) {
        if (kinds[f] < MF_KIND_IDENTITY || kinds[f] > MF_KIND_LAPLACIAN || ax_a[f] < 0 || ax_a[f] >= d ||
            ax_b[f] < 0 || ax_b[f] >= d || orders[f] < 0 || orders[f] > 2) {
            set_error("mf_phs_weights: bad family descriptor %d", f);
            return MF_ERR_ARG;
        }
        P.kinds[f] = kinds[f];
        P.ax_a[f] = ax_a[f];
        P.ax_b[f] = ax_b[f];
        P.orders[f] = orders[f];
        for (int j = 0; j < l; ++j) P.base_bot[f * MF_MAX_MONOMIALS + j] = base_bot[f * l + j];
    }
    for (int j = 0; j < l * d; ++j) P.expos[j] = expos[j];
    return MF_OK;
}

// phi(r): r^k (odd k, correctly rounded power standing in for glibc pow),
// r^k log r (even k; r^k by numba's integer power, exact replay)
__device__ __forceinline__ double phs_phi(double r, int k, int even) {
    if (!even) return pow_cr_int(r, k);
    return r > 0.0 ? __dmul_rn(numba_int_power(r, k), log(r)) : 0.0;
}

// q = prod_a local[a]^e_a, axis order, zero exponents skipped, from q = 1.0
__device__ __forceinline__ double phs_monomial(const double* loc, const int* e, int d) {
    double q = 1.0;
    for (int ax = 0; ax < d; ++ax)
        if (e[ax]) q = __dmul_rn(q, numba_int_power(loc[ax], e[ax]));
    return q;
}

// RHS top entries (L phi(|x - p_j|))(0) per family, before the s^-order factor
__device__ __forceinline__ void phs_rhs_top(const double* loc, int d, const PhsParams& P, double* top) {
    double r2 = 0.0;
    for (int ax = 0; ax < d; ++ax) r2 = __dadd_rn(r2, __dmul_rn(loc[ax], loc[ax]));
    double r = __dsqrt_rn(r2);
    double val = 0.0, d1r = 0.0, d2v = 0.0;
    const double kf = (double)P.k;
    if (r > 0.0) {
        if (P.even) {
            double lg = log(r);
            double rk2 = pow_cr_int(r, P.k - 2);
            val = __dmul_rn(numba_int_power(r, P.k), lg);
            d1r = __dmul_rn(rk2, __dadd_rn(__dmul_rn(kf, lg), 1.0));
            d2v = __dmul_rn(rk2, __dsub_rn(__dadd_rn(__dmul_rn((double)(P.k * P.k - P.k), lg), 2.0 * kf), 1.0));
        } else {
            double rk2 = pow_cr_int(r, P.k - 2);
            val = pow_cr_int(r, P.k);
            d1r = __dmul_rn(kf, rk2);
            d2v = __dmul_rn(__dmul_rn(kf, __dsub_rn(kf, 1.0)), rk2);
        }
    }
    for (int f = 0; f < P.nf; ++f) {
        int kind = P.kinds[f];
        double t;
        if (kind == MF_KIND_IDENTITY) {
            t = val;
        } else if (kind == MF_KIND_D1) {
            t = __dmul_rn(d1r, -loc[P.ax_a[f]]);
        } else if (kind == MF_KIND_D2) {
            double ee = r > 0.0 ? __ddiv_rn(__dmul_rn(loc[P.ax_a[f]], loc[P.ax_b[f]]), r2) : 0.0;
            double delta = P.ax_a[f] == P.ax_b[f] ? 1.0 : 0.0;
            t = __dadd_rn(__dmul_rn(d2v, ee), __dmul_rn(d1r, __dsub_rn(delta, ee)));
        } else {
            t = __dadd_rn(d2v, __dmul_rn((double)(d - 1), d1r));
        }
        top[f] = t;
    }
}

// FAST k = 3 (odd) right-hand side: r^3, 3 r, 6 r with FMA-contracted arithmetic
__device__ __forceinline__ void phs_rhs_top_k3(const double* loc, int d, const PhsParams& P, double* top) {
    double r2 = loc[0] * loc[0];
    for (int ax = 1; ax < d; ++ax) r2 = fma(loc[ax], loc[ax], r2);
    const double r = sqrt(r2);
    const double val = r2 * r, d1r = 3.0 * r, d2v = 6.0 * r;
    const double ir2 = r > 0.0 ? 1.0 / r2 : 0.0;
    for (int f = 0; f < P.nf; ++f) {
        const int kind = P.kinds[f];
        double t;
        if (kind == MF_KIND_IDENTITY) {
            t = val;
        } else if (kind == MF_KIND_D1) {
            t = -d1r * loc[P.ax_a[f]];
        } else if (kind == MF_KIND_D2) {
            const double ee = loc[P.ax_a[f]] * loc[P.ax_b[f]] * ir2;
            const double delta = P.ax_a[f] == P.ax_b[f] ? 1.0 : 0.0;
            t = fma(d2v, ee, d1r * (delta - ee));
        } else {
            t = fma((double)(d - 1), d1r, d2v);
        }
        top[f] = t;
    }
}

// deterministic +-1 probe vector for the conditioning estimate
__device__ __forceinline__ double probe_sign(int64_t idx, int r) {
    unsigned h = (unsigned)idx * 0x9E3779B1u ^ ((unsigned)r + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return (h & 0x80000000u) ? 1.0 : -1.0;
}

int launch_phs_fast(const PhsArgs& a, cudaStream_t st, int sms);
int launch_phs_ns_cta(const PhsArgs& a, cudaStream_t st, int sms);
int launch_phs_cta(const PhsArgs& a, bool replay, const int64_t* list, const int64_t* list_count,
                   int64_t max_count, cudaStream_t st, int sms);
int launch_phs_replay_reg(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count,
                          cudaStream_t st, int sms);

}  // namespace mf

// Dispatch of the register-resident shape solve (kernel template in phs_reg.cuh;
// each hot shape is instantiated in its own translation unit, phs_reg_<shape>.cu,
// so nvcc builds them in parallel).
#include "common.cuh"
#include "phs_params.cuh"

namespace mf {

template <int NN, int DEG, int DD, int NF, bool REPLAY>
int launch_reg(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count,
               cudaStream_t st, int sms);

template <int NN, int DEG, int DD, int NF>
int launch_ns2(const PhsArgs& a, cudaStream_t st, int sms);

template <bool REPLAY>
int dispatch_reg(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count,
                 cudaStream_t st, int sms) {
    const int n = a.n, l = a.P.l, d = a.P.d, nf = a.P.nf;
    // hot shapes of the BASELINE configs (C1/C4, C2, C3) and their neighbours
    // (launch_reg also checks that the exponent table is the graded-lex one)
    if (d == 3 && n == 35 && l == 10 && nf == 1) return launch_reg<35, 2, 3, 1, REPLAY>(a, list, list_count, max_count, st, sms);
    if (d == 2 && n == 15 && l == 6 && nf == 1) return launch_reg<15, 2, 2, 1, REPLAY>(a, list, list_count, max_count, st, sms);
    if (d == 2 && n == 25 && l == 6 && nf == 3) return launch_reg<25, 2, 2, 3, REPLAY>(a, list, list_count, max_count, st, sms);
    return MF_ERR_UNSUPPORTED;
}

// FAST/HYBRID first pass: HYBRID runs the nullspace kernel (phs_ns2.cuh) on the
// shapes it is instantiated for; FAST, and HYBRID on every other shape, the
// register rank-1 LU (phs_reg.cuh).
int launch_phs_fast(const PhsArgs& a, cudaStream_t st, int sms) {
    const int n = a.n, l = a.P.l, d = a.P.d, nf = a.P.nf;
    int rc = MF_ERR_UNSUPPORTED;
    if (d == 3 && n == 35 && l == 10 && nf == 1) rc = launch_ns2<35, 2, 3, 1>(a, st, sms);
    else if (d == 2 && n == 15 && l == 6 && nf == 1) rc = launch_ns2<15, 2, 2, 1>(a, st, sms);
    else if (d == 2 && n == 25 && l == 6 && nf == 3) rc = launch_ns2<25, 2, 2, 3>(a, st, sms);
    if (rc != MF_ERR_UNSUPPORTED) return rc;
    return dispatch_reg<false>(a, nullptr, nullptr, a.m, st, sms);
}

int launch_phs_replay_reg(const PhsArgs& a, const int64_t* list, const int64_t* list_count, int64_t max_count,
                          cudaStream_t st, int sms) {
    return dispatch_reg<true>(a, list, list_count, max_count, st, sms);
}

}  // namespace mf

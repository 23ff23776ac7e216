// Locality-ordered apply plan (sm_100a).
//
// The reference's node indices carry no spatial order (uniform random
// clouds), so a row-per-thread SpMV gathers u from random cache lines and is
// L2-bound.  The apply plan renumbers the rows/columns of the canonical CSR
// along a Morton (Z-order) curve of the node positions and stores the entries
// ELL-32 slot-major in that order: a warp's 32 rows are spatial neighbours,
// their columns hit the same few L1 lines, and the value/index streams stay
// contiguous.  Entry order inside each row is unchanged (ascending original
// column), so every row sum keeps scipy's addend order and results stay
// bitwise equal to the reference (storage.py:186-188).
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace mf {

// 32-bit Morton keys (10 bits per axis in 3D, 16 in 2D, 32 in 1D): a 1024^3
// lattice is far finer than any node spacing the plan is built for, and the
// radix sort needs 4 digit passes instead of 8 for 64-bit keys
__device__ __forceinline__ unsigned spread3(unsigned x) {  // 10 bits -> every 3rd bit
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}
__device__ __forceinline__ unsigned spread2(unsigned x) {  // 16 bits -> every 2nd bit
    x &= 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

__global__ void plan_bbox(const double* __restrict__ pos, int64_t N, int d, unsigned long long* bb) {
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < d; ++a) {
            double x = pos[i * d + a];
            mn[a] = fmin(mn[a], x);
            mx[a] = fmax(mx[a], x);
        }
    block_bbox_commit(mn, mx, d, bb);
}

__global__ void plan_keys(const double* __restrict__ pos, int64_t N, int d, const unsigned long long* __restrict__ bb,
                          unsigned* __restrict__ key, int32_t* __restrict__ val) {
    double lo[3], sc[3];
    // 24-bit keys (three radix passes): 2^24 Morton cells is ~16 per node at
    // N = 1M, enough for the gather locality the plan is for
    const int bits = d == 1 ? 24 : (d == 2 ? 12 : 8);
    const double span = (double)((1ull << bits) - 1);
    for (int a = 0; a < d; ++a) {
        lo[a] = from_ordered_bits(bb[a]);
        double ext = from_ordered_bits(bb[3 + a]) - lo[a];
        sc[a] = ext > 0.0 ? span / ext : 0.0;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned q[3] = {0, 0, 0};
        for (int a = 0; a < d; ++a) {
            double t = (pos[i * d + a] - lo[a]) * sc[a];
            t = t > 0.0 ? (t < span ? t : span) : 0.0;
            q[a] = (unsigned)t;
        }
        unsigned k;
        if (d == 1) k = q[0];
        else if (d == 2) k = spread2(q[0]) | (spread2(q[1]) << 1);
        else k = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
        key[i] = k;
        val[i] = (int32_t)i;
    }
}

__global__ void plan_invert(const int32_t* __restrict__ order, int64_t N, int32_t* __restrict__ inv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        inv[order[i]] = (int32_t)i;
}

// ELL-32 plan in the new order: row i' = old row order[i'], column c -> inv[c]
__global__ void plan_ell_build(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                               const double* __restrict__ data, int64_t N, int W, const int32_t* __restrict__ order,
                               const int32_t* __restrict__ inv, int32_t* __restrict__ ell_idx,
                               double* __restrict__ ell_val, int32_t* __restrict__ ell_len) {
    const int64_t total = ((N + 31) / 32) * 32 * (int64_t)W;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t tile = e / (32 * (int64_t)W);
        int rem = (int)(e - tile * 32 * (int64_t)W);
        int j = rem >> 5, lane = rem & 31;
        int64_t rn = tile * 32 + lane;
        int32_t ci = 0;
        double v = 0.0;
        if (rn < N) {
            const int64_t ro = order ? order[rn] : rn;
            const int32_t lo = indptr[ro], len = indptr[ro + 1] - lo;
            if (j == 0 && ell_len) ell_len[rn] = len;
            if (j < len) {
                const int32_t c = indices[lo + j];
                ci = inv ? inv[c] : c;
                if (data) v = data[lo + j];
            }
        }
        if (ell_idx) ell_idx[e] = ci;
        if (ell_val) ell_val[e] = v;
    }
    // W = 0 (no stored row has an entry): the loop above has no slots, the
    // lengths still have to be written (they are read by every apply)
    if (W == 0 && ell_len)
        for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
            const int64_t ro = order ? order[r] : r;
            ell_len[r] = indptr[ro + 1] - indptr[ro];
        }
}

// Block per 32-row tile: the tile's 32 W entries are built by one block, so
// the rows' CSR segments and the inverse-permutation lookups of their columns
// (spatial neighbours share columns) are re-read from this SM's L1 instead of
// being spread over several blocks and SMs; output order and values are the
// same as plan_ell_build's.
__global__ void __launch_bounds__(256) plan_ell_build_tile(const int32_t* __restrict__ indptr,
                                                           const int32_t* __restrict__ indices,
                                                           const double* __restrict__ data, int64_t N, int W,
                                                           const int32_t* __restrict__ order,
                                                           const int32_t* __restrict__ inv, int32_t* __restrict__ ell_idx,
                                                           double* __restrict__ ell_val, int32_t* __restrict__ ell_len) {
    const int64_t tiles = (N + 31) / 32;
    const int per = 32 * W;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t base = tile * per;
        for (int rem = threadIdx.x; rem < per; rem += blockDim.x) {
            const int j = rem >> 5, lane = rem & 31;
            const int64_t rn = tile * 32 + lane;
            int32_t ci = 0;
            double v = 0.0;
            if (rn < N) {
                const int64_t ro = order ? order[rn] : rn;
                const int32_t lo = indptr[ro], len = indptr[ro + 1] - lo;
                if (j == 0 && ell_len) ell_len[rn] = len;
                if (j < len) {
                    const int32_t c = indices[lo + j];
                    ci = inv ? inv[c] : c;
                    if (data) v = data[lo + j];
                }
            }
            if (ell_idx) ell_idx[base + rem] = ci;
            if (ell_val) ell_val[base + rem] = v;
        }
    }
}

__global__ void plan_gather(const double* __restrict__ src, const int32_t* __restrict__ order, int64_t N,
                            double* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[order[i]];
}

__global__ void plan_scatter(const double* __restrict__ src, const int32_t* __restrict__ order, int64_t N,
                             double* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        dst[order[i]] = src[i];
}

// row sums over the plan (thread per row, slot-major loads)
__global__ void __launch_bounds__(256) plan_apply_k(const int32_t* __restrict__ ell_idx,
                                                    const double* __restrict__ ell_val,
                                                    const int32_t* __restrict__ ell_len, int64_t N, int W,
                                                    const double* __restrict__ u, double* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        const int len = ell_len[r];
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double acc = 0.0;
#pragma unroll 5
        for (int j = 0; j < len; ++j) {
            const double a = __ldcs(ell_val + base + 32 * j);
            const int32_t c = __ldcs(ell_idx + base + 32 * j);
            acc = __dadd_rn(acc, __dmul_rn(a, __ldg(u + c)));
        }
        y[r] = acc;
    }
}

inline int grid_of(int64_t work, int threads, int per_sm = 8) { return grid_cap(work, threads, per_sm); }

// ---- operator combinations (storage.py:174-222) ------------------------------
// One pass over the shared index stream: per entry one column index, then per
// term one value and one field load; each term's sum runs in the row's addend
// order from 0.0 (separately rounded multiply and add), outputs add their terms
// in order onto 0.0.  NT = number of terms (compile time: the sums stay in
// registers); the plan variant scatters outputs to node order through `order`.
struct TermsDev {
    const double* val[MF_MAX_TERMS];
    const double* fld[MF_MAX_TERMS];
    double* out[MF_MAX_TERMS];
    int t0[MF_MAX_TERMS + 1];
    int nout;
};

template <int NT>
__device__ __forceinline__ void terms_finish(const TermsDev& T, const double (&s)[NT], int64_t dst) {
    for (int o = 0; o < T.nout; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (t >= T.t0[o] && t < T.t0[o + 1]) acc = __dadd_rn(acc, s[t]);
        T.out[o][dst] = acc;
    }
}

template <int NT>
__global__ void __launch_bounds__(256) plan_terms_k(const int32_t* __restrict__ ell_idx,
                                                    const int32_t* __restrict__ ell_len, int64_t N, int W,
                                                    const int32_t* __restrict__ order, const TermsDev T) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        const int len = ell_len[r];
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double s[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) s[t] = 0.0;
        for (int j = 0; j < len; ++j) {
            const int64_t e = base + 32 * j;
            const int32_t c = __ldcs(ell_idx + e);
#pragma unroll
            for (int t = 0; t < NT; ++t)
                s[t] = __dadd_rn(s[t], __dmul_rn(__ldcs(T.val[t] + e), __ldg(T.fld[t] + c)));
        }
        terms_finish<NT>(T, s, order ? (int64_t)order[r] : r);
    }
}
// every term reads the same field (several families of one operator applied to
// one field, WeightStore.apply_families): u[c] loaded once per entry, four
// entries in flight per row; each term's addends still in the row's order
template <int NT>
__global__ void __launch_bounds__(256) plan_terms1f_k(const int32_t* __restrict__ ell_idx,
                                                      const int32_t* __restrict__ ell_len, int64_t N, int W,
                                                      const int32_t* __restrict__ order, const TermsDev T) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double* __restrict__ u = T.fld[0];
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        const int len = ell_len[r];
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double s[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) s[t] = 0.0;
        int j = 0;
        for (; j + 4 <= len; j += 4) {
            int32_t c[4];
            double uc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = __ldcs(ell_idx + base + 32 * (j + q));
#pragma unroll
            for (int q = 0; q < 4; ++q) uc[q] = __ldg(u + c[q]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t e = base + 32 * (j + q);
#pragma unroll
                for (int t = 0; t < NT; ++t) s[t] = __dadd_rn(s[t], __dmul_rn(__ldcs(T.val[t] + e), uc[q]));
            }
        }
        for (; j < len; ++j) {
            const int64_t e = base + 32 * j;
            const double uc = __ldg(u + __ldcs(ell_idx + e));
#pragma unroll
            for (int t = 0; t < NT; ++t) s[t] = __dadd_rn(s[t], __dmul_rn(__ldcs(T.val[t] + e), uc));
        }
        terms_finish<NT>(T, s, order ? (int64_t)order[r] : r);
    }
}


template <int NT>
__global__ void __launch_bounds__(128) rows_terms_k(const int32_t* __restrict__ indptr,
                                                    const int32_t* __restrict__ indices,
                                                    const int64_t* __restrict__ sel, int64_t count, const TermsDev T) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
        const int64_t i = sel[k];
        double s[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) s[t] = 0.0;
        for (int32_t p = indptr[i]; p < indptr[i + 1]; ++p) {
            const int32_t c = indices[p];
#pragma unroll
            for (int t = 0; t < NT; ++t) s[t] = __dadd_rn(s[t], __dmul_rn(T.val[t][p], T.fld[t][c]));
        }
        terms_finish<NT>(T, s, k);
    }
}

}  // namespace mf

using namespace mf;

extern "C" int mf_order_workspace_size(int64_t N, size_t* bytes) {
    if (!bytes || N < 0) {
        set_error("mf_order_workspace_size: bad arguments");
        return MF_ERR_ARG;
    }
    size_t sort_bytes = 0;
    cub::DoubleBuffer<unsigned> k(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> v(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, k, v, (int)(N > 0 ? N : 1));
    Arena ar{nullptr, 0, 0, true};
    ar.take<unsigned long long>(6);
    ar.take<unsigned>(N);
    ar.take<unsigned>(N);
    ar.take<int32_t>(N);
    ar.take<char>(sort_bytes);
    *bytes = ar.off;
    return MF_OK;
}

extern "C" int mf_locality_order(const double* pos, int64_t N, int32_t d, int32_t* order, int32_t* inv, void* ws,
                                 size_t ws_bytes, void* stream) {
    MF_REQUIRE(d >= 1 && d <= MF_MAX_DIM && N >= 0 && N < 2147483647, "mf_locality_order: bad arguments");
    if (N == 0) return MF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    size_t sort_bytes = 0;
    cub::DoubleBuffer<unsigned> probe_k(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> probe_v(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, probe_k, probe_v, (int)N);
    Arena ar{(char*)ws, ws_bytes, 0, false};
    unsigned long long* bb = ar.take<unsigned long long>(6);
    unsigned* k0 = ar.take<unsigned>(N);
    unsigned* k1 = ar.take<unsigned>(N);
    int32_t* v0 = ar.take<int32_t>(N);
    char* tmp = ar.take<char>(sort_bytes);
    if (!ws || !ar.ok()) {
        set_error("mf_locality_order: workspace too small");
        return MF_ERR_WORKSPACE;
    }
    MF_CUDA_CHECK(cudaMemsetAsync(bb, 0xff, 3 * sizeof(unsigned long long), st));
    MF_CUDA_CHECK(cudaMemsetAsync(bb + 3, 0, 3 * sizeof(unsigned long long), st));
    plan_bbox<<<grid_of(N, 256, 4), 256, 0, st>>>(pos, N, d, bb);
    MF_LAUNCH_CHECK();
    plan_keys<<<grid_of(N, 256), 256, 0, st>>>(pos, N, d, bb, k0, v0);
    MF_LAUNCH_CHECK();
    cub::DoubleBuffer<unsigned> kb(k0, k1);
    cub::DoubleBuffer<int32_t> vb(v0, order);
    MF_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, kb, vb, (int)N, 0, 24, st));
    if (vb.Current() != order)
        MF_CUDA_CHECK(cudaMemcpyAsync(order, vb.Current(), sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
    if (inv) {
        plan_invert<<<grid_of(N, 256), 256, 0, st>>>(order, N, inv);
        MF_LAUNCH_CHECK();
    }
    return MF_OK;
}

extern "C" int mf_plan_build(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N, int32_t W,
                             const int32_t* order, const int32_t* inv, int32_t* ell_idx, double* ell_val,
                             int32_t* ell_len, void* stream) {
    MF_REQUIRE(N >= 0 && W >= 0 && (order != nullptr || inv == nullptr), "mf_plan_build: bad arguments");
    int64_t total = ((N + 31) / 32) * 32 * (int64_t)W;
    if (total == 0 && N == 0) return MF_OK;
    int64_t work = total > N ? total : N;
    // the tile build at 5 blocks per SM (C3 plan, order + ELL: 570 / 429 / 361 / 338
    // / 355 / 600 us at 2 / 3 / 4 / 5 / 6 / 8 blocks per SM, 444 us element-wise);
    // rows without a width (W = 0) only need their lengths
    if (W > 0)
        plan_ell_build_tile<<<grid_of((N + 31) / 32 * 256, 256, 5), 256, 0,
                              (cudaStream_t)stream>>>(indptr, indices, data, N, W, order, inv, ell_idx, ell_val,
                                                      ell_len);
    else
        plan_ell_build<<<grid_of(work, 256, 16), 256, 0, (cudaStream_t)stream>>>(indptr, indices, data, N, W, order,
                                                                                  inv, ell_idx, ell_val, ell_len);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_plan_apply(const int32_t* ell_idx, const double* ell_val, const int32_t* ell_len, int64_t N,
                             int32_t W, const int32_t* order, const double* u, double* y, double* scratch_u,
                             double* scratch_y, void* stream) {
    MF_REQUIRE(N >= 0 && W >= 0, "mf_plan_apply: bad arguments");
    if (N == 0) return MF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (!order) {
        plan_apply_k<<<grid_of(N, 256), 256, 0, st>>>(ell_idx, ell_val, ell_len, N, W, u, y);
        MF_LAUNCH_CHECK();
        return MF_OK;
    }
    MF_REQUIRE(scratch_u && scratch_y, "mf_plan_apply: an ordered plan needs two scratch vectors");
    plan_gather<<<grid_of(N, 256), 256, 0, st>>>(u, order, N, scratch_u);
    MF_LAUNCH_CHECK();
    plan_apply_k<<<grid_of(N, 256), 256, 0, st>>>(ell_idx, ell_val, ell_len, N, W, scratch_u, scratch_y);
    MF_LAUNCH_CHECK();
    plan_scatter<<<grid_of(N, 256), 256, 0, st>>>(scratch_y, order, N, y);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

namespace {
int terms_dev(const mf_terms_t* t, TermsDev& T) {
    MF_REQUIRE(t && t->nterm >= 1 && t->nterm <= MF_MAX_TERMS && t->nout >= 1 && t->nout <= MF_MAX_TERMS,
               "mf_*_terms: bad term / output counts");
    MF_REQUIRE(t->out_t0[0] == 0 && t->out_t0[t->nout] == t->nterm, "mf_*_terms: outputs must cover the terms in order");
    for (int o = 0; o < t->nout; ++o) {
        MF_REQUIRE(t->out_t0[o] <= t->out_t0[o + 1] && t->out[o], "mf_*_terms: bad output %d", o);
        T.out[o] = t->out[o];
        T.t0[o] = t->out_t0[o];
    }
    T.t0[t->nout] = t->out_t0[t->nout];
    for (int k = 0; k < t->nterm; ++k) {
        MF_REQUIRE(t->val[k] && t->fld[k], "mf_*_terms: term %d has no values or field", k);
        T.val[k] = t->val[k];
        T.fld[k] = t->fld[k];
    }
    for (int k = t->nterm; k < MF_MAX_TERMS; ++k) T.val[k] = T.val[0], T.fld[k] = T.fld[0];
    T.nout = t->nout;
    return MF_OK;
}

template <template <int> class L, class... A>
int dispatch_nt(int nt, A... a) {
    switch (nt) {
        case 1: return L<1>::go(a...);
        case 2: return L<2>::go(a...);
        case 3: return L<3>::go(a...);
        case 4: return L<4>::go(a...);
        case 5: case 6: return L<6>::go(a...);
        case 7: case 8: case 9: return L<9>::go(a...);
        default: return L<16>::go(a...);
    }
}

template <int NT>
struct PlanTermsL {
    static int go(const int32_t* idx, const int32_t* len, int64_t N, int W, const int32_t* order, const TermsDev* T,
                  cudaStream_t st) {
        bool one_field = true;
        for (int t = 1; t < NT; ++t) one_field = one_field && T->fld[t] == T->fld[0];
        if (one_field) plan_terms1f_k<NT><<<grid_of(N, 256), 256, 0, st>>>(idx, len, N, W, order, *T);
        else plan_terms_k<NT><<<grid_of(N, 256), 256, 0, st>>>(idx, len, N, W, order, *T);
        MF_LAUNCH_CHECK();
        return MF_OK;
    }
};
template <int NT>
struct RowsTermsL {
    static int go(const int32_t* ip, const int32_t* ix, const int64_t* sel, int64_t count, const TermsDev* T,
                  cudaStream_t st) {
        rows_terms_k<NT><<<grid_of(count, 128), 128, 0, st>>>(ip, ix, sel, count, *T);
        MF_LAUNCH_CHECK();
        return MF_OK;
    }
};
}  // namespace

extern "C" int mf_plan_apply_terms(const int32_t* ell_idx, const int32_t* ell_len, int64_t N, int32_t W,
                                   const int32_t* order, const mf_terms_t* terms, void* stream) {
    MF_REQUIRE(N >= 0 && W >= 0, "mf_plan_apply_terms: bad arguments");
    TermsDev T{};
    int rc = terms_dev(terms, T);
    if (rc != MF_OK || N == 0) return rc;
    // unused term slots (NT rounded up) add 0 * field to a sum nobody reads
    return dispatch_nt<PlanTermsL>(terms->nterm, ell_idx, ell_len, N, (int)W, order, (const TermsDev*)&T,
                                   (cudaStream_t)stream);
}

extern "C" int mf_apply_terms_rows(const int32_t* indptr, const int32_t* indices, const int64_t* sel, int64_t count,
                                   const mf_terms_t* terms, void* stream) {
    MF_REQUIRE(count >= 0, "mf_apply_terms_rows: bad count");
    TermsDev T{};
    int rc = terms_dev(terms, T);
    if (rc != MF_OK || count == 0) return rc;
    return dispatch_nt<RowsTermsL>(terms->nterm, indptr, indices, sel, count, (const TermsDev*)&T,
                                   (cudaStream_t)stream);
}

extern "C" int mf_permute(const double* src, const int32_t* order, int64_t N, int32_t scatter, double* dst,
                          void* stream) {
    MF_REQUIRE(N >= 0, "mf_permute: bad N");
    if (N == 0) return MF_OK;
    if (scatter) plan_scatter<<<grid_of(N, 256), 256, 0, (cudaStream_t)stream>>>(src, order, N, dst);
    else plan_gather<<<grid_of(N, 256), 256, 0, (cudaStream_t)stream>>>(src, order, N, dst);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

// rows in the plan's (Morton) order, columns in node numbering: the field is read
// in node order straight from L2 (it is N doubles) and each row's sum lands at
// y[order[r]] -- one launch, no permutes of the field or the result
__global__ void __launch_bounds__(256) plan_apply_direct_k(const int32_t* __restrict__ ell_idx,
                                                           const double* __restrict__ ell_val,
                                                           const int32_t* __restrict__ ell_len, int64_t N, int W,
                                                           const int32_t* __restrict__ order,
                                                           const double* __restrict__ u, double* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        const int len = ell_len[r];
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double acc = 0.0;
#pragma unroll 5
        for (int j = 0; j < len; ++j) {
            const double a = __ldcs(ell_val + base + 32 * j);
            const int32_t c = __ldcs(ell_idx + base + 32 * j);
            acc = __dadd_rn(acc, __dmul_rn(a, __ldg(u + c)));
        }
        y[order[r]] = acc;
    }
}

extern "C" int mf_plan_apply_direct(const int32_t* ell_idx, const double* ell_val, const int32_t* ell_len, int64_t N,
                                    int32_t W, const int32_t* order, const double* u, double* y, void* stream) {
    MF_REQUIRE(N >= 0 && W >= 0 && order, "mf_plan_apply_direct: bad arguments");
    if (N == 0) return MF_OK;
    plan_apply_direct_k<<<grid_of(N, 256), 256, 0, (cudaStream_t)stream>>>(ell_idx, ell_val, ell_len, N, W, order, u,
                                                                            y);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

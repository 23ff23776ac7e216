// Shared device helpers for the meshfree B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/meshfree_b200.h"

namespace mf {

constexpr unsigned FULL = 0xffffffffu;

// ---- error plumbing (host) --------------------------------------------------
void set_error(const char* fmt, ...);

#define MF_CUDA_CHECK(expr)                                                        \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::mf::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                            cudaGetErrorString(_e));                               \
            return MF_ERR_CUDA;                                                    \
        }                                                                          \
    } while (0)

void count_launch();

// Per-device properties, queried once per device (launchers size grids from them
// on every call; the runtime queries are not free on the enqueue path).
int dev_sms();            // multiprocessor count of the current device
int dev_max_smem_optin(); // opt-in dynamic shared memory per block
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device) and
// size; returns cudaSuccess or the error of the first call.
cudaError_t ensure_smem_attr(const void* kernel, int bytes);
template <class K>
inline cudaError_t ensure_smem(K* kernel, int bytes) { return ensure_smem_attr((const void*)kernel, bytes); }
// resident blocks per SM of (kernel, block size, dynamic smem), queried once
int occupancy_attr(const void* kernel, int threads, size_t smem);
template <class K>
inline int occupancy(K* kernel, int threads, size_t smem) { return occupancy_attr((const void*)kernel, threads, smem); }
// grid for a grid-stride kernel: ceil(work / threads) blocks, capped at per_sm per SM
inline int grid_cap(int64_t work, int threads, int per_sm) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)dev_sms() * per_sm;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}
#define MF_LAUNCH_CHECK()             \
    do {                              \
        ::mf::count_launch();         \
        MF_CUDA_CHECK(cudaGetLastError()); \
    } while (0)

#define MF_REQUIRE(cond, ...)                                                      \
    do {                                                                           \
        if (!(cond)) {                                                             \
            ::mf::set_error(__VA_ARGS__);                                          \
            return MF_ERR_ARG;                                                     \
        }                                                                          \
    } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
    char* base;
    size_t cap;
    size_t off = 0;
    bool dry;  // sizing pass: base may be null
    template <class T>
    T* take(size_t count) {
        size_t at = align_up(off);
        off = at + count * sizeof(T);
        return dry ? nullptr : reinterpret_cast<T*>(base + at);
    }
    bool ok() const { return dry || off <= cap; }
};

// ---- device helpers -----------------------------------------------------------

// Monotone map of a double onto uint64 (for atomic min/max over doubles).
// A value the compiler cannot prove loop-invariant: conditions on kernel
// parameters inside the big per-stencil loops would otherwise be unswitched,
// duplicating the whole loop body in the instruction cache.
__device__ __forceinline__ int opaque(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ unsigned long long ordered_bits(double x) {
    unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered_bits(unsigned long long u) {
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)u);
}

// Bounding-box reduction of a block (blockDim.x a multiple of 32, <= 1024): warp
// shuffles, then one warp over the per-warp partials, then one atomic per
// value and block on bb[0..d) (min) / bb[3..3+d) (max) as ordered bits --
// per-warp atomics on six addresses serialise at the L2.
__device__ __forceinline__ void block_bbox_commit(double mn[3], double mx[3], int d, unsigned long long* bb) {
    __shared__ double smn[3][32], smx[3][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int a = 0; a < d; ++a) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(FULL, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(FULL, mx[a], o));
        }
        if (lane == 0) {
            smn[a][w] = mn[a];
            smx[a][w] = mx[a];
        }
    }
    __syncthreads();
    if (w == 0) {
        for (int a = 0; a < d; ++a) {
            double vn = lane < nw ? smn[a][lane] : INFINITY, vx = lane < nw ? smx[a][lane] : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                vn = fmin(vn, __shfl_xor_sync(FULL, vn, o));
                vx = fmax(vx, __shfl_xor_sync(FULL, vx, o));
            }
            if (lane == 0) {
                atomicMin(&bb[a], ordered_bits(vn));
                atomicMax(&bb[3 + a], ordered_bits(vx));
            }
        }
    }
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// numba's integer power of a float base (numba/cpython/numbers.py int_power):
// r = 1; while e: if e & 1: r *= a; e >>= 1; a *= a.  Replayed op for op.
__device__ __forceinline__ double numba_int_power(double a, long long b) {
    double r = 1.0;
    bool inv = b < 0;
    unsigned long long e = (unsigned long long)(inv ? -b : b);
    while (e != 0) {
        if (e & 1) r = __dmul_rn(r, a);
        e >>= 1;
        a = __dmul_rn(a, a);
    }
    return inv ? __ddiv_rn(1.0, r) : r;
}

// ---- correctly rounded integer powers (stand-in for glibc pow) ---------------
// glibc's pow equals the correctly rounded result except in ~0.09% of calls
// (SURVEY.md §7 hard part 2); a double-double power is the closest portable
// reproduction.  Error of the unrounded double-double is ~1e-30 relative.
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    // explicit _rn intrinsics: the compiler must not contract these
    double p = __dmul_rn(a.hi, b.hi);
    double e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, e);
    e = fma(a.lo, b.hi, e);
    double s = __dadd_rn(p, e);
    return dd{s, __dsub_rn(e, __dsub_rn(s, p))};
}

__device__ __forceinline__ double pow_cr_int(double x, int k) {
    if (k == 0) return 1.0;
    if (k == 1) return x;
    if (k == -1) return __drcp_rn(x);
    int e = k < 0 ? -k : k;
    dd r{1.0, 0.0}, a{x, 0.0};
    bool first = true;
    while (e) {
        if (e & 1) {
            r = first ? a : dd_mul(r, a);
            first = false;
        }
        e >>= 1;
        if (e) a = dd_mul(a, a);
    }
    if (k > 0) return __dadd_rn(r.hi, r.lo);
    // 1 / (hi + lo), one Newton correction in double-double
    double q = __drcp_rn(r.hi);
    double t = fma(-r.hi, q, 1.0);
    t = fma(-r.lo, q, t);
    return fma(q, t, q);
}

}  // namespace mf

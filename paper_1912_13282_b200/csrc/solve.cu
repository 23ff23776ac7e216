// Implicit consumer of the weights, sm_100a:
//
//   mf_coo_to_csr     SparseSystem.finalize (assembly.py:91-108): committed rows
//                     (COO in commit order) -> canonical CSR, rows ascending,
//                     columns ascending
//   mf_assemble_rows  the row loop of solve_poisson_implicit (drivers.py:138-154)
//                     in one pass over a weight store's canonical structure:
//                     interior rows (term combinations), Dirichlet rows (1 on
//                     the diagonal), Neumann rows (normal combinations)
//   mf_color          Jones-Plassmann colouring of the symmetrised pattern
//   mf_ilu0_build     ILU(0) of the system in colour order (rows of one colour
//                     never couple, so each colour factors in parallel)
//   mf_ilu0_apply     M^-1 x: forward / backward substitution colour by colour
//   mf_bicgstab       scipy's bicgstab recurrence (solve.py:65-108 calls it)
//                     on the device, the host loop reading the scalars it
//                     branches on
//
// The reference preconditions with SuperLU's ILUT (spilu, solve.py:49-62),
// a sequential factorisation; the GPU substitutes ILU(0) in a parallel
// (multicolour) order.  Both converge BiCGStab to the same relative residual
// (rtol), so solutions agree to cond(A) * rtol, not bitwise.
#include <cfloat>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace mf {
namespace {

__device__ __forceinline__ unsigned prio_hash(unsigned i) {
    unsigned h = i * 0x9E3779B1u;
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    return h;
}
// strict order on (hash, index)
__device__ __forceinline__ bool higher(int a, int b) {
    const unsigned ha = prio_hash((unsigned)a), hb = prio_hash((unsigned)b);
    return ha > hb || (ha == hb && a > b);
}

// ---- COO -> canonical CSR ---------------------------------------------------
__global__ void coo_count_k(const int32_t* __restrict__ rows, int64_t nnz, int32_t* counts) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(counts + rows[e], 1);
}
__global__ void coo_scatter_k(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                              const double* __restrict__ vals, int64_t nnz, const int32_t* __restrict__ indptr,
                              int32_t* cursor, int32_t* indices, double* data) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = rows[e];
        const int at = indptr[r] + atomicAdd(cursor + r, 1);
        indices[at] = cols[e];
        data[at] = vals[e];
    }
}
// per-row insertion sort by column (columns are distinct within a row, so the
// result does not depend on the scatter order)
__global__ void row_sort_k(const int32_t* __restrict__ indptr, int64_t N, int32_t* indices, double* data) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        const int a = indptr[r], b = indptr[r + 1];
        for (int i = a + 1; i < b; ++i) {
            const int c = indices[i];
            const double v = data[i];
            int j = i - 1;
            while (j >= a && indices[j] > c) {
                indices[j + 1] = indices[j];
                data[j + 1] = data[j];
                --j;
            }
            indices[j + 1] = c;
            data[j + 1] = v;
        }
    }
}

// ---- batched assembly ---------------------------------------------------------
// kind: 1 interior, 2 Dirichlet, 3 Neumann.  Row lengths first.
__global__ void asm_len_k(const int32_t* __restrict__ s_indptr, const int8_t* __restrict__ kind, int64_t N,
                          int32_t* len, unsigned long long* missing) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = kind[i];
        int l = 0;
        if (k == 2) {
            l = 1;
        } else if (k == 1 || k == 3) {
            l = s_indptr[i + 1] - s_indptr[i];
            if (l == 0) atomicMin(missing, (unsigned long long)i);
        } else {
            atomicMin(missing, (unsigned long long)i);
        }
        len[i] = l;
    }
}
__global__ void asm_fill_k(const int32_t* __restrict__ s_indptr, const int32_t* __restrict__ s_indices,
                           const int32_t* __restrict__ s_perm, const double* __restrict__ v_int,
                           const double* __restrict__ v_neu, const int64_t* __restrict__ neu_row,
                           const int8_t* __restrict__ kind, int64_t N, int32_t n, const int32_t* __restrict__ indptr,
                           int32_t* indices, double* data) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = kind[i];
        const int o = indptr[i];
        if (k == 2) {
            indices[o] = (int32_t)i;
            data[o] = 1.0;
        } else if (k == 1 || k == 3) {
            const int a = s_indptr[i], b = s_indptr[i + 1];
            for (int p = a; p < b; ++p) {
                indices[o + p - a] = s_indices[p];
                const int src = s_perm[p];  // stencil-order slot (store row * n + j)
                data[o + p - a] = k == 1 ? v_int[src] : v_neu[neu_row[i] * n + (src % n)];
            }
        }
    }
}

// ---- Jones-Plassmann colouring --------------------------------------------------
// a node is blocked in round `rnd` when some uncoloured node of higher priority
// lists it in its row (the reverse direction of the pattern)
__global__ void jp_block_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t N,
                           const int32_t* __restrict__ color, int32_t* blocked, int rnd) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        if (color[j] >= 0) continue;
        for (int p = indptr[j]; p < indptr[j + 1]; ++p) {
            const int k = indices[p];
            if (k != j && color[k] < 0 && higher((int)j, k)) blocked[k] = rnd;
        }
    }
}
__global__ void jp_pick_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t N,
                          int32_t* color, const int32_t* __restrict__ blocked, unsigned long long* forbid, int rnd,
                          unsigned long long* left, int* overflow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (color[i] >= 0) continue;
        bool ok = blocked[i] != rnd;
        unsigned long long m0 = forbid[2 * i], m1 = forbid[2 * i + 1];
        for (int p = indptr[i]; ok && p < indptr[i + 1]; ++p) {
            const int k = indices[p];
            if (k == i) continue;
            const int ck = color[k];
            if (ck < 0) {
                if (higher(k, (int)i)) ok = false;
            } else if (ck < 64) {
                m0 |= 1ull << ck;
            } else {
                m1 |= 1ull << (ck - 64);
            }
        }
        if (!ok) {
            atomicAdd(left, 1ull);
            continue;
        }
        int c;
        if (~m0) c = __ffsll((long long)~m0) - 1;
        else if (~m1) c = 64 + __ffsll((long long)~m1) - 1;
        else {
            *overflow = 1;
            c = 127;
        }
        color[i] = c;
        for (int p = indptr[i]; p < indptr[i + 1]; ++p) {
            const int k = indices[p];
            if (k != i) atomicOr(forbid + 2 * k + (c >= 64), 1ull << (c & 63));
        }
    }
}
__global__ void color_hist_k(const int32_t* __restrict__ color, int64_t N, int32_t* hist) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + color[i], 1);
}
__global__ void color_scatter_k(const int32_t* __restrict__ color, int64_t N, const int32_t* __restrict__ off,
                                int32_t* cursor, int32_t* order) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = color[i];
        order[off[c] + atomicAdd(cursor + c, 1)] = (int32_t)i;
    }
}

// ---- ILU(0) in colour order ------------------------------------------------------
// part[p] = -1 (L: earlier colour), 0 (diagonal), +1 (U: later colour)
__global__ void ilu_part_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const int32_t* __restrict__ color, int64_t N, int8_t* part, int32_t* diag,
                           unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int ci = color[i];
        int dg = -1;
        for (int p = indptr[i]; p < indptr[i + 1]; ++p) {
            const int k = indices[p];
            if (k == i) {
                part[p] = 0;
                dg = p;
            } else {
                part[p] = color[k] < ci ? -1 : 1;
            }
        }
        diag[i] = dg;
        if (dg < 0) atomicMin(bad, (unsigned long long)i);
    }
}
__device__ __forceinline__ int find_col(const int32_t* __restrict__ idx, int a, int b, int c) {
    while (a < b) {
        const int m = (a + b) >> 1;
        const int v = idx[m];
        if (v < c) a = m + 1;
        else b = m;
    }
    return a;
}
// rows of colour c: IKJ update over the L entries in increasing colour order
__global__ void ilu_color_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* __restrict__ color, const int8_t* __restrict__ part,
                            const int32_t* __restrict__ diag, const int32_t* __restrict__ rows, int cnt, double* lu) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const int i = rows[t];
        const int a = indptr[i], b = indptr[i + 1];
        const int ci = color[i];
        for (int cc = 0; cc < ci; ++cc) {
            for (int p = a; p < b; ++p) {
                if (part[p] >= 0) continue;
                const int k = indices[p];
                if (color[k] != cc) continue;
                const double lik = lu[p] / lu[diag[k]];
                lu[p] = lik;
                for (int q = indptr[k]; q < indptr[k + 1]; ++q) {
                    if (part[q] <= 0) continue;  // U part of row k
                    const int j = indices[q];
                    const int at = find_col(indices, a, b, j);
                    if (at < b && indices[at] == j) lu[at] -= lik * lu[q];
                }
            }
        }
    }
}
__global__ void ilu_fwd_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                          const int8_t* __restrict__ part, const double* __restrict__ lu,
                          const int32_t* __restrict__ rows, int cnt, const double* __restrict__ x, double* y) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const int i = rows[t];
        double acc = x[i];
        for (int p = indptr[i]; p < indptr[i + 1]; ++p)
            if (part[p] < 0) acc -= lu[p] * y[indices[p]];
        y[i] = acc;
    }
}
__global__ void ilu_bwd_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                          const int8_t* __restrict__ part, const double* __restrict__ lu,
                          const int32_t* __restrict__ diag, const int32_t* __restrict__ rows, int cnt, double* y) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const int i = rows[t];
        double acc = y[i];
        for (int p = indptr[i]; p < indptr[i + 1]; ++p)
            if (part[p] > 0) acc -= lu[p] * y[indices[p]];
        y[i] = acc / lu[diag[i]];
    }
}

// ---- BiCGStab vector kernels ------------------------------------------------------
constexpr int RED_BLOCKS = 296, RED_THREADS = 256;

// partial[b] = sum over the block's strided slice of a.b (fixed grid: deterministic)
__global__ void __launch_bounds__(RED_THREADS) dot_partial_k(const double* __restrict__ a, const double* __restrict__ b,
                                                             int64_t N, double* partial) {
    __shared__ double sm[RED_THREADS / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < N; i += (int64_t)RED_BLOCKS * RED_THREADS)
        s = fma(a[i], b[i], s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < RED_THREADS / 32 ? sm[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}
__global__ void dot_final_k(const double* __restrict__ partial, double* out) {
    __shared__ double sm[RED_BLOCKS];
    for (int i = threadIdx.x; i < RED_BLOCKS; i += blockDim.x) sm[i] = partial[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < RED_BLOCKS; ++i) s += sm[i];
        *out = s;
    }
}
// r = b - A x (A x row by row in storage order, as csr_matvec)
__global__ void resid_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                        const double* __restrict__ data, const double* __restrict__ x, const double* __restrict__ b,
                        int64_t N, double* r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int p = indptr[i]; p < indptr[i + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(data[p], x[indices[p]]));
        r[i] = __dsub_rn(b[i], acc);
    }
}
__global__ void spmv_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                       const double* __restrict__ data, const double* __restrict__ x, int64_t N, double* y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int p = indptr[i]; p < indptr[i + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(data[p], x[indices[p]]));
        y[i] = acc;
    }
}
// numpy's in-place updates, one rounding per operation
__global__ void copy2_k(const double* __restrict__ a, int64_t N, double* b, double* c) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        b[i] = a[i];
        if (c) c[i] = a[i];
    }
}
__global__ void p_update_k(double* p, const double* __restrict__ v, const double* __restrict__ r, double omega,
                           double beta, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = __dadd_rn(__dmul_rn(__dsub_rn(p[i], __dmul_rn(omega, v[i])), beta), r[i]);
}
__global__ void axmy_k(double* r, const double* __restrict__ v, double alpha, int64_t N) {  // r -= alpha v
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = __dsub_rn(r[i], __dmul_rn(alpha, v[i]));
}
__global__ void xupd_k(double* x, const double* __restrict__ ph, double alpha, const double* __restrict__ sh,
                       double omega, int64_t N) {  // x += alpha phat; x += omega shat
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double t = __dadd_rn(x[i], __dmul_rn(alpha, ph[i]));
        if (sh) t = __dadd_rn(t, __dmul_rn(omega, sh[i]));
        x[i] = t;
    }
}

inline int vgrid(int64_t N) { return grid_cap(N, 256, 8); }

// ---- device-controlled iteration (graph-capturable) ---------------------------
// The same recurrence with every branch decided on the device: the scalars
// live in a BicgState, every kernel returns at once when `done` is set, so a
// graph of one iteration can be replayed any number of times past convergence
// without changing a bit.
struct BicgState {
    double atol, rho, rho_prev, alpha, omega, beta, rr, rv, ts, tt;
    long long it, maxiter;
    int done;   // 0 running, 1 finished
    int info;   // scipy's info once done
    int phase;  // (unused padding)
};

__device__ __forceinline__ double dot_sum(const double* __restrict__ partial) {
    double s = 0.0;
    for (int i = 0; i < RED_BLOCKS; ++i) s += partial[i];
    return s;
}
__global__ void __launch_bounds__(RED_THREADS) dot2_partial_k(const double* __restrict__ a, const double* __restrict__ b,
                                                              const double* __restrict__ c, const double* __restrict__ e,
                                                              int64_t N, double* partial, const BicgState* stt) {
    if (stt->done) return;
    __shared__ double sm[2][RED_THREADS / 32];
    double s0 = 0.0, s1 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < N; i += (int64_t)RED_BLOCKS * RED_THREADS) {
        s0 = fma(a[i], b[i], s0);
        if (c) s1 = fma(c[i], e[i], s1);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s0 += __shfl_xor_sync(FULL, s0, o);
        s1 += __shfl_xor_sync(FULL, s1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sm[0][threadIdx.x >> 5] = s0;
        sm[1][threadIdx.x >> 5] = s1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        s0 = threadIdx.x < RED_THREADS / 32 ? sm[0][threadIdx.x] : 0.0;
        s1 = threadIdx.x < RED_THREADS / 32 ? sm[1][threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            s0 += __shfl_xor_sync(FULL, s0, o);
            s1 += __shfl_xor_sync(FULL, s1, o);
        }
        if (threadIdx.x == 0) {
            partial[blockIdx.x] = s0;
            partial[RED_BLOCKS + blockIdx.x] = s1;
        }
    }
}
// step 1: ||r||, rho = (rt, r); the stop / breakdown tests and beta
__global__ void bicg_head_k(const double* __restrict__ partial, BicgState* stt) {
    if (threadIdx.x || stt->done) return;
    const double rr = dot_sum(partial), rho = dot_sum(partial + RED_BLOCKS);
    stt->rr = rr;
    if (stt->it >= stt->maxiter) {
        stt->done = 1;
        stt->info = (int)(stt->maxiter > 2147483647LL ? 2147483647LL : stt->maxiter);
        return;
    }
    if (sqrt(rr) < stt->atol) {
        stt->done = 1;
        stt->info = 0;
        return;
    }
    if (fabs(rho) < DBL_EPSILON * DBL_EPSILON) {
        stt->done = 1;
        stt->info = -10;
        return;
    }
    if (stt->it > 0) {
        if (fabs(stt->omega) < DBL_EPSILON * DBL_EPSILON) {
            stt->done = 1;
            stt->info = -11;
            return;
        }
        stt->beta = (rho / stt->rho_prev) * (stt->alpha / stt->omega);
    }
    stt->rho = rho;
}
__global__ void bicg_p_k(double* p, const double* __restrict__ v, const double* __restrict__ r, int64_t N,
                         const BicgState* stt) {
    if (stt->done) return;
    const bool first = stt->it == 0;
    const double om = stt->omega, be = stt->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = first ? r[i] : __dadd_rn(__dmul_rn(__dsub_rn(p[i], __dmul_rn(om, v[i])), be), r[i]);
}
// step 2: rv = (rt, v), alpha
__global__ void bicg_alpha_k(const double* __restrict__ partial, BicgState* stt) {
    if (threadIdx.x || stt->done) return;
    const double rv = dot_sum(partial);
    stt->rv = rv;
    if (rv == 0.0) {
        stt->done = 1;
        stt->info = -11;
        return;
    }
    stt->alpha = stt->rho / rv;
}
__global__ void bicg_axmy_k(double* r, const double* __restrict__ v, int64_t N, const BicgState* stt, int which) {
    if (stt->done) return;
    const double a = which == 0 ? stt->alpha : stt->omega;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = __dsub_rn(r[i], __dmul_rn(a, v[i]));
}
// step 3: ||s||: the half-step exit (x += alpha phat) decided here, applied by bicg_x_k
__global__ void bicg_mid_k(const double* __restrict__ partial, BicgState* stt) {
    if (threadIdx.x || stt->done) return;
    const double ss = dot_sum(partial);
    stt->rr = ss;
    if (sqrt(ss) < stt->atol) {
        stt->done = 2;  // half step: x += alpha phat still to apply
        stt->info = 0;
    }
}
__global__ void bicg_xhalf_k(double* x, const double* __restrict__ ph, int64_t N, BicgState* stt) {
    if (stt->done != 2) return;
    const double a = stt->alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], __dmul_rn(a, ph[i]));
}
__global__ void bicg_xhalf_done_k(BicgState* stt) {
    if (threadIdx.x == 0 && stt->done == 2) stt->done = 1;
}
// step 4: omega = (t, s) / (t, t)
__global__ void bicg_omega_k(const double* __restrict__ partial, BicgState* stt) {
    if (threadIdx.x || stt->done) return;
    stt->ts = dot_sum(partial);
    stt->tt = dot_sum(partial + RED_BLOCKS);
    stt->omega = stt->ts / stt->tt;
}
__global__ void bicg_x_k(double* x, const double* __restrict__ ph, const double* __restrict__ sh, int64_t N,
                         const BicgState* stt) {
    if (stt->done) return;
    const double a = stt->alpha, om = stt->omega;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(a, ph[i])), __dmul_rn(om, sh[i]));
}
__global__ void bicg_tail_k(BicgState* stt) {
    if (threadIdx.x || stt->done) return;
    stt->rho_prev = stt->rho;
    stt->it += 1;
}
// ILU(0) substitutions and products that stop with the iteration
__global__ void ilu_fwd_ctl_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                              const int8_t* __restrict__ part, const double* __restrict__ lu,
                              const int32_t* __restrict__ rows, int cnt, const double* __restrict__ x, double* y,
                              const BicgState* stt) {
    if (stt->done) return;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const int i = rows[t];
        double acc = x[i];
        for (int p = indptr[i]; p < indptr[i + 1]; ++p)
            if (part[p] < 0) acc -= lu[p] * y[indices[p]];
        y[i] = acc;
    }
}
__global__ void ilu_bwd_ctl_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                              const int8_t* __restrict__ part, const double* __restrict__ lu,
                              const int32_t* __restrict__ diag, const int32_t* __restrict__ rows, int cnt, double* y,
                              const BicgState* stt) {
    if (stt->done) return;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const int i = rows[t];
        double acc = y[i];
        for (int p = indptr[i]; p < indptr[i + 1]; ++p)
            if (part[p] > 0) acc -= lu[p] * y[indices[p]];
        y[i] = acc / lu[diag[i]];
    }
}
__global__ void spmv_ctl_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const double* __restrict__ data, const double* __restrict__ x, int64_t N, double* y,
                           const BicgState* stt) {
    if (stt->done) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int p = indptr[i]; p < indptr[i + 1]; ++p) acc = __dadd_rn(acc, __dmul_rn(data[p], x[indices[p]]));
        y[i] = acc;
    }
}
__global__ void copy_ctl_k(const double* __restrict__ a, int64_t N, double* b, const BicgState* stt) {
    if (stt->done) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
__global__ void bicg_init_k(const double* __restrict__ partial, BicgState* stt, double rtol, double atol,
                            long long maxiter) {
    if (threadIdx.x) return;
    const double bn = sqrt(dot_sum(partial));
    stt->atol = fmax(atol, rtol * bn);
    stt->it = 0;
    stt->maxiter = maxiter;
    stt->done = bn == 0.0 ? 3 : 0;  // 3: b == 0 (x = b, handled by the host)
    stt->info = 0;
    stt->rho_prev = stt->alpha = stt->omega = stt->beta = 0.0;
}

}  // namespace

// ILU(0) application (shared by mf_ilu0_apply and mf_bicgstab)
int ilu0_apply(const mf_ilu0_t* M, const double* x, double* y, cudaStream_t st) {
    for (int c = 0; c < M->ncolors; ++c) {
        const int a = M->color_off[c], cnt = M->color_off[c + 1] - a;
        if (cnt <= 0) continue;
        ilu_fwd_k<<<grid_cap(cnt, 128, 16), 128, 0, st>>>(M->indptr, M->indices, M->part, M->lu, M->order + a, cnt, x,
                                                          y);
        MF_LAUNCH_CHECK();
    }
    for (int c = M->ncolors - 1; c >= 0; --c) {
        const int a = M->color_off[c], cnt = M->color_off[c + 1] - a;
        if (cnt <= 0) continue;
        ilu_bwd_k<<<grid_cap(cnt, 128, 16), 128, 0, st>>>(M->indptr, M->indices, M->part, M->lu, M->diag, M->order + a,
                                                          cnt, y);
        MF_LAUNCH_CHECK();
    }
    return MF_OK;
}

}  // namespace mf

using namespace mf;

extern "C" int mf_assemble_workspace_size(int64_t N, size_t* bytes) {
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    *bytes = align_up((size_t)(N + 1) * 4) + align_up(scan) + 256;
    return MF_OK;
}

extern "C" int mf_coo_workspace_size(int64_t N, size_t* bytes) {
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    *bytes = align_up((size_t)(N + 1) * 4) * 2 + align_up(scan) + 256;
    return MF_OK;
}

extern "C" int mf_coo_to_csr(const int32_t* rows, const int32_t* cols, const double* vals, int64_t nnz, int64_t N,
                             int32_t* indptr, int32_t* indices, double* data, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(N >= 0 && nnz >= 0 && N < INT32_MAX && nnz < INT32_MAX, "mf_coo_to_csr: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    int32_t* counts = ar.take<int32_t>(N + 1);
    int32_t* cursor = ar.take<int32_t>(N + 1);
    void* tmp = ar.take<char>(scan);
    MF_REQUIRE(ar.ok() && ws, "mf_coo_to_csr: workspace too small");
    MF_CUDA_CHECK(cudaMemsetAsync(counts, 0, (N + 1) * 4, st));
    MF_CUDA_CHECK(cudaMemsetAsync(cursor, 0, (N + 1) * 4, st));
    if (nnz) {
        coo_count_k<<<grid_cap(nnz, 256, 8), 256, 0, st>>>(rows, nnz, counts);
        MF_LAUNCH_CHECK();
    }
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, scan, counts, indptr, (int)(N + 1), st));
    if (nnz) {
        coo_scatter_k<<<grid_cap(nnz, 256, 8), 256, 0, st>>>(rows, cols, vals, nnz, indptr, cursor, indices, data);
        MF_LAUNCH_CHECK();
    }
    if (N) {
        row_sort_k<<<vgrid(N), 256, 0, st>>>(indptr, N, indices, data);
        MF_LAUNCH_CHECK();
    }
    return MF_OK;
}

extern "C" int mf_assemble_rows(const int32_t* s_indptr, const int8_t* kind, int64_t N, int32_t* indptr,
                                int64_t* missing, int64_t* nnz_out, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(N >= 0 && N < INT32_MAX, "mf_assemble_rows: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    int32_t* len = ar.take<int32_t>(N + 1);
    void* tmp = ar.take<char>(scan);
    MF_REQUIRE(ar.ok() && ws, "mf_assemble_rows: workspace too small");
    MF_CUDA_CHECK(cudaMemsetAsync(missing, 0x7f, 8, st));
    MF_CUDA_CHECK(cudaMemsetAsync(len + N, 0, 4, st));
    if (N) {
        asm_len_k<<<vgrid(N), 256, 0, st>>>(s_indptr, kind, N, len, reinterpret_cast<unsigned long long*>(missing));
        MF_LAUNCH_CHECK();
    }
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, scan, len, indptr, (int)(N + 1), st));
    int32_t total = 0;
    MF_CUDA_CHECK(cudaMemcpyAsync(&total, indptr + N, 4, cudaMemcpyDeviceToHost, st));
    MF_CUDA_CHECK(cudaStreamSynchronize(st));
    *nnz_out = total;
    return MF_OK;
}

extern "C" int mf_assemble_fill(const int32_t* s_indptr, const int32_t* s_indices, const int32_t* s_perm, int32_t n,
                                const double* v_interior, const double* v_neumann, const int64_t* neumann_row,
                                const int8_t* kind, int64_t N, const int32_t* indptr, int32_t* indices, double* data,
                                void* stream) {
    MF_REQUIRE(N >= 0 && n >= 1, "mf_assemble_fill: bad sizes");
    if (N == 0) return MF_OK;
    asm_fill_k<<<vgrid(N), 256, 0, (cudaStream_t)stream>>>(s_indptr, s_indices, s_perm, v_interior, v_neumann,
                                                             neumann_row, kind, N, n, indptr, indices, data);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_ilu0_workspace_size(int64_t N, size_t* bytes) {
    *bytes = align_up((size_t)N * 4) * 2 + align_up((size_t)N * 16) + align_up(4 * 130) * 2 + 1024;
    return MF_OK;
}

// colours + colour-ordered rows + ILU(0) factors.  Caller-owned outputs:
// color (N int32), order (N int32), part (nnz int8), diag (N int32), lu (nnz f64);
// M is filled with the pointers and the colour offsets (host).
extern "C" int mf_ilu0_build(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N, int64_t nnz,
                             int32_t* color, int32_t* order, int8_t* part, int32_t* diag, double* lu, mf_ilu0_t* M,
                             int64_t* zero_pivot_row, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(N >= 1 && N < INT32_MAX && nnz >= N && M, "mf_ilu0_build: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    int32_t* blocked = ar.take<int32_t>(N);
    int32_t* cursor = ar.take<int32_t>(N);  // (colour cursors: first 130 entries)
    unsigned long long* forbid = ar.take<unsigned long long>(2 * N);
    int32_t* hist = ar.take<int32_t>(130);
    int32_t* off = ar.take<int32_t>(130);
    unsigned long long* ctl = ar.take<unsigned long long>(4);  // left, overflow, bad
    MF_REQUIRE(ar.ok() && ws, "mf_ilu0_build: workspace too small");
    MF_CUDA_CHECK(cudaMemsetAsync(color, 0xff, N * 4, st));
    MF_CUDA_CHECK(cudaMemsetAsync(blocked, 0, N * 4, st));
    MF_CUDA_CHECK(cudaMemsetAsync(forbid, 0, N * 16, st));
    MF_CUDA_CHECK(cudaMemsetAsync(ctl, 0, 32, st));
    const int g = vgrid(N);
    int rounds = 0;
    for (;; ++rounds) {
        MF_REQUIRE(rounds < 4096, "mf_ilu0_build: colouring did not finish");
        MF_CUDA_CHECK(cudaMemsetAsync(ctl, 0, 8, st));
        jp_block_k<<<g, 256, 0, st>>>(indptr, indices, N, color, blocked, rounds + 1);
        MF_LAUNCH_CHECK();
        jp_pick_k<<<g, 256, 0, st>>>(indptr, indices, N, color, blocked, forbid, rounds + 1, ctl,
                                     reinterpret_cast<int*>(ctl + 1));
        MF_LAUNCH_CHECK();
        unsigned long long h[2];
        MF_CUDA_CHECK(cudaMemcpyAsync(h, ctl, 16, cudaMemcpyDeviceToHost, st));
        MF_CUDA_CHECK(cudaStreamSynchronize(st));
        MF_REQUIRE(h[1] == 0, "mf_ilu0_build: more than 128 colours");
        if (h[0] == 0) break;
    }
    // colour-major row order
    MF_CUDA_CHECK(cudaMemsetAsync(hist, 0, 130 * 4, st));
    color_hist_k<<<g, 256, 0, st>>>(color, N, hist);
    MF_LAUNCH_CHECK();
    int hh[130];
    MF_CUDA_CHECK(cudaMemcpyAsync(hh, hist, 128 * 4, cudaMemcpyDeviceToHost, st));
    MF_CUDA_CHECK(cudaStreamSynchronize(st));
    int nc = 0;
    M->color_off[0] = 0;
    for (int c = 0; c < 128; ++c) {
        if (hh[c]) nc = c + 1;
        M->color_off[c + 1] = M->color_off[c] + hh[c];
    }
    M->ncolors = nc;
    MF_CUDA_CHECK(cudaMemcpyAsync(off, M->color_off, 129 * 4, cudaMemcpyHostToDevice, st));
    MF_CUDA_CHECK(cudaMemsetAsync(cursor, 0, 130 * 4, st));
    color_scatter_k<<<g, 256, 0, st>>>(color, N, off, cursor, order);
    MF_LAUNCH_CHECK();
    // L / diagonal / U split, then the factorisation colour by colour
    MF_CUDA_CHECK(cudaMemsetAsync(ctl + 2, 0x7f, 8, st));
    ilu_part_k<<<g, 256, 0, st>>>(indptr, indices, color, N, part, diag, ctl + 2);
    MF_LAUNCH_CHECK();
    MF_CUDA_CHECK(cudaMemcpyAsync(lu, data, nnz * 8, cudaMemcpyDeviceToDevice, st));
    for (int c = 1; c < nc; ++c) {
        const int a = M->color_off[c], cnt = M->color_off[c + 1] - a;
        if (cnt <= 0) continue;
        ilu_color_k<<<grid_cap(cnt, 128, 16), 128, 0, st>>>(indptr, indices, color, part, diag, order + a, cnt, lu);
        MF_LAUNCH_CHECK();
    }
    MF_CUDA_CHECK(cudaMemcpyAsync(zero_pivot_row, ctl + 2, 8, cudaMemcpyDeviceToDevice, st));
    M->indptr = indptr;
    M->indices = indices;
    M->part = part;
    M->diag = diag;
    M->lu = lu;
    M->order = order;
    M->rounds = rounds + 1;
    return MF_OK;
}

extern "C" int mf_ilu0_apply(const mf_ilu0_t* M, const double* x, double* y, void* stream) {
    MF_REQUIRE(M && M->ncolors >= 1, "mf_ilu0_apply: no factorisation");
    return ilu0_apply(M, x, y, (cudaStream_t)stream);
}

extern "C" int mf_bicgstab_workspace_size(int64_t N, size_t* bytes) {
    *bytes = align_up((size_t)N * 8) * 7 + align_up(2 * RED_BLOCKS * 8) + 1024;
    return MF_OK;
}

// scipy.sparse.linalg.bicgstab (scipy 1.18, _isolve/iterative.py) with x0 = x on
// entry; atol_eff = max(atol, rtol ||b||).  info: 0 converged, -10 rho breakdown,
// -11 omega / rv breakdown, maxiter when exhausted; *iterations counts the
// completed iterations (the reference's callback count).
extern "C" int mf_bicgstab(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N,
                           const mf_ilu0_t* M, const double* b, double* x, double rtol, double atol, int64_t maxiter,
                           int64_t* iterations, int32_t* info, double* residual_norm, void* ws, size_t ws_bytes,
                           void* stream) {
    MF_REQUIRE(N >= 1 && maxiter >= 0, "mf_bicgstab: bad sizes");
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    double* r = ar.take<double>(N);
    double* rt = ar.take<double>(N);
    double* p = ar.take<double>(N);
    double* v = ar.take<double>(N);
    double* ph = ar.take<double>(N);
    double* sh = ar.take<double>(N);
    double* t = ar.take<double>(N);
    double* partial = ar.take<double>(RED_BLOCKS);
    double* sc = ar.take<double>(8);
    MF_REQUIRE(ar.ok() && ws, "mf_bicgstab: workspace too small");
    const int g = vgrid(N);
    auto dot = [&](const double* a, const double* bb, double* out) -> int {
        dot_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, bb, N, partial);
        MF_LAUNCH_CHECK();
        dot_final_k<<<1, 256, 0, st>>>(partial, out);
        MF_LAUNCH_CHECK();
        return MF_OK;
    };
    auto fetch = [&](double* h, int cnt) -> int {
        MF_CUDA_CHECK(cudaMemcpyAsync(h, sc, cnt * 8, cudaMemcpyDeviceToHost, st));
        MF_CUDA_CHECK(cudaStreamSynchronize(st));
        return MF_OK;
    };
    auto precond = [&](const double* in, double* out) -> int {
        if (M) return ilu0_apply(M, in, out, st);
        copy2_k<<<g, 256, 0, st>>>(in, N, out, nullptr);
        MF_LAUNCH_CHECK();
        return MF_OK;
    };
#define MF_TRY(e)                \
    do {                         \
        int _rc = (e);           \
        if (_rc != MF_OK) return _rc; \
    } while (0)
    double h[4];
    MF_TRY(dot(b, b, sc));
    MF_TRY(fetch(h, 1));
    const double bnrm2 = sqrt(h[0]);
    *iterations = 0;
    *info = 0;
    if (bnrm2 == 0.0) {
        copy2_k<<<g, 256, 0, st>>>(b, N, x, nullptr);
        MF_LAUNCH_CHECK();
        *residual_norm = 0.0;
        return MF_OK;
    }
    const double atol_eff = fmax(atol, rtol * bnrm2);
    const double rhotol = DBL_EPSILON * DBL_EPSILON, omegatol = rhotol;
    resid_k<<<g, 256, 0, st>>>(indptr, indices, data, x, b, N, r);
    MF_LAUNCH_CHECK();
    copy2_k<<<g, 256, 0, st>>>(r, N, rt, nullptr);
    MF_LAUNCH_CHECK();
    double rho_prev = 0.0, omega = 0.0, alpha = 0.0;
    int64_t it = 0;
    for (; it < maxiter; ++it) {
        MF_TRY(dot(r, r, sc));
        MF_TRY(dot(rt, r, sc + 1));
        MF_TRY(fetch(h, 2));
        *residual_norm = sqrt(h[0]);
        if (sqrt(h[0]) < atol_eff) {
            *iterations = it;
            return MF_OK;
        }
        const double rho = h[1];
        if (fabs(rho) < rhotol) {
            *info = -10;
            *iterations = it;
            return MF_OK;
        }
        if (it > 0) {
            if (fabs(omega) < omegatol) {
                *info = -11;
                *iterations = it;
                return MF_OK;
            }
            const double beta = (rho / rho_prev) * (alpha / omega);
            p_update_k<<<g, 256, 0, st>>>(p, v, r, omega, beta, N);
            MF_LAUNCH_CHECK();
        } else {
            copy2_k<<<g, 256, 0, st>>>(r, N, p, nullptr);
            MF_LAUNCH_CHECK();
        }
        MF_TRY(precond(p, ph));
        spmv_k<<<g, 256, 0, st>>>(indptr, indices, data, ph, N, v);
        MF_LAUNCH_CHECK();
        MF_TRY(dot(rt, v, sc));
        MF_TRY(fetch(h, 1));
        const double rv = h[0];
        if (rv == 0.0) {
            *info = -11;
            *iterations = it;
            return MF_OK;
        }
        alpha = rho / rv;
        axmy_k<<<g, 256, 0, st>>>(r, v, alpha, N);  // r -= alpha v  (s = r)
        MF_LAUNCH_CHECK();
        MF_TRY(dot(r, r, sc));
        MF_TRY(fetch(h, 1));
        if (sqrt(h[0]) < atol_eff) {
            xupd_k<<<g, 256, 0, st>>>(x, ph, alpha, nullptr, 0.0, N);
            MF_LAUNCH_CHECK();
            *residual_norm = sqrt(h[0]);
            *iterations = it;
            return MF_OK;
        }
        MF_TRY(precond(r, sh));
        spmv_k<<<g, 256, 0, st>>>(indptr, indices, data, sh, N, t);
        MF_LAUNCH_CHECK();
        MF_TRY(dot(t, r, sc));
        MF_TRY(dot(t, t, sc + 1));
        MF_TRY(fetch(h, 2));
        omega = h[0] / h[1];
        xupd_k<<<g, 256, 0, st>>>(x, ph, alpha, sh, omega, N);
        MF_LAUNCH_CHECK();
        axmy_k<<<g, 256, 0, st>>>(r, t, omega, N);
        MF_LAUNCH_CHECK();
        rho_prev = rho;
    }
#undef MF_TRY
    *iterations = it;
    *info = (int32_t)(maxiter > INT32_MAX ? INT32_MAX : maxiter);
    return MF_OK;
}


// ---- device-controlled BiCGStab ---------------------------------------------------
// state: BICG_STATE_BYTES device bytes (mf_bicgstab_state_size); ws as mf_bicgstab.
extern "C" int mf_bicgstab_state_size(size_t* bytes) {
    *bytes = sizeof(BicgState);
    return MF_OK;
}

// r = b - A x, rt = r, ||b||, atol: the state is ready for mf_bicgstab_iter
extern "C" int mf_bicgstab_init(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N,
                                const double* b, const double* x, double rtol, double atol, int64_t maxiter,
                                void* state, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(N >= 1 && maxiter >= 0 && state, "mf_bicgstab_init: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    double* r = ar.take<double>(N);
    double* rt = ar.take<double>(N);
    for (int k = 0; k < 5; ++k) ar.take<double>(N);  // p, v, phat, shat, t (same layout as mf_bicgstab_iter)
    double* partial = ar.take<double>(2 * RED_BLOCKS);
    MF_REQUIRE(ar.ok() && ws, "mf_bicgstab_init: workspace too small");
    BicgState* stt = reinterpret_cast<BicgState*>(state);
    dot_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(b, b, N, partial);
    MF_LAUNCH_CHECK();
    bicg_init_k<<<1, 32, 0, st>>>(partial, stt, rtol, atol, (long long)maxiter);
    MF_LAUNCH_CHECK();
    const int g = vgrid(N);
    resid_k<<<g, 256, 0, st>>>(indptr, indices, data, x, b, N, r);
    MF_LAUNCH_CHECK();
    copy2_k<<<g, 256, 0, st>>>(r, N, rt, nullptr);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

// one iteration of scipy's recurrence, every step gated by the device state (a
// fixed launch sequence: capture it once in a graph and replay)
extern "C" int mf_bicgstab_iter(const int32_t* indptr, const int32_t* indices, const double* data, int64_t N,
                                const mf_ilu0_t* M, double* x, void* state, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(N >= 1 && state, "mf_bicgstab_iter: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    double* r = ar.take<double>(N);
    double* rt = ar.take<double>(N);
    double* p = ar.take<double>(N);
    double* v = ar.take<double>(N);
    double* ph = ar.take<double>(N);
    double* sh = ar.take<double>(N);
    double* t = ar.take<double>(N);
    double* partial = ar.take<double>(2 * RED_BLOCKS);
    MF_REQUIRE(ar.ok() && ws, "mf_bicgstab_iter: workspace too small");
    BicgState* stt = reinterpret_cast<BicgState*>(state);
    const int g = vgrid(N);
    auto precond = [&](const double* in, double* out) -> int {
        if (!M) {
            copy_ctl_k<<<g, 256, 0, st>>>(in, N, out, stt);
            MF_LAUNCH_CHECK();
            return MF_OK;
        }
        for (int c = 0; c < M->ncolors; ++c) {
            const int a = M->color_off[c], cnt = M->color_off[c + 1] - a;
            if (cnt <= 0) continue;
            ilu_fwd_ctl_k<<<grid_cap(cnt, 128, 16), 128, 0, st>>>(M->indptr, M->indices, M->part, M->lu,
                                                                  M->order + a, cnt, in, out, stt);
            MF_LAUNCH_CHECK();
        }
        for (int c = M->ncolors - 1; c >= 0; --c) {
            const int a = M->color_off[c], cnt = M->color_off[c + 1] - a;
            if (cnt <= 0) continue;
            ilu_bwd_ctl_k<<<grid_cap(cnt, 128, 16), 128, 0, st>>>(M->indptr, M->indices, M->part, M->lu, M->diag,
                                                                  M->order + a, cnt, out, stt);
            MF_LAUNCH_CHECK();
        }
        return MF_OK;
    };
    int rc;
    dot2_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(r, r, rt, r, N, partial, stt);
    MF_LAUNCH_CHECK();
    bicg_head_k<<<1, 32, 0, st>>>(partial, stt);
    MF_LAUNCH_CHECK();
    bicg_p_k<<<g, 256, 0, st>>>(p, v, r, N, stt);
    MF_LAUNCH_CHECK();
    if ((rc = precond(p, ph)) != MF_OK) return rc;
    spmv_ctl_k<<<g, 256, 0, st>>>(indptr, indices, data, ph, N, v, stt);
    MF_LAUNCH_CHECK();
    dot2_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(rt, v, nullptr, nullptr, N, partial, stt);
    MF_LAUNCH_CHECK();
    bicg_alpha_k<<<1, 32, 0, st>>>(partial, stt);
    MF_LAUNCH_CHECK();
    bicg_axmy_k<<<g, 256, 0, st>>>(r, v, N, stt, 0);
    MF_LAUNCH_CHECK();
    dot2_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(r, r, nullptr, nullptr, N, partial, stt);
    MF_LAUNCH_CHECK();
    bicg_mid_k<<<1, 32, 0, st>>>(partial, stt);
    MF_LAUNCH_CHECK();
    bicg_xhalf_k<<<g, 256, 0, st>>>(x, ph, N, stt);
    MF_LAUNCH_CHECK();
    bicg_xhalf_done_k<<<1, 32, 0, st>>>(stt);
    MF_LAUNCH_CHECK();
    if ((rc = precond(r, sh)) != MF_OK) return rc;
    spmv_ctl_k<<<g, 256, 0, st>>>(indptr, indices, data, sh, N, t, stt);
    MF_LAUNCH_CHECK();
    dot2_partial_k<<<RED_BLOCKS, RED_THREADS, 0, st>>>(t, r, t, t, N, partial, stt);
    MF_LAUNCH_CHECK();
    bicg_omega_k<<<1, 32, 0, st>>>(partial, stt);
    MF_LAUNCH_CHECK();
    bicg_x_k<<<g, 256, 0, st>>>(x, ph, sh, N, stt);
    MF_LAUNCH_CHECK();
    bicg_axmy_k<<<g, 256, 0, st>>>(r, t, N, stt, 1);
    MF_LAUNCH_CHECK();
    bicg_tail_k<<<1, 32, 0, st>>>(stt);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

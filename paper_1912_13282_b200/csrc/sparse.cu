// Canonical CSR assembly, explicit operator application and the fused
// forward-Euler heat step (sm_100a).
//
//   mf_csr_build / mf_csr_gather   WeightStore.matrix      (storage.py:156-170)
//   mf_apply                       WeightStore.apply_all   (storage.py:186-188)
//   mf_apply_rows                  WeightStore.apply       (storage.py:174-184)
//   mf_heat_steps                  run_heat_explicit loop  (drivers.py:87-110), on an apply plan (plan.cu)
//   mf_neumann_values              WeightStore.neumann_value (storage.py:226-250)
//
// Summation contract: scipy's csr_matvec accumulates each row in storage
// order from 0.0 with separately rounded multiply and add; the kernels here
// keep exactly that order (__dmul_rn/__dadd_rn), so the results are bitwise
// equal to the reference on the same CSR.
#include <cstdlib>

#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace mf {

constexpr double BLOWUP_LIMIT = 1e12;  // drivers.py:18

// ---------------------------------------------------------------------------
// CSR structure
// ---------------------------------------------------------------------------
__global__ void csr_mark_rows(const int64_t* __restrict__ rows, int64_t m, int64_t N,
                              int32_t* __restrict__ node_row, int32_t* __restrict__ dup) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = rows[r];
        if (node < 0 || node >= N) {
            atomicExch(dup, 2);
            continue;
        }
        int old = atomicCAS(&node_row[node], -1, (int)r);
        if (old != -1) atomicExch(dup, 1);
    }
}

// node_row[i] (-1 = not stored) -> row length n or 0, in place (plus a 0 at N)
__global__ void csr_counts(int32_t* __restrict__ node_row, int64_t N, int n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= N; i += (int64_t)gridDim.x * blockDim.x)
        node_row[i] = (i < N && node_row[i] >= 0) ? n : 0;
}

// One thread per stencil entry: its canonical slot is its rank by (column,
// slot) within the row -- the stable lexsort of storage.py:161.  Threads of a
// warp read the same row, so the inner loads are broadcasts.
__global__ void csr_fill(const int64_t* __restrict__ rows, const int32_t* __restrict__ st, int64_t m, int n,
                         const int32_t* __restrict__ indptr, int32_t* __restrict__ indices,
                         int32_t* __restrict__ perm) {
    const int64_t total = m * (int64_t)n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / n;
        const int j = (int)(e - r * n);
        const int32_t* src = st + r * n;
        const int32_t c = src[j];
        int rank = 0;
        for (int i = 0; i < n; ++i) {
            const int32_t ci = __ldg(src + i);
            rank += (ci < c) || (ci == c && i < j);
        }
        const int64_t base = indptr[rows[r]];
        indices[base + rank] = c;
        perm[base + rank] = (int32_t)e;
    }
}

// Same ranks, rows staged in shared memory as unique 32-bit keys column*64 + slot
// (N < 2^25, n <= 64), each row padded to a multiple of 4 with INT_MAX so a
// 16-byte load serves four comparisons.  A block takes CSR_ROWS rows at a time.
constexpr int CSR_ROWS = 32;

__global__ void __launch_bounds__(256) csr_fill_smem(const int64_t* __restrict__ rows, const int32_t* __restrict__ st,
                                                     int64_t m, int n, const int32_t* __restrict__ indptr,
                                                     int32_t* __restrict__ indices, int32_t* __restrict__ perm) {
    extern __shared__ __align__(16) int32_t sk[];  // CSR_ROWS x n4 keys
    const int n4 = (n + 3) & ~3;
    for (int64_t r0 = (int64_t)blockIdx.x * CSR_ROWS; r0 < m; r0 += (int64_t)gridDim.x * CSR_ROWS) {
        const int nr = (int)(m - r0 < CSR_ROWS ? m - r0 : CSR_ROWS);
        const int tot = nr * n;
        __syncthreads();
        for (int t = threadIdx.x; t < nr * n4; t += blockDim.x) {
            const int rr = t / n4, j = t - rr * n4;
            sk[t] = j < n ? (st[(r0 + rr) * n + j] << 6) | j : 0x7fffffff;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < tot; t += blockDim.x) {
            const int rr = t / n, j = t - rr * n;
            const int4* row = reinterpret_cast<const int4*>(sk + rr * n4);
            const int32_t ke = sk[rr * n4 + j];
            int rank = 0;
            for (int q = 0; q < (n4 >> 2); ++q) {
                const int4 v = row[q];
                rank += (v.x < ke) + (v.y < ke) + (v.z < ke) + (v.w < ke);
            }
            const int64_t r = r0 + rr;
            const int64_t base = indptr[rows[r]];
            indices[base + rank] = ke >> 6;
            perm[base + rank] = (int32_t)(r * n + j);
        }
    }
}

// Thread per row, rows staged through shared memory: a warp loads the keys
// column*64 + slot of its 32 rows with coalesced loads, each lane sorts its row
// in registers with a Batcher odd-even merge network over 64 positions pruned at
// compile time for the NR real inputs (positions >= NR hold +inf: comparators
// between two infs are dropped, one whose low input is inf is a register
// rename, one whose high input is inf a no-op), writes the sorted row back, and
// the warp stores the rows with coalesced writes.  The keys are unique, so the
// order is the stable (column, slot) lexsort of csr_fill.
template <int NR>
struct SortNet {
    static constexpr int P = NR <= 64 ? 64 : 128;  // network width (power of two >= NR)
    static constexpr int CAP = P == 64 ? 700 : 1600;
    int c[CAP][2];
    int nc;
    int out[P];
    constexpr SortNet() : c{}, nc(0), out{} {
        int map[P] = {};
        bool inf[P] = {};
        for (int i = 0; i < P; ++i) {
            map[i] = i;
            inf[i] = i >= NR;
        }
        for (int p = 1; p < P; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < P; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < P; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                            const int a = i + j, b = i + j + k;
                            if (inf[b]) continue;  // (both inf, or only the high one: no-op)
                            if (inf[a]) {          // low input inf: the values swap places
                                const int t = map[a];
                                map[a] = map[b];
                                map[b] = t;
                                inf[a] = false;
                                inf[b] = true;
                                continue;
                            }
                            c[nc][0] = map[a];
                            c[nc][1] = map[b];
                            ++nc;
                        }
        for (int i = 0; i < P; ++i) out[i] = map[i];
    }
};

// warps per block of csr_fill_net (the staged tiles must fit 48 KB of static shared memory)
template <int NR>
constexpr int csr_net_warps() {
    return NR <= 40 ? 8 : 4;
}

template <int NR>
__global__ void __launch_bounds__(csr_net_warps<NR>() * 32, NR <= 40 ? 4 : 2)
    csr_fill_net(const int64_t* __restrict__ rows, const int32_t* __restrict__ st, int64_t m,
                 const int32_t* __restrict__ indptr, int32_t* __restrict__ indices, int32_t* __restrict__ perm) {
    constexpr int PITCH = NR | 1;  // odd: lane-per-row accesses hit distinct banks
    constexpr int WPB = csr_net_warps<NR>();
    constexpr int SH = NR <= 64 ? 6 : 7;  // key = column << SH | slot
    constexpr SortNet<NR> net{};
    __shared__ int32_t sk[WPB][32 * PITCH];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int32_t* k = sk[wib];
    for (int64_t r0 = ((int64_t)blockIdx.x * WPB + wib) * 32; r0 < m; r0 += (int64_t)gridDim.x * WPB * 32) {
        const int nr = (int)(m - r0 < 32 ? m - r0 : 32);
        // coalesced staging of the tile's keys (rows are contiguous in `st`)
        for (int e = lane; e < nr * NR; e += 32) {
            const int rr = e / NR, j = e - rr * NR;
            k[rr * PITCH + j] = (st[r0 * NR + e] << SH) | j;
        }
        __syncwarp();
        if (lane < nr) {
            int key[NR];
#pragma unroll
            for (int j = 0; j < NR; ++j) key[j] = k[lane * PITCH + j];
#pragma unroll
            for (int t = 0; t < net.nc; ++t) {
                const int a = net.c[t][0], b = net.c[t][1];
                const int lo = min(key[a], key[b]), hi = max(key[a], key[b]);
                key[a] = lo;
                key[b] = hi;
            }
#pragma unroll
            for (int q = 0; q < NR; ++q) k[lane * PITCH + q] = key[net.out[q]];
        }
        __syncwarp();
        for (int rr = 0; rr < nr; ++rr) {
            const int64_t r = r0 + rr;
            const int64_t base = indptr[rows[r]];
            for (int q = lane; q < NR; q += 32) {
                const int kk = k[rr * PITCH + q];
                indices[base + q] = kk >> SH;
                perm[base + q] = (int32_t)(r * NR + (kk & ((1 << SH) - 1)));
            }
        }
        __syncwarp();
    }
}

__global__ void csr_gather_k(const int32_t* __restrict__ perm, const double* __restrict__ w, int64_t nnz,
                             double* __restrict__ data) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        data[p] = w[perm[p]];
}

// ---------------------------------------------------------------------------
// Row application.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double row_sum(const double* __restrict__ dv, const int32_t* __restrict__ iv,
                                          int lo, int hi, const double* __restrict__ u) {
    double acc = 0.0;
#pragma unroll 8
    for (int p = lo; p < hi; ++p) acc = __dadd_rn(acc, __dmul_rn(dv[p], __ldg(u + iv[p])));
    return acc;
}

// CSR, thread per row (general layout; the ELL plan below is the fast path)
__global__ void apply_csr_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const double* __restrict__ data, const double* __restrict__ u,
                            double* __restrict__ y, int64_t N) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = row_sum(data, indices, indptr[i], indptr[i + 1], u);
}

__global__ void apply_rows_k(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                             const double* __restrict__ data, const double* __restrict__ u,
                             const int64_t* __restrict__ sel, int64_t count, double* __restrict__ y) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = sel[k];
        y[k] = row_sum(data, indices, indptr[i], indptr[i + 1], u);
    }
}

struct HeatStep {
    const uint8_t* interior;
    const uint8_t* dirichlet;
    const double* g_dir;
    const double* source;
    const uint8_t* peak_skip;             // rows whose final value comes later (Neumann)
    double dt, D;
    unsigned long long* peak_out;         // this step's max|u| bits
    const unsigned long long* peak_prev;  // previous step's, or null
};

__device__ __forceinline__ bool step_blew_up(const unsigned long long* prev) {
    return prev && *prev > (unsigned long long)__double_as_longlong(BLOWUP_LIMIT);
}

// Thread per row over the ELL-32 plan: each warp-wide load of slot j is one
// contiguous 256 B (values) / 128 B (indices) segment.
template <bool HEAT>
__global__ void __launch_bounds__(256) ell_apply_k(const int32_t* __restrict__ ell_len,
                                                   const int32_t* __restrict__ ell_idx,
                                                   const double* __restrict__ ell_val, int64_t N, int W,
                                                   const double* __restrict__ u, double* __restrict__ y,
                                                   HeatStep hs) {
    if (HEAT && step_blew_up(hs.peak_prev)) return;
    unsigned long long peak = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ((N + 31) & ~31ll); r += stride) {
        const bool live = r < N;
        int len = live ? ell_len[r] : 0;
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double v;
        if (!HEAT) {
            double acc = 0.0;
#pragma unroll 5
            for (int j = 0; j < len; ++j) {
                double a = __ldcs(ell_val + base + 32 * j);
                int32_t c = __ldcs(ell_idx + base + 32 * j);
                acc = __dadd_rn(acc, __dmul_rn(a, __ldg(u + c)));
            }
            if (live) y[r] = acc;
        } else if (live) {
            v = u[r];
            if (hs.interior[r]) {
                double acc = 0.0;
#pragma unroll 5
                for (int j = 0; j < len; ++j) {
                    double a = __ldcs(ell_val + base + 32 * j);
                    int32_t c = __ldcs(ell_idx + base + 32 * j);
                    acc = __dadd_rn(acc, __dmul_rn(a, __ldg(u + c)));
                }
                double f = hs.source ? hs.source[r] : 0.0;
                // u + dt * (D * lap_u + f)   (drivers.py:93-96)
                v = __dadd_rn(v, __dmul_rn(hs.dt, __dadd_rn(__dmul_rn(hs.D, acc), f)));
            }
            if (hs.dirichlet[r]) v = hs.g_dir[r];
            y[r] = v;
            if (!(hs.peak_skip && hs.peak_skip[r])) {
                unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
                peak = b > peak ? b : peak;
            }
        }
    }
    if (HEAT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long ob = __shfl_xor_sync(FULL, peak, o);
            peak = ob > peak ? ob : peak;
        }
        if ((threadIdx.x & 31) == 0 && peak) atomicMax(hs.peak_out, peak);
    }
}

// ---------------------------------------------------------------------------
// Explicit Neumann closure (storage.py:226-250), one thread per listed node.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double neumann_coef(const mf_neumann_t& nm, int64_t k, int64_t base, int j) {
    // c = n_0 w_0 + n_1 w_1 + ... accumulated per axis (storage.py:231-234); normals are per listed node
    double c = __dmul_rn(nm.normals[k * nm.d + 0], nm.w_d1[base + j]);
    for (int a = 1; a < nm.d; ++a)
        c = __dadd_rn(c, __dmul_rn(nm.normals[k * nm.d + a], nm.w_d1[(int64_t)a * nm.mn + base + j]));
    return c;
}

__global__ void neumann_k(mf_neumann_t nm, const double* __restrict__ u, double* __restrict__ out,
                          double* __restrict__ u_scatter, unsigned long long* peak, int64_t* bad,
                          const unsigned long long* peak_prev) {
    if (step_blew_up(peak_prev)) return;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nm.count; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = nm.nodes[k];
        const int64_t base = nm.node_row[i] * nm.n;
        double ss = 0.0;
        for (int j = 0; j < nm.n; ++j) {
            double c = neumann_coef(nm, k, base, j);
            ss = fma(c, c, ss);
        }
        const double pivot = neumann_coef(nm, k, base, 0);
        double val;
        if (fabs(pivot) < 1e-12 * sqrt(ss)) {
            if (bad) atomicMin((unsigned long long*)bad, (unsigned long long)k);
            val = 0.0;
        } else {
            double acc = nm.gn[k];
            for (int j = 1; j < nm.n; ++j)
                acc = __dsub_rn(acc, __dmul_rn(neumann_coef(nm, k, base, j), u[nm.stencils[base + j]]));
            val = __ddiv_rn(acc, pivot);
        }
        if (out) out[k] = val;
        if (u_scatter) u_scatter[i] = val;
        if (peak) atomicMax(peak, (unsigned long long)__double_as_longlong(fabs(val)));
    }
}

// Heat step for rows of at most MAXW entries: a thread issues its row's whole
// index / value stream, then every u gather, then sums in storage order
// (bitwise the same as the batched loop above) -- more loads in flight per
// thread than the unroll-by-5 loop, whose gathers wait on each batch.
template <int MAXW, int CHUNK>
__global__ void __launch_bounds__(256) ell_heat_wide_k(const int32_t* __restrict__ ell_len,
                                                       const int32_t* __restrict__ ell_idx,
                                                       const double* __restrict__ ell_val, int64_t N, int W,
                                                       const double* __restrict__ u, double* __restrict__ y,
                                                       HeatStep hs) {
    if (step_blew_up(hs.peak_prev)) return;
    unsigned long long peak = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ((N + 31) & ~31ll); r += stride) {
        if (r >= N) continue;
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        double v = u[r];
        if (hs.interior[r]) {
            const int len = ell_len[r];
            double acc = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < MAXW; j0 += CHUNK) {
                double a[CHUNK], g[CHUNK];
                int32_t c[CHUNK];
#pragma unroll
                for (int j = 0; j < CHUNK; ++j) {
                    a[j] = j0 + j < len ? __ldcs(ell_val + base + 32 * (j0 + j)) : 0.0;
                    c[j] = j0 + j < len ? __ldcs(ell_idx + base + 32 * (j0 + j)) : 0;
                }
#pragma unroll
                for (int j = 0; j < CHUNK; ++j) g[j] = j0 + j < len ? __ldg(u + c[j]) : 0.0;
#pragma unroll
                for (int j = 0; j < CHUNK; ++j)
                    if (j0 + j < len) acc = __dadd_rn(acc, __dmul_rn(a[j], g[j]));
            }
            double f = hs.source ? hs.source[r] : 0.0;
            // u + dt * (D * lap_u + f)   (drivers.py:93-96)
            v = __dadd_rn(v, __dmul_rn(hs.dt, __dadd_rn(__dmul_rn(hs.D, acc), f)));
        }
        if (hs.dirichlet[r]) v = hs.g_dir[r];
        y[r] = v;
        if (!(hs.peak_skip && hs.peak_skip[r])) {
            unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
            peak = b > peak ? b : peak;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long ob = __shfl_xor_sync(FULL, peak, o);
        peak = ob > peak ? ob : peak;
    }
    if ((threadIdx.x & 31) == 0 && peak) atomicMax(hs.peak_out, peak);
}

// Packed heat step (mf_heat_pack): the step-invariant row data folded into one
// byte per row (length | interior << 5 | dirichlet << 6) and the column
// indices stored as 16-bit offsets from the row's own plan position -- in the
// Morton-ordered plan a stencil's columns are near its row.  Tiles with an
// offset outside int16 keep the 32-bit indices (tile_wide).  C4: 194 -> 161 MB
// read per step; the sums are the same as ell_heat_wide_k's, term for term.
constexpr int HEAT_META_LEN = 31, HEAT_META_INTERIOR = 32, HEAT_META_DIRICHLET = 64;

template <int MAXW, int CHUNK, bool WIDE>
__device__ __forceinline__ double heat_row_sum(const double* __restrict__ ell_val, const int32_t* __restrict__ ell_idx,
                                               const int16_t* __restrict__ ell_d16, const double* __restrict__ u,
                                               int64_t base, int32_t r, int len) {
    double acc = 0.0;
#pragma unroll
    for (int j0 = 0; j0 < MAXW; j0 += CHUNK) {
        double a[CHUNK], g[CHUNK];
        int32_t c[CHUNK];
#pragma unroll
        for (int j = 0; j < CHUNK; ++j) {
            a[j] = j0 + j < len ? __ldcs(ell_val + base + 32 * (j0 + j)) : 0.0;
            if (WIDE) c[j] = j0 + j < len ? __ldcs(ell_idx + base + 32 * (j0 + j)) : 0;
            else c[j] = j0 + j < len ? r + (int32_t)__ldcs(ell_d16 + base + 32 * (j0 + j)) : 0;
        }
#pragma unroll
        for (int j = 0; j < CHUNK; ++j) g[j] = j0 + j < len ? __ldg(u + c[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < CHUNK; ++j)
            if (j0 + j < len) acc = __dadd_rn(acc, __dmul_rn(a[j], g[j]));
    }
    return acc;
}

// With PDL (programmatic dependent launch) the next step's blocks start as the
// previous step's drain: they prefetch their first rows' operator entries
// (which do not depend on u) into L2, then wait for the previous grid.
template <int MAXW, int CHUNK, bool PDL>
__global__ void __launch_bounds__(256) ell_heat_packed_k(const uint8_t* __restrict__ meta,
                                                         const int16_t* __restrict__ ell_d16,
                                                         const uint8_t* __restrict__ tile_wide,
                                                         const int32_t* __restrict__ ell_idx,
                                                         const double* __restrict__ ell_val, int64_t N, int W,
                                                         const double* __restrict__ u, double* __restrict__ y,
                                                         HeatStep hs) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (PDL) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        const int64_t r0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (r0 < N) {
            const int64_t base = (r0 >> 5) * 32 * (int64_t)W + (r0 & 31);
            for (int j = 0; j < W; j += 2) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ell_val + base + 32 * j));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ell_d16 + base + 32 * j));
            }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (step_blew_up(hs.peak_prev)) return;
    unsigned long long peak = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ((N + 31) & ~31ll); r += stride) {
        if (r >= N) continue;
        const int64_t base = (r >> 5) * 32 * (int64_t)W + (r & 31);
        const int mt = meta[r];
        double v = u[r];
        if (mt & HEAT_META_INTERIOR) {
            const int len = mt & HEAT_META_LEN;
            const double acc = tile_wide[r >> 5]
                                   ? heat_row_sum<MAXW, CHUNK, true>(ell_val, ell_idx, ell_d16, u, base, (int32_t)r, len)
                                   : heat_row_sum<MAXW, CHUNK, false>(ell_val, ell_idx, ell_d16, u, base, (int32_t)r, len);
            double f = hs.source ? hs.source[r] : 0.0;
            // u + dt * (D * lap_u + f)   (drivers.py:93-96)
            v = __dadd_rn(v, __dmul_rn(hs.dt, __dadd_rn(__dmul_rn(hs.D, acc), f)));
        }
        if (mt & HEAT_META_DIRICHLET) v = hs.g_dir[r];
        y[r] = v;
        if (!(hs.peak_skip && hs.peak_skip[r])) {
            unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
            peak = b > peak ? b : peak;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long ob = __shfl_xor_sync(FULL, peak, o);
        peak = ob > peak ? ob : peak;
    }
    if ((threadIdx.x & 31) == 0 && peak) atomicMax(hs.peak_out, peak);
}

// One thread per ELL entry: the 16-bit offset, and the tile's wide flag when
// an offset does not fit; slot 0 also writes the row's meta byte.
__global__ void heat_pack_k(const int32_t* __restrict__ ell_len, const int32_t* __restrict__ ell_idx,
                            const uint8_t* __restrict__ interior, const uint8_t* __restrict__ dirichlet, int64_t N,
                            int W, int16_t* __restrict__ d16, uint8_t* __restrict__ meta, uint8_t* __restrict__ tile_wide) {
    const int64_t total = ((N + 31) / 32) * 32 * (int64_t)W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t tile = e / (32 * (int64_t)W);
        const int rem = (int)(e - tile * 32 * (int64_t)W);
        const int j = rem >> 5;
        const int64_t r = tile * 32 + (rem & 31);
        int16_t o = 0;
        if (r < N) {
            const int len = ell_len[r];
            if (j < len) {
                const int64_t dlt = (int64_t)ell_idx[e] - r;
                if (dlt >= -32768 && dlt <= 32767) o = (int16_t)dlt;
                else tile_wide[tile] = 1;
            }
            if (j == 0)
                meta[r] = (uint8_t)(len | (interior[r] ? HEAT_META_INTERIOR : 0) | (dirichlet[r] ? HEAT_META_DIRICHLET : 0));
        }
        d16[e] = o;
    }
}

inline int grid_for(int64_t work, int threads, int per_sm = 16) { return grid_cap(work, threads, per_sm); }

}  // namespace mf

using namespace mf;

extern "C" int mf_csr_workspace_size(int64_t N, size_t* bytes) {
    if (!bytes || N < 0) {
        set_error("mf_csr_workspace_size: bad arguments");
        return MF_ERR_ARG;
    }
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    Arena ar{nullptr, 0, 0, true};
    ar.take<int32_t>((size_t)N + 1);
    ar.take<int32_t>((size_t)N + 1);
    ar.take<char>(scan_bytes);
    *bytes = ar.off;
    return MF_OK;
}

extern "C" int mf_csr_build(const int64_t* rows, const int32_t* stencils, int64_t m, int32_t n, int64_t N,
                            int32_t* indptr, int32_t* indices, int32_t* perm, int32_t* dup_flag, void* ws,
                            size_t ws_bytes, void* stream) {
    MF_REQUIRE((n >= 1 || m == 0) && m >= 0 && N >= 0, "mf_csr_build: bad shape");
    MF_REQUIRE((double)m * n < 2147483647.0, "mf_csr_build: nnz %lld exceeds int32 indexing", (long long)(m * n));
    cudaStream_t st = (cudaStream_t)stream;
    MF_REQUIRE(N < 2147483647, "mf_csr_build: N exceeds int32 indexing");
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
    Arena ar{(char*)ws, ws_bytes, 0, false};
    int32_t* node_row = ar.take<int32_t>((size_t)N + 1);
    int32_t* counts = ar.take<int32_t>((size_t)N + 1);
    char* scan_tmp = ar.take<char>(scan_bytes);
    if (!ws || !ar.ok()) {
        set_error("mf_csr_build: workspace too small (%zu < %zu)", ws_bytes, ar.off);
        return MF_ERR_WORKSPACE;
    }
    MF_CUDA_CHECK(cudaMemsetAsync(node_row, 0xff, sizeof(int32_t) * (N + 1), st));
    if (dup_flag) MF_CUDA_CHECK(cudaMemsetAsync(dup_flag, 0, sizeof(int32_t), st));
    if (m > 0) {
        csr_mark_rows<<<grid_for(m, 256), 256, 0, st>>>(rows, m, N, node_row, dup_flag ? dup_flag : node_row + N);
        MF_LAUNCH_CHECK();
    }
    MF_CUDA_CHECK(cudaMemcpyAsync(counts, node_row, sizeof(int32_t) * (N + 1), cudaMemcpyDeviceToDevice, st));
    csr_counts<<<grid_for(N + 1, 256), 256, 0, st>>>(counts, N, n);
    MF_LAUNCH_CHECK();
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, indptr, (int)(N + 1), st));
    if (m > 0) {
        if (N < (1 << 25) && (n == 15 || n == 25 || n == 35)) {
            auto k = n == 15 ? csr_fill_net<15> : (n == 25 ? csr_fill_net<25> : csr_fill_net<35>);
            k<<<grid_for((m + 255) / 256 * 256, 256, 16), 256, 0, st>>>(rows, stencils, m, indptr, indices, perm);
        } else if (N < (1 << 24) && n == 70) {
            csr_fill_net<70><<<grid_for((m + 127) / 128 * 128, 128, 16), 128, 0, st>>>(rows, stencils, m, indptr,
                                                                                    indices, perm);
        } else if (N < (1 << 25) && n <= 64) {
            const int smem = CSR_ROWS * ((n + 3) & ~3) * (int)sizeof(int32_t);
            csr_fill_smem<<<grid_for((m + CSR_ROWS - 1) / CSR_ROWS, 1, 8), 256, smem, st>>>(rows, stencils, m, n,
                                                                                         indptr, indices, perm);
        } else {
            csr_fill<<<grid_for(m * (int64_t)n, 256, 16), 256, 0, st>>>(rows, stencils, m, n, indptr, indices, perm);
        }
        MF_LAUNCH_CHECK();
    }
    return MF_OK;
}

extern "C" int mf_csr_gather(const int32_t* perm, const double* w, int64_t nnz, double* data, void* stream) {
    MF_REQUIRE(nnz >= 0, "mf_csr_gather: bad nnz");
    if (nnz == 0) return MF_OK;
    csr_gather_k<<<grid_for(nnz, 256), 256, 0, (cudaStream_t)stream>>>(perm, w, nnz, data);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_apply(const int32_t* indptr, const int32_t* indices, const double* data, const double* u,
                        double* y, int64_t N, void* stream) {
    MF_REQUIRE(N >= 0, "mf_apply: bad N");
    if (N == 0) return MF_OK;
    apply_csr_k<<<grid_for(N, 256), 256, 0, (cudaStream_t)stream>>>(indptr, indices, data, u, y, N);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_apply_rows(const int32_t* indptr, const int32_t* indices, const double* data, const double* u,
                             const int64_t* sel, int64_t count, double* y, void* stream) {
    MF_REQUIRE(count >= 0, "mf_apply_rows: bad count");
    if (count == 0) return MF_OK;
    apply_rows_k<<<grid_for(count, 128), 128, 0, (cudaStream_t)stream>>>(indptr, indices, data, u, sel, count, y);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

// one explicit step on a block of rows (the row-partitioned heat loop,
// drivers.py:88-98 per block): lap = rows' Laplacian of the gathered field,
// interior u + dt * (D * lap + f) (f = 0.0 when absent, as the reference's
// `+ 0.0`), Dirichlet rows g, others unchanged; peak |u_new| as IEEE bits
__global__ void heat_rows_k(const double* __restrict__ lap, const double* __restrict__ u,
                            const uint8_t* __restrict__ interior, const uint8_t* __restrict__ dirichlet,
                            const double* __restrict__ g, const double* __restrict__ src, double dt, double D,
                            int64_t n, double* __restrict__ out, unsigned long long* peak) {
    unsigned long long mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = u[i];
        if (interior[i]) {
            const double f = src ? src[i] : 0.0;
            v = __dadd_rn(v, __dmul_rn(dt, __dadd_rn(__dmul_rn(D, lap[i]), f)));
        }
        if (dirichlet[i]) v = g[i];
        out[i] = v;
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
        mx = b > mx ? b : mx;
    }
    if (peak) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(FULL, mx, o);
            mx = t > mx ? t : mx;
        }
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(peak, mx);
    }
}

extern "C" int mf_heat_rows(const double* lap, const double* u, const uint8_t* interior, const uint8_t* dirichlet,
                            const double* g, const double* source, double dt, double diffusivity, int64_t n,
                            double* out, uint64_t* peak, void* stream) {
    MF_REQUIRE(n >= 0, "mf_heat_rows: bad n");
    if (n == 0) return MF_OK;
    heat_rows_k<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(lap, u, interior, dirichlet, g, source, dt,
                                                                      diffusivity, n, out,
                                                                      reinterpret_cast<unsigned long long*>(peak));
    MF_LAUNCH_CHECK();
    return MF_OK;
}

static int ell_grid(int64_t N) { return grid_for(((N + 31) / 32) * 32, 256, 8); }

extern "C" int mf_neumann_values(const mf_neumann_t* nm, const double* u, double* out, double* u_scatter,
                                 uint64_t* peak, int64_t* bad, void* stream) {
    MF_REQUIRE(nm && nm->n >= 1 && nm->d >= 1 && nm->d <= MF_MAX_DIM && nm->count >= 0,
               "mf_neumann_values: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (bad) MF_CUDA_CHECK(cudaMemsetAsync(bad, 0x7f, sizeof(int64_t), st));
    if (nm->count == 0) return MF_OK;
    neumann_k<<<grid_for(nm->count, 128), 128, 0, st>>>(*nm, u, out, u_scatter, (unsigned long long*)peak, bad,
                                                        nullptr);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_heat_pack(const int32_t* ell_len, const int32_t* ell_idx, const uint8_t* interior,
                            const uint8_t* dirichlet, int64_t N, int32_t W, int16_t* ell_d16, uint8_t* meta,
                            uint8_t* tile_wide, void* stream) {
    MF_REQUIRE(N >= 0 && W >= 0 && W <= HEAT_META_LEN, "mf_heat_pack: bad arguments (W %d)", (int)W);
    if (N == 0 || W == 0) return MF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    MF_CUDA_CHECK(cudaMemsetAsync(tile_wide, 0, (size_t)((N + 31) / 32), st));
    const int64_t total = ((N + 31) / 32) * 32 * (int64_t)W;
    heat_pack_k<<<grid_for(total, 256), 256, 0, st>>>(ell_len, ell_idx, interior, dirichlet, N, W, ell_d16, meta,
                                                       tile_wide);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_heat_steps(const int32_t* ell_len, const int32_t* ell_idx, const double* ell_val, int64_t N,
                             int32_t W, const uint8_t* interior, const uint8_t* dirichlet, const double* g_dir,
                             const double* source, double dt, double diffusivity, const mf_neumann_t* nm,
                             int64_t steps, double* u, double* scratch, uint64_t* peaks, const mf_heat_pack_t* pack,
                             void* stream) {
    MF_REQUIRE(N >= 0 && steps >= 0 && W >= 0, "mf_heat_steps: bad arguments");
    MF_REQUIRE(!pack || (pack->ell_d16 && pack->meta && pack->tile_wide && W <= 16),
               "mf_heat_steps: a packed plan needs ell_d16, meta and tile_wide, and rows of at most 16 entries");
    if (steps == 0 || N == 0) return MF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    MF_CUDA_CHECK(cudaMemsetAsync(peaks, 0, sizeof(uint64_t) * steps, st));
    // blocks per SM: the packed loop runs fastest at 4 x 256 threads (C4: 35 vs
    // 37-45 ms at 3, 5, 6, 8 or 16); the unpacked ones at 8
    const int grid = grid_for(((N + 31) / 32) * 32, 256, pack ? 4 : 8);
    const bool has_nm = nm && nm->count > 0;
    // programmatic dependent launch chains the packed steps (not with the Neumann pass in between)
    const bool pdl = !has_nm;
    double* buf[2] = {u, scratch};
    for (int64_t s = 0; s < steps; ++s) {
        const unsigned long long* prev = s ? (const unsigned long long*)(peaks + s - 1) : nullptr;
        unsigned long long* cur = (unsigned long long*)(peaks + s);
        HeatStep hs{interior, dirichlet, g_dir, source, has_nm ? nm->mask : nullptr, dt, diffusivity, cur, prev};
        double* u_old = buf[s & 1];
        double* u_new = buf[(s + 1) & 1];
        if (pack && pdl && s > 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            MF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, ell_heat_packed_k<16, 8, true>, pack->meta, pack->ell_d16,
                                             pack->tile_wide, ell_idx, ell_val, N, W, (const double*)u_old, u_new,
                                             hs));
        } else if (pack)
            ell_heat_packed_k<16, 8, false><<<grid, 256, 0, st>>>(pack->meta, pack->ell_d16, pack->tile_wide, ell_idx,
                                                                 ell_val, N, W, u_old, u_new, hs);
        else if (W <= 16)
            ell_heat_wide_k<16, 8><<<grid, 256, 0, st>>>(ell_len, ell_idx, ell_val, N, W, u_old, u_new, hs);
        else
            ell_apply_k<true><<<grid, 256, 0, st>>>(ell_len, ell_idx, ell_val, N, W, u_old, u_new, hs);
        MF_LAUNCH_CHECK();
        if (has_nm) {
            neumann_k<<<grid_for(nm->count, 128), 128, 0, st>>>(*nm, u_old, nullptr, u_new, cur, nullptr, prev);
            MF_LAUNCH_CHECK();
        }
    }
    if (steps & 1) MF_CUDA_CHECK(cudaMemcpyAsync(u, scratch, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    return MF_OK;
}

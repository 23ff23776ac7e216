// Node generation: the distance-acceptance pass of
// fill_interior (geometry/fill.py:38-117, driven by fill.py:204-298) on the GPU.
//
// The reference walks one generation's candidates strictly in order and
// accepts candidate c when no node accepted so far -- the nodes present
// before the generation and the candidates accepted earlier in it -- lies
// closer than gamma * min(h_c, h_j).  The same set is computed here in three
// passes, with the reference's distance arithmetic (sequential sum of
// squared differences from 0, no FMA) so every comparison decides alike:
//   1. every candidate against the nodes present before the generation, in
//      parallel (uniform cell grid of linked lists); survivors keep their order;
//   2. each survivor lists the EARLIER survivors it conflicts with (a grid of
//      the survivors);
//   3. the lexicographically-first greedy set over that conflict graph, by
//      rounds in one CTA: a survivor is rejected as soon as an earlier
//      conflicting survivor is accepted and accepted once every earlier
//      conflicting survivor is rejected -- exactly the sequential outcome.
// Accepted candidates are appended in candidate order and linked into the grid.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace mf {
namespace {

constexpr int MAXC = 64;  // earlier conflicting survivors listed per survivor

struct Grid {
    double lo[3];
    double cell;
    int dims[3];
    int d;
};

__device__ __forceinline__ int cell_coord(const Grid& g, double x, int a) {
    double t = floor((x - g.lo[a]) / g.cell);
    if (t < 0.0) t = 0.0;
    if (t > (double)(g.dims[a] - 1)) t = (double)(g.dims[a] - 1);
    return (int)t;
}
__device__ __forceinline__ int64_t cell_id(const Grid& g, const int* c) {
    int64_t id = c[0];
    for (int a = 1; a < g.d; ++a) id = id * g.dims[a] + c[a];
    return id;
}
// the reference's test: dist2 = sum (p_a - c_a)^2 from 0 in axis order, no FMA;
// lim = gamma * min(h_c, h_j); conflict when dist2 < lim * lim
__device__ __forceinline__ bool conflicts(const double* p, const double* c, int d, double gamma, double hc,
                                          double hj) {
    double dist2 = 0.0;
    for (int a = 0; a < d; ++a) {
        const double diff = __dsub_rn(p[a], c[a]);
        dist2 = __dadd_rn(dist2, __dmul_rn(diff, diff));
    }
    const double lim = __dmul_rn(gamma, fmin(hc, hj));
    return dist2 < __dmul_rn(lim, lim);
}

// visit every grid cell within `reach` cells of x; f(j) per listed node, stop when f returns true
template <class F>
__device__ bool scan_cells(const Grid& g, const double* x, int reach, const int32_t* __restrict__ head,
                           const int32_t* __restrict__ nxt, F f) {
    int c0[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < g.d; ++a) {
        c0[a] = cell_coord(g, x[a], a);
        lo[a] = max(0, c0[a] - reach);
        hi[a] = min(g.dims[a] - 1, c0[a] + reach);
    }
    int c[3];
    for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0])
        for (c[1] = lo[1]; c[1] <= (g.d > 1 ? hi[1] : lo[1]); ++c[1])
            for (c[2] = lo[2]; c[2] <= (g.d > 2 ? hi[2] : lo[2]); ++c[2]) {
                for (int j = head[cell_id(g, c)]; j >= 0; j = nxt[j])
                    if (f(j)) return true;
            }
    return false;
}

__device__ __forceinline__ int reach_of(const Grid& g, double gamma, double h) {
    return (int)ceil(gamma * h / g.cell) + 1;  // +1: rounding of the cell coordinates
}

__global__ void insert_k(const double* __restrict__ pos, int64_t a, int64_t b, Grid g, int32_t* head,
                         int32_t* nxt) {
    for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
        int c[3] = {0, 0, 0};
        for (int k = 0; k < g.d; ++k) c[k] = cell_coord(g, pos[i * g.d + k], k);
        nxt[i] = atomicExch(head + cell_id(g, c), (int32_t)i);
    }
}

// pass 1: survivors of the nodes present before the generation
__global__ void vs_existing_k(const double* __restrict__ pos, const double* __restrict__ hv, Grid g,
                              const int32_t* __restrict__ head, const int32_t* __restrict__ nxt,
                              const double* __restrict__ cand, const double* __restrict__ hc, int64_t M,
                              double gamma, int32_t* flag) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < M; c += (int64_t)gridDim.x * blockDim.x) {
        const double* x = cand + c * g.d;
        const double h = hc[c];
        const bool hit = scan_cells(g, x, reach_of(g, gamma, h), head, nxt,
                                    [&](int j) { return conflicts(pos + (int64_t)j * g.d, x, g.d, gamma, h, hv[j]); });
        flag[c] = hit ? 0 : 1;
    }
}
__global__ void compact_k(const int32_t* __restrict__ flag, const int32_t* __restrict__ at, int64_t M, int32_t* surv) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < M; c += (int64_t)gridDim.x * blockDim.x)
        if (flag[c]) surv[at[c]] = (int32_t)c;
}
// pass 2: survivors in their own grid (head2 over the same cells), earlier conflicts listed
__global__ void surv_insert_k(const double* __restrict__ cand, const int32_t* __restrict__ surv, int S, Grid g,
                              int32_t* head2, int32_t* nxt2) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        int c[3] = {0, 0, 0};
        for (int k = 0; k < g.d; ++k) c[k] = cell_coord(g, cand[(int64_t)surv[s] * g.d + k], k);
        nxt2[s] = atomicExch(head2 + cell_id(g, c), s);
    }
}
__global__ void surv_lists_k(const double* __restrict__ cand, const double* __restrict__ hc,
                             const int32_t* __restrict__ surv, int S, Grid g, const int32_t* __restrict__ head2,
                             const int32_t* __restrict__ nxt2, double gamma, int32_t* lst, int32_t* nlst,
                             int* overflow) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        const double* x = cand + (int64_t)surv[s] * g.d;
        const double h = hc[surv[s]];
        int k = 0;
        // survivors are listed by survivor index; only earlier ones matter.  The
        // reach of the later candidate covers the pair: lim <= gamma * h_s.
        scan_cells(g, x, reach_of(g, gamma, h), head2, nxt2, [&](int t) {
            if (t < s && conflicts(cand + (int64_t)surv[t] * g.d, x, g.d, gamma, h, hc[surv[t]])) {
                if (k < MAXC) lst[(int64_t)s * MAXC + k] = t;
                ++k;
            }
            return false;
        });
        if (k > MAXC) *overflow = 1;
        nlst[s] = k < MAXC ? k : MAXC;
    }
}
__global__ void surv_reset_k(const double* __restrict__ cand, const int32_t* __restrict__ surv, int S, Grid g,
                             int32_t* head2) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        int c[3] = {0, 0, 0};
        for (int k = 0; k < g.d; ++k) c[k] = cell_coord(g, cand[(int64_t)surv[s] * g.d + k], k);
        head2[cell_id(g, c)] = -1;
    }
}
// pass 3: greedy resolution in order, one CTA, rounds until every survivor is decided
__global__ void __launch_bounds__(1024) resolve_k(const int32_t* __restrict__ lst, const int32_t* __restrict__ nlst,
                                                  int S, int8_t* state, int* rounds) {
    __shared__ int undecided;
    for (int s = threadIdx.x; s < S; s += blockDim.x) state[s] = 0;
    __syncthreads();
    int r = 0;
    for (;; ++r) {
        if (threadIdx.x == 0) undecided = 0;
        __syncthreads();
        int mine = 0;
        for (int s = threadIdx.x; s < S; s += blockDim.x) {
            if (state[s] != 0) continue;
            bool all_rej = true, any_acc = false;
            for (int k = 0; k < nlst[s]; ++k) {
                const int8_t st = ((volatile int8_t*)state)[lst[(int64_t)s * MAXC + k]];
                any_acc |= st == 1;
                all_rej &= st == 2;
            }
            if (any_acc) state[s] = 2;
            else if (all_rej) state[s] = 1;
            else ++mine;
        }
        if (mine) atomicAdd(&undecided, mine);
        __syncthreads();
        if (undecided == 0) break;
        __syncthreads();
    }
    if (threadIdx.x == 0) *rounds = r + 1;
}
__global__ void acc_flag_k(const int8_t* __restrict__ state, int S, int32_t* flag) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) flag[s] = state[s] == 1;
}
__global__ void append_k(const int32_t* __restrict__ flag, const int32_t* __restrict__ at,
                         const int32_t* __restrict__ surv, int S, const double* __restrict__ cand,
                         const double* __restrict__ hc, int d, int64_t count, double* pos, double* hv,
                         int32_t* accepted_idx) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        if (!flag[s]) continue;
        const int64_t o = count + at[s];
        const int c = surv[s];
        for (int a = 0; a < d; ++a) pos[o * d + a] = cand[(int64_t)c * d + a];
        hv[o] = hc[c];
        accepted_idx[at[s]] = c;
    }
}

inline int g1(int64_t n) { return grid_cap(n, 256, 8); }

}  // namespace
}  // namespace mf

using namespace mf;

extern "C" int mf_fill_workspace_size(int64_t M, size_t* bytes) {
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(M + 1));
    *bytes = align_up((size_t)(M + 1) * 4) * 4 + align_up((size_t)M * MAXC * 4) + align_up((size_t)M * 4) +
             align_up((size_t)M) + align_up(scan) + 1024;
    return MF_OK;
}

extern "C" int mf_fill_insert(const double* pos, int64_t a, int64_t b, const mf_fill_grid_t* grid, int32_t* head,
                              int32_t* nxt, void* stream) {
    MF_REQUIRE(grid && grid->d >= 1 && grid->d <= 3 && a >= 0 && b >= a, "mf_fill_insert: bad arguments");
    if (b == a) return MF_OK;
    Grid g{};
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = grid->lo[k];
        g.dims[k] = grid->dims[k] > 0 ? grid->dims[k] : 1;
    }
    g.cell = grid->cell;
    g.d = grid->d;
    insert_k<<<g1(b - a), 256, 0, (cudaStream_t)stream>>>(pos, a, b, g, head, nxt);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

extern "C" int mf_fill_accept(double* pos, double* hv, int32_t* nxt, int64_t count, int64_t cap,
                              const mf_fill_grid_t* grid, int32_t* head, int32_t* head2, const double* cand,
                              const double* hc, int64_t M, double gamma, int32_t* accepted_idx,
                              int64_t* n_accepted, int32_t* rounds_out, void* ws, size_t ws_bytes, void* stream) {
    MF_REQUIRE(grid && grid->d >= 1 && grid->d <= 3 && M >= 0 && M < INT32_MAX && count >= 0,
               "mf_fill_accept: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    *n_accepted = 0;
    if (M == 0) return MF_OK;
    Grid g{};
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = grid->lo[k];
        g.dims[k] = grid->dims[k] > 0 ? grid->dims[k] : 1;
    }
    g.cell = grid->cell;
    g.d = grid->d;
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, (int32_t*)nullptr, (int32_t*)nullptr, (int)(M + 1));
    Arena ar{(char*)ws, ws_bytes, 0, ws == nullptr};
    int32_t* flag = ar.take<int32_t>(M + 1);
    int32_t* at = ar.take<int32_t>(M + 1);
    int32_t* surv = ar.take<int32_t>(M + 1);
    int32_t* nlst = ar.take<int32_t>(M + 1);
    int32_t* lst = ar.take<int32_t>((size_t)M * MAXC);
    int32_t* nxt2 = ar.take<int32_t>(M);
    int8_t* state = ar.take<int8_t>(M);
    void* tmp = ar.take<char>(scan);
    int* ctl = ar.take<int>(4);
    MF_REQUIRE(ar.ok() && ws, "mf_fill_accept: workspace too small");
    // 1. against the existing nodes
    vs_existing_k<<<g1(M), 256, 0, st>>>(pos, hv, g, head, nxt, cand, hc, M, gamma, flag);
    MF_LAUNCH_CHECK();
    MF_CUDA_CHECK(cudaMemsetAsync(flag + M, 0, 4, st));
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, scan, flag, at, (int)(M + 1), st));
    compact_k<<<g1(M), 256, 0, st>>>(flag, at, M, surv);
    MF_LAUNCH_CHECK();
    int32_t S = 0;
    MF_CUDA_CHECK(cudaMemcpyAsync(&S, at + M, 4, cudaMemcpyDeviceToHost, st));
    MF_CUDA_CHECK(cudaStreamSynchronize(st));
    if (S == 0) return MF_OK;
    // 2. earlier conflicting survivors
    MF_CUDA_CHECK(cudaMemsetAsync(ctl, 0, 16, st));
    surv_insert_k<<<g1(S), 256, 0, st>>>(cand, surv, S, g, head2, nxt2);
    MF_LAUNCH_CHECK();
    surv_lists_k<<<g1(S), 256, 0, st>>>(cand, hc, surv, S, g, head2, nxt2, gamma, lst, nlst, ctl);
    MF_LAUNCH_CHECK();
    surv_reset_k<<<g1(S), 256, 0, st>>>(cand, surv, S, g, head2);
    MF_LAUNCH_CHECK();
    // 3. the greedy set in candidate order
    resolve_k<<<1, 1024, 0, st>>>(lst, nlst, S, state, ctl + 1);
    MF_LAUNCH_CHECK();
    acc_flag_k<<<g1(S), 256, 0, st>>>(state, S, flag);
    MF_LAUNCH_CHECK();
    MF_CUDA_CHECK(cudaMemsetAsync(flag + S, 0, 4, st));
    MF_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, scan, flag, at, (int)(S + 1), st));
    int h[2];
    MF_CUDA_CHECK(cudaMemcpyAsync(h, ctl, 8, cudaMemcpyDeviceToHost, st));
    int32_t A = 0;
    MF_CUDA_CHECK(cudaMemcpyAsync(&A, at + S, 4, cudaMemcpyDeviceToHost, st));
    MF_CUDA_CHECK(cudaStreamSynchronize(st));
    MF_REQUIRE(h[0] == 0, "mf_fill_accept: more than %d earlier conflicts for one candidate", MAXC);
    if (rounds_out) *rounds_out = h[1];
    *n_accepted = A;
    if (A == 0) return MF_OK;
    MF_REQUIRE(count + A <= cap, "mf_fill_accept: capacity %lld exceeded", (long long)cap);
    append_k<<<g1(S), 256, 0, st>>>(flag, at, surv, S, cand, hc, g.d, count, pos, hv, accepted_idx);
    MF_LAUNCH_CHECK();
    insert_k<<<g1(A), 256, 0, st>>>(pos, count, count + A, g, head, nxt);
    MF_LAUNCH_CHECK();
    return MF_OK;
}

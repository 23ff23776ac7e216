// Microbenchmark: when does ptxas address a warp-uniform shared load through a
// uniform register (LDS [UR+imm], 0.5 SM-cycles per LDS.64 on B200) instead of
// a vector register (LDS [R+imm], ~1 cycle)?  Variants: per-warp base from the
// warp index, loads under a vote-uniform branch, 1-warp blocks.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lsu_probe3 tools/lsu_probe3.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;
constexpr int PER_WARP = 256;

// per-warp region selected by the warp index (threadIdx.x >> 5)
__global__ void k_warpbase(double* out) {
    __shared__ double s[16 * PER_WARP];
    for (int i = threadIdx.x; i < 16 * PER_WARP; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const double* w = s + (threadIdx.x >> 5) * PER_WARP;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += w[((i * 8 + u) & 31) * 8];
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// loads under a branch whose condition is a warp vote
__global__ void k_votebranch(double* out, int lim) {
    __shared__ double s[PER_WARP];
    for (int i = threadIdx.x; i < PER_WARP; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc[8] = {};
    const bool ok = __all_sync(0xffffffffu, lane < lim);
    if (ok) {
        for (int i = 0; i < ITER; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += s[((i * 8 + u) & 31) * 8];
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// 1-warp blocks, static shared array, lane-dependent work mixed in
__global__ void k_onewarp(double* out) {
    __shared__ double s[PER_WARP];
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < PER_WARP; i += 32) s[i] = i * 0.5;
    __syncwarp();
    double acc[8] = {};
    double x = s[lane];
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fma(x, acc[u], s[((i * 8 + u) & 31) * 8]);
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// explicit shared address from a uniform value via inline PTX (32-bit window address)
__global__ void k_ptx(double* out) {
    __shared__ double s[16 * PER_WARP];
    for (int i = threadIdx.x; i < 16 * PER_WARP; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(s) + __shfl_sync(0xffffffffu, (threadIdx.x >> 5), 0) * PER_WARP * 8;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double v;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + (unsigned)(((i * 8 + u) & 31) * 64)));
            acc[u] += v;
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

template <typename K, typename... A>
void run(const char* name, K k, int threads, int blocks_per_sm, double* out, int sms, A... args) {
    const int blocks = sms * blocks_per_sm;
    k<<<blocks, threads>>>(out, args...);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(out, args...);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_ops = (double)blocks * threads / 32 * ITER * 8;
    const double cyc = ms * 1e-3 * clk * 1e3 * sms;
    printf("%-16s %8.3f ms  %6.3f SM-cycles per warp-op (per SM)\n", name, ms, cyc / warp_ops);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("warpbase", k_warpbase, 512, 1, out, sms);
    run("votebranch", k_votebranch, 512, 4, out, sms, 40);
    run("onewarp", k_onewarp, 32, 32, out, sms);
    run("ptx", k_ptx, 512, 1, out, sms);
    return 0;
}

// Microbenchmark: cost of shared-memory broadcasts vs warp shuffles on B200.
// Each kernel issues ITER x 8 independent operations per warp; the printed
// figure is SM cycles per warp-instruction at full occupancy.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lsu_probe tools/lsu_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

__global__ void k_lds64_bcast(double* out) {
    __shared__ double s[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += s[(i * 8 + u) & 255];
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

__global__ void k_lds128_bcast(double* out) {
    __shared__ double2 s[128];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s[i] = make_double2(i, i + 1);
    __syncthreads();
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 v = s[(i * 8 + u) & 127];
            acc[u] += v.x * v.y;
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

__global__ void k_lds64_dist(double* out) {
    __shared__ double s[32 * 33];
    for (int i = threadIdx.x; i < 32 * 33; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += s[((i * 8 + u) & 31) * 33 + lane];
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

__global__ void k_shfl64(double* out) {
    const int lane = threadIdx.x & 31;
    double x = lane * 1.5;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += __shfl_sync(0xffffffffu, x, (i * 8 + u) & 31);
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

__global__ void k_dfma(double* out) {
    double acc[8];
    for (int u = 0; u < 8; ++u) acc[u] = threadIdx.x + u;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fma(acc[u], b, c);
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

template <typename K>
void run(const char* name, K k, double* out, int sms) {
    const int threads = 512, blocks = sms * 4;
    k<<<blocks, threads>>>(out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(out);
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
    run("lds64_bcast", k_lds64_bcast, out, sms);
    run("lds128_bcast", k_lds128_bcast, out, sms);
    run("lds64_dist", k_lds64_dist, out, sms);
    run("shfl64", k_shfl64, out, sms);
    run("dfma", k_dfma, out, sms);
    return 0;
}

// Microbenchmark: cost of warp-uniform (broadcast) shared loads as a function of
// the stride between consecutive loads and the access width, and of loads where
// the two half-warps read two different addresses (two stencils per warp).
// Each warp reads its own region (base from the warp index, like the shape
// kernels).  Printed: SM cycles per warp-instruction at full occupancy.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lsu_probe4 tools/lsu_probe4.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 2048;
constexpr int REGION = 1024;  // doubles per warp

// STRIDE in doubles between consecutive loads; W = 1 (LDS.64) or 2 (LDS.128);
// HALF: the upper half-warp reads an address OFF doubles further
template <int STRIDE, int W, int HALF, int OFF>
__global__ void k_bcast(double* out) {
    extern __shared__ double s[];
    for (int i = threadIdx.x; i < 4 * REGION; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const double* w = s + (threadIdx.x >> 5) * REGION + (HALF && lane >= 16 ? OFF : 0);
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int o = (((i * 8 + u) * STRIDE) & (REGION / 2 - 1)) & ~(W - 1);
            if (W == 1) {
                acc[u] += w[o];
            } else {
                const double2 v = *reinterpret_cast<const double2*>(w + o);
                acc[u] += v.x * v.y;
            }
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

template <typename K>
void run(const char* name, K k, double* out, int sms) {
    const int threads = 128, blocks = sms * 8;
    const size_t sm = 5 * REGION * sizeof(double);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<blocks, threads, sm>>>(out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<blocks, threads, sm>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_ops = (double)blocks * threads / 32 * ITER * 8;
    const double cyc = ms * 1e-3 * clk * 1e3 * sms;
    printf("%-34s %8.3f ms  %6.3f SM-cycles per warp-op (per SM)  %s\n", name, ms, cyc / warp_ops,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("lds64 uniform stride 1", k_bcast<1, 1, 0, 0>, out, sms);
    run("lds64 uniform stride 2", k_bcast<2, 1, 0, 0>, out, sms);
    run("lds64 uniform stride 8", k_bcast<8, 1, 0, 0>, out, sms);
    run("lds64 uniform stride 32", k_bcast<32, 1, 0, 0>, out, sms);
    run("lds64 uniform stride 33", k_bcast<33, 1, 0, 0>, out, sms);
    run("lds128 uniform stride 2", k_bcast<2, 2, 0, 0>, out, sms);
    run("lds128 uniform stride 8", k_bcast<8, 2, 0, 0>, out, sms);
    run("lds128 uniform stride 32", k_bcast<32, 2, 0, 0>, out, sms);
    run("lds64 half-warps off 1", k_bcast<1, 1, 1, 1>, out, sms);
    run("lds64 half-warps off 512+1", k_bcast<1, 1, 1, 513>, out, sms);
    run("lds128 half-warps off 2", k_bcast<2, 2, 1, 2>, out, sms);
    run("lds128 half-warps off 512+2", k_bcast<2, 2, 1, 514>, out, sms);
    run("lds128 half-warps off 512+4", k_bcast<2, 2, 1, 516>, out, sms);
    return 0;
}

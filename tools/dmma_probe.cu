// Microbenchmark: fp64 tensor-core (mma.sync m8n8k4 f64) vs DFMA throughput on this GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_k(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 123.456) out[0] = s;
}

__global__ void dfma_k(double* out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    const double b = 0.999999, c = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 123.456) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps = 4; warps <= 16; warps *= 2) {
        int blocks = sms * 4, threads = 32 * warps / 4 * 1;
        threads = 32 * warps;
        blocks = sms;
        int iters = 20000;
        dmma_k<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * blocks * (threads / 32);
        printf("DMMA m8n8k4: %d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
        dfma_k<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_k<<<blocks, threads>>>(out, iters / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * 16 * (iters / 4) * (double)blocks * threads;
        printf("DFMA        : %d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Does the fp64 tensor path (DMMA) share the DFMA datapath?  Time DMMA alone,
// DFMA alone and both interleaved (independent chains, same flop counts).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix_probe tools/fp64_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool DO_MMA, bool DO_FMA>
__global__ void mix_k(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    double c[8][2], f[8];
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = i; f[i] = threadIdx.x + i; }
    const double fb = 0.999999, fc = 1e-9;
    for (int it = 0; it < iters; ++it) {
        if (DO_MMA) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
        if (DO_FMA) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = fma(f[i], fb, fc);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
    if (s == 123.456) out[0] = s;
}

template <typename K>
float timeit(K k, double* out, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<sms * 2, 256>>>(out, 100);
    cudaEventRecord(e0);
    k<<<sms * 2, 256>>>(out, 20000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    float tm = timeit(mix_k<true, false>, out, sms);
    float tf = timeit(mix_k<false, true>, out, sms);
    float tb = timeit(mix_k<true, true>, out, sms);
    printf("DMMA alone %.3f ms, DFMA alone %.3f ms (same flops), both %.3f ms -> %s\n", tm, tf, tb,
           tb > 0.8 * (tm + tf) ? "shared datapath" : "separate pipes");
    return 0;
}

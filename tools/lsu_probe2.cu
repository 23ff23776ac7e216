// Microbenchmark: cost of shared-memory loads where groups of lanes share an
// address (one stencil per lane group), against warp-uniform and fully distinct
// 64-bit loads.  Printed: SM cycles per warp-instruction at full occupancy.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lsu_probe2 tools/lsu_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

// G = lanes per address group (32: uniform, 16: two addresses, 8: four, 4: eight, 1: distinct)
// the groups' addresses are consecutive doubles (distinct banks)
template <int G>
__global__ void k_lds64_grp(double* out) {
    __shared__ double s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane / G;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += s[(((i * 8 + u) & 31) * 32 + grp) & 2047];
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// four groups whose addresses are PITCH doubles apart (a per-stencil region each)
template <int PITCH>
__global__ void k_lds64_grp4_pitch(double* out) {
    __shared__ double s[4 * 1024];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 3;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += s[grp * PITCH + ((i * 8 + u) & 255)];
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// 128-bit loads shared by groups of 8 lanes (four addresses)
__global__ void k_lds128_grp8(double* out) {
    __shared__ double2 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double2(i, i + 1);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 3;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 v = s[(((i * 8 + u) & 63) * 16 + grp) & 1023];
            acc[u] += v.x * v.y;
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// distinct 64-bit stores, conflict-free
__global__ void k_sts64_dist(double* out) {
    __shared__ double s[32 * 33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double v = lane;
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s[((i * 8 + u + w) & 31) * 33 + lane] = v;
            v += 1.0;
        }
    }
    __syncthreads();
    if (s[lane] == 12345.0) out[0] = v;
}

// shuffle from one source lane per 8-lane group
__global__ void k_shfl64_grp8(double* out) {
    const int lane = threadIdx.x & 31;
    double x = lane * 1.5;
    double acc[8] = {};
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += __shfl_sync(0xffffffffu, x, (lane & ~7) | ((i * 8 + u) & 7));
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 12345.0) out[0] = t;
}

// DMMA m8n8k4 f64, 8 independent accumulators
__global__ void k_dmma(double* out) {
    const int lane = threadIdx.x & 31;
    double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    double c[8][2] = {};
    for (int i = 0; i < ITER / 4; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += c[u][0] + c[u][1];
    if (t == 12345.0) out[0] = t;
}

template <typename K>
void run(const char* name, K k, double* out, int sms, double ops_scale = 1.0) {
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
    const double warp_ops = (double)blocks * threads / 32 * ITER * 8 * ops_scale;
    const double cyc = ms * 1e-3 * clk * 1e3 * sms;
    printf("%-22s %8.3f ms  %6.3f SM-cycles per warp-op (per SM)\n", name, ms, cyc / warp_ops);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("lds64 uniform", k_lds64_grp<32>, out, sms);
    run("lds64 2 addr (16)", k_lds64_grp<16>, out, sms);
    run("lds64 4 addr (8)", k_lds64_grp<8>, out, sms);
    run("lds64 8 addr (4)", k_lds64_grp<4>, out, sms);
    run("lds64 16 addr (2)", k_lds64_grp<2>, out, sms);
    run("lds64 distinct", k_lds64_grp<1>, out, sms);
    run("lds64 4 addr pitch 1024", k_lds64_grp4_pitch<1024>, out, sms);
    run("lds64 4 addr pitch 1025", k_lds64_grp4_pitch<1025>, out, sms);
    run("lds64 4 addr pitch 1028", k_lds64_grp4_pitch<1028>, out, sms);
    run("lds128 4 addr (8)", k_lds128_grp8, out, sms);
    run("sts64 distinct", k_sts64_dist, out, sms);
    run("shfl64 grp8 src", k_shfl64_grp8, out, sms);
    run("dmma m8n8k4", k_dmma, out, sms, 0.25);
    return 0;
}

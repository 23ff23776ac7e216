// C-ABI housekeeping: version and per-thread error text.
#include <cstdarg>

#include "common.cuh"

#include <atomic>
#include <mutex>
#include <vector>

namespace mf {
static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
constexpr int MAX_DEV = 64;
struct DevProps {
    std::atomic<int> sms{0};
    std::atomic<int> smem{0};
};
DevProps g_props[MAX_DEV];
std::mutex g_attr_mu;
struct AttrRec {
    const void* fn;
    int dev;
    int bytes;
};
std::vector<AttrRec> g_attrs;
struct OccRec {
    const void* fn;
    int dev;
    int threads;
    size_t smem;
    int blocks;
};
std::vector<OccRec> g_occ;

int cur_dev() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < MAX_DEV ? dev : 0;
}
}  // namespace

int dev_sms() {
    const int dev = cur_dev();
    int v = g_props[dev].sms.load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        g_props[dev].sms.store(v, std::memory_order_relaxed);
    }
    return v;
}

int dev_max_smem_optin() {
    const int dev = cur_dev();
    int v = g_props[dev].smem.load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (v <= 0) v = 48 * 1024;
        g_props[dev].smem.store(v, std::memory_order_relaxed);
    }
    return v;
}

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;  // the default limit covers it
    const int dev = cur_dev();
    std::lock_guard<std::mutex> g(g_attr_mu);
    for (auto& r : g_attrs)
        if (r.fn == fn && r.dev == dev) {
            if (r.bytes >= bytes) return cudaSuccess;
            const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            if (e == cudaSuccess) r.bytes = bytes;
            return e;
        }
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) g_attrs.push_back({fn, dev, bytes});
    return e;
}

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
int occupancy_attr(const void* fn, int threads, size_t smem) {
    const int dev = cur_dev();
    std::lock_guard<std::mutex> g(g_attr_mu);
    for (auto& r : g_occ)
        if (r.fn == fn && r.dev == dev && r.threads == threads && r.smem == smem) return r.blocks;
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess || b < 1) b = 1;
    g_occ.push_back({fn, dev, threads, smem, b});
    return b;
}
}  // namespace mf

extern "C" int mf_abi_version(void) { return MF_ABI_VERSION; }
extern "C" const char* mf_last_error(void) { return mf::g_err; }

extern "C" long long mf_launch_count(void) { return mf::g_launches.load(); }

// ---- fp64 pipe probe: the denominator of the shape-solve roofline -----------
// 8 independent DFMA chains per thread; 2 flops per DFMA.
__global__ void dfma_probe_k(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 12345.0) out[0] = s;
}

extern "C" int mf_dfma_probe(int blocks, int threads, int iters, double* out, void* stream, double* flops) {
    dfma_probe_k<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters);
    MF_LAUNCH_CHECK();
    *flops = 2.0 * 8.0 * 16.0 * (double)iters * (double)blocks * (double)threads;
    return MF_OK;
}

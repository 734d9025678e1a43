// probe.cu -- ALU peak probes for the bench's second roofline (SURVEY.md 8(d):
// the merge is bound by int64 multiply-add issue, compositing by the FP64
// pipe).  Each thread runs 8 independent chains so issue, not latency, binds.
#include <cuda_runtime.h>

#include <cstdint>

#include "host.hpp"

namespace sphray_b200 {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_probe_int64(uint64_t seed, uint64_t* sink) {
    uint64_t a[kChains];
    const uint64_t x = seed | 1ull, y = seed ^ 0x9e3779b97f4a7c15ull;
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x + c;
#pragma unroll 4
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = a[c] * x + y;  // one int64 mul + one int64 add
    uint64_t r = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) r ^= a[c];
    if (r == 0x123456789ull) sink[0] = r;  // keeps the chains alive
}

__global__ void k_probe_fp64(double seed, double* sink) {
    double a[kChains];
    const double x = 0.999999 + seed * 1e-9, y = 1e-7;
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x + c;
#pragma unroll 4
    for (int i = 0; i < kIters; ++i)
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = fma(a[c], x, y);  // 2 flops
    double r = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) r += a[c];
    if (r == 1.2345) sink[0] = r;
}

template <class K, class... A>
double best_ms(K kern, int blocks, A... args) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, 256>>>(args...);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

}  // namespace

void probe_alu_peaks(int device, double* int64_gops, double* fp64_gflops) {
    if (cudaSetDevice(device) != cudaSuccess) fail(SPHRAY_ERR_CUDA, "probe: cudaSetDevice failed");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    void* sink = nullptr;
    if (cudaMalloc(&sink, 64) != cudaSuccess) fail(SPHRAY_ERR_CUDA, "probe: cudaMalloc failed");
    const int blocks = sms * 8;
    const double n = static_cast<double>(blocks) * 256 * kIters * kChains * 2;  // ops per launch
    const double ms_i = best_ms(k_probe_int64, blocks, static_cast<uint64_t>(12345), static_cast<uint64_t*>(sink));
    const double ms_f = best_ms(k_probe_fp64, blocks, 0.5, static_cast<double*>(sink));
    cudaFree(sink);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(SPHRAY_ERR_CUDA, std::string("probe: ") + cudaGetErrorString(e));
    *int64_gops = n / (ms_i * 1e-3) / 1e9;
    *fp64_gflops = n / (ms_f * 1e-3) / 1e9;
}

}  // namespace sphray_b200

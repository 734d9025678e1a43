// accumulate.cu -- accumulate<int64_t> (raycast.hpp:261-292) for explicit,
// sorted knot streams (one per ray), on the GPU: the merge of the render
// kernel without the window.  One warp per ray, lane-blocked: lane l takes the
// l-th contiguous run of the ray's knots, sums its jumps Taylor-shifted to the
// ray's first position tref, one warp scan per order (modulo 2^64, exact
// whenever the exact coefficients fit int64) gives every lane
// the sum of all earlier jumps, and each lane walks its run with the
// RayAccumulator recurrence (raycast.hpp:206-249).  Every step and every run
// start carries the render kernel's genuine-overflow tests
// (render_kernel.cuh shift_overflows / add_checked).  Output per knot: the
// coefficients after it and whether it closes its position (the last knot at
// a distinct t) -- the host keeps the closing ones, i.e. one FieldPiece per
// distinct position, in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "device_math.cuh"
#include "host.hpp"
#include "render.cuh"

namespace sphray_b200 {
namespace {

using namespace dev;

constexpr unsigned kFull = 0xffffffffu;
constexpr int kJ = kMaxDegree + 1;  // jumps per knot in the caller's layout

template <int D>
__device__ __forceinline__ bool shift_bad(const double (&v)[D + 1], double delta, const uint64_t (&w)[D + 1]) {
    double p[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) p[d] = v[d];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) p[j] = fma(delta, p[j + 1], p[j]);
    bool bad = false;
#pragma unroll
    for (int d = 0; d <= D; ++d)
        bad |= !(fabs(p[d] - static_cast<double>(static_cast<int64_t>(w[d]))) < 0x1p62);
    return bad;
}

template <int D>
__device__ __forceinline__ void to_double(const uint64_t (&a)[D + 1], double (&v)[D + 1]) {
#pragma unroll
    for (int d = 0; d <= D; ++d) v[d] = static_cast<double>(static_cast<int64_t>(a[d]));
}

template <int D>
__global__ void k_accumulate(const uint64_t* koff, const int64_t* kt, const int64_t* kb, const uint64_t* ray_ids,
                             size_t nrays, int64_t* out_a, uint8_t* closes, unsigned long long* ovf_ray) {
    const int lane = threadIdx.x & 31;
    const size_t warps = static_cast<size_t>(gridDim.x) * (blockDim.x >> 5);
    for (size_t r = static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrays;
         r += warps) {
        const uint64_t b0 = koff[r], b1 = koff[r + 1];
        if (b1 == b0) continue;
        const uint64_t n = b1 - b0, R = (n + 31) / 32;
        const uint64_t lo = static_cast<uint64_t>(lane) * R, hi = lo + R;
        const uint64_t k0 = b0 + (lo < n ? lo : n), k1 = b0 + (hi < n ? hi : n);
        const int64_t tref = kt[b0];
        uint64_t S[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) S[d] = 0;
        for (uint64_t k = k0; k < k1; ++k) {
            uint64_t g[D + 1];
#pragma unroll
            for (int d = 0; d <= D; ++d) g[d] = static_cast<uint64_t>(kb[k * kJ + d]);
            taylor_shift<D>(g, static_cast<uint64_t>(tref) - static_cast<uint64_t>(kt[k]));
#pragma unroll
            for (int d = 0; d <= D; ++d) S[d] += g[d];
        }
        uint64_t E[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) {
            uint64_t v = S[d];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t u = __shfl_up_sync(kFull, v, o);
                if (lane >= o) v += u;
            }
            E[d] = v - S[d];
        }
        bool bad = false;
        uint64_t Pc[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) Pc[d] = E[d];
        int64_t tcur = k0 < k1 ? kt[k0] : 0;
        if (k0 < k1) taylor_shift<D>(Pc, static_cast<uint64_t>(tcur) - static_cast<uint64_t>(tref));
        uint64_t Ps[D + 1];  // the run's entering state, for the cross-lane test
#pragma unroll
        for (int d = 0; d <= D; ++d) Ps[d] = Pc[d];
        for (uint64_t k = k0; k < k1; ++k) {
            const int64_t t = kt[k];
            if (t != tcur) {
                double v[D + 1];
                to_double<D>(Pc, v);
                const uint64_t dl = static_cast<uint64_t>(t) - static_cast<uint64_t>(tcur);
                taylor_shift<D>(Pc, dl);
                bad |= shift_bad<D>(v, static_cast<double>(static_cast<int64_t>(dl)), Pc);
                tcur = t;
            }
#pragma unroll
            for (int d = 0; d <= D; ++d) {
                const uint64_t j = static_cast<uint64_t>(kb[k * kJ + d]);
                const uint64_t s = Pc[d] + j;
                bad |= static_cast<int64_t>((Pc[d] ^ s) & (j ^ s)) < 0;
                Pc[d] = s;
            }
            const bool close = k + 1 == b1 || kt[k + 1] != t;
            closes[k] = close;
            if (close)
#pragma unroll
                for (int d = 0; d <= D; ++d) out_a[k * (D + 1) + d] = static_cast<int64_t>(Pc[d]);
        }
        // the state entering lane l's run must be the exact shift of lane l-1's end state
        const int64_t tl = static_cast<int64_t>(
            __shfl_up_sync(kFull, static_cast<unsigned long long>(k1 > k0 ? kt[k1 - 1] : 0), 1));
        double v[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d)
            v[d] = static_cast<double>(static_cast<int64_t>(__shfl_up_sync(kFull, static_cast<unsigned long long>(Pc[d]), 1)));
        if (lane > 0 && k0 < k1)
            bad |= shift_bad<D>(
                v, static_cast<double>(static_cast<int64_t>(static_cast<uint64_t>(kt[k0]) - static_cast<uint64_t>(tl))), Ps);
        if (__any_sync(kFull, bad) && lane == 0) atomicMin(ovf_ray, static_cast<unsigned long long>(ray_ids[r]));
    }
}

#define ACC_CUDA_OK(x)                                                             \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

struct Buf {
    void* p = nullptr;
    explicit Buf(size_t b) { ACC_CUDA_OK(cudaMalloc(&p, b ? b : 1)); }
    ~Buf() { cudaFree(p); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace

// Host side of sphray_accumulate.  knot_b: kMaxDegree + 1 jumps per knot.
void accumulate_knots(int D, size_t nrays, const uint64_t* ray_ids, const uint64_t* koff, const int64_t* kt,
                      const int64_t* kb, uint64_t* piece_off, int64_t* piece_t, int64_t* piece_a, uint64_t* ops,
                      cudaStream_t s) {
    if (D < 1 || D > kMaxDegree) fail(SPHRAY_ERR_CONFIG, "accumulate: degree out of range");
    if (nrays == 0) {
        if (piece_off) piece_off[0] = 0;
        return;
    }
    const uint64_t nk = koff[nrays];
    for (size_t r = 0; r < nrays; ++r) {
        if (koff[r + 1] < koff[r]) fail(SPHRAY_ERR_CONFIG, "accumulate: knot offsets decrease");
        for (uint64_t k = koff[r] + 1; k < koff[r + 1]; ++k)
            if (kt[k] < kt[k - 1])  // raycast.hpp:212-213
                fail(SPHRAY_ERR_NUMERIC, "accumulate: knots not sorted along the ray");
    }
    Buf dko((nrays + 1) * 8), dkt(nk * 8), dkb(nk * kJ * 8), drid(nrays * 8), da(nk * (D + 1) * 8), dcl(nk),
        dovf(8);
    ACC_CUDA_OK(cudaMemcpyAsync(dko.p, koff, (nrays + 1) * 8, cudaMemcpyHostToDevice, s));
    ACC_CUDA_OK(cudaMemcpyAsync(dkt.p, kt, nk * 8, cudaMemcpyHostToDevice, s));
    ACC_CUDA_OK(cudaMemcpyAsync(dkb.p, kb, nk * kJ * 8, cudaMemcpyHostToDevice, s));
    ACC_CUDA_OK(cudaMemcpyAsync(drid.p, ray_ids, nrays * 8, cudaMemcpyHostToDevice, s));
    ACC_CUDA_OK(cudaMemsetAsync(dovf.p, 0xff, 8, s));
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((nrays + 3) / 4, 148 * 16));
#define ACC_LAUNCH(DD)                                                                                   \
    k_accumulate<DD><<<blocks, 128, 0, s>>>(dko.as<uint64_t>(), dkt.as<int64_t>(), dkb.as<int64_t>(),   \
                                            drid.as<uint64_t>(), nrays, da.as<int64_t>(), dcl.as<uint8_t>(), \
                                            dovf.as<unsigned long long>())
    switch (D) {
        case 1: ACC_LAUNCH(1); break;
        case 2: ACC_LAUNCH(2); break;
        case 3: ACC_LAUNCH(3); break;
        case 4: ACC_LAUNCH(4); break;
        case 5: ACC_LAUNCH(5); break;
        default: ACC_LAUNCH(6); break;
    }
#undef ACC_LAUNCH
    ACC_CUDA_OK(cudaGetLastError());
    std::vector<int64_t> a(nk * (D + 1));
    std::vector<uint8_t> cl(nk);
    unsigned long long ovf = 0;
    ACC_CUDA_OK(cudaMemcpyAsync(a.data(), da.p, a.size() * 8, cudaMemcpyDeviceToHost, s));
    ACC_CUDA_OK(cudaMemcpyAsync(cl.data(), dcl.p, nk, cudaMemcpyDeviceToHost, s));
    ACC_CUDA_OK(cudaMemcpyAsync(&ovf, dovf.p, 8, cudaMemcpyDeviceToHost, s));
    ACC_CUDA_OK(cudaStreamSynchronize(s));
    if (ovf != ~0ull)
        fail(SPHRAY_ERR_OVERFLOW, "accumulate: integer overflow (ray " + std::to_string(ovf) + ")", -1, ovf);
    uint64_t np = 0;
    for (size_t r = 0; r < nrays; ++r) {
        if (piece_off) piece_off[r] = np;
        const uint64_t first = np;
        for (uint64_t k = koff[r]; k < koff[r + 1]; ++k) {
            if (!cl[k]) continue;
            if (piece_t) piece_t[np] = kt[k];
            if (piece_a)
                for (int d = 0; d <= D; ++d) piece_a[np * (D + 1) + d] = a[k * (D + 1) + d];
            ++np;
        }
        // RayAccumulator op count for P distinct positions (raycast.hpp:217-244)
        const uint64_t P = np - first;
        if (ops) ops[r] = P > 0 ? P * (D + 1) + (P - 1) * ((D + 1) * (3 * D + 4) / 2) : 0;
    }
    if (piece_off) piece_off[nrays] = np;
}

}  // namespace sphray_b200

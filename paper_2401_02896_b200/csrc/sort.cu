// sort.cu -- hand-written device scan and stable LSD radix sort (sm_100a) for
// the acceleration structure: the Morton order of the resident particle set,
// the per-frame depth order of the particles, the (tile, particle) binning,
// and the dataset-statistics medians.  No library kernels.
//
// Scan: three passes (block sums, one-block scan of the sums, block scans
// with their offsets); 2 reads + 1 write of the input.
//
// Radix sort, per 8-bit digit: (1) k_digit_hist -- per-tile digit counts
// written digit-major (count[d * tiles + b]); (2) the scan above turns them
// into the global output position of every (digit, tile) run; (3)
// k_digit_scatter -- each warp ranks its 512 consecutive items with
// __match_any_sync (stable: rounds of 32 in order, ranks within a round from
// the lane mask), the CTA folds the warp counts into per-(warp, digit)
// offsets in shared memory, and every item is written to
// base[digit] + warp offset + rank.  Stable, so LSD passes compose.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "render.cuh"

namespace sphray_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 8192
constexpr int kSortWarps = 8;
constexpr int kSortThreads = kSortWarps * 32;

#define SORT_CUDA_OK(x)                                                            \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

template <class T>
__device__ __forceinline__ T warp_incl(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// exclusive scan of the CTA's values (one per thread); returns the CTA total
template <class T>
__device__ __forceinline__ T block_excl(T v, T* wsum, T& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const T inc = warp_incl(v, lane);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T x = lane < nw ? wsum[lane] : T(0);
        const T xi = warp_incl(x, lane);
        if (lane < nw) wsum[lane] = xi - x;
        if (lane == nw - 1) wsum[32] = xi;
    }
    __syncthreads();
    const T out = wsum[warp] + inc - v;
    total = wsum[32];
    __syncthreads();
    return out;
}

// ---------------------------------------------------------------- scan
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* in, size_t n, T* sums) {
    __shared__ T wsum[33];
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) s += in[base + k];
    T total;
    (void)block_excl(s, wsum, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// one CTA: exclusive scan of m tile sums in place (m arbitrary, in chunks)
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* sums, size_t m, T* grand) {
    __shared__ T wsum[33];
    T carry = 0;
    for (size_t c0 = 0; c0 < m; c0 += kScanThreads) {
        const size_t i = c0 + threadIdx.x;
        const T v = i < m ? sums[i] : T(0);
        T total;
        const T ex = block_excl(v, wsum, total);
        if (i < m) sums[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && grand) *grand = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, T* out, size_t n, const T* sums) {
    __shared__ T wsum[33];
    const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
    T v[kScanItems];
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? in[base + k] : T(0);
        s += v[k];
    }
    T total;
    T run = block_excl(s, wsum, total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

// ---------------------------------------------------------------- radix sort
// Items per CTA tile: 4096 for 32-bit keys, 2048 for 64-bit keys (the tile is
// reordered in shared memory before it is written out).
template <class K>
constexpr int sort_rounds() {
    return sizeof(K) == 8 ? 8 : 16;
}
template <class K>
constexpr int sort_tile() {
    return kSortThreads * sort_rounds<K>();
}

template <class K>
__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const K* keys, size_t n, int shift,
                                                             uint32_t* counts, uint32_t tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(blockIdx.x) * sort_tile<K>();
#pragma unroll 4
    for (int k = 0; k < sort_rounds<K>(); ++k) {
        const size_t i = base + static_cast<size_t>(k) * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[static_cast<uint32_t>(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    counts[static_cast<size_t>(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one tile: each warp ranks its consecutive items per digit
// (__match_any_sync rounds of 32, in order); the tile is reordered by digit in
// shared memory and written out as contiguous runs (coalesced stores).
template <class K, bool VALS>
__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(const K* kin, K* kout, const uint32_t* vin,
                                                                uint32_t* vout, size_t n, int shift,
                                                                const uint32_t* offsets, uint32_t tiles) {
    constexpr int R = sort_rounds<K>(), T = sort_tile<K>();
    __shared__ uint32_t wc[kSortWarps][256];  // per-warp digit counters, then offsets within the digit
    __shared__ uint32_t dstart[256], gbase[256], wsum[33];
    __shared__ K skey[T];
    __shared__ uint32_t sval[VALS ? T : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const size_t tile0 = static_cast<size_t>(blockIdx.x) * T;
    const size_t base = tile0 + static_cast<size_t>(warp) * (32 * R);
    K key[R];
    uint32_t val[R];
    uint32_t rank[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const size_t i = base + static_cast<size_t>(r) * 32 + lane;
        const bool ok = i < n;
        key[r] = ok ? kin[i] : K(0);
        if constexpr (VALS) val[r] = ok ? vin[i] : 0u;
        const uint32_t dg = static_cast<uint32_t>(key[r] >> shift) & 255u;
        const unsigned peers = __match_any_sync(kFull, ok ? dg : 256u + lane);
        const uint32_t before = wc[warp][dg];
        rank[r] = before + __popc(peers & lanemask_lt());
        __syncwarp();
        if (ok && (peers & lanemask_lt()) == 0) wc[warp][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t cnt;
    {  // per digit: exclusive prefix over the warps; the tile's count and global base
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = wc[w][d];
            wc[w][d] = run;
            run += c;
        }
        cnt = run;
        gbase[d] = offsets[static_cast<size_t>(d) * tiles + blockIdx.x];
    }
    uint32_t total;
    dstart[threadIdx.x] = block_excl(cnt, wsum, total);  // syncs inside
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const size_t i = base + static_cast<size_t>(r) * 32 + lane;
        if (i < n) {
            const uint32_t dg = static_cast<uint32_t>(key[r] >> shift) & 255u;
            const uint32_t at = dstart[dg] + wc[warp][dg] + rank[r];
            skey[at] = key[r];
            if constexpr (VALS) sval[at] = val[r];
        }
    }
    __syncthreads();
    const uint32_t valid = static_cast<uint32_t>(n - tile0 < static_cast<size_t>(T) ? n - tile0 : T);
    for (uint32_t i = threadIdx.x; i < valid; i += kSortThreads) {
        const K k = skey[i];
        const uint32_t dg = static_cast<uint32_t>(k >> shift) & 255u;
        const uint32_t at = gbase[dg] + (i - dstart[dg]);
        kout[at] = k;
        if constexpr (VALS) vout[at] = sval[i];
    }
}

unsigned grid_of(size_t n, size_t per) { return static_cast<unsigned>((n + per - 1) / per); }

template <class T>
size_t scan_tmp_elems(size_t n) {
    return grid_of(n, kScanTile) + 1;
}

// exclusive scan; tmp holds scan_tmp_elems(n) elements; *total (device) optional
template <class T>
void scan_impl(const T* in, T* out, size_t n, T* tmp, T* total, cudaStream_t s) {
    if (n == 0) return;
    const unsigned g = grid_of(n, kScanTile);
    k_tile_sums<T><<<g, kScanThreads, 0, s>>>(in, n, tmp);
    k_scan_sums<T><<<1, kScanThreads, 0, s>>>(tmp, g, total);
    k_tile_scan<T><<<g, kScanThreads, 0, s>>>(in, out, n, tmp);
    SORT_CUDA_OK(cudaGetLastError());
}

template <class K>
void sort_impl(K* k0, K* k1, uint32_t* v0, uint32_t* v1, size_t n, int end_bit, void* tmp,
               cudaStream_t s, bool& result_in_first) {
    result_in_first = true;
    if (n == 0) return;
    if (n >= 0xffffffffull) fail(SPHRAY_ERR_CAPACITY, "radix sort: more than 2^32 - 1 items");
    const uint32_t tiles = grid_of(n, sort_tile<K>());
    const size_t m = static_cast<size_t>(256) * tiles;
    uint32_t* counts = static_cast<uint32_t*>(tmp);
    uint32_t* stmp = counts + m;
    K* src = k0;
    K* dst = k1;
    uint32_t* vs = v0;
    uint32_t* vd = v1;
    for (int shift = 0; shift < end_bit; shift += 8) {
        k_digit_hist<K><<<tiles, kSortThreads, 0, s>>>(src, n, shift, counts, tiles);
        scan_impl<uint32_t>(counts, counts, m, stmp, nullptr, s);
        if (vs)
            k_digit_scatter<K, true><<<tiles, kSortThreads, 0, s>>>(src, dst, vs, vd, n, shift, counts, tiles);
        else
            k_digit_scatter<K, false><<<tiles, kSortThreads, 0, s>>>(src, dst, nullptr, nullptr, n, shift,
                                                                     counts, tiles);
        SORT_CUDA_OK(cudaGetLastError());
        std::swap(src, dst);
        std::swap(vs, vd);
        result_in_first = !result_in_first;
    }
}

}  // namespace

size_t scan_tmp_bytes(size_t n) { return scan_tmp_elems<uint32_t>(n) * sizeof(uint32_t) + 16; }

void scan_u32(const uint32_t* in, uint32_t* out, size_t n, void* tmp, uint32_t* total_dev, cudaStream_t s) {
    scan_impl<uint32_t>(in, out, n, static_cast<uint32_t*>(tmp), total_dev, s);
}

size_t radix_tmp_bytes(size_t n) {
    const size_t tiles = grid_of(n, sort_tile<uint32_t>() < sort_tile<unsigned long long>()
                                        ? sort_tile<uint32_t>() : sort_tile<unsigned long long>());
    const size_t m = 256 * tiles;
    return (m + scan_tmp_elems<uint32_t>(m)) * sizeof(uint32_t) + 16;
}

int radix_passes(int end_bit) { return (end_bit + 7) / 8; }

// Stable LSD sort of (keys, values) on the low end_bit bits (values optional:
// vin == nullptr sorts keys only).  Buffers ping-pong; returns true when the
// sorted data ends in (kout, vout), false when in (kin, vin).
bool sort_pairs_u64(unsigned long long* kin, unsigned long long* kout, uint32_t* vin, uint32_t* vout,
                    size_t n, int end_bit, void* tmp, cudaStream_t s) {
    bool in_first = true;
    sort_impl<unsigned long long>(kin, kout, vin, vout, n, end_bit, tmp, s, in_first);
    return !in_first;
}

bool sort_pairs_u32(uint32_t* kin, uint32_t* kout, uint32_t* vin, uint32_t* vout, size_t n, int end_bit,
                    void* tmp, cudaStream_t s) {
    bool in_first = true;
    sort_impl<uint32_t>(kin, kout, vin, vout, n, end_bit, tmp, s, in_first);
    return !in_first;
}

}  // namespace sphray_b200

// render.cu -- the B200 hot path: per-ray candidate gather + exact hit test,
// quantized knot emission from the Lambda-indexed LUT, per-ray windowed sort
// and exact integer merge (prefix sum of Taylor-shifted jumps), transfer-
// function classification and front-to-back compositing with early ray
// termination.  One warp owns one ray; its pending knots live in a shared
// memory window that is flushed in depth order as the depth-sorted candidate
// list of its screen tile advances (the global knot array of the reference,
// raycast.hpp:448-455, is never materialised).
//
// Reference path replaced (all under /root/reference/proj/include/sphray):
//   particle_ray_footprint  raycast.hpp:128-184   -> k_prep (bbox) + tile binning + gather
//   detail::hit_ray         raycast.hpp:111-120   -> dev::hit_test + dev::lam_of
//   quantize_particle<Int>  quantize.hpp:199-250  -> quantize.cuh phases A/B
//   mirror_closure<T>       lut.hpp:100-168       -> quantize.cuh
//   sort_knots              raycast.hpp:188-194   -> flush-set select + warp radix sort
//   accumulate/RayAccumulator raycast.hpp:206-292 -> RayWorker::merge_composite / walk
//   composite/evaluate_piece/TransferFunction::sample raycast.hpp:295-381 -> Compositor
//   render_scene            raycast.hpp:414-497   -> k_render_rays + engine.cpp
#include <cuda_runtime.h>

#include <cstring>

#include "device_math.cuh"
#include "render.cuh"

namespace sphray_b200 {

using namespace dev;

namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
__global__ void k_prep(const PrepParams p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.n) return;
    const double4 a = p.pxyzh[i];
    const double support = dmul(p.q, a.w);  // raycast.hpp:131
    int px0, px1, py0, py1;
    footprint_bbox(p.cam, a.x, a.y, a.z, support, px0, px1, py0, py1);
    p.bbox[i] = make_int4(px0, px1, py0, py1);
    p.front[i] = __double2float_rd(front_bound(p.cam, a.x, a.y, a.z, support, a.w * p.reach_scale));
    uint32_t cnt = 0;
    if (px0 <= px1 && py0 <= py1) {
        const int tx0 = px0 >> kTileShift, tx1 = px1 >> kTileShift;
        const int ty0 = py0 >> kTileShift, ty1 = py1 >> kTileShift;
        if (p.nranks == 1) {
            cnt = static_cast<uint32_t>((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        } else {
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) cnt += ((ty * p.tiles_x + tx) % p.nranks) == p.rank;
        }
    }
    p.counts[i] = cnt;
    // X_d = (pow(tau,d)*mass)*value, Y_d = (sigma*density)*pow(h,d+3)   (quantize.hpp:221-222)
    const double4 m = p.mvr[i];
    double* xy = p.xy + static_cast<size_t>(i) * 3 * p.D;
    for (int d = 1; d <= p.D; ++d) {
        xy[d - 1] = dmul(dmul(p.powtau[d - 1], m.x), m.y);
        const double y = dmul(dmul(p.sigma, m.z), p.powh[static_cast<size_t>(i) * p.D + d - 1]);
        xy[p.D + d - 1] = y;
        xy[2 * p.D + d - 1] = recip_or_nan(y);
    }
}

__device__ __forceinline__ uint32_t orderable(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void k_depth_keys(const float* front, int n, uint32_t* keys, uint32_t* vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = orderable(front[i]);
    vals[i] = static_cast<uint32_t>(i);
}

// counts in depth order, and their exact 64-bit total (the entry count)
__global__ void k_gather_counts(const uint32_t* counts, const uint32_t* order, int n, uint32_t* out,
                                unsigned long long* total) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (j < n) {
        c = counts[order[j]];
        out[j] = static_cast<uint32_t>(c);
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, c);
}

// Entries of the particle at depth rank j, at offsets[j]: the entry array is
// in depth order, so a stable sort by tile leaves every tile's candidates
// sorted by their front bound (what the render kernel's flush bound needs).
__global__ void k_emit(const PrepParams p, const uint32_t* order, const uint32_t* offsets, uint32_t* keys,
                       uint32_t* vals) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.n) return;
    const uint32_t i = order[j];
    const int4 b = p.bbox[i];
    if (!(b.x <= b.y && b.z <= b.w)) return;
    uint32_t o = offsets[j];
    const int tx0 = b.x >> kTileShift, tx1 = b.y >> kTileShift;
    const int ty0 = b.z >> kTileShift, ty1 = b.w >> kTileShift;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            const uint32_t tile = static_cast<uint32_t>(ty * p.tiles_x + tx);
            if (p.nranks > 1 && static_cast<int>(tile % p.nranks) != p.rank) continue;
            keys[o] = p.nranks > 1 ? tile / p.nranks : tile;
            vals[o] = i;
            ++o;
        }
}

__global__ void k_tile_ranges(const uint32_t* keys, size_t m, uint32_t* begin, uint32_t* end) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) begin[t] = static_cast<uint32_t>(i);
    if (i == m - 1 || keys[i + 1] != t) end[t] = static_cast<uint32_t>(i + 1);
}

__global__ void k_records(const uint32_t* tile_keys, const uint32_t* cand, size_t m, const double4* pxyzh,
                          const int4* bbox, const float* front, int tiles_x, int rank, int nranks,
                          double4* cxyzh, uint4* cmeta) {
    const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const uint32_t i = cand[j];
    const uint32_t local = tile_keys[j];
    const uint32_t tile = nranks > 1 ? local * nranks + rank : local;
    const int tx0 = static_cast<int>(tile % tiles_x) * kTile, ty0 = static_cast<int>(tile / tiles_x) * kTile;
    const int4 b = bbox[i];
    const uint32_t x0 = max(b.x - tx0, 0), x1 = min(b.y - tx0, kTile - 1);
    const uint32_t y0 = max(b.z - ty0, 0), y1 = min(b.w - ty0, kTile - 1);
    cxyzh[j] = pxyzh[i];
    cmeta[j] = make_uint4(__float_as_uint(front[i]), i, x0 | (x1 << 4) | (y0 << 8) | (y1 << 12), 0u);
}

// skipped_particles (raycast.hpp:437-438, 452): particles with an empty footprint.
__global__ void k_reach(const CamConst cam, int n, double q, const double4* pxyzh,
                        const int4* bbox, unsigned long long* skipped) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool reach = false;
    if (i < n) {
        const int4 b = bbox[i];
        if (b.x <= b.y && b.z <= b.w) {
            const double4 a = pxyzh[i];
            const double support = dmul(q, a.w);
            double lam, t;
            const int cx = (b.x + b.y) >> 1, cy = (b.z + b.w) >> 1;
            reach = hit_ray(make_ray(cam, cx, cy), a.x, a.y, a.z, support, a.w, cam.near_plane,
                            cam.far_plane, lam, t);
            for (int py = b.z; py <= b.w && !reach; ++py)
                for (int px = b.x; px <= b.y && !reach; ++px)
                    reach = hit_ray(make_ray(cam, px, py), a.x, a.y, a.z, support, a.w,
                                    cam.near_plane, cam.far_plane, lam, t);
        }
    }
    const unsigned m = __ballot_sync(kFull, i < n && !reach);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(skipped, static_cast<unsigned long long>(__popc(m)));
}

__global__ void k_unpack(const double* packed, size_t per_rank, int nranks, int tiles_x, int W,
                         int H, double* out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<size_t>(W) * H) return;
    const int px = static_cast<int>(i % W), py = static_cast<int>(i / W);
    const uint64_t tile = static_cast<uint64_t>(py >> kTileShift) * tiles_x + (px >> kTileShift);
    const int rank = static_cast<int>(tile % nranks);
    const uint64_t local = tile / nranks;
    const size_t src = static_cast<size_t>(rank) * per_rank +
                       (local * kTileRays + ((py & (kTile - 1)) << kTileShift) + (px & (kTile - 1))) * 3;
    out[i * 3 + 0] = packed[src + 0];
    out[i * 3 + 1] = packed[src + 1];
    out[i * 3 + 2] = packed[src + 2];
}

__global__ void k_fill_bg(double* rgb, size_t npix, double r, double g, double b) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= npix) return;
    rgb[i * 3 + 0] = r;
    rgb[i * 3 + 1] = g;
    rgb[i * 3 + 2] = b;
}

// Morton order of the resident particle set (view independent).
__device__ __forceinline__ uint64_t spread21(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__global__ void k_morton(const sphray_particle* ps, size_t n, double lx, double ly, double lz,
                         double sx, double sy, double sz, unsigned long long* codes, uint32_t* idx) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto qz = [](double v, double l, double s) {
        double u = (v - l) * s;
        u = u < 0.0 ? 0.0 : (u > 2097151.0 ? 2097151.0 : u);
        return static_cast<uint64_t>(u);
    };
    const uint64_t x = qz(ps[i].x, lx, sx), y = qz(ps[i].y, ly, sy), z = qz(ps[i].z, lz, sz);
    codes[i] = spread21(x) | (spread21(y) << 1) | (spread21(z) << 2);
    idx[i] = static_cast<uint32_t>(i);
}

__global__ void k_scatter_scene(const sphray_particle* ps, const double* powh_in,
                                const uint32_t* perm, size_t n, int D, double4* pxyzh,
                                double4* mvr, double* powh, int32_t* orig) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = perm[i];
    const sphray_particle p = ps[s];
    pxyzh[i] = make_double4(p.x, p.y, p.z, p.h);
    mvr[i] = make_double4(p.mass, p.value, p.density, 0.0);
    for (int d = 0; d < D; ++d) powh[i * D + d] = powh_in[static_cast<size_t>(s) * D + d];
    orig[i] = static_cast<int32_t>(s);
}

// dataset_stats (quantize.hpp:129-165) on the resident scene: the four
// property columns for the medians, phi_max = max |(m v) / (((rho h) h) h)|
// in the reference's operation order, and the positivity check of h, rho.
// dataset_stats columns as orderable u64 keys (the IEEE bit pattern with the
// sign flipped / all bits flipped for negatives sorts like the doubles; -0.0
// and +0.0 compare equal in std::sort and both give the same median value).
__device__ __forceinline__ unsigned long long orderable_f64(double v) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_stats_columns(const double4* pxyzh, const double4* mvr, size_t n, unsigned long long* mass,
                                unsigned long long* density, unsigned long long* h, unsigned long long* value,
                                unsigned long long* phi_bits, unsigned int* bad) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long best = 0ull;
    bool b = false;
    if (i < n) {
        const double4 p = pxyzh[i];
        const double4 q = mvr[i];
        mass[i] = orderable_f64(q.x);
        value[i] = orderable_f64(q.y);
        density[i] = orderable_f64(q.z);
        h[i] = orderable_f64(p.w);
        b = !(p.w > 0.0) || !(q.z > 0.0);
        // p.mass * p.value / (p.density * p.h * p.h * p.h)   (host.cpp / quantize.hpp:141)
        const double num = __dmul_rn(q.x, q.y);
        const double den = __dmul_rn(__dmul_rn(__dmul_rn(q.z, p.w), p.w), p.w);
        const double phi = fabs(__ddiv_rn(num, den));
        best = phi == phi ? __double_as_longlong(phi) : 0ull;  // |phi| >= 0: bits order = value order
    }
    // warp max, one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long u = __shfl_xor_sync(0xffffffffu, best, o);
        best = u > best ? u : best;
    }
    const unsigned any_bad = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(phi_bits, best);
        if (any_bad) atomicOr(bad, 1u);
    }
}

}  // namespace

// defined in render_d<D>.cu (render_kernel.cuh)
template <int D, int M>
int render_occupancy_t(int warps, size_t smem, bool even);
template <int D, int M>
void launch_render_t(const FrameParams& P, int blocks, int warps, cudaStream_t s);
template <int D, int M>
void launch_quantize_hits_t(const QuantParams& Q, const sphray_particle* ps, const double* powh,
                            const double* powtau, size_t nhits, const double* tchi,
                            const double* lam, int64_t* knot_t, int64_t* knot_b,
                            int32_t* knot_count, cudaStream_t s);

// ===========================================================================
#define SPHRAY_CUDA_OK(x)                                                          \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

size_t warp_smem_bytes(int D, int cap, int mm, int jb) {
    (void)mm;
    return warp_bytes_for(D, cap, jb);
}

// Every (D, m) the reference admits: D in [1,6], m = ceil(K/2) in [1,4]
// (approx.hpp:27-30).  SPHRAY_FAST_BUILD keeps only the default D=3, m=2.
#ifdef SPHRAY_FAST_BUILD
#define SPHRAY_DISPATCH(D, MM_, ...)                          \
    switch ((D) * 10 + (MM_)) {                                \
        case 32: { constexpr int DD = 3, MM = 2; __VA_ARGS__; break; } \
        default: fail(SPHRAY_ERR_CONFIG, "unsupported (K, D) in this build"); \
    }
#else
#define SPHRAY_DISPATCH(D, MM_, ...)                          \
    switch ((D) * 10 + (MM_)) {                                \
        case 11: { constexpr int DD = 1, MM = 1; __VA_ARGS__; break; } \
        case 12: { constexpr int DD = 1, MM = 2; __VA_ARGS__; break; } \
        case 13: { constexpr int DD = 1, MM = 3; __VA_ARGS__; break; } \
        case 14: { constexpr int DD = 1, MM = 4; __VA_ARGS__; break; } \
        case 21: { constexpr int DD = 2, MM = 1; __VA_ARGS__; break; } \
        case 22: { constexpr int DD = 2, MM = 2; __VA_ARGS__; break; } \
        case 23: { constexpr int DD = 2, MM = 3; __VA_ARGS__; break; } \
        case 24: { constexpr int DD = 2, MM = 4; __VA_ARGS__; break; } \
        case 31: { constexpr int DD = 3, MM = 1; __VA_ARGS__; break; } \
        case 32: { constexpr int DD = 3, MM = 2; __VA_ARGS__; break; } \
        case 33: { constexpr int DD = 3, MM = 3; __VA_ARGS__; break; } \
        case 34: { constexpr int DD = 3, MM = 4; __VA_ARGS__; break; } \
        case 41: { constexpr int DD = 4, MM = 1; __VA_ARGS__; break; } \
        case 42: { constexpr int DD = 4, MM = 2; __VA_ARGS__; break; } \
        case 43: { constexpr int DD = 4, MM = 3; __VA_ARGS__; break; } \
        case 44: { constexpr int DD = 4, MM = 4; __VA_ARGS__; break; } \
        case 51: { constexpr int DD = 5, MM = 1; __VA_ARGS__; break; } \
        case 52: { constexpr int DD = 5, MM = 2; __VA_ARGS__; break; } \
        case 53: { constexpr int DD = 5, MM = 3; __VA_ARGS__; break; } \
        case 54: { constexpr int DD = 5, MM = 4; __VA_ARGS__; break; } \
        case 61: { constexpr int DD = 6, MM = 1; __VA_ARGS__; break; } \
        case 62: { constexpr int DD = 6, MM = 2; __VA_ARGS__; break; } \
        case 63: { constexpr int DD = 6, MM = 3; __VA_ARGS__; break; } \
        case 64: { constexpr int DD = 6, MM = 4; __VA_ARGS__; break; } \
        default: fail(SPHRAY_ERR_CONFIG, "unsupported (K, D) for the render kernel"); \
    }
#endif

int max_blocks_per_sm(int D, int mm, int warps, size_t smem, bool even) {
    int nb = 0;
    SPHRAY_DISPATCH(D, mm, { nb = render_occupancy_t<DD, MM>(warps, smem, even); });
    return nb;
}

void launch_render(const FrameParams& P, int D, int mm, int blocks, int warps, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(P.warp_bytes) * warps;
    (void)smem;
    SPHRAY_DISPATCH(D, mm, { launch_render_t<DD, MM>(P, blocks, warps, s); });
}

static unsigned grid_for(size_t n, int block) {
    return static_cast<unsigned>((n + block - 1) / block);
}

void launch_prep(const PrepParams& p, cudaStream_t s) {
    if (p.n == 0) return;
    k_prep<<<grid_for(p.n, 256), 256, 0, s>>>(p);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_depth_keys(const float* front, int n, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    if (n == 0) return;
    k_depth_keys<<<grid_for(n, 256), 256, 0, s>>>(front, n, keys, vals);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_gather_counts(const uint32_t* counts, const uint32_t* order, int n, uint32_t* out,
                          unsigned long long* total, cudaStream_t s) {
    if (n == 0) return;
    k_gather_counts<<<grid_for(n, 256), 256, 0, s>>>(counts, order, n, out, total);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_emit(const PrepParams& p, const uint32_t* order, const uint32_t* offsets, uint32_t* keys,
                 uint32_t* vals, cudaStream_t s) {
    if (p.n == 0) return;
    k_emit<<<grid_for(p.n, 256), 256, 0, s>>>(p, order, offsets, keys, vals);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_tile_ranges(const uint32_t* keys, size_t m, uint32_t* begin, uint32_t* end, cudaStream_t s) {
    if (m == 0) return;
    k_tile_ranges<<<grid_for(m, 256), 256, 0, s>>>(keys, m, begin, end);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_records(const uint32_t* tile_keys, const uint32_t* cand, size_t m, const double4* pxyzh,
                    const int4* bbox, const float* front, int tiles_x, int rank, int nranks,
                    double4* cxyzh, uint4* cmeta, cudaStream_t s) {
    if (m == 0) return;
    k_records<<<grid_for(m, 256), 256, 0, s>>>(tile_keys, cand, m, pxyzh, bbox, front, tiles_x, rank, nranks,
                                              cxyzh, cmeta);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_reach(const CamConst& cam, int n, double q, const double4* pxyzh, const int4* bbox,
                  unsigned long long* skipped, cudaStream_t s) {
    if (n == 0) return;
    k_reach<<<grid_for(n, 128), 128, 0, s>>>(cam, n, q, pxyzh, bbox, skipped);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_unpack(const double* packed, size_t per_rank, int nranks, int tiles_x, int W, int H,
                   double* out, cudaStream_t s) {
    k_unpack<<<grid_for(static_cast<size_t>(W) * H, 256), 256, 0, s>>>(packed, per_rank, nranks,
                                                                      tiles_x, W, H, out);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_fill_bg(double* rgb, size_t npix, const double* bg, cudaStream_t s) {
    if (npix == 0) return;
    k_fill_bg<<<grid_for(npix, 256), 256, 0, s>>>(rgb, npix, bg[0], bg[1], bg[2]);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_morton(const sphray_particle* ps, size_t n, const double* lo, const double* inv,
                   unsigned long long* codes, uint32_t* idx, cudaStream_t s) {
    if (n == 0) return;
    k_morton<<<grid_for(n, 256), 256, 0, s>>>(ps, n, lo[0], lo[1], lo[2], inv[0], inv[1], inv[2],
                                              codes, idx);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_scatter_scene(const sphray_particle* ps, const double* powh_in, const uint32_t* perm,
                          size_t n, int D, double4* pxyzh, double4* mvr, double* powh,
                          int32_t* orig, cudaStream_t s) {
    if (n == 0) return;
    k_scatter_scene<<<grid_for(n, 256), 256, 0, s>>>(ps, powh_in, perm, n, D, pxyzh, mvr, powh, orig);
    SPHRAY_CUDA_OK(cudaGetLastError());
}

void launch_quantize_hits(const QuantParams& Q, int D, const sphray_particle* ps,
                          const double* powh, const double* powtau, size_t nhits,
                          const double* tchi, const double* lam, int64_t* knot_t,
                          int64_t* knot_b, int32_t* knot_count, cudaStream_t s) {
    if (nhits == 0) return;
    const int mm = Q.m;
    SPHRAY_DISPATCH(D, mm, {
        launch_quantize_hits_t<DD, MM>(Q, ps, powh, powtau, nhits, tchi, lam, knot_t, knot_b,
                                       knot_count, s);
    });
}

namespace {
struct Scratch {  // RAII device scratch for the one-off statistics pass
    void* p = nullptr;
    explicit Scratch(size_t b) {
        if (cudaMalloc(&p, b ? b : 1) != cudaSuccess) fail(SPHRAY_ERR_CUDA, "dataset_stats: cudaMalloc failed");
    }
    ~Scratch() { cudaFree(p); }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};
}  // namespace

void device_dataset_stats(const double4* pxyzh, const double4* mvr, size_t n, cudaStream_t s,
                          double med[4], double* phi_max, bool* bad) {
    Scratch cols(n * 4 * sizeof(unsigned long long)), alt(n * sizeof(unsigned long long)), small(16),
        tmp(radix_tmp_bytes(n));
    unsigned long long* c = static_cast<unsigned long long*>(cols.p);
    unsigned long long* pb = static_cast<unsigned long long*>(small.p);
    SPHRAY_CUDA_OK(cudaMemsetAsync(small.p, 0, 16, s));
    k_stats_columns<<<grid_for(n, 256), 256, 0, s>>>(pxyzh, mvr, n, c, c + n, c + 2 * n, c + 3 * n, pb,
                                                     reinterpret_cast<unsigned int*>(pb + 1));
    SPHRAY_CUDA_OK(cudaGetLastError());
    unsigned long long* other = static_cast<unsigned long long*>(alt.p);
    for (int k = 0; k < 4; ++k) {
        // medians of sorted columns (detail::median, quantize.hpp:118-122)
        unsigned long long* col = c + k * n;
        const bool in_other = sort_pairs_u64(col, other, nullptr, nullptr, n, 64, tmp.p, s);
        const unsigned long long* sorted = in_other ? other : col;
        unsigned long long mid[2] = {0, 0};
        const size_t a = n % 2 ? n / 2 : n / 2 - 1;
        SPHRAY_CUDA_OK(cudaMemcpyAsync(mid, sorted + a, (n % 2 ? 1 : 2) * sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost, s));
        SPHRAY_CUDA_OK(cudaStreamSynchronize(s));
        double v[2];
        for (int j = 0; j < 2; ++j) {
            const unsigned long long u = (mid[j] & 0x8000000000000000ull) ? (mid[j] & ~0x8000000000000000ull) : ~mid[j];
            std::memcpy(&v[j], &u, sizeof(double));
        }
        med[k] = n % 2 ? v[0] : 0.5 * (v[0] + v[1]);
    }
    unsigned long long hb[2] = {0, 0};
    SPHRAY_CUDA_OK(cudaMemcpyAsync(hb, small.p, 16, cudaMemcpyDeviceToHost, s));
    SPHRAY_CUDA_OK(cudaStreamSynchronize(s));
    double pm;
    std::memcpy(&pm, &hb[0], sizeof(pm));
    *phi_max = pm;
    *bad = (hb[1] & 0xffffffffull) != 0;
}

}  // namespace sphray_b200

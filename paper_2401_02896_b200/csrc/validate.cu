// validate.cu -- the reference's `validate` groups (sphray_main.cpp:260-417,
// SURVEY.md 8(f1)) as GPU kernels over the device-resident scene:
//   group 2, exact superposition: every FieldPiece the render kernel's merge
//     produced is recomputed from the ray's knots by the explicit double sum
//     a_kd = sum_{t_i <= t_k} sum_{j >= d} C(j,d) b_ij (t_k - t_i)^(j-d)
//     in 128-bit integers (oracle::replay_ray, oracle.hpp:284-317, with
//     __int128 for BigInt) -- a method independent of the windowed merge;
//   group 3, dense-L2 envelope: the piecewise field against the exact SPH sum
//     (oracle::field_at, oracle.hpp:234-246) at the Simpson nodes of each
//     tested ray.
// Group 1 (telescoping) needs only the pieces and runs on the host.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_math.cuh"
#include "host.hpp"
#include "render.cuh"

namespace sphray_b200 {
namespace {

__global__ void k_inverse_perm(const int32_t* orig, size_t n, int32_t* inv) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) inv[orig[i]] = static_cast<int32_t>(i);
}

// per-hit particle records (original layout) and pow(h, d+3) from the
// Morton-ordered scene
__global__ void k_hit_records(const int64_t* pidx, size_t nh, const int32_t* inv,
                              const double4* pxyzh, const double4* mvr, const double* powh, int D,
                              sphray_particle* out, double* powh_out) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nh) return;
    const int32_t i = inv[pidx[k]];
    const double4 a = pxyzh[i], b = mvr[i];
    out[k] = sphray_particle{a.x, a.y, a.z, b.x, b.z, a.w, b.y};
    for (int d = 0; d < D; ++d) powh_out[k * D + d] = powh[static_cast<size_t>(i) * D + d];
}

__device__ __forceinline__ __int128 binom128(int n, int k) {
    __int128 r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

// Thread per piece: the explicit double sum over the ray's knots with t <= t_k.
// knot_off / piece_off: per-ray CSR (rays in the same order); knots sorted by t.
__global__ void k_replay(const uint64_t* knot_off, const int64_t* knot_t, const int64_t* knot_b,
                         const uint64_t* piece_off, const int64_t* piece_t, const int64_t* piece_a,
                         const uint32_t* piece_ray, size_t npieces, int D, unsigned int* ray_bad) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= npieces) return;
    const uint32_t r = piece_ray[k];
    const int64_t tk = piece_t[k];
    __int128 a[kMaxDegree + 1];
    for (int d = 0; d <= D; ++d) a[d] = 0;
    for (uint64_t i = knot_off[r]; i < knot_off[r + 1]; ++i) {
        const int64_t ti = knot_t[i];
        if (ti > tk) break;
        const __int128 dt = static_cast<__int128>(tk) - ti;
        for (int d = 0; d <= D; ++d) {
            __int128 pw = 1;
            for (int j = d; j <= D; ++j) {
                a[d] += binom128(j, d) * static_cast<__int128>(knot_b[i * (D + 1) + j]) * pw;
                pw *= dt;
            }
        }
    }
    bool ok = true;
    for (int d = 0; d <= D; ++d) ok &= a[d] == static_cast<__int128>(piece_a[k * (D + 1) + d]);
    if (!ok) atomicOr(&ray_bad[r], 1u);
}

// cubic B-spline, support radius 2 (oracle::cubic_w, oracle.hpp:29-35)
__device__ __forceinline__ double cubic_w(double r) {
    r = fabs(r);
    const double c = 1.0 / (4.0 * 3.14159265358979323846);
    if (r < 1.0) return c * (4.0 - 6.0 * r * r + 3.0 * r * r * r);
    if (r < 2.0) return c * (2.0 - r) * (2.0 - r) * (2.0 - r);
    return 0.0;
}

// Block per tested ray, thread per Simpson node: the piecewise approximation
// (evaluate_piece, raycast.hpp:295-301, on the last piece starting at or
// before t) and the exact superposed field at origin + dir t.
__global__ void k_l2_nodes(const CamConst cam, const uint32_t* ray_ids, const uint64_t* node_off,
                           const double* t0, const double* dtn, const uint64_t* piece_off,
                           const uint32_t* ray_piece_row, const int64_t* piece_t,
                           const int64_t* piece_a, int D, double tau, double sigma,
                           const double4* pxyzh, const double4* mvr, size_t n, double* approx,
                           double* exact) {
    const int r = blockIdx.x;
    const uint32_t id = ray_ids[r];
    const dev::RayD ray = dev::make_ray(cam, static_cast<int>(id % static_cast<uint32_t>(cam.W)),
                                   static_cast<int>(id / static_cast<uint32_t>(cam.W)));
    const uint64_t p0 = piece_off[ray_piece_row[r]], p1 = piece_off[ray_piece_row[r] + 1];
    const uint64_t nb = node_off[r], ne = node_off[r + 1];
    for (uint64_t q = nb + threadIdx.x; q < ne; q += blockDim.x) {
        const double t = t0[r] + static_cast<double>(q - nb) * dtn[r];
        uint64_t k = p0;
        while (k + 1 < p1 && static_cast<double>(piece_t[k + 1]) * tau <= t) ++k;
        const double x = t / tau - static_cast<double>(piece_t[k]);
        double acc = 0.0;
        for (int d = D; d >= 0; --d) acc = acc * x + static_cast<double>(piece_a[k * (D + 1) + d]);
        approx[q] = acc * sigma;
        const double px = ray.ox + ray.dx * t, py = ray.oy + ray.dy * t, pz = ray.oz + ray.dz * t;
        double f = 0.0;
        for (size_t i = 0; i < n; ++i) {
            const double4 a = pxyzh[i];
            const double dx = px - a.x, dy = py - a.y, dz = pz - a.z;
            const double rr = sqrt(dx * dx + dy * dy + dz * dz) / a.w;
            if (rr < 2.0) {
                const double4 b = mvr[i];
                f += b.x * b.y / (b.z * a.w * a.w * a.w) * cubic_w(rr);
            }
        }
        exact[q] = f;
    }
}

unsigned grid_of(size_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

#define SPHRAY_V_OK(x)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

void launch_hit_records(const int32_t* orig, size_t n, int32_t* inv, const int64_t* pidx, size_t nh,
                        const double4* pxyzh, const double4* mvr, const double* powh, int D,
                        sphray_particle* out, double* powh_out, cudaStream_t s) {
    k_inverse_perm<<<grid_of(n, 256), 256, 0, s>>>(orig, n, inv);
    SPHRAY_V_OK(cudaGetLastError());
    if (nh == 0) return;
    k_hit_records<<<grid_of(nh, 256), 256, 0, s>>>(pidx, nh, inv, pxyzh, mvr, powh, D, out, powh_out);
    SPHRAY_V_OK(cudaGetLastError());
}

void launch_replay(const uint64_t* knot_off, const int64_t* knot_t, const int64_t* knot_b,
                   const uint64_t* piece_off, const int64_t* piece_t, const int64_t* piece_a,
                   const uint32_t* piece_ray, size_t npieces, int D, unsigned int* ray_bad,
                   cudaStream_t s) {
    if (npieces == 0) return;
    k_replay<<<grid_of(npieces, 128), 128, 0, s>>>(knot_off, knot_t, knot_b, piece_off, piece_t,
                                                    piece_a, piece_ray, npieces, D, ray_bad);
    SPHRAY_V_OK(cudaGetLastError());
}

void launch_l2_nodes(const CamConst& cam, const uint32_t* ray_ids, int nrays, const uint64_t* node_off,
                     const double* t0, const double* dtn, const uint64_t* piece_off,
                     const uint32_t* ray_piece_row, const int64_t* piece_t, const int64_t* piece_a,
                     int D, double tau, double sigma, const double4* pxyzh, const double4* mvr,
                     size_t n, double* approx, double* exact, cudaStream_t s) {
    if (nrays == 0) return;
    k_l2_nodes<<<nrays, 256, 0, s>>>(cam, ray_ids, node_off, t0, dtn, piece_off, ray_piece_row,
                                     piece_t, piece_a, D, tau, sigma, pxyzh, mvr, n, approx, exact);
    SPHRAY_V_OK(cudaGetLastError());
}

}  // namespace sphray_b200

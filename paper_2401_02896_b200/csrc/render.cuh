// render.cuh -- device-side parameter blocks and launchers shared by the
// kernels (render.cu) and the engine (engine.cpp).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "host.hpp"

namespace sphray_b200 {

#ifndef SPHRAY_TILE_SHIFT
#define SPHRAY_TILE_SHIFT 3
#endif
constexpr int kTileShift = SPHRAY_TILE_SHIFT;  // 8x8-pixel screen tiles (2: 4x4)
constexpr int kTile = 1 << kTileShift;
constexpr int kTileRays = kTile * kTile;
constexpr int kHitQueue = 64;
// one extra slot per hit-queue array: the store target of lanes without a
// hit, so the gather's queue stores need no branch (0.45% per frame)
constexpr int kHqSlots = kHitQueue + 1;
constexpr int kTfPoint = 10;  // doubles per transfer-function point on the device
constexpr int kMaxJ = kMaxM * kMaxDegree;

// SPHRAY_STAGE=1: each warp prefetches its next 32 candidate records into
// shared memory with cp.async.bulk (TMA bulk copy) completing on an mbarrier,
// one gather step ahead of the hit tests.
#ifndef SPHRAY_STAGE
#define SPHRAY_STAGE 0
#endif
// SPHRAY_HQ_FRONT=1: the hit queue also keeps each hit's depth-sort front
// (the flush bound of the first queued hit is then a shared-memory read, not
// a dependent global load).
#ifndef SPHRAY_HQ_FRONT
#define SPHRAY_HQ_FRONT 1
#endif

#ifdef __CUDACC__
#define SPHRAY_HD __host__ __device__
#else
#define SPHRAY_HD
#endif

// Shared-memory bytes of one warp's knot window (layout: render_kernel.cuh carve()).
SPHRAY_HD inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// jb: bytes per jump (8; 16 for int_width 128)
SPHRAY_HD inline size_t warp_bytes_for(int D, int cap, int jb = 8) {
    size_t b = 0;
    b += align16(static_cast<size_t>(jb) * D * cap);  // pool: jumps of orders 1..D
    b += align16((jb == 16 ? 8 : 4) * static_cast<size_t>(cap));  // pt: position offsets
    b += align16(static_cast<size_t>(jb) * (D + 2));  // open piece
    b += align16(sizeof(double) * kHqSlots * 2);      // hit queue: d2, t_chi
    b += align16(sizeof(int32_t) * kHqSlots);         // hit queue: particle
#if SPHRAY_HQ_FRONT
    b += align16(sizeof(float) * kHqSlots);           // hit queue: front
#endif
    b += align16(sizeof(uint16_t) * cap * 2);         // ps, fl (+ flush set)
    b += align16(sizeof(uint32_t) * 256);             // radix bins
#if SPHRAY_STAGE
    b += 32 * 16 + 32 * 32 + 16;                      // staged candidate records + mbarrier
#endif
    return b;
}

// LUT + quanta view used by quantization (lut.hpp:25-52, quantize.hpp:44-51).
struct QuantParams {
    const double* lut_rows;  // N * (m + nj)
    int lut_stride, lut_N;
    double lut_dl, q;
    int K, m;
    double tau, sigma;
    double inv_tau, inv_dl;  // recip_or_nan(tau), recip_or_nan(lut_dl): division fast paths
    int w32;                 // int_width 32: every checked value must fit int32 (robust variant)
};

// Per-frame constants of the render kernel.
struct FrameParams {
    CamConst cam;
    QuantParams Q;
    // scene (Morton-ordered SoA)
    int n;
    const double4* pxyzh;  // x, y, z, h
    const double* xy;      // n * 3D: X_1..X_D, Y_1..Y_D (quantize.hpp:221-222), 1/Y_1..1/Y_D
    const int4* bbox;      // reference footprint bbox per particle (clipped)
    const float* front;    // knot-position lower bound (world units, rounded down)
    const int32_t* orig;   // original particle index
    // binning: the candidate records of every owned tile, in front order
    const double4* cxyzh;        // x, y, z, h of the candidate
    const uint4* cmeta;          // front (float bits), particle index, tile-local bbox (4 x 4 bits), 0
    const uint32_t* tile_begin;  // per owned tile
    const uint32_t* tile_end;
    int tiles_x, tiles_y;
    int rank, nranks;
    double inv_tau;   // 1 / tau for sample abscissae (compositing only)
    double inv_step;  // 1 / step (sample counts, checked against the exact quotient)
    // transfer function (raycast.hpp:313-338)
    const double* tf;  // ntf * kTfPoint: value, r, g, b, absorption, 4 slopes to the next point, pad
    int ntf;
    int tf0_clear;  // tf.sample(0).absorption == 0: zero pieces are exact no-ops
    double step;
    double bg[3];
    int mode;
    // knot window
    int cap;         // knot slots per warp
    int warp_bytes;  // dynamic smem per warp
    int tf_smem;     // bytes of the per-CTA shared copy of tf after the windows (0: read global)
    int robust;      // robust variant for this launch: 1 = rebasing window offsets, 2 = + int32 range tests
    int w128;        // int_width 128: the robust variant with a modulo-2^128 merge
    // work distribution
    unsigned long long* work_counter;
    uint64_t total_work;
    const uint32_t* ray_list;  // retry pass: explicit ray ids (else tile-major)
    int tile_row0, tile_col0;  // first tile row / column of the frame's work (pixel region)
    int tiles_wx;              // tile columns of the work
    int row_lo, row_hi;        // pixels rendered: py in [row_lo, row_hi),
    int col_lo, col_hi;        //                  px in [col_lo, col_hi)
    uint32_t* retry_list;
    unsigned int* retry_count;
    // output
    double* rgb;  // full image (packed == 0) or owned tiles, tile-major
    int packed;
    unsigned long long* stats;  // StatIndex
    sphray_ray_record* ray_rec;  // optional per-ray records, index (py - row_lo) * W + px
    // validation dumps (optional)
    unsigned long long* dump_count;  // [0] hits [1] pieces
    uint64_t dump_cap_hits, dump_cap_pieces;
    uint64_t* dump_hit_ray;
    int64_t* dump_hit_pidx;
    double* dump_hit_lam;
    double* dump_hit_tchi;
    uint64_t* dump_piece_ray;
    int64_t* dump_piece_t;
    int64_t* dump_piece_a;  // (D+1) per piece
};

enum StatIndex {
    kStatKnots = 0,
    kStatRays = 1,
    kStatIntOps = 2,
    kStatResidual = 3,
    kStatHits = 4,
    kStatMaxPending = 5,
    kStatOverflowKey = 6,
    kStatSkipped = 7,
    kStatTerminated = 29,  // rays that reached T <= 1e-3 (early ray termination)
    kStatAccumOverflowRay = 30,  // smallest ray whose merged coefficients left int64 (min; ~0: none)
    // work counters, filled only in -DSPHRAY_KSTATS=1 builds (diagnostics)
    kStatFlushes = 8,
    kStatScanned = 9,   // pending entries examined by flush selection
    kStatSelected = 10,  // knots finalised
    kStatChunks = 11,    // 32-knot merge chunks
    kStatRadixPasses = 12,
    kStatBatches = 13,   // insert_hits calls
    kStatSamples = 14,   // composited samples (lane path + balanced path)
    kStatBalanced = 15,  // chunks sent to the sample-parallel path
    kStatGather = 16,    // 32-candidate gather iterations
    kStatPeak0 = 17,     // rays by largest post-flush residual: <128, <192, <256, <320, <384, >=384
    kStatBits0 = 23,     // flushes by sort-key bits: <=8, <=10, <=12, <=14, <=16, >16
    kStatCount = 31
};
constexpr int kStatFirstK = kStatFlushes;

// Per-frame particle prep (view + quanta dependent).
struct PrepParams {
    CamConst cam;
    int n, D;
    double q, reach_scale;  // knot reach = h * reach_scale (largest LUT knot radius)
    const double4* pxyzh;
    const double4* mvr;    // mass, value, density
    const double* powh;    // n*D: pow(h, d+3)
    const double* powtau;  // D: pow(tau, d)
    double sigma;
    int4* bbox;
    float* front;
    double* xy;
    uint32_t* counts;
    int tiles_x, rank, nranks;
};

size_t warp_smem_bytes(int D, int cap, int m, int jb = 8);
int max_blocks_per_sm(int D, int m, int warps, size_t smem, bool even_k);
// dataset_stats (quantize.hpp:129-165) of the resident scene: medians of
// mass, density, h, value (med[0..3]), phi_max, and whether some particle has
// h <= 0 or density <= 0.
// validate.cu
void launch_hit_records(const int32_t* orig, size_t n, int32_t* inv, const int64_t* pidx, size_t nh,
                        const double4* pxyzh, const double4* mvr, const double* powh, int D,
                        sphray_particle* out, double* powh_out, cudaStream_t s);
void launch_replay(const uint64_t* knot_off, const int64_t* knot_t, const int64_t* knot_b,
                   const uint64_t* piece_off, const int64_t* piece_t, const int64_t* piece_a,
                   const uint32_t* piece_ray, size_t npieces, int D, unsigned int* ray_bad,
                   cudaStream_t s);
void launch_l2_nodes(const CamConst& cam, const uint32_t* ray_ids, int nrays, const uint64_t* node_off,
                     const double* t0, const double* dtn, const uint64_t* piece_off,
                     const uint32_t* ray_piece_row, const int64_t* piece_t, const int64_t* piece_a,
                     int D, double tau, double sigma, const double4* pxyzh, const double4* mvr,
                     size_t n, double* approx, double* exact, cudaStream_t s);

void device_dataset_stats(const double4* pxyzh, const double4* mvr, size_t n, cudaStream_t s,
                          double med[4], double* phi_max, bool* bad);
void launch_render(const FrameParams& P, int D, int m, int blocks, int warps, cudaStream_t s);
void launch_prep(const PrepParams& p, cudaStream_t s);
// depth order of the particles: keys = orderable(front), vals = index
void launch_depth_keys(const float* front, int n, uint32_t* keys, uint32_t* vals, cudaStream_t s);
// counts in depth order; *total (device, zeroed by the caller) += their sum
void launch_gather_counts(const uint32_t* counts, const uint32_t* order, int n, uint32_t* out,
                          unsigned long long* total, cudaStream_t s);
// (tile, particle) entries, particles visited in depth order
void launch_emit(const PrepParams& p, const uint32_t* order, const uint32_t* offsets, uint32_t* keys,
                 uint32_t* vals, cudaStream_t s);
void launch_tile_ranges(const uint32_t* keys, size_t m, uint32_t* begin, uint32_t* end, cudaStream_t s);
// candidate records in sorted (tile, front) order: the particle's x, y, z, h and
// (front, index, its reference bbox clipped to the tile in tile-local pixels)
void launch_records(const uint32_t* tile_keys, const uint32_t* cand, size_t m, const double4* pxyzh,
                    const int4* bbox, const float* front, int tiles_x, int rank, int nranks,
                    double4* cxyzh, uint4* cmeta, cudaStream_t s);
void launch_reach(const CamConst& cam, int n, double q, const double4* pxyzh, const int4* bbox,
                  unsigned long long* skipped, cudaStream_t s);
void launch_unpack(const double* packed, size_t per_rank, int nranks, int tiles_x, int W, int H,
                   double* out, cudaStream_t s);
void launch_fill_bg(double* rgb, size_t npix, const double* bg, cudaStream_t s);
void launch_morton(const sphray_particle* ps, size_t n, const double* lo, const double* inv,
                   unsigned long long* codes, uint32_t* idx, cudaStream_t s);
void launch_scatter_scene(const sphray_particle* ps, const double* powh_in, const uint32_t* perm,
                          size_t n, int D, double4* pxyzh, double4* mvr, double* powh,
                          int32_t* orig, cudaStream_t s);
void launch_quantize_hits(const QuantParams& Q, int D, const sphray_particle* ps,
                          const double* powh, const double* powtau, size_t nhits,
                          const double* tchi, const double* lam, int64_t* knot_t,
                          int64_t* knot_b, int32_t* knot_count, cudaStream_t s);

// accumulate.cu: accumulate<int64_t> for explicit knot streams (7 jumps per knot)
void accumulate_knots(int D, size_t nrays, const uint64_t* ray_ids, const uint64_t* koff, const int64_t* kt,
                      const int64_t* kb, uint64_t* piece_off, int64_t* piece_t, int64_t* piece_a, uint64_t* ops,
                      cudaStream_t s);
// sort.cu: hand-written scan and stable LSD radix sort
size_t scan_tmp_bytes(size_t n);
void scan_u32(const uint32_t* in, uint32_t* out, size_t n, void* tmp, uint32_t* total_dev, cudaStream_t s);
size_t radix_tmp_bytes(size_t n);
int radix_passes(int end_bit);
bool sort_pairs_u64(unsigned long long* kin, unsigned long long* kout, uint32_t* vin, uint32_t* vout,
                    size_t n, int end_bit, void* tmp, cudaStream_t s);
bool sort_pairs_u32(uint32_t* kin, uint32_t* kout, uint32_t* vin, uint32_t* vout, size_t n, int end_bit,
                    void* tmp, cudaStream_t s);

}  // namespace sphray_b200

/*
 * sphray_gpu.h -- C-ABI of the B200-native per-ray higher-order SPH field
 * approximation + compositing path (arXiv 2401.02896).
 *
 * Drop-in boundary for the reference's header-only renderer
 * (/root/reference/proj/include/sphray).  The reference has no FFI; its
 * interface is the C++ template `sphray::render_scene<Int>` and the sweep
 * functions it is built from.  Each entry point below names the reference
 * interface it replaces.  Plain POD structs, pointers and sizes only; no torch
 * or CUDA types cross this boundary.  All pointers are HOST pointers unless a
 * name says `device`.
 *
 * Errors mirror the reference's exception classes (errors.hpp:12-69) as
 * status codes; the C++ shim in sphray_gpu.hpp rethrows them as the matching
 * sphray:: exception.
 */
#ifndef SPHRAY_GPU_H
#define SPHRAY_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPHRAY_GPU_ABI_VERSION 2

/* errors.hpp:12-69 -> status codes.  CLI exit codes (sphray_main.cpp:442-462)
 * map CONFIG/IO -> 2, OVERFLOW -> 3, NUMERIC -> 4. */
typedef enum sphray_status {
    SPHRAY_OK = 0,
    SPHRAY_ERR_CONFIG = 1,   /* sphray::ConfigError   errors.hpp:18-21 */
    SPHRAY_ERR_IO = 2,       /* sphray::IoError       errors.hpp:24-27 */
    SPHRAY_ERR_OVERFLOW = 3, /* sphray::OverflowError errors.hpp:54-63 */
    SPHRAY_ERR_NUMERIC = 4,  /* sphray::NumericError  errors.hpp:66-69 */
    SPHRAY_ERR_CUDA = 5,     /* device failure / no CUDA device */
    SPHRAY_ERR_NCCL = 6,     /* tile gather failure */
    SPHRAY_ERR_CAPACITY = 7  /* a ray's knot window exceeded every window size */
} sphray_status;

/* == sphray::Particle (quantize.hpp:16-27) and one SPRT record (io.hpp:111-141). */
typedef struct sphray_particle {
    double x, y, z, mass, density, h, value;
} sphray_particle;

/* sphray::Camera (raycast.hpp:45-58). mode: 0 orthographic, 1 pinhole. */
typedef struct sphray_camera {
    int32_t mode;
    int32_t width;
    int32_t height;
    int32_t reserved;
    double position[3];
    double look_at[3];
    double up[3];
    double fov_deg;      /* vertical, pinhole only */
    double ortho_height; /* orthographic only */
    double near_plane;
    double far_plane;
} sphray_camera;

/* sphray::TfPoint (raycast.hpp:303-309). */
typedef struct sphray_tf_point {
    double value, r, g, b, absorption;
} sphray_tf_point;

/* sphray::Lut (lut.hpp:32-65) as a view of the .splt payload: `records` holds N
 * records of (lambda, error, ceil(K/2) knots, floor(K*D/2) jumps) doubles in
 * file order (lut.hpp:292-297), i.e. exactly the bytes after the .splt header. */
typedef struct sphray_lut_view {
    double q;
    int32_t K;
    int32_t D;
    int32_t N;
    int32_t reserved;
    const double* records;
} sphray_lut_view;

/* sphray::QuantaConfig (quantize.hpp:44-51). int_width: 32, 64 or 128 -- the
 * device arithmetic, as render_scene<Int> with Int of that width:
 * 32: every Checked value and merged coefficient must fit int32;
 * 64: int64 (the production kernel);
 * 128: 128-bit jumps and a modulo-2^128 merge (knot positions must fit int64,
 *      else SPHRAY_ERR_CAPACITY; validation outputs are int64 only).
 * A genuine overflow of the width raises SPHRAY_ERR_OVERFLOW naming the ray. */
typedef struct sphray_quanta {
    double tau;
    double sigma;
    int32_t int_width;
    int32_t reserved;
} sphray_quanta;

/* sphray::DatasetStats (quantize.hpp:31-40). */
typedef struct sphray_dataset_stats {
    double mass_r, density_r, h_r, value_r, phi_repr, a_max, clustering_factor;
    uint64_t count;
} sphray_dataset_stats;

/* Render modes. EXACT reproduces every sphray::RenderStats counter
 * (raycast.hpp:400-408): rays keep merging after they saturate.  FAST stops a
 * ray at early termination (image identical; knots/int_ops/residual counters
 * then cover only the traversed part). */
#define SPHRAY_MODE_EXACT 0
#define SPHRAY_MODE_FAST 1

/* sphray::RenderOptions (raycast.hpp:394-398) plus device-side knobs.
 * `threads` is accepted and ignored (the GPU grid replaces parallel_for). */
typedef struct sphray_render_options {
    double step;          /* <= 0 picks h_r / 8 (raycast.hpp:424) */
    double background[3];
    int32_t threads;
    int32_t mode;         /* SPHRAY_MODE_* */
    int32_t window;       /* knot window per ray (slots); 0 = auto */
    int32_t reserved;
} sphray_render_options;

/* sphray::RenderStats (raycast.hpp:400-408) + path counters. */
typedef struct sphray_render_stats {
    uint64_t particles;
    uint64_t skipped_particles;
    uint64_t knots;
    uint64_t rays_touched;
    uint64_t int_ops;
    uint64_t residual_failures;
    double step;
    uint64_t hits;            /* (ray, particle) pairs passing hit_ray */
    uint64_t candidates;      /* binned (tile, particle) entries */
    uint64_t window_retries;  /* rays re-run with a wider knot window */
    uint64_t max_window;      /* largest pending-knot count seen */
    double device_ms;         /* device time of the whole frame (CUDA events) */
    double bin_ms;            /* particle prep + tile binning (sort) */
    double render_ms;         /* the render kernel(s): gather, quantize, merge, composite */
    uint64_t launches;        /* kernels launched for the frame */
    uint64_t terminated_rays; /* rays whose transmittance reached <= 1e-3 (early termination) */
} sphray_render_stats;

/* Per-ray record of a frame rendered with records enabled
 * (sphray_context_set_rows): the RenderStats counters of one ray
 * (raycast.hpp:400-408, 471-493) and an order-independent checksum of its
 * merged FieldPieces (raycast.hpp:198-202, accumulate 261-292): the wrapping
 * uint64 sum over the ray's pieces of sphray_piece_mix(t, a, D).  In MODE_FAST
 * the counters of an early-terminated ray cover only the traversed part. */
typedef struct sphray_ray_record {
    uint64_t piece_checksum;
    uint32_t knots;   /* knots emitted on the ray (after the coincident merge) */
    uint32_t pieces;  /* distinct knot positions = FieldPieces */
    uint32_t hits;    /* (ray, particle) pairs passing hit_ray */
    uint32_t flags;   /* SPHRAY_RAY_* */
} sphray_ray_record;
#define SPHRAY_RAY_TOUCHED 1u     /* at least one knot */
#define SPHRAY_RAY_RESIDUAL 2u    /* trailing piece nonzero (residual_failures) */
#define SPHRAY_RAY_TERMINATED 4u  /* transmittance reached <= 1e-3 */

/* The piece hash of sphray_ray_record.piece_checksum: piece position t and
 * coefficients a_0..a_D. */
static inline uint64_t sphray_piece_mix(int64_t t, const int64_t* a, int D) {
    static const uint64_t M[8] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full,
                                  0x165667B19E3779F9ull, 0x27D4EB2F165667C5ull,
                                  0x94D049BB133111EBull, 0xBF58476D1CE4E5B9ull,
                                  0xD6E8FEB86659FD93ull, 0xFF51AFD7ED558CCDull};
    uint64_t x = (uint64_t)t * M[0];
    for (int d = 0; d <= D; ++d) x += (uint64_t)a[d] * M[d + 1];
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    return x;
}

/* OverflowError carries particle index and ray id (errors.hpp:54-63). */
typedef struct sphray_error {
    int32_t code;
    int32_t reserved;
    int64_t particle_index;
    uint64_t ray_id;
    char msg[256];
} sphray_error;

typedef struct sphray_context sphray_context;

/* Library/ABI identification. */
int sphray_abi_version(void);
const char* sphray_build_info(void);

/* One context per CUDA device; owns device memory, streams and the scene
 * cache.  Not re-entrant: one host thread per context. */
sphray_status sphray_context_create(int device, sphray_context** out, sphray_error* err);
void sphray_context_destroy(sphray_context* ctx);

/* Diagnostics (no reference counterpart): measured ALU issue peaks of a
 * device -- int64 multiply/add operations per second and fp64 flops per
 * second, in units of 1e9 -- the denominators of the benchmark's ALU
 * roofline for the merge. */
sphray_status sphray_probe_alu_peaks(int device, double* int64_gops, double* fp64_gflops,
                                     sphray_error* err);

/* Multi-GPU (one process per GPU): `unique_id` is 128 bytes produced by
 * sphray_comm_unique_id on rank 0 and broadcast by the caller.  Image tiles are
 * interleaved over ranks; finished tiles are gathered with NCCL over NVLink. */
sphray_status sphray_comm_unique_id(uint8_t unique_id[128], sphray_error* err);
sphray_status sphray_context_init_comm(sphray_context* ctx, int rank, int nranks,
                                       const uint8_t unique_id[128], sphray_error* err);

/* The same tile partition without a communicator: sphray_scene_render then
 * renders only this rank's tiles and returns them PACKED in rgb_out
 * (ceil(ntiles / nranks) tiles of 8x8 pixels, tile-major, RGB doubles; tile t
 * belongs to rank t % nranks).  Used to drive ranks from a host-side
 * collective and to test the sharded path on one device. */
sphray_status sphray_context_set_shard(sphray_context* ctx, int rank, int nranks,
                                       sphray_error* err);

/* Pixel region (no reference counterpart; used to check the benchmarked frame
 * against the reference's own sweep functions): subsequent renders of `ctx`
 * (sphray_scene_render, sphray_scene_hits, sphray_scene_pieces) trace only
 * the pixels px in [x0, x0 + w), py in [y0, y0 + h) of the camera -- the same
 * rays, bit for bit, as the full frame -- and sphray_scene_render writes
 * h * W * 3 doubles (rows y0 .. y0 + h - 1; pixels outside the region keep the
 * background).  w == 0 or h == 0 restores full frames.  record_rays != 0
 * makes every render also keep one sphray_ray_record per pixel of the region
 * (or frame), row-major over the region, fetched with sphray_context_ray_records.
 * Single-rank contexts only. */
sphray_status sphray_context_set_region(sphray_context* ctx, int32_t x0, int32_t y0, int32_t w,
                                        int32_t h, int32_t record_rays, sphray_error* err);
sphray_status sphray_context_ray_records(sphray_context* ctx, sphray_ray_record* out, size_t cap,
                                         size_t* count, sphray_error* err);

/* -------------------------------------------------------------------------
 * Drop-in for  template<class Int> Image render_scene(particles, cam, tf, lut,
 * qc, stats, opts, RenderStats*)   raycast.hpp:414-497.
 * Integer width comes from qc->int_width (dispatch_int_width, int_ops.hpp:113).
 * rgb_out: W*H*3 doubles, row-major, top row first (raycast.hpp:383-392).
 * ---------------------------------------------------------------------- */
sphray_status sphray_render_scene(sphray_context* ctx, const sphray_particle* particles,
                                  size_t n, const sphray_camera* cam,
                                  const sphray_tf_point* tf, size_t ntf,
                                  const sphray_lut_view* lut, const sphray_quanta* qc,
                                  const sphray_dataset_stats* stats,
                                  const sphray_render_options* opts, double* rgb_out,
                                  sphray_render_stats* out_stats, sphray_error* err);

/* Persistent form of the same call: the particle set and LUT are uploaded once
 * and stay resident in HBM; frames then only upload camera/TF/quanta.
 * sphray_scene_render with rgb_out == NULL leaves the image on the device
 * (sphray_scene_device_image returns it). */
sphray_status sphray_scene_upload(sphray_context* ctx, const sphray_particle* particles,
                                  size_t n, const sphray_lut_view* lut, sphray_error* err);
sphray_status sphray_scene_render(sphray_context* ctx, const sphray_camera* cam,
                                  const sphray_tf_point* tf, size_t ntf,
                                  const sphray_quanta* qc, const sphray_dataset_stats* stats,
                                  const sphray_render_options* opts, double* rgb_out,
                                  sphray_render_stats* out_stats, sphray_error* err);
const double* sphray_scene_device_image(sphray_context* ctx);
/* The resident scene: particle count and the LUT's K and D (piece_a of
 * sphray_scene_pieces holds D + 1 coefficients per piece).  ConfigError when
 * no scene is uploaded. */
sphray_status sphray_scene_info(sphray_context* ctx, size_t* n, int32_t* K, int32_t* D,
                                sphray_error* err);

/* The context's CUDA stream (cudaStream_t), for callers that time or order
 * work around the library's launches. */
void* sphray_context_stream(sphray_context* ctx);

/* -------------------------------------------------------------------------
 * Validation outputs (the reference's cmd_validate harness, sphray_main.cpp:
 * 260-417, and the sweep functions it drives).  Run on the resident scene.
 * ---------------------------------------------------------------------- */

/* particle_ray_footprint (raycast.hpp:128-184) for every particle, as a
 * ray-major list of hits.  Two-call protocol: pass cap = 0 to get the count. */
sphray_status sphray_scene_hits(sphray_context* ctx, const sphray_camera* cam,
                                uint64_t* ray_id, int64_t* particle_index, double* lam,
                                double* t_chi, size_t cap, size_t* count, sphray_error* err);

/* quantize_particle + sort_knots + accumulate (raycast.hpp:188-292) per ray:
 * the merged FieldPieces as CSR over touched rays.  piece_a holds D+1 int64
 * coefficients per piece.  Two-call protocol on (cap_rays, cap_pieces). */
sphray_status sphray_scene_pieces(sphray_context* ctx, const sphray_camera* cam,
                                  const sphray_quanta* qc, uint64_t* rays,
                                  uint64_t* piece_offsets, int64_t* piece_t, int64_t* piece_a,
                                  size_t cap_rays, size_t cap_pieces, size_t* n_rays,
                                  size_t* n_pieces, sphray_error* err);

/* accumulate<int64_t> (raycast.hpp:261-292) for explicit knot streams, one
 * per ray, on the GPU (the render kernel's merge without the window): ray r's
 * knots are [knot_offsets[r], knot_offsets[r+1]) of knot_t / knot_b, sorted by
 * t, with 7 (max_degree + 1) jumps per knot in knot_b (QuantizedKnot::b).
 * Output: one FieldPiece per distinct position as CSR -- piece_offsets
 * (nrays + 1), piece_t, piece_a (D + 1 per piece); capacity = total knots
 * suffices -- and per-ray RayAccumulator op counts (optional).  NumericError
 * for unsorted knots (raycast.hpp:212-213); OverflowError naming the ray for a
 * genuine int64 overflow of a coefficient (raycast.hpp:285-289); the
 * reference's spurious Delta t^D overflow is not reproduced. */
sphray_status sphray_accumulate(sphray_context* ctx, int D, size_t nrays, const uint64_t* ray_ids,
                                const uint64_t* knot_offsets, const int64_t* knot_t,
                                const int64_t* knot_b, uint64_t* piece_offsets, int64_t* piece_t,
                                int64_t* piece_a, uint64_t* ops, sphray_error* err);

/* quantize_particle<Int> (quantize.hpp:199-250) for explicit hits: knots of
 * hit i are written at [i*(K+1), i*(K+1)+count_i) with D+1 jumps each. */
sphray_status sphray_quantize_hits(sphray_context* ctx, const sphray_particle* particles,
                                   size_t nhits, const double* t_chi, const double* lam,
                                   const sphray_lut_view* lut, const sphray_quanta* qc,
                                   int64_t* knot_t, int64_t* knot_b, int32_t* knot_count,
                                   sphray_error* err);

/* -------------------------------------------------------------------------
 * Host-side inputs of the path (quantize.hpp:97-183), restated natively so a
 * caller needs nothing from the reference to drive the renderer.
 * ---------------------------------------------------------------------- */
sphray_status sphray_compute_dataset_stats(const sphray_particle* particles, size_t n,
                                           const sphray_lut_view* lut, double clustering_factor,
                                           sphray_dataset_stats* out, sphray_error* err);
/* The reference's `validate` checks (sphray_main.cpp:260-417) on the GPU for
 * the resident scene and one camera (the reference clamps it to 32 x 32):
 *   telescoping  -- every touched ray's trailing piece is zero;
 *   superposition -- every FieldPiece of the render kernel equals the explicit
 *                   128-bit double sum over the ray's knots (oracle replay);
 *   dense-L2     -- on the first 64 rays, the L2 distance between the
 *                   piecewise field and the exact SPH sum (composite Simpson,
 *                   n = max(64, len / (h_min / 64)) panels) relative to the
 *                   exact field's L2 norm stays within 4 hypot(E*, Q) on at
 *                   least 95% of the rays. */
typedef struct sphray_validate_report {
    uint64_t telescoping_rays, telescoping_bad;
    uint64_t superposition_rays, superposition_bad;
    uint64_t l2_rays, l2_bad;
    double l2_envelope;
    double l2_fraction_within;
    int32_t telescoping_pass, superposition_pass, l2_pass, pass;
} sphray_validate_report;
sphray_status sphray_scene_validate(sphray_context* ctx, const sphray_camera* cam,
                                    const sphray_quanta* qc, const sphray_dataset_stats* ds,
                                    sphray_validate_report* out, sphray_error* err);

/* -------------------------------------------------------------------------
 * File formats (io.hpp:62-216): SPRT binary / CSV particles (format sniffed
 * by magic), transfer-function CSV, binary PPM.  Loaders allocate with
 * malloc; release with sphray_free.  Errors: SPHRAY_ERR_IO (ConfigError for an
 * invalid transfer function, as the reference).
 * ---------------------------------------------------------------------- */
sphray_status sphray_particles_load(const char* path, sphray_particle** out, size_t* n,
                                    sphray_error* err);
sphray_status sphray_particles_save(const char* path, const sphray_particle* particles, size_t n,
                                    int binary, sphray_error* err);
sphray_status sphray_tf_load(const char* path, sphray_tf_point** out, size_t* n, sphray_error* err);
sphray_status sphray_ppm_save(const char* path, const double* rgb, int width, int height,
                              sphray_error* err);
/* load_camera (io.hpp:263-304): camera JSON with the reference's defaults,
 * validated like Camera::validate (ConfigError) */
sphray_status sphray_camera_load(const char* path, sphray_camera* out, sphray_error* err);
void sphray_free(void* p);
/* Loads a particle file and uploads it as the scene of `ctx`
 * (sphray_scene_upload semantics). */
sphray_status sphray_scene_upload_file(sphray_context* ctx, const char* path,
                                       const sphray_lut_view* lut, sphray_error* err);

/* dataset_stats (quantize.hpp:129-165) of the scene resident in `ctx`
 * (sphray_scene_upload), on the GPU: radix-sorted medians and a max
 * reduction -- bit-identical to sphray_compute_dataset_stats. */
sphray_status sphray_scene_dataset_stats(sphray_context* ctx, double clustering_factor,
                                         sphray_dataset_stats* out, sphray_error* err);
sphray_status sphray_choose_quanta(const sphray_lut_view* lut, const sphray_dataset_stats* ds,
                                   int int_width, double kappa, double kappa_prime,
                                   sphray_quanta* out, sphray_error* err);

/* serialize_lut / save_lut (lut.hpp:335-352, 395-399): the .splt file image of
 * a LUT view (kernel_id: up to 16 bytes, e.g. "cubic-bspline").  Two-call
 * protocol on cap for sphray_lut_serialize. */
sphray_status sphray_lut_serialize(const sphray_lut_view* lut, const char* kernel_id, uint8_t* out,
                                   size_t cap, size_t* nbytes, sphray_error* err);
sphray_status sphray_lut_save(const char* path, const sphray_lut_view* lut, const char* kernel_id,
                              sphray_error* err);

/* The reference CLI's render report (sphray_main.cpp:196-256), written next to
 * the image as "<out>.json": quanta, RenderStats, dataset statistics, errors
 * {E_star (overall_error, lut.hpp:284-290), Q_D (quantization_error,
 * quantize.hpp:64-73), combined}, overflow_count, K, D, kernel, seed, image --
 * the same JSON text (2-space indent).  stats == NULL or stats->particles == 0
 * gives the reference's empty-scene report.  kappa/kappa_prime <= 0 select the
 * cubic B-spline's constants.  Two-call protocol on cap (len excludes the NUL). */
sphray_status sphray_render_report(const sphray_lut_view* lut, const char* kernel_id,
                                   const sphray_dataset_stats* ds, const sphray_quanta* qc,
                                   const sphray_render_stats* stats, uint64_t seed,
                                   const char* image_path, double kappa, double kappa_prime,
                                   char* out, size_t cap, size_t* len, sphray_error* err);

/* .splt parsing (lut.hpp:354-393): validates the file image and copies the
 * header fields into *view.  view->records points into `bytes` (offset 44) when
 * that address is 8-byte aligned, else it is NULL and the caller supplies an
 * aligned copy of bytes[44:]. */
sphray_status sphray_lut_parse(const uint8_t* bytes, size_t nbytes, sphray_lut_view* view,
                               char kernel_id[17], sphray_error* err);

/* Synthetic scenes of BASELINE.json configs: 1 = blob 1e5,
 * 2 = blob 1M, 3 = clustered 16M, 4 = blob 4M, 5 = clustered 100M.  `n` may
 * override the particle count (0 = config default). Writes n records. */
sphray_status sphray_generate_scene(int config, size_t n, uint64_t seed,
                                    sphray_particle* out, sphray_error* err);
size_t sphray_scene_default_count(int config);

#ifdef __cplusplus
}
#endif

#endif /* SPHRAY_GPU_H */

// sphray_gpu.hpp -- header-only C++ drop-in over the C-ABI (sphray_gpu.h).
//
// Include AFTER the reference renderer's headers (<sphray/raycast.hpp>): this
// shim re-exposes the reference entry points with the reference's own types
// and exceptions, running the sm_100a path:
//
//   sphray::render_scene<Int>(particles, cam, tf, lut, qc, stats, opts, &rs)
//     -> sphray::gpu::render_scene<Int>(... same arguments ...)
//
// (raycast.hpp:414-497).  Errors come back as the matching sphray:: exception
// (errors.hpp:12-69); OverflowError keeps particle_index and ray_id.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <type_traits>
#include <vector>

#include "sphray_gpu.h"

namespace sphray::gpu {

[[noreturn]] inline void rethrow(sphray_status st, const sphray_error& e) {
    const std::string msg = e.msg;
    switch (st) {
        case SPHRAY_ERR_CONFIG: throw ConfigError(msg);
        case SPHRAY_ERR_IO: throw IoError(msg);
        case SPHRAY_ERR_OVERFLOW: throw OverflowError(msg, e.particle_index, e.ray_id);
        case SPHRAY_ERR_NUMERIC: throw NumericError(msg);
        default: throw Error("sphray_gpu: " + msg);
    }
}

inline void check(sphray_status st, const sphray_error& e) {
    if (st != SPHRAY_OK) rethrow(st, e);
}

// One CUDA device context (device memory, streams, resident scene).
class Device {
   public:
    explicit Device(int device = 0) {
        sphray_error e{};
        check(sphray_context_create(device, &ctx_, &e), e);
    }
    ~Device() { sphray_context_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    sphray_context* get() const { return ctx_; }

   private:
    sphray_context* ctx_ = nullptr;
};

inline Device& default_device() {
    static Device d(0);
    return d;
}

inline sphray_camera to_c(const Camera& c) {
    sphray_camera o{};
    o.mode = c.mode == Camera::Mode::pinhole ? 1 : 0;
    o.width = c.width;
    o.height = c.height;
    o.position[0] = c.position.x, o.position[1] = c.position.y, o.position[2] = c.position.z;
    o.look_at[0] = c.look_at.x, o.look_at[1] = c.look_at.y, o.look_at[2] = c.look_at.z;
    o.up[0] = c.up.x, o.up[1] = c.up.y, o.up[2] = c.up.z;
    o.fov_deg = c.fov_deg;
    o.ortho_height = c.ortho_height;
    o.near_plane = c.near;
    o.far_plane = c.far;
    return o;
}

// Lut -> .splt record layout (lut.hpp:292-297).
struct LutRecords {
    std::vector<double> records;
    sphray_lut_view view{};
};

inline LutRecords to_c(const Lut& lut) {
    LutRecords r;
    for (const auto& e : lut.entries) {
        r.records.push_back(e.lambda);
        r.records.push_back(e.error);
        r.records.insert(r.records.end(), e.knots.begin(), e.knots.end());
        r.records.insert(r.records.end(), e.s_hat.begin(), e.s_hat.end());
    }
    r.view.q = lut.q;
    r.view.K = lut.K;
    r.view.D = lut.D;
    r.view.N = static_cast<int32_t>(lut.entries.size());
    r.view.records = r.records.data();
    return r;
}

inline sphray_dataset_stats to_c(const DatasetStats& s) {
    return {s.mass_r, s.density_r, s.h_r, s.value_r, s.phi_repr, s.a_max, s.clustering_factor,
            static_cast<uint64_t>(s.count)};
}

// The device arithmetic for render_scene<Int>: int32_t -> every Checked
// value must fit int32 (int_width 32); int64_t -> int64 (64); Int128 on
// quanta of at most 64 bits -> the exact modulo-2^64 merge, which equals the
// Int128 result whenever that fits int64 and raises OverflowError otherwise
// (64); Int128 on w128 quanta -> 128-bit jumps and a modulo-2^128 merge (128;
// knot positions must fit int64, else CapacityError).
template <class Int>
constexpr int device_int_width(int quanta_bits) {
    if constexpr (std::is_same_v<Int, std::int32_t>) return 32;
    else if constexpr (std::is_same_v<Int, std::int64_t>) return 64;
    else return quanta_bits <= 64 ? 64 : 128;
}

// render_scene<Int>, raycast.hpp:414-497, on the B200 path.
template <class Int>
Image render_scene(std::span<const Particle> particles, const Camera& cam,
                   const TransferFunction& tf, const Lut& lut, const QuantaConfig& qc,
                   const DatasetStats& stats, const RenderOptions& opts,
                   RenderStats* out_stats = nullptr, Device* device = nullptr) {
    static_assert(sizeof(Particle) == sizeof(sphray_particle), "Particle layout");
    Device& dev = device ? *device : default_device();
    const sphray_camera c = to_c(cam);
    std::vector<sphray_tf_point> pts;
    for (const auto& p : tf.points) pts.push_back({p.value, p.r, p.g, p.b, p.absorption});
    const LutRecords L = to_c(lut);
    const sphray_quanta q{qc.tau, qc.sigma, device_int_width<Int>(static_cast<int>(qc.width)), 0};
    const sphray_dataset_stats ds = to_c(stats);
    sphray_render_options o{};
    o.step = opts.step;
    o.background[0] = opts.background.r;
    o.background[1] = opts.background.g;
    o.background[2] = opts.background.b;
    o.threads = opts.threads;
    o.mode = SPHRAY_MODE_EXACT;
    Image img;
    img.width = cam.width;
    img.height = cam.height;
    img.pixels.resize(static_cast<size_t>(cam.width > 0 ? cam.width : 0) *
                      (cam.height > 0 ? cam.height : 0));
    sphray_render_stats rs{};
    sphray_error e{};
    check(sphray_render_scene(dev.get(), reinterpret_cast<const sphray_particle*>(particles.data()),
                              particles.size(), &c, pts.data(), pts.size(), &L.view, &q, &ds, &o,
                              reinterpret_cast<double*>(img.pixels.data()), &rs, &e),
          e);
    if (out_stats) {
        out_stats->particles = rs.particles;
        out_stats->skipped_particles = rs.skipped_particles;
        out_stats->knots = rs.knots;
        out_stats->rays_touched = rs.rays_touched;
        out_stats->int_ops = rs.int_ops;
        out_stats->residual_failures = rs.residual_failures;
        out_stats->step = rs.step;
    }
    return img;
}

}  // namespace sphray::gpu

// api.cpp -- the extern "C" boundary (include/sphray_gpu.h).  Exceptions never
// cross it: every entry point converts to a status code + sphray_error.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <cstdlib>
#include <string>
#include <vector>

#include "engine.hpp"
#include "host.hpp"
#include "sphray_gpu.h"

using namespace sphray_b200;

namespace sphray_b200 {
void comm_unique_id(uint8_t out[128]);
}

struct sphray_context {
    std::unique_ptr<Engine> engine;
};

namespace {

void clear(sphray_error* e) {
    if (!e) return;
    e->code = SPHRAY_OK;
    e->reserved = 0;
    e->particle_index = -1;
    e->ray_id = 0;
    e->msg[0] = 0;
}

sphray_status set(sphray_error* e, sphray_status code, const char* msg, int64_t pidx = -1,
                  uint64_t ray = 0) {
    if (e) {
        e->code = code;
        e->particle_index = pidx;
        e->ray_id = ray;
        std::strncpy(e->msg, msg, sizeof(e->msg) - 1);
        e->msg[sizeof(e->msg) - 1] = 0;
    }
    return code;
}

template <class F>
sphray_status guarded(sphray_error* err, F&& f) {
    clear(err);
    try {
        f();
        return SPHRAY_OK;
    } catch (const ThrownError& t) {
        return set(err, t.code, t.what(), t.pidx, t.ray);
    } catch (const std::bad_alloc&) {
        return set(err, SPHRAY_ERR_CUDA, "out of host memory");
    } catch (const std::exception& x) {
        return set(err, SPHRAY_ERR_NUMERIC, x.what());
    }
}

Engine& engine(sphray_context* ctx) {
    if (!ctx || !ctx->engine) fail(SPHRAY_ERR_CONFIG, "null context");
    return *ctx->engine;
}

sphray_render_options default_opts() {
    sphray_render_options o{};
    o.mode = SPHRAY_MODE_EXACT;
    return o;
}

}  // namespace

extern "C" {

int sphray_abi_version(void) { return SPHRAY_GPU_ABI_VERSION; }

const char* sphray_build_info(void) {
    return "sphray_b200: sm_100a CUDA path (fp64 exact geometry, int64 exact merge), CUDA "
#ifdef __CUDACC_VER_MAJOR__
           "nvcc"
#endif
           " build " __DATE__;
}

sphray_status sphray_context_create(int device, sphray_context** out, sphray_error* err) {
    return guarded(err, [&] {
        if (!out) fail(SPHRAY_ERR_CONFIG, "null output pointer");
        *out = nullptr;
        auto ctx = std::make_unique<sphray_context>();
        ctx->engine = std::make_unique<Engine>(device);
        *out = ctx.release();
    });
}

void sphray_context_destroy(sphray_context* ctx) { delete ctx; }

sphray_status sphray_probe_alu_peaks(int device, double* int64_gops, double* fp64_gflops,
                                     sphray_error* err) {
    return guarded(err, [&] {
        if (!int64_gops || !fp64_gflops) fail(SPHRAY_ERR_CONFIG, "null output pointer");
        probe_alu_peaks(device, int64_gops, fp64_gflops);
    });
}

sphray_status sphray_comm_unique_id(uint8_t unique_id[128], sphray_error* err) {
    return guarded(err, [&] { comm_unique_id(unique_id); });
}

sphray_status sphray_context_init_comm(sphray_context* ctx, int rank, int nranks,
                                       const uint8_t unique_id[128], sphray_error* err) {
    return guarded(err, [&] { engine(ctx).init_comm(rank, nranks, unique_id); });
}

sphray_status sphray_context_set_shard(sphray_context* ctx, int rank, int nranks,
                                       sphray_error* err) {
    return guarded(err, [&] { engine(ctx).set_shard(rank, nranks); });
}

sphray_status sphray_scene_upload(sphray_context* ctx, const sphray_particle* particles, size_t n,
                                  const sphray_lut_view* lut, sphray_error* err) {
    return guarded(err, [&] {
        if (!lut) fail(SPHRAY_ERR_CONFIG, "null lut");
        engine(ctx).upload_scene(particles, n, *lut);
    });
}

sphray_status sphray_scene_render(sphray_context* ctx, const sphray_camera* cam,
                                  const sphray_tf_point* tf, size_t ntf, const sphray_quanta* qc,
                                  const sphray_dataset_stats* stats,
                                  const sphray_render_options* opts, double* rgb_out,
                                  sphray_render_stats* out_stats, sphray_error* err) {
    return guarded(err, [&] {
        if (!cam || !qc || !stats) fail(SPHRAY_ERR_CONFIG, "null camera/quanta/stats");
        const sphray_render_options o = opts ? *opts : default_opts();
        engine(ctx).render(*cam, tf, ntf, *qc, *stats, o, rgb_out, out_stats, nullptr);
    });
}

sphray_status sphray_scene_info(sphray_context* ctx, size_t* n, int32_t* K, int32_t* D,
                                sphray_error* err) {
    return guarded(err, [&] {
        Engine& e = engine(ctx);
        if (!e.has_scene()) fail(SPHRAY_ERR_CONFIG, "no scene uploaded");
        if (n) *n = e.scene_size();
        if (K) *K = e.scene_K();
        if (D) *D = e.scene_D();
    });
}

sphray_status sphray_context_set_region(sphray_context* ctx, int32_t x0, int32_t y0, int32_t w,
                                        int32_t h, int32_t record_rays, sphray_error* err) {
    return guarded(err, [&] { engine(ctx).set_region(x0, y0, w, h, record_rays != 0); });
}

sphray_status sphray_context_ray_records(sphray_context* ctx, sphray_ray_record* out, size_t cap,
                                         size_t* count, sphray_error* err) {
    return guarded(err, [&] {
        const size_t n = engine(ctx).ray_records(out, cap);
        if (count) *count = n;
    });
}

void* sphray_context_stream(sphray_context* ctx) {
    if (!ctx || !ctx->engine) return nullptr;
    return ctx->engine->stream();
}

const double* sphray_scene_device_image(sphray_context* ctx) {
    if (!ctx || !ctx->engine) return nullptr;
    return ctx->engine->device_image();
}

sphray_status sphray_render_scene(sphray_context* ctx, const sphray_particle* particles, size_t n,
                                  const sphray_camera* cam, const sphray_tf_point* tf, size_t ntf,
                                  const sphray_lut_view* lut, const sphray_quanta* qc,
                                  const sphray_dataset_stats* stats,
                                  const sphray_render_options* opts, double* rgb_out,
                                  sphray_render_stats* out_stats, sphray_error* err) {
    return guarded(err, [&] {
        if (!cam || !lut || !qc || !stats) fail(SPHRAY_ERR_CONFIG, "null camera/lut/quanta/stats");
        // validation order of render_scene: camera, then transfer function (raycast.hpp:419-420)
        (void)make_camera(*cam);
        const sphray_render_options o = opts ? *opts : default_opts();
        Engine& e = engine(ctx);
        e.upload_scene(particles, n, *lut);
        e.render(*cam, tf, ntf, *qc, *stats, o, rgb_out, out_stats, nullptr);
    });
}

sphray_status sphray_scene_hits(sphray_context* ctx, const sphray_camera* cam, uint64_t* ray_id,
                                int64_t* particle_index, double* lam, double* t_chi, size_t cap,
                                size_t* count, sphray_error* err) {
    return guarded(err, [&] {
        if (!cam || !count) fail(SPHRAY_ERR_CONFIG, "null camera/count");
        // the hit set does not depend on TF or quanta; use neutral ones
        const sphray_tf_point tf{0.0, 0.0, 0.0, 0.0, 0.0};
        // hits do not depend on the quanta; these keep every knot integer small
        sphray_quanta qc{};
        qc.tau = 1.0;
        qc.sigma = 1e300;
        qc.int_width = 64;
        sphray_dataset_stats ds{};
        ds.h_r = 1.0;
        Dumps d;
        d.hits = true;
        d.cap_hits = cap;
        Engine& e = engine(ctx);
        e.render(*cam, &tf, 1, qc, ds, default_opts(), nullptr, nullptr, &d);
        *count = d.n_hits;
        if (cap == 0) return;
        // ray-major, then particle index
        const size_t k = std::min<size_t>(cap, d.hit_ray.size());
        std::vector<size_t> order(k);
        std::iota(order.begin(), order.end(), size_t{0});
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            return d.hit_ray[a] != d.hit_ray[b] ? d.hit_ray[a] < d.hit_ray[b]
                                                : d.hit_pidx[a] < d.hit_pidx[b];
        });
        for (size_t i = 0; i < k; ++i) {
            if (ray_id) ray_id[i] = d.hit_ray[order[i]];
            if (particle_index) particle_index[i] = d.hit_pidx[order[i]];
            if (lam) lam[i] = d.hit_lam[order[i]];
            if (t_chi) t_chi[i] = d.hit_tchi[order[i]];
        }
    });
}

sphray_status sphray_scene_pieces(sphray_context* ctx, const sphray_camera* cam,
                                  const sphray_quanta* qc, uint64_t* rays, uint64_t* piece_offsets,
                                  int64_t* piece_t, int64_t* piece_a, size_t cap_rays,
                                  size_t cap_pieces, size_t* n_rays, size_t* n_pieces,
                                  sphray_error* err) {
    return guarded(err, [&] {
        if (!cam || !qc || !n_rays || !n_pieces) fail(SPHRAY_ERR_CONFIG, "null argument");
        const sphray_tf_point tf{0.0, 0.0, 0.0, 0.0, 0.0};
        sphray_dataset_stats ds{};
        ds.h_r = 1.0;
        Dumps d;
        d.pieces = true;
        d.cap_pieces = cap_pieces;
        Engine& e = engine(ctx);
        sphray_render_stats st{};
        e.render(*cam, &tf, 1, *qc, ds, default_opts(), nullptr, &st, &d);
        *n_pieces = d.n_pieces;
        *n_rays = st.rays_touched;
        if (cap_pieces == 0 || d.piece_t.size() < d.n_pieces) return;
        const size_t k = d.piece_t.size();
        std::vector<size_t> order(k);
        std::iota(order.begin(), order.end(), size_t{0});
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            return d.piece_ray[a] != d.piece_ray[b] ? d.piece_ray[a] < d.piece_ray[b]
                                                    : d.piece_t[a] < d.piece_t[b];
        });
        const int D1 = static_cast<int>(d.piece_a.size() / std::max<size_t>(k, 1));
        size_t r = 0;
        for (size_t i = 0; i < k; ++i) {
            const size_t o = order[i];
            if (i == 0 || d.piece_ray[o] != d.piece_ray[order[i - 1]]) {
                if (r < cap_rays) {
                    if (rays) rays[r] = d.piece_ray[o];
                    if (piece_offsets) piece_offsets[r] = i;
                }
                ++r;
            }
            if (piece_t) piece_t[i] = d.piece_t[o];
            if (piece_a)
                for (int j = 0; j < D1; ++j) piece_a[i * D1 + j] = d.piece_a[o * D1 + j];
        }
        if (piece_offsets && r <= cap_rays) piece_offsets[r] = k;
        *n_rays = r;
    });
}

sphray_status sphray_quantize_hits(sphray_context* ctx, const sphray_particle* particles,
                                   size_t nhits, const double* t_chi, const double* lam,
                                   const sphray_lut_view* lut, const sphray_quanta* qc,
                                   int64_t* knot_t, int64_t* knot_b, int32_t* knot_count,
                                   sphray_error* err) {
    return guarded(err, [&] {
        if (!lut || !qc) fail(SPHRAY_ERR_CONFIG, "null lut/quanta");
        engine(ctx).quantize_hits(particles, nhits, t_chi, lam, *lut, *qc, knot_t, knot_b, knot_count);
    });
}

sphray_status sphray_compute_dataset_stats(const sphray_particle* particles, size_t n,
                                           const sphray_lut_view* lut, double clustering_factor,
                                           sphray_dataset_stats* out, sphray_error* err) {
    return guarded(err, [&] {
        if (!lut || !out) fail(SPHRAY_ERR_CONFIG, "null lut/output");
        *out = dataset_stats(particles, n, make_lut(*lut), clustering_factor);
    });
}

sphray_status sphray_scene_validate(sphray_context* ctx, const sphray_camera* cam,
                                    const sphray_quanta* qc, const sphray_dataset_stats* ds,
                                    sphray_validate_report* out, sphray_error* err) {
    return guarded(err, [&] {
        if (!ctx || !cam || !qc || !ds || !out) fail(SPHRAY_ERR_CONFIG, "null argument");
        ctx->engine->validate(*cam, *qc, *ds, out);
    });
}

sphray_status sphray_particles_load(const char* path, sphray_particle** out, size_t* n,
                                    sphray_error* err) {
    return guarded(err, [&] {
        if (!path || !out || !n) fail(SPHRAY_ERR_CONFIG, "null argument");
        *out = nullptr;
        *n = 0;
        const auto ps = load_particles(path);
        auto* buf = static_cast<sphray_particle*>(std::malloc(std::max<size_t>(ps.size(), 1) * sizeof(sphray_particle)));
        if (!buf) fail(SPHRAY_ERR_IO, "out of host memory");
        std::memcpy(buf, ps.data(), ps.size() * sizeof(sphray_particle));
        *out = buf;
        *n = ps.size();
    });
}

sphray_status sphray_particles_save(const char* path, const sphray_particle* particles, size_t n,
                                    int binary, sphray_error* err) {
    return guarded(err, [&] {
        if (!path || (n && !particles)) fail(SPHRAY_ERR_CONFIG, "null argument");
        save_particles(particles, n, path, binary != 0);
    });
}

sphray_status sphray_tf_load(const char* path, sphray_tf_point** out, size_t* n, sphray_error* err) {
    return guarded(err, [&] {
        if (!path || !out || !n) fail(SPHRAY_ERR_CONFIG, "null argument");
        *out = nullptr;
        *n = 0;
        const auto tf = load_transfer_function(path);
        auto* buf = static_cast<sphray_tf_point*>(std::malloc(std::max<size_t>(tf.size(), 1) * sizeof(sphray_tf_point)));
        if (!buf) fail(SPHRAY_ERR_IO, "out of host memory");
        std::memcpy(buf, tf.data(), tf.size() * sizeof(sphray_tf_point));
        *out = buf;
        *n = tf.size();
    });
}

sphray_status sphray_ppm_save(const char* path, const double* rgb, int width, int height,
                              sphray_error* err) {
    return guarded(err, [&] {
        if (!path || (width > 0 && height > 0 && !rgb)) fail(SPHRAY_ERR_CONFIG, "null argument");
        save_ppm(rgb, width, height, path);
    });
}

sphray_status sphray_camera_load(const char* path, sphray_camera* out, sphray_error* err) {
    return guarded(err, [&] {
        if (!path || !out) fail(SPHRAY_ERR_CONFIG, "null argument");
        *out = load_camera(path);
    });
}

void sphray_free(void* p) { std::free(p); }

sphray_status sphray_scene_upload_file(sphray_context* ctx, const char* path,
                                       const sphray_lut_view* lut, sphray_error* err) {
    return guarded(err, [&] {
        if (!ctx || !path || !lut) fail(SPHRAY_ERR_CONFIG, "null argument");
        Engine& e = engine(ctx);
        if (is_sprt(path)) {
            // SPRT records land directly in pinned host memory (no pageable bounce)
            sphray_particle* stage = nullptr;
            const size_t n = read_sprt_into(path, [&](size_t k) { return stage = e.stage_particles(k); });
            e.upload_scene(stage, n, *lut);
        } else {
            const auto ps = load_particles(path);
            e.upload_scene(ps.data(), ps.size(), *lut);
        }
    });
}

sphray_status sphray_scene_dataset_stats(sphray_context* ctx, double clustering_factor,
                                         sphray_dataset_stats* out, sphray_error* err) {
    return guarded(err, [&] {
        if (!ctx || !out) fail(SPHRAY_ERR_CONFIG, "null context/output");
        *out = ctx->engine->scene_dataset_stats(clustering_factor);
    });
}

sphray_status sphray_accumulate(sphray_context* ctx, int D, size_t nrays, const uint64_t* ray_ids,
                                const uint64_t* knot_offsets, const int64_t* knot_t,
                                const int64_t* knot_b, uint64_t* piece_offsets, int64_t* piece_t,
                                int64_t* piece_a, uint64_t* ops, sphray_error* err) {
    return guarded(err, [&] {
        Engine& e = engine(ctx);
        if (nrays && (!ray_ids || !knot_offsets || (knot_offsets[nrays] && (!knot_t || !knot_b))))
            fail(SPHRAY_ERR_CONFIG, "accumulate: null input");
        e.accumulate(D, nrays, ray_ids, knot_offsets, knot_t, knot_b, piece_offsets, piece_t, piece_a, ops);
    });
}

sphray_status sphray_lut_serialize(const sphray_lut_view* lut, const char* kernel_id, uint8_t* out,
                                   size_t cap, size_t* nbytes, sphray_error* err) {
    return guarded(err, [&] {
        if (!lut) fail(SPHRAY_ERR_CONFIG, "null LUT view");
        const auto bytes = serialize_lut(*lut, kernel_id ? kernel_id : "");
        if (nbytes) *nbytes = bytes.size();
        if (out && cap) std::memcpy(out, bytes.data(), std::min(cap, bytes.size()));
    });
}

sphray_status sphray_lut_save(const char* path, const sphray_lut_view* lut, const char* kernel_id,
                              sphray_error* err) {
    return guarded(err, [&] {
        if (!lut || !path) fail(SPHRAY_ERR_CONFIG, "null argument");
        const auto bytes = serialize_lut(*lut, kernel_id ? kernel_id : "");
        std::FILE* f = std::fopen(path, "wb");
        if (!f) fail(SPHRAY_ERR_IO, std::string("lut: cannot open ") + path + " for writing");
        const size_t w = std::fwrite(bytes.data(), 1, bytes.size(), f);
        const int c = std::fclose(f);
        if (w != bytes.size() || c != 0) fail(SPHRAY_ERR_IO, "lut: write failure");
    });
}

sphray_status sphray_render_report(const sphray_lut_view* lut, const char* kernel_id,
                                   const sphray_dataset_stats* ds, const sphray_quanta* qc,
                                   const sphray_render_stats* stats, uint64_t seed,
                                   const char* image_path, double kappa, double kappa_prime,
                                   char* out, size_t cap, size_t* len, sphray_error* err) {
    return guarded(err, [&] {
        if (!(kappa > 0.0)) kappa = kCubicKappa;
        if (!(kappa_prime > 0.0)) kappa_prime = kCubicKappaPrime;
        const std::string txt = render_report_json(lut, kernel_id ? kernel_id : "", ds, qc, stats, seed,
                                                   image_path ? image_path : "", kappa, kappa_prime);
        if (len) *len = txt.size();
        if (out && cap) {
            const size_t k = std::min(cap - 1, txt.size());
            std::memcpy(out, txt.data(), k);
            out[k] = 0;
        }
    });
}

sphray_status sphray_choose_quanta(const sphray_lut_view* lut, const sphray_dataset_stats* ds,
                                   int int_width, double kappa, double kappa_prime,
                                   sphray_quanta* out, sphray_error* err) {
    return guarded(err, [&] {
        if (!lut || !ds || !out) fail(SPHRAY_ERR_CONFIG, "null argument");
        if (!(kappa > 0.0)) kappa = kCubicKappa;
        if (!(kappa_prime > 0.0)) kappa_prime = kCubicKappaPrime;
        *out = choose_quanta(make_lut(*lut), *ds, int_width, kappa, kappa_prime);
    });
}

// deserialize_lut (lut.hpp:354-393): header checks; records are returned in place.
sphray_status sphray_lut_parse(const uint8_t* bytes, size_t nbytes, sphray_lut_view* view,
                               char kernel_id[17], sphray_error* err) {
    return guarded(err, [&] {
        if (!bytes || !view) fail(SPHRAY_ERR_CONFIG, "null argument");
        auto need = [&](size_t at, size_t len) {
            if (at + len > nbytes) fail(SPHRAY_ERR_IO, "lut: truncated file");
        };
        need(0, 4);
        if (std::memcmp(bytes, "SPLT", 4) != 0) fail(SPHRAY_ERR_IO, "lut: bad magic");
        auto u32 = [&](size_t at) {
            need(at, 4);
            uint32_t v = 0;
            for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(bytes[at + i]) << (8 * i);
            return v;
        };
        auto f64 = [&](size_t at) {
            need(at, 8);
            uint64_t v = 0;
            for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(bytes[at + i]) << (8 * i);
            double d;
            std::memcpy(&d, &v, 8);
            return d;
        };
        const uint32_t version = u32(4);
        if (version != 1) fail(SPHRAY_ERR_IO, "lut: unsupported format version " + std::to_string(version));
        need(8, 16);
        if (kernel_id) {
            std::memcpy(kernel_id, bytes + 8, 16);
            kernel_id[16] = 0;
        }
        const double q = f64(24);
        const int K = static_cast<int>(u32(32));
        const int D = static_cast<int>(u32(36));
        const uint32_t N = u32(40);
        if (!(q > 0.0)) fail(SPHRAY_ERR_IO, "lut: invalid support radius");
        validate_approx(K, D);
        const int m = (K + 1) / 2, nj = K * D / 2;
        const size_t rec = 2 + m + nj;
        const size_t body = static_cast<size_t>(N) * rec * 8;
        need(44, body);
        if (44 + body != nbytes) fail(SPHRAY_ERR_IO, "lut: trailing bytes");
        double prev = -1.0;
        for (uint32_t i = 0; i < N; ++i) {
            const double lam = f64(44 + static_cast<size_t>(i) * rec * 8);
            if (!(lam > prev)) fail(SPHRAY_ERR_IO, "lut: distances not ascending");
            prev = lam;
        }
        // the 44-byte header leaves the records 4-byte aligned in a file image;
        // callers then pass an 8-byte aligned copy of bytes[44:] as records
        const bool aligned = (reinterpret_cast<uintptr_t>(bytes + 44) & 7) == 0;
        const double* recs = aligned ? reinterpret_cast<const double*>(bytes + 44) : nullptr;
        view->q = q;
        view->K = K;
        view->D = D;
        view->N = static_cast<int32_t>(N);
        view->reserved = 0;
        view->records = recs;
    });
}

size_t sphray_scene_default_count(int config) { return scene_default_count(config); }

sphray_status sphray_generate_scene(int config, size_t n, uint64_t seed, sphray_particle* out,
                                    sphray_error* err) {
    return guarded(err, [&] {
        if (!out) fail(SPHRAY_ERR_CONFIG, "null output");
        if (n == 0) n = scene_default_count(config);
        generate_scene(config, n, seed, out);
    });
}

}  // extern "C"

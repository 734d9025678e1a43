// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A thin extern "C" driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/sphray/*.hpp, header-only C++20).  It is
// compiled by oracle/Makefile into oracle/_ref/libsphray_ref.so; nothing of the
// reference source is copied into this repository.  Only tests/, bench.py's
// cpu_baseline / --impl reference legs and __graft_entry__.smoke() may load it.
//
// Build flags follow SURVEY.md section 8(a): -std=c++20 -O2, no -march, no FMA
// contraction, so every fp64 result is the one the reference CLI produces.
//
// Entry points mirror the reference call sites:
//   rp_render            -> sphray::render_scene<Int>          raycast.hpp:414-497
//   rp_footprint         -> sphray::particle_ray_footprint     raycast.hpp:128-184
//   rp_quantize          -> sphray::quantize_particle<Int>     quantize.hpp:199-250
//   rp_pipeline_*        -> sweep 1 + sort_knots + accumulate  raycast.hpp:188-292
//   rp_dataset_stats     -> sphray::dataset_stats              quantize.hpp:129-165
//   rp_choose_quanta     -> sphray::choose_quanta              quantize.hpp:169-183
//   rp_lut_build         -> sphray::build_lut + save_lut       lut.hpp:245-280, 395-399
//   rp_render_banded     -> SURVEY.md 8(d) banded CPU-baseline driver built only
//                           from the reference's public functions.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sphray/io.hpp"
#include "sphray/raycast.hpp"
#include "sphray_scenes.hpp"

using namespace sphray;

extern "C" {

typedef struct {
    double x, y, z, mass, density, h, value;
} rp_particle;

typedef struct {
    int mode;  // 0 orthographic, 1 pinhole
    int width, height;
    double position[3], look_at[3], up[3];
    double fov_deg, ortho_height, near_plane, far_plane;
} rp_camera;

typedef struct {
    double value, r, g, b, absorption;
} rp_tf_point;

typedef struct {
    double tau, sigma;
    int width_bits;
} rp_quanta;

typedef struct {
    double mass_r, density_r, h_r, value_r, phi_repr, a_max, clustering_factor;
    std::uint64_t count;
} rp_dstats;

typedef struct {
    std::uint64_t particles, skipped_particles, knots, rays_touched, int_ops, residual_failures;
    double step;
} rp_rstats;

typedef struct {
    std::uint64_t piece_checksum;  // sum of piece_mix over the ray's FieldPieces
    std::uint32_t knots, pieces, hits, flags;  // flags: 1 touched, 2 residual, 4 T <= 1e-3
} rp_ray_record;

typedef struct {
    int code;  // 0 ok, 1 config, 2 io, 3 overflow, 4 numeric, 5 other
    std::int64_t particle_index;
    std::uint64_t ray_id;
    char msg[256];
} rp_error;

}  // extern "C"

static_assert(sizeof(rp_particle) == sizeof(Particle), "particle layout");

namespace {

void set_err(rp_error* e, int code, const char* msg, std::int64_t pidx = -1,
             std::uint64_t ray = 0) {
    if (!e) return;
    e->code = code;
    e->particle_index = pidx;
    e->ray_id = ray;
    std::strncpy(e->msg, msg, sizeof(e->msg) - 1);
    e->msg[sizeof(e->msg) - 1] = 0;
}

template <class F>
int guarded(rp_error* err, F&& f) {
    if (err) set_err(err, 0, "");
    try {
        f();
        return 0;
    } catch (const OverflowError& e) {
        set_err(err, 3, e.what(), e.particle_index, e.ray_id);
        return 3;
    } catch (const ConfigError& e) {
        set_err(err, 1, e.what());
        return 1;
    } catch (const IoError& e) {
        set_err(err, 2, e.what());
        return 2;
    } catch (const NumericError& e) {
        set_err(err, 4, e.what());
        return 4;
    } catch (const std::exception& e) {
        set_err(err, 5, e.what());
        return 5;
    }
}

Camera to_cam(const rp_camera* c) {
    Camera cam;
    cam.mode = c->mode ? Camera::Mode::pinhole : Camera::Mode::orthographic;
    cam.position = {c->position[0], c->position[1], c->position[2]};
    cam.look_at = {c->look_at[0], c->look_at[1], c->look_at[2]};
    cam.up = {c->up[0], c->up[1], c->up[2]};
    cam.width = c->width;
    cam.height = c->height;
    cam.fov_deg = c->fov_deg;
    cam.ortho_height = c->ortho_height;
    cam.near = c->near_plane;
    cam.far = c->far_plane;
    return cam;
}

void from_cam(const Camera& cam, rp_camera* c) {
    c->mode = cam.mode == Camera::Mode::pinhole ? 1 : 0;
    c->position[0] = cam.position.x;
    c->position[1] = cam.position.y;
    c->position[2] = cam.position.z;
    c->look_at[0] = cam.look_at.x;
    c->look_at[1] = cam.look_at.y;
    c->look_at[2] = cam.look_at.z;
    c->up[0] = cam.up.x;
    c->up[1] = cam.up.y;
    c->up[2] = cam.up.z;
    c->width = cam.width;
    c->height = cam.height;
    c->fov_deg = cam.fov_deg;
    c->ortho_height = cam.ortho_height;
    c->near_plane = cam.near;
    c->far_plane = cam.far;
}

TransferFunction to_tf(const rp_tf_point* p, std::size_t n) {
    TransferFunction tf;
    for (std::size_t i = 0; i < n; ++i)
        tf.points.push_back({p[i].value, p[i].r, p[i].g, p[i].b, p[i].absorption});
    return tf;
}

QuantaConfig to_qc(const rp_quanta* q) {
    QuantaConfig qc;
    qc.tau = q->tau;
    qc.sigma = q->sigma;
    qc.width = int_width_from(q->width_bits);
    return qc;
}

DatasetStats to_ds(const rp_dstats* s) {
    DatasetStats d;
    d.mass_r = s->mass_r;
    d.density_r = s->density_r;
    d.h_r = s->h_r;
    d.value_r = s->value_r;
    d.phi_repr = s->phi_repr;
    d.a_max = s->a_max;
    d.clustering_factor = s->clustering_factor;
    d.count = s->count;
    return d;
}

void from_ds(const DatasetStats& d, rp_dstats* s) {
    s->mass_r = d.mass_r;
    s->density_r = d.density_r;
    s->h_r = d.h_r;
    s->value_r = d.value_r;
    s->phi_repr = d.phi_repr;
    s->a_max = d.a_max;
    s->clustering_factor = d.clustering_factor;
    s->count = d.count;
}

std::span<const Particle> to_span(const rp_particle* p, std::size_t n) {
    return {reinterpret_cast<const Particle*>(p), n};
}

const PiecewisePolynomialKernel& kern() {
    static const auto k = cubic_bspline();
    return k;
}

// Results of the reference sweeps 1-3 for validation (knots sorted per ray,
// pieces from accumulate<Int128>, which the reference treats as identical to
// the int64 path whenever the latter does not throw: raycast_tests.cpp:440-442).
struct Pipeline {
    int D = 0;
    std::vector<std::uint64_t> rays;          // touched rays, ascending
    std::vector<std::uint64_t> knot_off;      // CSR over rays into knots
    std::vector<std::int64_t> knot_t;         // sorted by (ray, t) (stable)
    std::vector<std::int64_t> knot_b;         // (D+1) per knot
    std::vector<std::uint64_t> piece_off;     // CSR over rays into pieces
    std::vector<std::int64_t> piece_t;
    std::vector<std::int64_t> piece_a;        // (D+1) per piece, low 64 bits
    std::vector<std::uint8_t> piece_fits;     // all (D+1) coefficients fit int64
    std::vector<std::uint64_t> ray_ops;       // int_ops per ray (Int128 path)
};


// The piece hash of sphray_ray_record.piece_checksum (include/sphray_gpu.h,
// sphray_piece_mix), restated here so the checker does not include product code.
std::uint64_t piece_mix(std::int64_t t, const std::int64_t* a, int D) {
    static const std::uint64_t M[8] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full,
                                       0x165667B19E3779F9ull, 0x27D4EB2F165667C5ull,
                                       0x94D049BB133111EBull, 0xBF58476D1CE4E5B9ull,
                                       0xD6E8FEB86659FD93ull, 0xFF51AFD7ED558CCDull};
    std::uint64_t x = static_cast<std::uint64_t>(t) * M[0];
    for (int d = 0; d <= D; ++d) x += static_cast<std::uint64_t>(a[d]) * M[d + 1];
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    return x;
}

// A pixel region [x0, x0 + w) x [y0, y0 + h) of the camera (w == 0: the frame).
struct Region {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;  // exclusive ends
    bool contains(int px, int py) const { return px >= x0 && px < x1 && py >= y0 && py < y1; }
};

Region make_region(const Camera& cam, int x0, int y0, int w, int h) {
    Region r;
    if (w <= 0 || h <= 0) {
        r.x1 = cam.width;
        r.y1 = cam.height;
        return r;
    }
    r.x0 = std::max(0, std::min(x0, cam.width));
    r.y0 = std::max(0, std::min(y0, cam.height));
    r.x1 = std::max(r.x0, std::min(x0 + w, cam.width));
    r.y1 = std::max(r.y0, std::min(y0 + h, cam.height));
    return r;
}

// The reference's conservative orthographic pixel bbox (raycast.hpp:136-149,
// same operations), used only to skip particles that cannot reach a region;
// pinhole cameras keep every particle.  Two pixels of slack on each side:
// this filter is the harness's, not the reference's.
bool may_reach(const Particle& p, const Camera& cam, double q, const Region& r) {
    if (cam.mode != Camera::Mode::orthographic) return true;
    const Vec3 chi{p.x, p.y, p.z};
    const double support = q * p.h;
    const Vec3 rel = chi - cam.position;
    const double hw = 0.5 * cam.ortho_height * cam.aspect();
    const double hh = 0.5 * cam.ortho_height;
    const double cx = rel.dot(cam.right());
    const double cy = rel.dot(cam.up_vector());
    const double x0 = std::floor((cx - support + hw) / (2 * hw) * cam.width - 0.5) - 1;
    const double x1 = std::ceil((cx + support + hw) / (2 * hw) * cam.width - 0.5) + 1;
    const double y0 = std::floor((hh - (cy + support)) / (2 * hh) * cam.height - 0.5) - 1;
    const double y1 = std::ceil((hh - (cy - support)) / (2 * hh) * cam.height - 0.5) + 1;
    if (!(x0 == x0 && x1 == x1 && y0 == y0 && y1 == y1)) return true;
    return !(y1 + 2 < r.y0 || y0 - 2 > r.y1 - 1 || x1 + 2 < r.x0 || x0 - 2 > r.x1 - 1);
}

template <class Int>
void collect_knots(std::span<const Particle> ps, const Camera& cam, const Lut& lut,
                   const QuantaConfig& qc, std::vector<QuantizedKnot<Int>>& knots,
                   int threads, const std::vector<std::uint8_t>* row_mask,
                   const Region* region = nullptr) {
    const int nthreads = resolve_threads(threads);
    std::vector<std::vector<QuantizedKnot<Int>>> buffers(ps.size() ? nthreads : 0);
    if (!ps.empty()) {
        const std::size_t chunk = (ps.size() + nthreads - 1) / nthreads;
        parallel_for(buffers.size(), nthreads, [&](std::size_t b) {
            const std::size_t lo = b * chunk;
            const std::size_t hi = std::min(lo + chunk, ps.size());
            for (std::size_t i = lo; i < hi; ++i) {
                if (region && !may_reach(ps[i], cam, lut.q, *region)) continue;
                auto hits = particle_ray_footprint(ps[i], cam, lut.q);
                for (const auto& hit : hits) {
                    if (row_mask && !(*row_mask)[hit.ray.py]) continue;
                    if (region && !region->contains(hit.ray.px, hit.ray.py)) continue;
                    auto ks = quantize_particle<Int>(ps[i], hit.ray.id, hit.t_chi, hit.lam, lut,
                                                     qc, static_cast<std::int64_t>(i));
                    buffers[b].insert(buffers[b].end(), ks.begin(), ks.end());
                }
            }
        });
    }
    for (auto& b : buffers) knots.insert(knots.end(), b.begin(), b.end());
}

}  // namespace

extern "C" {

int rp_lut_build(int K, int D, int N, std::uint64_t seed, int threads, const char* path,
                 double* estar, rp_error* err) {
    return guarded(err, [&] {
        LutBuildOptions o;
        o.seed = seed;
        o.threads = threads;
        const auto lut = build_lut(kern(), {K, D}, N, o);
        save_lut(lut, path);
        if (estar) *estar = overall_error(lut, kernel_constants(kern()));
    });
}

void* rp_lut_load(const char* path, rp_error* err) {
    Lut* out = nullptr;
    guarded(err, [&] { out = new Lut(load_lut(path)); });
    return out;
}

void rp_lut_free(void* lut) { delete static_cast<Lut*>(lut); }

int rp_lut_info(void* lutp, double* q, int* K, int* D, int* N) {
    const Lut& lut = *static_cast<Lut*>(lutp);
    *q = lut.q;
    *K = lut.K;
    *D = lut.D;
    *N = static_cast<int>(lut.entries.size());
    return 0;
}

int rp_lut_lookup(void* lutp, double lam, double* knots, double* s_hat, int* idx) {
    const Lut& lut = *static_cast<Lut*>(lutp);
    const LutEntry& e = lut.lookup(lam);
    for (std::size_t i = 0; i < e.knots.size(); ++i) knots[i] = e.knots[i];
    for (std::size_t i = 0; i < e.s_hat.size(); ++i) s_hat[i] = e.s_hat[i];
    *idx = (&e >= lut.entries.data() && &e < lut.entries.data() + lut.entries.size())
               ? static_cast<int>(&e - lut.entries.data())
               : -1;
    return 0;
}

int rp_kernel_constants(double* kappa, double* kappa_prime) {
    const auto c = kernel_constants(kern());
    *kappa = c.kappa;
    *kappa_prime = c.kappa_prime;
    return 0;
}

int rp_dataset_stats(const rp_particle* ps, std::size_t n, void* lutp, double clustering,
                     rp_dstats* out, rp_error* err) {
    return guarded(err, [&] {
        from_ds(dataset_stats(to_span(ps, n), *static_cast<Lut*>(lutp), clustering), out);
    });
}

int rp_choose_quanta(void* lutp, const rp_dstats* ds, int width_bits, rp_quanta* out,
                     rp_error* err) {
    return guarded(err, [&] {
        const Lut& lut = *static_cast<Lut*>(lutp);
        const auto c = kernel_constants(kern());
        const auto qc =
            choose_quanta({lut.K, lut.D}, c, lut.q, to_ds(ds), int_width_from(width_bits));
        out->tau = qc.tau;
        out->sigma = qc.sigma;
        out->width_bits = static_cast<int>(qc.width);
    });
}

int rp_camera_ray(const rp_camera* c, int px, int py, double* origin, double* dir,
                  std::uint64_t* id) {
    const Camera cam = to_cam(c);
    const Ray r = cam.ray_at(px, py);
    origin[0] = r.origin.x;
    origin[1] = r.origin.y;
    origin[2] = r.origin.z;
    dir[0] = r.dir.x;
    dir[1] = r.dir.y;
    dir[2] = r.dir.z;
    *id = r.id;
    return 0;
}

int rp_render(const rp_particle* ps, std::size_t n, const rp_camera* c, const rp_tf_point* tfp,
              std::size_t ntf, void* lutp, const rp_quanta* q, const rp_dstats* ds, double step,
              const double* bg, int threads, int accum_bits, double* rgb, rp_rstats* st,
              double* seconds, rp_error* err) {
    return guarded(err, [&] {
        const Camera cam = to_cam(c);
        const TransferFunction tf = to_tf(tfp, ntf);
        const Lut& lut = *static_cast<Lut*>(lutp);
        const QuantaConfig qc = to_qc(q);
        const DatasetStats dstats = to_ds(ds);
        RenderOptions opts;
        opts.step = step;
        opts.background = {bg[0], bg[1], bg[2]};
        opts.threads = threads;
        RenderStats rs;
        Image img;
        const auto t0 = std::chrono::steady_clock::now();
        if (accum_bits == 128)
            img = render_scene<Int128>(to_span(ps, n), cam, tf, lut, qc, dstats, opts, &rs);
        else if (accum_bits == 32)
            img = render_scene<std::int32_t>(to_span(ps, n), cam, tf, lut, qc, dstats, opts, &rs);
        else
            img = render_scene<std::int64_t>(to_span(ps, n), cam, tf, lut, qc, dstats, opts, &rs);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (std::size_t i = 0; i < img.pixels.size(); ++i) {
            rgb[3 * i + 0] = img.pixels[i].r;
            rgb[3 * i + 1] = img.pixels[i].g;
            rgb[3 * i + 2] = img.pixels[i].b;
        }
        if (st) {
            st->particles = rs.particles;
            st->skipped_particles = rs.skipped_particles;
            st->knots = rs.knots;
            st->rays_touched = rs.rays_touched;
            st->int_ops = rs.int_ops;
            st->residual_failures = rs.residual_failures;
            st->step = rs.step;
        }
    });
}

// All (ray, particle) hits, particle-major in reference order.  Returns the
// total count; arrays are filled up to cap.
// rp_footprint_region keeps only hits whose pixel lies in the region
// (x0, y0, w, h; w == 0: the whole frame).
std::int64_t rp_footprint_region(const rp_particle* ps, std::size_t n, const rp_camera* c, double q,
                                 int x0, int y0, int w, int h, std::uint64_t* ray,
                                 std::int64_t* pidx, double* lam, double* tchi, std::size_t cap,
                                 rp_error* err) {
    std::int64_t total = 0;
    const int rc = guarded(err, [&] {
        const Camera cam = to_cam(c);
        const Region reg = make_region(cam, x0, y0, w, h);
        const bool all = w <= 0 || h <= 0;
        for (std::size_t i = 0; i < n; ++i) {
            const Particle& p = reinterpret_cast<const Particle*>(ps)[i];
            if (!all && !may_reach(p, cam, q, reg)) continue;
            const auto hits = particle_ray_footprint(p, cam, q);
            for (const auto& h : hits) {
                if (!all && !reg.contains(h.ray.px, h.ray.py)) continue;
                if (static_cast<std::size_t>(total) < cap) {
                    ray[total] = h.ray.id;
                    pidx[total] = static_cast<std::int64_t>(i);
                    lam[total] = h.lam;
                    tchi[total] = h.t_chi;
                }
                ++total;
            }
        }
    });
    return rc ? -1 : total;
}

std::int64_t rp_footprint(const rp_particle* ps, std::size_t n, const rp_camera* c, double q,
                          std::uint64_t* ray, std::int64_t* pidx, double* lam, double* tchi,
                          std::size_t cap, rp_error* err) {
    return rp_footprint_region(ps, n, c, q, 0, 0, 0, 0, ray, pidx, lam, tchi, cap, err);
}

int rp_quantize(const rp_particle* p, std::uint64_t ray, double tchi, double lam, void* lutp,
                const rp_quanta* q, std::int64_t pidx, std::int64_t* t_out, std::int64_t* b_out,
                int cap, int* nout, rp_error* err) {
    return guarded(err, [&] {
        const auto ks = quantize_particle<std::int64_t>(*reinterpret_cast<const Particle*>(p), ray,
                                                        tchi, lam, *static_cast<Lut*>(lutp),
                                                        to_qc(q), pidx);
        *nout = static_cast<int>(ks.size());
        for (int i = 0; i < static_cast<int>(ks.size()) && i < cap; ++i) {
            t_out[i] = ks[i].t;
            for (int d = 0; d <= max_degree; ++d) b_out[i * (max_degree + 1) + d] = ks[i].b[d];
        }
    });
}

// Accumulate one ray's sorted knots with the reference RayAccumulator.
int rp_accumulate(const std::int64_t* t, const std::int64_t* b /* 7 per knot */, std::size_t n,
                  int D, int accum_bits, std::int64_t* piece_t, std::int64_t* piece_a /* 7 */,
                  std::size_t* npieces, std::uint64_t* ops, rp_error* err) {
    return guarded(err, [&] {
        auto run = [&](auto tag) {
            using Int = typename decltype(tag)::type;
            std::vector<QuantizedKnot<Int>> ks(n);
            for (std::size_t i = 0; i < n; ++i) {
                ks[i].ray = 0;
                ks[i].t = t[i];
                for (int d = 0; d <= max_degree; ++d) ks[i].b[d] = b[i * (max_degree + 1) + d];
            }
            std::uint64_t o = 0;
            const auto pcs = accumulate<Int>(ks, D, &o);
            *npieces = pcs.size();
            for (std::size_t i = 0; i < pcs.size(); ++i) {
                piece_t[i] = static_cast<std::int64_t>(pcs[i].t);
                for (int d = 0; d <= max_degree; ++d)
                    piece_a[i * (max_degree + 1) + d] = static_cast<std::int64_t>(pcs[i].a[d]);
            }
            if (ops) *ops = o;
        };
        if (accum_bits == 128)
            run(std::type_identity<Int128>{});
        else
            run(std::type_identity<std::int64_t>{});
    });
}

// composite() of raycast.hpp:356-381 on int64 pieces.
int rp_composite(const std::int64_t* piece_t, const std::int64_t* piece_a, std::size_t n,
                 const rp_quanta* q, int D, const rp_tf_point* tfp, std::size_t ntf, double step,
                 double t_min, double t_max, double* rgba, rp_error* err) {
    return guarded(err, [&] {
        std::vector<FieldPiece<std::int64_t>> pcs(n);
        for (std::size_t i = 0; i < n; ++i) {
            pcs[i].t = piece_t[i];
            for (int d = 0; d <= max_degree; ++d) pcs[i].a[d] = piece_a[i * (max_degree + 1) + d];
        }
        const auto out =
            composite<std::int64_t>(pcs, to_qc(q), D, to_tf(tfp, ntf), step, t_min, t_max);
        rgba[0] = out.r;
        rgba[1] = out.g;
        rgba[2] = out.b;
        rgba[3] = out.a;
    });
}

// Sweeps 1-3 with intermediate results kept (validation oracle).
void* rp_pipeline_run_region(const rp_particle* ps, std::size_t n, const rp_camera* c, void* lutp,
                             const rp_quanta* q, int threads, int x0, int y0, int w, int h,
                             rp_error* err) {
    auto pl = std::make_unique<Pipeline>();
    const int rc = guarded(err, [&] {
        const Camera cam = to_cam(c);
        cam.validate();
        const Lut& lut = *static_cast<Lut*>(lutp);
        const QuantaConfig qc = to_qc(q);
        const int D = lut.D;
        pl->D = D;
        const Region reg = make_region(cam, x0, y0, w, h);
        std::vector<QuantizedKnot<Int128>> knots;
        collect_knots<Int128>(to_span(ps, n), cam, lut, qc, knots, threads, nullptr,
                              (w > 0 && h > 0) ? &reg : nullptr);
        sort_knots(knots);
        std::vector<std::size_t> starts;
        for (std::size_t i = 0; i < knots.size(); ++i)
            if (i == 0 || knots[i].ray != knots[i - 1].ray) starts.push_back(i);
        starts.push_back(knots.size());
        const std::size_t nrays = starts.size() - 1;
        pl->knot_off.push_back(0);
        pl->piece_off.push_back(0);
        pl->knot_t.reserve(knots.size());
        pl->knot_b.reserve(knots.size() * (D + 1));
        for (const auto& k : knots) {
            pl->knot_t.push_back(static_cast<std::int64_t>(k.t));
            for (int d = 0; d <= D; ++d) pl->knot_b.push_back(static_cast<std::int64_t>(k.b[d]));
        }
        std::vector<std::vector<FieldPiece<Int128>>> pieces(nrays);
        std::vector<std::uint64_t> ops(nrays, 0);
        parallel_for(nrays, resolve_threads(threads), [&](std::size_t r) {
            const std::span<const QuantizedKnot<Int128>> stream(knots.data() + starts[r],
                                                                starts[r + 1] - starts[r]);
            pieces[r] = accumulate<Int128>(stream, D, &ops[r]);
        });
        const Int128 lo = static_cast<Int128>(INT64_MIN), hi = static_cast<Int128>(INT64_MAX);
        for (std::size_t r = 0; r < nrays; ++r) {
            pl->rays.push_back(knots[starts[r]].ray);
            pl->knot_off.push_back(starts[r + 1]);
            for (const auto& pc : pieces[r]) {
                pl->piece_t.push_back(static_cast<std::int64_t>(pc.t));
                bool fits = true;
                for (int d = 0; d <= D; ++d) {
                    pl->piece_a.push_back(static_cast<std::int64_t>(pc.a[d]));
                    if (pc.a[d] < lo || pc.a[d] > hi) fits = false;
                }
                pl->piece_fits.push_back(fits);
            }
            pl->piece_off.push_back(pl->piece_t.size());
            pl->ray_ops.push_back(ops[r]);
        }
    });
    if (rc) return nullptr;
    return pl.release();
}

void* rp_pipeline_run(const rp_particle* ps, std::size_t n, const rp_camera* c, void* lutp,
                      const rp_quanta* q, int threads, rp_error* err) {
    return rp_pipeline_run_region(ps, n, c, lutp, q, threads, 0, 0, 0, 0, err);
}

void rp_pipeline_sizes(void* h, std::uint64_t* nrays, std::uint64_t* nknots,
                       std::uint64_t* npieces, int* D) {
    const Pipeline& p = *static_cast<Pipeline*>(h);
    *nrays = p.rays.size();
    *nknots = p.knot_t.size();
    *npieces = p.piece_t.size();
    *D = p.D;
}

void rp_pipeline_get(void* h, std::uint64_t* rays, std::uint64_t* knot_off, std::int64_t* knot_t,
                     std::int64_t* knot_b, std::uint64_t* piece_off, std::int64_t* piece_t,
                     std::int64_t* piece_a, std::uint8_t* piece_fits, std::uint64_t* ray_ops) {
    const Pipeline& p = *static_cast<Pipeline*>(h);
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(rays, p.rays);
    cp(knot_off, p.knot_off);
    cp(knot_t, p.knot_t);
    cp(knot_b, p.knot_b);
    cp(piece_off, p.piece_off);
    cp(piece_t, p.piece_t);
    cp(piece_a, p.piece_a);
    cp(piece_fits, p.piece_fits);
    cp(ray_ops, p.ray_ops);
}

void rp_pipeline_free(void* h) { delete static_cast<Pipeline*>(h); }

// SURVEY.md 8(d) banded CPU baseline: rows whose mask byte is set are rendered
// with the reference's sweeps (footprint -> quantize -> sort_knots ->
// accumulate -> composite); the wall time of the whole band render is returned.
int rp_render_banded(const rp_particle* ps, std::size_t n, const rp_camera* c,
                     const rp_tf_point* tfp, std::size_t ntf, void* lutp, const rp_quanta* q,
                     double step, int threads, int accum_bits, const std::uint8_t* row_mask,
                     double* seconds, std::uint64_t* rays_touched, std::uint64_t* knots_out,
                     double* rgb_touched_sum, rp_error* err) {
    return guarded(err, [&] {
        const Camera cam = to_cam(c);
        const TransferFunction tf = to_tf(tfp, ntf);
        const Lut& lut = *static_cast<Lut*>(lutp);
        const QuantaConfig qc = to_qc(q);
        const int D = lut.D;
        std::vector<std::uint8_t> mask(row_mask, row_mask + cam.height);
        auto run = [&](auto tag) {
            using Int = typename decltype(tag)::type;
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<QuantizedKnot<Int>> knots;
            collect_knots<Int>(to_span(ps, n), cam, lut, qc, knots, threads, &mask);
            sort_knots(knots);
            std::vector<std::size_t> starts;
            for (std::size_t i = 0; i < knots.size(); ++i)
                if (i == 0 || knots[i].ray != knots[i - 1].ray) starts.push_back(i);
            starts.push_back(knots.size());
            const std::size_t nrays = starts.size() - 1;
            std::vector<double> sums(nrays, 0.0);
            parallel_for(nrays, resolve_threads(threads), [&](std::size_t r) {
                const std::span<const QuantizedKnot<Int>> stream(knots.data() + starts[r],
                                                                 starts[r + 1] - starts[r]);
                auto pieces = accumulate(stream, D);
                const Rgba px = composite<Int>(pieces, qc, D, tf, step, cam.near, cam.far);
                sums[r] = px.r + px.g + px.b;
            });
            const auto t1 = std::chrono::steady_clock::now();
            *seconds = std::chrono::duration<double>(t1 - t0).count();
            *rays_touched = nrays;
            *knots_out = knots.size();
            double s = 0.0;
            for (double v : sums) s += v;
            *rgb_touched_sum = s;
        };
        if (accum_bits == 128)
            run(std::type_identity<Int128>{});
        else
            run(std::type_identity<std::int64_t>{});
    });
}


// Pixels [x0, x0 + w) x [y0, y0 + h) of the full-frame render_scene, driven
// only by the reference's public functions on the SAME camera (so the rays are
// the frame's, bit for bit): particle_ray_footprint -> quantize_particle ->
// sort_knots -> accumulate -> composite, with render_scene's pixel formula
// (raycast.hpp:466-488).  Particles whose reference bbox misses the region are
// skipped first (may_reach; orthographic cameras only).  Outputs rows
// y0 .. y0+h-1 at full width (background outside the region) and one record
// per region pixel, row-major; *seconds is the wall time of the reference's
// sweeps (the region filter excluded).  The accumulator is int64, falling
// back to Int128 on the reference's OverflowError when allow_fallback
// (*bits_used tells which; raycast_tests.cpp:440-442 equates the two).
int rp_render_region(const rp_particle* ps, std::size_t n, const rp_camera* c,
                     const rp_tf_point* tfp, std::size_t ntf, void* lutp, const rp_quanta* q,
                     double step, const double* bg, int threads, int x0, int y0, int w, int h,
                     int allow_fallback, double* rgb, rp_ray_record* rec, rp_rstats* st,
                     double* seconds, int* bits_used, rp_error* err) {
    return guarded(err, [&] {
        const Camera cam = to_cam(c);
        cam.validate();
        const TransferFunction tf = to_tf(tfp, ntf);
        tf.validate();
        const Lut& lut = *static_cast<Lut*>(lutp);
        const QuantaConfig qc = to_qc(q);
        const int D = lut.D;
        const int W = cam.width;
        const Region reg = make_region(cam, x0, y0, w, h);
        const int RW = reg.x1 - reg.x0;
        const std::size_t nrow_px = static_cast<std::size_t>(reg.y1 - reg.y0) * W;
        const std::size_t nreg = static_cast<std::size_t>(reg.y1 - reg.y0) * RW;
        auto at = [&](std::uint64_t id) {
            return static_cast<std::size_t>(id / W - reg.y0) * RW + (id % W - reg.x0);
        };
        const std::span<const Particle> all = to_span(ps, n);
        std::vector<std::uint32_t> keep;
        for (std::size_t i = 0; i < n; ++i)
            if (may_reach(all[i], cam, lut.q, reg)) keep.push_back(static_cast<std::uint32_t>(i));
        const double stp = step;
        auto run = [&](auto tag) {
            using Int = typename decltype(tag)::type;
            const int nthreads = resolve_threads(threads);
            const auto t0 = std::chrono::steady_clock::now();
            // sweep 1 (raycast.hpp:427-446) over the particles that can reach the region
            std::vector<std::vector<QuantizedKnot<Int>>> buffers(nthreads);
            std::vector<std::vector<std::uint64_t>> hit_rays(nthreads);
            const std::size_t chunk = (keep.size() + nthreads - 1) / nthreads;
            parallel_for(buffers.size(), nthreads, [&](std::size_t b) {
                const std::size_t lo = b * chunk, hi = std::min(lo + chunk, keep.size());
                for (std::size_t k = lo; k < hi; ++k) {
                    const std::size_t i = keep[k];
                    auto hits = particle_ray_footprint(all[i], cam, lut.q);
                    for (const auto& hit : hits) {
                        if (!reg.contains(hit.ray.px, hit.ray.py)) continue;
                        hit_rays[b].push_back(hit.ray.id);
                        auto ks = quantize_particle<Int>(all[i], hit.ray.id, hit.t_chi, hit.lam, lut,
                                                         qc, static_cast<std::int64_t>(i));
                        buffers[b].insert(buffers[b].end(), ks.begin(), ks.end());
                    }
                }
            });
            std::vector<QuantizedKnot<Int>> knots;
            for (auto& b : buffers) knots.insert(knots.end(), b.begin(), b.end());
            buffers.clear();
            sort_knots(knots);  // sweep 2
            std::vector<std::size_t> starts;
            for (std::size_t i = 0; i < knots.size(); ++i)
                if (i == 0 || knots[i].ray != knots[i - 1].ray) starts.push_back(i);
            starts.push_back(knots.size());
            const std::size_t nrays = starts.size() - 1;
            std::vector<Rgb> px(nrow_px, Rgb{bg[0], bg[1], bg[2]});
            std::vector<std::vector<FieldPiece<Int>>> pieces(nrays);
            std::vector<std::uint64_t> ops(nrays, 0);
            std::vector<double> Tend(nrays, 1.0);
            parallel_for(nrays, nthreads, [&](std::size_t r) {  // sweep 3
                const std::span<const QuantizedKnot<Int>> stream(knots.data() + starts[r],
                                                                 starts[r + 1] - starts[r]);
                pieces[r] = accumulate(stream, D, &ops[r]);
                const std::uint64_t id = stream[0].ray;
                const Rgba cc = composite<Int>(pieces[r], qc, D, tf, stp, cam.near, cam.far);
                Tend[r] = 1.0 - cc.a;
                px[(id / W - reg.y0) * W + id % W] = {cc.r + (1.0 - cc.a) * bg[0],
                                                      cc.g + (1.0 - cc.a) * bg[1],
                                                      cc.b + (1.0 - cc.a) * bg[2]};
            });
            const auto t1 = std::chrono::steady_clock::now();
            *seconds = std::chrono::duration<double>(t1 - t0).count();
            for (std::size_t i = 0; i < nrow_px; ++i) {
                rgb[3 * i + 0] = px[i].r;
                rgb[3 * i + 1] = px[i].g;
                rgb[3 * i + 2] = px[i].b;
            }
            std::memset(rec, 0, nreg * sizeof(rp_ray_record));
            for (const auto& hr : hit_rays)
                for (std::uint64_t id : hr) rec[at(id)].hits++;
            rp_rstats s{};
            s.particles = n;
            s.knots = knots.size();
            s.rays_touched = nrays;
            s.step = stp;
            for (std::size_t r = 0; r < nrays; ++r) {
                rp_ray_record& o = rec[at(knots[starts[r]].ray)];
                o.knots = static_cast<std::uint32_t>(starts[r + 1] - starts[r]);
                o.pieces = static_cast<std::uint32_t>(pieces[r].size());
                o.flags = 1u;
                std::uint64_t cs = 0;
                for (const auto& pc : pieces[r]) {
                    std::int64_t a[max_degree + 1];
                    for (int d = 0; d <= D; ++d) a[d] = static_cast<std::int64_t>(pc.a[d]);
                    cs += piece_mix(static_cast<std::int64_t>(pc.t), a, D);
                }
                bool zero = true;
                for (int d = 0; d <= D; ++d)
                    if (pieces[r].back().a[d] != Int{}) zero = false;
                if (!zero) {
                    o.flags |= 2u;
                    ++s.residual_failures;
                }
                if (!(Tend[r] > 1e-3)) o.flags |= 4u;
                o.piece_checksum = cs;
                s.int_ops += ops[r];
            }
            *st = s;
        };
        try {
            *bits_used = 64;
            run(std::type_identity<std::int64_t>{});
        } catch (const OverflowError&) {
            if (!allow_fallback) throw;
            *bits_used = 128;
            run(std::type_identity<Int128>{});
        }
    });
}

// The reference CLI's render report (sphray_main.cpp:196-256): the CLI does
// not build here (CLI11 absent), so this restates the report construction of
// cmd_render around the reference's own render_scene<Int>, dataset_stats,
// choose_quanta, overall_error and quantization_error.  Writes the JSON text
// (dump(2) + newline) to out (cap bytes incl. NUL); returns its length.
std::int64_t rp_render_report(const rp_particle* ps, std::size_t n, const rp_camera* c,
                              const rp_tf_point* tfp, std::size_t ntf, void* lutp, int int_width,
                              std::uint64_t seed, const char* image, char* out, std::size_t cap,
                              rp_error* err) {
    std::string txt;
    const int rc = guarded(err, [&] {
        const Camera cam = to_cam(c);
        cam.validate();
        const TransferFunction tf = to_tf(tfp, ntf);
        const auto kernel = cubic_bspline();
        const auto width = int_width_from(int_width);
        nlohmann::json report;
        const std::span<const Particle> particles = to_span(ps, n);
        if (particles.empty()) {
            report["quanta"] = nullptr;
            report["stats"] = {{"particles", 0}, {"knots", 0}, {"rays_touched", 0}};
            report["errors"] = nullptr;
            report["overflow_count"] = 0;
        } else {
            const Lut& lut = *static_cast<Lut*>(lutp);
            const auto cc = kernel_constants(kernel);
            const ApproxConfig cfg{lut.K, lut.D};
            const auto stats = dataset_stats(particles, lut);
            const auto qc = choose_quanta(cfg, cc, kernel.q, stats, width);
            RenderOptions opts;
            RenderStats rs;
            (void)dispatch_int_width(width, [&](auto tag) {
                using Int = typename decltype(tag)::type;
                return render_scene<Int>(particles, cam, tf, lut, qc, stats, opts, &rs);
            });
            const double estar = overall_error(lut, cc);
            const double qd = quantization_error(cfg, cc, kernel.q, qc.tau / stats.h_r, qc.sigma / stats.phi_repr);
            report["quanta"] = {{"tau", qc.tau}, {"sigma", qc.sigma}, {"int_width", int_width}};
            report["stats"] = {{"particles", rs.particles},
                               {"skipped_particles", rs.skipped_particles},
                               {"knots", rs.knots},
                               {"rays_touched", rs.rays_touched},
                               {"int_ops", rs.int_ops},
                               {"residual_failures", rs.residual_failures},
                               {"step", rs.step}};
            report["dataset"] = {{"count", stats.count},
                                 {"h_r", stats.h_r},
                                 {"phi_repr", stats.phi_repr},
                                 {"a_max", stats.a_max},
                                 {"clustering_factor", stats.clustering_factor}};
            report["errors"] = {{"E_star", estar}, {"Q_D", qd}, {"combined", std::hypot(estar, qd)}};
            report["overflow_count"] = 0;
            report["K"] = lut.K;
            report["D"] = lut.D;
        }
        report["kernel"] = kernel.id;
        report["seed"] = seed;
        report["image"] = image ? image : "";
        txt = report.dump(2) + "\n";
    });
    if (rc) return -1;
    if (out && cap) {
        const std::size_t k = std::min(cap - 1, txt.size());
        std::memcpy(out, txt.data(), k);
        out[k] = 0;
    }
    return static_cast<std::int64_t>(txt.size());
}

int rp_generate_scene(int config, std::size_t n, std::uint64_t seed, rp_particle* out, rp_error* err) {
    return guarded(err, [&] {
        if (sphray_scenes::default_count(config) == 0) throw ConfigError("unknown scene config");
        if (n == 0) n = sphray_scenes::default_count(config);
        sphray_scenes::generate(config, n, seed, reinterpret_cast<sphray_scenes::Record*>(out));
    });
}

std::size_t rp_scene_default_count(int config) { return sphray_scenes::default_count(config); }

// Reference loaders (io.hpp) for the bundled desk scene fixtures.
std::int64_t rp_load_particles(const char* path, rp_particle* out, std::size_t cap,
                               rp_error* err) {
    std::int64_t n = -1;
    guarded(err, [&] {
        const auto ps = load_particles(path);
        n = static_cast<std::int64_t>(ps.size());
        for (std::size_t i = 0; i < ps.size() && i < cap; ++i)
            std::memcpy(&out[i], &ps[i], sizeof(Particle));
    });
    return n;
}

std::int64_t rp_load_tf(const char* path, rp_tf_point* out, std::size_t cap, rp_error* err) {
    std::int64_t n = -1;
    guarded(err, [&] {
        const auto tf = load_transfer_function(path);
        n = static_cast<std::int64_t>(tf.points.size());
        for (std::size_t i = 0; i < tf.points.size() && i < cap; ++i)
            out[i] = {tf.points[i].value, tf.points[i].r, tf.points[i].g, tf.points[i].b,
                      tf.points[i].absorption};
    });
    return n;
}

int rp_load_camera(const char* path, rp_camera* out, rp_error* err) {
    return guarded(err, [&] { from_cam(load_camera(path), out); });
}

}  // extern "C"

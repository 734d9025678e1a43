// oracle/shim_demo.cpp -- TEST INFRASTRUCTURE: the drop-in demonstration.
//
// A reference-side program that renders the scene of raycast_tests.cpp:390-443
// twice -- once with the reference's own sphray::render_scene<int64_t>, once
// with sphray::gpu::render_scene<int64_t> from include/sphray_gpu.hpp (the
// B200 path) -- with identical arguments, and prints the max |RGB difference|
// and both RenderStats.  Built by oracle/Makefile into oracle/_ref/shim_demo
// (needs /root/reference at build time; runs on the GPU box).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "sphray/raycast.hpp"
#include "sphray_gpu.hpp"

using namespace sphray;

static std::vector<Particle> random_cloud(std::mt19937_64& rng, int n, double spread, double d0,
                                          double d1) {
    auto u = [&](double lo, double hi) { return lo + (hi - lo) * double(rng() >> 11) * 0x1.0p-53; };
    std::vector<Particle> ps;
    for (int i = 0; i < n; ++i)
        ps.push_back({u(-spread, spread), u(-spread, spread), u(d0, d1), u(0.2, 2.0), u(0.5, 2.0),
                      u(0.1, 0.6), u(-1.0, 1.5)});
    return ps;
}

int main() {
    const auto kern = cubic_bspline();
    const Lut lut = build_lut(kern, {4, 3}, 16);
    std::mt19937_64 rng(31337);
    const auto ps = random_cloud(rng, 120, 1.6, -1.2, 1.2);
    Camera cam;
    cam.mode = Camera::Mode::orthographic;
    cam.position = {0, 0, 4};
    cam.look_at = {0, 0, 0};
    cam.width = 24;
    cam.height = 24;
    cam.ortho_height = 5.0;
    TransferFunction tf;
    tf.points = {{-0.5, 0, 0, 0.2, 0.1}, {0.5, 0.9, 0.3, 0.1, 1.4}};
    const auto stats = dataset_stats(ps, lut);
    const auto qc = choose_quanta({4, 3}, kernel_constants(kern), kern.q, stats, IntWidth::w64);
    RenderOptions opts;
    opts.background = {0.01, 0.02, 0.03};

    RenderStats rs_ref, rs_gpu;
    const Image a = render_scene<std::int64_t>(ps, cam, tf, lut, qc, stats, opts, &rs_ref);
    const Image b = gpu::render_scene<std::int64_t>(ps, cam, tf, lut, qc, stats, opts, &rs_gpu);
    double err = 0.0;
    for (size_t i = 0; i < a.pixels.size(); ++i)
        err = std::max({err, std::fabs(a.pixels[i].r - b.pixels[i].r),
                        std::fabs(a.pixels[i].g - b.pixels[i].g),
                        std::fabs(a.pixels[i].b - b.pixels[i].b)});
    std::printf("max_abs_rgb_diff %.3e\n", err);
    std::printf("ref knots %zu rays %zu int_ops %llu residual %zu skipped %zu\n", rs_ref.knots,
                rs_ref.rays_touched, (unsigned long long)rs_ref.int_ops, rs_ref.residual_failures,
                rs_ref.skipped_particles);
    std::printf("gpu knots %zu rays %zu int_ops %llu residual %zu skipped %zu\n", rs_gpu.knots,
                rs_gpu.rays_touched, (unsigned long long)rs_gpu.int_ops, rs_gpu.residual_failures,
                rs_gpu.skipped_particles);
    // the Int parameter selects the device arithmetic (dispatch_int_width,
    // int_ops.hpp:113-121): <int32_t> on w32 quanta, <Int128> on w64 quanta
    const auto qc32 = choose_quanta({4, 3}, kernel_constants(kern), kern.q, stats, IntWidth::w32);
    RenderStats r32a, r32b, r128a, r128b;
    const Image c32 = render_scene<std::int32_t>(ps, cam, tf, lut, qc32, stats, opts, &r32a);
    const Image d32 = gpu::render_scene<std::int32_t>(ps, cam, tf, lut, qc32, stats, opts, &r32b);
    const Image c128 = render_scene<Int128>(ps, cam, tf, lut, qc, stats, opts, &r128a);
    const Image d128 = gpu::render_scene<Int128>(ps, cam, tf, lut, qc, stats, opts, &r128b);
    double err32 = 0.0, err128 = 0.0;
    for (size_t i = 0; i < c32.pixels.size(); ++i) {
        err32 = std::max({err32, std::fabs(c32.pixels[i].r - d32.pixels[i].r),
                          std::fabs(c32.pixels[i].g - d32.pixels[i].g), std::fabs(c32.pixels[i].b - d32.pixels[i].b)});
        err128 = std::max({err128, std::fabs(c128.pixels[i].r - d128.pixels[i].r),
                           std::fabs(c128.pixels[i].g - d128.pixels[i].g),
                           std::fabs(c128.pixels[i].b - d128.pixels[i].b)});
    }
    std::printf("int32 max_abs_rgb_diff %.3e knots %zu/%zu; Int128 max_abs_rgb_diff %.3e int_ops %llu/%llu\n",
                err32, r32a.knots, r32b.knots, err128, (unsigned long long)r128a.int_ops,
                (unsigned long long)r128b.int_ops);
    // <Int128> on w128 quanta: the device's 128-bit merge
    const auto qcw = choose_quanta({4, 3}, kernel_constants(kern), kern.q, stats, IntWidth::w128);
    RenderStats rwa, rwb;
    const Image cw = render_scene<Int128>(ps, cam, tf, lut, qcw, stats, opts, &rwa);
    const Image dw = gpu::render_scene<Int128>(ps, cam, tf, lut, qcw, stats, opts, &rwb);
    double errw = 0.0;
    for (size_t i = 0; i < cw.pixels.size(); ++i)
        errw = std::max({errw, std::fabs(cw.pixels[i].r - dw.pixels[i].r), std::fabs(cw.pixels[i].g - dw.pixels[i].g),
                         std::fabs(cw.pixels[i].b - dw.pixels[i].b)});
    std::printf("Int128/w128 max_abs_rgb_diff %.3e knots %zu/%zu int_ops %llu/%llu\n", errw, rwa.knots, rwb.knots,
                (unsigned long long)rwa.int_ops, (unsigned long long)rwb.int_ops);
    const bool widths_ok = err32 <= 1e-4 && r32a.knots == r32b.knots && r32a.int_ops == r32b.int_ops &&
                           err128 <= 1e-4 && r128a.int_ops == r128b.int_ops && errw <= 1e-4 &&
                           rwa.knots == rwb.knots && rwa.int_ops == rwb.int_ops;
    // errors come back as the reference's exception types
    bool threw = false;
    try {
        Camera bad = cam;
        bad.width = 0;
        (void)gpu::render_scene<std::int64_t>(ps, bad, tf, lut, qc, stats, opts);
    } catch (const ConfigError&) {
        threw = true;
    }
    std::printf("config_error_rethrown %d\n", threw ? 1 : 0);
    const bool ok = err <= 1e-4 && rs_ref.knots == rs_gpu.knots &&
                    rs_ref.rays_touched == rs_gpu.rays_touched &&
                    rs_ref.int_ops == rs_gpu.int_ops && threw && widths_ok;
    std::printf("%s\n", ok ? "SHIM_OK" : "SHIM_MISMATCH");
    return ok ? 0 : 1;
}

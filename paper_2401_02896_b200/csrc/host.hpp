// host.hpp -- host-side pieces of the path: camera constants, LUT layout,
// dataset statistics / quanta (quantize.hpp:97-183), synthetic scenes.
//
// Everything here is compiled with -ffp-contract=off and no -march so fp64
// results equal the reference's (SURVEY.md 8(a) exactness cheat-sheet).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphray_gpu.h"

namespace sphray_b200 {

// Reference kernel constants of cubic_bspline() as kernel_constants()
// (kernel.hpp:158-190) computes them; pinned against oracle/_ref in tests.
constexpr double kCubicKappa = 0x1.68a53e31586eap-2;       // 0.35219285179310467
constexpr double kCubicKappaPrime = 0x1.5c74590f520d8p-3;  // 0.17014379098896515

constexpr int kMaxPieces = 8;  // approx.hpp:19
constexpr int kMaxDegree = 6;  // approx.hpp:20
constexpr int kMaxM = 4;       // ceil(kMaxPieces / 2)

// Internal exception carrying an ABI status; converted at the C boundary.
struct ThrownError : std::runtime_error {
    ThrownError(sphray_status c, const std::string& m, int64_t p, uint64_t r)
        : std::runtime_error(m), code(c), pidx(p), ray(r) {}
    sphray_status code;
    int64_t pidx;
    uint64_t ray;
};

[[noreturn]] void fail(sphray_status code, const std::string& msg, int64_t pidx = -1,
                       uint64_t ray = 0);

// ---------------------------------------------------------------------------
// Camera: the reference recomputes forward()/right()/up_vector() on every
// ray_at() call (raycast.hpp:70-100); they are pure functions of the camera,
// so they are evaluated once here with the same operation order.
struct CamConst {
    int32_t mode;  // 0 ortho, 1 pinhole
    int32_t W, H;
    int32_t pad;
    double pos[3];
    double fwd[3];
    double right[3];
    double upv[3];
    double aspect;     // (double)W / H                         raycast.hpp:78
    double hw, hh;     // 0.5*ortho_height*aspect, 0.5*ortho_height raycast.hpp:89-90
    double two_hw, two_hh;  // 2*hw, 2*hh                      raycast.hpp:142-149
    double th;         // tan(fov*pi/360) (glibc)               raycast.hpp:94
    double th_aspect;  // th * aspect                           raycast.hpp:163
    double near_plane, far_plane;
};

CamConst make_camera(const sphray_camera& c);  // validates like Camera::validate

// ---------------------------------------------------------------------------
// LUT in the device layout: per entry m knots then |J| jumps (f64), plus the
// basis index set (approx.hpp:44-54).
struct LutHost {
    double q = 0.0;
    int K = 0, D = 0, N = 0, m = 0, nj = 0;
    double delta_lambda = 0.0;  // q / N, lut.hpp:39
    double theta_max = 0.0;     // largest knot radius over all entries
    std::vector<double> rows;   // N * (m + nj)
    std::vector<int> idx_k, idx_d;  // basis index set
    std::vector<double> lambda, error;
};

LutHost make_lut(const sphray_lut_view& v);
void validate_tf(const sphray_tf_point* tf, size_t ntf);  // TransferFunction::validate

// io.cpp: io.hpp:62-216 restated
std::vector<sphray_particle> load_particles(const std::string& path);
bool is_sprt(const std::string& path);
size_t read_sprt_into(const std::string& path, const std::function<sphray_particle*(size_t)>& alloc);
void save_particles(const sphray_particle* ps, size_t n, const std::string& path, bool binary);
std::vector<sphray_tf_point> load_transfer_function(const std::string& path);
void save_ppm(const double* rgb, int W, int H, const std::string& path);
sphray_camera load_camera(const std::string& path);
std::vector<uint8_t> serialize_lut(const sphray_lut_view& v, const std::string& kernel_id);
std::string render_report_json(const sphray_lut_view* lut, const std::string& kernel_id,
                               const sphray_dataset_stats* ds, const sphray_quanta* qc,
                               const sphray_render_stats* st, uint64_t seed, const std::string& image,
                               double kappa, double kappa_prime);
// overall_error (lut.hpp:284-290) and quantization_error (quantize.hpp:64-73)
double overall_error(const LutHost& L, double kappa);
double quantization_error(const LutHost& L, double kappa, double kappa_prime, double tau_rel,
                          double sigma_rel);

// probe.cu: measured issue peaks (int64 mul/add ops/s, fp64 flops/s) of this GPU
void probe_alu_peaks(int device, double* int64_gops, double* fp64_gflops);
void validate_approx(int K, int D);  // ApproxConfig::validate approx.hpp:27-30

// ---------------------------------------------------------------------------
// Host precompute (quantize.hpp:118-183, lut.hpp:184-234).
sphray_dataset_stats dataset_stats(const sphray_particle* ps, size_t n, const LutHost& lut,
                                   double clustering_factor);
sphray_quanta choose_quanta(const LutHost& lut, const sphray_dataset_stats& ds, int width,
                            double kappa, double kappa_prime);
double entry_amplitude(const LutHost& lut, int entry);

// pow(h, d+3) for d = 1..D per particle (glibc pow, as quantize.hpp:222), the
// only libm call of quantize that depends on the particle.  Multithreaded.
void particle_powers(const sphray_particle* ps, size_t n, int D, double* out /* n*D */);
// the same, plus the coordinate bounding box (lo/hi x, y, z) in the same pass
void particle_powers_bbox(const sphray_particle* ps, size_t n, int D, double* out, double lo[3],
                          double hi[3]);

int host_threads();

// ---------------------------------------------------------------------------
size_t scene_default_count(int config);
void generate_scene(int config, size_t n, uint64_t seed, sphray_particle* out);

}  // namespace sphray_b200

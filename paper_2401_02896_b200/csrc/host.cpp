// host.cpp -- host-side pieces of the path (see host.hpp).
#include "host.hpp"
#include "sphray_scenes.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <numbers>
#include <random>
#include <stdexcept>
#include <mutex>
#include <thread>

namespace sphray_b200 {

void fail(sphray_status code, const std::string& msg, int64_t pidx, uint64_t ray) {
    throw ThrownError(code, msg, pidx, ray);
}

int host_threads() {
    if (const char* env = std::getenv("SPHRAY_THREADS")) {
        const int v = std::atoi(env);
        if (v >= 1) return v;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

template <class F>
static void parallel_chunks(size_t n, F&& fn) {
    const int T = std::max(1, std::min<int>(host_threads(), static_cast<int>((n + 65535) / 65536)));
    if (T <= 1) {
        fn(size_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const size_t chunk = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const size_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, lo, hi] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------------------
// Vec3 arithmetic in the reference's operation order (raycast.hpp:17-35).
namespace {
struct V3 {
    double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 o) {
    return {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
}
inline V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(V3 a) {
    const double n = norm(a);
    if (!(n > 0.0)) fail(SPHRAY_ERR_CONFIG, "cannot normalize a zero vector");
    return scale(a, 1.0 / n);
}
inline V3 v3(const double* p) { return {p[0], p[1], p[2]}; }
inline void put(double* o, V3 v) {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
}
}  // namespace

CamConst make_camera(const sphray_camera& c) {
    // Camera::validate, raycast.hpp:59-68
    if (c.width < 1 || c.height < 1) fail(SPHRAY_ERR_CONFIG, "camera: resolution must be positive");
    if (!(c.far_plane > c.near_plane))
        fail(SPHRAY_ERR_CONFIG, "camera: far plane must lie beyond near");
    if (c.mode != 0 && c.mode != 1) fail(SPHRAY_ERR_CONFIG, "camera: unknown mode");
    if (c.mode == 1 && !(c.fov_deg > 0.0 && c.fov_deg < 180.0))
        fail(SPHRAY_ERR_CONFIG, "camera: field of view must be inside (0, 180) degrees");
    if (c.mode == 0 && !(c.ortho_height > 0.0))
        fail(SPHRAY_ERR_CONFIG, "camera: orthographic height must be positive");
    const V3 fwd = normalized(sub(v3(c.look_at), v3(c.position)));  // raycast.hpp:70
    const V3 r0 = cross(fwd, v3(c.up));                                 // raycast.hpp:72
    if (!(norm(r0) > 1e-12)) fail(SPHRAY_ERR_CONFIG, "camera: up is parallel to view direction");
    const V3 right = normalized(r0);
    const V3 upv = cross(right, fwd);  // raycast.hpp:76

    CamConst k{};
    k.mode = c.mode;
    k.W = c.width;
    k.H = c.height;
    put(k.pos, v3(c.position));
    put(k.fwd, fwd);
    put(k.right, right);
    put(k.upv, upv);
    k.aspect = static_cast<double>(c.width) / c.height;
    k.hw = 0.5 * c.ortho_height * k.aspect;
    k.hh = 0.5 * c.ortho_height;
    k.two_hw = 2 * k.hw;
    k.two_hh = 2 * k.hh;
    k.th = std::tan(c.fov_deg * std::numbers::pi / 360.0);
    k.th_aspect = k.th * k.aspect;
    k.near_plane = c.near_plane;
    k.far_plane = c.far_plane;
    return k;
}

// ---------------------------------------------------------------------------
void validate_approx(int K, int D) {
    if (K < 1 || K > kMaxPieces) fail(SPHRAY_ERR_CONFIG, "K must be in [1, 8]");
    if (D < 1 || D > kMaxDegree) fail(SPHRAY_ERR_CONFIG, "D must be in [1, 6]");
}

LutHost make_lut(const sphray_lut_view& v) {
    validate_approx(v.K, v.D);
    if (!(v.q > 0.0)) fail(SPHRAY_ERR_IO, "lut: invalid support radius");
    if (v.N < 1) fail(SPHRAY_ERR_NUMERIC, "lut: empty table");
    if (!v.records) fail(SPHRAY_ERR_CONFIG, "lut: no records");
    LutHost L;
    L.q = v.q;
    L.K = v.K;
    L.D = v.D;
    L.N = v.N;
    L.m = (v.K + 1) / 2;  // positive_knot_count, approx.hpp:39
    // basis_index_set, approx.hpp:44-54
    for (int k = 1; k <= L.m; ++k)
        for (int d = 1; d <= v.D; ++d) {
            if (v.K % 2 == 1 && k == 1 && d % 2 == 1) continue;
            L.idx_k.push_back(k);
            L.idx_d.push_back(d);
        }
    L.nj = static_cast<int>(L.idx_k.size());
    L.delta_lambda = v.q / static_cast<double>(v.N);
    const int rec = 2 + L.m + L.nj;
    L.rows.resize(static_cast<size_t>(v.N) * (L.m + L.nj));
    double prev = -1.0;
    for (int i = 0; i < v.N; ++i) {
        const double* r = v.records + static_cast<size_t>(i) * rec;
        L.lambda.push_back(r[0]);
        L.error.push_back(r[1]);
        if (!(r[0] > prev)) fail(SPHRAY_ERR_IO, "lut: distances not ascending");
        prev = r[0];
        for (int j = 0; j < L.m + L.nj; ++j)
            L.rows[static_cast<size_t>(i) * (L.m + L.nj) + j] = r[2 + j];
        for (int k = 0; k < L.m; ++k) L.theta_max = std::max(L.theta_max, std::fabs(r[2 + k]));
    }
    return L;
}

// ---------------------------------------------------------------------------
// lut.hpp:100-168 in real arithmetic, as reconstruct_entry uses it.
namespace {
const long long kBinom[7][7] = {{1, 0, 0, 0, 0, 0, 0},  {1, 1, 0, 0, 0, 0, 0},
                                {1, 2, 1, 0, 0, 0, 0},  {1, 3, 3, 1, 0, 0, 0},
                                {1, 4, 6, 4, 1, 0, 0},  {1, 5, 10, 10, 5, 1, 0},
                                {1, 6, 15, 20, 15, 6, 1}};

struct DKnot {
    double pos;
    double b[kMaxDegree + 1];
};

std::vector<DKnot> mirror_closure_real(const double* pos /* m+1 */,
                                       const double (*bpos)[kMaxDegree + 1], int m, int K,
                                       int D) {
    double bneg[kMaxM][kMaxDegree + 1] = {};
    for (int k = 1; k <= m; ++k)
        for (int d = 0; d <= D; ++d)
            bneg[m - k][d] = (d % 2 == 1) ? bpos[k - 1][d] : -bpos[k - 1][d];
    auto offset = [&](int k) { return pos[k] - pos[0]; };
    double center[kMaxDegree + 1] = {};
    if (K % 2 == 0) {
        for (int d = 1; d <= D; d += 2) {
            double acc = 0.0;
            for (int k = 1; k <= m; ++k) {
                const double off = offset(k);
                double pw = 1.0;
                for (int j = d; j <= D; ++j) {
                    acc += static_cast<double>(kBinom[j][d]) * bneg[m - k][j] * pw;
                    if (j < D) pw = pw * off;
                }
            }
            center[d] = -(acc + acc);
        }
    } else {
        for (int d = (D % 2 == 1 ? D : D - 1); d >= 1; d -= 2) {
            double acc = 0.0;
            for (int k = 2; k <= m; ++k) acc += bneg[m - k][d];
            for (int k = 1; k <= m; ++k) {
                const double off = offset(k);
                double pw = off;
                for (int j = d + 1; j <= D; ++j) {
                    acc += static_cast<double>(kBinom[j][d]) * bneg[m - k][j] * pw;
                    if (j < D) pw = pw * off;
                }
            }
            bneg[m - 1][d] = -acc;
        }
    }
    std::vector<DKnot> out;
    for (int k = m; k >= 1; --k) {
        DKnot kn{};
        kn.pos = pos[0] + pos[0] - pos[k];
        for (int d = 0; d <= kMaxDegree; ++d) kn.b[d] = bneg[m - k][d];
        out.push_back(kn);
    }
    if (K % 2 == 0) {
        DKnot kn{};
        kn.pos = pos[0];
        for (int d = 0; d <= kMaxDegree; ++d) kn.b[d] = center[d];
        out.push_back(kn);
    }
    for (int k = 1; k <= m; ++k) {
        DKnot kn{};
        kn.pos = pos[k];
        for (int d = 0; d <= D; ++d)
            kn.b[d] = (d % 2 == 1) ? bneg[m - k][d] : -bneg[m - k][d];
        out.push_back(kn);
    }
    return out;
}
}  // namespace

// entry_amplitude + reconstruct_entry, lut.hpp:184-234.
double entry_amplitude(const LutHost& L, int entry) {
    const int m = L.m, D = L.D;
    const double* row = &L.rows[static_cast<size_t>(entry) * (L.m + L.nj)];
    double pos[kMaxM + 1] = {0.0};
    for (int k = 1; k <= m; ++k) pos[k] = row[k - 1];
    double bpos[kMaxM][kMaxDegree + 1] = {};
    for (int i = 0; i < L.nj; ++i) bpos[L.idx_k[i] - 1][L.idx_d[i]] = row[m + i];
    const auto knots = mirror_closure_real(pos, bpos, m, L.K, D);

    std::vector<double> positions;
    std::vector<std::array<double, kMaxDegree + 1>> local;
    std::array<double, kMaxDegree + 1> a{};
    double prev = 0.0;
    for (size_t i = 0; i < knots.size(); ++i) {
        if (i > 0) {
            const double dt = knots[i].pos - prev;
            std::array<double, kMaxDegree + 1> next{};
            for (int d = 0; d <= D; ++d) {
                double acc = knots[i].b[d];
                double pw = 1.0;
                for (int j = d; j <= D; ++j) {
                    acc += static_cast<double>(kBinom[j][d]) * a[j] * pw;
                    pw *= dt;
                }
                next[d] = acc;
            }
            a = next;
        } else {
            for (int d = 0; d <= kMaxDegree; ++d) a[d] = knots[i].b[d];
        }
        prev = knots[i].pos;
        positions.push_back(knots[i].pos);
        local.push_back(a);
    }
    auto eval_local = [&](size_t i, double x) {
        double r = 0.0;
        for (int d = D; d >= 0; --d) r = r * x + local[i][d];  // Polynomial::eval, n = D+1
        return r;
    };
    auto evaluate = [&](double t) {
        if (positions.empty() || t < positions.front() || t >= positions.back()) return 0.0;
        size_t i = 0;
        while (i + 1 < positions.size() && t >= positions[i + 1]) ++i;
        return eval_local(i, t - positions[i]);
    };
    double amp = 0.0;
    for (size_t i = 0; i + 1 < positions.size(); ++i)
        for (int s = 0; s <= 32; ++s) {
            const double t = positions[i] + (positions[i + 1] - positions[i]) * s / 32.0;
            amp = std::max(amp, std::abs(evaluate(t)));
        }
    return amp;
}

// ---------------------------------------------------------------------------
namespace {
double median(std::vector<double> v) {  // quantize.hpp:118-122
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}
}  // namespace

// TransferFunction::validate (raycast.hpp:316-324)
void validate_tf(const sphray_tf_point* tf, size_t ntf) {
    if (ntf == 0 || !tf) fail(SPHRAY_ERR_CONFIG, "transfer function: no control points");
    for (size_t i = 0; i < ntf; ++i) {
        if (tf[i].absorption < 0.0)
            fail(SPHRAY_ERR_CONFIG, "transfer function: absorption must be nonnegative");
        if (i > 0 && !(tf[i].value > tf[i - 1].value))
            fail(SPHRAY_ERR_CONFIG, "transfer function: values must be strictly increasing");
    }
}

// dataset_stats, quantize.hpp:129-165.
sphray_dataset_stats dataset_stats(const sphray_particle* ps, size_t n, const LutHost& L,
                                   double clustering_factor) {
    if (n == 0) fail(SPHRAY_ERR_CONFIG, "dataset_stats: empty particle set");
    if (!(clustering_factor > 0.0))
        fail(SPHRAY_ERR_CONFIG, "dataset_stats: clustering factor must be positive");
    std::vector<double> mass(n), density(n), h(n), value(n);
    double phi_max = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const auto& p = ps[i];
        if (!(p.h > 0.0) || !(p.density > 0.0))
            fail(SPHRAY_ERR_CONFIG,
                 "dataset_stats: particles need positive smoothing radius and density");
        mass[i] = p.mass;
        density[i] = p.density;
        h[i] = p.h;
        value[i] = p.value;
        phi_max = std::max(phi_max, std::abs(p.mass * p.value / (p.density * p.h * p.h * p.h)));
    }
    sphray_dataset_stats s{};
    s.mass_r = median(std::move(mass));
    s.density_r = median(std::move(density));
    s.h_r = median(std::move(h));
    s.value_r = median(std::move(value));
    s.phi_repr = s.mass_r * s.value_r / (s.density_r * s.h_r * s.h_r * s.h_r);
    s.clustering_factor = clustering_factor;
    s.count = n;
    double amp = 0.0;
    for (int e = 0; e < L.N; ++e) amp = std::max(amp, entry_amplitude(L, e));
    s.a_max = clustering_factor * phi_max * amp;
    return s;
}

// quantization_error_slope / optimal_tau / choose_quanta, quantize.hpp:55-183.
namespace {
double order_weight(double q, int d) {
    return 2.0 * std::pow(q, 2 * d + 3) / ((2 * d + 1) * (2 * d + 3));
}
}  // namespace

double overall_error(const LutHost& L, double kappa) {
    if (kappa <= 0.0) return 0.0;
    const double dl = L.delta_lambda;
    double acc = 0.0;
    for (int e = 0; e < L.N; ++e) acc += L.lambda[e] * L.error[e] * L.error[e] * dl;
    return std::sqrt(2.0 * std::numbers::pi * acc) / kappa;
}

double quantization_error(const LutHost& L, double kappa, double kappa_prime, double tau, double sigma) {
    if (!(tau > 0.0)) fail(SPHRAY_ERR_CONFIG, "quantization_error: tau must be positive");
    if (!(sigma >= 0.0)) fail(SPHRAY_ERR_CONFIG, "quantization_error: sigma must be nonnegative");
    double s = kappa_prime * kappa_prime * tau * tau;
    for (int d = 0; d <= L.D; ++d) s += order_weight(L.q, d) * sigma * sigma / std::pow(tau, 2 * d);
    return std::sqrt(s) / (4.0 * kappa);
}

namespace {
double slope(int D, double kappa, double kappa_prime, double q, double tau, double sigma) {
    double s = 2.0 * kappa_prime * kappa_prime * tau;
    for (int d = 1; d <= D; ++d)
        s -= 2.0 * d * order_weight(q, d) * sigma * sigma / std::pow(tau, 2 * d + 1);
    return s / (16.0 * kappa * kappa);
}
double optimal_tau(int D, double kappa, double kappa_prime, double q, double sigma) {
    if (!(sigma > 0.0))
        fail(SPHRAY_ERR_CONFIG,
             "optimal_tau: sigma must be positive (a zero value quantum drives tau to zero)");
    double lo = 1e-12, hi = 1e12;
    while (slope(D, kappa, kappa_prime, q, lo, sigma) > 0.0 && lo > 1e-300) lo *= 1e-3;
    while (slope(D, kappa, kappa_prime, q, hi, sigma) < 0.0 && hi < 1e300) hi *= 1e3;
    for (int it = 0; it < 300 && hi > lo * (1.0 + 1e-15); ++it) {
        const double mid = std::sqrt(lo * hi);
        if (slope(D, kappa, kappa_prime, q, mid, sigma) > 0.0)
            hi = mid;
        else
            lo = mid;
    }
    return std::sqrt(lo * hi);
}
}  // namespace

sphray_quanta choose_quanta(const LutHost& L, const sphray_dataset_stats& ds, int width,
                            double kappa, double kappa_prime) {
    if (width != 32 && width != 64 && width != 128)
        fail(SPHRAY_ERR_CONFIG, "int width must be one of 32, 64, 128");
    if (!(ds.a_max > 0.0)) fail(SPHRAY_ERR_CONFIG, "choose_quanta: a_max must be positive");
    if (!(ds.phi_repr > 0.0))
        fail(SPHRAY_ERR_CONFIG,
             "choose_quanta: representative contribution factor must be positive");
    if (!(ds.h_r > 0.0))
        fail(SPHRAY_ERR_CONFIG, "choose_quanta: representative smoothing radius must be positive");
    sphray_quanta qc{};
    qc.int_width = width;
    qc.sigma = ds.a_max / (std::ldexp(1.0, width - 1) - 1.0);  // int_max_double, int_ops.hpp:45
    qc.tau = optimal_tau(L.D, kappa, kappa_prime, L.q, qc.sigma / ds.phi_repr) * ds.h_r;
    return qc;
}

void particle_powers(const sphray_particle* ps, size_t n, int D, double* out) {
    parallel_chunks(n, [&](size_t lo, size_t hi) {
        double last_h = std::nan(""), last[kMaxDegree] = {};
        for (size_t i = lo; i < hi; ++i) {
            const double h = ps[i].h;
            if (!(h == last_h)) {
                for (int d = 1; d <= D; ++d) last[d - 1] = std::pow(h, d + 3);  // quantize.hpp:222
                last_h = h;
            }
            for (int d = 0; d < D; ++d) out[i * D + d] = last[d];
        }
    });
}

void particle_powers_bbox(const sphray_particle* ps, size_t n, int D, double* out, double lo[3],
                          double hi[3]) {
    lo[0] = hi[0] = ps[0].x;
    lo[1] = hi[1] = ps[0].y;
    lo[2] = hi[2] = ps[0].z;
    std::mutex mu;
    parallel_chunks(n, [&](size_t b, size_t e) {
        double last_h = std::nan(""), last[kMaxDegree] = {};
        double l[3] = {ps[b].x, ps[b].y, ps[b].z}, u[3] = {ps[b].x, ps[b].y, ps[b].z};
        for (size_t i = b; i < e; ++i) {
            const sphray_particle& p = ps[i];
            if (!(p.h == last_h)) {
                for (int d = 1; d <= D; ++d) last[d - 1] = std::pow(p.h, d + 3);  // quantize.hpp:222
                last_h = p.h;
            }
            for (int d = 0; d < D; ++d) out[i * D + d] = last[d];
            l[0] = std::min(l[0], p.x);
            l[1] = std::min(l[1], p.y);
            l[2] = std::min(l[2], p.z);
            u[0] = std::max(u[0], p.x);
            u[1] = std::max(u[1], p.y);
            u[2] = std::max(u[2], p.z);
        }
        std::lock_guard<std::mutex> g(mu);
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], l[a]);
            hi[a] = std::max(hi[a], u[a]);
        }
    });
}

// ---------------------------------------------------------------------------
// Synthetic scenes: include/sphray_scenes.hpp, shared with the
// reference-side harness so both arms draw byte-identical particles.
size_t scene_default_count(int config) { return sphray_scenes::default_count(config); }

void generate_scene(int config, size_t n, uint64_t seed, sphray_particle* out) {
    static_assert(sizeof(sphray_scenes::Record) == sizeof(sphray_particle), "record layout");
    if (sphray_scenes::default_count(config) == 0)
        fail(SPHRAY_ERR_CONFIG, "unknown scene config " + std::to_string(config));
    sphray_scenes::generate(config, n, seed, reinterpret_cast<sphray_scenes::Record*>(out));
}

}  // namespace sphray_b200

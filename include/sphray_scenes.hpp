// sphray_scenes.hpp -- the synthetic SPH scenes of BASELINE.json configs 1-5
// (SURVEY.md 8(d)), header-only so the B200 library (sphray_generate_scene)
// and the reference-side harness (oracle/_ref, the CPU baseline arm) draw
// byte-identical particle sets without linking one another.
//
//   config 1: 1e5-particle Gaussian blob, uniform h = 0.062
//   config 2: 1M blob, h = 0.029          config 4: 4M blob, h = 0.062 (1e5/n)^(1/3)
//   config 3: 16M clustered (256 Plummer halos + 10% uniform background in
//             [-3,3]^3), h = 1.2 (m / rho_model)^(1/3) from the analytic mixture
//   config 5: the config-3 generator at 100M
//
// Records are {x, y, z, mass, density, h, value} doubles (sphray::Particle,
// quantize.hpp:16-27).  std::mt19937_64 + libstdc++ distributions: the bytes
// depend only on (config, n, seed) and the standard library.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace sphray_scenes {

struct Record {
    double x, y, z, mass, density, h, value;
};

inline std::size_t default_count(int config) {
    switch (config) {
        case 1: return 100000;
        case 2: return 1000000;
        case 3: return 16777216;
        case 4: return 4194304;
        case 5: return 100000000;
    }
    return 0;
}

inline std::uint64_t default_seed(int config) { return (config == 3 || config == 5) ? 7 : 42; }

template <class F>
void for_chunks(std::size_t n, F&& fn) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t T = std::max<std::size_t>(1, std::min<std::size_t>(hw, (n + 65535) / 65536));
    if (T <= 1) {
        fn(std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const std::size_t chunk = (n + T - 1) / T;
    for (std::size_t t = 0; t < T; ++t) {
        const std::size_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

// Gaussian blob: chi ~ N(0, I3), mass 1/n, rho = exp(-|chi|^2/2) + 0.05, value = rho.
inline void blob(std::size_t n, std::uint64_t seed, double h, Record* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    const double mass = 1.0 / static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) {
        const double x = nd(rng), y = nd(rng), z = nd(rng);
        const double rho = std::exp(-(x * x + y * y + z * z) / 2.0) + 0.05;
        out[i] = {x, y, z, mass, rho, h, rho};
    }
}

// 256 Plummer halos (centres ~ 0.9 N(0, I3) inside |.| <= 2.5, scale radii
// log-uniform in [0.02, 0.3], Pareto(1.5) masses capped at 100) carrying 90% of
// the particles, plus a 10% uniform background in [-3,3]^3; density and value
// are the analytic mixture density, h = 1.2 (m / rho)^(1/3).
inline void clustered(std::size_t n, std::uint64_t seed, Record* out) {
    constexpr int kHalos = 256;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> nd(0.0, 1.0);
    double cx[kHalos], cy[kHalos], cz[kHalos], a[kHalos], w[kHalos];
    double wsum = 0.0;
    for (int i = 0; i < kHalos; ++i) {
        do {
            cx[i] = 0.9 * nd(rng);
            cy[i] = 0.9 * nd(rng);
            cz[i] = 0.9 * nd(rng);
        } while (std::fabs(cx[i]) > 2.5 || std::fabs(cy[i]) > 2.5 || std::fabs(cz[i]) > 2.5);
        a[i] = std::exp(std::log(0.02) + (std::log(0.3) - std::log(0.02)) * U(rng));
        w[i] = std::min(100.0, std::pow(1.0 - U(rng), -1.0 / 1.5));
        wsum += w[i];
    }
    for (int i = 0; i < kHalos; ++i) w[i] = 0.9 * w[i] / wsum;
    const double mass = 1.0 / static_cast<double>(n);
    std::size_t k = 0;
    for (int i = 0; i < kHalos && k < n; ++i) {
        const std::size_t cnt = std::min(n - k, static_cast<std::size_t>(w[i] * static_cast<double>(n)));
        for (std::size_t j = 0; j < cnt; ++j, ++k) {
            double r;
            do {
                const double u = std::max(U(rng), 1e-300);
                r = a[i] / std::sqrt(std::pow(u, -2.0 / 3.0) - 1.0);
            } while (!(r < 15.0 * a[i]));
            const double ct = 2.0 * U(rng) - 1.0, ph = 2.0 * std::numbers::pi * U(rng);
            const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
            out[k] = {cx[i] + r * st * std::cos(ph), cy[i] + r * st * std::sin(ph), cz[i] + r * ct,
                      mass, 0.0, 0.0, 0.0};
        }
    }
    for (; k < n; ++k)
        out[k] = {-3.0 + 6.0 * U(rng), -3.0 + 6.0 * U(rng), -3.0 + 6.0 * U(rng), mass, 0.0, 0.0, 0.0};
    double norm[kHalos];
    for (int i = 0; i < kHalos; ++i) norm[i] = w[i] * 3.0 / (4.0 * std::numbers::pi * a[i] * a[i] * a[i]);
    const double bg = 0.1 / 216.0;
    for_chunks(n, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t p = lo; p < hi; ++p) {
            double rho = bg;
            for (int i = 0; i < kHalos; ++i) {
                const double dx = out[p].x - cx[i], dy = out[p].y - cy[i], dz = out[p].z - cz[i];
                const double s = 1.0 + (dx * dx + dy * dy + dz * dz) / (a[i] * a[i]);
                rho += norm[i] / (s * s * std::sqrt(s));
            }
            out[p].density = rho;
            out[p].value = rho;
            out[p].h = 1.2 * std::cbrt(mass / rho);
        }
    });
}

// Throws std::invalid_argument for an unknown config.
inline void generate(int config, std::size_t n, std::uint64_t seed, Record* out) {
    switch (config) {
        case 1: blob(n, seed, n == 100000 ? 0.062 : 0.062 * std::cbrt(1e5 / n), out); return;
        case 2: blob(n, seed, n == 1000000 ? 0.029 : 0.062 * std::cbrt(1e5 / n), out); return;
        case 4: blob(n, seed, 0.062 * std::cbrt(1e5 / n), out); return;
        case 3:
        case 5: clustered(n, seed, out); return;
    }
    throw std::invalid_argument("unknown scene config " + std::to_string(config));
}

}  // namespace sphray_scenes

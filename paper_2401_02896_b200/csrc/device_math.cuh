// device_math.cuh -- exact fp64 / int64 building blocks of the path.
//
// Bit-exact parity with the reference (x86-64 SSE2, -O2, no FMA) needs every
// fp64 operation in the reference's order with no contraction: the
// __d{add,sub,mul,div,sqrt}_rn intrinsics are IEEE round-to-nearest and are
// never fused by nvcc.  libm calls that are not correctly rounded (tan, pow)
// are evaluated on the host with glibc (host.cpp) and passed in.
#pragma once

#include <cstdint>

#include "host.hpp"

namespace sphray_b200 {
namespace dev {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// Camera::ray_at (raycast.hpp:81-100).
struct RayD {
    double ox, oy, oz, dx, dy, dz;
};

__device__ __forceinline__ RayD make_ray(const CamConst& c, int px, int py) {
    const double u = dsub(dmul(ddiv(dadd(static_cast<double>(px), 0.5), static_cast<double>(c.W)), 2.0), 1.0);
    const double v = dsub(1.0, dmul(ddiv(dadd(static_cast<double>(py), 0.5), static_cast<double>(c.H)), 2.0));
    RayD r;
    if (c.mode == 0) {
        const double su = dmul(u, c.hw), sv = dmul(v, c.hh);
        r.ox = dadd(dadd(c.pos[0], dmul(c.right[0], su)), dmul(c.upv[0], sv));
        r.oy = dadd(dadd(c.pos[1], dmul(c.right[1], su)), dmul(c.upv[1], sv));
        r.oz = dadd(dadd(c.pos[2], dmul(c.right[2], su)), dmul(c.upv[2], sv));
        r.dx = c.fwd[0];
        r.dy = c.fwd[1];
        r.dz = c.fwd[2];
    } else {
        const double s1 = dmul(dmul(u, c.th), c.aspect), s2 = dmul(v, c.th);
        const double wx = dadd(dadd(c.fwd[0], dmul(c.right[0], s1)), dmul(c.upv[0], s2));
        const double wy = dadd(dadd(c.fwd[1], dmul(c.right[1], s1)), dmul(c.upv[1], s2));
        const double wz = dadd(dadd(c.fwd[2], dmul(c.right[2], s1)), dmul(c.upv[2], s2));
        const double n = dsqrt(dadd(dadd(dmul(wx, wx), dmul(wy, wy)), dmul(wz, wz)));
        const double inv = ddiv(1.0, n);
        r.ox = c.pos[0];
        r.oy = c.pos[1];
        r.oz = c.pos[2];
        r.dx = dmul(wx, inv);
        r.dy = dmul(wy, inv);
        r.dz = dmul(wz, inv);
    }
    return r;
}

// detail::hit_ray (raycast.hpp:111-120): the hit predicate, bit for bit.
__device__ __forceinline__ bool hit_ray(const RayD& r, double cx, double cy, double cz,
                                        double support, double h, double near_plane,
                                        double far_plane, double& lam, double& t_chi) {
    const double ocx = dsub(cx, r.ox), ocy = dsub(cy, r.oy), ocz = dsub(cz, r.oz);
    const double t = dadd(dadd(dmul(ocx, r.dx), dmul(ocy, r.dy)), dmul(ocz, r.dz));
    const double d2 =
        dsub(dadd(dadd(dmul(ocx, ocx), dmul(ocy, ocy)), dmul(ocz, ocz)), dmul(t, t));
    if (!(d2 < dmul(support, support))) return false;
    if (dadd(t, support) <= near_plane || dsub(t, support) >= far_plane) return false;
    lam = ddiv(dsqrt(d2 < 0.0 ? 0.0 : d2), h);  // std::max(d2, 0.0) keeps -0.0
    t_chi = t;
    return true;
}

// hit_ray split in two for the render kernel: the predicate returns d2 and
// t_chi; lam_of(d2, h) is the RayHit::lam of the same hit, computed later
// (per queued hit, not per tested candidate).  No early exits: the gather
// evaluates it on every lane and masks the result.
__device__ __forceinline__ bool hit_test(const RayD& r, double cx, double cy, double cz,
                                         double support, double near_plane, double far_plane,
                                         double& d2_out, double& t_chi) {
    const double ocx = dsub(cx, r.ox), ocy = dsub(cy, r.oy), ocz = dsub(cz, r.oz);
    const double t = dadd(dadd(dmul(ocx, r.dx), dmul(ocy, r.dy)), dmul(ocz, r.dz));
    const double d2 =
        dsub(dadd(dadd(dmul(ocx, ocx), dmul(ocy, ocy)), dmul(ocz, ocz)), dmul(t, t));
    d2_out = d2;
    t_chi = t;
    return (d2 < dmul(support, support)) & !(dadd(t, support) <= near_plane) &
           !(dsub(t, support) >= far_plane);
}
__device__ __forceinline__ double lam_of(double d2, double h) {
    return ddiv(dsqrt(d2 < 0.0 ? 0.0 : d2), h);
}

// Conservative pixel bbox of particle_ray_footprint (raycast.hpp:134-176).
// Returns px0,px1,py0,py1 already clipped to the image (empty if px0 > px1).
__device__ __forceinline__ int clamp_int(double v) {
    // static_cast<int> of an in-range double; out-of-range values cannot
    // reach a pixel either way, saturate them well inside int range.
    if (!(v > -1.0e9)) return -1000000000;
    if (!(v < 1.0e9)) return 1000000000;
    return static_cast<int>(v);
}

__device__ __forceinline__ void footprint_bbox(const CamConst& c, double x, double y, double z,
                                               double support, int& px0, int& px1, int& py0,
                                               int& py1) {
    px0 = 0;
    px1 = c.W - 1;
    py0 = 0;
    py1 = c.H - 1;
    const double rx = dsub(x, c.pos[0]), ry = dsub(y, c.pos[1]), rz = dsub(z, c.pos[2]);
    const double W = static_cast<double>(c.W), H = static_cast<double>(c.H);
    if (c.mode == 0) {
        const double cx = dadd(dadd(dmul(rx, c.right[0]), dmul(ry, c.right[1])), dmul(rz, c.right[2]));
        const double cy = dadd(dadd(dmul(rx, c.upv[0]), dmul(ry, c.upv[1])), dmul(rz, c.upv[2]));
        px0 = max(px0, clamp_int(floor(dsub(dmul(ddiv(dadd(dsub(cx, support), c.hw), c.two_hw), W), 0.5))) - 1);
        px1 = min(px1, clamp_int(ceil(dsub(dmul(ddiv(dadd(dadd(cx, support), c.hw), c.two_hw), W), 0.5))) + 1);
        py0 = max(py0, clamp_int(floor(dsub(dmul(ddiv(dsub(c.hh, dadd(cy, support)), c.two_hh), H), 0.5))) - 1);
        py1 = min(py1, clamp_int(ceil(dsub(dmul(ddiv(dsub(c.hh, dsub(cy, support)), c.two_hh), H), 0.5))) + 1);
    } else {
        const double depth = dadd(dadd(dmul(rx, c.fwd[0]), dmul(ry, c.fwd[1])), dmul(rz, c.fwd[2]));
        if (dsub(depth, support) > 0.0) {
            const double zmin = dsub(depth, support), zmax = dadd(depth, support);
            const double cx = dadd(dadd(dmul(rx, c.right[0]), dmul(ry, c.right[1])), dmul(rz, c.right[2]));
            const double cy = dadd(dadd(dmul(rx, c.upv[0]), dmul(ry, c.upv[1])), dmul(rz, c.upv[2]));
            auto ratio_lo = [&](double cc) {
                const double num = dsub(cc, support);
                return ddiv(num, num <= 0.0 ? zmin : zmax);
            };
            auto ratio_hi = [&](double cc) {
                const double num = dadd(cc, support);
                return ddiv(num, num >= 0.0 ? zmin : zmax);
            };
            const double u_lo = ddiv(ratio_lo(cx), c.th_aspect);
            const double u_hi = ddiv(ratio_hi(cx), c.th_aspect);
            const double v_lo = ddiv(ratio_lo(cy), c.th);
            const double v_hi = ddiv(ratio_hi(cy), c.th);
            px0 = max(px0, clamp_int(floor(dsub(dmul(dmul(dadd(u_lo, 1.0), 0.5), W), 0.5))) - 1);
            px1 = min(px1, clamp_int(ceil(dsub(dmul(dmul(dadd(u_hi, 1.0), 0.5), W), 0.5))) + 1);
            py0 = max(py0, clamp_int(floor(dsub(dmul(dmul(dsub(1.0, v_hi), 0.5), H), 0.5))) - 1);
            py1 = min(py1, clamp_int(ceil(dsub(dmul(dmul(dsub(1.0, v_lo), 0.5), H), 0.5))) + 1);
        }
    }
    px0 = max(px0, 0);
    py0 = max(py0, 0);
    px1 = min(px1, c.W - 1);
    py1 = min(py1, c.H - 1);
}

// Lower bound of the ray parameter of every knot this particle can emit on
// any ray that hits it (used only to schedule the per-ray knot window; any
// conservative bound is correct, a tighter one just flushes earlier).
__device__ __forceinline__ double front_bound(const CamConst& c, double x, double y, double z,
                                              double support, double reach) {
    const double rx = x - c.pos[0], ry = y - c.pos[1], rz = z - c.pos[2];
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double rn = sqrt(r2);
    double tlo;
    if (c.mode == 0) {
        const double depth = rx * c.fwd[0] + ry * c.fwd[1] + rz * c.fwd[2];
        const double slack = 1e-9 * (rn + fabs(c.pos[0]) + fabs(c.pos[1]) + fabs(c.pos[2]) +
                                     c.hw + c.hh + fabs(x) + fabs(y) + fabs(z) + 1e-300);
        tlo = depth - slack;
    } else {
        const double depth = rx * c.fwd[0] + ry * c.fwd[1] + rz * c.fwd[2];
        if (depth - support * (1.0 + 1e-9) > 0.0) {
            const double s2 = support * support;
            const double e = r2 - s2 - 1e-9 * r2;
            tlo = (e > 0.0 ? sqrt(e) : 0.0) - 1e-9 * (rn + 1e-300);
        } else {
            tlo = fmax(c.near_plane - support, -rn) - 1e-9 * (rn + fabs(c.near_plane) + support + 1e-300);
        }
    }
    const double f = tlo - reach;
    return f - 1e-9 * fabs(f);
}

// Lut::lookup (lut.hpp:43-52) for lam < q (quantize_particle returns before
// the zero entry: quantize.hpp:204).
static __device__ __noinline__ double div_exact(double a, double b) { return ddiv(a, b); }

// inv_dl = recip_or_nan(dl): x = lam/dl is taken as lam*inv_dl when that is
// farther than |x| 2^-50 from every integer (then floor and the tie test
// agree with the correctly rounded quotient), else divided exactly.
__device__ __forceinline__ int lut_index(double lam, double dl, double inv_dl, int N) {
    double x = lam * inv_dl;
    {
        const double f = floor(x);
        const double mg = fabs(x) * 0x1p-50;
        if (!(x - f > mg && (f + 1.0) - x > mg && fabs(x) < 0x1p49)) x = div_exact(lam, dl);
    }
    double i = floor(x);
    if (i == x && i > 0.0) i = dsub(i, 1.0);
    const double c = (i < 0.0) ? 0.0 : i;
    const long long idx = static_cast<long long>(c);
    return static_cast<int>(idx < N - 1 ? idx : N - 1);
}

// Checked<int64_t> (int_ops.hpp:63-99): the reference throws on overflow; the
// device keeps the wrapped value and raises a flag that aborts the render
// with OverflowError, naming the particle and ray like quantize.hpp:244-249.
__device__ __forceinline__ int64_t cadd(int64_t a, int64_t b, bool& o) {
    const int64_t r = static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
    o |= ((a ^ r) & (b ^ r)) < 0;
    return r;
}
__device__ __forceinline__ int64_t csub(int64_t a, int64_t b, bool& o) {
    const int64_t r = static_cast<int64_t>(static_cast<uint64_t>(a) - static_cast<uint64_t>(b));
    o |= ((a ^ b) & (a ^ r)) < 0;
    return r;
}
__device__ __forceinline__ int64_t cmul(int64_t a, int64_t b, bool& o) {
    const int64_t lo = static_cast<int64_t>(static_cast<uint64_t>(a) * static_cast<uint64_t>(b));
    const int64_t hi = __mul64hi(a, b);
    o |= hi != (lo >> 63);
    return lo;
}
__device__ __forceinline__ int64_t cneg(int64_t a, bool& o) {
    o |= a == INT64_MIN;
    return static_cast<int64_t>(0ull - static_cast<uint64_t>(a));
}

// Checked<int32_t> (int_ops.hpp:63-99) on top of the int64 arithmetic: every
// int32 operation's operands fit int32, so its exact result is the int64 one;
// `on` flags any result outside int32 (round_to_int<int32_t>'s range check is
// the same test).
__device__ __forceinline__ int64_t narrow32(int64_t v, bool on, bool& o) {
    if (on) o |= v != static_cast<int64_t>(static_cast<int32_t>(v));
    return v;
}

// round_to_int<int64_t> (int_ops.hpp:103-110): nearbyint (ties to even),
// then the range check [-2^63, 2^63).
__device__ __forceinline__ int64_t round_checked(double x, bool& o) {
    const double r = rint(x);
    const bool ok = r >= -9223372036854775808.0 && r < 9223372036854775808.0;
    o |= !ok;
    return ok ? __double2ll_rn(r) : 0;
}

// Correctly rounded reciprocal for the division fast paths below, or NaN
// (forcing the exact path) when it is not a normal number.
__host__ __device__ inline double recip_or_nan(double b) {
    const double y = 1.0 / b;
    const double ay = y < 0.0 ? -y : y;
    return (ay >= 0x1p-1000 && ay <= 0x1p1000) ? y : __builtin_nan("");
}

struct RintQ {
    int64_t v;
    bool ovf;
};
// Exact path, out of line: one copy of the division code for every call site.
static __device__ __noinline__ RintQ rint_div_exact(double a, double b) {
    bool o = false;
    const int64_t v = round_checked(ddiv(a, b), o);
    return {v, o};
}

// round_to_int(a / b) with the quotient correctly rounded as the reference
// computes it, from y = recip_or_nan(b).  q = a*y is within |q| 2^-51 of
// RN(a/b) (two roundings of relative size 2^-53); when q is farther than
// |q| 2^-50 from every half-integer, rint(q) == rint(RN(a/b)).  Otherwise
// (and for |q| >= 2^49, NaN, inf) the exact division decides.
__device__ __forceinline__ int64_t rint_div(double a, double b, double y, bool& o) {
    const double q = a * y;
    const double r = rint(q);
    const double aq = fabs(q);
    if (aq < 0x1p49 && fabs(q - r) < 0.5 - aq * 0x1p-50) return static_cast<int64_t>(r);
    const RintQ e = rint_div_exact(a, b);
    o |= e.ovf;
    return e.v;
}

// Taylor shift p(y) -> p(y + delta) modulo 2^64 (repeated Horner).  This is
// S(delta) of SURVEY.md 0.6: (S v)_d = sum_{j>=d} C(j,d) v_j delta^(j-d).
template <int D>
__device__ __forceinline__ void taylor_shift(uint64_t (&v)[D + 1], uint64_t delta) {
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) v[j] += delta * v[j + 1];
}

// The same for a delta below 2^32 (two positions of one flush window): the
// zero upper word saves one of the three IMADs of every 64-bit product.
template <int D>
__device__ __forceinline__ void taylor_shift(uint64_t (&v)[D + 1], uint32_t delta) {
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) v[j] += static_cast<uint64_t>(delta) * v[j + 1];
}

// The same modulo 2^128 (render_scene<Int128>, int_width 128); delta is a
// wrapped int64 position difference, sign-extended.
template <int D>
__device__ __forceinline__ void taylor_shift(unsigned __int128 (&v)[D + 1], uint64_t delta) {
    const unsigned __int128 dl =
        static_cast<unsigned __int128>(static_cast<__int128>(static_cast<int64_t>(delta)));
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) v[j] += dl * v[j + 1];
}

// ---------------------------------------------------------------------------
// Checked<Int128> (int_ops.hpp:63-99): wrapping __int128 arithmetic plus an
// overflow flag, for int_width 128 (quantize.hpp:199-250 with Int = Int128).
using i128 = __int128;
using u128 = unsigned __int128;
constexpr i128 kI128Min = static_cast<i128>(static_cast<u128>(1) << 127);

__device__ __forceinline__ i128 cadd(i128 a, i128 b, bool& o) {
    const i128 r = static_cast<i128>(static_cast<u128>(a) + static_cast<u128>(b));
    o |= ((a ^ r) & (b ^ r)) < 0;
    return r;
}
__device__ __forceinline__ i128 csub(i128 a, i128 b, bool& o) {
    const i128 r = static_cast<i128>(static_cast<u128>(a) - static_cast<u128>(b));
    o |= ((a ^ b) & (a ^ r)) < 0;
    return r;
}
__device__ __forceinline__ i128 cneg(i128 a, bool& o) {
    o |= a == kI128Min;
    return static_cast<i128>(static_cast<u128>(0) - static_cast<u128>(a));
}
// a * b, exact or flagged: magnitudes split in 64-bit limbs
__device__ __forceinline__ i128 cmul(i128 a, i128 b, bool& o) {
    const bool neg = (a < 0) != (b < 0);
    const u128 ua = a < 0 ? static_cast<u128>(0) - static_cast<u128>(a) : static_cast<u128>(a);
    const u128 ub = b < 0 ? static_cast<u128>(0) - static_cast<u128>(b) : static_cast<u128>(b);
    const uint64_t ah = static_cast<uint64_t>(ua >> 64), al = static_cast<uint64_t>(ua);
    const uint64_t bh = static_cast<uint64_t>(ub >> 64), bl = static_cast<uint64_t>(ub);
    bool big = ah != 0 && bh != 0;
    const u128 cross = static_cast<u128>(ah) * bl + static_cast<u128>(al) * bh;  // < 2^128 when !big
    big |= (cross >> 64) != 0;
    const u128 lo = static_cast<u128>(al) * bl;
    const u128 mag = lo + (cross << 64);
    big |= mag < lo;
    big |= neg ? mag > (static_cast<u128>(1) << 127) : (mag >> 127) != 0;
    o |= big;
    return static_cast<i128>(neg ? static_cast<u128>(0) - mag : mag);
}
__device__ __forceinline__ i128 cmul_binom(i128 a, long long c, bool& o) {
    if (c == 1) return a;
    return cmul(a, static_cast<i128>(c), o);
}
// round_to_int<Int128> (int_ops.hpp:103-110): nearbyint, range [-2^127, 2^127)
__device__ __forceinline__ i128 round_checked128(double x, bool& o) {
    const double r = rint(x);
    const bool ok = r >= -0x1p127 && r < 0x1p127;
    o |= !ok;
    return ok ? static_cast<i128>(r) : 0;
}
static __device__ __noinline__ i128 rint_div128_exact(double a, double b, bool* o) {
    bool f = false;
    const i128 v = round_checked128(ddiv(a, b), f);
    *o |= f;
    return v;
}
// round_to_int<Int128>(a / b) with the quotient rounded as the reference does
__device__ __forceinline__ i128 rint_div128(double a, double b, double y, bool& o) {
    const double q = a * y;
    const double r = rint(q);
    const double aq = fabs(q);
    if (aq < 0x1p49 && fabs(q - r) < 0.5 - aq * 0x1p-50) return static_cast<i128>(static_cast<int64_t>(r));
    return rint_div128_exact(a, b, &o);
}

}  // namespace dev
}  // namespace sphray_b200

// render_kernel.cuh -- the per-ray render kernel (warp per ray) and the
// explicit-hit quantization kernel, as templates over (D, m).  Each
// render_d<D>.cu instantiates them for one degree so the 24 (D, m) variants
// compile in parallel.  See render.cu for the reference mapping.
//
// Per-ray knot window (shared memory, one per warp):
//   pt     cap u32: knot position as an offset from the ray's base tb (the
//          first flush bound: every knot of the ray is >= it)
//   pool   D x cap u64: the knot's jumps of orders 1..D (order 0 is
//          structurally zero)
//   ps     pending knots (slot ids), UNSORTED: inserting a batch is an append
//   fl     free-slot stack [0, nfree); directly above it, during a flush, the
//          flush set fs = fl + nfree: pending knots with t < F, selected by a
//          ballot scan and sorted (warp LSD radix) only when they are final;
//          once merged they are free slots already (nfree += nsel)
//   open   the last piece (t, a_0..a_D), whose end is the first knot of the
//          next flush set
#pragma once

#include <cuda_runtime.h>

#include "device_math.cuh"
#include "quantize.cuh"
#include "render.cuh"

#ifndef SPHRAY_GATHER_TO
#define SPHRAY_GATHER_TO 32  // hits queued before an insert/flush step (<= kHitQueue)
#endif
#ifndef SPHRAY_INSERT_ROUNDS
#define SPHRAY_INSERT_ROUNDS 1  // 32-hit insert rounds per step
#endif
#ifndef SPHRAY_FLUSH_AT
#define SPHRAY_FLUSH_AT 4  // flush once the pending list holds SPHRAY_FLUSH_AT/8 of the window
#endif
#ifndef SPHRAY_KSTATS
#define SPHRAY_KSTATS 0
#endif
// diagnostic work counters (render.cuh StatIndex), compiled out by default
#define SPHRAY_KS(idx, v)                                                            \
    do {                                                                             \
        if (SPHRAY_KSTATS && lane == 0)                                              \
            atomicAdd(&P.stats[idx], static_cast<unsigned long long>(v));            \
    } while (0)
#ifndef SPHRAY_COLD_OUTLINE
#define SPHRAY_COLD_OUTLINE 1  // rarely executed code out of line (the kernel is instruction-cache bound)
#endif
#ifndef SPHRAY_MAXNREG
#define SPHRAY_MAXNREG 168
#endif

namespace sphray_b200 {
namespace rk {

using namespace dev;

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// floor(front / tau) - 2: every knot of a not-yet-inserted candidate has
// t >= this (front is a conservative bound, see dev::front_bound).
__device__ __forceinline__ int64_t knot_floor(float front, double inv_tau) {
    // a multiply by 1/tau (relative error ~2^-52) instead of the division:
    // the bound only has to stay below the knots, one more unit of slack
    // covers the rounding for |v| < 2^52
    const double v = floor(static_cast<double>(front) * inv_tau) - 3.0;
    if (!(v > -9.2e18)) return INT64_MIN;
    if (!(v < 9.2e18)) return INT64_MAX;
    return static_cast<int64_t>(v);
}

// TransferFunction::sample (raycast.hpp:326-337).  The device TF holds
// kTfPoint doubles per point: value, r, g, b, absorption and the four slopes
// to the next point, so the interpolation is one fma per channel,
// c_a + (v - value_a) * slope_a (within a few ulps of the reference's
// c_a + t (c_b - c_a); inside the RGB tolerance).  Clamping uses w = 0,
// which reproduces the end point exactly.
constexpr int kTfStride = kTfPoint;

// TF readers: the per-CTA shared copy (ld.shared) or global memory; a point's
// 10 doubles are 16-byte aligned, read in pairs (value, r) (g, b) (ab, sr)
// (sg, sb) (sab, pad).
struct TfShared {
    uint32_t base;
    __device__ __forceinline__ double operator()(int k) const {
        double v;
        asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * static_cast<uint32_t>(k)));
        return v;
    }
    __device__ __forceinline__ double2 pair(int k) const {
        double2 v;
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(base + 8u * static_cast<uint32_t>(k)));
        return v;
    }
};
struct TfGlobal {
    const double* p;
    __device__ __forceinline__ double operator()(int k) const { return __ldg(p + k); }
    __device__ __forceinline__ double2 pair(int k) const {
        return __ldg(reinterpret_cast<const double2*>(p + k));
    }
};

template <class Ld>
__device__ __forceinline__ void tf_sample(const Ld& ld, int n, double v, double& r, double& g,
                                          double& b, double& ab) {
    const int last = kTfStride * (n - 1);
    const bool lo = v <= ld(0), hi = v >= ld(last);
    int a = 0;
    if (!lo && !hi) {  // the reference's linear search for the bracket (a branch-free
        int i = kTfStride;  // count measured 2.7% / 13% slower: the loop mostly exits at once)
        while (ld(i) < v) i += kTfStride;
        a = i - kTfStride;
    }
    if (hi) a = last;
    const double2 p0 = ld.pair(a), p1 = ld.pair(a + 2), p2 = ld.pair(a + 4), p3 = ld.pair(a + 6),
                  p4 = ld.pair(a + 8);
    const double w = (lo || hi) ? 0.0 : v - p0.x;
    r = fma(w, p2.y, p0.y);
    g = fma(w, p3.x, p1.x);
    b = fma(w, p3.y, p1.y);
    ab = fma(w, p4.x, p2.x);
}

// n = max(2, ceil((hi - lo) / step)) exactly as the reference counts samples
// (raycast.hpp:367): a multiply by 1/step, with the exact division only when
// the quotient is within rounding distance of an integer.
static __device__ __noinline__ int sample_count_long(double len, double step, double q) {
    double c = ceil(q);
    if (fabs(q - rint(q)) <= 1e-12 * q + 1e-300) c = ceil(div_exact(len, step));
    return c > 2.0 ? static_cast<int>(c) : 2;
}
__device__ __forceinline__ int sample_count(double len, double step, double inv_step) {
    const double q = len * inv_step;
    if (q < 1.9) return 2;  // len/step < 2 for sure: the common case
    if (SPHRAY_COLD_OUTLINE) return sample_count_long(len, step, q);
    double c = ceil(q);
    if (fabs(q - rint(q)) <= 1e-12 * q + 1e-300) c = ceil(div_exact(len, step));
    return c > 2.0 ? static_cast<int>(c) : 2;
}

// alpha = 1 - exp(-x) (raycast.hpp:372) in fp64: below 1/16 the Taylor series
// of 1 - e^-x to x^8 (truncation < x^9/9! < 2e-17 relative), else
// 1 - exp(-x) as the reference writes it (CUDA's exp is within 1 ulp of
// glibc's).  Either way alpha is within a few ulps of the reference's, so the
// early-termination test T <= 1e-3 sees the same transmittance to ~1e-15.
#ifndef SPHRAY_ALPHA_MODE
#define SPHRAY_ALPHA_MODE 0  // 0: fp64 (series + exp); 1: round-1 fp32 (diagnostics)
#endif
#ifndef SPHRAY_PF_L1
#define SPHRAY_PF_L1 1  // L1 prefetch of the candidate batch this many batches ahead (0: off)
#endif
#ifndef SPHRAY_SHIFT32
#define SPHRAY_SHIFT32 1  // in-window Taylor shifts with a 32-bit delta
#endif
#ifndef SPHRAY_OVF_CHECK
#define SPHRAY_OVF_CHECK 1  // genuine-overflow test of the merge (0: off, diagnostics only)
#endif
// alpha for x >= 2^-8: the series to x^6 below 1/16 (relative error < 7e-13),
// else 1 - exp(-x) as the reference writes it (CUDA's exp is within 1 ulp of
// glibc's; several hundred SASS instructions, hence out of line: at config 3
// nearly every sample takes the short series).
static __device__ __noinline__ double alpha_wide(double x) {
    if (x < 0.0625) {
        double s = 1.0 / 5040.0;
        s = fma(s, -x, 1.0 / 720.0);
        s = fma(s, -x, 1.0 / 120.0);
        s = fma(s, -x, 1.0 / 24.0);
        s = fma(s, -x, 1.0 / 6.0);
        s = fma(s, -x, 0.5);
        s = fma(s, -x, 1.0);
        return s * x;
    }
    return 1.0 - exp(-x);
}
static __device__ __noinline__ double one_minus_exp_neg_ool(double x) { return 1.0 - exp(-x); }
__device__ __forceinline__ double alpha_of(double x) {
    if (SPHRAY_ALPHA_MODE == 1) {
        if (x < 0.05) return x * (1.0 - x * (0.5 - x * (1.0 / 6.0 - x * (1.0 / 24.0))));
        return 1.0 - static_cast<double>(__expf(-static_cast<float>(x)));
    }
    if (x < 0x1p-8) {  // series to x^4 (relative error < x^5/6! < 1.2e-15)
        double s = 1.0 / 120.0;
        s = fma(s, -x, 1.0 / 24.0);
        s = fma(s, -x, 1.0 / 6.0);
        s = fma(s, -x, 0.5);
        s = fma(s, -x, 1.0);
        return s * x;
    }
    if (SPHRAY_COLD_OUTLINE == 2) return alpha_wide(x);
    if (x < 0.0625) {
        double s = 1.0 / 5040.0;
        s = fma(s, -x, 1.0 / 720.0);
        s = fma(s, -x, 1.0 / 120.0);
        s = fma(s, -x, 1.0 / 24.0);
        s = fma(s, -x, 1.0 / 6.0);
        s = fma(s, -x, 0.5);
        s = fma(s, -x, 1.0);
        return s * x;
    }
    if (SPHRAY_COLD_OUTLINE) return one_minus_exp_neg_ool(x);
    return 1.0 - exp(-x);
}

// sphray_piece_mix (include/sphray_gpu.h) of one FieldPiece, for the per-ray
// piece checksum of sphray_ray_record.
// The merge's integer: U = uint64_t (int_width 32 / 64) or unsigned __int128
// (int_width 128); SOf<U> is its signed twin.
template <class U>
using SOf = std::conditional_t<sizeof(U) == 16, __int128, int64_t>;

template <class U>
__device__ __forceinline__ U shfl_up_u(U v, int o) {
    if constexpr (sizeof(U) == 16) {
        const uint64_t lo = __shfl_up_sync(kFull, static_cast<unsigned long long>(v), o);
        const uint64_t hi = __shfl_up_sync(kFull, static_cast<unsigned long long>(v >> 64), o);
        return (static_cast<U>(hi) << 64) | lo;
    } else {
        return __shfl_up_sync(kFull, static_cast<unsigned long long>(v), o);
    }
}
template <class U>
__device__ __forceinline__ U shfl_idx_u(U v, int src) {
    if constexpr (sizeof(U) == 16) {
        const uint64_t lo = __shfl_sync(kFull, static_cast<unsigned long long>(v), src);
        const uint64_t hi = __shfl_sync(kFull, static_cast<unsigned long long>(v >> 64), src);
        return (static_cast<U>(hi) << 64) | lo;
    } else {
        return __shfl_sync(kFull, static_cast<unsigned long long>(v), src);
    }
}
template <class U>
__device__ __forceinline__ U warp_incl_scan_u(U v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const U u = shfl_up_u(v, o);
        if (lane >= o) v += u;
    }
    return v;
}
template <class U>
__device__ __forceinline__ double to_double(U a) {
    return static_cast<double>(static_cast<SOf<U>>(a));
}

template <int D, class U>
__device__ __forceinline__ uint64_t piece_mix(int64_t t, const U (&a)[D + 1]) {
    constexpr uint64_t M[8] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full, 0x165667B19E3779F9ull,
                               0x27D4EB2F165667C5ull, 0x94D049BB133111EBull, 0xBF58476D1CE4E5B9ull,
                               0xD6E8FEB86659FD93ull, 0xFF51AFD7ED558CCDull};
    uint64_t x = static_cast<uint64_t>(t) * M[0];
#pragma unroll
    for (int d = 0; d <= D; ++d) x += static_cast<uint64_t>(a[d]) * M[d + 1];  // low 64 bits
    x ^= x >> 31;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 29;
    return x;
}

// Genuine-overflow test of one Taylor shift (RayAccumulator::advance,
// raycast.hpp:232-249).  The merge runs modulo 2^64, which equals the exact
// (Int128) result whenever the exact coefficients fit int64.
// Given an exact input polynomial v (as doubles) and the wrapped result w of
// shifting it by delta, the exact result is predicted in fp64 (relative error
// ~2^-50 of the terms); |prediction - w| >= 2^62 means the exact coefficient
// left int64 -- the case where render_scene<int64_t> throws OverflowError and
// a wrapped merge would silently give a wrong field.  A non-finite prediction
// (astronomic terms) counts as overflow too.
// TOP = false skips order D: a Taylor shift leaves the top coefficient
// unchanged, so when v is the exact double image of the shifted state's own
// pre-shift integers (the walk), that order cannot differ.
template <int D, class U, bool TOP = true>
__device__ __forceinline__ bool shift_overflows(const double (&v)[D + 1], double delta,
                                                const U (&w)[D + 1]) {
    constexpr double kLim = sizeof(U) == 16 ? 0x1p126 : 0x1p62;
    if (!SPHRAY_OVF_CHECK) return false;
    double p[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) p[d] = v[d];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = D - 1; j >= i; --j) p[j] = fma(delta, p[j + 1], p[j]);
    bool bad = false;
#pragma unroll
    for (int d = 0; d <= (TOP ? D : D - 1); ++d)
        bad |= !(fabs(p[d] - to_double(w[d])) < kLim);
    return bad;
}

// a += j modulo 2^64 (2^128), flagging signed overflow (Checked<Int> +, int_ops.hpp:73-80)
template <class U>
__device__ __forceinline__ U add_checked(U a, U j, bool& o) {
    const U r = a + j;
    if (SPHRAY_OVF_CHECK) o |= static_cast<SOf<U>>((a ^ r) & (j ^ r)) < 0;
    return r;
}

struct WarpMem {
    void* pt;        // cap: position offsets (u32; u64 for int_width 128, see the file comment)
    void* pool;      // D x cap: jumps of orders 1..D (the merge's integer, 8 or 16 bytes)
    void* open;      // D+2: the open piece (t, a_0..a_D)
    double* hq_d2;  // hit queue (candidate order): squared distance of closest approach
    double* hq_t;
    int32_t* hq_p;
    float* hq_f;    // SPHRAY_HQ_FRONT: the hit's particle front (depth-sort key)
    uint16_t* ps;   // pending slots, unsorted
    uint16_t* fl;   // free slot stack (+ the flush set above it)
    uint32_t* hist;  // 256: radix-sort bins
    uint4* st_meta;   // SPHRAY_STAGE: 32 staged candidate records {front, particle, bbox, 0}
    double4* st_xyzh; //               and their {x, y, z, h}
    uint64_t* bar;    //               the mbarrier their bulk copy completes on
};

__device__ inline WarpMem carve(char* base, int D, int cap, int jb) {
    // layout must match warp_bytes_for (render.cuh); jb = bytes per jump
    // (16 also selects 8-byte position offsets)
    WarpMem w;
    char* p = base;
    w.pool = p;
    p += align16(static_cast<size_t>(jb) * D * cap);
    w.pt = p;
    p += align16((jb == 16 ? 8 : 4) * static_cast<size_t>(cap));
    w.open = p;
    p += align16(static_cast<size_t>(jb) * (D + 2));
    w.hq_d2 = reinterpret_cast<double*>(p);
    w.hq_t = w.hq_d2 + kHqSlots;
    p += align16(sizeof(double) * kHqSlots * 2);
    w.hq_p = reinterpret_cast<int32_t*>(p);
    p += align16(sizeof(int32_t) * kHqSlots);
    w.hq_f = reinterpret_cast<float*>(p);
    if (SPHRAY_HQ_FRONT) p += align16(sizeof(float) * kHqSlots);
    w.ps = reinterpret_cast<uint16_t*>(p);
    w.fl = w.ps + cap;
    p += align16(sizeof(uint16_t) * cap * 2);
    w.hist = reinterpret_cast<uint32_t*>(p);
    p += align16(sizeof(uint32_t) * 256);
    w.st_meta = reinterpret_cast<uint4*>(p);
    p += 32 * 16;
    w.st_xyzh = reinterpret_cast<double4*>(p);
    p += 32 * 32;
    w.bar = reinterpret_cast<uint64_t*>(p);
    return w;
}

// cp.async.bulk (bulk TMA) of candidate records into shared memory, completing
// on an mbarrier (transaction count = bytes).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

// Piece compositing (composite(), raycast.hpp:356-381), shared by the lane
// walk and the out-of-line early-termination replay.
template <int D, bool TS>
struct Compositor {
    const FrameParams& P;
    uint32_t tf_sa;  // shared address of the CTA's TF copy (TS)

    // Samples of one piece, front to back, from transmittance T0 (composite(),
    // raycast.hpp:369-377): midpoints lo + (s + 1/2) dt as the reference
    // places them, taken here as the piece-local abscissa x = x0 + (s + 1/2) dx
    // (x0 = lo/tau - t_piece, dx = dt/tau; evaluate_piece, raycast.hpp:295-301)
    // and fp64 Horner on the coefficients, times sigma; alpha = 1 - exp(-ab dt)
    // via alpha_of; colour and transmittance accumulate in fp64.  With `stop`
    // the reference's T > 1e-3 check runs before every sample (the
    // early-termination replay).  (Evaluating two samples per iteration for
    // ILP measured 7% slower on config 3: more registers, longer code.)
    __device__ __forceinline__ void sample_eval(const double (&c)[D + 1], double x, double dt,
                                                double& alpha, double& r, double& g,
                                                double& b) const {
        double acc = c[D];
#pragma unroll
        for (int d = D - 1; d >= 0; --d) acc = fma(acc, x, c[d]);
        acc *= P.Q.sigma;  // evaluate_piece (raycast.hpp:295-301): Horner on a_d, then x sigma
        double ab;
        if constexpr (TS)
            tf_sample(TfShared{tf_sa}, P.ntf, acc, r, g, b, ab);
        else
            tf_sample(TfGlobal{P.tf}, P.ntf, acc, r, g, b, ab);
        alpha = alpha_of(ab * dt);
    }

    __device__ __forceinline__ void sample_piece(const double (&c)[D + 1], double x0, double dx,
                                                 double dt, int n, double T0, bool stop,
                                                 double& Tout, double& cr, double& cg,
                                                 double& cb) const {
        Tout = T0;
        cr = cg = cb = 0.0;
        double sh = 0.5;  // s + 1/2 carried as a double (exact; no int -> double per sample)
        for (int s = 0; s < n; ++s) {
            if (stop && !(Tout > 1e-3)) break;
            double a, r, g, b;
            sample_eval(c, fma(sh, dx, x0), dt, a, r, g, b);
            sh += 1.0;
            const double ta = Tout * a;
            cr = fma(ta, r, cr);
            cg = fma(ta, g, cg);
            cb = fma(ta, b, cb);
            Tout = Tout * (1.0 - a);
        }
    }

    // Per-piece setup of composite() (raycast.hpp:364-372): [lo, hi] =
    // [t_s tau, t_e tau] cut to [near, far], n = max(2, ceil((hi-lo)/step))
    // samples of width dt = (hi-lo)/n, the piece polynomial in double, and
    // the piece-local abscissa x0 + (s + 1/2) dx of sample s.
    // Returns 0 when nothing is sampled (empty interval, or a zero piece
    // under a transfer function that is clear at 0: alpha = 1 - exp(-0) = 0).
    template <class U>
    __device__ __forceinline__ int piece_setup(int64_t ts, int64_t te, const U (&a)[D + 1],
                                               double (&c)[D + 1], double& x0, double& dx,
                                               double& dt) const {
        double A[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) A[d] = to_double(a[d]);
        return piece_setup_d(ts, te, A, c, x0, dx, dt);
    }
    // the same from the coefficients already converted to double (exact
    // integers up to rounding; zero exactly when the integer is zero)
    __device__ __forceinline__ int piece_setup_d(int64_t ts, int64_t te, const double (&A)[D + 1],
                                                 double (&c)[D + 1], double& x0, double& dx,
                                                 double& dt) const {
        const double a_lo = dmul(static_cast<double>(ts), P.Q.tau);
        const double a_hi = dmul(static_cast<double>(te), P.Q.tau);
        const double lo = (a_lo < P.cam.near_plane) ? P.cam.near_plane : a_lo;
        const double hi = (P.cam.far_plane < a_hi) ? P.cam.far_plane : a_hi;
        // branch-free: an empty interval or a clear zero piece just yields
        // n = 0 (len <= 0 counts as 2 samples and is never divided); the
        // branchy form with early returns measured 0.8% slower per frame
        const double len = dsub(hi, lo);
        const int n = sample_count(len, P.step, P.inv_step);
        dt = n == 2 ? len * 0.5 : div_exact(len, static_cast<double>(n));
        bool zero = true;
#pragma unroll
        for (int d = 0; d <= D; ++d) {
            zero &= A[d] == 0.0;
            c[d] = A[d];
        }
        x0 = fma(lo, P.inv_tau, -static_cast<double>(ts));
        dx = dt * P.inv_tau;
        return ((hi > lo) & !(zero & (P.tf0_clear != 0))) ? n : 0;
    }

    // Samples one piece into a lane's running (T, colour).
    template <class U>
    __device__ __forceinline__ void composite_piece(int64_t ts, int64_t te, const U (&a)[D + 1],
                                                    bool stop, double& Tl, double& cr, double& cg,
                                                    double& cb, int& nsmp) const {
        double A[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) A[d] = to_double(a[d]);
        composite_piece_d(ts, te, A, stop, Tl, cr, cg, cb, nsmp);
    }
    __device__ __forceinline__ void composite_piece_d(int64_t ts, int64_t te, const double (&A)[D + 1],
                                                      bool stop, double& Tl, double& cr, double& cg,
                                                      double& cb, int& nsmp) const {
        double c[D + 1], x0 = 0.0, dx = 0.0, dt = 0.0;
        const int n = piece_setup_d(ts, te, A, c, x0, dx, dt);
        nsmp += n;  // n == 0 runs no sample and adds zeros (no early return)
        double To, r, g, b;
        sample_piece(c, x0, dx, dt, n, Tl, stop, To, r, g, b);
        cr += r;
        cg += g;
        cb += b;
        Tl = To;
    }

};

template <int D, class U>
struct ReplayIn {
    U E[D + 1];   // sum of the jumps before the run, around tref
    U oa[D + 1];  // the previous open piece (lead lane)
    int64_t ot;
    bool lead;
    double Tb;  // the run's true starting transmittance
};
struct ReplayOut {
    double T, r, g, b;
};

// Early-termination replay of one lane's run (raycast.hpp:363, 369): the walk
// of RayWorker::walk from the true T with the per-sample stop test.  Out of
// line: it runs at most once per ray, and the render kernel is
// instruction-cache bound.
template <int D, bool TS, class U, class PT>
__device__ __noinline__ ReplayOut replay_run(const FrameParams& P, uint32_t tf_sa, const uint16_t* fs,
                                             const PT* pt, const U* pool, int cap,
                                             int64_t tb, int64_t tref, int k0, int k1, int nsel,
                                             ReplayIn<D, U> in) {
    const Compositor<D, TS> cmp{P, tf_sa};
    double Tl = in.Tb, cr = 0.0, cg = 0.0, cb = 0.0;
    int nsmp = 0;
    int64_t tcur = tb + static_cast<int64_t>(pt[fs[k0]]);
    if (in.lead) cmp.composite_piece(in.ot, tcur, in.oa, true, Tl, cr, cg, cb, nsmp);
    U Pc[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) Pc[d] = in.E[d];
    taylor_shift<D>(Pc, static_cast<uint64_t>(tcur) - static_cast<uint64_t>(tref));
    int64_t tn = tcur;
    for (int k = k0; k < k1; ++k) {
        const int s = fs[k];
        const int64_t t = tn;
        if (t != tcur) {
            taylor_shift<D>(Pc, static_cast<uint64_t>(t) - static_cast<uint64_t>(tcur));
            tcur = t;
        }
#pragma unroll
        for (int d = 1; d <= D; ++d) Pc[d] += pool[(d - 1) * cap + s];
        const bool more = k + 1 < nsel;
        tn = more ? tb + static_cast<int64_t>(pt[fs[k + 1]]) : t;
        if (more && tn != t) cmp.composite_piece(t, tn, Pc, true, Tl, cr, cg, cb, nsmp);
    }
    return {Tl, cr, cg, cb};
}

// One warp renders one ray at a time.  TS: the transfer function is read
// from the CTA's shared copy (else from global memory).
// REC: the per-ray records (piece checksums) are compiled in; the production
// kernel is instantiated with and without them (the checksum code costs ~2% of
// the frame even when disabled at run time), the robust variant always has them.
template <int D, int M, bool TS, int DUMP, bool EVEN, bool REC, class U = uint64_t>
class RayWorker {
   public:
    static constexpr int KN = 2 * M + 1;  // knots per hit, at most
    const FrameParams& P;
    WarpMem w;
    int lane;
    uint32_t tf_sa;  // shared address of the CTA's TF copy (TS)
    uint64_t ray_id = 0;
    // warp-uniform ray state
    int np = 0, nfree = 0;
    uint16_t* fs = nullptr;  // flush set of the current flush (w.fl + nfree)
    int64_t tb = 0;          // position base of pt[]
    bool has_base = false;
    using S = SOf<U>;
    static constexpr bool kW64 = sizeof(U) == 8;
    static constexpr bool kRobust = DUMP >= 1;  // rebasing + insert splitting
    static constexpr bool kDump = DUMP >= 2;    // validation dumps + int32 range tests
    // window position offsets from tb: 32 bits (a live window spans < 2^32
    // quanta), 64 bits for int_width 128 (tiny tau: one particle's knots can
    // span more than 2^32 quanta)
    using PT = std::conditional_t<kW64, uint32_t, uint64_t>;
    static constexpr uint64_t kSpan = kW64 ? 0x100000000ull : 0x8000000000000000ull;
    U G[D + 1];  // running sum of jumps shifted to tref (mod 2^64, 2^128)
    int64_t tref = 0;
    bool has_ref = false;
    bool has_open = false;  // w.open holds the last piece
    double T = 1.0;
    double Cr = 0.0, Cg = 0.0, Cb = 0.0;  // per-lane partial colour sums (reduced in finish)
    bool term = false;
    unsigned long long knots = 0, pieces = 0, hits = 0;
    int max_pending = 0;
    int max_resid = 0;  // SPHRAY_KSTATS: largest pending set left by a flush
    uint64_t csum = 0;  // per-lane share of the ray's piece checksum (P.ray_rec)
    bool aovf = false;  // a merged coefficient left int64 (shift_overflows / add_checked)
    uint32_t st_phase = 0;  // SPHRAY_STAGE: parity of the staging mbarrier
    bool st_inflight = false;

    Compositor<D, TS> cmp;

    __device__ RayWorker(const FrameParams& p, WarpMem wm, int l, uint32_t t)
        : P(p), w(wm), lane(l), tf_sa(t), cmp{p, t} {}

    __device__ __forceinline__ PT* pt_p() const { return static_cast<PT*>(w.pt); }
    // Taylor shift by the distance between two positions of the window
    // (below kSpan: 2^32 for the 32-bit offsets of int_width 32/64)
    __device__ __forceinline__ static void win_shift(U (&v)[D + 1], uint64_t dl) {
        if constexpr (kW64 && SPHRAY_SHIFT32)
            taylor_shift<D>(v, static_cast<uint32_t>(dl));
        else
            taylor_shift<D>(v, dl);
    }
    __device__ __forceinline__ int64_t pool_t(int slot) const {
        return tb + static_cast<int64_t>(pt_p()[slot]);
    }
    __device__ __forceinline__ U& pool_c(int d, int slot) const {
        return static_cast<U*>(w.pool)[(d - 1) * P.cap + slot];
    }
    __device__ __forceinline__ U* open_p() const { return static_cast<U*>(w.open);
    }

    __device__ void reset() {
        np = 0;
        nfree = P.cap;
        for (int i = lane; i < P.cap; i += 32) w.fl[i] = static_cast<uint16_t>(P.cap - 1 - i);
#pragma unroll
        for (int d = 0; d <= D; ++d) G[d] = 0;
        tref = 0;
        has_ref = false;
        has_open = false;
        tb = 0;
        has_base = false;
        T = 1.0;
        Cr = Cg = Cb = 0.0;
        term = false;
        knots = pieces = hits = 0;
        max_pending = 0;
        max_resid = 0;
        csum = 0;
        aovf = false;
        __syncwarp();
    }

    // Lane-sequential walk over the sorted flush-set knots [k0, k1) -- the
    // RayAccumulator recurrence (raycast.hpp:206-244) on one lane: Pc enters
    // as the sum of every earlier jump around tref, is moved to each knot by
    // a Taylor shift and takes its jumps; the last knot at a position closes
    // the piece that starts there, which is composited up to the next knot
    // (or kept as the open piece when it is the set's last).  `lead`: lane 0
    // first composites the previous flush's open piece (ot, oa).  stop: the
    // early-termination replay (absolute T, no side effects).
    __device__ void walk(int k0, int k1, int nsel, U (&Pc)[D + 1], bool comp, bool stop,
                         bool lead, int64_t ot, const U (&oa)[D + 1], double& Tl, double& cr,
                         double& cg, double& cb, int& npc, int& nsmp) {
        if (k0 >= k1) return;
        int64_t tcur = pool_t(fs[k0]);
        if (lead && comp) cmp.composite_piece(ot, tcur, oa, stop, Tl, cr, cg, cb, nsmp);
        taylor_shift<D>(Pc, static_cast<uint64_t>(tcur) - static_cast<uint64_t>(tref));
        int64_t tn = tcur;
        // the last emitted piece's coefficients as doubles: the overflow test's
        // input for the next shift and the compositing input (one conversion)
        double A[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) A[d] = 0.0;
        for (int k = k0; k < k1; ++k) {
            const int s = fs[k];
            const int64_t t = tn;
            const bool more = k + 1 < nsel;
            // the next knot's position and this knot's jumps are loaded before
            // the shift: their shared-memory latency overlaps it
            const int64_t tnext = more ? pool_t(fs[k + 1]) : t;
            U jmp[D + 1];
#pragma unroll
            for (int d = 1; d <= D; ++d) jmp[d] = pool_c(d, s);
            // branch-free: a shift by 0 (more jumps at the position) is the
            // identity; every nonzero shift follows an emission in this run,
            // whose doubles A feed the overflow test
            const uint64_t dl = static_cast<uint64_t>(t) - static_cast<uint64_t>(tcur);
            win_shift(Pc, dl);
            if (SPHRAY_OVF_CHECK)
                aovf |= (dl != 0) & shift_overflows<D, U, false>(A, static_cast<double>(static_cast<int64_t>(dl)), Pc);
            tcur = t;
#pragma unroll
            for (int d = 1; d <= D; ++d) {
                Pc[d] = add_checked(Pc[d], jmp[d], aovf);
                if constexpr (kDump && kW64) narrow32(static_cast<int64_t>(Pc[d]), P.Q.w32, aovf);
            }
            tn = tnext;
            if (more && tn == t) continue;  // more jumps at this position
            ++npc;
#pragma unroll
            for (int d = 0; d <= D; ++d) A[d] = to_double(Pc[d]);
            if constexpr (kDump && kW64)
#pragma unroll
                for (int d = 0; d <= D; ++d) narrow32(static_cast<int64_t>(Pc[d]), P.Q.w32, aovf);
            if constexpr (REC)
                if (P.ray_rec && !stop) csum += piece_mix<D, U>(t, Pc);
            if constexpr (kDump)
                if (!stop && P.dump_piece_t) dump_piece(t, Pc);
            if (!more) {
                if (!stop) {
                    open_p()[0] = static_cast<U>(static_cast<S>(t));
#pragma unroll
                    for (int d = 0; d <= D; ++d) open_p()[1 + d] = Pc[d];
                }
            } else if (comp) {
                cmp.composite_piece_d(t, tn, A, stop, Tl, cr, cg, cb, nsmp);
            }
        }
    }

    // validation dump of one FieldPiece
    // (int_width 128: the low 64 bits of each coefficient)
    __device__ __forceinline__ void dump_piece(int64_t t, const U (&a)[D + 1]) const {
        const unsigned long long at = atomicAdd(&P.dump_count[1], 1ull);
        if (at < P.dump_cap_pieces) {
            P.dump_piece_ray[at] = ray_id;
            P.dump_piece_t[at] = t;
#pragma unroll
            for (int d = 0; d <= D; ++d) P.dump_piece_a[at * (D + 1) + d] = static_cast<int64_t>(a[d]);
        }
    }

    // Merge + composite the sorted flush set fs[0, nsel), lane-blocked: lane
    // l owns the run [l R, l R + R).  (1) each lane sums its jumps shifted to
    // tref; (2) one exclusive warp scan per order gives every lane the sum of
    // all earlier jumps (exact modulo 2^64, so equal to RayAccumulator's Int128
    // result whenever that fits int64); (3) each lane walks its run (walk()),
    // compositing its pieces from T = 1; (4) one warp combine (prefix product
    // of the lanes' transmittances) folds the runs into the ray, and the first
    // lane that brings T to <= 1e-3 replays its run with the reference's
    // per-sample stop test (raycast.hpp:363, 369).
    __device__ void merge_composite(int nsel) {
        const int R = (nsel + 31) >> 5;
        const int k0 = min(lane * R, nsel), k1 = min(k0 + R, nsel);
        if (!has_ref) {
            tref = pool_t(fs[0]);
            has_ref = true;
        }
        // Sg = sum over the run of each knot's jumps shifted to tref, summed
        // forward: the partial sum moves knot to knot by in-window (< 2^32)
        // shifts and takes each knot's jumps (b_0 == 0 for every knot), and
        // one shift carries it to tref -- modulo 2^64 the same value as
        // shifting every knot to tref (shifts compose: p(y+a)(y+b) = p(y+a+b))
        U Sg[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) Sg[d] = 0;
        int64_t ta = k0 < k1 ? pool_t(fs[k0]) : tref;
        for (int k = k0; k < k1; ++k) {
            const int s = fs[k];
            const int64_t t = pool_t(s);
            if (t != ta) win_shift(Sg, static_cast<uint64_t>(t) - static_cast<uint64_t>(ta));
            ta = t;
#pragma unroll
            for (int d = 1; d <= D; ++d) Sg[d] += pool_c(d, s);
        }
        taylor_shift<D>(Sg, static_cast<uint64_t>(tref) - static_cast<uint64_t>(ta));
        U E[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) {
            const U inc = warp_incl_scan_u(Sg[d], lane);
            E[d] = G[d] + (inc - Sg[d]);
            G[d] += shfl_idx_u(inc, 31);
        }
        const bool lead = lane == 0 && has_open;
        int64_t ot = 0;
        U oa[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) oa[d] = 0;
        if (lead) {
            ot = static_cast<int64_t>(open_p()[0]);
#pragma unroll
            for (int d = 0; d <= D; ++d) oa[d] = open_p()[1 + d];
        }
        __syncwarp();
        const bool comp = !term;
        double Tl = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
        int npc = 0, nsmp = 0;
        U Pc[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) Pc[d] = E[d];
        walk(k0, k1, nsel, Pc, comp, false, lead, ot, oa, Tl, cr, cg, cb, npc, nsmp);
        __syncwarp();
        // Overflow test of each run's first shift (the walk tests the rest):
        // the state entering lane l's run (every jump before it, taken from the
        // scan) must be the exact shift of lane l-1's end state -- or, for
        // lane 0, of the previous flush's open piece.
        {
            const int64_t tlast = k1 > k0 ? pool_t(fs[k1 - 1]) : 0;
            int64_t tp = static_cast<int64_t>(__shfl_up_sync(kFull, static_cast<unsigned long long>(tlast), 1));
            double v[D + 1];
#pragma unroll
            for (int d = 0; d <= D; ++d) {
                const U up = shfl_up_u(Pc[d], 1);
                v[d] = to_double(lane == 0 ? oa[d] : up);
            }
            if (lane == 0) tp = ot;
            if (k0 < k1 && (lane > 0 || lead)) {
                const int64_t t0 = pool_t(fs[k0]);
                U Ps[D + 1];
#pragma unroll
                for (int d = 0; d <= D; ++d) Ps[d] = E[d];
                taylor_shift<D>(Ps, static_cast<uint64_t>(t0) - static_cast<uint64_t>(tref));
                aovf |= shift_overflows<D>(
                    v, static_cast<double>(static_cast<int64_t>(static_cast<uint64_t>(t0) - static_cast<uint64_t>(tp))), Ps);
            }
        }
        has_open = true;
        pieces += __reduce_add_sync(kFull, static_cast<unsigned>(npc));
        if (SPHRAY_KSTATS) {
            const unsigned ns = __reduce_add_sync(kFull, static_cast<unsigned>(nsmp));
            SPHRAY_KS(kStatSamples, ns);
        }
        if (comp) {
            double pre = Tl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double u = __shfl_up_sync(kFull, pre, o);
                if (lane >= o) pre *= u;
            }
            double excl = __shfl_up_sync(kFull, pre, 1);
            if (lane == 0) excl = 1.0;
            const double Tb = T * excl;  // T before this lane's run
            const double Ta = Tb * Tl;   // and after it
            const unsigned failm = __ballot_sync(kFull, nsmp > 0 && !(Ta > 1e-3));
            const int f = failm ? __ffs(failm) - 1 : 32;
            if (lane < f) {
                Cr = fma(Tb, cr, Cr);
                Cg = fma(Tb, cg, Cg);
                Cb = fma(Tb, cb, Cb);
            }
            double Tend = __shfl_sync(kFull, Ta, 31);
            if (f < 32) {
                double T2 = Tb;
                if (lane == f) {
                    ReplayIn<D, U> in;
#pragma unroll
                    for (int d = 0; d <= D; ++d) {
                        in.E[d] = E[d];
                        in.oa[d] = oa[d];
                    }
                    in.ot = ot;
                    in.lead = lead;
                    in.Tb = Tb;
                    const ReplayOut o = replay_run<D, TS, U, PT>(P, tf_sa, fs, pt_p(), static_cast<const U*>(w.pool), P.cap, tb, tref, k0,
                                                          k1, nsel, in);
                    T2 = o.T;
                    Cr += o.r;
                    Cg += o.g;
                    Cb += o.b;
                }
                Tend = __shfl_sync(kFull, T2, f);
                term = true;
            }
            T = Tend;
        }
        // every slot of the set is free again: fs sits right above the free
        // stack (the open piece lives in w.open)
        nfree += nsel;
        __syncwarp();
    }

    // Sort fs[0, nsel) by knot position: warp LSD radix sort on (t - tmin),
    // 8 bits per pass (flush sets usually span < 2^16 tau: two passes).  The
    // first pass ranks with shared atomics (its input order is arbitrary);
    // later passes scatter stably, ranks within a round of 32 from match.any
    // (a per-bit ballot version measured 2% slower).
    __device__ void sort_flush_radix(int nsel, PT tmin, int bits) {
        const PT* pt = pt_p();
        uint16_t* src = fs;
        uint16_t* dst = w.ps + np;  // free scratch: np + nsel <= cap
#pragma unroll 1
        for (int shift = 0; shift < bits; shift += 8) {
            SPHRAY_KS(kStatRadixPasses, 1);
            reinterpret_cast<uint4*>(w.hist)[lane] = make_uint4(0u, 0u, 0u, 0u);
            reinterpret_cast<uint4*>(w.hist)[lane + 32] = make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
#pragma unroll 1
            for (int c0 = 0; c0 < nsel; c0 += 32) {  // warp-uniform trip count
                const int i = c0 + lane;
                if (i < nsel) {
                    const uint32_t dg = static_cast<uint32_t>((pt[src[i]] - tmin) >> shift) & 255u;
                    atomicAdd(&w.hist[dg], 1u);
                }
            }
            __syncwarp();
            // exclusive prefix of the 256 bins: 8 per lane
            uint32_t loc[8], run = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                loc[k] = run;
                run += w.hist[lane * 8 + k];
            }
            const uint32_t before = warp_incl_scan(run, lane) - run;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) w.hist[lane * 8 + k] = before + loc[k];
            __syncwarp();
            if (shift == 0) {
                // the first pass needs no stability (the input order is
                // arbitrary): atomic ranks
#pragma unroll 1
                for (int c0 = 0; c0 < nsel; c0 += 32) {
                    const int i = c0 + lane;
                    if (i < nsel) {
                        const int sl = src[i];
                        const uint32_t dg = static_cast<uint32_t>(pt[sl] - tmin) & 255u;
                        dst[atomicAdd(&w.hist[dg], 1u)] = static_cast<uint16_t>(sl);
                    }
                }
                __syncwarp();
                uint16_t* tmp = src;
                src = dst;
                dst = tmp;
                continue;
            }
#pragma unroll 1
            for (int c0 = 0; c0 < nsel; c0 += 32) {
                const int i = c0 + lane;
                const bool valid = i < nsel;
                const int sl = valid ? src[i] : 0;
                const uint32_t dg = valid ? static_cast<uint32_t>((pt[sl] - tmin) >> shift) & 255u : 0u;
                const unsigned peers = __match_any_sync(kFull, valid ? dg : 256u + lane);
                const unsigned below = peers & lanemask_lt();
                const uint32_t base = valid ? w.hist[dg] : 0u;
                __syncwarp();
                if (valid) {
                    dst[base + __popc(below)] = static_cast<uint16_t>(sl);
                    if (below == 0) w.hist[dg] = base + __popc(peers);
                }
                __syncwarp();
            }
            uint16_t* tmp = src;
            src = dst;
            dst = tmp;
        }
        if (src != fs) {
            for (int i = lane; i < nsel; i += 32) fs[i] = src[i];
            __syncwarp();
        }
    }

    // Finalise every pending knot with t < F (all of them if all_): select
    // and sort them, merge equal positions, and turn each distinct position
    // into a FieldPiece -- the running polynomial being the prefix sum of the
    // jumps Taylor-shifted to a common origin tref (exact modulo 2^64, so
    // equal to RayAccumulator's Int128 result whenever that fits int64).
    __device__ void flush(int64_t F, bool all_) {
        // ---- select t < F into fs, compact the rest of ps in place
        fs = w.fl + nfree;  // [nfree, nfree + np) is free space above the stack
        int nsel = 0, nkeep = 0;
        // F as an offset from tb, clamped to [0, kSpan]
        const uint64_t dF = static_cast<uint64_t>(F) - static_cast<uint64_t>(tb);
        const uint64_t Fo = all_ ? kSpan : (F <= tb ? 0ull : (dF > kSpan ? kSpan : dF));
        // Robust variants (DUMP >= 1): every knot kept pending (and every later one)
        // is >= F, so the position base moves up to F in this pass and pt[]
        // offsets only span the live window, not the whole ray (small tau,
        // long rays).  The set being flushed keeps the old base until merged.
        const int64_t tb_next = (kRobust && !all_ && F > tb) ? F : tb;
        const PT keep_shift = (kRobust && Fo > 0 && Fo < kSpan) ? static_cast<PT>(Fo) : PT(0);
        PT tmin = ~PT(0), tmax = 0;
        PT* pt = pt_p();
        for (int c0 = 0; c0 < np; c0 += 32) {
            const int i = c0 + lane;
            const bool valid = i < np;
            const int s = valid ? w.ps[i] : 0;
            const PT t = valid ? pt[s] : PT(0);
            const bool sel = valid && static_cast<uint64_t>(t) < Fo;
            // one ballot: the valid lanes are a prefix, so a kept lane's rank
            // among the kept ones is (its lane) - (selected lanes below it)
            const unsigned msel = __ballot_sync(kFull, sel);
            const int below = __popc(msel & lanemask_lt());
            __syncwarp();
            // branch-free: one predicated store through a selected pointer
            // (the if/else form measured 1.8% slower per frame)
            uint16_t* const dp = sel ? fs + (nsel + below) : w.ps + (nkeep + lane - below);
            if (valid) *dp = static_cast<uint16_t>(s);
            tmin = sel && t < tmin ? t : tmin;
            tmax = sel && t > tmax ? t : tmax;
            if (keep_shift && valid && !sel) pt[s] = t - keep_shift;
            const int ns = __popc(msel);
            nsel += ns;
            nkeep += min(32, np - c0) - ns;
        }
        __syncwarp();
        SPHRAY_KS(kStatFlushes, 1);
        SPHRAY_KS(kStatScanned, np);
        SPHRAY_KS(kStatSelected, nsel);
        np = nkeep;
        if (SPHRAY_KSTATS && np > max_resid) max_resid = np;
        if (nsel == 0) {
            tb = tb_next;
            return;
        }
        int bits;
        if constexpr (kW64) {
            tmin = __reduce_min_sync(kFull, tmin);
            tmax = __reduce_max_sync(kFull, tmax);
            const uint32_t range = tmax - tmin;
            bits = range == 0 ? 0 : 32 - __clz(static_cast<int>(range));
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const PT a = __shfl_xor_sync(kFull, static_cast<unsigned long long>(tmin), o);
                const PT b = __shfl_xor_sync(kFull, static_cast<unsigned long long>(tmax), o);
                tmin = a < tmin ? a : tmin;
                tmax = b > tmax ? b : tmax;
            }
            const PT range = tmax - tmin;
            bits = range == 0 ? 0 : 64 - __clzll(static_cast<long long>(range));
        }
        if (SPHRAY_KSTATS) {
            const int bb = bits <= 8 ? 0 : bits <= 10 ? 1 : bits <= 12 ? 2 : bits <= 14 ? 3 : bits <= 16 ? 4 : 5;
            SPHRAY_KS(kStatBits0 + bb, 1);
        }
        if (nsel > 1) sort_flush_radix(nsel, tmin, bits);

        merge_composite(nsel);
        tb = tb_next;
    }

    __device__ void report_overflow(int pi) {
        const unsigned long long key = (static_cast<unsigned long long>(P.orig[pi]) << 32) | ray_id;
        atomicMin(&P.stats[kStatOverflowKey], key);
    }

    // Quantize the first nq queued hits (lane per hit) and append their knots
    // to the pending list.  Returns false if the window is too small.
    // 0: inserted; 1: the window is full; 2: a position falls outside the
    // 32-bit offset range of the current base.
    __device__ int insert_hits(int nq, int64_t F) {
        const bool act = lane < nq;
        int pi = 0;
        double lam = 0.0, tchi = 0.0, h = 0.0;
        if (act) {
            pi = w.hq_p[lane];
            tchi = w.hq_t[lane];
            h = P.pxyzh[pi].w;
            lam = lam_of(w.hq_d2[lane], h);  // RayHit::lam, raycast.hpp:118
        }
        bool ovf = false;
        HitPositions<M> hp;
        bool emits = act && quantize_positions<M, EVEN, kDump>(P.Q, h, lam, tchi, hp, ovf);
        int nk = emits ? hp.nk : 0;
        if (ovf) {
            report_overflow(pi);
            nk = 0;
            emits = false;
        }
        const int off = warp_incl_scan(nk, lane) - nk;
        const int total = __shfl_sync(kFull, off + nk, 31);
        SPHRAY_KS(kStatBatches, 1);
        if (total == 0) return 0;
        if (total > nfree) return 1;  // the caller flushed; the window is genuinely full
        const int slot0 = nfree - total + off;  // this lane's slots: fl[slot0 .. slot0 + nk)
        if (!has_base) {
            // every knot of the ray is >= the current flush bound
            tb = F;
            has_base = true;
        }
        bool far_ = false;  // a knot more than 2^32 quanta from tb
        if (emits) {
            double X[3 * D];
            const double* xs = P.xy + static_cast<size_t>(pi) * (3 * D);
#pragma unroll
            for (int d = 0; d < 3 * D; ++d) X[d] = xs[d];
            auto sink = [&](int o, int64_t t, const S (&b)[D + 1]) {
                const int slot = w.fl[slot0 + o];
                // b[0] is structurally zero (lut.hpp:107-166): only orders 1..D are stored
                const uint64_t to = static_cast<uint64_t>(t) - static_cast<uint64_t>(tb);
                far_ |= t < tb || (kW64 && to > 0xffffffffull);
                pt_p()[slot] = static_cast<PT>(to);
#pragma unroll
                for (int d = 1; d <= D; ++d) pool_c(d, slot) = static_cast<U>(b[d]);
                w.ps[np + off + o] = static_cast<uint16_t>(slot);
            };
            quantize_emit<D, M, EVEN, decltype(sink)&, kDump, S>(P.Q, X, hp, ovf, sink);
            if (ovf) report_overflow(pi);
        }
        // a ray spanning more than 2^32 position quanta does not fit the
        // 32-bit offsets: treated like a window overflow (retry pass, then
        // CapacityError)
        if (__any_sync(kFull, far_)) return 2;
        __syncwarp();
        nfree -= total;
        np += total;
        knots += total;
        if (np > max_pending) max_pending = np;
        return 0;
    }

    // front (depth-sort key) of the first queued hit
    __device__ __forceinline__ float head_front() const {
        return SPHRAY_HQ_FRONT ? w.hq_f[0] : P.front[w.hq_p[0]];
    }

    // Drop the first nq queued hits (up to 63 queued: shift in chunks of 32).
    __device__ __forceinline__ void drop_queued(int nq, int& hq_n) {
        const int rest = hq_n - nq;
        for (int c0 = 0; c0 < rest; c0 += 32) {
            const int i = c0 + lane;
            int32_t qp = 0;
            double ql = 0.0, qt = 0.0;
            float qf = 0.f;
            if (i < rest) {
                qp = w.hq_p[nq + i];
                if (SPHRAY_HQ_FRONT) qf = w.hq_f[nq + i];
                ql = w.hq_d2[nq + i];
                qt = w.hq_t[nq + i];
            }
            __syncwarp();
            if (i < rest) {
                w.hq_p[i] = qp;
                if (SPHRAY_HQ_FRONT) w.hq_f[i] = qf;
                w.hq_d2[i] = ql;
                w.hq_t[i] = qt;
            }
            __syncwarp();
        }
        hq_n = rest;
    }

    // Prefetch the candidate records [c0, min(c0 + 32, ce)) into the warp's
    // staging buffer (one elected lane issues the two bulk copies).
    __device__ __forceinline__ void stage_issue(uint32_t c0, uint32_t ce) {
        if (lane == 0) {
            const uint32_t nrec = min(32u, ce - c0);
            const uint32_t bar = smem_addr(w.bar);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, nrec * 48u);
            bulk_g2s(smem_addr(w.st_meta), P.cmeta + c0, nrec * 16u, bar);
            bulk_g2s(smem_addr(w.st_xyzh), P.cxyzh + c0, nrec * 32u, bar);
        }
        st_inflight = true;
    }
    __device__ __forceinline__ void stage_wait() {
        mbar_wait(smem_addr(w.bar), st_phase);
        st_phase ^= 1u;
        st_inflight = false;
    }
    __device__ __forceinline__ void stage_drain() {
        if (SPHRAY_STAGE && st_inflight) stage_wait();
    }

    // One ray; returns false if the knot window overflowed (ray is retried).
    __device__ bool run(int px, int py) {
        stage_drain();
        reset();
        const RayD ray = make_ray(P.cam, px, py);
        const int tile = (py >> kTileShift) * P.tiles_x + (px >> kTileShift);
        const int local = P.nranks > 1 ? tile / P.nranks : tile;
        const uint32_t cb = P.tile_begin[local], ce = P.tile_end[local];
        const uint32_t lx = static_cast<uint32_t>(px & (kTile - 1)), ly = static_cast<uint32_t>(py & (kTile - 1));
        const double near_plane = P.cam.near_plane, far_plane = P.cam.far_plane;
        uint32_t cursor = cb;
        int hq_n = 0;
        if (SPHRAY_STAGE && cursor < ce) stage_issue(cursor, ce);
        while (true) {
            // ---- gather: exact hit test of 32 candidates at a time
            while (hq_n < SPHRAY_GATHER_TO && hq_n <= kHitQueue - 32 && cursor < ce) {
                SPHRAY_KS(kStatGather, 1);
                const uint32_t c = cursor + lane;
                bool hit = false;
                double d2 = 0.0, tchi = 0.0;
                uint32_t pi = 0;
                uint4 mt = make_uint4(0u, 0u, 0u, 0u);
                double4 p = make_double4(0.0, 0.0, 0.0, 0.0);
                if (SPHRAY_STAGE) {
                    // records staged by the previous step's bulk copy; the next
                    // batch is requested as soon as this one is in registers
                    stage_wait();
                    if (c < ce) {
                        mt = w.st_meta[lane];
                        p = w.st_xyzh[lane];
                    }
                    __syncwarp();
                    if (cursor + 32 < ce) stage_issue(cursor + 32, ce);
                } else {
                    // the tile's candidate record (coalesced: consecutive lanes read
                    // consecutive records, both loads issued together); lanes
                    // past the list re-read the last one (cursor < ce)
                    const uint32_t cc = c < ce ? c : ce - 1;
                    mt = P.cmeta[cc];
                    p = P.cxyzh[cc];
                    if (SPHRAY_PF_L1 && c + 32 * SPHRAY_PF_L1 < ce) {
                        // pull a later batch's records from L2 into L1 while
                        // this one is tested
                        const uint32_t cn = c + 32 * SPHRAY_PF_L1;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.cmeta + cn));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.cxyzh + cn));
                    }
                }
                {
                    // branch-free: every lane runs the exact test, the range and
                    // bbox tests only mask it (divergent lanes would idle anyway;
                    // the branchy form measured 0.9% slower per frame)
                    pi = mt.y;
                    const bool inb = (c < ce) & (lx >= (mt.z & 15u)) & (lx <= ((mt.z >> 4) & 15u)) &
                                     (ly >= ((mt.z >> 8) & 15u)) & (ly <= ((mt.z >> 12) & 15u));
                    hit = inb & hit_test(ray, p.x, p.y, p.z, dmul(P.Q.q, p.w), near_plane,
                                         far_plane, d2, tchi);
                }
                const unsigned m = __ballot_sync(kFull, hit);
                {
                    // no branch: lanes without a hit store to the dummy slot
                    const int at = hit ? hq_n + __popc(m & lanemask_lt()) : kHitQueue;
                    w.hq_p[at] = static_cast<int32_t>(pi);
                    if (SPHRAY_HQ_FRONT) w.hq_f[at] = __uint_as_float(mt.x);
                    w.hq_d2[at] = d2;
                    w.hq_t[at] = tchi;
                }
                if (kDump && P.dump_hit_ray && m) {
                    unsigned long long base = 0;
                    if (lane == 0)
                        base = atomicAdd(&P.dump_count[0], static_cast<unsigned long long>(__popc(m)));
                    base = __shfl_sync(kFull, base, 0);
                    if (hit) {
                        const unsigned long long at = base + __popc(m & lanemask_lt());
                        if (at < P.dump_cap_hits) {
                            P.dump_hit_ray[at] = ray_id;
                            P.dump_hit_pidx[at] = P.orig[pi];
                            P.dump_hit_lam[at] = lam_of(d2, P.pxyzh[pi].w);
                            P.dump_hit_tchi[at] = tchi;
                        }
                    }
                }
                hq_n += __popc(m);
                hits += __popc(m);
                cursor += 32;
            }
            __syncwarp();
            // ---- insert as many queued hits as the window surely takes (each
            // emits at most KN knots), then flush: every knot below F -- the
            // bound of the first hit still queued, or of the next untested
            // candidate (both depth-sorted) -- is final.
            bool stuck = false;
            int nq_cap = 32;
#pragma unroll 1
            for (int round = 0; round < SPHRAY_INSERT_ROUNDS && hq_n > 0; ++round) {
                const int nq = min(min(hq_n, nq_cap), nfree / KN);
                if (nq == 0) {
                    stuck = round == 0;
                    break;
                }
                const int64_t F0 = knot_floor(head_front(), P.inv_tau);
                const int rc = insert_hits(nq, F0);
                if (rc == 1) return false;
                if (rc == 2) {
                    // positions beyond the 32-bit offsets of the base: the
                    // main pass hands the ray to the robust retry variant,
                    // which finalises what it can (moving the base up to F0)
                    // and inserts fewer hits at a time
                    if (!kRobust) return false;
                    const int np0 = np;
                    flush(F0, false);
                    if (nq == 1 && np == np0) return false;  // no progress possible
                    nq_cap = max(1, nq / 2);
                    --round;
                    continue;
                }
                drop_queued(nq, hq_n);
            }
            const bool final_ = hq_n == 0 && cursor >= ce;
            int64_t F = INT64_MAX;
            if (!final_) {
                const float fr = hq_n > 0 ? head_front() : __uint_as_float(P.cmeta[cursor].x);
                F = knot_floor(fr, P.inv_tau);
            }
            if (final_ || stuck || nfree < 32 * KN || np >= (P.cap * SPHRAY_FLUSH_AT) / 8) {
                const int np0 = np;
                flush(F, final_);
                if (stuck && np == np0) return false;  // nothing final: the window is too small
            }
            if (final_) break;
            if (term && P.mode == SPHRAY_MODE_FAST) break;
        }
        return true;
    }

    __device__ void finish(double* out, int px, int py) {
        const double sr = warp_sum(Cr), sg = warp_sum(Cg), sb = warp_sum(Cb);
        const bool ovf_any = __any_sync(kFull, aovf);
        uint64_t cs = 0;
        if constexpr (REC) {
            if (P.ray_rec) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(kFull, csum, o);
                cs = csum;
            }
        }
        if (lane == 0) {
            double r = P.bg[0], g = P.bg[1], b = P.bg[2];
            if (knots > 0) {
                // pixel = C + (1 - a) * background, a = 1 - T (raycast.hpp:379, 486-488)
                const double a = 1.0 - T;
                r = sr + (1.0 - a) * P.bg[0];
                g = sg + (1.0 - a) * P.bg[1];
                b = sb + (1.0 - a) * P.bg[2];
            }
            out[0] = r;
            out[1] = g;
            out[2] = b;
            const bool complete = !(term && P.mode == SPHRAY_MODE_FAST);
            bool residual = false;  // raycast.hpp:477-480: trailing piece must be zero
            if (knots > 0 && complete && has_open) {
#pragma unroll
                for (int d = 0; d <= D; ++d) residual |= open_p()[1 + d] != 0;
            }
            // RayAccumulator op count for P distinct positions (raycast.hpp:217-244)
            const unsigned long long Pp = pieces;
            const unsigned long long ops =
                Pp > 0 ? Pp * (D + 1) + (Pp - 1) * ((D + 1) * (3 * D + 4) / 2) : 0ull;
            if (knots) {
                atomicAdd(&P.stats[kStatKnots], knots);
                atomicAdd(&P.stats[kStatRays], 1ull);
                atomicAdd(&P.stats[kStatIntOps], ops);
                if (residual) atomicAdd(&P.stats[kStatResidual], 1ull);
            }
            if (term) atomicAdd(&P.stats[kStatTerminated], 1ull);
            if (ovf_any) atomicMin(&P.stats[kStatAccumOverflowRay], static_cast<unsigned long long>(ray_id));
            if (hits) atomicAdd(&P.stats[kStatHits], hits);
            atomicMax(&P.stats[kStatMaxPending], static_cast<unsigned long long>(max_pending));
            if (REC && P.ray_rec) {
                sphray_ray_record rec;
                rec.piece_checksum = cs;
                rec.knots = static_cast<uint32_t>(knots);
                rec.pieces = static_cast<uint32_t>(pieces);
                rec.hits = static_cast<uint32_t>(hits);
                rec.flags = (knots > 0 ? SPHRAY_RAY_TOUCHED : 0u) | (residual ? SPHRAY_RAY_RESIDUAL : 0u) |
                            (term ? SPHRAY_RAY_TERMINATED : 0u);
                P.ray_rec[static_cast<size_t>(py - P.row_lo) * (P.col_hi - P.col_lo) + (px - P.col_lo)] = rec;
            }
            if (SPHRAY_KSTATS) {
                const int b = max_resid < 128 ? 0 : max_resid < 192 ? 1 : max_resid < 256 ? 2
                            : max_resid < 320 ? 3 : max_resid < 384 ? 4 : 5;
                atomicAdd(&P.stats[kStatPeak0 + b], 1ull);
            }
        }
        __syncwarp();
    }
};

// W128: the merge runs modulo 2^128 (int_width 128; robust variant only)
template <int D, int M, bool TS, int DUMP, bool EVEN, bool REC, bool W128 = false>
__global__ void __maxnreg__(SPHRAY_MAXNREG) k_render_rays(const __grid_constant__ FrameParams P) {
    using U = std::conditional_t<W128, unsigned __int128, uint64_t>;
    extern __shared__ __align__(16) char smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const WarpMem wm = carve(smem + static_cast<size_t>(warp) * P.warp_bytes, D, P.cap, static_cast<int>(sizeof(U)));
    uint32_t tf_sa = 0;
    if constexpr (TS) {
        double* st = reinterpret_cast<double*>(smem + static_cast<size_t>(blockDim.x >> 5) * P.warp_bytes);
        for (int i = threadIdx.x; i < P.ntf * kTfStride; i += blockDim.x) st[i] = P.tf[i];
        __syncthreads();
        tf_sa = static_cast<uint32_t>(__cvta_generic_to_shared(st));
    }
    RayWorker<D, M, TS, DUMP, EVEN, REC, U> rw(P, wm, lane, tf_sa);
    if (SPHRAY_STAGE && lane == 0) mbar_init(smem_addr(wm.bar));
    __syncwarp();
    while (true) {
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(P.work_counter, 1ull);
        item = __shfl_sync(kFull, item, 0);
        if (item >= P.total_work) break;
        int px, py;
        if (P.ray_list) {
            const uint32_t rid = P.ray_list[item];
            px = static_cast<int>(rid % static_cast<uint32_t>(P.cam.W));
            py = static_cast<int>(rid / static_cast<uint32_t>(P.cam.W));
        } else {
            const uint64_t local = item / kTileRays;
            const int r = static_cast<int>(item % kTileRays);
            const uint64_t tile =
                P.nranks > 1 ? local * P.nranks + P.rank
                             : (local / P.tiles_wx + P.tile_row0) * static_cast<uint64_t>(P.tiles_x) +
                                   P.tile_col0 + local % P.tiles_wx;
            const int tx = static_cast<int>(tile % P.tiles_x), ty = static_cast<int>(tile / P.tiles_x);
            px = tx * kTile + (r & (kTile - 1));
            py = ty * kTile + (r >> kTileShift);
        }
        if (px >= P.col_hi || px < P.col_lo || py >= P.row_hi || py < P.row_lo) continue;
        rw.ray_id = static_cast<uint64_t>(py) * P.cam.W + px;
        uint64_t out_index = rw.ray_id;
        if (P.packed) {
            const uint64_t tile = static_cast<uint64_t>(py >> kTileShift) * P.tiles_x + (px >> kTileShift);
            out_index = (tile / P.nranks) * kTileRays + ((py & (kTile - 1)) << kTileShift) + (px & (kTile - 1));
        }
        if (rw.run(px, py)) {
            rw.finish(P.rgb + out_index * 3, px, py);
        } else if (lane == 0) {
            const unsigned at = atomicAdd(P.retry_count, 1u);
            P.retry_list[at] = static_cast<uint32_t>(rw.ray_id);
        }
        __syncwarp();
    }
    rw.stage_drain();  // no bulk copy may still target this CTA's shared memory
}

// quantize_particle for explicit hits (validation entry point).
template <int D, int M, bool EVEN>
__global__ void k_quantize_hits(const QuantParams Q, const sphray_particle* ps, const double* powh,
                                const double* powtau, size_t nhits, const double* tchi,
                                const double* lam, int64_t* knot_t, int64_t* knot_b,
                                int32_t* knot_count) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nhits) return;
    constexpr int KN = 2 * M + 1;
    const sphray_particle p = ps[i];
    bool ovf = false;
    HitPositions<M> hp;
    if (!quantize_positions<M, EVEN, true>(Q, p.h, lam[i], tchi[i], hp, ovf)) {
        knot_count[i] = ovf ? -1 : 0;
        return;
    }
    double X[3 * D];
    for (int d = 1; d <= D; ++d) {
        X[d - 1] = dmul(dmul(powtau[d - 1], p.mass), p.value);
        X[D + d - 1] = dmul(dmul(Q.sigma, p.density), powh[i * D + d - 1]);
        X[2 * D + d - 1] = recip_or_nan(X[D + d - 1]);
    }
    const int stride = Q.K + 1;
    auto sink = [&](int o, int64_t t, const int64_t (&b)[D + 1]) {
        if (o < KN && o < stride) {
            knot_t[i * stride + o] = t;
            for (int d = 0; d <= D; ++d) knot_b[(i * stride + o) * (D + 1) + d] = b[d];
        }
    };
    quantize_emit<D, M, EVEN, decltype(sink)&, true>(Q, X, hp, ovf, sink);
    knot_count[i] = ovf ? -1 : hp.nk;
}

}  // namespace rk

#define SPHRAY_RK_CUDA_OK(x)                                                       \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

template <int D, int M, bool EVEN>
int render_occupancy_tt(int warps, size_t smem) {
    int nb = 0;
    SPHRAY_RK_CUDA_OK(cudaFuncSetAttribute(rk::k_render_rays<D, M, true, 0, EVEN, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    SPHRAY_RK_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, rk::k_render_rays<D, M, true, 0, EVEN, false>, warps * 32, smem));
    return nb;
}

template <int D, int M>
int render_occupancy_t(int warps, size_t smem, bool even) {
    return even ? render_occupancy_tt<D, M, true>(warps, smem) : render_occupancy_tt<D, M, false>(warps, smem);
}

template <int D, int M, bool EVEN>
void launch_render_tt(const FrameParams& P, int blocks, int warps, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(P.warp_bytes) * warps + P.tf_smem;
    // Validation dumps, the retry pass and int_width 32 / 128 frames use the
    // full robust instantiation (DUMP = 2: dump code, int32 range tests,
    // per-flush rebasing of the 32-bit window offsets, batch splitting; TF in
    // global memory).  Frames whose rays span more than 2^31 quanta (small
    // tau) take the lean robust one (DUMP = 1: rebasing and splitting only,
    // TF in shared memory).  The production kernel carries none of it (it is
    // instruction-cache sensitive).
    const bool full = P.dump_hit_ray || P.dump_piece_t || P.ray_list || P.robust == 2 ||
                      (P.robust && !P.tf_smem);
    auto kern = P.w128 ? rk::k_render_rays<D, M, false, 2, EVEN, true, true>
                : full ? rk::k_render_rays<D, M, false, 2, EVEN, true>
                : P.robust ? rk::k_render_rays<D, M, true, 1, EVEN, true>
                : P.tf_smem ? (P.ray_rec ? rk::k_render_rays<D, M, true, 0, EVEN, true>
                                         : rk::k_render_rays<D, M, true, 0, EVEN, false>)
                            : rk::k_render_rays<D, M, false, 0, EVEN, true>;
    SPHRAY_RK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    kern<<<blocks, warps * 32, smem, s>>>(P);
    SPHRAY_RK_CUDA_OK(cudaGetLastError());
}

// the parity of K selects the closure at compile time (quantize.cuh)
template <int D, int M>
void launch_render_t(const FrameParams& P, int blocks, int warps, cudaStream_t s) {
    if ((P.Q.K & 1) == 0)
        launch_render_tt<D, M, true>(P, blocks, warps, s);
    else
        launch_render_tt<D, M, false>(P, blocks, warps, s);
}

template <int D, int M>
void launch_quantize_hits_t(const QuantParams& Q, const sphray_particle* ps, const double* powh,
                            const double* powtau, size_t nhits, const double* tchi,
                            const double* lam, int64_t* knot_t, int64_t* knot_b,
                            int32_t* knot_count, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>((nhits + 127) / 128);
    if ((Q.K & 1) == 0)
        rk::k_quantize_hits<D, M, true><<<g, 128, 0, s>>>(Q, ps, powh, powtau, nhits, tchi, lam,
                                                           knot_t, knot_b, knot_count);
    else
        rk::k_quantize_hits<D, M, false><<<g, 128, 0, s>>>(Q, ps, powh, powtau, nhits, tchi, lam,
                                                            knot_t, knot_b, knot_count);
    SPHRAY_RK_CUDA_OK(cudaGetLastError());
}

#define SPHRAY_INSTANTIATE(D, M)                                                             \
    template int render_occupancy_t<D, M>(int, size_t, bool);                                \
    template void launch_render_t<D, M>(const FrameParams&, int, int, cudaStream_t);         \
    template void launch_quantize_hits_t<D, M>(const QuantParams&, const sphray_particle*,   \
                                               const double*, const double*, size_t,         \
                                               const double*, const double*, int64_t*,       \
                                               int64_t*, int32_t*, cudaStream_t);

}  // namespace sphray_b200

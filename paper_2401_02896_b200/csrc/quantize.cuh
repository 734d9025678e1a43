// quantize.cuh -- quantize_particle<int64_t> (quantize.hpp:199-250) with the
// integer mirror closure (lut.hpp:100-168), split in two phases so the render
// kernel can allocate window slots between them:
//   phase A (positions)    quantize.hpp:211-216, lut.hpp:147-166
//   phase B (coefficients) quantize.hpp:218-242, lut.hpp:104-145
// Checked<int64_t> semantics: wrapping arithmetic plus an overflow flag.
#pragma once

#include <type_traits>

#include "device_math.cuh"
#include "render.cuh"

namespace sphray_b200 {
namespace dev {

constexpr long long binom(int n, int k) {
    long long r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

// Checked multiply by a binomial c > 0 (Checked<int64_t> *); c is a
// constant after unrolling, so the bounds fold and c == 1 costs nothing.
__device__ __forceinline__ int64_t cmul_binom(int64_t a, long long c, bool& o) {
    if (c == 1) return a;
    o |= a > INT64_MAX / c || a < INT64_MIN / c;
    return static_cast<int64_t>(static_cast<uint64_t>(a) * static_cast<uint64_t>(c));
}

template <int M>
struct HitPositions {
    static constexpr int KN = 2 * M + 1;
    int64_t pos[M + 1];  // pos[0] centre, pos[k] positive knots
    int64_t kpos[KN];    // emission order -m..-1, [0], 1..m (nondecreasing); odd K: no centre
    int nraw;            // emitted entries before the coincident merge (2m+1 or 2m)
    int nk;              // distinct positions (knots actually emitted)
    const double* row;   // LUT entry: m knots then |J| jumps
};

// Phase A.  Returns false when quantize_particle emits nothing (lam >= q,
// quantize.hpp:204).  All array indices are compile-time (M and the parity of
// K are template parameters) so nothing spills to local memory.
// N32: the kernel variant that serves int_width 32 (Q.w32 at run time):
// every Checked value also has to fit int32 (narrow32).
template <int M, bool EVEN, bool N32 = false>
__device__ __forceinline__ bool quantize_positions(const QuantParams& Q, double h, double lam,
                                                   double tchi, HitPositions<M>& hp,
                                                   bool& ovf) {
    const bool n32 = N32 && Q.w32;
    constexpr int KN = HitPositions<M>::KN;
    constexpr bool even = EVEN;  // K even (compile time: dead closure code stays out)
    hp.nraw = even ? KN : KN - 1;
    hp.nk = 0;
#pragma unroll
    for (int k = 0; k <= M; ++k) hp.pos[k] = 0;
#pragma unroll
    for (int q = 0; q < KN; ++q) hp.kpos[q] = 0;
    if (!(lam < Q.q)) return false;
    const int e = lut_index(lam, Q.lut_dl, Q.inv_dl, Q.lut_N);
    hp.row = Q.lut_rows + static_cast<size_t>(e) * Q.lut_stride;
    hp.pos[0] = narrow32(rint_div(tchi, Q.tau, Q.inv_tau, ovf), n32, ovf);
#pragma unroll
    for (int k = 1; k <= M; ++k)
        hp.pos[k] = narrow32(
            cadd(hp.pos[0], narrow32(rint_div(dmul(h, hp.row[k - 1]), Q.tau, Q.inv_tau, ovf), n32, ovf), ovf),
            n32, ovf);
    const int64_t twice = narrow32(cadd(hp.pos[0], hp.pos[0], ovf), n32, ovf);
    bool ov2 = false;  // the negative side is evaluated for all k; flags count once
#pragma unroll
    for (int i = 0; i < M; ++i) hp.kpos[i] = narrow32(csub(twice, hp.pos[M - i], ov2), n32, ov2);  // lut.hpp:150
    ovf |= ov2;
    // positive side (lut.hpp:154-166): even K puts the centre at index m
#pragma unroll
    for (int j = 0; j <= M; ++j) {
        const int64_t ev = (j == 0) ? hp.pos[0] : hp.pos[j];
        const int64_t od = (j < M) ? hp.pos[j + 1] : 0;
        hp.kpos[M + j] = even ? ev : od;
    }
    hp.nk = 1;
#pragma unroll
    for (int q = 1; q < KN; ++q)
        if (q < hp.nraw && hp.kpos[q] != hp.kpos[q - 1]) ++hp.nk;
    return true;
}

// Phase B.  X[0..D) = (pow(tau,d)*mass)*value, X[D..2D) = (sigma*density)*pow(h,d+3)
// (quantize.hpp:221-222 with the libm parts precomputed on the host),
// X[2D..3D) = recip_or_nan(X[D..2D)) for rint_div.
// sink(o, t, b) receives distinct knot o (0..nk) with its D+1 jumps.
// S: the Checked integer of the jumps -- int64_t, or __int128 for int_width
// 128 (positions stay int64: the window's positions are int64).
template <class S>
__device__ __forceinline__ S rint_div_s(double a, double b, double y, bool& o) {
    if constexpr (sizeof(S) == 16) return rint_div128(a, b, y, o);
    else return rint_div(a, b, y, o);
}
template <class S>
__device__ __forceinline__ S narrow_s(S v, bool on, bool& o) {
    if constexpr (sizeof(S) == 16) return v;
    else return narrow32(v, on, o);
}

template <int D, int M, bool EVEN, class Sink, bool N32 = false, class S = int64_t>
__device__ __forceinline__ void quantize_emit(const QuantParams& Q, const double* X,
                                              const HitPositions<M>& hp, bool& ovf,
                                              Sink&& sink) {
    using U = std::conditional_t<sizeof(S) == 16, unsigned __int128, uint64_t>;
    constexpr S kMin = static_cast<S>(static_cast<U>(1) << (8 * sizeof(S) - 1));
    const bool n32 = N32 && Q.w32;
    auto nw = [&](S v) { return narrow_s<S>(v, n32, ovf); };
    constexpr int m = M;
    constexpr int KN = HitPositions<M>::KN;
    constexpr bool even = EVEN;  // K even (compile time: dead closure code stays out)
    S negk[M][D + 1];  // negk[k-1] == bneg[m-k] of lut.hpp:106
    S center[D + 1];
#pragma unroll
    for (int k = 0; k < M; ++k)
#pragma unroll
        for (int d = 0; d <= D; ++d) negk[k][d] = 0;
#pragma unroll
    for (int d = 0; d <= D; ++d) center[d] = 0;
    const int c1 = even ? D : D / 2;  // index-set entries with k == 1 (approx.hpp:48-51)
#pragma unroll
    for (int k = 1; k <= M; ++k) {
#pragma unroll
        for (int d = 1; d <= D; ++d) {
            int ii;
            if (k == 1) {
                if (!even && (d & 1)) continue;
                ii = even ? d - 1 : d / 2 - 1;
            } else {
                ii = c1 + (k - 2) * D + (d - 1);
            }
            const S bp = nw(rint_div_s<S>(dmul(X[d - 1], hp.row[m + ii]), X[D + d - 1], X[2 * D + d - 1], ovf));
            negk[k - 1][d] = (d & 1) ? bp : nw(cneg(bp, ovf));  // lut.hpp:107-109
        }
    }
    if (even) {
        // even K: the centre knot carries the odd-order jumps (lut.hpp:118-130)
#pragma unroll
        for (int d = 1; d <= D; d += 2) {
            S acc = 0;
#pragma unroll
            for (int k = 1; k <= M; ++k) {
                const S off = nw(static_cast<S>(csub(hp.pos[k], hp.pos[0], ovf)));
                S pw = 1;  // off^(j-d), built one step at a time as lut.hpp:123-126
#pragma unroll
                for (int j = d; j <= D; ++j) {
                    S t = nw(cmul_binom(negk[k - 1][j], binom(j, d), ovf));
                    if (j > d) t = nw(cmul(t, pw, ovf));  // * 1 at j == d
                    acc = nw(cadd(acc, t, ovf));
                    if (j < D) pw = (j == d) ? off : nw(cmul(pw, off, ovf));
                }
            }
            center[d] = nw(cneg(nw(cadd(acc, acc, ovf)), ovf));
        }
    } else {
        // odd K: the innermost pair closes, descending odd d (lut.hpp:131-145)
#pragma unroll
        for (int d = (D % 2 == 1 ? D : D - 1); d >= 1; d -= 2) {
            S acc = 0;
#pragma unroll
            for (int k = 2; k <= M; ++k) acc = nw(cadd(acc, negk[k - 1][d], ovf));
#pragma unroll
            for (int k = 1; k <= M; ++k) {
                const S off = nw(static_cast<S>(csub(hp.pos[k], hp.pos[0], ovf)));
                S pw = off;
#pragma unroll
                for (int j = d + 1; j <= D; ++j) {
                    acc = nw(cadd(acc, nw(cmul(nw(cmul_binom(negk[k - 1][j], binom(j, d), ovf)), pw, ovf)), ovf));
                    if (j < D) pw = nw(cmul(pw, off, ovf));
                }
            }
            negk[0][d] = nw(cneg(acc, ovf));
        }
    }
    // jumps in emission order (lut.hpp:147-166), static indices like kpos
    auto jump = [&](int q, int d) -> S {
        if (q < M) return negk[M - 1 - q][d];
        const int j = q - M;  // even: 0 = centre, k = j; odd: k = j + 1
        if (even) {
            if (j == 0) return center[d];
            const S v = negk[j - 1][d];
            return (d & 1) ? v : static_cast<S>(static_cast<U>(0) - static_cast<U>(v));
        }
        if (j + 1 > M) return 0;
        const S v = negk[j][d];
        return (d & 1) ? v : static_cast<S>(static_cast<U>(0) - static_cast<U>(v));
    };
    // the positive side negates even orders (checked in the reference)
#pragma unroll
    for (int k = 1; k <= M; ++k)
#pragma unroll
        for (int d = 0; d <= D; d += 2)
            ovf |= negk[k - 1][d] == kMin || (n32 && negk[k - 1][d] == INT32_MIN);
    // coincident merge of quantize.hpp:229-242
    S cur[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) cur[d] = jump(0, d);
    int o = 0;
#pragma unroll
    for (int q = 1; q < KN; ++q) {
        if (q < hp.nraw) {
            if (hp.kpos[q] == hp.kpos[q - 1]) {
#pragma unroll
                for (int d = 0; d <= D; ++d) cur[d] = nw(cadd(cur[d], jump(q, d), ovf));
            } else {
                sink(o++, hp.kpos[q - 1], cur);
#pragma unroll
                for (int d = 0; d <= D; ++d) cur[d] = jump(q, d);
            }
        }
    }
    sink(o, even ? hp.kpos[KN - 1] : hp.kpos[KN - 2], cur);
}

}  // namespace dev
}  // namespace sphray_b200

/*
 * oracle/sphray_oracle.c -- TEST INFRASTRUCTURE: a plain-C restatement of the
 * reference's per-ray path (/root/reference/proj/include/sphray), used only by
 * tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() as the
 * CHECKER.  It is never linked into, or called by, the product.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by the unmodified reference (oracle/_ref,
 * tests/golden/make_golden.py) and against the reference's own known-answer
 * tests (raycast_tests.cpp, quantize_tests.cpp, lut_tests.cpp).
 *
 * Compiled with -O2 -ffp-contract=off and no -march (reference flags,
 * proj/CMakeLists.txt:11): every fp64 expression keeps the reference's order.
 * Integers: checked int64 for quantization (Checked<int64_t>, int_ops.hpp:63-99)
 * and exact __int128 accumulation (the reference's Int128 path), reporting a
 * merged coefficient that does not fit int64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OP_MAX_DEGREE 6
#define OP_MAX_M 4

typedef struct {
    double x, y, z, mass, density, h, value;
} op_particle;

typedef struct {
    int mode; /* 0 orthographic, 1 pinhole */
    int width, height;
    double position[3], look_at[3], up[3];
    double fov_deg, ortho_height, near_plane, far_plane;
} op_camera;

typedef struct {
    double q;
    int K, D, N;
    const double* records; /* N x (2 + m + |J|) doubles, .splt record order */
} op_lut;

typedef struct {
    double value, r, g, b, absorption;
} op_tf;

typedef struct {
    uint64_t particles, skipped_particles, knots, rays_touched, int_ops, residual_failures;
    double step;
} op_stats;

enum { OP_OK = 0, OP_CONFIG = 1, OP_OVERFLOW = 3, OP_NUMERIC = 4, OP_NOMEM = 5 };

/* ---------------------------------------------------------------- vectors
 * raycast.hpp:17-35 */
typedef struct {
    double x, y, z;
} v3;

static v3 v_add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v_sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v_scale(v3 a, double s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double v_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v_cross(v3 a, v3 o) {
    v3 r = {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
    return r;
}
static double v_norm(v3 a) { return sqrt(v_dot(a, a)); }
static int v_normalized(v3 a, v3* out) {
    const double n = v_norm(a);
    if (!(n > 0.0)) return OP_CONFIG;
    *out = v_scale(a, 1.0 / n);
    return OP_OK;
}
static v3 v_of(const double* p) { v3 r = {p[0], p[1], p[2]}; return r; }

/* ---------------------------------------------------------------- camera
 * Camera::validate / forward / right / up_vector / ray_at, raycast.hpp:59-100 */
typedef struct {
    v3 pos, fwd, right, upv;
} cam_frame;

static int cam_frame_of(const op_camera* c, cam_frame* f) {
    if (c->width < 1 || c->height < 1) return OP_CONFIG;
    if (!(c->far_plane > c->near_plane)) return OP_CONFIG;
    if (c->mode == 1 && !(c->fov_deg > 0.0 && c->fov_deg < 180.0)) return OP_CONFIG;
    if (c->mode == 0 && !(c->ortho_height > 0.0)) return OP_CONFIG;
    if (v_normalized(v_sub(v_of(c->look_at), v_of(c->position)), &f->fwd)) return OP_CONFIG;
    const v3 r = v_cross(f->fwd, v_of(c->up));
    if (!(v_norm(r) > 1e-12)) return OP_CONFIG;
    if (v_normalized(r, &f->right)) return OP_CONFIG;
    f->upv = v_cross(f->right, f->fwd);
    f->pos = v_of(c->position);
    return OP_OK;
}

static double cam_aspect(const op_camera* c) { return (double)c->width / c->height; }

static void ray_at(const op_camera* c, const cam_frame* f, int px, int py, v3* o, v3* d) {
    const double u = (px + 0.5) / c->width * 2.0 - 1.0;
    const double v = 1.0 - (py + 0.5) / c->height * 2.0;
    if (c->mode == 0) {
        const double hw = 0.5 * c->ortho_height * cam_aspect(c);
        const double hh = 0.5 * c->ortho_height;
        *o = v_add(v_add(f->pos, v_scale(f->right, u * hw)), v_scale(f->upv, v * hh));
        *d = f->fwd;
    } else {
        const double th = tan(c->fov_deg * 3.14159265358979323846 / 360.0);
        *o = f->pos;
        v3 w = v_add(v_add(f->fwd, v_scale(f->right, u * th * cam_aspect(c))), v_scale(f->upv, v * th));
        v_normalized(w, d);
    }
}

int op_camera_ray(const op_camera* c, int px, int py, double* origin, double* dir) {
    cam_frame f;
    const int rc = cam_frame_of(c, &f);
    if (rc) return rc;
    v3 o, d;
    ray_at(c, &f, px, py, &o, &d);
    origin[0] = o.x; origin[1] = o.y; origin[2] = o.z;
    dir[0] = d.x; dir[1] = d.y; dir[2] = d.z;
    return OP_OK;
}

/* detail::hit_ray, raycast.hpp:111-120 */
static int hit_ray(v3 o, v3 d, v3 chi, double support, double h, double near_plane,
                   double far_plane, double* lam, double* t_chi) {
    const v3 oc = v_sub(chi, o);
    const double t = v_dot(oc, d);
    const double d2 = v_dot(oc, oc) - t * t;
    if (!(d2 < support * support)) return 0;
    if (t + support <= near_plane || t - support >= far_plane) return 0;
    *lam = sqrt(d2 < 0.0 ? 0.0 : d2) / h; /* std::max(d2, 0.0) */
    *t_chi = t;
    return 1;
}

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

/* particle_ray_footprint, raycast.hpp:128-184 (pixel bbox, then exact test).
 * Writes up to cap hits; *n receives the total. */
int op_footprint(const op_particle* p, const op_camera* c, double q, uint64_t* ray, double* lam,
                 double* tchi, size_t cap, size_t* n) {
    cam_frame f;
    const int rc = cam_frame_of(c, &f);
    if (rc) return rc;
    const v3 chi = {p->x, p->y, p->z};
    const double support = q * p->h;
    int px0 = 0, px1 = c->width - 1, py0 = 0, py1 = c->height - 1;
    const v3 rel = v_sub(chi, f.pos);
    if (c->mode == 0) {
        const double hw = 0.5 * c->ortho_height * cam_aspect(c);
        const double hh = 0.5 * c->ortho_height;
        const double cx = v_dot(rel, f.right), cy = v_dot(rel, f.upv);
        px0 = imax(px0, (int)floor((cx - support + hw) / (2 * hw) * c->width - 0.5) - 1);
        px1 = imin(px1, (int)ceil((cx + support + hw) / (2 * hw) * c->width - 0.5) + 1);
        py0 = imax(py0, (int)floor((hh - (cy + support)) / (2 * hh) * c->height - 0.5) - 1);
        py1 = imin(py1, (int)ceil((hh - (cy - support)) / (2 * hh) * c->height - 0.5) + 1);
    } else {
        const double depth = v_dot(rel, f.fwd);
        if (depth - support > 0.0) {
            const double zmin = depth - support, zmax = depth + support;
            const double cx = v_dot(rel, f.right), cy = v_dot(rel, f.upv);
            const double th = tan(c->fov_deg * 3.14159265358979323846 / 360.0);
#define RATIO_LO(cc) (((cc) - support) / ((cc) - support <= 0.0 ? zmin : zmax))
#define RATIO_HI(cc) (((cc) + support) / ((cc) + support >= 0.0 ? zmin : zmax))
            const double u_lo = RATIO_LO(cx) / (th * cam_aspect(c));
            const double u_hi = RATIO_HI(cx) / (th * cam_aspect(c));
            const double v_lo = RATIO_LO(cy) / th;
            const double v_hi = RATIO_HI(cy) / th;
#undef RATIO_LO
#undef RATIO_HI
            px0 = imax(px0, (int)floor((u_lo + 1.0) * 0.5 * c->width - 0.5) - 1);
            px1 = imin(px1, (int)ceil((u_hi + 1.0) * 0.5 * c->width - 0.5) + 1);
            py0 = imax(py0, (int)floor((1.0 - v_hi) * 0.5 * c->height - 0.5) - 1);
            py1 = imin(py1, (int)ceil((1.0 - v_lo) * 0.5 * c->height - 0.5) + 1);
        }
    }
    size_t k = 0;
    for (int py = imax(py0, 0); py <= imin(py1, c->height - 1); ++py)
        for (int px = imax(px0, 0); px <= imin(px1, c->width - 1); ++px) {
            v3 o, d;
            double l, t;
            ray_at(c, &f, px, py, &o, &d);
            if (hit_ray(o, d, chi, support, p->h, c->near_plane, c->far_plane, &l, &t)) {
                if (k < cap) {
                    ray[k] = (uint64_t)py * (uint64_t)c->width + (uint64_t)px;
                    lam[k] = l;
                    tchi[k] = t;
                }
                ++k;
            }
        }
    *n = k;
    return OP_OK;
}

/* ---------------------------------------------------------------- LUT
 * Lut::lookup lut.hpp:43-52 (lam < q) and basis_index_set approx.hpp:44-54 */
static int lut_m(const op_lut* L) { return (L->K + 1) / 2; }
static int lut_nj(const op_lut* L) { return L->K * L->D / 2; }

int op_lut_index(const op_lut* L, double lam) {
    const double x = lam / (L->q / (double)L->N);
    double i = floor(x);
    if (i == x && i > 0.0) i -= 1.0;
    const size_t idx = (size_t)(i < 0.0 ? 0.0 : i);
    return (int)(idx < (size_t)(L->N - 1) ? idx : (size_t)(L->N - 1));
}

/* ---------------------------------------------------------------- checked ints
 * Checked<int64_t> int_ops.hpp:63-99, round_to_int int_ops.hpp:103-110 */
static int64_t c_add(int64_t a, int64_t b, int* o) { int64_t r; *o |= __builtin_add_overflow(a, b, &r); return r; }
static int64_t c_sub(int64_t a, int64_t b, int* o) { int64_t r; *o |= __builtin_sub_overflow(a, b, &r); return r; }
static int64_t c_mul(int64_t a, int64_t b, int* o) { int64_t r; *o |= __builtin_mul_overflow(a, b, &r); return r; }
static int64_t c_neg(int64_t a, int* o) { int64_t r; *o |= __builtin_sub_overflow((int64_t)0, a, &r); return r; }
static int64_t round_i64(double x, int* o) {
    const double r = nearbyint(x);
    const double hi = ldexp(1.0, 63);
    if (!(r >= -hi && r < hi)) { *o = 1; return 0; }
    return (int64_t)r;
}

static const long long BINOM[7][7] = {{1, 0, 0, 0, 0, 0, 0},  {1, 1, 0, 0, 0, 0, 0},
                                      {1, 2, 1, 0, 0, 0, 0},  {1, 3, 3, 1, 0, 0, 0},
                                      {1, 4, 6, 4, 1, 0, 0},  {1, 5, 10, 10, 5, 1, 0},
                                      {1, 6, 15, 20, 15, 6, 1}};

/* quantize_particle<int64_t> quantize.hpp:199-250 with mirror_closure
 * lut.hpp:100-168.  Knots: t_out[i], b_out[i*7 + d]. */
int op_quantize(const op_particle* p, double t_chi, double lam, const op_lut* L, double tau,
                double sigma, int64_t* t_out, int64_t* b_out, int* nout) {
    *nout = 0;
    if (!(lam < L->q)) return OP_OK;
    const int K = L->K, D = L->D, m = lut_m(L), nj = lut_nj(L);
    const double* e = L->records + (size_t)op_lut_index(L, lam) * (2 + m + nj) + 2;
    int ovf = 0;
    int64_t pos[OP_MAX_M + 1] = {0};
    pos[0] = round_i64(t_chi / tau, &ovf);
    for (int k = 1; k <= m; ++k) pos[k] = c_add(pos[0], round_i64(p->h * e[k - 1] / tau, &ovf), &ovf);
    int64_t bpos[OP_MAX_M][OP_MAX_DEGREE + 1];
    memset(bpos, 0, sizeof(bpos));
    int i = 0;
    for (int k = 1; k <= m; ++k)
        for (int d = 1; d <= D; ++d) {
            if (K % 2 == 1 && k == 1 && d % 2 == 1) continue;
            const double raw = pow(tau, d) * p->mass * p->value * e[m + i] /
                               (sigma * p->density * pow(p->h, d + 3));
            bpos[k - 1][d] = round_i64(raw, &ovf);
            ++i;
        }
    /* mirror_closure (lut.hpp:100-168) */
    int64_t bneg[OP_MAX_M][OP_MAX_DEGREE + 1];
    memset(bneg, 0, sizeof(bneg));
    for (int k = 1; k <= m; ++k)
        for (int d = 0; d <= D; ++d) bneg[m - k][d] = (d % 2 == 1) ? bpos[k - 1][d] : c_neg(bpos[k - 1][d], &ovf);
    int64_t center[OP_MAX_DEGREE + 1] = {0};
    if (K % 2 == 0) {
        for (int d = 1; d <= D; d += 2) {
            int64_t acc = 0;
            for (int k = 1; k <= m; ++k) {
                const int64_t off = c_sub(pos[k], pos[0], &ovf);
                int64_t pw = 1;
                for (int j = d; j <= D; ++j) {
                    acc = c_add(acc, c_mul(c_mul(BINOM[j][d], bneg[m - k][j], &ovf), pw, &ovf), &ovf);
                    if (j < D) pw = c_mul(pw, off, &ovf);
                }
            }
            center[d] = c_neg(c_add(acc, acc, &ovf), &ovf);
        }
    } else {
        for (int d = (D % 2 == 1 ? D : D - 1); d >= 1; d -= 2) {
            int64_t acc = 0;
            for (int k = 2; k <= m; ++k) acc = c_add(acc, bneg[m - k][d], &ovf);
            for (int k = 1; k <= m; ++k) {
                const int64_t off = c_sub(pos[k], pos[0], &ovf);
                int64_t pw = off;
                for (int j = d + 1; j <= D; ++j) {
                    acc = c_add(acc, c_mul(c_mul(BINOM[j][d], bneg[m - k][j], &ovf), pw, &ovf), &ovf);
                    if (j < D) pw = c_mul(pw, off, &ovf);
                }
            }
            bneg[m - 1][d] = c_neg(acc, &ovf);
        }
    }
    /* assembly -m..-1, [0], 1..m and coincident merge (quantize.hpp:229-242) */
    int64_t kt[2 * OP_MAX_M + 1], kb[2 * OP_MAX_M + 1][OP_MAX_DEGREE + 1];
    int nk = 0;
    for (int k = m; k >= 1; --k) {
        kt[nk] = c_sub(c_add(pos[0], pos[0], &ovf), pos[k], &ovf);
        for (int d = 0; d <= OP_MAX_DEGREE; ++d) kb[nk][d] = bneg[m - k][d];
        ++nk;
    }
    if (K % 2 == 0) {
        kt[nk] = pos[0];
        for (int d = 0; d <= OP_MAX_DEGREE; ++d) kb[nk][d] = center[d];
        ++nk;
    }
    for (int k = 1; k <= m; ++k) {
        kt[nk] = pos[k];
        for (int d = 0; d <= OP_MAX_DEGREE; ++d) kb[nk][d] = 0;
        for (int d = 0; d <= D; ++d) kb[nk][d] = (d % 2 == 1) ? bneg[m - k][d] : c_neg(bneg[m - k][d], &ovf);
        ++nk;
    }
    int n = 0;
    for (int q = 0; q < nk; ++q) {
        if (n > 0 && t_out[n - 1] == kt[q]) {
            for (int d = 0; d <= D; ++d) b_out[(n - 1) * 7 + d] = c_add(b_out[(n - 1) * 7 + d], kb[q][d], &ovf);
        } else {
            t_out[n] = kt[q];
            for (int d = 0; d <= OP_MAX_DEGREE; ++d) b_out[n * 7 + d] = kb[q][d];
            ++n;
        }
    }
    *nout = n;
    return ovf ? OP_OVERFLOW : OP_OK;
}

/* ---------------------------------------------------------------- accumulate
 * accumulate<Int128> + RayAccumulator, raycast.hpp:206-292.  Knots sorted by t.
 * Returns OP_OVERFLOW if a merged coefficient does not fit int64 (the pieces
 * are still written, low 64 bits). */
int op_accumulate(const int64_t* t, const int64_t* b, size_t n, int D, int64_t* piece_t,
                  int64_t* piece_a, size_t* npieces, uint64_t* ops) {
    __int128 a[OP_MAX_DEGREE + 1] = {0};
    int64_t t_prev = 0;
    int started = 0, fits = 1;
    uint64_t o = 0;
    size_t np = 0, i = 0;
    while (i < n) {
        size_t j = i + 1;
        __int128 jump[OP_MAX_DEGREE + 1];
        for (int d = 0; d <= D; ++d) jump[d] = b[i * 7 + d];
        while (j < n && t[j] == t[i]) {
            for (int d = 0; d <= D; ++d) jump[d] += b[j * 7 + d];
            ++j;
        }
        if (started && !(t_prev < t[i])) return OP_NUMERIC;
        if (started) {
            const __int128 dt = (__int128)t[i] - (__int128)t_prev;
            __int128 next[OP_MAX_DEGREE + 1];
            for (int d = 0; d <= D; ++d) {
                __int128 acc = 0, pw = 1;
                for (int jj = d; jj <= D; ++jj) {
                    acc += (__int128)BINOM[jj][d] * a[jj] * pw;
                    o += 2;
                    if (jj < D) {
                        pw *= dt;
                        ++o;
                    }
                }
                next[d] = acc;
            }
            for (int d = 0; d <= D; ++d) a[d] = next[d];
        }
        t_prev = t[i];
        started = 1;
        for (int d = 0; d <= D; ++d) {
            a[d] += jump[d];
            ++o;
        }
        piece_t[np] = t[i];
        for (int d = 0; d <= OP_MAX_DEGREE; ++d) piece_a[np * 7 + d] = 0;
        for (int d = 0; d <= D; ++d) {
            piece_a[np * 7 + d] = (int64_t)a[d];
            if (a[d] < (__int128)INT64_MIN || a[d] > (__int128)INT64_MAX) fits = 0;
        }
        ++np;
        i = j;
    }
    *npieces = np;
    if (ops) *ops = o;
    return fits ? OP_OK : OP_OVERFLOW;
}

/* ---------------------------------------------------------------- composite
 * evaluate_piece raycast.hpp:295-301, TransferFunction::sample 326-337,
 * composite 356-381 */
static void tf_sample(const op_tf* p, size_t n, double v, op_tf* out) {
    if (v <= p[0].value) { *out = p[0]; return; }
    if (v >= p[n - 1].value) { *out = p[n - 1]; return; }
    size_t i = 1;
    while (p[i].value < v) ++i;
    const op_tf* a = &p[i - 1];
    const op_tf* b = &p[i];
    const double w = (v - a->value) / (b->value - a->value);
    out->value = v;
    out->r = a->r + w * (b->r - a->r);
    out->g = a->g + w * (b->g - a->g);
    out->b = a->b + w * (b->b - a->b);
    out->absorption = a->absorption + w * (b->absorption - a->absorption);
}

int op_composite(const int64_t* piece_t, const int64_t* piece_a, size_t n, double tau, double sigma,
                 int D, const op_tf* tf, size_t ntf, double step, double t_min, double t_max,
                 double* rgba) {
    double T = 1.0, r = 0.0, g = 0.0, b = 0.0;
    if (!(step > 0.0)) return OP_CONFIG;
    for (size_t i = 0; i + 1 < n && T > 1e-3; ++i) {
        const double a_lo = (double)piece_t[i] * tau, a_hi = (double)piece_t[i + 1] * tau;
        const double lo = a_lo < t_min ? t_min : a_lo;
        const double hi = t_max < a_hi ? t_max : a_hi;
        if (!(hi > lo)) continue;
        const int c = (int)ceil((hi - lo) / step);
        const int ns = c > 2 ? c : 2;
        const double dt = (hi - lo) / ns;
        for (int s = 0; s < ns && T > 1e-3; ++s) {
            const double t = lo + (s + 0.5) * dt;
            const double x = t / tau - (double)piece_t[i];
            double acc = 0.0;
            for (int d = D; d >= 0; --d) acc = acc * x + (double)piece_a[i * 7 + d];
            op_tf m;
            tf_sample(tf, ntf, acc * sigma, &m);
            const double alpha = 1.0 - exp(-m.absorption * dt);
            r += T * alpha * m.r;
            g += T * alpha * m.g;
            b += T * alpha * m.b;
            T *= 1.0 - alpha;
        }
    }
    rgba[0] = r;
    rgba[1] = g;
    rgba[2] = b;
    rgba[3] = 1.0 - T;
    return OP_OK;
}

/* ---------------------------------------------------------------- render
 * render_scene raycast.hpp:414-497, single-threaded, Int128 accumulation. */
typedef struct {
    uint64_t ray;
    int64_t t;
    int64_t b[7];
} op_knot;

static int knot_cmp(const void* pa, const void* pb) {
    const op_knot* a = (const op_knot*)pa;
    const op_knot* b = (const op_knot*)pb;
    if (a->ray != b->ray) return a->ray < b->ray ? -1 : 1;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    return 0;
}

int op_render(const op_particle* ps, size_t n, const op_camera* cam, const op_tf* tf, size_t ntf,
              const op_lut* L, double tau, double sigma, double h_r, double step_opt,
              const double* bg, double* rgb, op_stats* st, int64_t* err_particle,
              uint64_t* err_ray) {
    cam_frame f;
    if (cam_frame_of(cam, &f)) return OP_CONFIG;
    if (ntf == 0) return OP_CONFIG;
    for (size_t i = 0; i < ntf; ++i) {
        if (tf[i].absorption < 0.0) return OP_CONFIG;
        if (i > 0 && !(tf[i].value > tf[i - 1].value)) return OP_CONFIG;
    }
    const int D = L->D;
    memset(st, 0, sizeof(*st));
    st->particles = n;
    st->step = step_opt > 0.0 ? step_opt : h_r / 8.0;
    size_t cap = 1024, nk = 0, hcap = 1024;
    op_knot* knots = (op_knot*)malloc(cap * sizeof(op_knot));
    uint64_t* hr = (uint64_t*)malloc(hcap * 8);
    double* hl = (double*)malloc(hcap * 8);
    double* ht = (double*)malloc(hcap * 8);
    if (!knots || !hr || !hl || !ht) return OP_NOMEM;
    int rc = OP_OK;
    for (size_t i = 0; i < n && rc == OP_OK; ++i) {
        size_t nh = 0;
        op_footprint(&ps[i], cam, L->q, hr, hl, ht, hcap, &nh);
        if (nh > hcap) {
            hcap = nh;
            hr = (uint64_t*)realloc(hr, hcap * 8);
            hl = (double*)realloc(hl, hcap * 8);
            ht = (double*)realloc(ht, hcap * 8);
            op_footprint(&ps[i], cam, L->q, hr, hl, ht, hcap, &nh);
        }
        if (nh == 0) st->skipped_particles++;
        for (size_t h = 0; h < nh; ++h) {
            int64_t t[9], b[9 * 7];
            int cnt = 0;
            if (op_quantize(&ps[i], ht[h], hl[h], L, tau, sigma, t, b, &cnt) != OP_OK) {
                rc = OP_OVERFLOW;
                if (err_particle) *err_particle = (int64_t)i;
                if (err_ray) *err_ray = hr[h];
                break;
            }
            for (int k = 0; k < cnt; ++k) {
                if (nk == cap) {
                    cap *= 2;
                    knots = (op_knot*)realloc(knots, cap * sizeof(op_knot));
                }
                knots[nk].ray = hr[h];
                knots[nk].t = t[k];
                memcpy(knots[nk].b, &b[k * 7], 7 * 8);
                ++nk;
            }
        }
    }
    free(hr);
    free(hl);
    free(ht);
    if (rc != OP_OK) {
        free(knots);
        return rc;
    }
    st->knots = nk;
    qsort(knots, nk, sizeof(op_knot), knot_cmp);
    const size_t npix = (size_t)cam->width * cam->height;
    for (size_t i = 0; i < npix; ++i) {
        rgb[3 * i] = bg[0];
        rgb[3 * i + 1] = bg[1];
        rgb[3 * i + 2] = bg[2];
    }
    int64_t* kt = (int64_t*)malloc((nk + 1) * 8);
    int64_t* kb = (int64_t*)malloc((nk + 1) * 7 * 8);
    int64_t* pt = (int64_t*)malloc((nk + 1) * 8);
    int64_t* pa = (int64_t*)malloc((nk + 1) * 7 * 8);
    size_t s = 0;
    while (s < nk) {
        size_t e = s;
        while (e < nk && knots[e].ray == knots[s].ray) {
            kt[e - s] = knots[e].t;
            memcpy(&kb[(e - s) * 7], knots[e].b, 7 * 8);
            ++e;
        }
        size_t np = 0;
        uint64_t ops = 0;
        op_accumulate(kt, kb, e - s, D, pt, pa, &np, &ops);
        st->rays_touched++;
        st->int_ops += ops;
        int zero = 1;
        for (int d = 0; d <= D; ++d)
            if (pa[(np - 1) * 7 + d] != 0) zero = 0;
        st->residual_failures += !zero;
        double c[4];
        if (op_composite(pt, pa, np, tau, sigma, D, tf, ntf, st->step, cam->near_plane,
                         cam->far_plane, c) != OP_OK) {
            rc = OP_CONFIG;
            break;
        }
        const uint64_t id = knots[s].ray;
        rgb[3 * id] = c[0] + (1.0 - c[3]) * bg[0];
        rgb[3 * id + 1] = c[1] + (1.0 - c[3]) * bg[1];
        rgb[3 * id + 2] = c[2] + (1.0 - c[3]) * bg[2];
        s = e;
    }
    free(kt);
    free(kb);
    free(pt);
    free(pa);
    free(knots);
    return rc;
}

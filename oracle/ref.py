"""ctypes wrapper around oracle/_ref/libsphray_ref.so -- TEST INFRASTRUCTURE.

The library is the UNMODIFIED reference (header-only C++20 under
/root/reference/proj/include) compiled by oracle/Makefile around
oracle/ref_driver.cpp.  Only tests/, bench.py (cpu_baseline leg and
``--impl reference``) and __graft_entry__.smoke() may use it, and only as the
checker / CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsphray_ref.so")

MAX_DEGREE = 6


class RpParticle(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("x", "y", "z", "mass", "density", "h", "value")]


class RpCamera(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("width", C.c_int),
        ("height", C.c_int),
        ("position", C.c_double * 3),
        ("look_at", C.c_double * 3),
        ("up", C.c_double * 3),
        ("fov_deg", C.c_double),
        ("ortho_height", C.c_double),
        ("near_plane", C.c_double),
        ("far_plane", C.c_double),
    ]


class RpTf(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("value", "r", "g", "b", "absorption")]


class RpQuanta(C.Structure):
    _fields_ = [("tau", C.c_double), ("sigma", C.c_double), ("width_bits", C.c_int)]


class RpDStats(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mass_r", "density_r", "h_r", "value_r", "phi_repr",
                                           "a_max", "clustering_factor")] + [("count", C.c_uint64)]


class RpRStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("particles", "skipped_particles", "knots",
                                           "rays_touched", "int_ops", "residual_failures")] + [
        ("step", C.c_double)]


class RpRayRecord(C.Structure):
    _fields_ = [("piece_checksum", C.c_uint64), ("knots", C.c_uint32), ("pieces", C.c_uint32),
                ("hits", C.c_uint32), ("flags", C.c_uint32)]


RAY_RECORD_DTYPE = np.dtype([("piece_checksum", "<u8"), ("knots", "<u4"), ("pieces", "<u4"),
                             ("hits", "<u4"), ("flags", "<u4")])


class RpError(C.Structure):
    _fields_ = [("code", C.c_int), ("particle_index", C.c_int64), ("ray_id", C.c_uint64),
                ("msg", C.c_char * 256)]


class RefError(RuntimeError):
    def __init__(self, err: RpError):
        self.code = err.code
        self.particle_index = err.particle_index
        self.ray_id = err.ray_id
        super().__init__(f"reference error {err.code}: {err.msg.decode(errors='replace')}")


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        _lib = C.CDLL(LIB_PATH)
        _lib.rp_lut_load.restype = C.c_void_p
        _lib.rp_lut_load.argtypes = [C.c_char_p, C.POINTER(RpError)]
        _lib.rp_lut_free.argtypes = [C.c_void_p]
        _lib.rp_pipeline_run.restype = C.c_void_p
        _lib.rp_pipeline_run_region.restype = C.c_void_p
        _lib.rp_footprint.restype = C.c_int64
        _lib.rp_footprint_region.restype = C.c_int64
        _lib.rp_load_particles.restype = C.c_int64
        _lib.rp_load_tf.restype = C.c_int64
        _lib.rp_scene_default_count.restype = C.c_size_t
        _lib.rp_render_report.restype = C.c_int64
    return _lib


def _check(rc: int, err: RpError):
    if rc != 0:
        raise RefError(err)


PARTICLE_DTYPE = np.dtype([(n, "<f8") for n in ("x", "y", "z", "mass", "density", "h", "value")])


def as_particles(arr) -> np.ndarray:
    """(n,7) float64 or structured array -> contiguous (n,7) float64."""
    a = np.ascontiguousarray(arr)
    if a.dtype == PARTICLE_DTYPE:
        a = a.view("<f8").reshape(-1, 7)
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 7)
    return a


def _pp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(RpParticle)) if a.size else None


@dataclass
class Camera:
    mode: str = "orthographic"
    position: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    width: int = 64
    height: int = 64
    fov_deg: float = 60.0
    ortho_height: float = 2.0
    near: float = 0.0
    far: float = 1e30

    def c(self) -> RpCamera:
        c = RpCamera()
        c.mode = 1 if self.mode == "pinhole" else 0
        c.width, c.height = self.width, self.height
        c.position[:] = self.position
        c.look_at[:] = self.look_at
        c.up[:] = self.up
        c.fov_deg, c.ortho_height = self.fov_deg, self.ortho_height
        c.near_plane, c.far_plane = self.near, self.far
        return c


def _tf(points):
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 5)
    arr = (RpTf * max(1, len(pts)))()
    for i, p in enumerate(pts):
        arr[i] = RpTf(*p)
    return arr, len(pts)


class Lut:
    def __init__(self, path: str):
        err = RpError()
        self.path = path
        self.h = lib().rp_lut_load(path.encode(), C.byref(err))
        if not self.h:
            raise RefError(err)
        q, K, D, N = C.c_double(), C.c_int(), C.c_int(), C.c_int()
        lib().rp_lut_info(C.c_void_p(self.h), C.byref(q), C.byref(K), C.byref(D), C.byref(N))
        self.q, self.K, self.D, self.N = q.value, K.value, D.value, N.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.rp_lut_free(C.c_void_p(self.h))
            self.h = None

    def lookup(self, lam: float):
        kn = (C.c_double * 8)()
        sh = (C.c_double * 64)()
        idx = C.c_int()
        lib().rp_lut_lookup(C.c_void_p(self.h), C.c_double(lam), kn, sh, C.byref(idx))
        m = (self.K + 1) // 2
        return idx.value, list(kn[:m]), list(sh[: self.K * self.D // 2])


def build_lut(K: int, D: int, N: int, path: str, seed: int = 0, threads: int = 0) -> float:
    err = RpError()
    estar = C.c_double()
    _check(lib().rp_lut_build(K, D, N, C.c_uint64(seed), threads, path.encode(), C.byref(estar),
                              C.byref(err)), err)
    return estar.value


def kernel_constants():
    k, kp = C.c_double(), C.c_double()
    lib().rp_kernel_constants(C.byref(k), C.byref(kp))
    return k.value, kp.value


def dataset_stats(particles, lut: Lut, clustering: float = 16.0) -> RpDStats:
    a = as_particles(particles)
    out, err = RpDStats(), RpError()
    _check(lib().rp_dataset_stats(_pp(a), C.c_size_t(len(a)), C.c_void_p(lut.h),
                                  C.c_double(clustering), C.byref(out), C.byref(err)), err)
    return out


def choose_quanta(lut: Lut, ds: RpDStats, width_bits: int = 64) -> RpQuanta:
    out, err = RpQuanta(), RpError()
    _check(lib().rp_choose_quanta(C.c_void_p(lut.h), C.byref(ds), width_bits, C.byref(out),
                                  C.byref(err)), err)
    return out


def camera_ray(cam: Camera, px: int, py: int):
    o = (C.c_double * 3)()
    d = (C.c_double * 3)()
    rid = C.c_uint64()
    c = cam.c()
    lib().rp_camera_ray(C.byref(c), px, py, o, d, C.byref(rid))
    return tuple(o), tuple(d), rid.value


def render(particles, cam: Camera, tf, lut: Lut, qc: RpQuanta, ds: RpDStats, step: float = 0.0,
           background=(0.0, 0.0, 0.0), threads: int = 0, accum_bits: int = 64):
    """sphray::render_scene<Int>: returns (rgb (H,W,3) float64, stats dict, seconds)."""
    a = as_particles(particles)
    c = cam.c()
    tfa, ntf = _tf(tf)
    rgb = np.zeros((cam.height, cam.width, 3), dtype=np.float64)
    st, err = RpRStats(), RpError()
    sec = C.c_double()
    bg = (C.c_double * 3)(*background)
    _check(lib().rp_render(_pp(a), C.c_size_t(len(a)), C.byref(c), tfa, C.c_size_t(ntf),
                           C.c_void_p(lut.h), C.byref(qc), C.byref(ds), C.c_double(step), bg,
                           threads, accum_bits, rgb.ctypes.data_as(C.POINTER(C.c_double)),
                           C.byref(st), C.byref(sec), C.byref(err)), err)
    stats = {f: getattr(st, f) for f, _ in RpRStats._fields_}
    return rgb, stats, sec.value


def render_robust(particles, cam, tf, lut, qc, ds, step=0.0, background=(0, 0, 0), threads=0):
    """render_scene<int64_t>; on the reference's (possibly spurious) OverflowError, the same
    quanta through render_scene<Int128> (raycast_tests.cpp:440-442: identical when both run)."""
    try:
        return render(particles, cam, tf, lut, qc, ds, step, background, threads, 64) + (64,)
    except RefError as e:
        if e.code != 3:
            raise
        return render(particles, cam, tf, lut, qc, ds, step, background, threads, 128) + (128,)


def footprint(particles, cam: Camera, q: float, region=(0, 0, 0, 0)):
    """All hits (ray id, particle index, lam, t_chi), particle-major, reference order;
    `region` (x0, y0, w, h) keeps only hits on those pixels (w == 0: the frame)."""
    a = as_particles(particles)
    c = cam.c()
    err = RpError()
    R = [int(v) for v in region]
    n = lib().rp_footprint_region(_pp(a), C.c_size_t(len(a)), C.byref(c), C.c_double(q), *R,
                                  None, None, None, None, C.c_size_t(0), C.byref(err))
    if n < 0:
        raise RefError(err)
    ray = np.zeros(n, np.uint64)
    pidx = np.zeros(n, np.int64)
    lam = np.zeros(n, np.float64)
    tchi = np.zeros(n, np.float64)
    P = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
    n2 = lib().rp_footprint_region(_pp(a), C.c_size_t(len(a)), C.byref(c), C.c_double(q), *R,
                                   P(ray, C.c_uint64), P(pidx, C.c_int64), P(lam, C.c_double),
                                   P(tchi, C.c_double), C.c_size_t(n), C.byref(err))
    assert n2 == n
    return ray, pidx, lam, tchi


def quantize(particle, ray: int, tchi: float, lam: float, lut: Lut, qc: RpQuanta, pidx: int = -1):
    p = RpParticle(*[float(v) for v in np.asarray(particle, dtype=np.float64).reshape(7)])
    t = (C.c_int64 * 16)()
    b = (C.c_int64 * (16 * (MAX_DEGREE + 1)))()
    n = C.c_int()
    err = RpError()
    _check(lib().rp_quantize(C.byref(p), C.c_uint64(ray), C.c_double(tchi), C.c_double(lam),
                             C.c_void_p(lut.h), C.byref(qc), C.c_int64(pidx), t, b, 16,
                             C.byref(n), C.byref(err)), err)
    ts = np.array(t[: n.value], dtype=np.int64)
    bs = np.array(b[: n.value * (MAX_DEGREE + 1)], dtype=np.int64).reshape(-1, MAX_DEGREE + 1)
    return ts, bs


def accumulate(t, b, D: int, accum_bits: int = 128):
    t = np.ascontiguousarray(t, dtype=np.int64)
    b = np.zeros((len(t), MAX_DEGREE + 1), dtype=np.int64) if b is None else \
        np.ascontiguousarray(b, dtype=np.int64).reshape(-1, MAX_DEGREE + 1)
    n = len(t)
    pt = np.zeros(max(n, 1), np.int64)
    pa = np.zeros((max(n, 1), MAX_DEGREE + 1), np.int64)
    npc = C.c_size_t()
    ops = C.c_uint64()
    err = RpError()
    P = lambda x: x.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    _check(lib().rp_accumulate(P(t), P(b), C.c_size_t(n), D, accum_bits, P(pt), P(pa),
                               C.byref(npc), C.byref(ops), C.byref(err)), err)
    return pt[: npc.value], pa[: npc.value], ops.value


def composite(piece_t, piece_a, qc: RpQuanta, D: int, tf, step: float, t_min: float,
              t_max: float):
    pt = np.ascontiguousarray(piece_t, dtype=np.int64)
    pa = np.ascontiguousarray(piece_a, dtype=np.int64).reshape(-1, MAX_DEGREE + 1)
    tfa, ntf = _tf(tf)
    out = (C.c_double * 4)()
    err = RpError()
    P = lambda x: x.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    _check(lib().rp_composite(P(pt), P(pa), C.c_size_t(len(pt)), C.byref(qc), D, tfa,
                              C.c_size_t(ntf), C.c_double(step), C.c_double(t_min),
                              C.c_double(t_max), out, C.byref(err)), err)
    return tuple(out)


def pipeline(particles, cam: Camera, lut: Lut, qc: RpQuanta, threads: int = 0,
             region=(0, 0, 0, 0)):
    """Sweeps 1-2 + accumulate<Int128>: dict of CSR arrays (rays, knots, pieces, ops);
    `region` (x0, y0, w, h) restricts the rays to those pixels (w == 0: the frame)."""
    a = as_particles(particles)
    c = cam.c()
    err = RpError()
    R = [int(v) for v in region]
    h = lib().rp_pipeline_run_region(_pp(a), C.c_size_t(len(a)), C.byref(c), C.c_void_p(lut.h),
                                     C.byref(qc), threads, *R, C.byref(err))
    if not h:
        raise RefError(err)
    try:
        nr, nk, npc, D = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        lib().rp_pipeline_sizes(C.c_void_p(h), C.byref(nr), C.byref(nk), C.byref(npc),
                                C.byref(D))
        nr, nk, npc, D = nr.value, nk.value, npc.value, D.value
        out = dict(
            D=D,
            rays=np.zeros(nr, np.uint64),
            knot_off=np.zeros(nr + 1, np.uint64),
            knot_t=np.zeros(nk, np.int64),
            knot_b=np.zeros((nk, D + 1), np.int64),
            piece_off=np.zeros(nr + 1, np.uint64),
            piece_t=np.zeros(npc, np.int64),
            piece_a=np.zeros((npc, D + 1), np.int64),
            piece_fits=np.zeros(npc, np.uint8),
            ray_ops=np.zeros(nr, np.uint64),
        )
        P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
        lib().rp_pipeline_get(C.c_void_p(h), *[P(out[k]) for k in (
            "rays", "knot_off", "knot_t", "knot_b", "piece_off", "piece_t", "piece_a",
            "piece_fits", "ray_ops")])
        return out
    finally:
        lib().rp_pipeline_free(C.c_void_p(h))


def render_banded(particles, cam: Camera, tf, lut: Lut, qc: RpQuanta, step: float, row_mask,
                  threads: int = 0, accum_bits: int = 64):
    a = as_particles(particles)
    c = cam.c()
    tfa, ntf = _tf(tf)
    mask = np.ascontiguousarray(row_mask, dtype=np.uint8)
    sec, rays, knots, s = C.c_double(), C.c_uint64(), C.c_uint64(), C.c_double()
    err = RpError()
    _check(lib().rp_render_banded(_pp(a), C.c_size_t(len(a)), C.byref(c), tfa, C.c_size_t(ntf),
                                  C.c_void_p(lut.h), C.byref(qc), C.c_double(step), threads,
                                  accum_bits, mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                                  C.byref(sec), C.byref(rays), C.byref(knots), C.byref(s),
                                  C.byref(err)), err)
    return dict(seconds=sec.value, rays_touched=rays.value, knots=knots.value, rgb_sum=s.value)


def load_particles(path: str) -> np.ndarray:
    err = RpError()
    n = lib().rp_load_particles(path.encode(), None, C.c_size_t(0), C.byref(err))
    if n < 0:
        raise RefError(err)
    out = np.zeros((n, 7), np.float64)
    lib().rp_load_particles(path.encode(), out.ctypes.data_as(C.POINTER(RpParticle)),
                            C.c_size_t(n), C.byref(err))
    return out


def load_tf(path: str) -> np.ndarray:
    err = RpError()
    arr = (RpTf * 256)()
    n = lib().rp_load_tf(path.encode(), arr, C.c_size_t(256), C.byref(err))
    if n < 0:
        raise RefError(err)
    return np.array([[arr[i].value, arr[i].r, arr[i].g, arr[i].b, arr[i].absorption]
                     for i in range(n)], dtype=np.float64)


def load_camera(path: str) -> Camera:
    err = RpError()
    c = RpCamera()
    _check(lib().rp_load_camera(path.encode(), C.byref(c), C.byref(err)), err)
    return Camera(mode="pinhole" if c.mode else "orthographic", position=tuple(c.position),
                  look_at=tuple(c.look_at), up=tuple(c.up), width=c.width, height=c.height,
                  fov_deg=c.fov_deg, ortho_height=c.ortho_height, near=c.near_plane,
                  far=c.far_plane)


def render_region(particles, cam: Camera, tf, lut: Lut, qc: RpQuanta, step: float, x0: int,
                  y0: int, w: int, h: int, background=(0.0, 0.0, 0.0), threads: int = 0,
                  allow_fallback=True):
    """Pixels [x0, x0+w) x [y0, y0+h) of the full-frame render_scene through the
    reference's own sweep functions on the same camera (rp_render_region): returns
    (rgb of rows y0..y0+h-1 (h, W, 3), per-pixel records (RAY_RECORD_DTYPE, row-major
    over the region), stats dict, seconds of the reference sweeps, accumulator bits)."""
    a = as_particles(particles)
    c = cam.c()
    tfa, ntf = _tf(tf)
    y0c = max(0, min(y0, cam.height))
    y1c = max(y0c, min(y0 + h, cam.height))
    x0c = max(0, min(x0, cam.width))
    x1c = max(x0c, min(x0 + w, cam.width))
    rgb = np.zeros((y1c - y0c, cam.width, 3), np.float64)
    rec = np.zeros((y1c - y0c) * (x1c - x0c), RAY_RECORD_DTYPE)
    st, err, sec, bits = RpRStats(), RpError(), C.c_double(), C.c_int()
    bg = (C.c_double * 3)(*background)
    _check(lib().rp_render_region(_pp(a), C.c_size_t(len(a)), C.byref(c), tfa, C.c_size_t(ntf),
                                  C.c_void_p(lut.h), C.byref(qc), C.c_double(step), bg, threads,
                                  x0, y0, w, h, int(bool(allow_fallback)),
                                  rgb.ctypes.data_as(C.POINTER(C.c_double)),
                                  rec.ctypes.data_as(C.c_void_p), C.byref(st), C.byref(sec),
                                  C.byref(bits), C.byref(err)), err)
    stats = {f: getattr(st, f) for f, _ in RpRStats._fields_}
    return rgb, rec, stats, sec.value, bits.value


def render_rows(particles, cam: Camera, tf, lut: Lut, qc: RpQuanta, step: float, row0: int,
                nrows: int, background=(0.0, 0.0, 0.0), threads: int = 0, allow_fallback=True):
    """Full-width rows [row0, row0+nrows): render_region over those rows."""
    return render_region(particles, cam, tf, lut, qc, step, 0, row0, cam.width, nrows,
                         background, threads, allow_fallback)


def generate_scene(config: int, n: int = 0, seed=None) -> np.ndarray:
    """The synthetic scenes of BASELINE.json (include/sphray_scenes.hpp, compiled into
    oracle/_ref): byte-identical to the product's sphray_generate_scene."""
    if seed is None:
        seed = 7 if config in (3, 5) else 42
    if n == 0:
        n = lib().rp_scene_default_count(int(config))
    out = np.zeros((n, 7), np.float64)
    err = RpError()
    _check(lib().rp_generate_scene(int(config), C.c_size_t(n), C.c_uint64(seed), _pp(out),
                                   C.byref(err)), err)
    return out


def piece_mix(t, a, D: int) -> np.ndarray:
    """sphray_piece_mix (include/sphray_gpu.h) vectorised over pieces (t (P,), a (P, >=D+1))."""
    M = np.array([0x9E3779B97F4A7C15, 0xC2B2AE3D27D4EB4F, 0x165667B19E3779F9,
                  0x27D4EB2F165667C5, 0x94D049BB133111EB, 0xBF58476D1CE4E5B9,
                  0xD6E8FEB86659FD93, 0xFF51AFD7ED558CCD], dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.asarray(t, np.int64).view(np.uint64) * M[0]
        A = np.asarray(a, np.int64).view(np.uint64)
        for d in range(D + 1):
            x = x + A[:, d] * M[d + 1]
        x = x ^ (x >> np.uint64(31))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(29))
    return x


def render_report(particles, cam: Camera, tf, lut: Lut, int_width: int = 64, seed: int = 0,
                  image: str = "") -> str:
    """The reference CLI's render report JSON text (rp_render_report)."""
    a = as_particles(particles)
    c = cam.c()
    tfa, ntf = _tf(tf)
    err = RpError()
    args = (_pp(a), C.c_size_t(len(a)), C.byref(c), tfa, C.c_size_t(ntf), C.c_void_p(lut.h),
            int_width, C.c_uint64(seed), image.encode())
    n = lib().rp_render_report(*args, None, C.c_size_t(0), C.byref(err))
    if n < 0:
        raise RefError(err)
    buf = C.create_string_buffer(n + 1)
    lib().rp_render_report(*args, buf, C.c_size_t(n + 1), C.byref(err))
    return buf.value.decode()

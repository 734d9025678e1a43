"""ctypes wrapper of oracle/_build/libsphray_oracle.so (oracle/sphray_oracle.c) --
TEST INFRASTRUCTURE: the plain-C restatement of the reference path, the checker
for the GPU parity tests and the ``kind: port`` CPU baseline.  Never product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libsphray_oracle.so")


class OpCamera(C.Structure):
    _fields_ = [("mode", C.c_int), ("width", C.c_int), ("height", C.c_int),
                ("position", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_deg", C.c_double), ("ortho_height", C.c_double),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class OpLut(C.Structure):
    _fields_ = [("q", C.c_double), ("K", C.c_int), ("D", C.c_int), ("N", C.c_int),
                ("records", C.POINTER(C.c_double))]


class OpStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("particles", "skipped_particles", "knots",
                                           "rays_touched", "int_ops", "residual_failures")] + [
        ("step", C.c_double)]


class PortError(RuntimeError):
    def __init__(self, code, msg=""):
        self.code = code
        super().__init__(f"oracle port error {code} {msg}")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.check_call(["make", "-s", "-C", HERE, "port"])
        _lib = C.CDLL(LIB_PATH)
    return _lib


def camera(mode="orthographic", position=(0, 0, 0), look_at=(0, 0, -1), up=(0, 1, 0), width=64,
           height=64, fov_deg=60.0, ortho_height=2.0, near=0.0, far=1e30) -> OpCamera:
    c = OpCamera()
    c.mode = 1 if mode == "pinhole" else 0
    c.width, c.height = width, height
    c.position[:] = [float(v) for v in position]
    c.look_at[:] = [float(v) for v in look_at]
    c.up[:] = [float(v) for v in up]
    c.fov_deg, c.ortho_height, c.near_plane, c.far_plane = fov_deg, ortho_height, near, far
    return c


class Lut:
    """.splt file -> op_lut (records copied 8-byte aligned)."""

    def __init__(self, path: str):
        raw = open(path, "rb").read()
        assert raw[:4] == b"SPLT"
        self.q = np.frombuffer(raw[24:32], "<f8")[0]
        self.K, self.D, self.N = (int(np.frombuffer(raw[o:o + 4], "<u4")[0]) for o in (32, 36, 40))
        self.records = np.frombuffer(raw[44:], "<f8").copy()
        self.c = OpLut(self.q, self.K, self.D, self.N,
                       self.records.ctypes.data_as(C.POINTER(C.c_double)))


def _pp(a):
    return np.ascontiguousarray(a, np.float64).ctypes.data_as(C.c_void_p)


def footprint_particle(p, cam: OpCamera, q: float):
    p = np.ascontiguousarray(p, np.float64)
    n = C.c_size_t()
    lib().op_footprint(_pp(p), C.byref(cam), C.c_double(q), None, None, None, C.c_size_t(0),
                       C.byref(n))
    k = n.value
    ray = np.zeros(k, np.uint64)
    lam = np.zeros(k, np.float64)
    tchi = np.zeros(k, np.float64)
    rc = lib().op_footprint(_pp(p), C.byref(cam), C.c_double(q), ray.ctypes.data_as(C.c_void_p),
                            lam.ctypes.data_as(C.c_void_p), tchi.ctypes.data_as(C.c_void_p),
                            C.c_size_t(k), C.byref(n))
    if rc:
        raise PortError(rc)
    return ray, lam, tchi


def footprint(particles, cam: OpCamera, q: float):
    rays, pids, lams, ts = [], [], [], []
    for i, p in enumerate(np.asarray(particles, np.float64).reshape(-1, 7)):
        r, l, t = footprint_particle(p, cam, q)
        rays.append(r)
        pids.append(np.full(len(r), i, np.int64))
        lams.append(l)
        ts.append(t)
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)  # noqa: E731
    return cat(rays, np.uint64), cat(pids, np.int64), cat(lams, np.float64), cat(ts, np.float64)


def lut_index(lut: Lut, lam: float) -> int:
    lib().op_lut_index.restype = C.c_int
    return lib().op_lut_index(C.byref(lut.c), C.c_double(lam))


def quantize(p, t_chi: float, lam: float, lut: Lut, tau: float, sigma: float):
    t = np.zeros(9, np.int64)
    b = np.zeros((9, 7), np.int64)
    n = C.c_int()
    rc = lib().op_quantize(_pp(np.asarray(p, np.float64)), C.c_double(t_chi), C.c_double(lam),
                           C.byref(lut.c), C.c_double(tau), C.c_double(sigma),
                           t.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), C.byref(n))
    if rc:
        raise PortError(rc)
    return t[: n.value], b[: n.value]


def accumulate(t, b, D: int):
    t = np.ascontiguousarray(t, np.int64)
    bb = np.zeros((len(t), 7), np.int64)
    if len(t):
        b = np.asarray(b, np.int64).reshape(len(t), -1)
        bb[:, : b.shape[1]] = b
    pt = np.zeros(max(1, len(t)), np.int64)
    pa = np.zeros((max(1, len(t)), 7), np.int64)
    np_ = C.c_size_t()
    ops = C.c_uint64()
    rc = lib().op_accumulate(t.ctypes.data_as(C.c_void_p), bb.ctypes.data_as(C.c_void_p),
                             C.c_size_t(len(t)), C.c_int(D), pt.ctypes.data_as(C.c_void_p),
                             pa.ctypes.data_as(C.c_void_p), C.byref(np_), C.byref(ops))
    if rc and rc != 3:
        raise PortError(rc)
    return pt[: np_.value], pa[: np_.value], ops.value, rc == 0


def composite(piece_t, piece_a, tau, sigma, D, tf, step, t_min, t_max):
    pt = np.ascontiguousarray(piece_t, np.int64)
    pa = np.zeros((len(pt), 7), np.int64)
    a = np.asarray(piece_a, np.int64).reshape(len(pt), -1)
    pa[:, : a.shape[1]] = a
    tfa = np.ascontiguousarray(tf, np.float64).reshape(-1, 5)
    out = np.zeros(4, np.float64)
    rc = lib().op_composite(pt.ctypes.data_as(C.c_void_p), pa.ctypes.data_as(C.c_void_p),
                            C.c_size_t(len(pt)), C.c_double(tau), C.c_double(sigma), C.c_int(D),
                            tfa.ctypes.data_as(C.c_void_p), C.c_size_t(len(tfa)),
                            C.c_double(step), C.c_double(t_min), C.c_double(t_max),
                            out.ctypes.data_as(C.c_void_p))
    if rc:
        raise PortError(rc)
    return out


def camera_ray(cam: OpCamera, px: int, py: int):
    o = np.zeros(3)
    d = np.zeros(3)
    rc = lib().op_camera_ray(C.byref(cam), px, py, o.ctypes.data_as(C.c_void_p),
                             d.ctypes.data_as(C.c_void_p))
    if rc:
        raise PortError(rc)
    return o, d


def render(particles, cam: OpCamera, tf, lut: Lut, tau, sigma, h_r, step=0.0, bg=(0, 0, 0)):
    """render_scene (raycast.hpp:414-497), single-threaded, Int128 accumulation."""
    ps = np.ascontiguousarray(particles, np.float64).reshape(-1, 7)
    tfa = np.ascontiguousarray(tf, np.float64).reshape(-1, 5)
    rgb = np.zeros((cam.height, cam.width, 3), np.float64)
    st = OpStats()
    ep, er = C.c_int64(-1), C.c_uint64(0)
    bgv = np.ascontiguousarray(bg, np.float64)
    rc = lib().op_render(ps.ctypes.data_as(C.c_void_p), C.c_size_t(len(ps)), C.byref(cam),
                         tfa.ctypes.data_as(C.c_void_p), C.c_size_t(len(tfa)), C.byref(lut.c),
                         C.c_double(tau), C.c_double(sigma), C.c_double(h_r), C.c_double(step),
                         bgv.ctypes.data_as(C.c_void_p), rgb.ctypes.data_as(C.c_void_p),
                         C.byref(st), C.byref(ep), C.byref(er))
    if rc:
        err = PortError(rc)
        err.particle_index, err.ray_id = ep.value, er.value
        raise err
    return rgb, {f: getattr(st, f) for f, _ in OpStats._fields_}

"""sphray_b200 -- B200-native per-ray higher-order SPH field approximation + DVR.

Host-side mirror of the reference renderer's interface for this path
(/root/reference/proj/include/sphray): the same names, argument meaning and
error behaviour, calling the sm_100a CUDA path through the C-ABI in
``include/sphray_gpu.h`` (``libsphray_b200.so``, built in-tree).  There is no
CPU fallback: without the built library or a CUDA device every render entry
point raises.

Reference interface mirrored (file:line under proj/include/sphray):
  Camera                 raycast.hpp:45-101
  TfPoint / TransferFunction raycast.hpp:303-338
  Lut, load_lut          lut.hpp:32-65, 354-405
  QuantaConfig           quantize.hpp:44-51
  DatasetStats, dataset_stats, choose_quanta  quantize.hpp:31-40, 129-183
  RenderOptions, RenderStats, render_scene    raycast.hpp:394-497
  Error hierarchy        errors.hpp:12-69
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "Error", "ConfigError", "IoError", "OverflowError", "NumericError", "CudaError",
    "NcclError", "CapacityError", "Camera", "TfPoint", "TransferFunction", "Lut", "load_lut",
    "QuantaConfig", "DatasetStats", "RenderOptions", "RenderStats", "Image", "Context",
    "render_scene", "dataset_stats", "choose_quanta", "generate_scene", "lib_path", "load_library",
    "MODE_EXACT", "MODE_FAST", "KAPPA_CUBIC", "KAPPA_PRIME_CUBIC",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libsphray_b200.so"

MODE_EXACT = 0
MODE_FAST = 1
# kernel_constants(cubic_bspline()) as the reference computes them (kernel.hpp:158-190)
KAPPA_CUBIC = float.fromhex("0x1.68a53e31586eap-2")
KAPPA_PRIME_CUBIC = float.fromhex("0x1.5c74590f520d8p-3")


# --------------------------------------------------------------------------- errors
class Error(RuntimeError):
    """sphray::Error (errors.hpp:12-15)."""


class ConfigError(Error):
    """sphray::ConfigError (errors.hpp:18-21)."""


class IoError(Error):
    """sphray::IoError (errors.hpp:24-27)."""


class OverflowError(Error):  # noqa: A001 -- mirrors sphray::OverflowError
    """sphray::OverflowError (errors.hpp:54-63): carries particle_index and ray_id."""

    def __init__(self, msg: str, particle_index: int = -1, ray_id: int = 0):
        super().__init__(msg)
        self.particle_index = particle_index
        self.ray_id = ray_id


class NumericError(Error):
    """sphray::NumericError (errors.hpp:66-69)."""


class CudaError(Error):
    """Device failure or no CUDA device (the path has no CPU fallback)."""


class NcclError(Error):
    """Tile-gather failure."""


class CapacityError(Error):
    """A ray's pending-knot window exceeded every window size."""


_STATUS = {1: ConfigError, 2: IoError, 3: OverflowError, 4: NumericError, 5: CudaError,
           6: NcclError, 7: CapacityError}


# --------------------------------------------------------------------------- C structs
class _Particle(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("x", "y", "z", "mass", "density", "h", "value")]


class _Camera(C.Structure):
    _fields_ = [("mode", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("reserved", C.c_int32), ("position", C.c_double * 3),
                ("look_at", C.c_double * 3), ("up", C.c_double * 3), ("fov_deg", C.c_double),
                ("ortho_height", C.c_double), ("near_plane", C.c_double),
                ("far_plane", C.c_double)]


class _TfPoint(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("value", "r", "g", "b", "absorption")]


class _ValidateReport(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("telescoping_rays", "telescoping_bad",
                                          "superposition_rays", "superposition_bad",
                                          "l2_rays", "l2_bad")] + \
               [("l2_envelope", C.c_double), ("l2_fraction_within", C.c_double)] + \
               [(n, C.c_int32) for n in ("telescoping_pass", "superposition_pass", "l2_pass",
                                         "pass_")]


class _LutView(C.Structure):
    _fields_ = [("q", C.c_double), ("K", C.c_int32), ("D", C.c_int32), ("N", C.c_int32),
                ("reserved", C.c_int32), ("records", C.POINTER(C.c_double))]


class _Quanta(C.Structure):
    _fields_ = [("tau", C.c_double), ("sigma", C.c_double), ("int_width", C.c_int32),
                ("reserved", C.c_int32)]


class _DStats(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mass_r", "density_r", "h_r", "value_r", "phi_repr",
                                           "a_max", "clustering_factor")] + [
        ("count", C.c_uint64)]


class _Options(C.Structure):
    _fields_ = [("step", C.c_double), ("background", C.c_double * 3), ("threads", C.c_int32),
                ("mode", C.c_int32), ("window", C.c_int32), ("reserved", C.c_int32)]


class _RStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("particles", "skipped_particles", "knots",
                                           "rays_touched", "int_ops", "residual_failures")] + [
        ("step", C.c_double)] + [(n, C.c_uint64) for n in (
            "hits", "candidates", "window_retries", "max_window")] + [
        ("device_ms", C.c_double), ("bin_ms", C.c_double), ("render_ms", C.c_double),
        ("launches", C.c_uint64), ("terminated_rays", C.c_uint64)]


class _RayRecord(C.Structure):
    _fields_ = [("piece_checksum", C.c_uint64), ("knots", C.c_uint32), ("pieces", C.c_uint32),
                ("hits", C.c_uint32), ("flags", C.c_uint32)]


RAY_RECORD_DTYPE = np.dtype([("piece_checksum", "<u8"), ("knots", "<u4"), ("pieces", "<u4"),
                             ("hits", "<u4"), ("flags", "<u4")])
RAY_TOUCHED, RAY_RESIDUAL, RAY_TERMINATED = 1, 2, 4


class _Error(C.Structure):
    _fields_ = [("code", C.c_int32), ("reserved", C.c_int32), ("particle_index", C.c_int64),
                ("ray_id", C.c_uint64), ("msg", C.c_char * 256)]


_lib = None


def lib_path() -> str:
    return os.environ.get("SPHRAY_B200_LIB", os.path.join(HERE, LIB_NAME))


def load_library():
    """Loads the in-tree C-ABI library; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise CudaError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; "
                        "g.build()'` (the sm_100a path has no CPU fallback)")
    L = C.CDLL(path)
    P = C.POINTER
    L.sphray_abi_version.restype = C.c_int
    L.sphray_build_info.restype = C.c_char_p
    L.sphray_context_create.argtypes = [C.c_int, P(C.c_void_p), P(_Error)]
    L.sphray_context_destroy.argtypes = [C.c_void_p]
    L.sphray_probe_alu_peaks.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(_Error)]
    L.sphray_comm_unique_id.argtypes = [C.c_char_p, P(_Error)]
    L.sphray_context_init_comm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, P(_Error)]
    L.sphray_context_set_shard.argtypes = [C.c_void_p, C.c_int, C.c_int, P(_Error)]
    L.sphray_context_set_region.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_int32, P(_Error)]
    L.sphray_scene_info.argtypes = [C.c_void_p, P(C.c_size_t), P(C.c_int32), P(C.c_int32), P(_Error)]
    L.sphray_context_ray_records.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, P(C.c_size_t),
                                             P(_Error)]
    L.sphray_render_scene.argtypes = [C.c_void_p, P(_Particle), C.c_size_t, P(_Camera),
                                      P(_TfPoint), C.c_size_t, P(_LutView), P(_Quanta),
                                      P(_DStats), P(_Options), P(C.c_double), P(_RStats),
                                      P(_Error)]
    L.sphray_scene_upload.argtypes = [C.c_void_p, P(_Particle), C.c_size_t, P(_LutView), P(_Error)]
    L.sphray_scene_render.argtypes = [C.c_void_p, P(_Camera), P(_TfPoint), C.c_size_t,
                                      P(_Quanta), P(_DStats), P(_Options), P(C.c_double),
                                      P(_RStats), P(_Error)]
    L.sphray_scene_device_image.argtypes = [C.c_void_p]
    L.sphray_scene_device_image.restype = C.c_void_p
    L.sphray_context_stream.argtypes = [C.c_void_p]
    L.sphray_context_stream.restype = C.c_void_p
    L.sphray_scene_hits.argtypes = [C.c_void_p, P(_Camera), P(C.c_uint64), P(C.c_int64),
                                    P(C.c_double), P(C.c_double), C.c_size_t, P(C.c_size_t),
                                    P(_Error)]
    L.sphray_scene_pieces.argtypes = [C.c_void_p, P(_Camera), P(_Quanta), P(C.c_uint64),
                                      P(C.c_uint64), P(C.c_int64), P(C.c_int64), C.c_size_t,
                                      C.c_size_t, P(C.c_size_t), P(C.c_size_t), P(_Error)]
    L.sphray_quantize_hits.argtypes = [C.c_void_p, P(_Particle), C.c_size_t, P(C.c_double),
                                       P(C.c_double), P(_LutView), P(_Quanta), P(C.c_int64),
                                       P(C.c_int64), P(C.c_int32), P(_Error)]
    L.sphray_compute_dataset_stats.argtypes = [P(_Particle), C.c_size_t, P(_LutView), C.c_double,
                                               P(_DStats), P(_Error)]
    L.sphray_particles_load.argtypes = [C.c_char_p, P(P(_Particle)), P(C.c_size_t), P(_Error)]
    L.sphray_particles_save.argtypes = [C.c_char_p, P(_Particle), C.c_size_t, C.c_int, P(_Error)]
    L.sphray_tf_load.argtypes = [C.c_char_p, P(P(_TfPoint)), P(C.c_size_t), P(_Error)]
    L.sphray_ppm_save.argtypes = [C.c_char_p, P(C.c_double), C.c_int, C.c_int, P(_Error)]
    L.sphray_free.argtypes = [C.c_void_p]
    L.sphray_camera_load.argtypes = [C.c_char_p, P(_Camera), P(_Error)]
    L.sphray_scene_upload_file.argtypes = [C.c_void_p, C.c_char_p, P(_LutView), P(_Error)]
    L.sphray_scene_validate.argtypes = [C.c_void_p, P(_Camera), P(_Quanta), P(_DStats),
                                        P(_ValidateReport), P(_Error)]
    L.sphray_scene_dataset_stats.argtypes = [C.c_void_p, C.c_double, P(_DStats), P(_Error)]
    L.sphray_choose_quanta.argtypes = [P(_LutView), P(_DStats), C.c_int, C.c_double, C.c_double,
                                       P(_Quanta), P(_Error)]
    L.sphray_lut_parse.argtypes = [C.c_void_p, C.c_size_t, P(_LutView), C.c_char_p, P(_Error)]
    L.sphray_generate_scene.argtypes = [C.c_int, C.c_size_t, C.c_uint64, P(_Particle), P(_Error)]
    L.sphray_accumulate.argtypes = [C.c_void_p, C.c_int, C.c_size_t] + [C.c_void_p] * 8 + [P(_Error)]
    L.sphray_lut_serialize.argtypes = [P(_LutView), C.c_char_p, C.c_void_p, C.c_size_t, P(C.c_size_t),
                                       P(_Error)]
    L.sphray_lut_save.argtypes = [C.c_char_p, P(_LutView), C.c_char_p, P(_Error)]
    L.sphray_render_report.argtypes = [P(_LutView), C.c_char_p, P(_DStats), P(_Quanta), P(_RStats),
                                       C.c_uint64, C.c_char_p, C.c_double, C.c_double, C.c_char_p,
                                       C.c_size_t, P(C.c_size_t), P(_Error)]
    L.sphray_scene_default_count.argtypes = [C.c_int]
    L.sphray_scene_default_count.restype = C.c_size_t
    for name in ("sphray_context_create", "sphray_comm_unique_id", "sphray_context_init_comm",
                 "sphray_context_set_shard", "sphray_context_set_region", "sphray_scene_info",
                 "sphray_context_ray_records",
                 "sphray_render_scene", "sphray_scene_upload", "sphray_scene_render",
                 "sphray_scene_hits", "sphray_scene_pieces", "sphray_quantize_hits",
                 "sphray_compute_dataset_stats", "sphray_choose_quanta", "sphray_lut_parse",
                 "sphray_generate_scene", "sphray_lut_serialize", "sphray_accumulate", "sphray_lut_save",
                 "sphray_render_report"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int, err: _Error):
    if rc == 0:
        return
    msg = err.msg.decode(errors="replace")
    cls = _STATUS.get(rc, Error)
    if cls is OverflowError:
        raise OverflowError(msg, err.particle_index, err.ray_id)
    raise cls(msg)


# --------------------------------------------------------------------------- value types
@dataclass
class Camera:
    """sphray::Camera (raycast.hpp:45-58); mode 'orthographic' or 'pinhole'."""
    mode: str = "orthographic"
    position: Sequence[float] = (0.0, 0.0, 0.0)
    look_at: Sequence[float] = (0.0, 0.0, -1.0)
    up: Sequence[float] = (0.0, 1.0, 0.0)
    width: int = 64
    height: int = 64
    fov_deg: float = 60.0
    ortho_height: float = 2.0
    near: float = 0.0
    far: float = 1e30

    def _c(self) -> _Camera:
        c = _Camera()
        if self.mode not in ("orthographic", "pinhole"):
            raise ConfigError("camera json: mode must be 'orthographic' or 'pinhole'")
        c.mode = 1 if self.mode == "pinhole" else 0
        c.width, c.height = int(self.width), int(self.height)
        c.position[:] = [float(v) for v in self.position]
        c.look_at[:] = [float(v) for v in self.look_at]
        c.up[:] = [float(v) for v in self.up]
        c.fov_deg, c.ortho_height = float(self.fov_deg), float(self.ortho_height)
        c.near_plane, c.far_plane = float(self.near), float(self.far)
        return c


@dataclass
class TfPoint:
    value: float = 0.0
    r: float = 0.0
    g: float = 0.0
    b: float = 0.0
    absorption: float = 0.0


@dataclass
class TransferFunction:
    """sphray::TransferFunction (raycast.hpp:313-338)."""
    points: list = field(default_factory=list)

    @classmethod
    def from_array(cls, arr) -> "TransferFunction":
        a = np.asarray(arr, dtype=np.float64).reshape(-1, 5)
        return cls([TfPoint(*row) for row in a])

    def _c(self):
        n = len(self.points)
        arr = (_TfPoint * max(1, n))()
        for i, p in enumerate(self.points):
            if isinstance(p, TfPoint):
                arr[i] = _TfPoint(p.value, p.r, p.g, p.b, p.absorption)
            else:
                arr[i] = _TfPoint(*[float(v) for v in p])
        return arr, n


@dataclass
class QuantaConfig:
    """sphray::QuantaConfig (quantize.hpp:44-51)."""
    tau: float = 0.0
    sigma: float = 0.0
    width: int = 64

    def _c(self) -> _Quanta:
        return _Quanta(self.tau, self.sigma, int(self.width), 0)


@dataclass
class DatasetStats:
    """sphray::DatasetStats (quantize.hpp:31-40)."""
    mass_r: float = 0.0
    density_r: float = 0.0
    h_r: float = 0.0
    value_r: float = 0.0
    phi_repr: float = 0.0
    a_max: float = 0.0
    clustering_factor: float = 0.0
    count: int = 0

    def _c(self) -> _DStats:
        return _DStats(self.mass_r, self.density_r, self.h_r, self.value_r, self.phi_repr,
                       self.a_max, self.clustering_factor, int(self.count))

    @classmethod
    def _from(cls, s: _DStats) -> "DatasetStats":
        return cls(s.mass_r, s.density_r, s.h_r, s.value_r, s.phi_repr, s.a_max,
                   s.clustering_factor, s.count)


@dataclass
class RenderOptions:
    """sphray::RenderOptions (raycast.hpp:394-398) + the device-side mode/window knobs."""
    step: float = 0.0
    background: Sequence[float] = (0.0, 0.0, 0.0)
    threads: int = 1
    mode: int = MODE_EXACT
    window: int = 0

    def _c(self) -> _Options:
        o = _Options()
        o.step = float(self.step)
        o.background[:] = [float(v) for v in self.background]
        o.threads, o.mode, o.window = int(self.threads), int(self.mode), int(self.window)
        return o


@dataclass
class RenderStats:
    """sphray::RenderStats (raycast.hpp:400-408) + path counters."""
    particles: int = 0
    skipped_particles: int = 0
    knots: int = 0
    rays_touched: int = 0
    int_ops: int = 0
    residual_failures: int = 0
    step: float = 0.0
    hits: int = 0
    candidates: int = 0
    window_retries: int = 0
    max_window: int = 0
    device_ms: float = 0.0
    bin_ms: float = 0.0
    render_ms: float = 0.0
    launches: int = 0
    terminated_rays: int = 0

    @classmethod
    def _from(cls, s: _RStats) -> "RenderStats":
        return cls(**{f: getattr(s, f) for f, _ in _RStats._fields_})


@dataclass
class Image:
    """sphray::Image (raycast.hpp:383-392): pixels (H, W, 3) float64, top row first."""
    width: int
    height: int
    pixels: np.ndarray


class Lut:
    """sphray::Lut (lut.hpp:32-65) held as the raw .splt bytes."""

    def __init__(self, data: bytes):
        self._buf = np.frombuffer(bytes(data), dtype=np.uint8).copy()  # 8-byte aligned copy
        L = load_library()
        self._view = _LutView()
        kid = C.create_string_buffer(17)
        err = _Error()
        _check(L.sphray_lut_parse(self._buf.ctypes.data, self._buf.size, C.byref(self._view), kid,
                                  C.byref(err)), err)
        self.kernel_id = kid.value.decode()
        # 8-byte aligned copy of the records (the .splt header is 44 bytes)
        self._records = np.frombuffer(self._buf[44:].tobytes(), dtype="<f8").copy()
        self._view.records = self._records.ctypes.data_as(C.POINTER(C.c_double))
        self.q, self.K, self.D, self.N = self._view.q, self._view.K, self._view.D, self._view.N

    @property
    def view(self) -> _LutView:
        return self._view

    def records(self) -> np.ndarray:
        m, nj = (self.K + 1) // 2, self.K * self.D // 2
        return self._records.reshape(self.N, 2 + m + nj)

    def serialize(self) -> bytes:
        """serialize_lut (lut.hpp:335-352): the .splt file image."""
        L = load_library()
        n, err = C.c_size_t(), _Error()
        kid = self.kernel_id.encode()
        _check(L.sphray_lut_serialize(C.byref(self._view), kid, None, 0, C.byref(n), C.byref(err)), err)
        out = (C.c_uint8 * n.value)()
        _check(L.sphray_lut_serialize(C.byref(self._view), kid, out, n.value, C.byref(n), C.byref(err)), err)
        return bytes(out)


def save_lut(lut: "Lut", path: str) -> None:
    """save_lut (lut.hpp:395-399)."""
    L = load_library()
    err = _Error()
    _check(L.sphray_lut_save(os.fsencode(path), C.byref(lut.view), lut.kernel_id.encode(), C.byref(err)), err)


def render_report(lut: "Lut", stats: "DatasetStats", qc: "QuantaConfig", rstats: "RenderStats",
                  seed: int = 0, image: str = "") -> str:
    """The reference CLI's `render` report JSON (sphray_main.cpp:196-256)."""
    L = load_library()
    ds, q = stats._c(), qc._c()
    rs = _RStats(**{f: getattr(rstats, f) for f, _ in _RStats._fields_}) if rstats is not None else None
    n, err = C.c_size_t(), _Error()
    args = (C.byref(lut.view), lut.kernel_id.encode(), C.byref(ds), C.byref(q),
            C.byref(rs) if rs is not None else None, C.c_uint64(seed), image.encode(), 0.0, 0.0)
    _check(L.sphray_render_report(*args, None, 0, C.byref(n), C.byref(err)), err)
    buf = C.create_string_buffer(n.value + 1)
    _check(L.sphray_render_report(*args, buf, n.value + 1, C.byref(n), C.byref(err)), err)
    return buf.value.decode()


def load_lut(path: str) -> Lut:
    """load_lut (lut.hpp:401-405)."""
    try:
        with open(path, "rb") as f:
            return Lut(f.read())
    except FileNotFoundError as e:
        raise IoError(f"lut: cannot open {path}") from e


def _particles(arr) -> np.ndarray:
    a = np.ascontiguousarray(arr, dtype=np.float64)
    if a.ndim == 1 and a.size % 7 == 0:
        a = a.reshape(-1, 7)
    if a.ndim != 2 or a.shape[1] != 7:
        raise ConfigError("particles must be an (n, 7) array of x,y,z,mass,density,h,value")
    return a


def _pp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(_Particle)) if a.size else None


def dataset_stats(particles, lut: Lut, clustering_factor: float = 16.0) -> DatasetStats:
    """dataset_stats (quantize.hpp:129-165), restated natively."""
    L = load_library()
    a = _particles(particles)
    out, err = _DStats(), _Error()
    _check(L.sphray_compute_dataset_stats(_pp(a), len(a), C.byref(lut.view), clustering_factor,
                                          C.byref(out), C.byref(err)), err)
    return DatasetStats._from(out)


def choose_quanta(lut: Lut, stats: DatasetStats, width: int = 64,
                  kappa: float = KAPPA_CUBIC, kappa_prime: float = KAPPA_PRIME_CUBIC) -> QuantaConfig:
    """choose_quanta (quantize.hpp:169-183) with the cubic B-spline's kernel constants."""
    L = load_library()
    out, err = _Quanta(), _Error()
    ds = stats._c()
    _check(L.sphray_choose_quanta(C.byref(lut.view), C.byref(ds), int(width), kappa, kappa_prime,
                                  C.byref(out), C.byref(err)), err)
    return QuantaConfig(out.tau, out.sigma, out.int_width)


def load_particles(path: str) -> np.ndarray:
    """load_particles (io.hpp:141-151): SPRT binary or CSV -> (n, 7) float64
    rows x, y, z, mass, density, h, value."""
    L = load_library()
    ptr, n, err = C.POINTER(_Particle)(), C.c_size_t(), _Error()
    _check(L.sphray_particles_load(os.fsencode(path), C.byref(ptr), C.byref(n), C.byref(err)), err)
    try:
        out = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(n.value * 7,)).copy()
    finally:
        L.sphray_free(ptr)
    return out.reshape(n.value, 7)


def save_particles(particles, path: str, binary: bool = False) -> None:
    """save_particles (io.hpp:153-161)."""
    L = load_library()
    a = _particles(particles)
    err = _Error()
    _check(L.sphray_particles_save(os.fsencode(path), _pp(a), len(a), int(binary), C.byref(err)), err)


def load_transfer_function(path: str) -> "TransferFunction":
    """load_transfer_function (io.hpp:158-190): sorted, validated."""
    L = load_library()
    ptr, n, err = C.POINTER(_TfPoint)(), C.c_size_t(), _Error()
    _check(L.sphray_tf_load(os.fsencode(path), C.byref(ptr), C.byref(n), C.byref(err)), err)
    try:
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(n.value * 5,)).copy()
    finally:
        L.sphray_free(ptr)
    return TransferFunction.from_array(arr.reshape(n.value, 5))


def load_camera(path: str) -> "Camera":
    """load_camera (io.hpp:294-304)."""
    L = load_library()
    c, err = _Camera(), _Error()
    _check(L.sphray_camera_load(os.fsencode(path), C.byref(c), C.byref(err)), err)
    return Camera(mode="pinhole" if c.mode == 1 else "orthographic", position=tuple(c.position),
                  look_at=tuple(c.look_at), up=tuple(c.up), width=c.width, height=c.height,
                  fov_deg=c.fov_deg, ortho_height=c.ortho_height, near=c.near_plane,
                  far=c.far_plane)


def save_ppm(rgb, path: str) -> None:
    """save_ppm (io.hpp:193-210): (H, W, 3) linear RGB clamped to [0, 1], 8 bits."""
    L = load_library()
    a = np.ascontiguousarray(rgb, dtype=np.float64)
    err = _Error()
    _check(L.sphray_ppm_save(os.fsencode(path), a.ctypes.data_as(C.POINTER(C.c_double)),
                             a.shape[1], a.shape[0], C.byref(err)), err)


def probe_alu_peaks(device: int = 0) -> dict:
    """Measured int64 multiply/add and fp64 FMA issue peaks of `device`."""
    L = load_library()
    gi, gf, err = C.c_double(), C.c_double(), _Error()
    _check(L.sphray_probe_alu_peaks(device, C.byref(gi), C.byref(gf), C.byref(err)), err)
    return {"int64_gops": gi.value, "fp64_gflops": gf.value}


def generate_scene(config: int, n: int = 0, seed: Optional[int] = None) -> np.ndarray:
    """Synthetic SPH scenes of BASELINE.json configs 1-5: (n, 7) float64."""
    L = load_library()
    if n == 0:
        n = L.sphray_scene_default_count(int(config))
    if seed is None:
        seed = 7 if config in (3, 5) else 42
    out = np.zeros((n, 7), dtype=np.float64)
    err = _Error()
    _check(L.sphray_generate_scene(int(config), n, C.c_uint64(seed), _pp(out), C.byref(err)), err)
    return out


class Context:
    """One CUDA device: resident scene + frame renders (sphray_context)."""

    def __init__(self, device: int = 0):
        self._L = load_library()
        self._h = C.c_void_p()
        err = _Error()
        _check(self._L.sphray_context_create(int(device), C.byref(self._h), C.byref(err)), err)
        self._lut = None
        self._n = 0

    def close(self):
        if self._h:
            self._L.sphray_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @staticmethod
    def comm_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        err = _Error()
        _check(L.sphray_comm_unique_id(buf, C.byref(err)), err)
        return buf.raw

    def init_comm(self, rank: int, nranks: int, unique_id: bytes):
        """NCCL communicator for the tile gather: render() then returns the full image."""
        err = _Error()
        _check(self._L.sphray_context_init_comm(self._h, rank, nranks, unique_id, C.byref(err)), err)
        self._shard = (0, 1)

    def set_shard(self, rank: int, nranks: int):
        """Render only tiles t with t % nranks == rank; render() then returns them packed."""
        err = _Error()
        _check(self._L.sphray_context_set_shard(self._h, rank, nranks, C.byref(err)), err)
        self._shard = (rank, nranks)

    def set_region(self, x0: int = 0, y0: int = 0, w: int = 0, h: int = 0, record: bool = False):
        """Trace only pixels [x0, x0+w) x [y0, y0+h) of later frames (the same rays
        as the full frame; w or h == 0: full frames); render() then returns rows
        y0 .. y0+h-1.  record: keep one per-ray record (knots, pieces, hits,
        flags, piece checksum) per pixel of the region, row-major."""
        err = _Error()
        _check(self._L.sphray_context_set_region(self._h, int(x0), int(y0), int(w), int(h),
                                                 int(bool(record)), C.byref(err)), err)
        self._rows = (int(y0), int(h) if w > 0 else 0)

    def scene_info(self) -> dict:
        """The resident scene: particle count n and the LUT's K, D (sphray_scene_info)."""
        n, K, D, err = C.c_size_t(), C.c_int32(), C.c_int32(), _Error()
        _check(self._L.sphray_scene_info(self._h, C.byref(n), C.byref(K), C.byref(D), C.byref(err)), err)
        return {"n": n.value, "K": K.value, "D": D.value}

    def ray_records(self) -> np.ndarray:
        """Per-ray records of the last frame (row-major over the band), RAY_RECORD_DTYPE."""
        cnt, err = C.c_size_t(), _Error()
        _check(self._L.sphray_context_ray_records(self._h, None, 0, C.byref(cnt), C.byref(err)), err)
        out = np.zeros(cnt.value, RAY_RECORD_DTYPE)
        _check(self._L.sphray_context_ray_records(self._h, out.ctypes.data_as(C.c_void_p), len(out),
                                                  C.byref(cnt), C.byref(err)), err)
        return out

    def upload(self, particles, lut: Lut):
        a = _particles(particles)
        err = _Error()
        _check(self._L.sphray_scene_upload(self._h, _pp(a), len(a), C.byref(lut.view),
                                           C.byref(err)), err)
        self._lut = lut
        self._n = len(a)

    def render(self, cam: Camera, tf: TransferFunction, qc: QuantaConfig, stats: DatasetStats,
               opts: Optional[RenderOptions] = None, to_host: bool = True):
        opts = opts or RenderOptions()
        c = cam._c()
        tfa, ntf = tf._c()
        q, ds, o = qc._c(), stats._c(), opts._c()
        rs, err = _RStats(), _Error()
        shard = getattr(self, "_shard", (0, 1))
        if shard[1] > 1:
            from . import dist as _d
            nt = _d.tile_grid(cam.width, cam.height)[2]
            shape = (_d.packed_tiles_per_rank(shard[1], nt) * _d.TILE * _d.TILE * 3,)
        else:
            r0, nr = getattr(self, "_rows", (0, 0))
            rows = cam.height if nr == 0 else max(0, min(r0 + nr, cam.height) - min(r0, cam.height))
            shape = (rows, cam.width, 3)
        rgb = np.empty(shape, dtype=np.float64) if to_host else None
        _check(self._L.sphray_scene_render(
            self._h, C.byref(c), tfa, ntf, C.byref(q), C.byref(ds), C.byref(o),
            rgb.ctypes.data_as(C.POINTER(C.c_double)) if to_host else None, C.byref(rs),
            C.byref(err)), err)
        img = Image(cam.width, shape[0] if shard[1] == 1 else cam.height, rgb) if to_host else None
        return img, RenderStats._from(rs)

    def stream_ptr(self) -> int:
        """The library's cudaStream_t (for torch.cuda.ExternalStream / event timing)."""
        return int(self._L.sphray_context_stream(self._h) or 0)

    def device_image_ptr(self) -> int:
        return int(self._L.sphray_scene_device_image(self._h) or 0)

    def hits(self, cam: Camera):
        """All (ray, particle) hits of the resident scene (particle_ray_footprint, raycast.hpp:128)."""
        c = cam._c()
        cnt, err = C.c_size_t(), _Error()
        _check(self._L.sphray_scene_hits(self._h, C.byref(c), None, None, None, None, 0,
                                         C.byref(cnt), C.byref(err)), err)
        n = cnt.value
        ray = np.zeros(n, np.uint64)
        pidx = np.zeros(n, np.int64)
        lam = np.zeros(n, np.float64)
        tchi = np.zeros(n, np.float64)
        P = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
        _check(self._L.sphray_scene_hits(self._h, C.byref(c), P(ray, C.c_uint64),
                                         P(pidx, C.c_int64), P(lam, C.c_double),
                                         P(tchi, C.c_double), n, C.byref(cnt), C.byref(err)), err)
        return ray, pidx, lam, tchi

    def pieces(self, cam: Camera, qc: QuantaConfig):
        """Merged FieldPieces per touched ray (accumulate, raycast.hpp:261-292) as CSR."""
        c, q = cam._c(), qc._c()
        nr, npc, err = C.c_size_t(), C.c_size_t(), _Error()
        _check(self._L.sphray_scene_pieces(self._h, C.byref(c), C.byref(q), None, None, None, None,
                                           0, 0, C.byref(nr), C.byref(npc), C.byref(err)), err)
        D = self.scene_info()["D"]  # the stride the library writes (the resident scene's degree)
        rays = np.zeros(nr.value, np.uint64)
        off = np.zeros(nr.value + 1, np.uint64)
        pt = np.zeros(npc.value, np.int64)
        pa = np.zeros((npc.value, D + 1), np.int64)
        P = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
        _check(self._L.sphray_scene_pieces(self._h, C.byref(c), C.byref(q), P(rays, C.c_uint64),
                                           P(off, C.c_uint64), P(pt, C.c_int64),
                                           P(pa, C.c_int64), len(rays), len(pt), C.byref(nr),
                                           C.byref(npc), C.byref(err)), err)
        return dict(rays=rays, piece_off=off, piece_t=pt, piece_a=pa)

    def validate(self, cam: Camera, qc: QuantaConfig, ds: DatasetStats) -> dict:
        """The reference's `validate` groups (sphray_main.cpp:260-417) for the
        uploaded scene: telescoping, exact superposition (128-bit replay of
        every piece), dense-L2 envelope.  Like the reference, callers clamp the
        camera to 32 x 32 (validate_camera())."""
        rep, err = _ValidateReport(), _Error()
        _check(self._L.sphray_scene_validate(self._h, C.byref(cam._c()), C.byref(qc._c()),
                                             C.byref(ds._c()), C.byref(rep), C.byref(err)), err)
        out = {k: getattr(rep, k) for k, _ in _ValidateReport._fields_}
        out["pass"] = bool(out.pop("pass_"))
        for k in ("telescoping_pass", "superposition_pass", "l2_pass"):
            out[k] = bool(out[k])
        return out

    def upload_file(self, path: str, lut: Lut) -> None:
        """Loads a particle file (SPRT / CSV) and makes it the resident scene."""
        err = _Error()
        _check(self._L.sphray_scene_upload_file(self._h, os.fsencode(path), C.byref(lut.view),
                                                C.byref(err)), err)
        self._lut = lut
        self._n = self.scene_info()["n"]

    def dataset_stats(self, clustering_factor: float = 16.0) -> DatasetStats:
        """dataset_stats (quantize.hpp:129-165) of the uploaded scene, on the GPU."""
        out, err = _DStats(), _Error()
        _check(self._L.sphray_scene_dataset_stats(self._h, clustering_factor, C.byref(out),
                                                  C.byref(err)), err)
        return DatasetStats._from(out)

    def accumulate(self, knot_t, knot_b, D: int, ray_offsets=None, ray_ids=None):
        """accumulate<int64_t> (raycast.hpp:261-292) for explicit knot streams on
        the GPU.  knot_t (n,), knot_b (n, <=7) jumps; ray_offsets (nrays+1) CSR
        (default: one ray), ray_ids for error reports.  Returns
        (piece_offsets, piece_t, piece_a (P, D+1), ops per ray)."""
        kt = np.ascontiguousarray(knot_t, np.int64)
        kb = np.zeros((len(kt), 7), np.int64)
        if len(kt):
            b = np.asarray(knot_b, np.int64).reshape(len(kt), -1)
            kb[:, : b.shape[1]] = b
        off = np.ascontiguousarray([0, len(kt)] if ray_offsets is None else ray_offsets, np.uint64)
        nr = len(off) - 1
        rid = np.ascontiguousarray(np.arange(nr) if ray_ids is None else ray_ids, np.uint64)
        poff = np.zeros(nr + 1, np.uint64)
        pt = np.zeros(max(len(kt), 1), np.int64)
        pa = np.zeros((max(len(kt), 1), D + 1), np.int64)
        ops = np.zeros(max(nr, 1), np.uint64)
        err = _Error()
        P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
        _check(self._L.sphray_accumulate(self._h, int(D), nr, P(rid), P(off), P(kt), P(kb), P(poff), P(pt),
                                         P(pa), P(ops), C.byref(err)), err)
        npc = int(poff[-1])
        return poff, pt[:npc], pa[:npc], ops[:nr]

    def quantize_hits(self, particles, t_chi, lam, lut: Lut, qc: QuantaConfig):
        """quantize_particle (quantize.hpp:199-250) for explicit hits (one particle row each)."""
        a = _particles(particles)
        n = len(a)
        t_chi = np.ascontiguousarray(t_chi, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
        K1, D = lut.K + 1, lut.D
        kt = np.zeros((n, K1), np.int64)
        kb = np.zeros((n, K1, D + 1), np.int64)
        kc = np.zeros(n, np.int32)
        q, err = qc._c(), _Error()
        P = lambda x, t: x.ctypes.data_as(C.POINTER(t))  # noqa: E731
        _check(self._L.sphray_quantize_hits(self._h, _pp(a), n, P(t_chi, C.c_double),
                                            P(lam, C.c_double), C.byref(lut.view), C.byref(q),
                                            P(kt, C.c_int64), P(kb, C.c_int64), P(kc, C.c_int32),
                                            C.byref(err)), err)
        return kt, kb, kc


_default_ctx: Optional[Context] = None


def _ctx() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


def render_scene(particles, cam: Camera, tf: TransferFunction, lut: Lut, qc: QuantaConfig,
                 stats: DatasetStats, opts: Optional[RenderOptions] = None,
                 ctx: Optional[Context] = None):
    """render_scene<Int> (raycast.hpp:414-497) on the B200 path: returns (Image, RenderStats).

    The integer width comes from ``qc.width`` like dispatch_int_width (int_ops.hpp:113)."""
    ctx = ctx or _ctx()
    a = _particles(particles)
    opts = opts or RenderOptions()
    c = cam._c()
    tfa, ntf = tf._c()
    q, ds, o = qc._c(), stats._c(), opts._c()
    rs, err = _RStats(), _Error()
    rgb = np.empty((cam.height, cam.width, 3), dtype=np.float64)
    _check(ctx._L.sphray_render_scene(ctx._h, _pp(a), len(a), C.byref(c), tfa, ntf,
                                      C.byref(lut.view), C.byref(q), C.byref(ds), C.byref(o),
                                      rgb.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rs),
                                      C.byref(err)), err)
    ctx._lut = lut
    ctx._n = len(a)
    return Image(cam.width, cam.height, rgb), RenderStats._from(rs)

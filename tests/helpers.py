"""Shared test fixtures: the reference tests' scene generators restated in Python.

``random_cloud`` follows raycast_tests.cpp:34-44 exactly (std::mt19937_64 draws,
u = lo + (hi - lo) * (rng() >> 11) * 2^-53), so the same seeds give the same
particles the reference's own tests use.
"""
from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LUTS = os.path.join(ROOT, "data", "luts")
REF_DATA = "/root/reference/proj/data"
GOLDEN = os.path.join(ROOT, "tests", "golden")

# SURVEY.md 8(d) synthetic TF: abs(0) = 0, so empty gaps are exact no-ops
SYNTH_TF = np.array([[0.0, 0.02, 0.02, 0.10, 0.0], [0.2, 0.05, 0.10, 0.45, 0.35],
                     [0.6, 0.10, 0.35, 0.80, 0.9], [1.0, 1.0, 0.85, 0.30, 2.4]])
# raycast_tests.cpp:403 (absorption at 0 is nonzero: gaps must be sampled)
TEST_TF = np.array([[-0.5, 0.0, 0.0, 0.2, 0.1], [0.5, 0.9, 0.3, 0.1, 1.4]])


def lut_path(K=4, D=3, N=1024):
    return os.path.join(LUTS, f"cubic_K{K}_D{D}_N{N}.splt")


class MT19937_64:
    """std::mt19937_64."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def random_cloud(rng: MT19937_64, n: int, spread: float, depth0: float, depth1: float):
    """raycast_tests.cpp:34-44."""
    def u(lo, hi):
        return lo + (hi - lo) * float(rng() >> 11) * 2.0 ** -53

    out = []
    for _ in range(n):
        out.append([u(-spread, spread), u(-spread, spread), u(depth0, depth1), u(0.2, 2.0),
                    u(0.5, 2.0), u(0.1, 0.6), u(-1.0, 1.5)])
    return np.array(out, dtype=np.float64)


def synth_camera_kwargs(width, height):
    """SURVEY.md 8(d) orthographic camera."""
    return dict(mode="orthographic", position=(0.0, 0.0, 8.0), look_at=(0.0, 0.0, 0.0),
                up=(0.0, 1.0, 0.0), width=width, height=height, ortho_height=6.0, near=0.0,
                far=1e30)


def render_test_camera_kwargs():
    """raycast_tests.cpp:394-400."""
    return dict(mode="orthographic", position=(0.0, 0.0, 4.0), look_at=(0.0, 0.0, 0.0),
                up=(0.0, 1.0, 0.0), width=24, height=24, ortho_height=5.0)


def footprint_test_cameras():
    """raycast_tests.cpp:155-166: an orthographic and a pinhole camera."""
    ortho = dict(mode="orthographic", width=28, height=20, position=(0.3, -0.2, 4.0),
                 look_at=(0.0, 0.1, 0.0), up=(0.2, 1.0, 0.1), ortho_height=5.0)
    pin = dict(ortho, mode="pinhole", fov_deg=55.0)
    return ortho, pin

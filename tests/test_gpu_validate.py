"""The reference's `validate` command (sphray_main.cpp:260-417)
run on the GPU: telescoping, exact superposition and dense-L2 envelope groups.

Checker: the golden scenes (pieces produced by the unmodified reference) and a
numpy restatement of the reference's group-3 formulas (oracle.hpp:29-62,
234-246; lut.hpp:284-290; quantize.hpp:64-73) on the reference's own pieces."""
import math

import numpy as np
import pytest

import paper_2401_02896_b200 as S
from oracle import ref
from tests import helpers as H
from tests.test_gpu_parity import load, quanta

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = S.Context(0)
    yield c
    c.close()


def clamp32(ck):
    ck = dict(ck)
    ck["width"], ck["height"] = min(ck["width"], 32), min(ck["height"], 32)
    return ck


def cubic_w(r):
    r = np.abs(r)
    c = 1.0 / (4.0 * math.pi)
    return np.where(r < 1.0, c * (4.0 - 6.0 * r * r + 3.0 * r ** 3),
                    np.where(r < 2.0, c * (2.0 - r) ** 3, 0.0))


def envelope(lut, qc, ds):
    kappa, kappa_p = ref.kernel_constants()
    rec = lut.records()
    dl = lut.q / lut.N
    estar = math.sqrt(2.0 * math.pi * float(np.sum(rec[:, 0] * rec[:, 1] ** 2 * dl))) / kappa
    tq, sq = qc.tau / ds.h_r, qc.sigma / ds.phi_repr
    s = kappa_p ** 2 * tq * tq
    for d in range(lut.D + 1):
        s += 2.0 * lut.q ** (2 * d + 3) / ((2 * d + 1) * (2 * d + 3)) * sq * sq / tq ** (2 * d)
    return 4.0 * math.hypot(estar, math.sqrt(s) / (4.0 * kappa))


def l2_bad_numpy(g, ck, lut, qc, ds):
    """Group 3 restated on the reference's pieces for the first 64 rays."""
    ps = g["particles"]  # x y z mass density h value
    env = envelope(lut, qc, ds)
    h_step = ps[:, 5].min() / 64.0
    rays, off = g["pl_rays"], g["pl_piece_off"]
    pt, pa = g["pl_piece_t"], g["pl_piece_a"]
    cam = ref.Camera(**ck)
    tested = bad = 0
    for r in range(len(rays)):
        if tested == 64:
            break
        a, b = int(off[r]), int(off[r + 1])
        t0, t1 = float(pt[a]) * qc.tau, float(pt[b - 1]) * qc.tau
        if not t1 > t0:
            continue
        n = max(64, int((t1 - t0) / h_step))
        n += n % 2
        ts = t0 + np.arange(n + 1) * ((t1 - t0) / n)
        k = np.searchsorted(pt[a:b].astype(np.float64) * qc.tau, ts, side="right") - 1
        k = np.clip(k, 0, b - a - 1) + a
        x = ts / qc.tau - pt[k].astype(np.float64)
        acc = np.zeros_like(ts)
        for d in range(lut.D, -1, -1):
            acc = acc * x + pa[k, d].astype(np.float64)
        approx = acc * qc.sigma
        o, dirv, _ = ref.camera_ray(cam, int(rays[r] % ck["width"]), int(rays[r] // ck["width"]))
        pos = np.asarray(o)[None, :] + np.asarray(dirv)[None, :] * ts[:, None]
        rr = np.sqrt(((pos[:, None, :] - ps[None, :, :3]) ** 2).sum(-1)) / ps[None, :, 5]
        phi = ps[:, 3] * ps[:, 6] / (ps[:, 4] * ps[:, 5] ** 3)
        exact = (phi[None, :] * cubic_w(rr)).sum(-1)
        w = np.full(n + 1, 2.0)
        w[1::2] = 4.0
        w[0] = w[-1] = 1.0
        hh = (t1 - t0) / n
        num = math.sqrt(max(float((w * (approx - exact) ** 2).sum()) * hh / 3.0, 0.0))
        den = math.sqrt(max(float((w * exact ** 2).sum()) * hh / 3.0, 0.0))
        tested += 1
        bad += den > 0.0 and num / den > env
    return tested, bad, env


@pytest.mark.parametrize("name", ["render_test", "kd_K3_D2", "kd_K5_D4"])
def test_validate_groups_match_reference(ctx, name):
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ctx.upload(g["particles"], lut)
    ck = clamp32(g["ck"])
    assert ck == g["ck"]  # these goldens are already validation-sized
    qc = quanta(g)
    ds = S.dataset_stats(g["particles"], lut)
    rep = ctx.validate(S.Camera(**ck), qc, ds)
    # group 1: one trailing zero piece per touched ray (reference stats)
    assert rep["telescoping_rays"] == int(g["stat_rays_touched"])
    assert rep["telescoping_bad"] == int(g["stat_residual_failures"]) == 0
    # group 2: every GPU piece equals the 128-bit replay
    assert rep["superposition_rays"] == len(g["pl_rays"]) and rep["superposition_bad"] == 0
    # group 3: same rays tested, same verdicts as the restated oracle
    tested, bad, env = l2_bad_numpy(g, ck, lut, qc, ds)
    assert rep["l2_envelope"] == pytest.approx(env, rel=1e-12)
    assert (rep["l2_rays"], rep["l2_bad"]) == (tested, bad)
    assert rep["pass"] == (rep["l2_fraction_within"] >= 0.95)


def test_validate_desk_scene_passes(ctx):
    """The bundled desk scene passes validation (cli_tests.cpp:343-357 checks
    residual_failures == 0 on it)."""
    g = load("desk")
    lut = S.load_lut(g["lut_path"])
    ctx.upload(g["particles"], lut)
    ds = S.dataset_stats(g["particles"], lut)
    rep = ctx.validate(S.Camera(**clamp32(g["ck"])), quanta(g), ds)
    assert rep["telescoping_bad"] == 0 and rep["superposition_bad"] == 0
    assert rep["telescoping_rays"] > 0 and rep["l2_rays"] > 0


def test_validate_generated_blob_1024_entry_lut(ctx):
    """A config-1-family scene with the default 1024-entry LUT, against the
    reference's own pieces (oracle/_ref accumulate<Int128>)."""
    ps = S.generate_scene(1, n=3000)
    ck = H.synth_camera_kwargs(32, 32)
    path = H.lut_path(4, 3, 1024)
    lut = S.load_lut(path)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    ctx.upload(ps, lut)
    rep = ctx.validate(S.Camera(**ck), qc, ds)
    r = ref.pipeline(ps, ref.Camera(**ck), ref.Lut(path), ref.RpQuanta(qc.tau, qc.sigma, 64))
    g = {"particles": ps, "pl_rays": r["rays"], "pl_piece_off": r["piece_off"],
         "pl_piece_t": r["piece_t"], "pl_piece_a": r["piece_a"]}
    assert rep["telescoping_bad"] == 0 and rep["superposition_bad"] == 0
    assert rep["superposition_rays"] == len(r["rays"])
    tested, bad, env = l2_bad_numpy(g, ck, lut, qc, ds)
    assert (rep["l2_rays"], rep["l2_bad"]) == (tested, bad)

"""Integer-overflow semantics of the GPU path.

The reference computes in Checked<Int> and throws OverflowError -- for
quantization naming the particle and ray (quantize.hpp:244-249), for the merge
naming the ray (raycast.hpp:285-289).  The B200 merge runs modulo 2^64 (exact
whenever the exact coefficients fit int64) and tests every
shift and jump add for a genuine overflow (render_kernel.cuh shift_overflows /
add_checked):

* a genuine overflow (the exact Int128 FieldPieces of some ray do not fit
  int64) raises OverflowError naming a ray, particle index -1, never a wrong
  image;
* the reference's *spurious* overflow (Delta t^D of an empty gap, raycast.hpp:
  236-244) is not reproduced: the GPU returns the image of the Int128 path,
  which the reference's own test equates with the int64 one
  (raycast_tests.cpp:440-442).
"""
import numpy as np
import pytest

import paper_2401_02896_b200 as S
from oracle import ref
from tests import helpers as H

pytestmark = pytest.mark.gpu

LUT = H.lut_path(4, 3, 1024)
CAM = dict(mode="orthographic", position=(0.0, 0.0, 8.0), look_at=(0.0, 0.0, 0.0),
           up=(0.0, 1.0, 0.0), width=8, height=8, ortho_height=0.4)


@pytest.fixture(scope="module")
def ctx():
    c = S.Context(0)
    yield c
    c.close()


def bad_rays(ps, rl, rqc):
    """Rays whose exact (Int128) FieldPieces leave int64."""
    p = ref.pipeline(ps, ref.Camera(**CAM), rl, rqc)
    out = set()
    for i, r in enumerate(p["rays"]):
        a, b = int(p["piece_off"][i]), int(p["piece_off"][i + 1])
        if not p["piece_fits"][a:b].all():
            out.add(int(r))
    return out


def test_genuine_merge_overflow_raises(ctx):
    """Two coincident particles whose sum exceeds int64 at a sigma 12x below
    choose_quanta's (the reference's int64 path throws too)."""
    ps = np.array([[0.0, 0.0, 0.0, 1.0, 1.0, 0.3, 1.0], [0.0, 0.0, 0.0, 1.0, 1.0, 0.3, 1.0],
                   [0.05, 0.02, -0.01, 1.0, 1.0, 0.3, 1.0]])
    lut, rl = S.load_lut(LUT), ref.Lut(LUT)
    ds = S.dataset_stats(ps, lut)
    qc0 = S.choose_quanta(lut, ds)
    qc = S.QuantaConfig(qc0.tau, qc0.sigma / 12.0, 64)
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    bad = bad_rays(ps, rl, rqc)
    assert bad
    with pytest.raises(ref.RefError) as er:
        ref.render(ps, ref.Camera(**CAM), H.SYNTH_TF, rl, rqc, ref.dataset_stats(ps, rl), threads=1)
    assert er.value.code == 3
    for mode in (S.MODE_EXACT, S.MODE_FAST):
        with pytest.raises(S.OverflowError) as e:
            S.render_scene(ps, S.Camera(**CAM), S.TransferFunction.from_array(H.SYNTH_TF), lut, qc,
                           ds, S.RenderOptions(mode=mode), ctx=ctx)
        assert e.value.particle_index == -1
        assert "accumulate" in str(e.value) and f"ray {e.value.ray_id}" in str(e.value)
        # the named ray genuinely overflows, or is the one the reference names
        assert e.value.ray_id in bad or e.value.ray_id == er.value.ray_id


def test_in_range_sigma_renders(ctx):
    """The same scene at choose_quanta's sigma: no overflow, reference image."""
    ps = np.array([[0.0, 0.0, 0.0, 1.0, 1.0, 0.3, 1.0], [0.0, 0.0, 0.0, 1.0, 1.0, 0.3, 1.0],
                   [0.05, 0.02, -0.01, 1.0, 1.0, 0.3, 1.0]])
    lut, rl = S.load_lut(LUT), ref.Lut(LUT)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    assert not bad_rays(ps, rl, rqc)
    img, st = S.render_scene(ps, S.Camera(**CAM), S.TransferFunction.from_array(H.SYNTH_TF), lut,
                             qc, ds, S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    rgb, rst, _, _ = ref.render_robust(ps, ref.Camera(**CAM), H.SYNTH_TF, rl, rqc,
                                       ref.dataset_stats(ps, rl))
    assert np.abs(img.pixels - rgb).max() <= 1e-4
    assert st.int_ops == rst["int_ops"] and st.residual_failures == 0


def test_spurious_reference_overflow_is_not_reproduced(ctx):
    """Clusters 6 units apart at tau = 1e-6: the reference's int64 advance()
    overflows on Delta t^3 across the empty gap (raycast.hpp:236-244) although
    every exact coefficient fits; the GPU returns the Int128 image."""
    ps = np.array([[0.0, 0.0, 1.0, 1.0, 1.0, 0.3, 1.0], [0.02, 0.0, -5.0, 1.0, 1.0, 0.3, 1.0],
                   [0.0, 0.03, -2.5, 1.0, 1.0, 0.25, 1.0]])
    lut, rl = S.load_lut(LUT), ref.Lut(LUT)
    ds = S.dataset_stats(ps, lut)
    qc0 = S.choose_quanta(lut, ds)
    qc = S.QuantaConfig(1e-6, qc0.sigma, 64)
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    rds = ref.dataset_stats(ps, rl)
    with pytest.raises(ref.RefError) as er:
        ref.render(ps, ref.Camera(**CAM), H.SYNTH_TF, rl, rqc, rds, threads=1)
    assert er.value.code == 3
    assert not bad_rays(ps, rl, rqc)
    rgb, rst, _ = ref.render(ps, ref.Camera(**CAM), H.SYNTH_TF, rl, rqc, rds, accum_bits=128)
    img, st = S.render_scene(ps, S.Camera(**CAM), S.TransferFunction.from_array(H.SYNTH_TF), lut,
                             qc, ds, S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    assert np.abs(img.pixels - rgb).max() <= 1e-4
    for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
        assert getattr(st, k) == rst[k], k


def test_quantize_overflow_names_particle_and_ray(ctx):
    """quantize_tests.cpp:316-343 at render level: an outlier particle far
    beyond the budget of the dataset statistics overflows quantization; the
    error names the first (particle, ray) like the reference (quantize.hpp:244-249)."""
    ps = H.random_cloud(H.MT19937_64(11), 30, 0.15, -0.3, 0.3)
    lut, rl = S.load_lut(LUT), ref.Lut(LUT)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    ps2 = ps.copy()
    ps2[7, 3] = 1e12  # mass: b_d far beyond int64
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    with pytest.raises(ref.RefError) as er:
        ref.render(ps2, ref.Camera(**CAM), H.SYNTH_TF, rl, rqc, ref.dataset_stats(ps, rl), threads=1)
    assert er.value.code == 3 and er.value.particle_index == 7
    with pytest.raises(S.OverflowError) as e:
        S.render_scene(ps2, S.Camera(**CAM), S.TransferFunction.from_array(H.SYNTH_TF), lut, qc, ds,
                       ctx=ctx)
    assert e.value.particle_index == 7
    assert "particle 7" in str(e.value)


# --------------------------------------------------------------------------- int_width 32
# render_scene<int32_t> (dispatch_int_width, int_ops.hpp:113-121): every
# Checked<int32_t> value of quantize_particle and every merged coefficient must
# fit int32; the GPU computes in int64 and tests the int32 range of each.

@pytest.mark.parametrize("case", ["render_test", "blob", "render_test_K2D1"])
def test_int32_renders_match_reference(ctx, case):
    if case == "blob":
        ps, ck, tf, lp = ref.generate_scene(1, 3000), H.synth_camera_kwargs(48, 48), H.SYNTH_TF, \
            H.lut_path(4, 3, 1024)
    else:
        ps = H.random_cloud(H.MT19937_64(31337), 120, 1.6, -1.2, 1.2)
        ck, tf = H.render_test_camera_kwargs(), H.TEST_TF
        lp = H.lut_path(2, 1, 1024) if case.endswith("K2D1") else H.lut_path(4, 3, 16)
    lut, rl = S.load_lut(lp), ref.Lut(lp)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds, 32)
    rds = ref.dataset_stats(ps, rl)
    rqc = ref.choose_quanta(rl, rds, 32)
    assert (qc.tau, qc.sigma, qc.width) == (rqc.tau, rqc.sigma, 32)
    rgb, rst, _ = ref.render(ps, ref.Camera(**ck), tf, rl, rqc, rds, accum_bits=32)
    img, st = S.render_scene(ps, S.Camera(**ck), S.TransferFunction.from_array(tf), lut, qc, ds,
                             S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    assert np.abs(img.pixels - rgb).max() <= 1e-4
    for k in ("knots", "rays_touched", "int_ops", "residual_failures", "skipped_particles"):
        assert getattr(st, k) == rst[k], k


def test_int32_distant_particle_overflows_but_int64_renders(ctx, tmp_path):
    """cli_tests.cpp:252-273: a particle 2e7 away overflows 32-bit knot
    positions (OverflowError naming particle and ray, exit code 3 in the CLI)
    but renders at 64 bits."""
    small = np.array([[-0.8, 0.5, 0.3, 1.0, 1.2, 0.6, 1.5], [0.4, -0.6, -0.4, 0.8, 0.9, 0.8, 2.0],
                      [0.9, 0.8, 0.8, 1.2, 1.1, 0.5, 0.7], [-0.3, -0.9, -0.9, 0.6, 1.0, 0.9, 1.1],
                      [0.1, 0.2, 0.5, 1.5, 1.4, 0.7, 2.4], [-1.0, -0.2, 0.0, 0.9, 0.8, 0.6, 0.9],
                      [0.0, 0.0, -2e7, 1.0, 1.0, 0.5, 1.0]])
    ck = dict(mode="orthographic", position=(0.0, 0.0, 4.0), look_at=(0.0, 0.0, 0.0),
              up=(0.0, 1.0, 0.0), width=16, height=16, ortho_height=4.0)
    tf = np.array([[0.0, 0.0, 0.0, 0.0, 0.0], [1.0, 1.0, 0.5, 0.2, 2.0], [5.0, 1.0, 1.0, 1.0, 4.0]])
    lp = str(tmp_path / "k2d1n8.splt")
    ref.build_lut(2, 1, 8, lp)  # lut-build --K 2 --D 1 -N 8
    lut, rl = S.load_lut(lp), ref.Lut(lp)
    ds, rds = S.dataset_stats(small, lut), ref.dataset_stats(small, rl)
    q32, r32 = S.choose_quanta(lut, ds, 32), ref.choose_quanta(rl, rds, 32)
    with pytest.raises(ref.RefError) as er:
        ref.render(small, ref.Camera(**ck), tf, rl, r32, rds, accum_bits=32)
    with pytest.raises(S.OverflowError) as e:
        S.render_scene(small, S.Camera(**ck), S.TransferFunction.from_array(tf), lut, q32, ds, ctx=ctx)
    assert (e.value.particle_index, e.value.ray_id) == (er.value.particle_index, er.value.ray_id)
    q64, r64 = S.choose_quanta(lut, ds, 64), ref.choose_quanta(rl, rds, 64)
    rgb, rst, _ = ref.render(small, ref.Camera(**ck), tf, rl, r64, rds, accum_bits=64)
    img, st = S.render_scene(small, S.Camera(**ck), S.TransferFunction.from_array(tf), lut, q64, ds,
                             S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    assert np.abs(img.pixels - rgb).max() <= 1e-4
    for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
        assert getattr(st, k) == rst[k], k


# --------------------------------------------------------------------------- int_width 128
# render_scene<Int128> on w128 quanta: 128-bit jumps and a modulo-2^128 merge
# (robust kernel variant); knot positions stay int64.

@pytest.mark.parametrize("case", ["render_test", "blob"])
def test_int128_renders_match_reference(ctx, case):
    if case == "blob":
        ps, ck, tf, lp = ref.generate_scene(1, 3000), H.synth_camera_kwargs(48, 48), H.SYNTH_TF, \
            H.lut_path(4, 3, 1024)
    else:
        ps = H.random_cloud(H.MT19937_64(31337), 120, 1.6, -1.2, 1.2)
        ck, tf, lp = H.render_test_camera_kwargs(), H.TEST_TF, H.lut_path(4, 3, 16)
    lut, rl = S.load_lut(lp), ref.Lut(lp)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds, 128)
    rds = ref.dataset_stats(ps, rl)
    rqc = ref.choose_quanta(rl, rds, 128)
    assert (qc.tau, qc.sigma, qc.width) == (rqc.tau, rqc.sigma, 128)
    rgb, rst, _ = ref.render(ps, ref.Camera(**ck), tf, rl, rqc, rds, accum_bits=128)
    img, st = S.render_scene(ps, S.Camera(**ck), S.TransferFunction.from_array(tf), lut, qc, ds,
                             S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    assert np.abs(img.pixels - rgb).max() <= 1e-4
    for k in ("knots", "rays_touched", "int_ops", "residual_failures", "skipped_particles"):
        assert getattr(st, k) == rst[k], k
    # per-ray FieldPiece checksums (low 64 bits of the 128-bit coefficients)
    ctx.upload(ps, lut)
    ctx.set_region(0, 0, 0, 0, record=True)
    try:
        ctx.render(S.Camera(**ck), S.TransferFunction.from_array(tf), qc, ds, S.RenderOptions(mode=S.MODE_EXACT))
        rec = ctx.ray_records()
    finally:
        ctx.set_region()
    _, rrec, _, _, bits = ref.render_region(ps, ref.Camera(**ck), tf, rl, rqc, st.step, 0, 0, ck["width"],
                                            ck["height"])
    assert bits == 128
    for k in ("knots", "pieces", "hits", "piece_checksum"):
        np.testing.assert_array_equal(rec[k], rrec[k])


def test_int128_positions_beyond_int64_fail_loudly(ctx):
    """Degree-1 tables at 128 bits quantize positions below 1e-19: t / tau leaves
    int64, which the device's window does not represent (CapacityError, never
    a wrong image)."""
    ps = ref.generate_scene(1, 500)
    lp = H.lut_path(2, 1, 1024)
    lut = S.load_lut(lp)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds, 128)
    assert qc.tau < 1e-18
    with pytest.raises(S.CapacityError):
        S.render_scene(ps, S.Camera(**H.synth_camera_kwargs(16, 16)), S.TransferFunction.from_array(H.SYNTH_TF),
                       lut, qc, ds, ctx=ctx)

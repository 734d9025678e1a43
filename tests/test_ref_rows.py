"""CPU checks of the reference-side row-band driver (oracle/_ref rp_render_rows)
that the bench's parity block and the config-3 GPU band test rely on.

* rows rendered by the reference's own sweep functions on the full camera are
  bit-identical to the same rows of render_scene (raycast.hpp:414-497);
* the per-ray records (knots, pieces, piece checksum, residual flag) equal the
  reference pipeline's per-ray CSR (accumulate<Int128>, raycast.hpp:261-292),
  with the checksum restated in numpy (sphray_piece_mix, include/sphray_gpu.h);
* the synthetic-scene generator compiled into oracle/_ref and the product's
  sphray_generate_scene (include/sphray_scenes.hpp) give identical bytes.
"""
import numpy as np
import pytest

from oracle import ref
from tests import helpers as H

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def scene():
    ps = ref.generate_scene(1, 6000)
    rl = ref.Lut(H.lut_path(4, 3, 1024))
    ds = ref.dataset_stats(ps, rl)
    qc = ref.choose_quanta(rl, ds)
    cam = ref.Camera(**H.synth_camera_kwargs(40, 40))
    return ps, rl, ds, qc, cam


def test_rows_equal_full_frame(scene):
    ps, rl, ds, qc, cam = scene
    rgb, st, _, bits = ref.render_robust(ps, cam, H.SYNTH_TF, rl, qc, ds, background=(0.1, 0.2, 0.3))
    for r0, nr in ((0, 40), (13, 4), (37, 9)):
        rr, rec, rst, _, _ = ref.render_rows(ps, cam, H.SYNTH_TF, rl, qc, ds.h_r / 8.0, r0, nr,
                                             background=(0.1, 0.2, 0.3))
        assert (rr == rgb[r0:r0 + nr]).all()
        assert rst["knots"] == int(rec["knots"].sum())
        if (r0, nr) == (0, 40):
            for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
                assert rst[k] == st[k], k


def test_row_records_match_pipeline(scene):
    ps, rl, ds, qc, cam = scene
    _, rec, _, _, _ = ref.render_rows(ps, cam, H.SYNTH_TF, rl, qc, ds.h_r / 8.0, 0, cam.height)
    p = ref.pipeline(ps, cam, rl, qc)
    D = p["D"]
    mix = ref.piece_mix(p["piece_t"], p["piece_a"], D)
    touched = np.zeros(len(rec), bool)
    for i, r in enumerate(p["rays"]):
        a, b = int(p["piece_off"][i]), int(p["piece_off"][i + 1])
        with np.errstate(over="ignore"):
            cs = np.uint64(mix[a:b].sum(dtype=np.uint64))
        o = rec[int(r)]
        assert o["piece_checksum"] == cs
        assert o["pieces"] == b - a
        assert o["knots"] == int(p["knot_off"][i + 1] - p["knot_off"][i])
        assert o["flags"] & 1
        assert bool(o["flags"] & 2) == bool(p["piece_a"][b - 1].any())
        touched[int(r)] = True
    assert (rec["knots"][~touched] == 0).all()


def test_scene_generators_identical():
    import paper_2401_02896_b200 as S

    for config, n in ((1, 20000), (3, 40000), (4, 5000)):
        a = S.generate_scene(config, n=n)
        b = ref.generate_scene(config, n)
        assert a.tobytes() == b.tobytes(), config


def test_region_footprint_and_pipeline_are_frame_subsets(scene):
    """The region filters (a conservative particle pre-filter + the pixel test)
    drop nothing the full frame has inside the region."""
    ps, rl, ds, qc, cam = scene
    region = (11, 17, 9, 5)
    x0, y0, w, h = region
    ray, pid, lam, t = ref.footprint(ps, cam, rl.q)
    px, py = ray % cam.width, ray // cam.width
    inside = (px >= x0) & (px < x0 + w) & (py >= y0) & (py < y0 + h)
    r2, p2, l2, t2 = ref.footprint(ps, cam, rl.q, region=region)
    assert inside.sum() > 100
    np.testing.assert_array_equal(r2, ray[inside])
    np.testing.assert_array_equal(p2, pid[inside])
    np.testing.assert_array_equal(l2.view(np.uint64), lam[inside].view(np.uint64))
    full = ref.pipeline(ps, cam, rl, qc)
    sub = ref.pipeline(ps, cam, rl, qc, region=region)
    rx, ry = full["rays"] % cam.width, full["rays"] // cam.width
    keep = np.nonzero((rx >= x0) & (rx < x0 + w) & (ry >= y0) & (ry < y0 + h))[0]
    np.testing.assert_array_equal(sub["rays"], full["rays"][keep])
    pieces = np.concatenate([np.arange(int(full["piece_off"][i]), int(full["piece_off"][i + 1]))
                             for i in keep])
    np.testing.assert_array_equal(sub["piece_t"], full["piece_t"][pieces])
    np.testing.assert_array_equal(sub["piece_a"], full["piece_a"][pieces])
    rgb, rec, _, _, _ = ref.render_region(ps, cam, H.SYNTH_TF, rl, qc, ds.h_r / 8.0, *region)
    frame, _, _, _ = ref.render_robust(ps, cam, H.SYNTH_TF, rl, qc, ds)
    assert (rgb[:, x0:x0 + w] == frame[y0:y0 + h, x0:x0 + w]).all()
    assert (rgb[:, :x0] == 0).all() and len(rec) == w * h

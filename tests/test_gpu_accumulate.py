"""sphray_accumulate: accumulate<int64_t> (raycast.hpp:261-292) for explicit
knot streams on the GPU, against the reference's own accumulator KATs
(raycast_tests.cpp:257-318) and the reference's accumulate<Int128> on real
knot streams (oracle/_ref pipeline): pieces bit-exact, op counts exact."""
import numpy as np
import pytest

import paper_2401_02896_b200 as S
from oracle import ref
from tests import helpers as H

pytestmark = pytest.mark.gpu

INT64_MAX = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def ctx():
    c = S.Context(0)
    yield c
    c.close()


def test_ramp_kat(ctx):
    """raycast_tests.cpp:257-283: a unit ramp from t=0, flat from t=3, back to 0 at t=5."""
    kt = np.array([0, 3, 5])
    kb = np.array([[0, 1], [0, -1], [-3, 0]])
    off, pt, pa, ops = ctx.accumulate(kt, kb, D=1)
    np.testing.assert_array_equal(pt, [0, 3, 5])
    np.testing.assert_array_equal(pa, [[0, 1], [3, 0], [0, 0]])
    assert ops[0] > 0
    with pytest.raises(S.NumericError):
        ctx.accumulate(np.array([0, 5, 4]), np.zeros((3, 2)), D=1)


def test_equal_positions_and_overflow_kat(ctx):
    """raycast_tests.cpp:285-318: equal positions merge (a0 = 2 then 0); a
    genuine overflow names the ray (ray 9)."""
    off, pt, pa, ops = ctx.accumulate([2, 2, 6], [[5], [-3], [-2]], D=2, ray_ids=[4])
    np.testing.assert_array_equal(pt, [2, 6])
    assert pa[0, 0] == 2 and pa[1, 0] == 0 and ops[0] > 0
    off, pt, pa, ops = ctx.accumulate(np.zeros(0), np.zeros((0, 3)), D=2)
    assert len(pt) == 0
    with pytest.raises(S.OverflowError) as e:
        ctx.accumulate([0, 1000], [[0, INT64_MAX // 2], [0, 0]], D=1, ray_ids=[9])
    assert e.value.ray_id == 9 and "ray 9" in str(e.value) and e.value.particle_index == -1


@pytest.mark.parametrize("K,D", [(4, 3), (3, 2), (5, 4)])
def test_streams_match_reference_int128(ctx, K, D):
    ps = ref.generate_scene(1, 3000)
    path = H.lut_path(K, D, 1024 if (K, D) == (4, 3) else 64)
    rl = ref.Lut(path)
    ds = ref.dataset_stats(ps, rl)
    qc = ref.choose_quanta(rl, ds)
    p = ref.pipeline(ps, ref.Camera(**H.synth_camera_kwargs(40, 40)), rl, qc)
    assert p["piece_fits"].all()
    off, pt, pa, ops = ctx.accumulate(p["knot_t"], p["knot_b"], D=D, ray_offsets=p["knot_off"],
                                      ray_ids=p["rays"])
    np.testing.assert_array_equal(off, p["piece_off"])
    np.testing.assert_array_equal(pt, p["piece_t"])
    np.testing.assert_array_equal(pa, p["piece_a"])
    np.testing.assert_array_equal(ops, p["ray_ops"])

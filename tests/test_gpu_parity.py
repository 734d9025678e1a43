"""GPU parity: the sm_100a path against the reference on identical inputs.

Checkers: the golden fixtures of tests/golden/ (produced by the UNMODIFIED
reference through oracle/_ref by tests/golden/make_golden.py) and, for
generated scenes, oracle/_ref run live on the GPU box's host.

Bars:
  * hit sets (ray, particle, lam, t_chi): bit-exact
  * per-hit knots and merged FieldPiece coefficients: bit-exact integers
    (reference accumulate<Int128> on w64 quanta, identical to the int64 path
    whenever that does not throw: raycast_tests.cpp:440-442)
  * RGB: |gpu - reference| <= 1e-4 absolute per channel.  Both compute in
    fp64; the residual differences are CUDA-vs-glibc exp ulps and the order of
    the front-to-back sum (observed ~1e-15).
  * RenderStats particles / skipped / knots / rays_touched / int_ops /
    residual_failures / step: exact (EXACT mode)
"""
import hashlib
import os

import numpy as np
import pytest

import paper_2401_02896_b200 as S
from oracle import ref
from tests import helpers as H

pytestmark = pytest.mark.gpu

RGB_TOL = 1e-4
GOLDEN_SCENES = ["render_test", "footprint_ortho", "footprint_pinhole", "clip_planes", "desk",
                 "blob3000", "kd_K3_D2", "kd_K5_D4", "kd_K2_D3", "kd_K6_D6", "kd_K7_D5"]


@pytest.fixture(scope="module")
def ctx():
    c = S.Context(0)
    yield c
    c.close()


def load(name):
    z = np.load(os.path.join(H.GOLDEN, name + ".npz"))
    g = {k: z[k] for k in z.files}
    ck = dict(mode=str(g["cam_mode"]), position=tuple(g["cam_position"]),
              look_at=tuple(g["cam_look_at"]), up=tuple(g["cam_up"]), width=int(g["cam_width"]),
              height=int(g["cam_height"]), fov_deg=float(g["cam_fov_deg"]),
              ortho_height=float(g["cam_ortho_height"]), near=float(g["cam_near"]),
              far=float(g["cam_far"]))
    g["ck"] = ck
    g["lut_path"] = os.path.join(H.LUTS, str(g["lut"]))
    return g


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def quanta(g):
    return S.QuantaConfig(float(g["tau"]), float(g["sigma"]), 64)


def dstats(g, ps, lut):
    return S.dataset_stats(ps, lut)


@pytest.mark.parametrize("name", GOLDEN_SCENES)
def test_hit_sets_bit_exact(ctx, name):
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ctx.upload(g["particles"], lut)
    ray, pid, lam, t = ctx.hits(S.Camera(**g["ck"]))
    if "digest_hits" in g:
        # reference order is particle-major; compare in the same order
        o = np.lexsort((ray, pid))
        assert len(ray) == int(g["n_hits"])
        assert digest(ray[o], pid[o], lam[o], t[o]) == str(g["digest_hits"])
        return
    o = np.lexsort((g["hit_pidx"], g["hit_ray"]))
    np.testing.assert_array_equal(ray, g["hit_ray"][o])
    np.testing.assert_array_equal(pid, g["hit_pidx"][o])
    np.testing.assert_array_equal(lam.view(np.uint64), g["hit_lam"][o].view(np.uint64))
    np.testing.assert_array_equal(t.view(np.uint64), g["hit_tchi"][o].view(np.uint64))


@pytest.mark.parametrize("name", [n for n in GOLDEN_SCENES if n not in ("desk", "blob3000")])
def test_knots_bit_exact(ctx, name):
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ps = g["particles"]
    kt, kb, kc = ctx.quantize_hits(ps[g["hit_pidx"]], g["hit_tchi"], g["hit_lam"], lut, quanta(g))
    np.testing.assert_array_equal(kc, g["knot_count"])
    off = np.concatenate([[0], np.cumsum(g["knot_count"])])
    D1 = lut.D + 1
    for i in range(len(kc)):
        np.testing.assert_array_equal(kt[i, : kc[i]], g["knot_t"][off[i]:off[i + 1]])
        np.testing.assert_array_equal(kb[i, : kc[i]], g["knot_b"][off[i]:off[i + 1], :D1])


@pytest.mark.parametrize("name", GOLDEN_SCENES)
def test_field_pieces_bit_exact(ctx, name):
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ctx.upload(g["particles"], lut)
    p = ctx.pieces(S.Camera(**g["ck"]), quanta(g))
    np.testing.assert_array_equal(p["rays"], g["pl_rays"])
    np.testing.assert_array_equal(p["piece_off"], g["pl_piece_off"])
    if "digest_pieces" in g:
        assert len(p["piece_t"]) == int(g["n_pieces"])
        # the reference stores 7 coefficients (max_degree + 1) per piece
        pa = np.zeros((len(p["piece_a"]), lut.D + 1), np.int64)
        pa[:] = p["piece_a"]
        assert digest(p["rays"], p["piece_off"], p["piece_t"], pa) == str(g["digest_pieces"])
        return
    assert g["pl_piece_fits"].all()
    np.testing.assert_array_equal(p["piece_t"], g["pl_piece_t"])
    np.testing.assert_array_equal(p["piece_a"], g["pl_piece_a"])


@pytest.mark.parametrize("name", GOLDEN_SCENES)
@pytest.mark.parametrize("mode", [S.MODE_EXACT, S.MODE_FAST])
def test_render_matches_reference(ctx, name, mode):
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ps = g["particles"]
    ds = S.dataset_stats(ps, lut)
    assert ds.h_r == float(g["h_r"]) and ds.a_max == float(g["a_max"])
    qc = S.choose_quanta(lut, ds)
    assert qc.tau == float(g["tau"]) and qc.sigma == float(g["sigma"])
    img, st = S.render_scene(ps, S.Camera(**g["ck"]), S.TransferFunction.from_array(g["tf"]), lut,
                             qc, ds, S.RenderOptions(background=tuple(g["background"]), mode=mode),
                             ctx=ctx)
    err = np.abs(img.pixels - g["rgb"]).max()
    assert err <= RGB_TOL, err
    assert st.particles == int(g["stat_particles"])
    assert st.skipped_particles == int(g["stat_skipped_particles"])
    assert st.step == float(g["stat_step"])
    if mode == S.MODE_EXACT:
        for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
            assert getattr(st, k) == int(g["stat_" + k]), (k, getattr(st, k), int(g["stat_" + k]))


def _blob(n, w):
    ps = S.generate_scene(1, n=n)
    return ps, H.synth_camera_kwargs(w, w)


def test_generated_blob_against_live_reference(ctx):
    """A generated config-1-family scene, checked against oracle/_ref on this host."""
    ps, ck = _blob(20000, 96)
    lut = S.load_lut(H.lut_path(4, 3, 1024))
    rl = ref.Lut(H.lut_path(4, 3, 1024))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    rds = ref.dataset_stats(ps, rl)
    ctx.upload(ps, lut)
    ray, pid, lam, t = ctx.hits(S.Camera(**ck))
    r_ray, r_pid, r_lam, r_t = ref.footprint(ps, ref.Camera(**ck), lut.q)
    o = np.lexsort((r_pid, r_ray))
    np.testing.assert_array_equal(ray, r_ray[o])
    np.testing.assert_array_equal(pid, r_pid[o])
    np.testing.assert_array_equal(lam.view(np.uint64), r_lam[o].view(np.uint64))
    np.testing.assert_array_equal(t.view(np.uint64), r_t[o].view(np.uint64))
    p = ctx.pieces(S.Camera(**ck), qc)
    r = ref.pipeline(ps, ref.Camera(**ck), rl, rqc)
    np.testing.assert_array_equal(p["rays"], r["rays"])
    np.testing.assert_array_equal(p["piece_t"], r["piece_t"])
    np.testing.assert_array_equal(p["piece_a"], r["piece_a"])
    img, st = S.render_scene(ps, S.Camera(**ck), S.TransferFunction.from_array(H.SYNTH_TF), lut, qc,
                             ds, ctx=ctx)
    rgb, rst, _, _ = ref.render_robust(ps, ref.Camera(**ck), H.SYNTH_TF, rl, rqc, rds)
    assert np.abs(img.pixels - rgb).max() <= RGB_TOL
    for k in ("knots", "rays_touched", "int_ops", "residual_failures", "skipped_particles"):
        assert getattr(st, k) == rst[k], k


def test_early_termination_opaque(ctx):
    """Opaque media saturate and exit early (raycast_tests.cpp:382-387)."""
    g = load("blob3000")
    lut = S.load_lut(g["lut_path"])
    rl = ref.Lut(g["lut_path"])
    ps = g["particles"]
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    rds = ref.dataset_stats(ps, rl)
    dense = np.array([[0.0, 1.0, 0.5, 0.25, 0.0], [0.01, 1.0, 0.5, 0.25, 500.0]])
    rgb, rst, _, _ = ref.render_robust(ps, ref.Camera(**g["ck"]), dense, rl,
                                       ref.RpQuanta(qc.tau, qc.sigma, 64), rds)
    assert (rgb.sum(axis=2) > 0.5).any()
    for mode in (S.MODE_EXACT, S.MODE_FAST):
        img, st = S.render_scene(ps, S.Camera(**g["ck"]), S.TransferFunction.from_array(dense), lut,
                                 qc, ds, S.RenderOptions(mode=mode), ctx=ctx)
        assert np.abs(img.pixels - rgb).max() <= RGB_TOL
        if mode == S.MODE_EXACT:
            assert st.knots == rst["knots"] and st.int_ops == rst["int_ops"]


def test_empty_scene_paints_background(ctx):
    """raycast_tests.cpp:445-470."""
    lut = S.load_lut(H.lut_path(4, 3, 16))
    cam = S.Camera(width=6, height=4)
    img, st = S.render_scene(np.zeros((0, 7)), cam, S.TransferFunction.from_array([[0, 0, 0, 0, 0.5]]),
                             lut, S.QuantaConfig(0.1, 1.0, 64), S.DatasetStats(h_r=1.0),
                             S.RenderOptions(background=(0.25, 0.5, 0.75)), ctx=ctx)
    assert st.particles == 0 and st.knots == 0 and st.rays_touched == 0
    assert (img.pixels == np.array([0.25, 0.5, 0.75])).all()


def test_permutation_invariance(ctx):
    """raycast_tests.cpp:422-432: permuting the input changes no bit."""
    g = load("render_test")
    lut = S.load_lut(g["lut_path"])
    ps = g["particles"]
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    args = (S.Camera(**g["ck"]), S.TransferFunction.from_array(g["tf"]), lut, qc, ds,
            S.RenderOptions(background=tuple(g["background"])))
    img, st = S.render_scene(ps, *args, ctx=ctx)
    for seed in (1, 2, 3):
        p2 = ps[np.random.default_rng(seed).permutation(len(ps))]
        img2, st2 = S.render_scene(p2, *args, ctx=ctx)
        assert (img2.pixels == img.pixels).all()
        assert st2.knots == st.knots and st2.residual_failures == 0


def test_small_window_retry_is_exact(ctx):
    """A tiny knot window forces the wide-window retry pass; results must not change."""
    ps, ck = _blob(20000, 64)
    lut = S.load_lut(H.lut_path(4, 3, 1024))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    cam, tf = S.Camera(**ck), S.TransferFunction.from_array(H.SYNTH_TF)
    img, st = S.render_scene(ps, cam, tf, lut, qc, ds, S.RenderOptions(), ctx=ctx)
    img2, st2 = S.render_scene(ps, cam, tf, lut, qc, ds, S.RenderOptions(window=192), ctx=ctx)
    assert st2.window_retries > 0
    # exact integers; only the fp64 association of the compositing sum follows
    # the window's flush points
    assert np.abs(img2.pixels - img.pixels).max() <= 1e-12
    assert st2.knots == st.knots and st2.int_ops == st.int_ops


def test_validation_errors(ctx):
    lut = S.load_lut(H.lut_path(4, 3, 16))
    ps = H.random_cloud(H.MT19937_64(1), 10, 1.0, -1.0, 1.0)
    tf = S.TransferFunction.from_array([[0, 0, 0, 0, 0.5]])
    q, d = S.QuantaConfig(0.1, 1.0), S.DatasetStats(h_r=1.0)
    with pytest.raises(S.ConfigError):
        S.render_scene(ps, S.Camera(width=0), tf, lut, q, d, ctx=ctx)
    with pytest.raises(S.ConfigError):
        S.render_scene(ps, S.Camera(), S.TransferFunction.from_array([[1, 0, 0, 0, 0], [1, 0, 0, 0, 0]]),
                       lut, q, d, ctx=ctx)
    with pytest.raises(S.ConfigError):
        S.render_scene(ps, S.Camera(), S.TransferFunction.from_array([[0, 0, 0, 0, -1.0]]), lut, q, d,
                       ctx=ctx)


@pytest.mark.parametrize("name", ["render_test", "blob3000", "desk"])
@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_sharded_tiles_match_single_gpu(name, nranks):
    """Image-tile sharding: each rank renders tiles t % G == r
    into its packed buffer (the kernel's packed write path); gathered and
    unpacked with the layout k_unpack uses, the image is bit-identical to the
    single-rank render, and the per-rank counters sum to the same totals."""
    from tests import dist_layout as SD

    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ps = g["particles"]
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    cam = S.Camera(**g["ck"])
    tf = S.TransferFunction.from_array(g["tf"])
    opts = S.RenderOptions(background=tuple(g["background"]))
    with S.Context(0) as full:
        full.upload(ps, lut)
        img, st = full.render(cam, tf, qc, ds, opts)
    packed, sums = [], dict(knots=0, rays_touched=0, int_ops=0, hits=0)
    for r in range(nranks):
        with S.Context(0) as c:
            c.set_shard(r, nranks)
            c.upload(ps, lut)
            part, pst = c.render(cam, tf, qc, ds, opts)
            packed.append(part.pixels)
            for k in sums:
                sums[k] += getattr(pst, k)
    rgb = SD.unpack(np.concatenate(packed), nranks, cam.width, cam.height)
    assert (rgb == img.pixels).all()
    for k, v in sums.items():
        assert v == getattr(st, k), k


def _ulps(x, j):
    """x moved by j ulps."""
    x = np.asarray(x, np.float64)
    return np.nextafter(x, np.where(j >= 0, np.inf, -np.inf)) if abs(j) == 1 else \
        _ulps(np.nextafter(x, np.where(j >= 0, np.inf, -np.inf)), j - np.sign(j))


@pytest.mark.parametrize("lutname", [(4, 3, 1024), (5, 4, 64)])
def test_quantize_near_ties_live_reference(ctx, lutname):
    """The quantize divisions run as reciprocal multiplies with an exactness
    guard (device_math.cuh rint_div / lut_index).  Hits built to land within a
    few ulps of the rounding boundaries -- t_chi/tau at half-integers,
    h*u_k/tau at half-integers, lam/dl at LUT entry edges and lam = 0 -- must
    still quantize bit-identically to the reference (oracle/_ref live)."""
    path = H.lut_path(*lutname)
    lut, rl = S.load_lut(path), ref.Lut(path)
    rng = np.random.default_rng(5)
    tau, sigma = 1.0 / 1000, 2.0 ** -40  # |coefficients| up to ~2^53: both paths
    dl = lut.q / lut.N
    rec = lut.records()
    m = (lut.K + 1) // 2
    n = 3000
    ps = np.zeros((n, 7))
    ps[:, 3] = rng.uniform(0.5, 2.0, n)       # mass
    ps[:, 4] = rng.uniform(0.5, 2.0, n)       # density
    ps[:, 5] = rng.uniform(0.01, 0.1, n)      # h
    ps[:, 6] = rng.uniform(-1.0, 1.0, n)      # value
    e = rng.integers(0, lut.N, n)
    lam = e * dl
    k = rng.integers(-4000, 4000, n)
    tchi = (k + 0.5) * tau
    j = rng.integers(-3, 4, n)
    kind = np.arange(n) % 4
    for i in range(n):
        if kind[i] == 0 and j[i] != 0:      # t_chi / tau near a half-integer
            tchi[i] = _ulps(tchi[i], int(j[i]))
        elif kind[i] == 1:                  # lam / dl near an entry edge (or 0)
            lam[i] = 0.0 if j[i] == 0 or e[i] == 0 else _ulps(lam[i], int(j[i]))
        elif kind[i] == 2:                  # h * u_1 / tau near a half-integer
            u1 = rec[min(e[i], lut.N - 1), 2]
            h = (rng.integers(20, 200) + 0.5) * tau / u1
            ps[i, 5] = h if j[i] == 0 else float(_ulps(h, int(j[i])))
            lam[i] = (e[i] + 0.5) * dl
    lam = np.minimum(lam, lut.q * (1 - 1e-12))
    kt, kb, kc = ctx.quantize_hits(ps, tchi, lam, lut, S.QuantaConfig(tau, sigma, 64))
    rqc = ref.RpQuanta(tau, sigma, 64)
    D1 = lut.D + 1
    for i in range(n):
        rt, rb = ref.quantize(ps[i], 0, float(tchi[i]), float(lam[i]), rl, rqc)
        assert kc[i] == len(rt), i
        np.testing.assert_array_equal(kt[i, : kc[i]], rt, err_msg=str(i))
        np.testing.assert_array_equal(kb[i, : kc[i]], rb[:, :D1], err_msg=str(i))


@pytest.mark.parametrize("name", ["render_test", "desk", "blob3000", "kd_K6_D6"])
def test_scene_dataset_stats_on_gpu(ctx, name):
    """dataset_stats on the resident scene (GPU radix-sort medians + max
    reduction) equals the host restatement field for field,
    and both equal the reference's."""
    g = load(name)
    lut = S.load_lut(g["lut_path"])
    ps = g["particles"]
    for sub in (ps, ps[:-1]):  # even and odd counts
        ctx.upload(sub, lut)
        dg = ctx.dataset_stats()
        dh = S.dataset_stats(sub, lut)
        dr = ref.dataset_stats(sub, ref.Lut(g["lut_path"]))
        for k in ("mass_r", "density_r", "h_r", "value_r", "phi_repr", "a_max", "count"):
            assert getattr(dg, k) == getattr(dh, k), k
            assert getattr(dg, k) == getattr(dr, k), k


def test_scene_dataset_stats_rejects_bad_particles(ctx):
    lut = S.load_lut(H.lut_path(4, 3, 16))
    ps = H.random_cloud(H.MT19937_64(3), 50, 1.0, -1.0, 1.0)
    ps[7, 5] = 0.0  # h = 0
    ctx.upload(ps, lut)
    with pytest.raises(S.ConfigError):
        ctx.dataset_stats()


def test_alu_peak_probe():
    """The bench's ALU-roofline denominators come from a live probe."""
    pk = S.probe_alu_peaks(0)
    assert 1e3 < pk["int64_gops"] < 1e6 and 1e3 < pk["fp64_gflops"] < 1e6, pk


def test_ray_spanning_beyond_32bit_offsets_fails_loudly(ctx):
    """Knot positions are kept as 32-bit offsets per ray; a ray whose knots
    span more than 2^32 quanta cannot be represented and must fail with
    CapacityError (never a wrong image).  (The reference's int64 path throws
    OverflowError on such a ray: Delta t^D overflows in advance().)"""
    ps = np.array([[0.0, 0.0, 0.0, 1.0, 1.0, 0.3, 1.0],
                   [0.0, 0.0, -2.0, 1.0, 1.0, 0.3, 1.0]])
    lut = S.load_lut(H.lut_path(4, 3, 1024))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    qc = S.QuantaConfig(1e-10, qc.sigma, 64)
    cam = S.Camera(**H.synth_camera_kwargs(8, 8))
    with pytest.raises(S.CapacityError):
        S.render_scene(ps, cam, S.TransferFunction.from_array(H.SYNTH_TF), lut, qc, ds, ctx=ctx)


def test_scene_upload_from_file(ctx, tmp_path):
    """sphray_scene_upload_file == loading + sphray_scene_upload."""
    g = load("render_test")
    lut = S.load_lut(g["lut_path"])
    path = str(tmp_path / "scene.sprt")
    S.save_particles(g["particles"], path, binary=True)
    ctx.upload_file(path, lut)
    ray, pid, lam, t = ctx.hits(S.Camera(**g["ck"]))
    o = np.lexsort((g["hit_pidx"], g["hit_ray"]))
    np.testing.assert_array_equal(pid, g["hit_pidx"][o])
    np.testing.assert_array_equal(t.view(np.uint64), g["hit_tchi"][o].view(np.uint64))


@pytest.mark.parametrize("K", [2, 4])
def test_degree_one_small_tau_live_reference(ctx, K):
    """D = 1 LUTs give a tiny tau (~1e-9 here), so one ray's knot positions
    span far more than 2^32 quanta; the window's 32-bit offsets are rebased at
    every flush and only the live window must fit.  Checked against the live
    reference (pieces bit-exact, image <= 1e-4, stats exact)."""
    ps, ck = _blob(3000, 32)
    path = H.lut_path(K, 1, 1024)
    lut, rl = S.load_lut(path), ref.Lut(path)
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    assert qc.tau < 1e-8
    rqc = ref.RpQuanta(qc.tau, qc.sigma, 64)
    ctx.upload(ps, lut)
    p = ctx.pieces(S.Camera(**ck), qc)
    r = ref.pipeline(ps, ref.Camera(**ck), rl, rqc)
    np.testing.assert_array_equal(p["rays"], r["rays"])
    np.testing.assert_array_equal(p["piece_t"], r["piece_t"])
    np.testing.assert_array_equal(p["piece_a"], r["piece_a"])
    img, st = S.render_scene(ps, S.Camera(**ck), S.TransferFunction.from_array(H.SYNTH_TF), lut, qc,
                             ds, S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    rgb, rst, _, _ = ref.render_robust(ps, ref.Camera(**ck), H.SYNTH_TF, rl, rqc,
                                       ref.dataset_stats(ps, rl))
    assert np.abs(img.pixels - rgb).max() <= RGB_TOL
    for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
        assert getattr(st, k) == rst[k], k


def test_large_transfer_function_global_variant(ctx):
    """A TF too large for the per-CTA shared copy (> 4 KB: 60 points) runs the
    production kernel that reads it from global memory; same bars."""
    v = np.linspace(-0.2, 2.5, 60)
    tf = np.stack([v, 0.5 + 0.4 * np.sin(3 * v), 0.5 + 0.4 * np.cos(2 * v), 0.3 + 0.2 * np.sin(v),
                   0.1 + 0.8 * v * v], axis=1)
    ps, ck = _blob(5000, 48)
    lut = S.load_lut(H.lut_path(4, 3, 1024))
    rl = ref.Lut(H.lut_path(4, 3, 1024))
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds)
    rds = ref.dataset_stats(ps, rl)
    img, st = S.render_scene(ps, S.Camera(**ck), S.TransferFunction.from_array(tf), lut, qc, ds,
                             S.RenderOptions(mode=S.MODE_EXACT), ctx=ctx)
    rgb, rst, _, _ = ref.render_robust(ps, ref.Camera(**ck), tf, rl, ref.RpQuanta(qc.tau, qc.sigma, 64), rds)
    assert np.abs(img.pixels - rgb).max() <= RGB_TOL
    for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
        assert getattr(st, k) == rst[k], k

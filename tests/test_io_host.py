"""File formats: the library's particle / transfer-function
readers and PPM writer against the reference's own (io.hpp:62-216, through
oracle/_ref).  CPU only: no compute on the GPU."""
import os

import numpy as np
import pytest

import paper_2401_02896_b200 as S
from oracle import ref
from tests import helpers as H

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

CODE = {S.ConfigError: 1, S.IoError: 2}


def outcome_ours(fn, *a):
    try:
        return "ok", fn(*a)
    except (S.ConfigError, S.IoError) as e:
        return CODE[type(e)], None


def outcome_ref(fn, *a):
    try:
        return "ok", fn(*a)
    except ref.RefError as e:
        return e.code, None


def cloud(n=200, seed=5):
    ps = H.random_cloud(H.MT19937_64(seed), n, 1.0, -1.0, 1.0)
    ps[:, 6] = np.random.default_rng(seed).normal(size=n)  # signed values
    return ps


@pytest.mark.parametrize("binary", [False, True])
def test_particles_round_trip_matches_reference(tmp_path, binary):
    ps = cloud()
    path = str(tmp_path / ("p.sprt" if binary else "p.csv"))
    S.save_particles(ps, path, binary=binary)
    ours = S.load_particles(path)
    theirs = ref.load_particles(path)
    assert ours.shape == theirs.shape == ps.shape
    assert (ours.view(np.uint64) == theirs.view(np.uint64)).all()
    assert (ours.view(np.uint64) == ps.view(np.uint64)).all()  # %.17g round trip is exact


CSV_CASES = {
    "ok_spaces": "x,y,z,mass,density,h,value\n 1 , 2,3,4,5,6,7\n\n-1e-3,2.5,0x1p-2,1,1,0.5,-inf\n",
    "bad_header": "x,y,z,mass,rho,h,value\n1,2,3,4,5,6,7\n",
    "empty": "",
    "short_row": "x,y,z,mass,density,h,value\n1,2,3,4,5,6\n",
    "not_number": "x,y,z,mass,density,h,value\n1,2,3,4,5,6,seven\n",
    "trailing_junk": "x,y,z,mass,density,h,value\n1,2,3,4,5,6,7x\n",
    "h_zero": "x,y,z,mass,density,h,value\n1,2,3,4,5,0,7\n",
    "density_neg": "x,y,z,mass,density,h,value\n1,2,3,4,-5,1,7\n",
    "nan_value": "x,y,z,mass,density,h,value\n1,2,3,4,5,1,nan\n",
    "inf_position": "x,y,z,mass,density,h,value\ninf,2,3,4,5,1,7\n",
}


@pytest.mark.parametrize("case", sorted(CSV_CASES))
def test_particle_csv_syntax_and_validation_match_reference(tmp_path, case):
    path = str(tmp_path / "p.csv")
    open(path, "w").write(CSV_CASES[case])
    a, va = outcome_ours(S.load_particles, path)
    b, vb = outcome_ref(ref.load_particles, path)
    assert a == b, (case, a, b)
    if a == "ok":
        assert (va.view(np.uint64) == vb.view(np.uint64)).all()


def test_particle_binary_errors_match_reference(tmp_path):
    ps = cloud(10)
    path = str(tmp_path / "p.sprt")
    S.save_particles(ps, path, binary=True)
    raw = open(path, "rb").read()
    for name, data in [("truncated", raw[:-3]), ("header_only", raw[:8]),
                       ("bad_h", raw[:12 + 5 * 8] + np.float64(-1.0).tobytes() + raw[12 + 6 * 8:])]:
        p = str(tmp_path / (name + ".sprt"))
        open(p, "wb").write(data)
        a, _ = outcome_ours(S.load_particles, p)
        b, _ = outcome_ref(ref.load_particles, p)
        assert a == b != "ok", name
    a, _ = outcome_ours(S.load_particles, str(tmp_path / "missing.sprt"))
    b, _ = outcome_ref(ref.load_particles, str(tmp_path / "missing.sprt"))
    assert a == b == 2


TF_CASES = {
    "header_unsorted": "value,r,g,b,absorption\n0.6,0.1,0.35,0.8,0.9\n0,0.02,0.02,0.1,0\n0.2,.05,.1,.45,.35\n",
    "no_header": "-0.5, 0, 0, 0.2, 0.1\n0.5, 0.9, 0.3, 0.1, 1.4\n",
    "duplicate_value": "0,0,0,0,0\n0,1,1,1,1\n",
    "negative_absorption": "0,0,0,0,-1\n",
    "empty": "\n\n",
    "four_cells": "0,0,0,0\n",
}


@pytest.mark.parametrize("case", sorted(TF_CASES))
def test_transfer_function_csv_matches_reference(tmp_path, case):
    path = str(tmp_path / "tf.csv")
    open(path, "w").write(TF_CASES[case])
    a, va = outcome_ours(S.load_transfer_function, path)
    b, vb = outcome_ref(ref.load_tf, path)
    assert a == b, (case, a, b)
    if a == "ok":
        got = np.array([[p.value, p.r, p.g, p.b, p.absorption] for p in va.points])
        assert (got == vb).all()


def test_ppm_writer_bytes(tmp_path):
    rng = np.random.default_rng(1)
    img = rng.uniform(-0.2, 1.2, size=(5, 7, 3))
    img[0, 0] = [0.5 / 255, 1.5 / 255, 254.5 / 255]  # halfway cases: lround rounds away from 0
    path = str(tmp_path / "i.ppm")
    S.save_ppm(img, path)
    data = open(path, "rb").read()
    head = b"P6\n7 5\n255\n"
    assert data[:len(head)] == head
    want = np.floor(255.0 * np.clip(img, 0.0, 1.0) + 0.5).astype(np.uint8).tobytes()
    assert data[len(head):] == want


def test_bundled_desk_files_if_present():
    """The reference's own data files load identically (skipped off-container)."""
    root = "/root/reference/proj/data"
    if not os.path.isdir(root):
        pytest.skip("reference data not present")
    for f in os.listdir(root):
        p = os.path.join(root, f)
        if f.endswith(".csv") and "tf" in f:
            a = S.load_transfer_function(p)
            b = ref.load_tf(p)
            assert np.array_equal(np.array([[q.value, q.r, q.g, q.b, q.absorption] for q in a.points]), b)
        elif f.endswith((".csv", ".sprt", ".bin")) and "tf" not in f:
            try:
                b = ref.load_particles(p)
            except ref.RefError:
                continue
            a = S.load_particles(p)
            assert (a.view(np.uint64) == b.view(np.uint64)).all(), f


CAM_CASES = {
    "bundled_like": '{"mode": "pinhole", "position": [0.0, 0.55, 3.4], "look_at": [0,0,0], '
                    '"up": [0,1,0], "width": 256, "height": 192, "fov_deg": 42.0, "near": 0.0, "far": 100.0}',
    "defaults": "{}",
    "ortho": '{"mode": "orthographic", "position": [0,0,8], "look_at": [0,0,0], "ortho_height": 6}',
    "bad_mode": '{"mode": "fisheye"}',
    "bad_vec": '{"position": [0, 1]}',
    "bad_json": '{"mode": ',
    "zero_width": '{"width": 0}',
    "degenerate_up": '{"position": [0,0,0], "look_at": [0,1,0], "up": [0,1,0]}',
    "bad_fov": '{"mode": "pinhole", "fov_deg": 180}',
    "string_width": '{"width": "wide"}',
}


@pytest.mark.parametrize("case", sorted(CAM_CASES))
def test_camera_json_matches_reference(tmp_path, case):
    path = str(tmp_path / "cam.json")
    open(path, "w").write(CAM_CASES[case])
    a, va = outcome_ours(S.load_camera, path)
    b, vb = outcome_ref(ref.load_camera, path)
    assert a == b, (case, a, b)
    if a == "ok":
        for k in ("mode", "position", "look_at", "up", "width", "height", "fov_deg",
                  "ortho_height", "near", "far"):
            assert getattr(va, k) == getattr(vb, k) or tuple(getattr(va, k)) == tuple(getattr(vb, k)), k


def _msg_ours(fn, *a):
    try:
        fn(*a)
        return "ok"
    except (S.ConfigError, S.IoError) as e:
        return str(e)


def _msg_ref(fn, *a):
    try:
        fn(*a)
        return "ok"
    except ref.RefError as e:
        return str(e).split(": ", 1)[1]


def test_particle_binary_error_messages_match_reference(tmp_path):
    """read_particles_binary (io.hpp:118-138): truncation reports 'truncated
    file'; a bad record before the truncation point is reported first."""
    ps = cloud(10)
    path = str(tmp_path / "p.sprt")
    S.save_particles(ps, path, binary=True)
    raw = open(path, "rb").read()
    bad = raw[:12 + 5 * 8] + np.float64(-1.0).tobytes() + raw[12 + 6 * 8:]
    for name, data in [("truncated", raw[:-3]), ("bad_then_truncated", bad[:-3]),
                       ("bad_magic", b"SPRX" + raw[4:])]:
        p = str(tmp_path / (name + ".sprt"))
        open(p, "wb").write(data)
        assert _msg_ours(S.load_particles, p) == _msg_ref(ref.load_particles, p), name


@pytest.mark.parametrize("name", sorted(os.listdir(H.LUTS)))
def test_lut_serialize_is_the_reference_file(tmp_path, name):
    """serialize_lut / save_lut (lut.hpp:335-352, 395-399): the committed tables
    were written by the reference's save_lut; re-serialising gives the same bytes."""
    path = os.path.join(H.LUTS, name)
    lut = S.load_lut(path)
    raw = open(path, "rb").read()
    assert lut.serialize() == raw
    out = str(tmp_path / name)
    S.save_lut(lut, out)
    assert open(out, "rb").read() == raw


@pytest.mark.parametrize("width", [32, 64])
def test_render_report_matches_reference_cli(width):
    """The CLI's render report (sphray_main.cpp:196-256), field for field and
    byte for byte, given the same RenderStats (here the reference's own)."""
    ps = H.random_cloud(H.MT19937_64(31337), 120, 1.6, -1.2, 1.2)
    ck = H.render_test_camera_kwargs()
    lp = H.lut_path(4, 3, 16)
    rl, lut = ref.Lut(lp), S.load_lut(lp)
    want = ref.render_report(ps, ref.Camera(**ck), H.TEST_TF, rl, width, seed=5, image="out.ppm")
    ds = S.dataset_stats(ps, lut)
    qc = S.choose_quanta(lut, ds, width)
    rds = ref.dataset_stats(ps, rl)
    _, rst, _ = ref.render(ps, ref.Camera(**ck), H.TEST_TF, rl, ref.choose_quanta(rl, rds, width), rds,
                           accum_bits=width)
    got = S.render_report(lut, ds, qc, S.RenderStats(**rst), seed=5, image="out.ppm")
    assert got == want
    empty = ref.render_report(np.zeros((0, 7)), ref.Camera(**ck), H.TEST_TF, rl, width, seed=5,
                              image="out.ppm")
    assert S.render_report(lut, ds, qc, None, seed=5, image="out.ppm") == empty

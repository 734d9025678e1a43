"""CPU: the C-ABI library loads, exports every entry point include/sphray_gpu.h
declares, fails loudly without a GPU, and its host-side logic (dataset stats,
quanta, .splt parsing, scene generators) matches the reference bit for bit."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2401_02896_b200 as S
from tests import helpers as H

HEADER = os.path.join(H.ROOT, "include", "sphray_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    inline = set(re.findall(r"static\s+inline\s+[\w\s\*]+?\b(sphray_[a-z_0-9]+)\s*\(", text))
    return sorted(set(re.findall(r"\b(sphray_[a-z_0-9]+)\s*\(", text)) - inline)


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("sphray_render_scene", "sphray_scene_upload", "sphray_scene_render",
                 "sphray_scene_hits", "sphray_scene_pieces", "sphray_quantize_hits",
                 "sphray_context_create", "sphray_context_init_comm", "sphray_lut_parse",
                 "sphray_compute_dataset_stats", "sphray_choose_quanta"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = S.load_library()
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing
    assert L.sphray_abi_version() == 2


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", S.lib_path()], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(S.CudaError):
        S.Context(0)


def test_lut_parse_and_malformed_files(tmp_path):
    lut = S.load_lut(H.lut_path(4, 3, 1024))
    assert (lut.kernel_id, lut.q, lut.K, lut.D, lut.N) == ("cubic-bspline", 2.0, 4, 3, 1024)
    raw = open(H.lut_path(4, 3, 16), "rb").read()
    with pytest.raises(S.IoError):
        S.Lut(b"XXXX" + raw[4:])  # bad magic (lut_tests.cpp:254-293)
    with pytest.raises(S.IoError):
        S.Lut(raw[:-3])  # truncated
    with pytest.raises(S.IoError):
        S.Lut(raw + b"\0")  # trailing bytes
    bad = bytearray(raw)
    bad[4] = 2  # version
    with pytest.raises(S.IoError):
        S.Lut(bytes(bad))
    with pytest.raises(S.IoError):
        S.load_lut(str(tmp_path / "missing.splt"))


@pytest.mark.parametrize("name", ["desk", "render_test", "blob3000", "kd_K7_D5", "kd_K6_D6"])
def test_dataset_stats_and_quanta_match_reference(name):
    z = np.load(os.path.join(H.GOLDEN, name + ".npz"))
    lut = S.load_lut(os.path.join(H.LUTS, str(z["lut"])))
    ds = S.dataset_stats(z["particles"], lut)
    assert ds.h_r == float(z["h_r"]) and ds.a_max == float(z["a_max"])
    assert ds.phi_repr == float(z["phi_repr"])
    qc = S.choose_quanta(lut, ds)
    assert qc.tau == float(z["tau"]) and qc.sigma == float(z["sigma"])


def test_kernel_constants_pinned_to_reference():
    try:
        from oracle import ref
        if not ref.available():
            raise ImportError
    except ImportError:
        pytest.skip("oracle/_ref not built")
    k, kp = ref.kernel_constants()
    assert k == S.KAPPA_CUBIC and kp == S.KAPPA_PRIME_CUBIC


def test_dataset_stats_errors():
    lut = S.load_lut(H.lut_path(4, 3, 16))
    with pytest.raises(S.ConfigError):
        S.dataset_stats(np.zeros((0, 7)), lut)
    with pytest.raises(S.ConfigError):
        S.dataset_stats(np.array([[0, 0, 0, 1, 0.0, 0.1, 1]]), lut)  # zero density
    with pytest.raises(S.ConfigError):
        S.choose_quanta(lut, S.DatasetStats(h_r=1.0, phi_repr=1.0, a_max=0.0))


@pytest.mark.parametrize("config", [1, 2, 4])
def test_blob_generator_is_deterministic(config):
    n = 5000
    a = S.generate_scene(config, n=n)
    b = S.generate_scene(config, n=n)
    assert a.shape == (n, 7) and (a == b).all()
    rho = np.exp(-(a[:, 0] ** 2 + a[:, 1] ** 2 + a[:, 2] ** 2) / 2.0) + 0.05
    np.testing.assert_allclose(a[:, 4], rho, rtol=1e-15)
    assert (a[:, 4] == a[:, 6]).all() and (a[:, 3] == 1.0 / n).all()


def test_clustered_generator_spans_decades_of_h():
    a = S.generate_scene(3, n=200000)
    h = a[:, 5]
    assert (h > 0).all() and h.max() / h.min() > 100.0
    assert (a[:, 4] == a[:, 6]).all()
    b = S.generate_scene(3, n=200000)
    assert (a == b).all()

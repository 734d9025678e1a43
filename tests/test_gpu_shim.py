"""GPU: the C++ drop-in.  oracle/_ref/shim_demo is a reference-side program
(built against the unmodified reference headers) that calls
sphray::render_scene<int64_t> and sphray::gpu::render_scene<int64_t>
(include/sphray_gpu.hpp) with identical arguments and compares them."""
import os
import subprocess

import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu
DEMO = os.path.join(H.ROOT, "oracle", "_ref", "shim_demo")


def test_cpp_shim_is_a_drop_in():
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/shim_demo not built (needs /root/reference at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "SHIM_OK" in out.stdout

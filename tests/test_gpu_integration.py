"""The INTEGRATION.md drop-in on the GPU: the reference's own solve_krylov
driving the GPU LinearOps (oracle/_ref/linearop_demo, compiled against the
unmodified reference headers), and the bench/smoke entry points."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "linearop_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="linearop_demo not built (reference sources absent at build time)")
@pytest.mark.parametrize("args", [["10000", "50", "1.0", "3000", "8", "0"], ["10000", "50", "0.5", "2001", "8", "1"],
                                  ["20000", "10", "1.0", "1", "4", "1"]])
def test_reference_krylov_with_gpu_linearops(args):
    r = subprocess.run([DEMO, *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def test_smoke_entry_point():
    import __graft_entry__ as g
    g.smoke()

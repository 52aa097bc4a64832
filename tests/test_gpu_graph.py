"""CUDA-graph step ranges (dg_engine_run_steps, DG_RUN_GRAPH) are bit-exact
vs the oracle's fp32 mirror at BASELINE config 1's shape (8 nodes, 2^20
params, 100 steps), on the default and the x-double-buffered kernel paths."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {"default": {}, "pingpong_legacy": {"DG_XSHARE": "0", "DG_PINGPONG_MIN_NC": "1"}}


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("d", [1 << 20, 5003])
def test_graph_steps_bit_exact(path, d):
    p = subprocess.run([sys.executable, os.path.join(HERE, "graph_parity_main.py"), str(d)],
                       env={**os.environ, **PATHS[path]}, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]

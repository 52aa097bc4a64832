"""Bounds checks without compute-sanitizer (closed on this pool): NaN canaries
in the row padding of every engine buffer survive every kernel path, and the
results stay bit-exact vs the oracle (tests/guard_main.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
LEGACY = {"DG_XSHARE": "0"}
PATHS = {"default": {}, "xshare_pairs": {"DG_XSHARE_PAIRS": "1"},
         "legacy": {**LEGACY}, "pingpong": {**LEGACY, "DG_PINGPONG_MIN_NC": "1"},
         "tma": {**LEGACY, "DG_TMA": "2", "DG_PINGPONG_MIN_NC": "0"},
         "coop": {**LEGACY, "DG_TMA": "0", "DG_COOP_MIN_NC": "2", "DG_PINGPONG_MIN_NC": "0"},
         "warps": {**LEGACY, "DG_TMA": "0", "DG_PINGPONG_MIN_NC": "1", "DG_WARPS_MIN_NC": "1"}}


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("d", [1003, 4099])
def test_padding_canaries_survive(path, d):
    p = subprocess.run([sys.executable, os.path.join(HERE, "guard_main.py"), str(d)], env={**os.environ, **PATHS[path]},
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]

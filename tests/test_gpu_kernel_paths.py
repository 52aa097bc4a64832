"""Every fused-kernel path (x-sharing kernel = default, the legacy
warp-specialised TMA, cooperative, per-thread and warp-per-node kernels) must be
bit-exact against the oracle's fp32 mirror for every topology; the path is
chosen by env knobs read once per process, hence one subprocess per path."""
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
PATHS = {"default": {},                       # x-sharing kernel
         "xshare_small_grid": {"DG_WAVES": "0.3"},
         "legacy": {**LEGACY},
         "pingpong_all": {**LEGACY, "DG_PINGPONG_MIN_NC": "1"},
         "tma_all": {**LEGACY, "DG_TMA": "2", "DG_PINGPONG_MIN_NC": "0"},
         "tma_pingpong": {**LEGACY, "DG_TMA": "2", "DG_PINGPONG_MIN_NC": "1"},
         "per_thread_all": {**LEGACY, "DG_TMA": "0", "DG_COOP_MIN_NC": "99", "DG_PINGPONG_MIN_NC": "0"},
         "coop_all": {**LEGACY, "DG_TMA": "0", "DG_COOP_MIN_NC": "2", "DG_PINGPONG_MIN_NC": "0"},
         "warps_all": {**LEGACY, "DG_TMA": "0", "DG_PINGPONG_MIN_NC": "1", "DG_WARPS_MIN_NC": "1"},
         # fault injection (SPEC.md:317 Jacobi snapshot): a 2 ms spin before every
         # step and the stale x buffer overwritten with NaN as soon as it is free
         "fault_pingpong": {**LEGACY, "DG_PINGPONG_MIN_NC": "1", "DG_FAULT_POISON": "1",
                            "DG_FAULT_DELAY_US": "2000"},
         "fault_default": {"DG_FAULT_POISON": "1", "DG_FAULT_DELAY_US": "2000"}}


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("d", [5003, 300_001])
def test_kernel_path_bit_exact(path, d):
    env = {**os.environ, **PATHS[path]}
    p = subprocess.run([sys.executable, os.path.join(HERE, "engine_parity_main.py"), str(d)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]

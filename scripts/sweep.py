"""Kernel-variant sweep on one GPU: runs bench.py (kernel/step numbers only)
for each variant library in build/variants and for DG_WAVES settings.
Usage (on the GPU box): python scripts/sweep.py [extra bench args]"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
extra = sys.argv[1:]
base = dict(kv.split("=", 1) for kv in os.environ.get("SWEEP_ENV", "").split() if "=" in kv)
runs = [("default", dict(base))]
for lib in sorted(glob.glob(os.path.join(ROOT, "build", "variants", "libdg_*.so"))):
    runs.append((os.path.basename(lib)[6:-3], {**base, "DG_LIB": lib}))
if not base:
    runs.append(("waves2", {"DG_WAVES": "2"}))
for name, env in runs:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "30", "--warmup", "4", "--no-e2e",
           "--no-cpu-baseline"] + extra
    p = subprocess.run(cmd, env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    line = next((l for l in p.stdout.splitlines() if l.startswith("{")), None)
    if not line:
        print(f"{name:10s} FAILED rc={p.returncode} {p.stderr[-400:]}", flush=True)
        continue
    j = json.loads(line)
    r = j["roofline"]
    print(f"{name:10s} value={j['value']:.4e} ms/step={j['ms_per_step']:.3f} kernel={r['achieved']:.0f} GB/s "
          f"frac={r['frac']:.3f} step_frac={j['step_roofline']['frac']:.3f}", flush=True)

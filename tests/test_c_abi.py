"""The C ABI from a native C caller (tests/c_abi_main.c, compiled with gcc
against include/dg.h and linked with libdg.so): struct layouts agree with the
ctypes mirror, schedules agree with the oracle, and (GPU) 12 engine steps
driven from C are bit-exact vs the oracle's fp32 mirror."""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2410_11998_b200")
SRC = os.path.join(ROOT, "tests", "c_abi_main.c")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libdg.so")):
        pytest.fail("libdg.so not built (python -c 'import __graft_entry__ as g; g.build()')")
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    out = str(tmp_path_factory.mktemp("cabi") / "c_abi_main")
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Werror", "-o", out, SRC, "-I", os.path.join(ROOT, "include"),
                    "-L", LIBDIR, "-ldg", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


def run(exe, *args):
    p = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    return p.stdout.splitlines()


def test_struct_layouts_match_ctypes(exe, dg):
    mirror = {"dg_adam_cfg": dg._AdamCfg, "dg_validation": dg._Validation, "dg_engine_config": dg._EngineConfig,
              "dg_engine_stats": dg._EngineStats, "dg_rm_params": dg._RmParams}
    import ctypes
    seen = {k: set() for k in mirror}
    for line in run(exe, "layout"):
        f = line.split()
        if f[0] == "sizeof":
            assert ctypes.sizeof(mirror[f[1]]) == int(f[2]), line
        elif f[0] == "field":
            desc = getattr(mirror[f[1]], f[2])
            assert (desc.offset, desc.size) == (int(f[3]), int(f[4])), line
            seen[f[1]].add(f[2])
    for name, cls in mirror.items():  # every ctypes field exists in C (no extra or renamed fields)
        assert seen[name] == {n for n, _ in cls._fields_}, name


def test_schedules_from_c_match_oracle(exe, oracle):
    makers = {"complete8": lambda: oracle.make_complete(8), "one_peer_ring8": lambda: oracle.make_one_peer_ring(8),
              "one_peer_exponential8": lambda: oracle.make_one_peer_exponential(8),
              "one_peer_exponential16": lambda: oracle.make_one_peer_exponential(16),
              "aer8_2": lambda: oracle.make_aer(8, 2),
              "static_exponential8": lambda: oracle.make_static_exponential(8)}
    cur, checked = None, 0
    for line in run(exe, "schedules"):
        f = line.split()
        if f[0] == "schedule":
            cur = makers[f[1]]()
            kv = dict(x.split("=") for x in f[2:])
            assert (int(kv["n"]), int(kv["period"]), int(kv["wpn"])) == (cur.workers, cur.period,
                                                                          cur.workers_per_node), line
            assert kv["name"] == {"aer8_2": "aer"}.get(f[1], f[1].rstrip("0123456789")), line
        elif f[0] == "round":
            r, i = int(f[1]), int(f[3].rstrip(":"))
            idx, w = cur.neighbors_at(r)[i]
            got = [x.split(":") for x in f[4:]]
            assert [int(a) for a, _ in got] == list(idx), line
            assert [float(b) for _, b in got] == list(w), line   # %.17g round-trips exactly
            checked += 1
        elif f[0] == "validate":
            assert f[2] == "pass=1", line
        elif f[0] == "error":
            assert f[2] == "rc=2", line                         # DG_CONFIG_ERROR (ConfigError)
    assert checked > 100


@pytest.mark.gpu
def test_engine_from_c_bit_exact(exe, oracle, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "state.bin")
    run(exe, "engine", out)
    n, d, T, seed = 8, 4099, 12, 2410
    raw = np.fromfile(out, np.float32)
    cfgs = [(0, dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1), ("x", "m", "v")),
            (1, dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4), ("x", "m", "v", "b"))]
    pos = 0
    for algo, c, keys in cfgs:
        st = oracle.init_state(n, d, seed, True, np.float32, algo)
        oracle.run(oracle.make_one_peer_ring(n), algo, oracle.OptimizerConfig(**c), seed, st, 1, T, T)
        for k in keys:
            got = raw[pos:pos + n * d].reshape(n, d)
            pos += n * d
            assert np.array_equal(got.view(np.uint32), st[k].view(np.uint32)), (algo, k)
    assert pos == raw.size


def test_cpp_adapter_compiles_and_matches_oracle(oracle, tmp_path):
    """a declab-shaped C++20 adapter over dg.h (RAII
    schedule, errors.hpp taxonomy) compiled with g++ and checked vs the oracle."""
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = str(tmp_path / "cpp_adapter")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp_adapter_main.cpp"), "-I", os.path.join(ROOT, "include"),
                    "-L", LIBDIR, "-ldg", f"-Wl,-rpath,{LIBDIR}"], check=True)
    makers = {"one_peer_exponential8": lambda: oracle.make_one_peer_exponential(8),
              "aer8_2": lambda: oracle.make_aer(8, 2),
              "static_exponential8": lambda: oracle.make_static_exponential(8)}
    cur, rows = None, 0
    out = run(exe)
    for line in out:
        f = line.split()
        if f[0] == "schedule":
            cur = makers[f[1]]()
        elif f[0] == "round":
            r, i = int(f[1]), int(f[3].rstrip(":"))
            assert [int(x) for x in f[4:]] == list(cur.neighbors_at(r)[i][0]), line
            rows += 1
        elif f[0] == "validate":
            assert f[-1] == "pass=1", line
    assert rows == 8 * (3 + 4 + 1)
    assert out[-1] == "error ConfigError"

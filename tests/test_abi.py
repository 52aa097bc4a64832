"""The drop-in boundary: libdg.so loads without a GPU and exports exactly the
C ABI declared in include/dg.h; the product never links the oracle."""
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dg.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_api():
    names = declared()
    for must in ("dg_make_one_peer_ring", "dg_make_one_peer_exponential", "dg_make_aer",
                 "dg_make_static_exponential", "dg_schedule_neighbors", "dg_schedule_matrix",
                 "dg_dadam_step_f32", "dg_accum_adam_step_f32", "dg_engine_create", "dg_engine_step"):
        assert must in names


def test_library_exports_every_declared_symbol(dg):
    L = dg.lib()
    for name in declared():
        assert hasattr(L, name), name
    assert set(declared()) == set(dg.SIGNATURES), "ctypes signature table out of sync with dg.h"


def test_exports_are_c_symbols_and_no_oracle():
    so = dg_path()
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for name in declared():
        assert name in syms, name  # unmangled => extern "C"
    assert not any(s.startswith("or_") or s.startswith("ref_") for s in syms)
    ldd = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "declab" not in ldd
    assert "libnccl" in ldd


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", dg_path()], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def dg_path():
    import paper_2410_11998_b200 as dg
    return dg.library_path()


def test_errors_map_to_reference_taxonomy(dg):
    import pytest
    with pytest.raises(dg.ConfigError) as e:
        dg.make_aer(6, 4)
    assert e.value.code == 2 and isinstance(e.value, ValueError)
    assert dg.DivergenceError.code == 3 and dg.InvariantError.code == 4


def test_every_engine_knob_is_documented():
    """Every environment knob the library reads is listed in INTEGRATION.md section 7."""
    import glob
    root = ROOT
    knobs = set()
    for f in glob.glob(os.path.join(root, "paper_2410_11998_b200", "csrc", "*.*")):
        if f.endswith((".cu", ".cuh", ".cpp", ".hpp")):
            src = open(f).read()
            knobs |= set(re.findall(r'getenv\("([A-Z_0-9]+)"\)', src))
            knobs |= set(re.findall(r'env_int\("([A-Z_0-9]+)"', src))
    doc = open(os.path.join(root, "INTEGRATION.md")).read()
    assert knobs and all(f"`{k}`" in doc for k in knobs), sorted(k for k in knobs if f"`{k}`" not in doc)

"""Generate the golden fixtures in tests/golden/ from the REFERENCE build.

Run here (where /root/reference exists) after `make -C oracle`:
    python tests/golden/make_golden.py

Every value below comes from oracle/_ref/libdeclab_ref.so, i.e. the
reference's own proj/src/rng.cpp and proj/src/vec.cpp compiled from
/root/reference (see oracle/Makefile), composed per SPEC.md:272-298 in
oracle/ref_shim.cpp.  The fixtures let the GPU box (which has no
/root/reference) pin the oracle restatement.

Neighbour tables come from the SPEC's schedule definitions (the reference has
no topology.cpp); they are written out explicitly here, independent of both
oracle.cpp and libdg, and stored in the fixture.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SEED = 2410


def rng_kats():
    keys = [(0, 1, 0, 0), (42, 4, 0, 0), (42, 2, 3, 7), (42, 6, 7, 0), (2410, 2, 5, 100),
            (2410, 4, 0, 0), (2410, 6, 63, 0), (2**64 - 1, 3, 2**40, 2**33)]
    R = O.ref()
    out = []
    for k in keys:
        u = np.empty(8, np.uint64)
        R.ref_rng_u64(*k, 8, u)
        unit = np.empty(8, np.float64)
        R.ref_rng_unit(*k, 8, unit)
        out.append({"key": list(k), "u64": [int(x) for x in u], "unit": [float(x).hex() for x in unit]})
    speed = [R.ref_speed_multiplier(1, 0, 0, 0.0134, k) for k in range(5)]
    m = np.array([0.5, -2.0, 1e-12, 3.0]); v = np.array([0.25, 4.0, 1e-30, 0.0])
    div = np.empty(4)
    R.ref_div_by_sqrt_plus_eps(m, v, 4, 1e-8, div)
    return {"streams": out, "speed_multiplier_sigma2_0.0134": [float(x).hex() for x in speed],
            "div_by_sqrt_plus_eps": {"m": m.tolist(), "v": v.tolist(), "eps": 1e-8,
                                     "out": [float(x).hex() for x in div]}}


# Schedules written from the SPEC / Appendix B definitions.
def tables_ring(n):
    r1 = [sorted({i, i ^ 1}) for i in range(n)]
    r2 = [sorted({i, (i + 1) % n if i % 2 else (i - 1) % n}) for i in range(n)]
    return [r1, r2], [[[0.5, 0.5]] * n] * 2


def tables_aer8_2():  # Appendix B: r1 {0,1}{2,3}{4..7}; r2 {0..3}{4,5}{6,7}; r3 {0,1,4,5}{2,3}{6,7}; r4 {2,3,6,7}{0,1}{4,5}
    groups = [[[0, 1], [2, 3], [4, 5, 6, 7]], [[0, 1, 2, 3], [4, 5], [6, 7]],
              [[0, 1, 4, 5], [2, 3], [6, 7]], [[2, 3, 6, 7], [0, 1], [4, 5]]]
    idx, w = [], []
    for gs in groups:
        ri, rw = [None] * 8, [None] * 8
        for g in gs:
            for i in g:
                ri[i] = g
                rw[i] = [1.0 / len(g)] * len(g)
        idx.append(ri)
        w.append(rw)
    return idx, w


def tables_static_exp8():  # {i, i+-1, i+-2, i+4}, w = 1/6
    idx = [sorted({i, (i + 1) % 8, (i - 1) % 8, (i + 2) % 8, (i - 2) % 8, (i + 4) % 8}) for i in range(8)]
    return [idx], [[[1.0 / 6] * 6] * 8]


def pack(idx, w, n):
    P = len(idx)
    maxdeg = max(len(x) for r in idx for x in r)
    I = np.zeros((P, n, maxdeg), np.int32)
    W = np.zeros((P, n, maxdeg), np.float64)
    Cn = np.zeros((P, n), np.int32)
    for r in range(P):
        for i in range(n):
            I[r, i, :len(idx[r][i])] = idx[r][i]
            W[r, i, :len(idx[r][i])] = w[r][i]
            Cn[r, i] = len(idx[r][i])
    return I, W, Cn, maxdeg


def ref_trajectory(name, idx, w, n, d, algo, cfg, T, dispersed):
    import ctypes as C
    I, W, Cn, maxdeg = pack(idx, w, n)
    st = O.init_state(n, d, SEED, dispersed, np.float64, algo)
    el = C.c_double()
    c = cfg.c()
    R = O.ref()
    rc = R.ref_run(algo, n, d, len(idx), maxdeg, I.reshape(-1), W.reshape(-1), Cn.reshape(-1),
                   C.byref(c), SEED, 1, T, T, 1, 1, None, st["x"].reshape(-1), st["m"].reshape(-1),
                   st["v"].reshape(-1), None if st["b"] is None else st["b"].ctypes.data_as(C.c_void_p),
                   C.byref(el))
    assert rc == 0, R.ref_last_error()
    arrs = {"x": st["x"], "m": st["m"], "v": st["v"], "nbr_idx": I, "nbr_w": W, "nbr_cnt": Cn}
    if st["b"] is not None:
        arrs["b"] = st["b"]
    meta = dict(name=name, n=n, d=d, algo=algo, T=T, seed=SEED, dispersed=dispersed,
                alpha=cfg.alpha, beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps, s=cfg.s,
                paper_literal=cfg.paper_literal)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=json.dumps(meta), **arrs)


def main():
    with open(os.path.join(OUT, "rng_kat.json"), "w") as f:
        json.dump(rng_kats(), f, indent=1)
    dadam = O.OptimizerConfig(2e-3, 0.974, 0.999, 1e-8, 1).rounded_f32()
    accum = O.OptimizerConfig(8e-4, 0.9, 0.999, 1e-8, 4).rounded_f32()
    ring_i, ring_w = tables_ring(8)
    ref_trajectory("ref_ring8_dadam", ring_i, ring_w, 8, 256, O.DADAM, dadam, 100, True)
    ref_trajectory("ref_ring8_accum4", ring_i, ring_w, 8, 256, O.ACCUM, accum, 100, True)
    ai, aw = tables_aer8_2()
    ref_trajectory("ref_aer8_accum4", ai, aw, 8, 128, O.ACCUM, accum, 100, True)
    si, sw = tables_static_exp8()
    ref_trajectory("ref_staticexp8_dadam", si, sw, 8, 128, O.DADAM, dadam, 100, False)
    lit = O.OptimizerConfig(8e-4, 0.9, 0.999, 1e-8, 4, True).rounded_f32()
    ref_trajectory("ref_ring8_accum4_literal", ring_i, ring_w, 8, 64, O.ACCUM, lit, 40, True)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

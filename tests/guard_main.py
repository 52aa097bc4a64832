"""Subprocess body for tests/test_gpu_guard.py: bounds checks of every kernel
path without compute-sanitizer (closed on this pool).  Each node's bucket
row is d_pad = round_up(d, 64) floats; the kernels own [0, d).  The padding
[d, d_pad) of every buffer (x, both x buffers when ping-ponged, g, m, v,
acc) is filled with a NaN canary before stepping and must be bit-identical
afterwards, and the results must stay bit-exact vs the oracle (a write past
the row end would land in the next node's row).  Argument: d (not a multiple
of 64).  Exit code 0 = clean."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2410_11998_b200.ddp import device_view  # noqa: E402

SEED = 2410
CANARY = np.uint32(0x7FBADBAD)
TOPOS = [("make_one_peer_ring", "ONE_PEER_RING", (8,)), ("make_one_peer_exponential", "ONE_PEER_EXP", (8,)),
         ("make_static_exponential", "STATIC_EXP", (8,)), ("make_aer", "AER", (8, 2)),
         ("make_complete", "COMPLETE", (8,)), ("make_static_exponential", "STATIC_EXP", (16,))]
CFG = {0: dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1),
       1: dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)}


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 1003
    d_pad = (d + 63) // 64 * 64
    assert d_pad > d
    T = 12
    bad = 0
    for fn, kind, args in TOPOS:
        for algo in (0, 1):
            eng = dg.Engine(getattr(dg, fn)(*args), d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T)
            n = eng.local_nodes
            kinds = [dg.X, dg.G, dg.M, dg.V] + ([dg.ACC] if algo else [])
            guarded = {}   # device pointer of a row -> torch view of its padding

            def guard_all(first_time_zero):
                nonlocal bad
                for w in kinds:
                    for i in range(n):
                        p = eng.buffer(i, w)
                        if p in guarded:
                            continue
                        pad = device_view(p, d_pad)[d:]
                        torch.cuda.synchronize()
                        if first_time_zero and not torch.all(pad.view(torch.int32) == 0):
                            print(f"PADDING WRITTEN (fresh buffer) {fn}{args} algo={algo} kind={w} node={i}", flush=True)
                            bad += 1
                        pad.view(torch.int32).fill_(int(CANARY.view(np.int32)))
                        guarded[p] = pad
                torch.cuda.synchronize()

            eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
            guard_all(False)
            for t in range(1, T + 1):
                eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
                eng.step(t)
                eng.sync()
                guard_all(True)   # a buffer that just became current (ping-pong) must be untouched too
            for p, pad in guarded.items():
                if not torch.all(pad.view(torch.int32) == int(CANARY.view(np.int32))):
                    print(f"CANARY OVERWRITTEN {fn}{args} algo={algo} ptr={p:#x}", flush=True)
                    bad += 1
            st = O.init_state(n, d, SEED, True, np.float32, algo)
            O.run(O.make(getattr(O, kind), *args), algo, O.OptimizerConfig(**CFG[algo]), SEED, st, 1, T, T)
            for k, w in [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo else []):
                got = np.stack([eng.download(i, w) for i in range(n)])
                if not np.array_equal(got.view(np.uint32), st[k].view(np.uint32)):
                    print(f"MISMATCH {fn}{args} algo={algo} {k}", flush=True)
                    bad += 1
            eng.close()
    print("ok" if not bad else f"{bad} problems")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

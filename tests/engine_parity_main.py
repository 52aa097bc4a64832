"""Subprocess body for tests/test_gpu_kernel_paths.py: runs the fused engine
over every topology/algorithm with whatever kernel-path env (DG_TMA,
DG_COOP_MIN_NC) the parent set, and checks bit-exactness against the
oracle's fp32 mirror.  Exit code 0 = all equal."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

SEED = 2410
TOPOS = [("make_one_peer_ring", "ONE_PEER_RING", (8,)), ("make_one_peer_exponential", "ONE_PEER_EXP", (8,)),
         ("make_static_exponential", "STATIC_EXP", (8,)), ("make_aer", "AER", (8, 2)),
         ("make_aer", "AER", (16, 4)), ("make_complete", "COMPLETE", (8,)),
         ("make_static_exponential", "STATIC_EXP", (16,)), ("make_complete", "COMPLETE", (16,)),
         # > 16 resident nodes: legacy rounds run in several launches (<= 16 members each)
         ("make_one_peer_exponential", "ONE_PEER_EXP", (64,)), ("make_static_exponential", "STATIC_EXP", (32,))]
CFG = {0: dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1),
       1: dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)}


def main():
    d, T = int(sys.argv[1]) if len(sys.argv) > 1 else 5003, 12
    bad = 0
    for fn, kind, args in TOPOS:
        for algo in (0, 1):
            eng = dg.Engine(getattr(dg, fn)(*args), d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T)
            eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
            for t in range(1, T + 1):
                eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
                eng.step(t)
            eng.sync()
            st = O.init_state(eng.local_nodes, d, SEED, True, np.float32, algo)
            O.run(O.make(getattr(O, kind), *args), algo, O.OptimizerConfig(**CFG[algo]), SEED, st, 1, T, T)
            keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo else [])
            for k, w in keys:
                got = np.stack([eng.download(i, w) for i in range(eng.local_nodes)])
                if not np.array_equal(got.view(np.uint32), st[k].view(np.uint32)):
                    print(f"MISMATCH {fn}{args} algo={algo} {k}", flush=True)
                    bad += 1
            eng.close()
    print("ok" if not bad else f"{bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

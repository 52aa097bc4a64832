"""Subprocess body for tests/test_gpu_graph.py: dg_engine_run_steps with CUDA
graphs (DG_RUN_GRAPH) vs the oracle's fp32 mirror, gradient held fixed (a
graph replays the same kernels; g is an input the caller refreshes between
ranges).  Ranges are captured, replayed twice (the second replay of the same
t-range re-runs those iterations on the evolved state, as the oracle does) and
mixed with eager steps; with DG_PINGPONG_MIN_NC=1 (legacy kernels) every
round flips the x buffer, so replays must start from the captured buffer.
Argument: d (>= 100000: BASELINE config 1's ring only).  Exit code 0 = all equal."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

SEED = 2410
CFG = {0: dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1),
       1: dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)}
TOPOS = [("make_one_peer_ring", "ONE_PEER_RING", (8,)), ("make_static_exponential", "STATIC_EXP", (8,)),
         ("make_one_peer_exponential", "ONE_PEER_EXP", (8,))]
# (t_first, t_last, graph) in call order; T = 100 (BASELINE config 1: 100 steps)
PLAN = [(1, 3, False), (4, 51, True), (52, 52, False), (53, 56, True), (53, 56, True), (57, 96, True),
        (97, 100, True)]


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    topos = TOPOS if d < 100_000 else TOPOS[:1]   # full config-1 size: its own topology (ring)
    T = 100
    bad = 0
    for fn, kind, args in topos:
        for algo in (0, 1):
            eng = dg.Engine(getattr(dg, fn)(*args), d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T)
            eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
            eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, 1)
            n = eng.local_nodes
            st = O.init_state(n, d, SEED, True, np.float32, algo)
            g = np.stack([O.fill_f32(SEED, O.MINIBATCH, i, 1, d) for i in range(n)])
            osched = O.make(getattr(O, kind), *args)
            ocfg = O.OptimizerConfig(**CFG[algo])
            for t0, t1, graph in PLAN:
                eng.run_steps(t0, t1, graph=graph)
                O.run_fixed_g(osched, algo, ocfg, st, g, t0, t1, T)
            eng.sync()
            stats = eng.stats()
            keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo else [])
            for k, w in keys:
                got = np.stack([eng.download(i, w) for i in range(n)])
                if not np.array_equal(got.view(np.uint32), st[k].view(np.uint32)):
                    print(f"MISMATCH {fn}{args} algo={algo} {k}", flush=True)
                    bad += 1
            steps = sum(t1 - t0 + 1 for t0, t1, _ in PLAN)
            if stats["steps"] != steps:
                print(f"STATS steps {stats['steps']} != {steps}", flush=True)
                bad += 1
            print(f"{fn}{args} algo={algo} steps={stats['steps']} launches={stats['kernel_launches']}", flush=True)
            eng.close()
    print("ok" if not bad else f"{bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

"""Shared helpers for full-size (BASELINE configs 2-5) parity checks: run the
fused engine on the full bucket, gather sampled columns on the device, replay
exactly those columns with the oracle (every column evolves independently),
and compare bit-exactly with the fp32 mirror and norm-wise with fp64."""
import numpy as np

SEED = 2410
CFG = {0: dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1),
       1: dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)}


def sample_columns(d, n=32768, seed=7):
    rng = np.random.default_rng(seed)
    cols = rng.choice(d, size=min(n, d), replace=False)
    extra = [0, 1, 2, 3, d - 1, d - 2, d - 3, d - 4, d // 2]
    return np.unique(np.concatenate([cols, [c for c in extra if 0 <= c < d]])).astype(np.uint64)


def run_engine_cols(dg, sched, d, algo, T, cols, **engine_kw):
    eng = dg.Engine(sched, d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T, **engine_kw)
    eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
    for t in range(1, T + 1):
        eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
        eng.step(t)
    eng.sync()
    keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo == 1 else [])
    got = {k: np.stack([eng.gather(i, w, cols) for i in range(eng.local_nodes)]) for k, w in keys}
    first, nl = eng.first_node, eng.local_nodes
    eng.close()
    return got, first, nl


def check_against_oracle(O, osched, algo, T, cols, got, first, nl, normwise):
    """Returns a list of failure strings (empty = pass)."""
    bad = []
    ocfg = O.OptimizerConfig(**CFG[algo])
    f32 = O.run_cols(osched, algo, ocfg, SEED, cols, True, 1, T, T, np.float32)
    f64 = O.run_cols(osched, algo, ocfg.rounded_f32(), SEED, cols, True, 1, T, T, np.float64)
    for k in got:
        want = f32[k][first:first + nl]
        if not np.array_equal(got[k].view(np.uint32), want.view(np.uint32)):
            nbad = int((got[k].view(np.uint32) != want.view(np.uint32)).sum())
            bad.append(f"{k}: {nbad} columns differ from the fp32 mirror")
        if k in ("x", "m", "v"):
            for i in range(nl):
                e = normwise(got[k][i], f64[k][first + i])
                if e > 1e-6:
                    bad.append(f"{k}[{first + i}] norm-wise {e:.3e} > 1e-6 vs fp64")
    return bad

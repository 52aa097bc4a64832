"""GPU parity: libdg's CUDA path vs the CPU oracle on identical synthetic
buckets and seeds (SURVEY.md 8(c) parity protocol).

* BIT-EXACT (elementwise, fp32 bit patterns) against the oracle's fp32 mirror
  (oracle.cpp, SURVEY.md Appendix A op order);
* within 1e-6 NORM-WISE relative (||a-b||_2/||b||_2, per state tensor per node)
  against the fp64 oracle fed fp32-rounded hyperparameters after 100 steps
  (north_star tolerance; elementwise 1e-6 vs fp64 is infeasible).
"""
import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

SEED = 2410
DADAM_CFG = dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1)
ACCUM_CFG = dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bit_exact(a, b, what):
    ba, bb = bits(a), bits(b)
    if not np.array_equal(ba, bb):
        bad = np.flatnonzero(ba != bb)
        raise AssertionError(f"{what}: {bad.size} mismatching elements, first at {bad[0]}: "
                             f"{np.asarray(a).ravel()[bad[0]]!r} vs {np.asarray(b).ravel()[bad[0]]!r}")


def cfgs(dg, oracle, algo, paper_literal=False):
    c = DADAM_CFG if algo == 0 else ACCUM_CFG
    return (dg.OptimizerConfig(**c, paper_literal=paper_literal),
            oracle.OptimizerConfig(**c, paper_literal=paper_literal))


# --------------------------------------------------------------------------- synthetic inputs
@pytest.mark.parametrize("key", [(SEED, 2, 0, 1), (SEED, 2, 7, 100), (SEED, 4, 0, 0), (42, 6, 63, 0)])
@pytest.mark.parametrize("n", [1, 7, 4096, 1_000_003])
def test_fill_synthetic_bit_exact(dg, oracle, key, n):
    out = torch.empty(n, device="cuda", dtype=torch.float32)
    dg.fill_synthetic(out, *key)
    torch.cuda.synchronize()
    assert_bit_exact(out.cpu().numpy(), oracle.fill_f32(*key, n), "fill")


# --------------------------------------------------------------------------- semantic per-node API
def _rand(rng, n, scale=1.0):
    return (rng.standard_normal(n) * scale).astype(np.float32)


@pytest.mark.parametrize("offset", [0, 1])          # 1 => unaligned views => scalar path
@pytest.mark.parametrize("n", [1, 5, 1023, 65536 + 3])
def test_semantic_dadam_step_bit_exact(dg, oracle, n, offset):
    rng = np.random.default_rng(n + offset)
    dcfg, ocfg = cfgs(dg, oracle, 0)
    host = {k: _rand(rng, n + offset) for k in ("x", "g", "m", "mixed")}
    host["v"] = np.abs(_rand(rng, n + offset))
    dev = {k: torch.from_numpy(v.copy()).cuda()[offset:] for k, v in host.items()}
    ref = {k: v[offset:].copy() for k, v in host.items()}
    for t in (1, 2, 7):
        dg.dadam_step(dev["x"], dev["g"], dev["m"], dev["v"], dev["mixed"], dcfg, t)
        oracle.dadam_step(ref["x"], ref["g"], ref["m"], ref["v"], ref["mixed"], ocfg, t)
    dg.check_divergence()
    for k in ("x", "m", "v"):
        assert_bit_exact(dev[k].cpu().numpy(), ref[k], k)


@pytest.mark.parametrize("paper_literal", [False, True])
def test_semantic_accum_step_bit_exact(dg, oracle, paper_literal):
    n, T = 4099, 12
    rng = np.random.default_rng(11)
    dcfg, ocfg = cfgs(dg, oracle, 1, paper_literal)
    host = {k: _rand(rng, n) for k in ("x", "m", "b")}
    host["v"] = np.abs(_rand(rng, n))
    dev = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    ref = {k: v.copy() for k, v in host.items()}
    for t in range(1, T + 1):  # crosses three fold boundaries (t = 4, 8, 12)
        g = _rand(rng, n)
        mixed = _rand(rng, n)
        dg.accum_adam_step(dev["x"], torch.from_numpy(g).cuda(), dev["m"], dev["v"], dev["b"],
                           torch.from_numpy(mixed).cuda(), dcfg, t, T)
        oracle.accum_adam_step(ref["x"], g, ref["m"], ref["v"], ref["b"], mixed, ocfg, t, T)
        for k in ("x", "m", "v", "b"):
            assert_bit_exact(dev[k].cpu().numpy(), ref[k], f"{k}@t={t}")


@pytest.mark.parametrize("count", [1, 2, 6, 16, 17, 40])
def test_gossip_mix_bit_exact(dg, count):
    n = 10007
    rng = np.random.default_rng(count)
    xs = [_rand(rng, n) for _ in range(count)]
    w = rng.random(count)
    w /= w.sum()
    out = torch.empty(n, device="cuda")
    dg.gossip_mix(out, [torch.from_numpy(x).cuda() for x in xs], w)
    acc = np.zeros(n)
    for k in range(count):  # ascending order, fp64 accumulation, one rounding
        acc = acc + w[k] * xs[k].astype(np.float64)
    assert_bit_exact(out.cpu().numpy(), acc.astype(np.float32), "mix")


def test_semantic_step_errors(dg):
    z = torch.zeros(4, device="cuda")
    dcfg = dg.OptimizerConfig()
    with pytest.raises(dg.ConfigError):
        dg.dadam_step(z, z, z, z, z, dcfg, 0)
    with pytest.raises(dg.ConfigError):
        dg.accum_adam_step(z, z, z, z, z, z, dg.OptimizerConfig(s=4), 1, 6)   # T mod s
    with pytest.raises(dg.ConfigError):
        dg.dadam_step(z, z, z, z, torch.zeros(5, device="cuda"), dcfg, 1)     # length mismatch


def test_semantic_divergence(dg):
    x = torch.ones(64, device="cuda")
    g = torch.ones(64, device="cuda")
    g[17] = float("inf")
    m, v = torch.zeros(64, device="cuda"), torch.zeros(64, device="cuda")
    dg.dadam_step(x, g, m, v, x.clone(), dg.OptimizerConfig(), 5)
    with pytest.raises(dg.DivergenceError) as e:
        dg.check_divergence()
    assert e.value.iteration == 5
    dg.check_divergence()  # flag cleared


# --------------------------------------------------------------------------- fused engine
def run_engine(dg, sched, d, algo, dcfg, T, dispersed=True, t_stop=None, world=1, rank=0, device=0,
               nccl_id=None, chunk=0):
    eng = dg.Engine(sched, d, dcfg, algo=algo, total_steps=T, world_size=world, rank=rank, device=device,
                    nccl_id=nccl_id, chunk=chunk)
    if dispersed:
        eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
    else:
        eng.fill_synthetic(dg.X, SEED, dg.Stream.INIT_MODEL, False, 0)
    for t in range(1, (t_stop or T) + 1):
        eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)   # g_i^(t)
        eng.step(t)
    eng.sync()
    return eng


def engine_state(dg, eng, algo):
    keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo == 1 else [])
    return {k: np.stack([eng.download(i, w) for i in range(eng.local_nodes)]) for k, w in keys}


def oracle_state(oracle, osched, d, algo, ocfg, T, dtype, dispersed=True, t_stop=None):
    st = oracle.init_state(osched.workers, d, SEED, dispersed, dtype, algo)
    oracle.run(osched, algo, ocfg if dtype == np.float32 else ocfg.rounded_f32(), SEED, st, 1,
               t_stop or T, T)
    return st


@pytest.mark.parametrize("algo", [0, 1])
@pytest.mark.parametrize("d", [1 << 20, 1_000_003])
def test_engine_config1_ring8_100_steps(dg, oracle, algo, d):
    """BASELINE config 1: 8 simulated nodes, one-peer ring, 1M-param bucket, 100 steps."""
    T = 100
    dcfg, ocfg = cfgs(dg, oracle, algo)
    eng = run_engine(dg, dg.make_one_peer_ring(8), d, algo, dcfg, T)
    got = engine_state(dg, eng, algo)
    eng.close()
    osched = oracle.make_one_peer_ring(8)
    f32 = oracle_state(oracle, osched, d, algo, ocfg, T, np.float32)
    for k in got:
        assert_bit_exact(got[k], f32[k], k)
    f64 = oracle_state(oracle, osched, d, algo, ocfg, T, np.float64)
    worst = 0.0
    for k in ("x", "m", "v"):
        for i in range(8):
            e = normwise(got[k][i], f64[k][i])
            worst = max(worst, e)
            assert e <= 1e-6, (k, i, e)
    print(f"config1 algo={algo} d={d}: worst norm-wise rel err vs fp64 = {worst:.3e}")


def test_engine_accum_mid_group_t98(dg, oracle):
    # at T=100 with s=4 the accumulator is identically zero; t=98 checks b != 0 too
    dcfg, ocfg = cfgs(dg, oracle, 1)
    d = 1 << 16
    eng = run_engine(dg, dg.make_one_peer_ring(8), d, 1, dcfg, 100, t_stop=98)
    got = engine_state(dg, eng, 1)
    f32 = oracle_state(oracle, oracle.make_one_peer_ring(8), d, 1, ocfg, 100, np.float32, t_stop=98)
    assert got["b"].any()
    for k in got:
        assert_bit_exact(got[k], f32[k], k)
    f64 = oracle_state(oracle, oracle.make_one_peer_ring(8), d, 1, ocfg, 100, np.float64, t_stop=98)
    for i in range(8):
        assert normwise(got["b"][i], f64["b"][i]) <= 1e-6


TOPOS = [("make_one_peer_exponential", "ONE_PEER_EXP", (8,)),
         ("make_static_exponential", "STATIC_EXP", (8,)),
         ("make_aer", "AER", (8, 2)),
         ("make_aer", "AER", (16, 4)),          # 16 resident nodes, groups of 8
         ("make_complete", "COMPLETE", (8,)),
         ("make_one_peer_ring", "ONE_PEER_RING", (2,)),
         ("make_one_peer_exponential", "ONE_PEER_EXP", (16,)),
         ("make_static_exponential", "STATIC_EXP", (5,))]


@pytest.mark.parametrize("fn,kind,args", TOPOS)
@pytest.mark.parametrize("algo", [0, 1])
def test_engine_topologies_bit_exact(dg, oracle, fn, kind, args, algo):
    d, T = 4099, 24
    dcfg, ocfg = cfgs(dg, oracle, algo)
    eng = run_engine(dg, getattr(dg, fn)(*args), d, algo, dcfg, T, dispersed=(algo == 0))
    got = engine_state(dg, eng, algo)
    f32 = oracle_state(oracle, oracle.make(getattr(oracle, kind), *args), d, algo, ocfg, T, np.float32,
                       dispersed=(algo == 0))
    for k in got:
        assert_bit_exact(got[k], f32[k], k)


def test_engine_paper_literal(dg, oracle):
    dcfg, ocfg = cfgs(dg, oracle, 1, paper_literal=True)
    d, T = 1000, 16
    eng = run_engine(dg, dg.make_aer(8, 2), d, 1, dcfg, T)
    got = engine_state(dg, eng, 1)
    f32 = oracle_state(oracle, oracle.make_aer(8, 2), d, 1, ocfg, T, np.float32)
    for k in got:
        assert_bit_exact(got[k], f32[k], k)


def test_engine_divergence_reports_iteration(dg):
    d = 1024
    eng = dg.Engine(dg.make_one_peer_ring(8), d, dg.OptimizerConfig(), total_steps=10)
    eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
    for t in range(1, 6):
        eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
        if t == 3:
            bad = np.zeros(d, np.float32)
            bad[100] = np.nan
            eng.upload(5, dg.G, bad)
        eng.step(t)
    with pytest.raises(dg.DivergenceError) as e:
        eng.sync()
    assert e.value.iteration == 3


def test_engine_config_errors(dg):
    with pytest.raises(dg.ConfigError):
        dg.Engine(dg.make_one_peer_ring(8), 100, dg.OptimizerConfig(s=4), algo=dg.ACCUM, total_steps=6)
    eng = dg.Engine(dg.make_one_peer_ring(8), 100, dg.OptimizerConfig(), total_steps=10)
    with pytest.raises(dg.ConfigError):
        eng.step(0)
    with pytest.raises(dg.ConfigError):
        eng.download(8, dg.X)
    with pytest.raises(dg.ConfigError):
        dg.Engine(dg.make_one_peer_exponential(128), 100, dg.OptimizerConfig())  # > 64 nodes on one GPU


def test_engine_upload_download_roundtrip(dg):
    eng = dg.Engine(dg.make_one_peer_ring(4), 333, dg.OptimizerConfig())
    a = np.arange(333, dtype=np.float32)
    eng.upload(2, dg.M, a)
    assert np.array_equal(eng.download(2, dg.M), a)
    assert np.array_equal(eng.download(2, dg.M, 10, 5), a[10:15])
    st = eng.stats()
    assert st["local_nodes"] == 4 and st["first_node"] == 0 and st["d"] == 333

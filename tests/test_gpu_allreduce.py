"""All-Reduce Adam (Alg. 2),
the comparison baseline, on the engine vs the oracle (fp32 mirror bit-exact,
fp64 norm-wise), plus the SPEC examples and the consistency error."""
import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

SEED = 2410
CFG = dict(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, s=1)   # PAPER.md:1153 (All-Reduce baseline)


def run(dg, n, d, T, x0=None):
    eng = dg.Engine(dg.make_complete(n), d, dg.OptimizerConfig(**CFG), algo=dg.ALLREDUCE, total_steps=T)
    if x0 is None:
        eng.fill_synthetic(dg.X, SEED, dg.Stream.INIT_MODEL, False, 0)   # shared x^(0)
    else:
        for i in range(n):
            eng.upload(i, dg.X, x0[i])
    for t in range(1, T + 1):
        eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
        eng.step(t)
    return eng


@pytest.mark.parametrize("n,d", [(8, 100_003), (1, 4099), (16, 5000)])
def test_allreduce_adam_bit_exact(dg, oracle, n, d):
    T = 20
    eng = run(dg, n, d, T)
    eng.sync()
    got = {k: np.stack([eng.download(i, w) for i in range(n)]) for k, w in (("x", dg.X), ("m", dg.M), ("v", dg.V))}
    eng.close()
    s = oracle.make_complete(n)
    f32 = oracle.init_state(n, d, SEED, False, np.float32)
    oracle.run(s, oracle.ALLREDUCE, oracle.OptimizerConfig(**CFG), SEED, f32, 1, T)
    f64 = oracle.init_state(n, d, SEED, False, np.float64)
    oracle.run(s, oracle.ALLREDUCE, oracle.OptimizerConfig(**CFG).rounded_f32(), SEED, f64, 1, T)
    for k in got:
        assert np.array_equal(got[k].view(np.uint32), f32[k].view(np.uint32)), k
        assert np.all(got[k] == got[k][0])                      # all workers identical
        assert normwise(got[k][0], f64[k][0]) <= 1e-6, k


def test_allreduce_opposite_gradients(dg):
    # N=2, g1 = -g2 -> gbar = 0: from the zero state x is unchanged;
    # with nonzero moments m decays by beta1 (and v by beta2) exactly.
    d = 1000
    x = np.linspace(-1, 1, d, dtype=np.float32)
    g = np.linspace(-2, 3, d, dtype=np.float32)
    for m0, v0 in ((0.0, 0.0), (0.5, 1.0)):
        eng = dg.Engine(dg.make_complete(2), d, dg.OptimizerConfig(**CFG), algo=dg.ALLREDUCE)
        for i in range(2):
            eng.upload(i, dg.X, x)
            eng.upload(i, dg.M, np.full(d, m0, np.float32))
            eng.upload(i, dg.V, np.full(d, v0, np.float32))
        eng.upload(0, dg.G, g)
        eng.upload(1, dg.G, -g)
        eng.step(1)
        eng.sync()
        assert np.array_equal(eng.download(1, dg.M), np.full(d, np.float32(0.9) * np.float32(m0), np.float32))
        assert np.array_equal(eng.download(0, dg.V), np.full(d, np.float32(0.999) * np.float32(v0), np.float32))
        if m0 == 0.0:
            assert np.array_equal(eng.download(0, dg.X), x)
        eng.close()


def test_allreduce_diverged_workers_is_invariant_error(dg):
    d, n = 512, 4
    x0 = np.zeros((n, d), np.float32)
    x0[2, 7] = 1e-3
    eng = run(dg, n, d, 3, x0=x0)
    with pytest.raises(dg.InvariantError):
        eng.sync()

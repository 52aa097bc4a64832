"""on-device consensus error / gossip_consensus
(topology.hpp:90-100) against the fp64 oracle restatement."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

CASES = [("make_one_peer_exponential", "ONE_PEER_EXP", (8,), 3), ("make_one_peer_exponential", "ONE_PEER_EXP", (16,), 4),
         ("make_aer", "AER", (16, 4), 4), ("make_complete", "COMPLETE", (8,), 1),
         ("make_one_peer_ring", "ONE_PEER_RING", (8,), None), ("make_static_exponential", "STATIC_EXP", (8,), None),
         ("make_one_peer_ring", "ONE_PEER_RING", (4,), 2)]


@pytest.mark.parametrize("fn,kind,args,exact_at", CASES)
def test_gossip_consensus_matches_oracle(dg, oracle, fn, kind, args, exact_at):
    rng = np.random.default_rng(3)
    s = getattr(dg, fn)(*args)
    n, d, rounds = s.workers(), 10007, 12
    x0 = rng.standard_normal((n, d)).astype(np.float32)
    got = dg.gossip_consensus(s, x0, rounds)
    want = oracle.gossip_consensus(oracle.make(getattr(oracle, kind), *args), x0.astype(np.float64), rounds)
    assert got[0] == 1.0
    assert np.all(np.abs(got - want) <= 1e-5 + 1e-4 * want), (got, want)
    assert np.all(np.diff(got) <= 1e-7)                       # non-increasing
    if exact_at is not None:                                  # exact consensus
        # error[t] is measured against the preserved initial mean xbar^(0)
        # (topology.hpp:90-100).  At exact consensus every fp32 x_i equals the
        # fp32 rounding of xbar^(0), so the error is one rounding (<= 2^-24
        # relative per element, squared) rather than exactly 0: ~1e-16 here.
        assert got[exact_at] <= 1e-12, got[exact_at]
        assert want[exact_at] <= 1e-12, want[exact_at]


def test_gossip_consensus_zero_dispersion(dg):
    s = dg.make_one_peer_ring(8)
    x0 = np.tile(np.linspace(-1, 1, 257, dtype=np.float32), (8, 1))
    assert np.all(dg.gossip_consensus(s, x0, 5) == 0.0)


def test_engine_consensus_mean_preserved(dg, oracle):
    # mean preservation under the fused DAdam step with zero gradients
    s = dg.make_static_exponential(8)
    rng = np.random.default_rng(4)
    x0 = rng.standard_normal((8, 4099)).astype(np.float32)
    eng = dg.Engine(s, 4099, dg.OptimizerConfig())
    for i in range(8):
        eng.upload(i, dg.X, x0[i])
    _, m0 = eng.consensus()
    for t in range(1, 11):
        eng.step(t)
    disp, m1 = eng.consensus()
    eng.close()
    assert abs(m1 - m0) / m0 < 1e-6
    xbar = x0.astype(np.float64).mean(0)
    assert abs(m0 - float(xbar @ xbar)) / m0 < 1e-12

"""Topology / peer-schedule generator of libdg (host side, no GPU).

Follows the SPEC.md topology examples and acceptance criteria #1/#2
(SPEC.md:98-188, 571-572), and requires the product's closed-form peer tables
to be BIT-EXACT against the oracle's dense-matrix restatement for every round
(north_star: "peer schedules and neighbour indices bit-exact").
"""
import numpy as np
import pytest

BUILDERS = [
    ("make_complete", "COMPLETE", lambda n: (n,), [1, 2, 4, 5, 8, 16, 32]),
    ("make_one_peer_ring", "ONE_PEER_RING", lambda n: (n,), [2, 4, 8, 16, 32, 64]),
    ("make_one_peer_exponential", "ONE_PEER_EXP", lambda n: (n,), [2, 4, 8, 16, 32, 64]),
    ("make_static_exponential", "STATIC_EXP", lambda n: (n,), [2, 3, 4, 6, 8, 16, 32, 64]),
]
AER_CASES = [(2, 1), (4, 1), (8, 1), (8, 2), (8, 4), (16, 2), (16, 4), (32, 4), (64, 8), (64, 1), (12, 3)]


def _pairs(dg, oracle):
    for fn, kind, args, ns in BUILDERS:
        for n in ns:
            yield f"{fn}({n})", getattr(dg, fn)(*args(n)), oracle.make(getattr(oracle, kind), *args(n))
    for n, wpn in AER_CASES:
        yield f"make_aer({n},{wpn})", dg.make_aer(n, wpn), oracle.make(oracle.AER, n, wpn)


def test_schedules_bit_exact_vs_oracle(dg, oracle):
    for name, s, o in _pairs(dg, oracle):
        assert s.workers() == o.workers and s.period() == o.period, name
        assert s.workers_per_node() == o.workers_per_node and s.is_static() == o.is_static, name
        for r in range(1, 2 * s.period() + 2):  # two full periods: periodicity too
            assert np.array_equal(s.matrix_at(r), o.matrix_at(r)), (name, r)
            for (a, wa), (b, wb) in zip(s.neighbors_and_weights_at(r), o.neighbors_at(r)):
                assert a == b and np.array_equal(wa, wb), (name, r)


def test_every_round_valid(dg):
    # acceptance #1: every matrix of every topology at N in {2,4,8,16,32} passes to 1e-12
    for n in (2, 4, 8, 16, 32):
        scheds = [dg.make_complete(n), dg.make_one_peer_ring(n), dg.make_one_peer_exponential(n),
                  dg.make_static_exponential(n), dg.make_aer(n, 1)]
        if n >= 4:
            scheds.append(dg.make_aer(n, 2))
        for s in scheds:
            for r in range(1, s.period() + 1):
                w = s.matrix_at(r)
                v = dg.validate(w)
                assert v.passed(), (s.name(), n, r)
                assert np.abs(w - w.T).max() <= 1e-12
                assert np.abs(w.sum(0) - 1).max() <= 1e-12 and np.abs(w.sum(1) - 1).max() <= 1e-12


def test_neighbors_include_self_ascending(dg):
    s = dg.make_aer(16, 4)
    for r in range(1, s.period() + 1):
        for i, nb in enumerate(s.neighbors_at(r)):
            assert i in nb and nb == sorted(nb)


# ------------------------------------------------------------------ SPEC examples
def test_complete_examples(dg):
    assert np.all(dg.make_complete(4).matrix_at(1) == 0.25)
    assert dg.make_complete(1).matrix_at(1).tolist() == [[1.0]]
    assert abs(dg.spectral_lambda(dg.make_complete(4).matrix_at(1))) < 1e-12


def test_one_peer_ring_examples(dg):
    s = dg.make_one_peer_ring(4)
    blk = np.array([[.5, .5], [.5, .5]])
    want = np.block([[blk, np.zeros((2, 2))], [np.zeros((2, 2)), blk]])
    assert np.array_equal(s.matrix_at(1), want)
    prod = s.matrix_at(2) @ s.matrix_at(1)
    assert np.allclose(prod, 0.25, atol=1e-15)
    s2 = dg.make_one_peer_ring(2)
    assert np.array_equal(s2.matrix_at(1), blk) and np.array_equal(s2.matrix_at(2), blk)
    with pytest.raises(dg.ConfigError):
        dg.make_one_peer_ring(7)


def test_one_peer_exponential_examples(dg):
    s = dg.make_one_peer_exponential(16)
    assert s.neighbors_at(3)[0] == [0, 4]
    assert dg.effective_lambda(dg.make_one_peer_exponential(8)) < 1e-12
    assert np.array_equal(dg.make_one_peer_exponential(2).matrix_at(1), np.full((2, 2), .5))
    with pytest.raises(dg.ConfigError):
        dg.make_one_peer_exponential(12)


def test_aer_examples(dg):
    s = dg.make_aer(16, 4)
    nb = s.neighbors_at(1)
    assert nb[0] == list(range(4)) and nb[5] == list(range(4, 8)) and nb[9] == list(range(8, 16))
    prod = np.eye(16)
    for r in range(1, s.period() + 1):
        prod = s.matrix_at(r) @ prod
    assert np.allclose(prod, 1 / 16, atol=1e-14)
    g = dg.make_aer(8, 4)
    assert g.period() == 1 and np.allclose(g.matrix_at(1), 1 / 8)
    # Appendix B: AER(8, 2) rounds follow Fig. 9's merge order (2,3),(0,1),(0,2),(1,3)
    a = dg.make_aer(8, 2)
    assert a.neighbors_at(1)[4] == [4, 5, 6, 7] and a.neighbors_at(1)[0] == [0, 1]
    assert a.neighbors_at(2)[0] == [0, 1, 2, 3]
    assert a.neighbors_at(3)[0] == [0, 1, 4, 5]
    assert a.neighbors_at(4)[2] == [2, 3, 6, 7]
    with pytest.raises(dg.ConfigError):
        dg.make_aer(12, 2)  # M = 6 not a power of two


def test_static_exponential_n8(dg):
    s = dg.make_static_exponential(8)
    assert s.is_static() and s.neighbors_at(1)[0] == [0, 1, 2, 4, 6, 7]
    assert np.allclose(s.matrix_at(1)[0][[0, 1, 2, 4, 6, 7]], 1 / 6)
    assert abs(dg.spectral_lambda(s.matrix_at(1)) - 1 / 3) < 1e-12


def test_validate_examples(dg):
    assert dg.validate(np.full((4, 4), .25)).passed()
    # SPEC.md:134 says "not symmetric, columns != 1"; the columns of this matrix do
    # sum to 1 -- it is the ROWS (1.1, 0.9) that fail, which is what we assert.
    bad = dg.validate(np.array([[.6, .5], [.4, .5]]))
    assert not bad.passed() and not bad.symmetric and not bad.rows_stochastic and bad.cols_stochastic
    assert dg.validate(np.eye(3)).passed()
    assert abs(dg.spectral_lambda(np.eye(4)) - 1) < 1e-12
    m = np.kron(np.eye(2), np.full((2, 2), .5))
    assert abs(dg.spectral_lambda(m) - 1) < 1e-12
    with pytest.raises(dg.ConfigError):
        dg.spectral_lambda(np.array([[.6, .5], [.4, .5]]))


def test_lambda_vs_oracle(dg, oracle):
    for name, s, o in _pairs(dg, oracle):
        assert abs(dg.effective_lambda(s) - oracle.effective_lambda(o)) < 1e-9, name
        for r in range(1, s.period() + 1):
            w = s.matrix_at(r)
            assert abs(dg.spectral_lambda(w) - oracle.spectral_lambda(w)) < 1e-9, name
    ring8 = dg.effective_lambda(dg.make_one_peer_ring(8))
    assert 0 < ring8 < 1


def test_effective_lambda_permutation_invariant(dg):
    rng = np.random.default_rng(1)
    s = dg.make_one_peer_ring(8)
    p = rng.permutation(8)
    P = np.eye(8)[p]
    rounds = [P @ s.matrix_at(r) @ P.T for r in (1, 2)]
    s2 = dg.from_matrices("perm", 1, rounds)
    assert abs(dg.effective_lambda(s) - dg.effective_lambda(s2)) < 1e-12


def test_from_matrices_rejects(dg):
    with pytest.raises(dg.ConfigError):
        dg.from_matrices("asym", 1, [np.array([[.6, .5], [.4, .5]])])
    with pytest.raises(dg.ConfigError):  # disconnected union graph
        dg.from_matrices("eye", 1, [np.eye(4)])
    s = dg.from_matrices("ring", 1, [dg.make_one_peer_ring(6).matrix_at(r) for r in (1, 2)])
    assert s.period() == 2 and s.neighbors_at(2)[5] == [0, 5]


def test_round_zero_is_config_error(dg):
    s = dg.make_one_peer_ring(4)
    with pytest.raises(dg.ConfigError):
        s.matrix_at(0)


def test_gossip_consensus_oracle_properties(oracle):
    # SPEC.md:162-167 (oracle restatement of gossip_consensus): mean preservation,
    # non-increasing C(t), exact consensus after one period for one-peer exp / AER(16,4)
    rng = np.random.default_rng(2)
    for s, exact_at in ((oracle.make_one_peer_exponential(16), 4), (oracle.make_aer(16, 4), 4),
                        (oracle.make_complete(8), 1), (oracle.make_one_peer_ring(4), 2)):
        x0 = rng.standard_normal((s.workers, 64))
        err = oracle.gossip_consensus(s, x0, 8)
        assert err[0] == 1.0 and np.all(np.diff(err) <= 1e-15)
        assert err[exact_at] <= 1e-12
    s = oracle.make_one_peer_ring(8)
    assert np.all(oracle.gossip_consensus(s, np.ones((8, 4)), 3) == 0)


def test_schedule_names_and_describe(dg):
    # MixingSchedule::name() (topology.hpp:50) and MixingValidation::describe() (topology.hpp:33)
    assert dg.make_complete(4).name() == "complete"
    assert dg.make_one_peer_ring(8).name() == "one_peer_ring"
    assert dg.make_one_peer_exponential(8).name() == "one_peer_exponential"
    assert dg.make_aer(8, 2).name() == "aer"
    assert dg.make_static_exponential(8).name() == "static_exponential"
    s = dg.from_matrices("my ring", 1, [dg.make_one_peer_ring(4).matrix_at(1), dg.make_one_peer_ring(4).matrix_at(2)])
    assert s.name() == "my ring" and s.period() == 2
    v = dg.validate(dg.make_complete(4).matrix_at(1))
    assert v.passed() and v.describe().startswith("valid:")
    bad = dg.validate(np.array([[0.6, 0.5], [0.4, 0.5]]))
    assert not bad.passed()
    txt = bad.describe()
    assert txt.startswith("INVALID:") and "symmetric=NO" in txt and "rows_stochastic=NO" in txt


def test_consensus_trajectory_csv(dg, tmp_path):
    # trajectory export `round,consensus_error`; host-only part of f2
    tr = dg.ConsensusTrajectory([1.0, 0.25, 0.0])
    assert np.all(tr == np.array([1.0, 0.25, 0.0])) and tr.error.dtype == np.float64
    path = tmp_path / "c.csv"
    tr.to_csv(str(path))
    assert path.read_text().splitlines() == ["round,consensus_error", "0,1", "1,0.25", "2,0"]

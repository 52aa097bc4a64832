"""Pins the CPU oracle (oracle/oracle.cpp) before it is trusted as the checker.

* RNG: SURVEY.md Appendix C KATs and tests/golden/rng_kat.json, both produced by
  the reference's own rng.cpp.
* Step math: golden trajectories from the reference's vec.cpp primitives
  (tests/golden/ref_*.npz, see make_golden.py) must be reproduced BIT-EXACTLY by
  the fp64 restatement; the live reference build (oracle/_ref) is compared too
  when present.
* SPEC.md optimizer examples and acceptance criterion #3.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, normwise

SEED = 2410


# --------------------------------------------------------------------------- rng
def test_rng_appendix_c_kats(oracle):
    # SURVEY.md Appendix C (computed from the reference rng.cpp)
    kats = [((0, 1, 0, 0), 0xf19264ec81b77bd5, 0xa9d7508c3805069e, 0.77590505174671232),
            ((42, 4, 0, 0), 0x03790e927dd8fa64, 0x635761dd5eb8dfa9, 0.0013493599932684619),
            ((42, 2, 3, 7), 0x9a6f31e46f41b7c9, 0xd927c36340277f72, 0.51819688540888054),
            ((42, 6, 7, 0), 0x8619a129634821aa, 0x26d4fababf19a6fe, 0.27359325172711058)]
    for key, u0, u1, unit2 in kats:
        u = oracle.rng_u64(*key, 2)
        assert int(u[0]) == u0 and int(u[1]) == u1
        assert oracle.rng_unit(*key, 1, first=2)[0] == unit2


def test_rng_golden_vectors(oracle):
    with open(os.path.join(GOLDEN, "rng_kat.json")) as f:
        g = json.load(f)
    for s in g["streams"]:
        assert [int(x) for x in oracle.rng_u64(*s["key"], 8)] == s["u64"]
        assert [float(x).hex() for x in oracle.rng_unit(*s["key"], 8)] == s["unit"]


def test_rng_skip_ahead_matches_sequential(oracle):
    # draw k of a stream == k-th next_u64 (rng.cpp:35-38): skip-ahead is exact
    seq = oracle.rng_u64(7, 2, 3, 9, 1000)
    for first in (0, 1, 17, 999):
        assert oracle.rng_u64(7, 2, 3, 9, 1, first=first)[0] == seq[first]


def test_fill_f32_is_one_rounding(oracle):
    u = oracle.rng_unit(SEED, 2, 0, 1, 4096)
    want = (2.0 * u - 1.0).astype(np.float32)
    assert np.array_equal(oracle.fill_f32(SEED, 2, 0, 1, 4096), want)
    assert want.min() >= -1.0 and want.max() <= 1.0


def test_div_by_sqrt_plus_eps_golden(oracle):
    with open(os.path.join(GOLDEN, "rng_kat.json")) as f:
        g = json.load(f)["div_by_sqrt_plus_eps"]
    m, v = np.array(g["m"]), np.array(g["v"])
    want = [float.fromhex(h) for h in g["out"]]
    # vec.cpp:51-57: eps OUTSIDE the square root
    got = m / (np.sqrt(v) + g["eps"])
    assert got.tolist() == want


# --------------------------------------------------------------------------- golden trajectories
def _golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return json.loads(str(z["meta"])), z


GOLDEN_RUNS = ["ref_ring8_dadam", "ref_ring8_accum4", "ref_aer8_accum4", "ref_staticexp8_dadam",
               "ref_ring8_accum4_literal"]
KINDS = {"ring8": ("ONE_PEER_RING", 8, 1), "aer8": ("AER", 8, 2), "staticexp8": ("STATIC_EXP", 8, 1)}


def _sched_for(oracle, name):
    kind, n, wpn = KINDS[name.split("_")[1]]
    return oracle.make(getattr(oracle, kind), n, wpn)


@pytest.mark.parametrize("name", GOLDEN_RUNS)
def test_oracle_schedule_matches_golden_tables(oracle, name):
    meta, z = _golden(name)
    s = _sched_for(oracle, name)
    idx, w, cnt, _ = s.tables()
    assert np.array_equal(idx[:, :, :z["nbr_idx"].shape[2]], z["nbr_idx"])
    assert np.array_equal(w[:, :, :z["nbr_w"].shape[2]], z["nbr_w"])
    assert np.array_equal(cnt, z["nbr_cnt"])


@pytest.mark.parametrize("name", GOLDEN_RUNS)
def test_oracle_fp64_bit_exact_vs_reference_golden(oracle, name):
    meta, z = _golden(name)
    s = _sched_for(oracle, name)
    cfg = oracle.OptimizerConfig(meta["alpha"], meta["beta1"], meta["beta2"], meta["eps"], meta["s"],
                                 meta["paper_literal"])
    st = oracle.init_state(meta["n"], meta["d"], meta["seed"], meta["dispersed"], np.float64, meta["algo"])
    oracle.run(s, meta["algo"], cfg, meta["seed"], st, 1, meta["T"], meta["T"])
    for k in ("x", "m", "v") + (("b",) if meta["algo"] == oracle.ACCUM else ()):
        assert np.array_equal(st[k], z[k]), k


@pytest.mark.parametrize("name", GOLDEN_RUNS)
def test_fp32_mirror_normwise_vs_reference_golden(oracle, name):
    meta, z = _golden(name)
    s = _sched_for(oracle, name)
    cfg = oracle.OptimizerConfig(meta["alpha"], meta["beta1"], meta["beta2"], meta["eps"], meta["s"],
                                 meta["paper_literal"])
    st = oracle.init_state(meta["n"], meta["d"], meta["seed"], meta["dispersed"], np.float32, meta["algo"])
    oracle.run(s, meta["algo"], cfg, meta["seed"], st, 1, meta["T"], meta["T"])
    for k in ("x", "m", "v"):
        for i in range(meta["n"]):
            assert normwise(st[k][i], z[k][i]) <= 1e-6, (k, i)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                                    "libdeclab_ref.so")), reason="reference build absent")
@pytest.mark.parametrize("kind,n,wpn", [("ONE_PEER_RING", 8, 1), ("ONE_PEER_EXP", 16, 1), ("AER", 16, 4),
                                        ("STATIC_EXP", 8, 1), ("COMPLETE", 4, 1)])
@pytest.mark.parametrize("algo", [0, 1])
def test_oracle_fp64_bit_exact_vs_live_reference(oracle, kind, n, wpn, algo):
    s = oracle.make(getattr(oracle, kind), n, wpn)
    cfg = oracle.OptimizerConfig() if algo == 0 else oracle.OptimizerConfig(8e-4, 0.9, 0.999, 1e-8, 4)
    a = oracle.init_state(n, 333, SEED, True, np.float64, algo)
    b = {k: (None if v is None else v.copy()) for k, v in a.items()}
    oracle.run(s, algo, cfg, SEED, a, 1, 24, 24)
    oracle.ref_run(s, algo, cfg, SEED, b, 1, 24, 24)
    for k in a:
        if a[k] is not None:
            assert np.array_equal(a[k], b[k]), k


# --------------------------------------------------------------------------- SPEC examples (optim)
def test_dadam_first_step_is_minus_alpha_sign(oracle):
    # N=1, x0=1, g=2, alpha=0.1, eps=1e-8, t=1 -> x1 ~ 0.9
    cfg = oracle.OptimizerConfig(0.1, 0.9, 0.999, 1e-8)
    x, g, m, v = (np.array([1.0]), np.array([2.0]), np.zeros(1), np.zeros(1))
    mixed = x.copy()
    oracle.dadam_step(x, g, m, v, mixed, cfg, 1)
    assert abs(x[0] - 0.9) < 1e-8


def test_dadam_zero_grad_complete_averages(oracle):
    # zero gradients, 2 workers, complete W, x=(2,0) -> both 1
    s = oracle.make_complete(2)
    st = {"x": np.array([[2.0], [0.0]]), "m": np.zeros((2, 1)), "v": np.zeros((2, 1)), "b": None}
    # zero gradients: run the single-node step with explicit g = 0
    w = s.matrix_at(1)
    for i in range(2):
        mixed = np.array([w[i, 0] * 2.0 + w[i, 1] * 0.0])
        x = st["x"][i].copy()
        oracle.dadam_step(x, np.zeros(1), st["m"][i], st["v"][i], mixed, oracle.OptimizerConfig(), 1)
        assert x[0] == 1.0


def test_dadam_t0_is_config_error(oracle):
    x = np.zeros(1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.dadam_step(x, x.copy(), x.copy(), x.copy(), x.copy(), oracle.OptimizerConfig(), 0)
    assert e.value.code == oracle.CONFIG_ERROR


def test_dadam_n1_is_textbook_adam(oracle):
    # SPEC.md:313, acceptance #3(a): N=1 DAdam == textbook Adam (eps outside sqrt) to 1e-12, 100 steps
    rng = np.random.default_rng(0)
    cfg = oracle.OptimizerConfig(1e-2, 0.9, 0.999, 1e-8)
    x = rng.standard_normal(64)
    m = np.zeros(64); v = np.zeros(64)
    xa, ma, va = x.copy(), m.copy(), v.copy()
    for t in range(1, 101):
        g = rng.standard_normal(64)
        oracle.dadam_step(x, g, m, v, x.copy(), cfg, t)
        ma = 0.9 * ma + 0.1 * g
        va = 0.999 * va + 0.001 * g * g
        xa = xa - 1e-2 * (ma / (1 - 0.9 ** t)) / (np.sqrt(va / (1 - 0.999 ** t)) + 1e-8)
        assert np.max(np.abs(x - xa)) <= 1e-12


@pytest.mark.parametrize("seed", range(20))
def test_accum_s1_equals_dadam(oracle, seed):
    # SPEC.md:296,312, acceptance #3(b): AccumAdam(s=1) == DAdam state-for-state, 100 steps
    s = oracle.make_one_peer_ring(4)
    cfg = oracle.OptimizerConfig(2e-3, 0.9, 0.999, 1e-8, 1)
    a = oracle.init_state(4, 32, seed, True, np.float64, oracle.DADAM)
    b = oracle.init_state(4, 32, seed, True, np.float64, oracle.ACCUM)
    oracle.run(s, oracle.DADAM, cfg, seed, a, 1, 100)
    oracle.run(s, oracle.ACCUM, cfg, seed, b, 1, 100, 100)
    for k in ("x", "m", "v"):
        assert np.array_equal(a[k], b[k]), k
    assert not b["b"].any()


def test_accum_s2_hand_unroll(oracle):
    # constant g, s=2: m at t=2 is (1-b1) g, m_hat^(1) = (1-b1) g
    b1 = 0.9
    cfg = oracle.OptimizerConfig(1e-3, b1, 0.999, 1e-8, 2)
    g = np.array([0.5, -1.5])
    x, mh, vh, b = np.ones(2), np.zeros(2), np.zeros(2), np.zeros(2)
    oracle.accum_adam_step(x, g, mh, vh, b, x.copy(), cfg, 1, 2)
    assert not mh.any() and np.array_equal(b, g / 2)
    x_before = x.copy()
    oracle.accum_adam_step(x, g, mh, vh, b, x.copy(), cfg, 2, 2)
    m_t2 = (1 - b1) * g  # transient m at t=2 (m_hat^(0) = 0)
    c1 = 1 / (1 - b1)
    v_t2 = 0.001 * g * g
    want = x_before - 1e-3 * (c1 * m_t2) / (np.sqrt(v_t2 / (1 - 0.999)) + 1e-8)
    assert np.allclose(x, want, rtol=0, atol=1e-15)
    assert np.allclose(mh, (1 - b1) * g, rtol=1e-15) and not b.any()


def test_accum_momentum_identity(oracle):
    # SPEC.md:298 / PAPER.md:2167-2171: m^(t) = (1-b1)(g^(t) + b1 G^(t^-1) + ... + b1^(t^-1) G^(1))
    s_, b1 = 4, 0.9
    cfg = oracle.OptimizerConfig(1e-3, b1, 0.999, 1e-8, s_)
    rng = np.random.default_rng(3)
    gs = [rng.standard_normal(8) for _ in range(12)]
    x, mh, vh, b = np.zeros(8), np.zeros(8), np.zeros(8), np.zeros(8)
    for t in range(1, 13):
        that = math.ceil(t / s_)
        G = [np.mean(gs[(k - 1) * s_:k * s_], axis=0) for k in range(1, that)]
        want_m = (1 - b1) * (gs[t - 1] + sum(b1 ** (that - k) * G[k - 1] for k in range(1, that)))
        got_m = b1 * mh + (1 - b1) * gs[t - 1]  # m_t as Alg. 3 line 6 forms it from the state
        assert np.allclose(got_m, want_m, rtol=1e-12, atol=1e-14), t
        oracle.accum_adam_step(x, gs[t - 1], mh, vh, b, x.copy(), cfg, t, 12)


def test_accum_errors(oracle):
    z = np.zeros(1)
    cfg = oracle.OptimizerConfig(1e-3, 0.9, 0.999, 1e-8, 4)
    for t, T in ((1, 6), (9, 8), (0, 8)):  # T mod s != 0, t > T, t == 0
        with pytest.raises(oracle.OracleError) as e:
            oracle.accum_adam_step(z.copy(), z, z.copy(), z.copy(), z.copy(), z, cfg, t, T)
        assert e.value.code == oracle.CONFIG_ERROR


def test_divergence_error_names_iteration(oracle):
    s = oracle.make_one_peer_ring(2)
    st = oracle.init_state(2, 8, SEED, True, np.float64)
    st["x"][1, 3] = np.inf
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(s, oracle.DADAM, oracle.OptimizerConfig(), SEED, st, 1, 5)
    assert e.value.code == oracle.DIVERGENCE and e.value.iteration == 1


def test_cta_contract(oracle):
    # the step depends on neighbours only through x^(t-1): corrupting a
    # neighbour's iteration-t state after mixing does not change node 0's result.
    cfg = oracle.OptimizerConfig()
    rng = np.random.default_rng(5)
    xs = rng.standard_normal((2, 16))
    mixed = 0.5 * xs[0] + 0.5 * xs[1]
    g = rng.standard_normal(16)
    outs = []
    for corrupt in (False, True):
        x0, m0, v0 = xs[0].copy(), np.zeros(16), np.zeros(16)
        if corrupt:
            xs_t = xs.copy()
            xs_t[1] = np.nan  # neighbour's iteration-t state, after mixing was formed
        oracle.dadam_step(x0, g, m0, v0, mixed, cfg, 1)
        outs.append(x0)
    assert np.array_equal(outs[0], outs[1])


def test_fp32_mirror_normwise_vs_fp64_config1_small(oracle):
    # fp32 mirror within 1e-6 norm-wise of fp64 fed fp32-rounded hyperparameters
    s = oracle.make_one_peer_ring(8)
    for algo, cfg in ((0, oracle.OptimizerConfig()), (1, oracle.OptimizerConfig(8e-4, 0.9, 0.999, 1e-8, 4))):
        a = oracle.init_state(8, 4096, SEED, True, np.float32, algo)
        b = oracle.init_state(8, 4096, SEED, True, np.float64, algo)
        oracle.run(s, algo, cfg, SEED, a, 1, 100, 100)
        oracle.run(s, algo, cfg.rounded_f32(), SEED, b, 1, 100, 100)
        for k in ("x", "m", "v"):
            for i in range(8):
                assert normwise(a[k][i], b[k][i]) <= 1e-6, (algo, k, i)

"""ctypes view of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
reference legs, always as the checker (or the timed CPU baseline), never as
the product path.  Two libraries:

* ``liboracle.so``              -- our restatement (oracle/oracle.cpp)
* ``_ref/libdeclab_ref.so``     -- the reference's own vec.cpp + rng.cpp
                                   (compiled from /root/reference) + ref_shim.cpp
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OK, CONFIG_ERROR, DIVERGENCE, INVARIANT = 0, 2, 3, 4
COMPLETE, ONE_PEER_RING, ONE_PEER_EXP, AER, STATIC_EXP = range(5)
DADAM, ACCUM, ALLREDUCE = 0, 1, 2
# rng.hpp:9-16
DATASET, MINIBATCH, SPEED_NOISE, INIT_MODEL, TAU_SAMPLE, CONSENSUS_INIT = 1, 2, 3, 4, 5, 6

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code, msg, iteration=None):
        super().__init__(f"[{code}] {msg}")
        self.code, self.iteration = code, iteration


class AdamCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("s", C.c_int), ("paper_literal", C.c_int)]


class Validation(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("symmetric", "nonnegative", "rows_stochastic",
                                       "cols_stochastic", "eigenvalues_in_range")] + \
               [(k, C.c_double) for k in ("max_asymmetry", "min_entry", "max_row_error",
                                          "max_col_error", "min_eigenvalue", "max_eigenvalue")]

    def passed(self):
        return bool(self.symmetric and self.nonnegative and self.rows_stochastic
                    and self.cols_stochastic and self.eigenvalues_in_range)


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        L = _load(os.path.join(HERE, "liboracle.so"))
        L.or_last_error.restype = C.c_char_p
        L.or_last_divergence_iteration.restype = C.c_long
        L.or_rng_u64.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _u64p]
        L.or_rng_unit.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_size_t, _dp]
        L.or_fill_f32.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_size_t, _fp]
        L.or_make.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.or_from_matrices.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.or_free.argtypes = [C.c_void_p]
        L.or_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4
        L.or_matrix.argtypes = [C.c_void_p, C.c_long, _dp]
        L.or_neighbors.argtypes = [C.c_void_p, C.c_long, C.c_int, np.ctypeslib.ndpointer(np.int32),
                                   _dp, C.c_int, C.POINTER(C.c_int)]
        L.or_validate.argtypes = [_dp, C.c_int, C.POINTER(Validation)]
        L.or_spectral_lambda.argtypes = [_dp, C.c_int, C.POINTER(C.c_double)]
        L.or_effective_lambda.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.or_gossip_consensus.argtypes = [C.c_void_p, _dp, C.c_int, C.c_size_t, C.c_int, C.c_int, _dp]
        for nm, p in (("f64", _dp), ("f32", _fp)):
            getattr(L, f"or_dadam_step_{nm}").argtypes = [p, p, p, p, p, C.c_size_t, C.POINTER(AdamCfg), C.c_long]
            getattr(L, f"or_accum_adam_step_{nm}").argtypes = [p, p, p, p, p, p, C.c_size_t,
                                                               C.POINTER(AdamCfg), C.c_long, C.c_long]
            getattr(L, f"or_run_{nm}").argtypes = [C.c_void_p, C.c_int, C.POINTER(AdamCfg), C.c_uint64,
                                                   C.c_size_t, C.c_long, C.c_long, C.c_long, C.c_int,
                                                   p, p, p, C.c_void_p]
        for nm, p in (("f64", _dp), ("f32", _fp)):
            getattr(L, f"or_run_cols_{nm}").argtypes = [C.c_void_p, C.c_int, C.POINTER(AdamCfg), C.c_uint64, _u64p,
                                                        C.c_size_t, C.c_int, C.c_long, C.c_long, C.c_long,
                                                        C.c_int, p, p, p, C.c_void_p]
        L.or_step_all_f64.argtypes = [C.c_void_p, C.c_int, C.POINTER(AdamCfg), C.c_size_t, C.c_long,
                                      C.c_long, C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_void_p]
        L.or_step_all_f32.argtypes = [C.c_void_p, C.c_int, C.POINTER(AdamCfg), C.c_size_t, C.c_long,
                                      C.c_long, C.c_int, _fp, _fp, _fp, _fp, _fp, C.c_void_p]
        _lib = L
    return _lib


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libdeclab_ref.so"))


def ref():
    global _ref
    if _ref is None:
        R = _load(os.path.join(HERE, "_ref", "libdeclab_ref.so"))
        R.ref_last_error.restype = C.c_char_p
        R.ref_rng_u64.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_size_t, _u64p]
        R.ref_rng_unit.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_size_t, _dp]
        R.ref_speed_multiplier.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int]
        R.ref_speed_multiplier.restype = C.c_double
        R.ref_div_by_sqrt_plus_eps.argtypes = [_dp, _dp, C.c_size_t, C.c_double, _dp]
        R.ref_run.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_int, C.c_int,
                              np.ctypeslib.ndpointer(np.int32), _dp, np.ctypeslib.ndpointer(np.int32),
                              C.POINTER(AdamCfg), C.c_uint64, C.c_long, C.c_long, C.c_long, C.c_int,
                              C.c_int, C.c_void_p, _dp, _dp, _dp, C.c_void_p, C.POINTER(C.c_double)]
        _ref = R
    return _ref


def _check(rc):
    if rc != OK:
        L = lib()
        it = L.or_last_divergence_iteration() if rc == DIVERGENCE else None
        raise OracleError(rc, L.or_last_error().decode(), it)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ rng
def rng_u64(seed, purpose, worker, iteration, n, first=0):
    out = np.empty(n, np.uint64)
    lib().or_rng_u64(seed, purpose, worker, iteration, first, n, out)
    return out


def rng_unit(seed, purpose, worker, iteration, n, first=0):
    out = np.empty(n, np.float64)
    lib().or_rng_unit(seed, purpose, worker, iteration, first, n, out)
    return out


def fill_f32(seed, purpose, worker, iteration, n):
    out = np.empty(n, np.float32)
    lib().or_fill_f32(seed, purpose, worker, iteration, n, out)
    return out


# ------------------------------------------------------------------ topology
class Schedule:
    """Oracle MixingSchedule (topology.hpp:40-63)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        w, p, k, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().or_info(self._h, C.byref(w), C.byref(p), C.byref(k), C.byref(s)))
        self.workers, self.period, self.workers_per_node, self.is_static = w.value, p.value, k.value, bool(s.value)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            try:
                lib().or_free(self._h)
            except Exception:
                pass

    @property
    def handle(self):
        return self._h

    def matrix_at(self, rnd):
        w = np.empty((self.workers, self.workers), np.float64)
        _check(lib().or_matrix(self._h, rnd, w))
        return w

    def neighbors_at(self, rnd):
        out = []
        for i in range(self.workers):
            idx = np.empty(self.workers, np.int32)
            w = np.empty(self.workers, np.float64)
            cnt = C.c_int()
            _check(lib().or_neighbors(self._h, rnd, i, idx, w, self.workers, C.byref(cnt)))
            out.append((idx[:cnt.value].tolist(), w[:cnt.value].copy()))
        return out

    def tables(self):
        """period x n x maxdeg neighbour index / weight tables + counts (for ref_run)."""
        n, P = self.workers, self.period
        rows = [self.neighbors_at(r + 1) for r in range(P)]
        maxdeg = max(len(ix) for rr in rows for ix, _ in rr)
        idx = np.zeros((P, n, maxdeg), np.int32)
        w = np.zeros((P, n, maxdeg), np.float64)
        cnt = np.zeros((P, n), np.int32)
        for r in range(P):
            for i, (ix, ww) in enumerate(rows[r]):
                idx[r, i, :len(ix)] = ix
                w[r, i, :len(ix)] = ww
                cnt[r, i] = len(ix)
        return idx, w, cnt, maxdeg


def make(kind, n, wpn=1):
    h = C.c_void_p()
    _check(lib().or_make(kind, n, wpn, C.byref(h)))
    return Schedule(h.value)


def make_complete(n):
    return make(COMPLETE, n)


def make_one_peer_ring(n):
    return make(ONE_PEER_RING, n)


def make_one_peer_exponential(n):
    return make(ONE_PEER_EXP, n)


def make_aer(n, workers_per_node):
    return make(AER, n, workers_per_node)


def make_static_exponential(n):
    return make(STATIC_EXP, n)


def from_matrices(mats, workers_per_node=1):
    mats = np.ascontiguousarray(mats, np.float64)
    P, n, _ = mats.shape
    h = C.c_void_p()
    _check(lib().or_from_matrices(mats.reshape(-1), n, P, workers_per_node, C.byref(h)))
    return Schedule(h.value)


def validate(w):
    w = np.ascontiguousarray(w, np.float64)
    out = Validation()
    _check(lib().or_validate(w.reshape(-1), w.shape[0], C.byref(out)))
    return out


def spectral_lambda(w):
    w = np.ascontiguousarray(w, np.float64)
    out = C.c_double()
    _check(lib().or_spectral_lambda(w.reshape(-1), w.shape[0], C.byref(out)))
    return out.value


def effective_lambda(s):
    out = C.c_double()
    _check(lib().or_effective_lambda(s.handle, C.byref(out)))
    return out.value


def gossip_consensus(s, x0, rounds, threads=0):
    x0 = np.ascontiguousarray(x0, np.float64)
    err = np.empty(rounds + 1, np.float64)
    _check(lib().or_gossip_consensus(s.handle, x0.reshape(-1), x0.shape[0], x0.shape[1], rounds, threads, err))
    return err


# ------------------------------------------------------------------ optim
@dataclass
class OptimizerConfig:
    """OptimizerConfig."""
    alpha: float = 2e-3
    beta1: float = 0.974
    beta2: float = 0.999
    eps: float = 1e-8
    s: int = 1
    paper_literal: bool = False

    def c(self):
        return AdamCfg(self.alpha, self.beta1, self.beta2, self.eps, self.s, int(self.paper_literal))

    def rounded_f32(self):
        """Hyperparameters rounded through fp32."""
        f = lambda v: float(np.float32(v))
        return OptimizerConfig(f(self.alpha), f(self.beta1), f(self.beta2), f(self.eps), self.s, self.paper_literal)


def dadam_step(x, g, m, v, mixed, cfg, t):
    """In-place single-worker DAdam step; dtype picks fp64 / fp32 mirror."""
    fn = lib().or_dadam_step_f64 if x.dtype == np.float64 else lib().or_dadam_step_f32
    c = cfg.c()
    _check(fn(x, g, m, v, mixed, x.size, C.byref(c), t))


def accum_adam_step(x, g, m_hat, v_hat, b, mixed, cfg, t, T):
    """In-place single-worker AccumAdam step."""
    fn = lib().or_accum_adam_step_f64 if x.dtype == np.float64 else lib().or_accum_adam_step_f32
    c = cfg.c()
    _check(fn(x, g, m_hat, v_hat, b, mixed, x.size, C.byref(c), t, T))


def init_state(n, d, seed, dispersed, dtype=np.float32, algo=DADAM):
    """x^(0): shared InitModel stream (Alg. 1 line 1) or per-node ConsensusInit stream."""
    x = np.empty((n, d), np.float32)
    for i in range(n):
        x[i] = fill_f32(seed, CONSENSUS_INIT, i, 0, d) if dispersed else fill_f32(seed, INIT_MODEL, 0, 0, d)
    x = x.astype(dtype)
    z = lambda: np.zeros((n, d), dtype)
    return {"x": x, "m": z(), "v": z(), "b": z() if algo == ACCUM else None}


def run(s, algo, cfg, seed, state, t_begin, t_end, T=0, threads=0):
    """Run steps t_begin..t_end for all nodes in place (fp64 or fp32 per state dtype)."""
    x = state["x"]
    n, d = x.shape
    assert n == s.workers
    fn = lib().or_run_f64 if x.dtype == np.float64 else lib().or_run_f32
    c = cfg.c()
    _check(fn(s.handle, algo, C.byref(c), seed, d, t_begin, t_end, T, threads,
              x.reshape(-1), state["m"].reshape(-1), state["v"].reshape(-1), _ptr(state["b"])))
    return state


def run_fixed_g(s, algo, cfg, state, g, t_begin, t_end, T=0, threads=0):
    """fp32 mirror (or fp64) steps t_begin..t_end with the gradient g (n x d) held fixed."""
    x = state["x"]
    n, d = x.shape
    xprev = np.empty_like(x)
    f64 = x.dtype == np.float64
    fn = lib().or_step_all_f64 if f64 else lib().or_step_all_f32
    g = np.ascontiguousarray(g, x.dtype)
    c = cfg.c()
    for t in range(t_begin, t_end + 1):
        _check(fn(s.handle, algo, C.byref(c), d, t, T, threads, g.reshape(-1), x.reshape(-1), xprev.reshape(-1),
                  state["m"].reshape(-1), state["v"].reshape(-1), _ptr(state["b"])))
    return state


def ref_run(s, algo, cfg, seed, state, t_begin, t_end, T=0, threads=0, g_fixed=None):
    """Reference CPU path (vec.cpp primitives + parallel_for), fp64; returns step-loop seconds."""
    R = ref()
    idx, w, cnt, maxdeg = s.tables()
    x = state["x"]
    n, d = x.shape
    c = cfg.c()
    el = C.c_double()
    rc = R.ref_run(algo, n, d, s.period, maxdeg, idx.reshape(-1), w.reshape(-1), cnt.reshape(-1),
                   C.byref(c), seed, t_begin, t_end, T, threads, int(g_fixed is None), _ptr(g_fixed),
                   x.reshape(-1), state["m"].reshape(-1), state["v"].reshape(-1), _ptr(state["b"]),
                   C.byref(el))
    if rc != OK:
        raise OracleError(rc, R.ref_last_error().decode())
    return el.value


def run_cols(s, algo, cfg, seed, cols, dispersed, t_begin, t_end, T=0, dtype=np.float32, threads=0):
    """Replay the columns `cols` of a full-size bucket (oracle.h or_run_cols_*).
    Returns {"x","m","v"[,"b"]} arrays of shape (workers, len(cols))."""
    cols = np.ascontiguousarray(cols, np.uint64)
    n, nc = s.workers, cols.size
    st = {k: np.zeros((n, nc), dtype) for k in ("x", "m", "v")}
    st["b"] = np.zeros((n, nc), dtype) if algo == ACCUM else None
    fn = lib().or_run_cols_f32 if dtype == np.float32 else lib().or_run_cols_f64
    c = cfg.c()
    _check(fn(s.handle, algo, C.byref(c), seed, cols, nc, int(dispersed), t_begin, t_end, T, threads,
              st["x"].reshape(-1), st["m"].reshape(-1), st["v"].reshape(-1), _ptr(st["b"])))
    return st

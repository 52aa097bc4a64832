"""B200-native decentralized gossip + Adam step (arXiv 2410.11998), Python view.

A thin ctypes mirror of the reference's operator API (namespace ``declab``:
``MixingSchedule``, ``make_*``, ``validate``, ``spectral_lambda``,
``effective_lambda``, ``OptimizerConfig``, ``dadam_step``, ``accum_adam_step``)
over the C ABI in ``include/dg.h`` (``libdg.so``, sm_100a CUDA + NCCL).  Same
names, same argument meaning and the same error taxonomy (errors.hpp:8-26):
``ConfigError`` / ``DivergenceError(iteration)`` / ``InvariantError``.

There is no CPU fallback: every compute call goes to libdg.so and fails loudly
when the library or a GPU is missing.  PyTorch is used only as plumbing
(device tensors and streams) for the per-node semantic step.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "DGError", "ConfigError", "DivergenceError", "InvariantError", "CudaError", "NcclError",
    "MixingSchedule", "MixingValidation", "make_complete", "make_one_peer_ring",
    "make_one_peer_exponential", "make_aer", "make_static_exponential", "from_matrices",
    "validate", "spectral_lambda", "effective_lambda", "OptimizerConfig", "gossip_mix",
    "dadam_step", "accum_adam_step", "check_divergence", "fill_synthetic", "Engine",
    "nccl_unique_id", "plan_exchange", "library_path", "DADAM", "ACCUM", "ALLREDUCE", "gossip_consensus",
    "ConsensusTrajectory",
    "TRANSPORT_AUTO", "TRANSPORT_NCCL", "TRANSPORT_P2P",
    "X", "G", "M", "V", "ACC", "Stream",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# DG_LIB overrides the library path (kernel-variant sweeps, scripts/sweep.py).
_LIB_PATH = os.environ.get("DG_LIB") or os.path.join(HERE, "libdg.so")

DADAM, ACCUM, ALLREDUCE = 0, 1, 2
TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_P2P = 0, 1, 2
ENGINE_IN_PLACE = 1
RUN_GRAPH, RUN_CAPTURE_ONLY = 1, 2
X, G, M, V, ACC = 0, 1, 2, 3, 4


class Stream:
    """StreamRng purposes (rng.hpp:9-16)."""
    DATASET, MINIBATCH, SPEED_NOISE, INIT_MODEL, TAU_SAMPLE, CONSENSUS_INIT = 1, 2, 3, 4, 5, 6


# ----------------------------------------------------------------------------- errors
class DGError(RuntimeError):
    code = 1

    def __init__(self, msg, iteration=None):
        super().__init__(msg)
        self.iteration = iteration


class ConfigError(DGError, ValueError):       # errors.hpp:10-12 (exit 2)
    code = 2


class DivergenceError(DGError):               # errors.hpp:16-20 (exit 3)
    code = 3


class InvariantError(DGError):                # errors.hpp:24-26 (exit 4)
    code = 4


class CudaError(DGError):
    code = 5


class NcclError(DGError):
    code = 6


_ERRORS = {2: ConfigError, 3: DivergenceError, 4: InvariantError, 5: CudaError, 6: NcclError}


# ----------------------------------------------------------------------------- ctypes
class _AdamCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("s", C.c_int), ("paper_literal", C.c_int)]


class _Validation(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("symmetric", "nonnegative", "rows_stochastic",
                                       "cols_stochastic", "eigenvalues_in_range")] + \
               [(k, C.c_double) for k in ("max_asymmetry", "min_entry", "max_row_error",
                                          "max_col_error", "min_eigenvalue", "max_eigenvalue")]


class _EngineConfig(C.Structure):
    _fields_ = [("schedule", C.c_void_p), ("world_size", C.c_int), ("rank", C.c_int),
                ("device", C.c_int), ("nccl_id", C.c_void_p), ("d", C.c_size_t),
                ("chunk", C.c_size_t), ("algo", C.c_int), ("adam", _AdamCfg),
                ("total_steps", C.c_long), ("transport", C.c_int), ("flags", C.c_int)]


class _RmParams(C.Structure):
    _fields_ = [("N", C.c_int), ("b", C.c_int), ("theta", C.c_double), ("gamma", C.c_double),
                ("omega", C.c_double), ("sigma2", C.c_double), ("workers_per_node", C.c_int),
                ("normalized", C.c_int), ("allow_omega_above_one", C.c_int)]


class _EngineStats(C.Structure):
    _fields_ = [("local_nodes", C.c_int), ("first_node", C.c_int), ("nodes", C.c_int),
                ("world_size", C.c_int), ("rank", C.c_int), ("d", C.c_size_t),
                ("chunk", C.c_size_t), ("kernel_launches", C.c_long), ("steps", C.c_long),
                ("bytes_sent", C.c_double), ("bytes_received", C.c_double),
                ("hbm_bytes", C.c_double), ("nccl_version", C.c_long), ("kernel_ms", C.c_double),
                ("timed_launches", C.c_long), ("timed_hbm_bytes", C.c_double), ("transport", C.c_int),
                ("barriers", C.c_long), ("remote_kernel_ms", C.c_double), ("remote_bytes", C.c_double)]


_lib = None

# Exported symbols and their ctypes signatures (also the ABI-completeness list
# checked by tests/test_abi.py against include/dg.h).
_VP, _I, _L, _SZ, _D = C.c_void_p, C.c_int, C.c_long, C.c_size_t, C.c_double
_IP, _DP, _FP = C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float)
SIGNATURES = {
    "dg_last_error": ([], C.c_char_p),
    "dg_last_divergence_iteration": ([], _L),
    "dg_version": ([], _I),
    "dg_make_complete": ([_I, C.POINTER(_VP)], _I),
    "dg_make_one_peer_ring": ([_I, C.POINTER(_VP)], _I),
    "dg_make_one_peer_exponential": ([_I, C.POINTER(_VP)], _I),
    "dg_make_aer": ([_I, _I, C.POINTER(_VP)], _I),
    "dg_make_static_exponential": ([_I, C.POINTER(_VP)], _I),
    "dg_schedule_from_matrices": ([_DP, _I, _I, _I, C.POINTER(_VP)], _I),
    "dg_schedule_from_matrices_named": ([C.c_char_p, _DP, _I, _I, _I, C.POINTER(_VP)], _I),
    "dg_schedule_name": ([_VP, C.c_char_p, _SZ, C.POINTER(_SZ)], _I),
    "dg_validation_pass": ([C.POINTER(_Validation)], _I),
    "dg_validation_describe": ([C.POINTER(_Validation), C.c_char_p, _SZ, C.POINTER(_SZ)], _I),
    "dg_schedule_info": ([_VP, _IP, _IP, _IP, _IP], _I),
    "dg_schedule_neighbors": ([_VP, _L, _I, _IP, _DP, _I, _IP], _I),
    "dg_schedule_matrix": ([_VP, _L, _DP], _I),
    "dg_schedule_free": ([_VP], None),
    "dg_validate": ([_DP, _I, C.POINTER(_Validation)], _I),
    "dg_spectral_lambda": ([_DP, _I, _DP], _I),
    "dg_effective_lambda": ([_VP, _DP], _I),
    "dg_gossip_mix_f32": ([_VP, C.POINTER(_VP), _DP, _I, _SZ, _VP], _I),
    "dg_dadam_step_f32": ([_VP, _VP, _VP, _VP, _VP, _SZ, C.POINTER(_AdamCfg), _L, _VP], _I),
    "dg_accum_adam_step_f32": ([_VP, _VP, _VP, _VP, _VP, _VP, _SZ, C.POINTER(_AdamCfg), _L, _L, _VP], _I),
    "dg_step_check_divergence": ([_VP], _I),
    "dg_fill_synthetic_f32": ([_VP, _SZ, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, _VP], _I),
    "dg_nccl_unique_id": ([_VP], _I),
    "dg_engine_create": ([C.POINTER(_EngineConfig), C.POINTER(_VP)], _I),
    "dg_engine_buffer": ([_VP, _I, _I, C.POINTER(_VP)], _I),
    "dg_engine_upload": ([_VP, _I, _I, _VP, _SZ, _SZ], _I),
    "dg_engine_download": ([_VP, _I, _I, _VP, _SZ, _SZ], _I),
    "dg_engine_fill_synthetic": ([_VP, _I, C.c_uint64, C.c_uint32, _I, C.c_uint64], _I),
    "dg_engine_gather": ([_VP, _I, _I, _VP, _SZ, _VP], _I),
    "dg_engine_consensus": ([_VP, _DP, _DP], _I),
    "dg_engine_consensus_fix_mean": ([_VP], _I),
    "dg_engine_step": ([_VP, _L], _I),
    "dg_engine_run_steps": ([_VP, _L, _L, _I], _I),
    "dg_engine_sync": ([_VP], _I),
    "dg_engine_streams": ([_VP, C.POINTER(_VP), C.POINTER(_VP)], _I),
    "dg_engine_get_stats": ([_VP, C.POINTER(_EngineStats)], _I),
    "dg_engine_destroy": ([_VP], None),
    "dg_engine_set_timing": ([_VP, _I], _I),
    "dg_engine_step_range": ([_VP, _L, _SZ, _SZ], _I),
    "dg_engine_wait_stream": ([_VP, _VP], _I),
    "dg_engine_join": ([_VP, _VP], _I),
    "dg_plan_exchange": ([_VP, _I, _I, _L, _IP, _IP, _IP, _IP, _IP, _IP, _I], _I),
    "dg_rm_simulate": ([_I, C.POINTER(_RmParams), _VP, _L, C.c_uint64, _DP, _DP], _I),
    "dg_rm_closed_form_speedup": ([_D, _I, _I, _D, _DP], _I),
    "dg_rm_speed_multiplier": ([C.c_uint64, C.c_uint64, C.c_uint64, _D, _DP], _I),
}


def library_path():
    return _LIB_PATH


def lib():
    """Load libdg.so (built in-tree by __graft_entry__.build()); no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback for the gossip step)")
        L = C.CDLL(_LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes, fn.restype = args, res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        L = lib()
        msg = L.dg_last_error().decode()
        cls = _ERRORS.get(rc, DGError)
        it = L.dg_last_divergence_iteration() if rc == 3 else None
        raise cls(msg, it)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


# ----------------------------------------------------------------------------- topology
@dataclass
class MixingValidation:
    """MixingValidation (topology.hpp:16-34)."""
    symmetric: bool
    nonnegative: bool
    rows_stochastic: bool
    cols_stochastic: bool
    eigenvalues_in_range: bool
    max_asymmetry: float
    min_entry: float
    max_row_error: float
    max_col_error: float
    min_eigenvalue: float
    max_eigenvalue: float

    def _c(self):
        return _Validation(*(int(getattr(self, f)) if i < 5 else float(getattr(self, f))
                             for i, (f, _) in enumerate(_Validation._fields_)))

    def passed(self) -> bool:  # MixingValidation::pass() (topology.hpp:29-32)
        c = self._c()
        return bool(lib().dg_validation_pass(C.byref(c)))

    def describe(self) -> str:  # MixingValidation::describe() (topology.hpp:33)
        c = self._c()
        buf = C.create_string_buffer(512)
        n = C.c_size_t()
        _check(lib().dg_validation_describe(C.byref(c), buf, len(buf), C.byref(n)))
        return buf.value.decode()


class MixingSchedule:
    """Immutable periodic mixing schedule (topology.hpp:40-63); 1-based rounds."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        n = C.c_size_t()
        _check(lib().dg_schedule_name(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().dg_schedule_name(self._h, buf, len(buf), C.byref(n)))
        self._name = buf.value.decode()
        w, p, k, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().dg_schedule_info(self._h, C.byref(w), C.byref(p), C.byref(k), C.byref(s)))
        self._workers, self._period, self._wpn, self._static = w.value, p.value, k.value, bool(s.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.dg_schedule_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def workers(self) -> int:
        return self._workers

    def period(self) -> int:
        return self._period

    def workers_per_node(self) -> int:
        return self._wpn

    def name(self) -> str:  # topology.hpp:50 (dg_schedule_name)
        return self._name

    def is_static(self) -> bool:
        return self._static

    def matrix_at(self, rnd: int) -> np.ndarray:
        n = self._workers
        w = np.empty((n, n), np.float64)
        _check(lib().dg_schedule_matrix(self._h, rnd, _dptr(w)))
        return w

    def neighbors_at(self, rnd: int) -> List[List[int]]:
        return [ix for ix, _ in self.neighbors_and_weights_at(rnd)]

    def neighbors_and_weights_at(self, rnd: int):
        out = []
        n = self._workers
        idx = (C.c_int * n)()
        w = np.empty(n, np.float64)
        cnt = C.c_int()
        for i in range(n):
            _check(lib().dg_schedule_neighbors(self._h, rnd, i, idx, _dptr(w), n, C.byref(cnt)))
            out.append((list(idx[:cnt.value]), w[:cnt.value].copy()))
        return out


def _make(fn, *args):
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return MixingSchedule(h.value)


def make_complete(n: int) -> MixingSchedule:                      # topology.hpp:65-66
    return _make(lib().dg_make_complete, n)


def make_one_peer_ring(n: int) -> MixingSchedule:                 # topology.hpp:67-69
    return _make(lib().dg_make_one_peer_ring, n)


def make_one_peer_exponential(n: int) -> MixingSchedule:          # topology.hpp:70-72
    return _make(lib().dg_make_one_peer_exponential, n)


def make_aer(n: int, workers_per_node: int) -> MixingSchedule:    # topology.hpp:73-78
    return _make(lib().dg_make_aer, n, workers_per_node)


def make_static_exponential(n: int) -> MixingSchedule:            # new
    return _make(lib().dg_make_static_exponential, n)


def from_matrices(name: str, workers_per_node: int, rounds: Sequence[np.ndarray]) -> MixingSchedule:
    """MixingSchedule::from_matrices (topology.hpp:44-45)."""
    mats = np.ascontiguousarray(np.stack([np.asarray(r, np.float64) for r in rounds]))
    P, n, n2 = mats.shape
    if n != n2:
        raise ConfigError("from_matrices: matrices must be square")
    return _make(lib().dg_schedule_from_matrices_named, name.encode(), _dptr(mats), n, P, workers_per_node)


def validate(w) -> MixingValidation:                              # topology.hpp:80
    w = np.ascontiguousarray(w, np.float64)
    out = _Validation()
    _check(lib().dg_validate(_dptr(w), w.shape[0], C.byref(out)))
    return MixingValidation(*(bool(getattr(out, f)) if i < 5 else getattr(out, f)
                              for i, (f, _) in enumerate(_Validation._fields_)))


def spectral_lambda(w) -> float:                                  # topology.hpp:82-84
    w = np.ascontiguousarray(w, np.float64)
    out = C.c_double()
    _check(lib().dg_spectral_lambda(_dptr(w), w.shape[0], C.byref(out)))
    return out.value


def effective_lambda(s: MixingSchedule) -> float:                 # topology.hpp:86-88
    out = C.c_double()
    _check(lib().dg_effective_lambda(s.handle, C.byref(out)))
    return out.value


def plan_exchange(s: MixingSchedule, world_size: int, rank: int, rnd: int):
    """The gossip exchange the engine issues for (rank, round): (sends, recvs) lists of (peer, node)."""
    cap = max(64, 4 * s.workers())
    sp, sn, rp, rn = ((C.c_int * cap)() for _ in range(4))
    ns, nr = C.c_int(), C.c_int()
    _check(lib().dg_plan_exchange(s.handle, world_size, rank, rnd, sp, sn, C.byref(ns),
                                  rp, rn, C.byref(nr), cap))
    return ([(sp[k], sn[k]) for k in range(ns.value)], [(rp[k], rn[k]) for k in range(nr.value)])


# ----------------------------------------------------------------------------- optim
@dataclass
class OptimizerConfig:
    """OptimizerConfig; defaults = DAdam of PAPER.md:1139."""
    alpha: float = 2e-3
    beta1: float = 0.974
    beta2: float = 0.999
    eps: float = 1e-8
    s: int = 1
    paper_literal: bool = False

    def _c(self) -> _AdamCfg:
        return _AdamCfg(self.alpha, self.beta1, self.beta2, self.eps, int(self.s), int(self.paper_literal))


def _dev(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ConfigError(f"{name}: expected a contiguous float32 CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def gossip_mix(mixed, xs, weights, stream=None):
    """mixed <- sum_k w_k xs_k in the given (ascending-j) order, on the GPU."""
    n = mixed.numel()
    for x in xs:
        if x.numel() != n:
            raise ConfigError("gossip_mix: length mismatch")
    ptrs = (C.c_void_p * max(1, len(xs)))(*[_dev(x, "xs").value for x in xs])
    w = np.ascontiguousarray(weights, np.float64)
    _check(lib().dg_gossip_mix_f32(_dev(mixed, "mixed"), ptrs, _dptr(w), len(xs), n, _stream(stream)))


def _same_len(*ts):
    n = ts[0].numel()
    if any(t.numel() != n for t in ts):
        raise ConfigError("length mismatch")  # vec.cpp:11-14
    return n


def dadam_step(x, g, m, v, mixed, cfg: OptimizerConfig, t: int, stream=None):
    """dadam_step, in place on fp32 CUDA tensors."""
    n = _same_len(x, g, m, v, mixed)
    c = cfg._c()
    _check(lib().dg_dadam_step_f32(_dev(x, "x"), _dev(g, "g"), _dev(m, "m"), _dev(v, "v"),
                                   _dev(mixed, "mixed"), n, C.byref(c), t, _stream(stream)))


def accum_adam_step(x, g, m_hat, v_hat, b_acc, mixed, cfg: OptimizerConfig, t: int, T: int, stream=None):
    """accum_adam_step, in place on fp32 CUDA tensors."""
    n = _same_len(x, g, m_hat, v_hat, b_acc, mixed)
    c = cfg._c()
    _check(lib().dg_accum_adam_step_f32(_dev(x, "x"), _dev(g, "g"), _dev(m_hat, "m_hat"),
                                        _dev(v_hat, "v_hat"), _dev(b_acc, "b_acc"), _dev(mixed, "mixed"),
                                        n, C.byref(c), t, T, _stream(stream)))


def check_divergence(stream=None):
    """Raise DivergenceError(iteration) if a semantic step produced a non-finite state."""
    _check(lib().dg_step_check_divergence(_stream(stream)))


def fill_synthetic(out, seed: int, purpose: int, worker: int, iteration: int, stream=None):
    """out[e] = (float)(2u-1), u = draw e of StreamRng(seed, purpose, worker, iteration)."""
    _check(lib().dg_fill_synthetic_f32(_dev(out, "out"), out.numel(), seed, purpose, worker,
                                       iteration, _stream(stream)))


# ----------------------------------------------------------------------------- consensus (f2)
class ConsensusTrajectory(np.ndarray):
    """ConsensusTrajectory (topology.hpp:90-96): error[t], t = 0..rounds, as a
    float64 array (so arithmetic and comparisons work elementwise)."""

    def __new__(cls, error):
        return np.asarray(error, np.float64).view(cls)

    @property
    def error(self) -> np.ndarray:
        return self.view(np.ndarray)

    def to_csv(self, path_or_file) -> None:
        """Trajectory export, columns `round,consensus_error`."""
        lines = ["round,consensus_error"] + [f"{t},{e:.17g}" for t, e in enumerate(self.error)]
        text = "\n".join(lines) + "\n"
        if hasattr(path_or_file, "write"):
            path_or_file.write(text)
        else:
            with open(path_or_file, "w") as f:
                f.write(text)


def gossip_consensus(schedule: MixingSchedule, x0: np.ndarray, rounds: int, device: int = 0) -> ConsensusTrajectory:
    """gossip_consensus (topology.hpp:90-100) on one GPU:
    x <- W^(t) x for t = 1..rounds on fp32 buckets (fp64 mixing accumulation),
    error[t] = sum_i ||x_i - xbar0||^2 / sum_i ||x_i^0 - xbar0||^2 with xbar0 the
    preserved initial mean (fixed on the device before round 1); zero initial
    dispersion gives an all-zero trajectory.  The step is the fused engine with
    zero gradients, where DAdam reduces exactly to x <- mix."""
    x0 = np.ascontiguousarray(x0, np.float32)
    n, d = x0.shape
    if n != schedule.workers():
        raise ConfigError("gossip_consensus: x0 size mismatch")
    if rounds < 0:
        raise ConfigError("gossip_consensus: rounds < 0")
    eng = Engine(schedule, d, OptimizerConfig(), device=device)
    try:
        for i in range(n):
            eng.upload(i, X, x0[i])
        err = np.zeros(rounds + 1)
        eng.consensus_fix_mean()
        d0, _ = eng.consensus()
        if d0 == 0.0:
            return ConsensusTrajectory(err)
        err[0] = 1.0
        for t in range(1, rounds + 1):
            eng.step(t)
            err[t] = eng.consensus()[0] / d0
        eng.sync()
        return ConsensusTrajectory(err)
    finally:
        eng.close()


# ----------------------------------------------------------------------------- engine
def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().dg_nccl_unique_id(buf))
    return bytes(buf)


class Engine:
    """Fused gossip + Adam engine for the nodes resident on one GPU (dg_engine_*)."""

    def __init__(self, schedule: MixingSchedule, d: int, cfg: OptimizerConfig, algo: int = DADAM,
                 total_steps: int = 0, world_size: int = 1, rank: int = 0, device: int = 0,
                 nccl_id: Optional[bytes] = None, chunk: int = 0, transport: int = TRANSPORT_AUTO,
                 flags: int = 0):
        self.schedule = schedule
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_char * 128).from_buffer_copy(nccl_id)
        ec = _EngineConfig(schedule.handle.value, world_size, rank, device,
                           C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                           d, chunk, algo, cfg._c(), total_steps, transport, flags)
        h = C.c_void_p()
        _check(lib().dg_engine_create(C.byref(ec), C.byref(h)))
        self._h = h
        self.algo, self.cfg, self.d = algo, cfg, d
        st = self.stats()
        self.local_nodes, self.first_node = st["local_nodes"], st["first_node"]

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dg_engine_destroy(self._h)
            self._h = None

    __del__ = close

    def buffer(self, local: int, which: int) -> int:
        p = C.c_void_p()
        _check(lib().dg_engine_buffer(self._h, local, which, C.byref(p)))
        return p.value

    def upload(self, local: int, which: int, host: np.ndarray, offset: int = 0):
        if host.dtype != np.float32 or not host.flags.c_contiguous:
            raise ConfigError("upload: expected a contiguous float32 array")
        _check(lib().dg_engine_upload(self._h, local, which, host.ctypes.data_as(_VP), offset, host.size))

    def upload_ptr(self, local: int, which: int, host_ptr: int, count: int, offset: int = 0):
        _check(lib().dg_engine_upload(self._h, local, which, C.c_void_p(host_ptr), offset, count))

    def download(self, local: int, which: int, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        count = self.d - offset if count is None else count
        out = np.empty(count, np.float32)
        _check(lib().dg_engine_download(self._h, local, which, out.ctypes.data_as(_VP), offset, count))
        return out

    def gather(self, local: int, which: int, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, np.uint64)
        out = np.empty(idx.size, np.float32)
        _check(lib().dg_engine_gather(self._h, local, which, idx.ctypes.data_as(_VP), idx.size,
                                      out.ctypes.data_as(_VP)))
        return out

    def consensus_fix_mean(self):
        """Fix xbar of later consensus() calls to the current mean (collective)."""
        _check(lib().dg_engine_consensus_fix_mean(self._h))

    def consensus(self):
        """(sum_i ||x_i - xbar||^2, ||xbar||^2) over all nodes; collective across ranks."""
        a, b = C.c_double(), C.c_double()
        _check(lib().dg_engine_consensus(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def fill_synthetic(self, which: int, seed: int, purpose: int, per_node: bool, iteration: int):
        _check(lib().dg_engine_fill_synthetic(self._h, which, seed, purpose, int(per_node), iteration))

    def step(self, t: int):
        _check(lib().dg_engine_step(self._h, t))

    def run_steps(self, t_first: int, t_last: int, graph: bool = True, capture_only: bool = False):
        """Steps t_first..t_last; graph=True replays them as one cached CUDA graph
        (dg_engine_run_steps), identical results to calling step(t) for each t."""
        flags = (RUN_GRAPH if graph else 0) | (RUN_CAPTURE_ONLY if capture_only else 0)
        _check(lib().dg_engine_run_steps(self._h, t_first, t_last, flags))

    def step_range(self, t: int, off: int, length: int):
        _check(lib().dg_engine_step_range(self._h, t, off, length))

    def wait_stream(self, stream):
        _check(lib().dg_engine_wait_stream(self._h, _stream(stream)))

    def join(self, stream):
        _check(lib().dg_engine_join(self._h, _stream(stream)))

    def sync(self):
        _check(lib().dg_engine_sync(self._h))

    def streams(self):
        a, b = C.c_void_p(), C.c_void_p()
        _check(lib().dg_engine_streams(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_timing(self, on: bool):
        _check(lib().dg_engine_set_timing(self._h, int(on)))

    def stats(self) -> dict:
        s = _EngineStats()
        _check(lib().dg_engine_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _EngineStats._fields_}

"""Runtime model over libdg's native
simulator (dg_rm_*): per-iteration runtimes of All-Reduce, decentralized and
SGP-variant training from the dependency recurrences of PAPER.md Appendix A.5
and A.8.1, Eq. (3), Monte-Carlo speedup with common random numbers, and the
Gantt timeline export of Fig. 1."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import MixingSchedule, _check, _dptr, _RmParams, lib

ALLREDUCE, DECENTRALIZED, SGP = 0, 1, 2


@dataclass
class RuntimeParams:
    """RuntimeParams."""
    N: int = 8
    b: int = 4
    theta: float = 0.2
    gamma: float = 0.1
    omega: float = 1.0
    sigma2: float = 0.0
    workers_per_node: int = 1
    normalized: bool = False
    allow_omega_above_one: bool = False

    def _c(self):
        return _RmParams(self.N, self.b, self.theta, self.gamma, self.omega, self.sigma2, self.workers_per_node,
                         int(self.normalized), int(self.allow_omega_above_one))


def _simulate(mode, params: RuntimeParams, T: int, seed: int, schedule: Optional[MixingSchedule],
              timeline: bool):
    rt = np.empty(T, np.float64)
    tl = np.empty((T, params.N, 1 + 3 * params.b), np.float64) if timeline else None
    c = params._c()
    _check(lib().dg_rm_simulate(mode, C.byref(c), schedule.handle if schedule is not None else None, T, seed,
                                _dptr(rt), _dptr(tl) if tl is not None else None))
    return (rt, tl) if timeline else rt


def simulate_allreduce(params: RuntimeParams, T: int, seed: int = 0, timeline: bool = False):
    return _simulate(ALLREDUCE, params, T, seed, None, timeline)


def simulate_decentralized(params: RuntimeParams, T: int, seed: int = 0,
                           schedule: Optional[MixingSchedule] = None, timeline: bool = False):
    return _simulate(DECENTRALIZED, params, T, seed, schedule, timeline)


def simulate_sgp_variant(params: RuntimeParams, T: int, seed: int = 0,
                         schedule: Optional[MixingSchedule] = None, timeline: bool = False):
    return _simulate(SGP, params, T, seed, schedule, timeline)


def closed_form_speedup(gamma: float, N: int, b: int, theta: float) -> float:
    out = C.c_double()
    _check(lib().dg_rm_closed_form_speedup(gamma, N, b, theta, C.byref(out)))
    return out.value


def speed_multiplier(seed: int, worker: int, iteration: int, sigma2: float) -> float:
    out = C.c_double()
    _check(lib().dg_rm_speed_multiplier(seed, worker, iteration, sigma2, C.byref(out)))
    return out.value


def monte_carlo_speedup(params: RuntimeParams, T: int, replicates: int, seed: int = 0,
                        schedule: Optional[MixingSchedule] = None) -> Tuple[float, float]:
    """Mean All-Reduce / mean decentralized per-iteration runtime over replicates
    (common random numbers: same p^(i,t) draws per replicate); returns
    (speedup, 95% normal-approximation half-width over per-replicate ratios)."""
    if replicates < 1:
        raise ValueError("replicates >= 1")
    ratios = []
    for r in range(replicates):
        ar = simulate_allreduce(params, T, seed + r).mean()
        de = simulate_decentralized(params, T, seed + r, schedule).mean()
        ratios.append(ar / de)
    ratios = np.asarray(ratios)
    half = 1.96 * ratios.std(ddof=1) / math.sqrt(replicates) if replicates > 1 else 0.0
    return float(ratios.mean()), float(half)


def export_timeline(params: RuntimeParams, timeline: np.ndarray, mode: int, T: Optional[int] = None,
                    p: Optional[np.ndarray] = None) -> List[tuple]:
    """Gantt rows (worker, iteration, task, bucket, start, end), start = end - duration
    (SPEC.md:480-485), sorted by (worker, start).  p: speed multipliers [T, N] (default 1)."""
    T = timeline.shape[0] if T is None else T
    N, b = params.N, params.b
    rows = []
    for t in range(T):
        for i in range(N):
            rec = timeline[t, i]
            pi = 1.0 if p is None else p[t, i]
            fwd = pi * (b / N if (mode == ALLREDUCE and not params.normalized) else 1.0 / N)
            rows.append((i, t + 1, "F", 0, rec[0] - fwd, rec[0]))
            for k in range(1, b + 1):
                rows.append((i, t + 1, f"B_{k}", k, rec[k] - pi * 2.0 / N, rec[k]))
                if mode == ALLREDUCE:
                    rows.append((i, t + 1, f"C_{k}", k, rec[2 * b + k] - params.gamma, rec[2 * b + k]))
                else:
                    rows.append((i, t + 1, f"U_{k}", k, rec[b + k] - params.theta, rec[b + k]))
                    rows.append((i, t + 1, f"C_{k}", k, rec[2 * b + k] - params.omega * params.gamma,
                                 rec[2 * b + k]))
            if mode == ALLREDUCE:
                rows.append((i, t + 1, "U", 0, rec[b + 1] - params.theta * b, rec[b + 1]))
    rows.sort(key=lambda r: (r[0], r[4]))
    return rows

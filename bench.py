#!/usr/bin/env python3
"""Benchmark: fused gossip + DAdam step, param-updates/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (config.workload), numbered as BASELINE.md / SURVEY.md (1-5 =
BASELINE.json configs[0..4]); --config picks one, the default is
  N = 1: config 3 -- 8 simulated nodes on one B200, static exponential graph,
          350M-param flat fp32 bucket per node, DAdam (alpha 2e-3, betas
          0.974/0.999): the largest BASELINE config that fits
          one GPU (56 GB);
  N > 1: config 4 -- 8 nodes, alternating (AER) topology, 1.3B-param bucket,
          AccumAdam s=4, the config BASELINE names for 2/4/8-GPU
          scaling (208 GB: does not fit one GPU); strong scaling, nodes
          block-partitioned over the N GPUs.
A "step" is one dg_engine_step(t) over every resident node's full bucket:
mixing with the round-t peers (remote x^(t-1) read in-kernel over NVLink),
Adam moments and the model update, in one fused sm_100a kernel launch.

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 2410
METRIC = "gossip+DAdam param-updates/sec"
UNIT = "param-updates/s"
HBM_PER_UPDATE = 28.0          # B per DAdam param-update
HBM_PER_REMOTE = 12.0          # B of HBM per received remote bucket param (send read + slot write + read)
NVL_MEASURED = 770e9           # B/s per direction, measured peer copy (B200_PROFILING.md)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=None,
                   help="BASELINE config (1-based); default 3 at N=1, 4 at N>1")
    p.add_argument("--nodes", type=int, default=None, help="total nodes (overrides the config)")
    p.add_argument("--nodes-per-gpu", type=int, default=None, help="weak scaling: nodes per GPU")
    p.add_argument("--bucket-params", dest="d", type=int, default=None)
    p.add_argument("--topology", default=None,
                   choices=["one_peer_exponential", "one_peer_ring", "static_exponential", "aer"])
    p.add_argument("--algo", choices=["dadam", "accum", "allreduce"], default=None)
    p.add_argument("--chunk", type=int, default=0)
    p.add_argument("--transport", choices=["p2p", "nccl"], default="p2p")
    p.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                   help="replay the timed steps as one CUDA graph (dg_engine_run_steps); auto = on for "
                        "buckets below 2^27 params per GPU (launch-bound, e.g. config 1)")
    p.add_argument("--e2e-steps", type=int, default=4)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-clocks", action="store_true", help="do not sample nvidia-smi during the timed region")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


# BASELINE.json configs (numbered 1-5 as in BASELINE.md / SURVEY.md)
CONFIGS = {
    1: dict(topology="one_peer_ring", nodes=8, d=1 << 20, algo="accum",
            text="config 1: 8 simulated nodes, ring, 1M-param bucket, AccumAdam s=4"),
    2: dict(topology="one_peer_exponential", nodes=8, d=125_000_000, algo="dadam",
            text="config 2: 8 nodes, one-peer exponential, 125M-param bucket (GPT-2 small size), DAdam"),
    3: dict(topology="static_exponential", nodes=8, d=350_000_000, algo="dadam",
            text="config 3: 8 nodes, static exponential, 350M-param bucket, DAdam"),
    4: dict(topology="aer", nodes=8, d=1_300_000_000, algo="accum",
            text="config 4: 8 nodes, alternating (AER) topology, 1.3B-param bucket, AccumAdam s=4"),
    5: dict(topology="one_peer_exponential", nodes=64, d=125_000_000, algo="dadam",
            text="config 5: 64 simulated nodes, one-peer exponential, 125M params per node"),
}


def resolve(a, world):
    """Fill the workload from --config (default 3 at N=1, 4 at N>1); explicit
    flags override single fields.  Sets a.nodes (total) and a.scaling."""
    if a.config is None:
        a.config = 3 if world == 1 else 4
    c = CONFIGS[a.config]
    a.topology = a.topology or c["topology"]
    a.algo = a.algo or c["algo"]
    a.d = a.d or c["d"]
    custom = any(getattr(a, k) != c[k] for k in ("topology", "algo", "d"))
    if a.nodes_per_gpu:
        a.nodes, a.scaling = a.nodes_per_gpu * world, "weak"
    else:
        a.nodes = a.nodes or c["nodes"]
        a.scaling = "strong"
    custom |= a.nodes != c["nodes"]
    a.workload = (f"BASELINE {c['text']}" if not custom else
                  f"custom (from BASELINE config {a.config}): {a.nodes} nodes, "
                  f"{a.topology.replace('_', ' ')}, {a.d:,}-param bucket, {a.algo}")
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def make_schedule(mod, topo, n):
    if topo == "one_peer_exponential":
        return mod.make_one_peer_exponential(n)
    if topo == "one_peer_ring":
        return mod.make_one_peer_ring(n)
    if topo == "static_exponential":
        return mod.make_static_exponential(n)
    return mod.make_aer(n, 2)


def hyper(algo):
    if algo == "dadam":
        return dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1)
    if algo == "allreduce":
        return dict(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, s=1)     # PAPER.md:1153 (All-Reduce Adam)
    return dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)


def algo_code(dg, algo):
    return {"dadam": dg.DADAM, "accum": dg.ACCUM, "allreduce": dg.ALLREDUCE}[algo]


def config_block(a, world, nodes):
    return {
        "workload": a.workload, "baseline_config": a.config,
        "nodes": nodes, "nodes_per_gpu": nodes / world, "params_per_node": a.d,
        "topology": a.topology, "algo": a.algo, "seed": SEED,
        "parallelism": (f"gossip over {world} GPU(s), nodes block-partitioned; remote buckets "
                        + ("read in-kernel from peer HBM over NVLink (CUDA IPC)" if a.transport == "p2p"
                           else "via chunked NCCL send/recv over NVLink")),
        "transport": a.transport,
        "cuda_graph": bool(getattr(a, "use_graph", False)),
        "l2": ("no flush needed: every step streams >= 28 GB per GPU, > 126 MB L2" if a.d * nodes >= 1 << 27
               else "inputs smaller than L2: no flush (config 1 is a small-bucket, launch-bound case)"),
        "inputs": "synthetic StreamRng buckets (x0 ConsensusInit, g Minibatch@t=1 held fixed across timed steps)",
    }


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]) * 1e9, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650e9, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_traffic(key):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows, self.proc, self.th = [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        loaded = [float(r[1]) for r in self.rows if len(r) >= 9 and r[3].isdigit() and int(r[3]) > 0]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(loaded or sm) if (loaded or sm) else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def per_update_bytes(algo, t, s):
    """DAdam 28 B; AccumAdam 28 B, 36 B on the fold step (t % s == 0)."""
    return 36.0 if algo == "accum" and t % s == 0 else HBM_PER_UPDATE


class NvlCounters:
    """NVLink data counters of this rank's GPU, read through NVML around the
    timed region (hardware counters, not CUDA-event estimates).  Tries the
    per-link data-throughput fields (KiB) first, then the per-link byte
    counters; `read()` returns (tx_bytes, rx_bytes) summed over the links."""
    LINKS = 18

    def __init__(self, local):
        self.h, self.src, self.err = None, None, None
        try:
            import pynvml
            import torch
            self.nv = pynvml
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(local).uuid)
            self.uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.h = pynvml.nvmlDeviceGetHandleByUUID(self.uuid)
            for tx, rx, scale, name in (
                    (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                     1024.0, "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB, per link)"),
                    (pynvml.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, pynvml.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
                     1.0, "NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES (per link)")):
                self.ids, self.scale, self.src = (tx, rx), scale, name
                try:
                    if self.read() is not None:
                        return
                except Exception as e:  # noqa: BLE001
                    self.err = f"{name}: {e}"
            errs = self.err
            self.src = "nvidia-smi"
            if self.read() is None:
                self.src = None
                self.err = f"{errs}; {self.err}"
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def read(self):
        if self.src == "nvidia-smi":
            return self._read_smi()
        if self.h is None or self.ids is None:
            return None
        q = [(fid, link) for fid in self.ids for link in range(self.LINKS)]
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, q)
        out = [0.0, 0.0]
        ok = False
        codes = set()
        for k, v in enumerate(vals):
            if v.nvmlReturn != 0:
                codes.add(int(v.nvmlReturn))
                continue
            ok = True
            x = {0: v.value.dVal, 1: v.value.uiVal, 2: v.value.ulVal, 3: v.value.ullVal,
                 4: v.value.sllVal, 5: v.value.siVal}.get(int(v.valueType), v.value.ullVal)
            out[k // self.LINKS] += float(x) * self.scale
        if not ok:
            self.err = f"{self.src}: nvmlReturn codes {sorted(codes)}"
        return tuple(out) if ok else None

    def _read_smi(self):
        """`nvidia-smi nvlink -gt d`: per-link Data Tx / Rx counters in KiB."""
        import re
        p = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", self.uuid], capture_output=True, text=True,
                           timeout=30)
        tx = rx = 0.0
        hits = 0
        for m in re.finditer(r"Data\s+(Tx|Rx)\s*:\s*([0-9]+)\s*KiB", p.stdout):
            hits += 1
            if m.group(1) == "Tx":
                tx += float(m.group(2)) * 1024.0
            else:
                rx += float(m.group(2)) * 1024.0
        if not hits:
            self.err = (self.err or "") + f"; nvidia-smi nvlink -gt d: {p.stdout[:200]!r} {p.stderr[:200]!r}"
            return None
        return tx, rx


def step_roofline(sched, world, d, steps_t, hbm_bw, transport, algo="dadam", s=1):
    """SURVEY.md 8(d) per-GPU step bound, summed over the timed rounds:
    max over GPUs of max(HBM bytes / BW_HBM, NVLink bytes / BW_NVL).
    NCCL transport: every received remote bucket costs 12 B/param of HBM (owner
    read for the send, recv-slot write, kernel read).  P2P transport: the fused
    kernel reads remote buckets over NVLink, so HBM pays only the owner-side
    read (4 B/param per bucket served to a peer)."""
    import paper_2410_11998_b200 as dg
    n = sched.workers()
    if algo == "allreduce":  # column sums (8 B/elem written + read) + ring all-reduce of fp64 sums
        nl = -(-n // world)
        t_hbm = d * (HBM_PER_UPDATE * nl + 16.0) / hbm_bw
        t_nvl = (2.0 * (world - 1) / world) * 8.0 * d / NVL_MEASURED if world > 1 else 0.0
        return len(steps_t) * max(t_hbm, t_nvl)
    total = 0.0
    cache = {}
    for t in steps_t:
        r = (t - 1) % sched.period() + 1
        per_update = per_update_bytes(algo, t, s)
        if (r, per_update) not in cache:
            worst = 0.0
            for g in range(world):
                sends, recvs = dg.plan_exchange(sched, world, g, r)
                nl = sum(1 for i in range(n) if i * world // n == g)
                if transport == "p2p":
                    remote_hbm = 4.0 * len(sends)
                else:
                    remote_hbm = HBM_PER_REMOTE * len(recvs)
                t_hbm = d * (per_update * nl + remote_hbm) / hbm_bw
                t_nvl = 4.0 * d * max(len(recvs), len(sends)) / NVL_MEASURED
                worst = max(worst, t_hbm, t_nvl)
            cache[(r, per_update)] = worst
        total += cache[(r, per_update)]
    return total


# ------------------------------------------------------------------------- CPU legs
def cpu_reference_run(a, nodes_sample, d_sample, steps, threads):
    """The reference CPU path (oracle/_ref: reference vec.cpp + parallel_for) on a
    bounded sample; returns (updates/s, kind, note)."""
    import numpy as np
    from oracle import pyoracle as O
    h = hyper(a.algo)
    cfg = O.OptimizerConfig(**h)
    algo = algo_code(O, a.algo)
    s = {"one_peer_exponential": O.make_one_peer_exponential, "one_peer_ring": O.make_one_peer_ring,
         "static_exponential": O.make_static_exponential}.get(a.topology, lambda n: O.make_aer(n, 2))(nodes_sample)
    st = O.init_state(nodes_sample, d_sample, SEED, True, np.float64, algo)
    g = np.stack([O.fill_f32(SEED, O.MINIBATCH, i, 1, d_sample) for i in range(nodes_sample)]).astype(np.float64)
    T = 4 * (steps + 1)
    if O.ref_available():
        el = O.ref_run(s, algo, cfg, SEED, st, 1, steps, T, threads, g_fixed=g)
        kind = "reference"
        note = ("oracle/_ref: the reference's proj/src/vec.cpp + rng.cpp + parallel.hpp compiled from "
                "/root/reference, step composed per SPEC.md:272-280 (upstream ships no step code)")
    else:
        import ctypes as C
        L = O.lib()
        xprev = np.empty_like(st["x"])
        c = cfg.c()
        t0 = time.perf_counter()
        for t in range(1, steps + 1):
            rc = L.or_step_all_f64(s.handle, algo, C.byref(c), d_sample, t, T, threads, g.reshape(-1),
                                   st["x"].reshape(-1), xprev.reshape(-1), st["m"].reshape(-1),
                                   st["v"].reshape(-1), None)
            assert rc == 0
        el = time.perf_counter() - t0
        kind = "port"
        note = "oracle/oracle.cpp fp64 restatement (reference build absent)"
    return nodes_sample * d_sample * steps / el, kind, note, el


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(a, budget_s):
    import numpy as np  # noqa: F401
    threads = os.cpu_count() or 1
    nodes_sample, d_sample = 8, min(a.d, 1 << 21)
    # calibrate: 2 steps, then size the run to ~budget_s
    rate, _, _, el = cpu_reference_run(a, nodes_sample, d_sample, 2, threads)
    steps = max(3, int(budget_s * rate / (nodes_sample * d_sample)))
    rate, kind, note, el = cpu_reference_run(a, nodes_sample, d_sample, steps, threads)
    # Exec::Serial: one thread, a quarter of the sample
    serial, _, _, _ = cpu_reference_run(a, nodes_sample, d_sample, max(2, steps // 4), 1)
    return {"value": rate, "unit": UNIT, "cores": min(threads, nodes_sample), "host_threads": threads,
            "serial_value": serial, "cpu_model": cpu_model(),
            "kind": kind,
            "sample": (f"{nodes_sample} nodes x {d_sample:,} params (fp64), {steps} steps of the same "
                       f"topology/algorithm, g held fixed; {el:.1f} s wall; OpenMP over nodes "
                       f"(parallel.hpp:13-23 caps useful threads at the node count); {note}")}


# ------------------------------------------------------------------------- reference arm
def run_reference(a):
    rank, _, world = dist_env()
    if rank != 0:
        return
    resolve(a, world)
    nodes = a.nodes
    threads = os.cpu_count() or 1
    nodes_sample, d_sample = 8, min(a.d, 1 << 21)
    rate, kind, note, el = cpu_reference_run(a, nodes_sample, d_sample, a.warmup + a.steps, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * nodes_sample * d_sample / rate,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(a, world, nodes),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": min(threads, nodes_sample), "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{nodes_sample} nodes x {d_sample:,} params per step (bounded sample of "
                                   f"the workload), {a.warmup + a.steps} steps, {el:.1f} s; {note}"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- our arm
def run_ours(a):
    import numpy as np
    import torch
    import paper_2410_11998_b200 as dg

    rank, local, world = dist_env()
    if world != a.gpus:
        a.gpus = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    resolve(a, world)
    nodes = a.nodes
    sched = make_schedule(dg, a.topology, nodes)
    algo = algo_code(dg, a.algo)
    h = hyper(a.algo)
    total_t = a.warmup + a.steps + a.e2e_steps + 8
    total_t += (-total_t) % 4
    nccl_id = None
    if world > 1:
        obj = [dg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = dg.Engine(sched, a.d, dg.OptimizerConfig(**h), algo=algo, total_steps=total_t, world_size=world,
                    rank=rank, device=local, nccl_id=nccl_id, chunk=a.chunk,
                    transport=dg.TRANSPORT_P2P if a.transport == "p2p" else dg.TRANSPORT_NCCL)
    if a.algo == "allreduce":   # All-Reduce Adam: workers share x^(0) (Alg. 2 line 1)
        eng.fill_synthetic(dg.X, SEED, dg.Stream.INIT_MODEL, False, 0)
    else:                        # dispersed models so mixing is exercised from step 1
        eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
    eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, 1)
    eng.sync()
    comp_ptr, _ = eng.streams()
    comp = torch.cuda.ExternalStream(comp_ptr)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    use_graph = a.use_graph = a.graph == "on" or (a.graph == "auto" and a.d * nodes // world < (1 << 27)
                                    and a.algo != "allreduce")
    t = 0
    if use_graph:   # warm-up range captured + replayed, the timed range captured (not run) here
        eng.run_steps(1, a.warmup, graph=True)
        t = a.warmup
        eng.run_steps(t + 1, t + a.steps, graph=True, capture_only=True)
    else:
        for _ in range(a.warmup):
            t += 1
            eng.step(t)
    eng.sync()

    clocks = ClockSampler()
    if rank == 0 and not a.no_clocks:
        clocks.start()
        time.sleep(0.3)
    # ---- timed region: K steps, CUDA events on the engine's compute stream
    eng.set_timing(False)
    eng.set_timing(True)
    launches0 = eng.stats()["kernel_launches"]
    nvc = NvlCounters(local) if world > 1 else None
    nv0 = nvc.read() if nvc else None   # (before the barrier: host work here would skew the ranks' start)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(comp)
    timed_t = list(range(t + 1, t + a.steps + 1))
    if use_graph:
        eng.run_steps(t + 1, t + a.steps, graph=True)
        t += a.steps
    else:
        for _ in range(a.steps):
            t += 1
            eng.step(t)
    ev1.record(comp)
    eng.sync()
    torch.cuda.synchronize()
    barrier()
    nv1 = nvc.read() if nvc else None
    ms = ev0.elapsed_time(ev1)
    st = eng.stats()
    eng.set_timing(False)
    clk = clocks.stop() if rank == 0 and not a.no_clocks else None
    ms_max = max_over_ranks(ms)
    launches = st["kernel_launches"] - launches0
    nvl_counters = None
    if nvc is not None:   # hardware NVLink counters of every rank, gathered to rank 0
        mine = None
        if nv0 is not None and nv1 is not None:
            tx, rx = nv1[0] - nv0[0], nv1[1] - nv0[1]
            mine = {"rank": rank, "tx_bytes_per_step": tx / a.steps, "rx_bytes_per_step": rx / a.steps,
                    "rx_GBps_over_timed_region": rx / (ms / 1e3) / 1e9,
                    "rx_GBps_over_exchange_kernels": (rx / (st["remote_kernel_ms"] / 1e3) / 1e9
                                                      if st["remote_kernel_ms"] > 0 else None),
                    "algorithmic_remote_bytes_per_step": st["remote_bytes"] / a.steps}
        allc = [None] * world
        dist.all_gather_object(allc, mine)
        if all(c is not None for c in allc):
            rxk = [c["rx_GBps_over_exchange_kernels"] for c in allc if c["rx_GBps_over_exchange_kernels"]]
            nvl_counters = {"source": nvc.src, "per_rank": allc,
                            "min_rx_GBps_over_exchange_kernels": min(rxk) if rxk else None,
                            "peak": NVL_MEASURED / 1e9, "nominal": 900.0, "unit": "GB/s",
                            "frac_of_measured": (min(rxk) * 1e9 / NVL_MEASURED) if rxk else None,
                            "what": ("per GPU, NVLink data bytes received during the timed region (NVML "
                                     "hardware counters read before/after it) over the summed CUDA-event "
                                     "time of the exchange-round fused launches; counters include the "
                                     "1-element barrier all-reduces")}
        else:
            nvl_counters = {"unavailable": nvc.err or "NVML NVLink counters not readable"}
    value = nodes * a.d * a.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (fused gossip+Adam), live CUDA events
    hbm_bw, peak_src = read_peaks()
    kern_s = st["kernel_ms"] / 1e3
    achieved = st["timed_hbm_bytes"] / kern_s if kern_s > 0 else 0.0
    per_launch = st["timed_hbm_bytes"] / max(1, st["timed_launches"])
    transport = "p2p" if st["transport"] == dg.TRANSPORT_P2P else "nccl"
    roof_step_s = step_roofline(sched, world, a.d, timed_t, hbm_bw, transport, algo=a.algo, s=h["s"])

    # ---- end to end through the public API: pinned host g -> H2D each step, step, D2H status
    e2e = None
    if not a.no_e2e and a.e2e_steps > 0:
        nl = eng.local_nodes
        host = torch.empty((nl, a.d), dtype=torch.float32, pin_memory=True)
        for i in range(nl):
            host[i].copy_(torch.from_numpy(eng.download(i, dg.G)))
        barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            t += 1
            for i in range(nl):
                eng.upload_ptr(i, dg.G, host[i].data_ptr(), a.d)
            eng.step(t)
            eng.sync()            # D2H read of the step's status (divergence flag, 4 B)
        w1 = time.perf_counter()
        e2e_s = max_over_ranks(w1 - w0)
        e2e = {"value": nodes * a.d * a.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": 4 * nl * a.d * world, "d2h_bytes_per_step": 4 * world,
               "steps": a.e2e_steps,
               "note": "pinned host gradients copied H2D every step (PCIe-bound), device-resident x/m/v"}
        del host

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a, a.cpu_seconds)

    if rank == 0:
        key = f"{a.topology}/{a.algo}/n{nodes}/g{world}/d{a.d}"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_block(a, world, nodes),
            "roofline": {"bound": "hbm", "achieved": achieved / 1e9, "peak": hbm_bw / 1e9, "unit": "GB/s",
                         "frac": achieved / hbm_bw, "traffic": read_traffic(key),
                         "algorithmic_bytes_per_launch": per_launch,
                         "bytes_per_param_update": (HBM_PER_UPDATE if a.algo != "accum" else
                                                    "28 (36 on fold steps t % s == 0)"),
                         "kernel_ms_per_launch": st["kernel_ms"] / max(1, st["timed_launches"]),
                         "kernel_share_of_step": st["kernel_ms"] / ms if ms > 0 else None,
                         "peak_source": peak_src,
                         "kernel": ("gossip_adam_xshare<DEG,ALGO,FOLD,COLW> (csrc/xshare.cuh)"
                                    if os.environ.get("DG_XSHARE", "1") != "0" else
                                    "legacy.cu register-streaming kernels (DG_XSHARE=0)")},
            "step_roofline": {"bound_ms_per_step": 1e3 * roof_step_s / a.steps,
                              "frac": (roof_step_s * 1e3) / ms_max,
                              "model": ("SURVEY.md 8(d): per round, max over GPUs of max(HBM bytes/BW_HBM, "
                                        f"NVLink bytes/770 GB/s), {transport} transport"),
                              "nvlink_bytes_received_per_step": st["bytes_received"] / max(1, st["steps"])},
            "nvlink": ({"achieved": st["remote_bytes"] / (st["remote_kernel_ms"] / 1e3) / 1e9,
                        "peak": NVL_MEASURED / 1e9, "nominal": 900.0, "unit": "GB/s",
                        "frac": st["remote_bytes"] / (st["remote_kernel_ms"] / 1e3) / NVL_MEASURED,
                        "frac_of_nominal": st["remote_bytes"] / (st["remote_kernel_ms"] / 1e3) / 900e9,
                        "bytes_per_step": st["remote_bytes"] / a.steps,
                        "kernel_ms_per_step": st["remote_kernel_ms"] / a.steps,
                        "what": "remote x^(t-1) buckets read in-kernel over NVLink by the exchange-round "
                                "fused launches (per direction; every GPU both reads and serves)",
                        "peak_source": "measured peer read bandwidth, B200_PROFILING.md (775 GB/s LDG.128)",
                        "hw_counters": ("NVML/nvidia-smi NVLink counters unsupported on this B200 pool; ncu "
                                        "nvlrx__bytes of the same kernels in a single-process probe: "
                                        "profiles/r2_nvl_probe.md (data bytes = 1.000x algorithmic, 715 GB/s)")}
                       if st["remote_kernel_ms"] > 0 else None),
            "nvlink_counters": nvl_counters,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
            "nvlink_bytes_sent_per_step": st["bytes_sent"] / max(1, st["steps"]),
            "nccl_version": st["nccl_version"],
        }
        print(json.dumps(line), flush=True)
    if dist:   # no peer may still read this rank's IPC-exported x when it is freed
        dist.barrier()
    eng.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()

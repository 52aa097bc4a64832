"""Per-round step timing on N GPUs (torchrun), for tuning the exchange:
    torchrun --nproc-per-node N scripts/round_timing.py [--nodes-per-gpu 8] [--d 125000000]
Each step is bracketed by CUDA events on the engine's compute stream with a
barrier in between, so the printed ms are per round of the schedule."""
import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nodes-per-gpu", type=int, default=8)
ap.add_argument("--bucket-params", dest="d", type=int, default=125_000_000)
ap.add_argument("--topology", default="one_peer_exponential")
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--periods", type=int, default=2)
ap.add_argument("--b2b", action="store_true", help="steps back to back (no barrier/sync between them), events per step")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
n = a.nodes_per_gpu * world
sched = {"one_peer_exponential": dg.make_one_peer_exponential, "static_exponential": dg.make_static_exponential,
         "one_peer_ring": dg.make_one_peer_ring}.get(a.topology, lambda k: dg.make_aer(k, 2))(n)
obj = [dg.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
eng = dg.Engine(sched, a.d, dg.OptimizerConfig(), world_size=world, rank=rank, device=local, nccl_id=obj[0],
                chunk=a.chunk)
eng.fill_synthetic(dg.X, 2410, 6, True, 0)
eng.fill_synthetic(dg.G, 2410, 2, True, 1)
comp = torch.cuda.ExternalStream(eng.streams()[0])
P = sched.period()
t = 0
for _ in range(P):
    t += 1
    eng.step(t)
eng.sync()
res = {}
if a.b2b:   # the bench's regime: per-step events on the compute stream, no host sync in between
    evs = []
    dist.barrier()
    torch.cuda.synchronize()
    for _ in range(a.periods * P):
        t += 1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        eng.step(t)
        e1.record(comp)
        evs.append(((t - 1) % P + 1, e0, e1))
    eng.sync()
    tot = torch.tensor([evs[0][1].elapsed_time(evs[-1][2]) / len(evs)], device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"b2b first-to-last per step (incl. gaps between steps): {tot.item():.3f} ms", flush=True)
    for r, e0, e1 in evs:
        ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        res.setdefault(r, []).append(ms.item())
for _ in range(0 if a.b2b else a.periods * P):
    t += 1
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    eng.step(t)
    e1.record(comp)
    eng.sync()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    res.setdefault((t - 1) % P + 1, []).append(ms.item())
if rank == 0:
    sends, recvs = {}, {}
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("DG_", "NCCL_P2P", "NCCL_MIN", "NCCL_MAX")))
    line = " ".join(f"r{r}:{min(v):.2f}/{sum(v) / len(v):.2f}/{max(v):.2f}" for r, v in sorted(res.items()))
    avg = sum(sum(v) / len(v) for v in res.values()) / len(res)
    print(f"[{tag or 'default'}]{' b2b' if a.b2b else ''} chunk={a.chunk} rounds(ms min/mean/max) {line} "
          f"avg(mean)={avg:.2f}", flush=True)
eng.close()
dist.destroy_process_group()

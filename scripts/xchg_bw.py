"""Exchange bandwidth per direction of the transports the f1 DDP wrapper can
use: torchrun --nproc-per-node 2 scripts/xchg_bw.py [--range] [--transport nccl|p2p].
Engine with one node per GPU, one-peer exponential (every round swaps the whole
bucket with the peer).  NCCL: with DG_DIAG_SKIP_KERNEL=1 the exchange alone.
In-place P2P (--range --transport p2p): the update kernel itself reads the
peer's bucket over NVLink, so the line reports the whole range step and the
NVLink rate of its in-kernel reads.  Prints one line on rank 0."""
import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=125_000_000)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--range", action="store_true", help="in-place engine, whole-bucket step_range (f1 path)")
ap.add_argument("--tag", default="")
ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
obj = [dg.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
sched = dg.make_one_peer_exponential(world)
eng = dg.Engine(sched, a.d, dg.OptimizerConfig(), world_size=world, rank=rank, device=local, nccl_id=obj[0],
                chunk=a.chunk, transport=dg.TRANSPORT_NCCL if a.transport == "nccl" else dg.TRANSPORT_P2P,
                flags=dg.ENGINE_IN_PLACE if a.range else 0)
comp = torch.cuda.ExternalStream(eng.streams()[0])


def step(t):
    if a.range:
        eng.step_range(t, 0, a.d)
    else:
        eng.step(t)


for t in range(1, 4):
    step(t)
eng.sync()
eng.set_timing(True)
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(comp)
for t in range(4, 4 + a.iters):
    step(t)
e1.record(comp)
eng.sync()
ms = torch.tensor([e0.elapsed_time(e1) / a.iters], device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
st = eng.stats()
if rank == 0:
    gbs = 4.0 * a.d / (ms.item() / 1e3) / 1e9
    nvl = (st["remote_bytes"] / (st["remote_kernel_ms"] / 1e3) / 1e9) if st["remote_kernel_ms"] > 0 else None
    print(f"xchg {a.tag} transport={st['transport']} d={a.d} chunk={st['chunk']} range={a.range} "
          f"ms/step={ms.item():.3f} GB/s per direction={gbs:.1f} in-kernel NVLink GB/s={nvl}", flush=True)
eng.close()
dist.barrier()
dist.destroy_process_group()

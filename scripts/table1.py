"""Table-1 analogue on B200: gossip-averaging time per
iteration for 16 workers, three 25 MB fp32 tensors (19.66M params) per worker,
per topology, for both transports, next to All-Reduce Adam on the same buffers.
Run with torchrun on 4 GPUs (4 workers per GPU):
    torchrun --nproc-per-node 4 scripts/table1.py [--transport p2p|nccl]
Zero gradients make the fused DAdam step exactly x <- W x (pure averaging)."""
import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--transport", default="p2p")
ap.add_argument("--iters", type=int, default=48)
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
N, D = 16, 3 * 25 * 1024 * 1024 // 4
tp = dg.TRANSPORT_P2P if a.transport == "p2p" else dg.TRANSPORT_NCCL
rows = []
for name, sched, algo in (("Complete", dg.make_complete(N), dg.DADAM),
                          ("One-peer Exp", dg.make_one_peer_exponential(N), dg.DADAM),
                          ("One-peer Ring", dg.make_one_peer_ring(N), dg.DADAM),
                          ("AER (m=4)", dg.make_aer(N, 4), dg.DADAM),
                          ("All-Reduce Adam", dg.make_complete(N), dg.ALLREDUCE)):
    obj = [dg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    eng = dg.Engine(sched, D, dg.OptimizerConfig(alpha=1e-3, beta1=0.9), algo=algo, world_size=world, rank=rank,
                    device=local, nccl_id=obj[0], transport=tp)
    eng.fill_synthetic(dg.X, 2410, 4, False, 0)   # shared x0 (All-Reduce needs identical workers)
    comp = torch.cuda.ExternalStream(eng.streams()[0])
    for t in range(1, 9):
        eng.step(t)
    eng.sync()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for t in range(9, 9 + a.iters):
        eng.step(t)
    e1.record(comp)
    eng.sync()
    ms = torch.tensor([e0.elapsed_time(e1) / a.iters], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    rows.append((name, ms.item()))
    eng.close()
    dist.barrier()
if rank == 0:
    print(f"| topology ({N} workers on {world} B200, 3 x 25 MB fp32, transport {a.transport}) | ms / iteration | "
          f"x 8196 iterations (s) |")
    print("|---|---|---|")
    for name, ms in rows:
        print(f"| {name} | {ms:.3f} | {ms * 8196 / 1e3:.2f} |")
dist.destroy_process_group()

"""Training-iteration benchmark for the f1 wrapper, torchrun
one process per GPU.  Model: MLP stack (fp32 master weights, bf16 autocast
matmuls).  Modes, each timed over --iters iterations (max over ranks):
  gossip      DecentralizedDataParallel, 25 MB buckets: bucket updates start
              inside backward; default transport (in-place P2P: peers' buckets read
              in-kernel over NVLink, per-bucket stream-memory flags)
  gossip_nccl same with the NCCL transport (next-iteration send/recv pre-posted,
              PAPER.md:302-304)
  gossip_1b   same wrapper, one bucket (update after the whole backward)
  ddp_adam    torch DDP (bucketed NCCL all-reduce) + torch.optim.Adam(fused=True):
              the paper's All-Reduce baseline
  local_adam  no communication (compute + fused Adam only): lower bound
"""
import argparse
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from paper_2410_11998_b200.ddp import DecentralizedDataParallel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--width", type=int, default=2048)
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--batch", type=int, default=8192)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--topology", default="one_peer_exponential")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))


def make_model():
    torch.manual_seed(0)
    layers = []
    for _ in range(a.layers):
        layers += [torch.nn.Linear(a.width, 4 * a.width), torch.nn.GELU(), torch.nn.Linear(4 * a.width, a.width)]
    return torch.nn.Sequential(*layers).cuda()


def run(mode):
    model = make_model()
    nparams = sum(p.numel() for p in model.parameters())
    cfg = dg.OptimizerConfig(alpha=1e-4, beta1=0.9, beta2=0.999, eps=1e-8)
    if mode.startswith("gossip"):
        net = DecentralizedDataParallel(model, topology=a.topology, optimizer=cfg,
                                        bucket_cap_mb=1e9 if mode == "gossip_1b" else 25.0,
                                        transport="nccl" if mode == "gossip_nccl" else "auto")
        opt = None
    elif mode == "ddp_adam":
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
        opt = torch.optim.Adam(net.parameters(), lr=1e-4, fused=True)
    else:
        net, opt = model, torch.optim.Adam(model.parameters(), lr=1e-4, fused=True)
    x = torch.randn(a.batch, a.width, device="cuda")

    def it():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = net(x).float().pow(2).mean()
        loss.backward()
        if opt is not None:
            opt.step()
            opt.zero_grad(set_to_none=False)

    for _ in range(3):
        it()
    if mode.startswith("gossip"):
        net.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(a.iters):
        it()
    if mode.startswith("gossip"):
        net.synchronize()
    torch.cuda.synchronize()
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / a.iters], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    extra = (f" buckets={len(net.buckets)} transport={ {1: 'nccl', 2: 'p2p'}[net.engine.stats()['transport']] }"
             if mode.startswith("gossip") else "")
    del net, opt, model
    torch.cuda.empty_cache()
    return ms.item(), nparams, extra


res = [(m, *run(m)) for m in ("local_adam", "ddp_adam", "gossip_1b", "gossip_nccl", "gossip")]
if rank == 0:
    print(f"| mode ({world} B200, {res[0][2] / 1e6:.0f}M params, batch {a.batch}, {a.topology}) | ms / iteration |")
    print("|---|---|")
    for m, ms, n, extra in res:
        print(f"| {m}{extra} | {ms:.2f} |")
dist.destroy_process_group()

"""torchrun body for tests/test_multigpu.py::test_ddp_multigpu: the per-bucket
grad-hook wrapper on every rank (NCCL bucketed exchange pre-posted for the next
iteration) against the plain-PyTorch reference (all_gather + mix + Adam)."""
import copy
import os
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import paper_2410_11998_b200 as dg  # noqa: E402
from ddp_reference import ReferenceDAdam  # noqa: E402
from paper_2410_11998_b200.ddp import DecentralizedDataParallel  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.backends.cuda.matmul.allow_tf32 = False
    bad = 0
    for topo in ("one_peer_exponential", "one_peer_ring", "complete"):
        if topo == "one_peer_ring" and world % 2:
            continue
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.GELU(), torch.nn.Linear(256, 10)).cuda()
        ref_model = copy.deepcopy(model)
        cfg = dg.OptimizerConfig(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8)
        ddp = DecentralizedDataParallel(model, topology=topo, optimizer=cfg, bucket_cap_mb=0.02,
                                        transport=os.environ.get("MP_DDP_TRANSPORT", "auto"))
        names = {id(p): n for n, p in ddp.module.named_parameters()}
        layout = [((names[id(p)], p.numel()), o) for p, o in ddp._layout]
        ref = ReferenceDAdam(ref_model, layout, ddp.d, ddp.schedule, cfg, world, rank)
        gen = torch.Generator(device="cuda").manual_seed(100 + rank)      # different data per worker
        for it in range(10):
            xb = torch.randn(16, 64, device="cuda", generator=gen)
            yb = torch.randint(0, 10, (16,), device="cuda", generator=gen)
            torch.nn.functional.cross_entropy(ddp(xb), yb).backward()
            ref.step(lambda m: torch.nn.functional.cross_entropy(m(xb), yb))
        ddp.synchronize()
        got, want = ddp.flat_parameters(), ref.x
        err = float((got.double() - want.double()).norm() / want.double().norm())
        exact = bool(torch.equal(got, want))
        tr = {1: "nccl", 2: "p2p"}.get(ddp.engine.stats()["transport"])
        print(f"rank {rank}: {topo} transport={tr} buckets={len(ddp.buckets)} normwise={err:.3e} bit_exact={exact}",
              flush=True)
        # the reference uses the same separate fp32 ops and fp64 mixing: bit-identical by construction
        bad += (err > 1e-6) or not exact
        dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: {'ok' if not bad else 'FAIL'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

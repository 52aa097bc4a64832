"""Calibrate the runtime model (Appendix A.5) with
B200 timings and check its prediction against measured training iterations.
torchrun, one process per GPU:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 scripts/rm_calibrate.py

Measured per GPU on the f1 model (MLP stack, scripts/ddp_bench.py), medians of
CUDA-event timings, max over ranks:
  t_fb      forward + backward of one worker's batch   -> time unit u = N * t_fb / 3
            (the model's fwd + bwd of one bucket is 1/N + 2/N)
  t_upd     the engine's fused DAdam update of the whole model (one bucket)  -> theta = t_upd / u
  t_ar      NCCL all-reduce of the fp32 gradient bucket                         -> gamma = t_ar / u
  t_gossip  one gossip exchange of the bucket (send + recv with one peer)      -> omega = t_gossip / t_ar
Then dg_rm_simulate (b = 1, sigma^2 = 0) predicts the All-Reduce and the
decentralized per-iteration time (x u), compared with the measured iteration
of torch DDP + fused Adam and of DecentralizedDataParallel (one bucket)."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from paper_2410_11998_b200 import runtime_model as rm  # noqa: E402
from paper_2410_11998_b200.ddp import DecentralizedDataParallel  # noqa: E402

WIDTH, LAYERS, BATCH, REPS = 2048, 12, 8192, 12
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))


def make_model():
    torch.manual_seed(0)
    layers = []
    for _ in range(LAYERS):
        layers += [torch.nn.Linear(WIDTH, 4 * WIDTH), torch.nn.GELU(), torch.nn.Linear(4 * WIDTH, WIDTH)]
    return torch.nn.Sequential(*layers).cuda()


def med_ms(fn, reps=REPS):
    """median CUDA-event time of fn() on the current stream, max over ranks"""
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = torch.tensor([sorted(ts)[len(ts) // 2]], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def wall_ms(it, sync, iters=20):
    for _ in range(3):
        it()
    sync()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(iters):
        it()
    sync()
    torch.cuda.synchronize()
    t = torch.tensor([(time.perf_counter() - t0) * 1e3 / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


model = make_model()
P = sum(p.numel() for p in model.parameters())
x = torch.randn(BATCH, WIDTH, device="cuda")


def fwd_bwd():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = model(x).float().pow(2).mean()
    loss.backward()


t_fb = med_ms(fwd_bwd)
flat = torch.randn(P, device="cuda")
t_ar = med_ms(lambda: dist.all_reduce(flat))
recv = torch.empty_like(flat)
peer = rank ^ 1 if world > 1 else rank


def exchange():
    if world > 1:
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, flat, peer), dist.P2POp(dist.irecv, recv, peer)]):
            r.wait()


t_gossip = med_ms(exchange)
eng = dg.Engine(dg.make_complete(1), P, dg.OptimizerConfig(alpha=1e-4, beta1=0.9), algo=dg.DADAM,
                device=local)
eng.fill_synthetic(dg.X, 1, dg.Stream.CONSENSUS_INIT, True, 0)
eng.fill_synthetic(dg.G, 1, dg.Stream.MINIBATCH, True, 1)
step = [0]


def upd():
    step[0] += 1
    eng.step(step[0])
    eng.join(torch.cuda.current_stream())


t_upd = med_ms(upd)
eng.sync()
eng.close()
del flat, recv
opt = torch.optim.Adam(model.parameters(), lr=1e-4, fused=True)
t_adam = med_ms(opt.step)
del opt

# measured iterations: torch DDP + fused Adam (All-Reduce) and the gossip wrapper (one bucket)
ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
opt = torch.optim.Adam(ddp.parameters(), lr=1e-4, fused=True)


def it_ddp():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = ddp(x).float().pow(2).mean()
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=False)


m_ar = wall_ms(it_ddp, lambda: None)
del ddp, opt, model
torch.cuda.empty_cache()
model = make_model()
net = DecentralizedDataParallel(model, topology="one_peer_exponential",
                                optimizer=dg.OptimizerConfig(alpha=1e-4, beta1=0.9), bucket_cap_mb=1e9)


def it_gossip():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = net(x).float().pow(2).mean()
    loss.backward()


m_dec = wall_ms(it_gossip, net.synchronize)

if rank == 0:
    u = world * t_fb / 3.0
    prm = rm.RuntimeParams(N=world, b=1, theta=t_upd / u, gamma=t_ar / u, omega=min(1.0, t_gossip / t_ar),
                           sigma2=0.0, normalized=True)
    T = 40
    ar = rm.simulate_allreduce(prm, T)[-10:].mean() * u
    prm_ar = rm.RuntimeParams(**{**prm.__dict__, "theta": t_adam / u})
    ar_adam = rm.simulate_allreduce(prm_ar, T)[-10:].mean() * u
    dec = rm.simulate_decentralized(prm, T, schedule=dg.make_one_peer_exponential(world))[-10:].mean() * u
    print(f"## f4 calibration on {world} B200 ({P / 1e6:.0f}M-param MLP, batch {BATCH}/GPU, one bucket)\n")
    print("| measured | ms | model parameter |")
    print("|---|---|---|")
    print(f"| forward + backward t_fb | {t_fb:.3f} | unit u = N t_fb / 3 = {u:.3f} ms |")
    print(f"| engine DAdam update t_upd | {t_upd:.3f} | theta = {prm.theta:.4f} |")
    print(f"| torch fused Adam step | {t_adam:.3f} | theta_AR = {t_adam / u:.4f} |")
    print(f"| NCCL all-reduce of the bucket t_ar | {t_ar:.3f} | gamma = {prm.gamma:.4f} |")
    print(f"| one-peer exchange t_gossip | {t_gossip:.3f} | omega = {prm.omega:.4f} |")
    print()
    print("| iteration | model ms | measured ms |")
    print("|---|---|---|")
    print(f"| All-Reduce (DDP + fused Adam; model theta_AR) | {ar_adam:.2f} | {m_ar:.2f} |")
    print(f"| All-Reduce (model with the engine's theta) | {ar:.2f} | — |")
    print(f"| decentralized (gossip wrapper, one-peer exp) | {dec:.2f} | {m_dec:.2f} |")
    print(f"\nspeedup: model {ar_adam / dec:.3f}, measured {m_ar / m_dec:.3f}; "
          f"Eq. (3) best case {rm.closed_form_speedup(prm.gamma, world, 1, prm.theta):.3f}")
net.synchronize()
dist.destroy_process_group()

"""torchrun body for tests/test_multigpu.py: one process per GPU, nodes
block-partitioned over ranks, NCCL send/recv gossip exchange through libdg.
Every rank checks its resident nodes bit-exactly against the oracle's fp32
mirror run of ALL nodes on the CPU (so results are placement-invariant:
identical to the 1-GPU run).  Small chunks force the chunked, double-buffered
exchange pipeline.  Exit code 0 = all equal on this rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_11998_b200 as dg  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

SEED = 2410
TRANSPORT = {"nccl": dg.TRANSPORT_NCCL, "p2p": dg.TRANSPORT_P2P}[os.environ.get("MP_TRANSPORT", "p2p")]
CFG = {0: dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1),
       1: dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4)}
CASES = [("make_one_peer_exponential", "ONE_PEER_EXP", (8,)), ("make_one_peer_ring", "ONE_PEER_RING", (8,)),
         ("make_static_exponential", "STATIC_EXP", (8,)), ("make_aer", "AER", (8, 2)),
         ("make_complete", "COMPLETE", (8,)), ("make_one_peer_exponential", "ONE_PEER_EXP", (16,)),
         # >= 4 ranks: 16 resident nodes whose round graph has > 32 distinct sources (oversize plan)
         ("make_static_exponential", "STATIC_EXP", (64,))]


def fullsize(rank, world, local):
    """BASELINE configs 4 (AER(8,2), 1.3B, AccumAdam s=4) and 5 (64 nodes one-peer
    exponential, 125M per node; needs 4 GPUs) at full size, sampled columns."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from conftest import normwise
    from fullsize import check_against_oracle, run_engine_cols, sample_columns
    # T = 100 steps (north_star: "within 1e-6 relative after 100 steps")
    cases = [("config4_aer_1.3B_accum", "make_aer", "AER", (8, 2), 1_300_000_000, 1, 100)]
    if world >= 4:
        cases.append(("config5_64nodes_125M", "make_one_peer_exponential", "ONE_PEER_EXP", (64,), 125_000_000, 0, 100))
    bad = 0
    for name, fn, kind, args, d, algo, T in cases:
        obj = [dg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cols = sample_columns(d)
        got, first, nl = run_engine_cols(dg, getattr(dg, fn)(*args), d, algo, T, cols, world_size=world,
                                         rank=rank, device=local, nccl_id=obj[0], transport=TRANSPORT)
        errs = check_against_oracle(O, O.make(getattr(O, kind), *args), algo, T, cols, got, first, nl, normwise)
        print(f"rank {rank}: {name} nodes {first}..{first + nl - 1}: {'ok' if not errs else errs[:3]}", flush=True)
        bad += len(errs)
        dist.barrier()
    return bad


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    if os.environ.get("MP_FULLSIZE"):
        bad = fullsize(rank, world, local)
        dist.destroy_process_group()
        print(f"rank {rank}: {'ok' if not bad else f'{bad} failures'}", flush=True)
        sys.exit(1 if bad else 0)
    d = int(os.environ.get("MP_D", "100003"))
    chunk = int(os.environ.get("MP_CHUNK", "16384"))
    T = 12
    bad = 0
    for fn, kind, args in CASES:
        if -(-args[0] // world) > 64:  # engine limit: <= 64 resident nodes per GPU
            continue
        for algo in (0, 1):
            obj = [dg.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            sched = getattr(dg, fn)(*args)
            eng = dg.Engine(sched, d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T, world_size=world,
                            rank=rank, device=local, nccl_id=obj[0], chunk=chunk, transport=TRANSPORT)
            eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
            for t in range(1, T + 1):
                eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
                eng.step(t)
            eng.sync()
            st = O.init_state(sched.workers(), d, SEED, True, np.float32, algo)
            O.run(O.make(getattr(O, kind), *args), algo, O.OptimizerConfig(**CFG[algo]), SEED, st, 1, T, T)
            keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo else [])
            f = eng.first_node
            stats = eng.stats()
            # f2: collective consensus error over all ranks vs the mirror's states
            disp, msq = eng.consensus()
            xb = st["x"].astype(np.float64).mean(0)
            want_disp = float(((st["x"].astype(np.float64) - xb) ** 2).sum())
            if abs(disp - want_disp) > 1e-9 * want_disp or abs(msq - float(xb @ xb)) > 1e-9 * float(xb @ xb):
                print(f"rank {rank}: CONSENSUS MISMATCH {fn}{args} {disp} vs {want_disp}", flush=True)
                bad += 1
            for k, w in keys:
                got = np.stack([eng.download(i, w) for i in range(eng.local_nodes)])
                want = st[k][f:f + eng.local_nodes]
                if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                    print(f"rank {rank}: MISMATCH {fn}{args} algo={algo} {k}", flush=True)
                    bad += 1
            print(f"rank {rank}: {fn}{args} algo={algo} transport={stats['transport']} nodes {f}..{f + eng.local_nodes - 1} "
                  f"sent {stats['bytes_sent'] / 1e6:.1f} MB launches {stats['kernel_launches']} "
                  f"barriers {stats['barriers']}", flush=True)
            eng.close()
            dist.barrier()
    # f1 path: in-place engine (x never moves), dg_engine_step_range over three
    # ranges per iteration -- P2P: peers' publish buffers read in-kernel,
    # ordered by per-range stream-memory flags; NCCL: pre-posted send/recv
    cuts = [0, 40000, 70016, d] if d > 70016 else [0, d]
    for fn, kind, args in [("make_one_peer_exponential", "ONE_PEER_EXP", (8,)),
                           ("make_static_exponential", "STATIC_EXP", (8,)), ("make_one_peer_ring", "ONE_PEER_RING", (8,))]:
        for algo in (0, 1):
            obj = [dg.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            eng = dg.Engine(getattr(dg, fn)(*args), d, dg.OptimizerConfig(**CFG[algo]), algo=algo, total_steps=T,
                            world_size=world, rank=rank, device=local, nccl_id=obj[0], transport=TRANSPORT,
                            flags=dg.ENGINE_IN_PLACE)
            eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
            for t in range(1, T + 1):
                eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
                for k in range(len(cuts) - 1):
                    eng.step_range(t, cuts[k], cuts[k + 1] - cuts[k])
            eng.sync()
            st = O.init_state(8, d, SEED, True, np.float32, algo)
            O.run(O.make(getattr(O, kind), *args), algo, O.OptimizerConfig(**CFG[algo]), SEED, st, 1, T, T)
            f = eng.first_node
            keys = [("x", dg.X), ("m", dg.M), ("v", dg.V)] + ([("b", dg.ACC)] if algo else [])
            for k, w in keys:
                got = np.stack([eng.download(i, w) for i in range(eng.local_nodes)])
                if not np.array_equal(got.view(np.uint32), st[k][f:f + eng.local_nodes].view(np.uint32)):
                    print(f"rank {rank}: MISMATCH in-place {fn}{args} algo={algo} {k}", flush=True)
                    bad += 1
            stats = eng.stats()
            print(f"rank {rank}: in-place {fn}{args} algo={algo} transport={stats['transport']} ranges={len(cuts) - 1}"
                  f" launches {stats['kernel_launches']}", flush=True)
            eng.close()
            dist.barrier()
    # f3: All-Reduce Adam across ranks (NCCL all-reduce of fp64 gradient column sums)
    for n_nodes in (8, 16):
        obj = [dg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        acfg = dict(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, s=1)
        eng = dg.Engine(dg.make_complete(n_nodes), d, dg.OptimizerConfig(**acfg), algo=dg.ALLREDUCE, total_steps=T,
                        world_size=world, rank=rank, device=local, nccl_id=obj[0], transport=TRANSPORT)
        eng.fill_synthetic(dg.X, SEED, dg.Stream.INIT_MODEL, False, 0)
        for t in range(1, T + 1):
            eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
            eng.step(t)
        eng.sync()
        st = O.init_state(n_nodes, d, SEED, False, np.float32)
        O.run(O.make_complete(n_nodes), O.ALLREDUCE, O.OptimizerConfig(**acfg), SEED, st, 1, T)
        f = eng.first_node
        for k, w in (("x", dg.X), ("m", dg.M), ("v", dg.V)):
            got = np.stack([eng.download(i, w) for i in range(eng.local_nodes)])
            if not np.array_equal(got.view(np.uint32), st[k][f:f + eng.local_nodes].view(np.uint32)):
                print(f"rank {rank}: MISMATCH allreduce n={n_nodes} {k}", flush=True)
                bad += 1
        eng.close()
        dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: {'ok' if not bad else f'{bad} mismatches'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

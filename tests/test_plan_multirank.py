"""Multi-GPU host logic on CPU: world_size 2 / 4 / 8 gloo ranks each build their
round plans through libdg (dg_plan_exchange) and check, via gloo collectives,
that every rank's sends to a peer are exactly that peer's receives from it, in
the same (node-ascending) order NCCL's per-peer in-order matching needs, and
that the receives cover every remote neighbour the rank mixes."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [("make_one_peer_exponential", (8,)), ("make_one_peer_exponential", (64,)),
         ("make_one_peer_ring", (8,)), ("make_static_exponential", (8,)), ("make_aer", (8, 2)),
         ("make_aer", (16, 2)), ("make_complete", (8,)), ("make_static_exponential", (64,)),
         ("make_aer", (64, 8))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2410_11998_b200 as dg
        for fn, args in CASES:
            s = getattr(dg, fn)(*args)
            n = s.workers()
            if world > n:
                continue
            if -(-n // world) > 64:  # engine limit: <= 64 resident nodes per GPU
                try:
                    dg.plan_exchange(s, world, rank, 1)
                    raise AssertionError("expected ConfigError for > 64 resident nodes")
                except dg.ConfigError:
                    continue
            owner = [i * world // n for i in range(n)]
            for r in range(1, s.period() + 1):
                sends, recvs = dg.plan_exchange(s, world, rank, r)
                allp = [None] * world
                dist.all_gather_object(allp, (sends, recvs))
                for peer in range(world):
                    if peer == rank:
                        continue
                    mine_to_peer = [node for p_, node in sends if p_ == peer]
                    peer_from_me = [node for p_, node in allp[peer][1] if p_ == rank]
                    assert mine_to_peer == peer_from_me, (fn, args, r, rank, peer)
                    assert mine_to_peer == sorted(mine_to_peer)
                # receives == remote neighbours actually mixed here
                mine = [i for i in range(n) if owner[i] == rank]
                need = sorted({j for i in mine for j in s.neighbors_at(r)[i] if owner[j] != rank},
                              key=lambda j: (owner[j], j))
                assert [node for _, node in recvs] == need, (fn, r, rank)
                assert all(owner[node] == rank for _, node in sends)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, None))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_plans_match_across_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v is None for v in res.values()), res

"""DecentralizedDataParallel: the paper's PyTorch extension,
driving the B200 engine bucket by bucket from backward hooks.

One process per GPU, one decentralized worker (node) per GPU ("one GPU per
worker").  The wrapped module's parameters and gradients become
views of the engine's flat fp32 x / g buckets (no copies).  Parameters are laid
out in reverse registration order (approximately backward order, like DDP) and
grouped into buckets of <= bucket_cap_mb.  Every parameter gets a
post_accumulate_grad_hook (PyTorch >= 2.1); when the last gradient of a bucket
has been accumulated, the hook hands the bucket to dg_engine_step_range:

    wait for the bucket's round-t exchange (posted at t-1)   T_Uk = max{T_Bk, T_Ck^(t-1)} + theta
    update the bucket (mix with the round-t peers + Adam)    U_k
    post the bucket's round-(t+1) exchange                   C_k

so the gossip of bucket k overlaps the rest of backward and the next forward.
Transport (`transport=`): "auto" (default) = P2P when CUDA IPC works: the
update kernel reads the peers' x^(t-1) of the bucket in-kernel over NVLink
from their publish buffers, ordered by per-bucket stream-memory flags (no
copies, no NCCL kernels); "nccl" = NCCL send/recv of the bucket pre-posted at
t-1, as described above.
Buckets launch in a fixed global order (bucket 0, 1, ... on every rank) however
autograd orders the hooks.  An iteration starts with the first hook of a
backward and ends at the next forward (which joins the engine's stream);
eval / no_grad forwards never step, and no_sync() accumulates gradients over
several backwards.  No optimizer is needed: the engine performs the DAdam /
AccumAdam update.
"""
from __future__ import annotations

from contextlib import contextmanager
from typing import Callable, List, Optional

import torch

from . import (DADAM, ENGINE_IN_PLACE, G, TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_P2P, X, ConfigError, Engine,
               OptimizerConfig,
               make_aer, make_complete, make_one_peer_exponential, make_one_peer_ring, make_static_exponential,
               nccl_unique_id)

_TOPOLOGIES = {
    "one_peer_exponential": make_one_peer_exponential,
    "one_peer_ring": make_one_peer_ring,
    "static_exponential": make_static_exponential,
    "complete": make_complete,
}


class _DeviceArray:
    """Zero-copy fp32 view of engine memory for torch.as_tensor (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_view(ptr: int, n: int) -> torch.Tensor:
    return torch.as_tensor(_DeviceArray(ptr, n), device="cuda")


def _round_up(n: int, a: int = 64) -> int:
    return (n + a - 1) // a * a


class DecentralizedDataParallel(torch.nn.Module):
    def __init__(self, module: torch.nn.Module, topology="one_peer_exponential",
                 optimizer: Optional[OptimizerConfig] = None, algo: int = DADAM, total_steps: int = 0,
                 bucket_cap_mb: float = 25.0, aer_workers_per_node: int = 1, transport: str = "auto"):
        super().__init__()
        import torch.distributed as dist
        self.module = module
        self.world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank() if self.world > 1 else 0
        self.device = torch.cuda.current_device()
        if self.world == 1:                     # a single worker has no peers: W = [1]
            sched = make_complete(1)
        elif isinstance(topology, str):
            sched = (make_aer(self.world, aer_workers_per_node) if topology == "aer"
                     else _TOPOLOGIES[topology](self.world))
        elif isinstance(topology, Callable):
            sched = topology(self.world)
        else:
            sched = topology
        if sched.workers() != self.world:
            raise ConfigError("DecentralizedDataParallel: the schedule must have one worker per process")
        self.schedule = sched
        params = [p for p in module.parameters() if p.requires_grad]
        if not params:
            raise ConfigError("DecentralizedDataParallel: no trainable parameters")
        # flat layout in backward-ish order, 64-float aligned parameters, <= cap buckets
        cap = max(64, int(bucket_cap_mb * (1 << 20) / 4))
        self._layout: List[tuple] = []          # (param, offset)
        buckets: List[list] = []                 # [start, end, [params]]
        off = 0
        for p in reversed(params):
            n = p.numel()
            if not buckets or (off - buckets[-1][0] + n > cap and buckets[-1][2]):
                buckets.append([off, off, []])
            self._layout.append((p, off))
            buckets[-1][2].append(p)
            off += _round_up(n)
            buckets[-1][1] = off
        self.d = off
        self.buckets = [(b[0], b[1], b[2]) for b in buckets]
        nccl_id = None
        if self.world > 1:
            obj = [nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        self.engine = Engine(sched, self.d, optimizer or OptimizerConfig(), algo=algo, total_steps=total_steps,
                             world_size=self.world, rank=self.rank, device=self.device, nccl_id=nccl_id,
                             transport={"auto": TRANSPORT_AUTO, "p2p": TRANSPORT_P2P,
                                        "nccl": TRANSPORT_NCCL}[transport], flags=ENGINE_IN_PLACE)
        self._x = device_view(self.engine.buffer(0, X), self.d)
        self._g = device_view(self.engine.buffer(0, G), self.d)
        with torch.no_grad():
            for p, o in self._layout:                 # x^(0) <- x^(0) of rank 0 (Alg. 1 line 1)
                self._x[o:o + p.numel()].copy_(p.detach().reshape(-1))
            if self.world > 1:
                dist.broadcast(self._x, src=0)
            torch.cuda.current_stream().synchronize()
        for p, o in self._layout:                     # parameters / gradients = views of the buckets
            p.data = self._x[o:o + p.numel()].view_as(p)
            p.grad = self._g[o:o + p.numel()].view_as(p)
        self._bucket_of = {}
        for b, (_, _, ps) in enumerate(self.buckets):
            for p in ps:
                self._bucket_of[id(p)] = b
                p.register_post_accumulate_grad_hook(self._on_grad)
        self.t = 0                       # iterations whose step has been issued (or is in flight)
        self._active = False             # a backward of iteration t is firing hooks
        self._sync = True                # False inside no_sync(): accumulate, no step
        self._zero_next = False          # g was consumed by a step: zero before the next accumulation
        self._pending = [len(b[2]) for b in self.buckets]
        self._ready = [False] * len(self.buckets)
        self._next = 0                   # next bucket to launch (fixed global order 0, 1, ...)
        self._views = {id(p): self._g[o:o + p.numel()].view_as(p) for p, o in self._layout}

    # ------------------------------------------------------------------ hooks
    def _on_grad(self, p: torch.Tensor):
        view = self._views[id(p)]
        if p.grad is None or p.grad.data_ptr() != view.data_ptr():
            # zero_grad(set_to_none=True) or a rebound .grad detached the
            # parameter from the engine's g bucket: copy the fresh gradient back
            # into the bucket and re-attach the view
            with torch.no_grad():
                if p.grad is None:
                    view.zero_()
                else:
                    view.copy_(p.grad)
            p.grad = view
        if not self._sync:
            return
        if not self._active:             # first hook of a backward: iteration t+1 begins
            self._active = True
            self.t += 1
            self._pending = [len(b[2]) for b in self.buckets]
            self._ready = [False] * len(self.buckets)
            self._next = 0
        b = self._bucket_of[id(p)]
        self._pending[b] -= 1
        if self._pending[b] == 0:
            self._ready[b] = True
            self._drain()

    def _drain(self):
        # Buckets launch strictly in index order on every rank (NCCL
        # point-to-point is matched by issue order; the P2P
        # transport assigns per-bucket flags in first-use order), like
        # torch DDP's next_bucket_: a bucket that becomes ready early waits for
        # its predecessors.
        while self._next < len(self.buckets) and self._ready[self._next]:
            self._launch(self._next)
            self._next += 1

    def _launch(self, b: int):
        start, end, _ = self.buckets[b]
        self.engine.wait_stream(torch.cuda.current_stream())   # g of this bucket is complete
        self.engine.step_range(self.t, start, min(end, self.d) - start)

    def finish_iteration(self):
        """Launch the buckets of the running iteration that have not launched yet
        (unused parameters never fire hooks), in order, then make the current
        stream wait for every bucket update of the iteration."""
        if self._active:
            for b in range(self.buckets.__len__()):
                self._ready[b] = True
            self._drain()
            self._active = False
            self._zero_next = True
        self.engine.join(torch.cuda.current_stream())

    @contextmanager
    def no_sync(self):
        """Gradient accumulation: backward passes inside accumulate into the
        engine's g bucket without stepping; the first backward outside steps."""
        old, self._sync = self._sync, False
        try:
            yield
        finally:
            self._sync = old

    def forward(self, *args, **kwargs):
        # A backward that fired hooks since the last forward completed an
        # iteration: finish it (x^(t) must be final before this forward reads
        # it).  Evaluation / no_grad forwards and forwards inside no_sync()
        # never start a step.
        self.finish_iteration()
        if self._zero_next and self.training and torch.is_grad_enabled():
            with torch.no_grad():
                self._g.zero_()
            self._zero_next = False
        return self.module(*args, **kwargs)

    def synchronize(self):
        """Finish the current iteration and wait for every queued update (raises
        DivergenceError(t) on a non-finite state)."""
        self.finish_iteration()
        self.engine.sync()

    def flat_parameters(self) -> torch.Tensor:
        return self._x

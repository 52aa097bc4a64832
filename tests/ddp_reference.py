"""Plain-PyTorch decentralized Adam used as the checker for the DDP wrapper
(tests only): per iteration, gradients at x^(t-1) from the same model, x^(t-1)
of every rank via all_gather, mixed = sum_{j in N_i} w_ij x_j (fp64 accumulate,
ascending j, one rounding), then Alg. 1 lines 4-6 with separate fp32 ops and the
same fp32-derived scalars as the engine."""
import math

import numpy as np
import torch


def scalars(cfg, t):
    f = lambda v: float(np.float32(v))
    b1, b2 = f(cfg.beta1), f(cfg.beta2)
    return dict(b1=b1, omb1=1.0 - b1, b2=b2, omb2=1.0 - b2, c1=1.0 / (1.0 - b1 ** t),
                c2=1.0 / (1.0 - b2 ** t), neg_alpha=-f(cfg.alpha), eps=f(cfg.eps))


class ReferenceDAdam:
    def __init__(self, model, layout, d, schedule, cfg, world, rank):
        self.model, self.layout, self.d = model, layout, d
        self.schedule, self.cfg, self.world, self.rank = schedule, cfg, world, rank
        self.x = torch.zeros(d, device="cuda")
        with torch.no_grad():
            for (name, n), o in layout:
                self.x[o:o + n].copy_(dict(model.named_parameters())[name].detach().reshape(-1))
        if world > 1:
            import torch.distributed as dist
            dist.broadcast(self.x, src=0)
        self.m = torch.zeros(d, device="cuda")
        self.v = torch.zeros(d, device="cuda")
        self.t = 0

    def _load(self):
        params = dict(self.model.named_parameters())
        with torch.no_grad():
            for (name, n), o in self.layout:
                params[name].copy_(self.x[o:o + n].view_as(params[name]))

    def step(self, loss_fn):
        import torch.distributed as dist
        self.t += 1
        self._load()
        self.model.zero_grad(set_to_none=False)
        loss_fn(self.model).backward()
        g = torch.zeros(self.d, device="cuda")
        params = dict(self.model.named_parameters())
        for (name, n), o in self.layout:
            g[o:o + n] = params[name].grad.reshape(-1)
        if self.world > 1:
            xs = [torch.empty_like(self.x) for _ in range(self.world)]
            dist.all_gather(xs, self.x)
        else:
            xs = [self.x]
        idx, w = self.schedule.neighbors_and_weights_at(self.t)[self.rank]
        acc = torch.zeros(self.d, dtype=torch.float64, device="cuda")
        for j, wj in zip(idx, w):
            acc = acc + float(wj) * xs[j].double()
        mixed = acc.float()
        s = scalars(self.cfg, self.t)
        self.m = self.m * s["b1"] + g * s["omb1"]
        self.v = self.v * s["b2"] + (g * g) * s["omb2"]
        direction = (self.m * s["c1"]) / (torch.sqrt(self.v * s["c2"]) + s["eps"])
        self.x = mixed + direction * s["neg_alpha"]

"""the per-bucket grad-hook wrapper.
Engine-level dg_engine_step_range parity, and DecentralizedDataParallel on one
GPU (N=1: DAdam == textbook Adam) against a plain-PyTorch
reference of the same update."""
import numpy as np
import pytest

from conftest import normwise

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

SEED = 2410


@pytest.mark.parametrize("algo", [0, 1])
def test_step_range_matches_oracle(dg, oracle, algo):
    c = (dict(alpha=2e-3, beta1=0.974, beta2=0.999, eps=1e-8, s=1) if algo == 0 else
         dict(alpha=8e-4, beta1=0.9, beta2=0.999, eps=1e-8, s=4))
    d, T = 10_000, 12
    ranges = [(0, 3008), (3008, 4992), (8000, 2000)]      # buckets tiling [0, d)
    for fn, kind, args in (("make_one_peer_ring", "ONE_PEER_RING", (8,)), ("make_static_exponential", "STATIC_EXP", (8,))):
        eng = dg.Engine(getattr(dg, fn)(*args), d, dg.OptimizerConfig(**c), algo=algo, total_steps=T,
                        flags=dg.ENGINE_IN_PLACE)
        eng.fill_synthetic(dg.X, SEED, dg.Stream.CONSENSUS_INIT, True, 0)
        x_ptr = eng.buffer(0, dg.X)
        for t in range(1, T + 1):
            eng.fill_synthetic(dg.G, SEED, dg.Stream.MINIBATCH, True, t)
            for off, n in reversed(ranges):
                eng.step_range(t, off, n)
        eng.sync()
        assert eng.buffer(0, dg.X) == x_ptr                # in place: x never moves
        st = oracle.init_state(8, d, SEED, True, np.float32, algo)
        oracle.run(oracle.make(getattr(oracle, kind), *args), algo, oracle.OptimizerConfig(**c), SEED, st, 1, T, T)
        for k, w in (("x", dg.X), ("m", dg.M), ("v", dg.V)):
            got = np.stack([eng.download(i, w) for i in range(8)])
            assert np.array_equal(got.view(np.uint32), st[k].view(np.uint32)), (fn, algo, k)
        eng.close()


def _mlp():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.GELU(), torch.nn.Linear(256, 256), torch.nn.GELU(),
                               torch.nn.Linear(256, 10)).cuda()


def test_ddp_single_gpu_matches_reference(dg):
    import copy
    from ddp_reference import ReferenceDAdam
    from paper_2410_11998_b200.ddp import DecentralizedDataParallel
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    model = _mlp()
    ref_model = copy.deepcopy(model)
    cfg = dg.OptimizerConfig(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8)
    ddp = DecentralizedDataParallel(model, optimizer=cfg, bucket_cap_mb=0.1)   # several buckets
    assert len(ddp.buckets) >= 3
    layout = []
    names = {id(p): n for n, p in ddp.module.named_parameters()}
    for p, o in ddp._layout:
        layout.append(((names[id(p)], p.numel()), o))
    ref = ReferenceDAdam(ref_model, layout, ddp.d, ddp.schedule, cfg, 1, 0)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for it in range(15):
        xb = torch.randn(32, 64, device="cuda", generator=gen)
        yb = torch.randint(0, 10, (32,), device="cuda", generator=gen)
        loss = torch.nn.functional.cross_entropy(ddp(xb), yb)
        loss.backward()
        ref.step(lambda m: torch.nn.functional.cross_entropy(m(xb), yb))
    ddp.synchronize()
    got = ddp.flat_parameters().cpu().numpy()
    want = ref.x.cpu().numpy()
    assert normwise(got, want) <= 1e-6
    assert loss.item() < 2.5


def test_ddp_eval_no_sync_and_zero_grad(dg):
    """eval / no_grad forwards never step; no_sync() accumulates two
    backwards into one step; zero_grad(set_to_none=True) re-attaches the
    gradient to the engine's bucket (compared with the plain-PyTorch reference)."""
    import copy
    from ddp_reference import ReferenceDAdam
    from paper_2410_11998_b200.ddp import DecentralizedDataParallel
    torch.backends.cuda.matmul.allow_tf32 = False
    model = _mlp()
    ref_model = copy.deepcopy(model)
    cfg = dg.OptimizerConfig(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8)
    ddp = DecentralizedDataParallel(model, optimizer=cfg, bucket_cap_mb=0.1)
    names = {id(p): n for n, p in ddp.module.named_parameters()}
    layout = [((names[id(p)], p.numel()), o) for p, o in ddp._layout]
    ref = ReferenceDAdam(ref_model, layout, ddp.d, ddp.schedule, cfg, 1, 0)
    gen = torch.Generator(device="cuda").manual_seed(5)
    batch = lambda: (torch.randn(32, 64, device="cuda", generator=gen), torch.randint(0, 10, (32,), device="cuda", generator=gen))
    ce = torch.nn.functional.cross_entropy
    x0 = ddp.flat_parameters().clone()
    ddp.eval()
    with torch.no_grad():
        for _ in range(3):
            ddp(batch()[0])
    ddp.synchronize()
    assert ddp.t == 0 and torch.equal(ddp.flat_parameters(), x0)
    ddp.train()
    for it in range(4):
        (x1, y1), (x2, y2) = batch(), batch()
        with ddp.no_sync():
            ce(ddp(x1), y1).backward()
        ce(ddp(x2), y2).backward()
        ref.step(lambda m: ce(m(x1), y1) + ce(m(x2), y2))
        if it == 1:
            ddp.module.zero_grad(set_to_none=True)
            ddp.synchronize()
            # the step of iteration 2 already consumed g; the next accumulation re-binds the views
    ddp.synchronize()
    assert ddp.t == 4
    assert normwise(ddp.flat_parameters().cpu().numpy(), ref.x.cpu().numpy()) <= 1e-6

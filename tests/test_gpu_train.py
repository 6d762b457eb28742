"""The training restatement (paper_2310_00177_b200/train.py, torch) computes
the same network as the CUDA kernels: outputs agree to f32 rounding on random
weights and geometry; its operator equals the CUDA spmv."""
import numpy as np
import pytest

from paper_2310_00177_b200 import scenes

pytestmark = pytest.mark.gpu


def test_torch_network_matches_cuda(b200):
    import torch

    from paper_2310_00177_b200 import train

    t = scenes.random_types((32, 32, 32), 5)
    p = b200.init_params(4, 13)
    ctx = b200.Context(3, t.shape, p)
    ctx.set_mask(t)
    x = np.random.default_rng(2).standard_normal(t.shape).astype(np.float32)
    want = ctx.net_apply(x)
    geo = train.Geometry(t, 4, torch.device("cuda"))
    flat = torch.tensor(p.flat, device="cuda")
    got = train.net_apply(train.unflatten(flat, 4), geo, torch.tensor(x, device="cuda")[None], 4)[0].cpu().numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-5
    # the loss operator is the solve's operator
    v = np.random.default_rng(3).standard_normal(ctx.n_fluid)
    full = np.zeros(t.size)
    full[t.reshape(-1) == 0] = v
    av = train.poisson(geo, torch.tensor(full.reshape(t.shape), device="cuda")[None])[0].cpu().numpy().reshape(-1)
    assert np.allclose(av[t.reshape(-1) == 0], ctx.spmv(v), rtol=0, atol=1e-12)

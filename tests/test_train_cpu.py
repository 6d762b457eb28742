"""The training restatement (paper_2310_00177_b200/train.py) on CPU against
the oracle: the torch network equals the restated network to f32 rounding
and its operator equals the oracle's spmv (small grids)."""
import numpy as np
import pytest

from paper_2310_00177_b200 import scenes

torch = pytest.importorskip("torch")


def test_torch_network_and_operator_match_oracle(oracle):
    from paper_2310_00177_b200 import train

    t = scenes.random_types((16, 16, 16), 9)
    p = oracle.init_params(3, 3, 21)
    octx = oracle.context(t, p, 3)
    x = np.random.default_rng(4).standard_normal(t.shape).astype(np.float32)
    want = octx.net_apply(x.reshape(-1)).reshape(t.shape)
    geo = train.Geometry(t, 3, torch.device("cpu"))
    got = train.net_apply(train.unflatten(torch.tensor(p), 3), geo, torch.tensor(x)[None], 3)[0].numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-5
    v = np.random.default_rng(5).standard_normal(int((t == 0).sum()))
    full = np.zeros(t.size)
    full[t.reshape(-1) == 0] = v
    av = train.poisson(geo, torch.tensor(full.reshape(t.shape))[None])[0].numpy().reshape(-1)
    assert np.allclose(av[t.reshape(-1) == 0], oracle.spmv(t, v), rtol=0, atol=1e-12)

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


@pytest.mark.ref
@pytest.mark.parametrize("depth", [2, 3])
def test_loss_and_gradient_match_reference_backward(ref, depth):
    """The torch restatement's loss and autograd gradient against the
    reference's hand-written backward pass (backward_batch<float>,
    train.hpp:94-150 over net/backward.hpp:46-169) on a 2D mixed-BC frame:
    same weights, same right-hand sides, the reference's un-normalised loss."""
    from paper_2310_00177_b200 import train

    n = 32
    c = np.arange(n) + 0.5
    y, x = np.meshgrid(c, c, indexing="ij")
    t = np.zeros((n, n), np.uint8)
    t[y >= 0.7 * n] = 1
    t[(x < 0.3 * n) & (y < 0.25 * n)] = 2
    t[0, :] = t[-1, :] = t[:, 0] = t[:, -1] = 2
    p = ref.init_params_2d(depth, 5)
    fl = t.reshape(-1) == 0
    rhs = np.stack([ref.rhs_normal(100 + i, t.size)[fl] for i in range(4)])
    want_loss, want_g = ref.backward_2d(t, p, depth, rhs)

    geo = train.Geometry(t, depth, torch.device("cpu"))
    flat = torch.tensor(p, requires_grad=True)
    b = torch.zeros((4, t.size), dtype=torch.float64)
    b[:, torch.tensor(fl)] = torch.tensor(rhs)
    L = train.loss(train.unflatten(flat, depth, dim=2), geo, b.view(4, n, n), depth, normalize=False)
    L.backward()
    got = flat.grad.numpy()
    assert abs(L.item() - want_loss) <= 1e-5 * want_loss
    assert np.linalg.norm(got - want_g) <= 1e-4 * np.linalg.norm(want_g)
    # the comparison is not vacuous: most weights get a gradient
    assert np.count_nonzero(want_g) > 0.5 * want_g.size

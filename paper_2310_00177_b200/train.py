"""Training of 3D network weights — offline, not the solve.

The reference trains its 2D network with a hand-written backward pass
(`train.cpp:76-151`, `backward.hpp:46-169`) on the loss ||b - A P(b)||_2
(`train.hpp:40-91`) with Adam (`train.cpp:25-56`). This module restates the
same network (`NetContext::build` / `apply`, `net/forward.hpp:56-129`, in the
3D conventions of DESIGN.md) as differentiable torch ops and trains it with
torch autograd on the GPU. Training is a one-off offline step: the weights it
writes (`save_npm`, dim 3) are loaded by the CUDA solve path, which never runs
torch. `torch_net_apply` is checked against the CUDA kernels' `net_apply` on
random weights (tests/test_gpu_train.py).

Network, per level l (3 planes of pooled one-hot masks, padded with the solid
ring):
    K_l(x)[s] = B[s] + sum_{c,t} W[s,c,t] I_pad(c, x + off(t))   (conv3d)
    apply(K, v)(x) = sum_s K(x)[s] v_pad(x + off(s))
    down: y_l = apply(Kd_l, x_l), x_{l+1} = avg_pool(y_l); coarsest: y = apply(Kc, x)
    up:   out_l = z_a,l y_l + z_b,l apply(Ku_l, upsample(out_{l+1}))
    z = bias + (1 / (27 n_l)) sum_{c,t} K[c,t] F[c,t],  F[c,t] = sum_x I_pad(c, x + off(t))
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

S = 27
WN, KN = S * 3 * S, 3 * S  # 3D conv weights (2187), linear block (81)


def sizes(dim: int) -> tuple[int, int, int]:
    """(slots, conv weights, linear-block weights): 3D 27/2187/81, 2D 9/243/27
    (params.hpp:14-26)."""
    s = 27 if dim == 3 else 9
    return s, s * 3 * s, 3 * s


def level_count(depth: int, dim: int = 3) -> int:
    s, wn, kn = sizes(dim)
    return (depth - 1) * (2 * (wn + s) + 2 * (kn + 1)) + (wn + s)


def unflatten(flat: torch.Tensor, depth: int, dim: int = 3) -> dict:
    """for_each_span order (params.hpp:66-80): per level l < L-1 down W,B;
    up W,B; lin_a K,bias; lin_b K,bias; then the coarse W,B."""
    s, wn, kn = sizes(dim)
    p, o = {}, 0

    def take(n):
        nonlocal o
        v = flat[o:o + n]
        o += n
        return v

    for l in range(depth - 1):
        p[f"dW{l}"], p[f"dB{l}"] = take(wn), take(s)
        p[f"uW{l}"], p[f"uB{l}"] = take(wn), take(s)
        p[f"aK{l}"], p[f"ab{l}"] = take(kn), take(1)
        p[f"bK{l}"], p[f"bb{l}"] = take(kn), take(1)
    p["cW"], p["cB"] = take(wn), take(s)
    assert o == flat.numel()
    return p


def _offsets(dim: int):
    """window offsets in slot order (x fastest, then y, then z)"""
    if dim == 3:
        return [(dz, dy, dx) for dz in range(3) for dy in range(3) for dx in range(3)]
    return [(dy, dx) for dy in range(3) for dx in range(3)]


def _shift(v: torch.Tensor, off, shape):
    """v padded by one: the window view at offset off, shape `shape` (trailing dims)"""
    return v[(..., *[slice(o, o + n) for o, n in zip(off, shape)])]


class Geometry:
    """Per-frame constants of one cell-type grid (2D or 3D): padded level
    images, window sums, the fluid mask and the Poisson operator's diagonal."""

    def __init__(self, types: np.ndarray, depth: int, device) -> None:
        t = torch.as_tensor(np.ascontiguousarray(types), device=device).long()
        self.dim = t.dim()
        self.shape = tuple(t.shape)
        pool = F.avg_pool3d if self.dim == 3 else F.avg_pool2d
        pw = (1, 1) * self.dim
        img = torch.stack([(t == c).float() for c in range(3)])  # (3, *shape)
        self.ipad, self.F, self.n = [], [], []
        for l in range(depth):
            if l > 0:
                img = pool(img[None], 2)[0]
            pad = F.pad(img, pw)
            pad[2] = F.pad(img[2], pw, value=1.0)  # the solid ring
            self.ipad.append(pad)
            shp = tuple(img.shape[1:])
            fs = torch.stack([_shift(pad, off, shp).sum(dim=tuple(range(1, self.dim + 1)))
                              for off in _offsets(self.dim)], dim=1)  # (3, S)
            self.F.append(fs.double())
            self.n.append(int(np.prod(shp)))
        self.fluid = (t == 0)
        # diagonal of the reduced Poisson row: non-solid in-domain face neighbours
        ns = F.pad((t != 2).float(), pw)
        diag = torch.zeros_like(t, dtype=torch.float64)
        for off in _faces(self.dim):
            diag += _shift(ns, off, self.shape).double()
        self.diag = diag * self.fluid


def _faces(dim: int):
    if dim == 3:
        return [(0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)]
    return [(0, 1), (2, 1), (1, 0), (1, 2)]


def kernels(ipad: torch.Tensor, W: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """build_kernels (kernels.hpp:121-144): (S, *shape)."""
    dim = ipad.dim() - 1
    s = 27 if dim == 3 else 9
    if dim == 3:
        return F.conv3d(ipad[None], W.view(s, 3, 3, 3, 3), B)[0]
    return F.conv2d(ipad[None], W.view(s, 3, 3, 3), B)[0]


def apply(K: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """apply_kernels (kernels.hpp:147-172) on a batch v: (nb, *shape)."""
    dim = v.dim() - 1
    shp = tuple(v.shape[1:])
    vp = F.pad(v, (1, 1) * dim)
    out = torch.zeros_like(v)
    for s, off in enumerate(_offsets(dim)):
        out = out + K[s] * _shift(vp, off, shp)
    return out


def net_apply(p: dict, geo: Geometry, x: torch.Tensor, depth: int) -> torch.Tensor:
    """NetContext::apply (forward.hpp:95-129) on a batch x: (nb, *shape)."""
    dim = geo.dim
    pool = F.avg_pool3d if dim == 3 else F.avg_pool2d
    s = 27 if dim == 3 else 9
    ys, cur = [], x
    for l in range(depth - 1):
        y = apply(kernels(geo.ipad[l], p[f"dW{l}"], p[f"dB{l}"]), cur)
        ys.append(y)
        cur = pool(y[:, None], 2)[:, 0]
    out = apply(kernels(geo.ipad[depth - 1], p["cW"], p["cB"]), cur)
    for l in range(depth - 2, -1, -1):
        up = out
        for d in range(1, dim + 1):
            up = up.repeat_interleave(2, d)
        u = apply(kernels(geo.ipad[l], p[f"uW{l}"], p[f"uB{l}"]), up)
        norm = 1.0 / (s * geo.n[l])  # forward.hpp:78 (9 n_l in 2D, 27 n_l in 3D)
        za = p[f"ab{l}"][0] + norm * (p[f"aK{l}"].view(3, s).double() * geo.F[l]).sum().float()
        zb = p[f"bb{l}"][0] + norm * (p[f"bK{l}"].view(3, s).double() * geo.F[l]).sum().float()
        out = za * ys[l] + zb * u
    return out


def poisson(geo: Geometry, v: torch.Tensor) -> torch.Tensor:
    """A v for full-grid batches with zeros off fluid (assemble_poisson[_3d])."""
    vp = F.pad(v, (1, 1) * geo.dim)
    nb = torch.zeros_like(v)
    for off in _faces(geo.dim):
        nb = nb + _shift(vp, off, geo.shape)
    return (geo.diag * v - nb) * geo.fluid


def loss(p: dict, geo: Geometry, b: torch.Tensor, depth: int, normalize: bool = True) -> torch.Tensor:
    """Mean over the batch of ||b - A P(b)|| (loss_one, train.hpp:69-91, and
    backward_batch's batch mean, :94-150); normalize divides each by ||b|| so
    every frame weighs the same (False: the reference's loss)."""
    d = net_apply(p, geo, b.float(), depth).double() * geo.fluid
    r = b - poisson(geo, d)
    nr = r.flatten(1).norm(dim=1)
    return (nr / b.flatten(1).norm(dim=1) if normalize else nr).mean()


def smooth_rhs(geo: Geometry, nb: int, gen: torch.Generator, sweeps: int) -> torch.Tensor:
    """Right-hand sides weighted to the operator's low end (the slow modes of
    CG, like the reference's Ritz-vector datasets, dataset.cpp:34-59): white
    noise on fluid cells smoothed by `sweeps` damped-Jacobi sweeps of A."""
    b = torch.randn((nb,) + geo.shape, generator=gen, device=geo.fluid.device, dtype=torch.float64) * geo.fluid
    inv = torch.where(geo.diag > 0, 1.0 / geo.diag.clamp(min=1), torch.zeros_like(geo.diag))
    for _ in range(sweeps):
        b = b - (2.0 / 3.0) * inv * poisson(geo, b)
    return b / b.flatten(1).norm(dim=1).view(-1, 1, 1, 1)


class RitzSet:
    """Right-hand sides from Ritz vectors of a frame's operator, the paper's
    training data (after DCDM): m steps of Lanczos with full
    reorthogonalisation on the reduced operator (fluid cells), the Ritz
    vectors Y = Q S of the tridiagonal's eigenpairs, and random combinations
    b = Y c, normalised, with the coefficients of the low half of the spectrum
    weighted `low_weight` times the rest. The reference generates its 2D sets
    the same way (dataset.cpp:34-59, lanczos.cpp:25-82)."""

    def __init__(self, geo: Geometry, m: int, gen: torch.Generator, low_weight: float = 9.0) -> None:
        dev = geo.fluid.device
        self.geo = geo
        self.idx = geo.fluid.reshape(-1).nonzero().squeeze(1)
        nf = self.idx.numel()
        m = min(m, nf)
        Q = torch.empty((m, nf), dtype=torch.float64, device=dev)
        q = torch.randn(nf, generator=gen, device=dev, dtype=torch.float64)
        q /= q.norm()
        alpha = torch.zeros(m, dtype=torch.float64, device=dev)
        beta = torch.zeros(m, dtype=torch.float64, device=dev)
        prev = torch.zeros_like(q)
        for j in range(m):
            Q[j] = q
            w = self.apply_a(q) - (beta[j - 1] * prev if j else 0.0)
            alpha[j] = torch.dot(w, q)
            w = w - alpha[j] * q
            for _ in range(2):  # full reorthogonalisation
                w = w - Q[: j + 1].T @ (Q[: j + 1] @ w)
            b = w.norm()
            if j + 1 < m:
                beta[j] = b
                prev, q = q, w / b
        T = torch.diag(alpha) + torch.diag(beta[: m - 1], 1) + torch.diag(beta[: m - 1], -1)
        theta, S = torch.linalg.eigh(T)  # ascending
        self.theta = theta
        # Ritz vectors Y = Q^T S by ascending Ritz value, (nf, m), in row chunks
        # and stored as bf16 (a training set of random combinations needs no more)
        self.Y = torch.empty((nf, m), dtype=torch.bfloat16, device=dev)
        for r0 in range(0, nf, 1 << 20):
            self.Y[r0:r0 + (1 << 20)] = (Q[:, r0:r0 + (1 << 20)].T @ S).to(torch.bfloat16)
        del Q
        w = torch.ones(m, dtype=torch.float32, device=dev)
        w[: m // 2] = low_weight
        self.weight = w

    def apply_a(self, v: torch.Tensor) -> torch.Tensor:
        full = torch.zeros(self.geo.fluid.numel(), dtype=v.dtype, device=v.device)
        full[self.idx] = v
        return poisson(self.geo, full.view((1,) + self.geo.shape)).reshape(-1)[self.idx]

    def sample(self, nb: int, gen: torch.Generator) -> torch.Tensor:
        c = torch.randn((self.Y.shape[1], nb), generator=gen, device=self.Y.device) * self.weight[:, None]
        bf = (self.Y @ c.to(torch.bfloat16)).double().T  # (nb, nf)
        bf = bf / bf.norm(dim=1, keepdim=True)
        out = torch.zeros((nb, self.geo.fluid.numel()), dtype=torch.float64, device=bf.device)
        out[:, self.idx] = bf
        return out.view((nb,) + self.geo.shape)


def train(frames, depth: int, steps: int, lr: float, init: np.ndarray, nb: int, seed: int, device,
          log=print, max_sweeps: int = 40, ritz_m: int = 0, ritz_every: int = 1) -> np.ndarray:
    """Adam on the flat parameter vector (adam_update, train.cpp:25-56)."""
    flat = torch.tensor(init, dtype=torch.float32, device=device, requires_grad=True)
    opt = torch.optim.Adam([flat], lr=lr, betas=(0.9, 0.999), eps=1e-8)
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, T_max=max(steps, 1), eta_min=lr * 0.05)
    geos = [Geometry(t, depth, device) for t in frames]
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    # Ritz-vector right-hand sides (the paper's data) on every ritz_every-th frame
    ritz = {}
    if ritz_m > 0:
        for i, geo in enumerate(geos):
            if i % ritz_every == 0:
                ritz[i] = RitzSet(geo, ritz_m, gen)
        log(f"ritz sets: {len(ritz)} frames x {ritz_m} Lanczos vectors")
    for step in range(steps):
        gi = step % len(geos)
        geo = geos[gi]
        sweeps = int(torch.randint(0, max_sweeps, (1,), generator=gen, device=device).item())
        b = ritz[gi].sample(nb, gen) if gi in ritz else smooth_rhs(geo, nb, gen, sweeps)
        opt.zero_grad()
        L = loss(unflatten(flat, depth), geo, b, depth)
        L.backward()
        opt.step()
        sched.step()
        if step % 100 == 0 or step == steps - 1:
            log(f"step {step:5d} loss {L.item():.5f} (sweeps {sweeps})")
        if not math.isfinite(L.item()):
            raise RuntimeError("train: non-finite loss")
    return flat.detach().cpu().numpy()

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
WN, KN = S * 3 * S, 3 * S  # conv weights (2187), linear block (81)


def level_count(depth: int) -> int:
    return (depth - 1) * (2 * (WN + S) + 2 * (KN + 1)) + (WN + S)


def unflatten(flat: torch.Tensor, depth: int) -> dict:
    """for_each_span order (params.hpp:66-80, 3D): per level l < L-1 down W,B;
    up W,B; lin_a K,bias; lin_b K,bias; then the coarse W,B."""
    p, o = {}, 0

    def take(n):
        nonlocal o
        v = flat[o:o + n]
        o += n
        return v

    for l in range(depth - 1):
        p[f"dW{l}"], p[f"dB{l}"] = take(WN), take(S)
        p[f"uW{l}"], p[f"uB{l}"] = take(WN), take(S)
        p[f"aK{l}"], p[f"ab{l}"] = take(KN), take(1)
        p[f"bK{l}"], p[f"bb{l}"] = take(KN), take(1)
    p["cW"], p["cB"] = take(WN), take(S)
    assert o == flat.numel()
    return p


class Geometry:
    """Per-frame constants of one cell-type grid: padded level images, window
    sums, the fluid mask and the Poisson operator's diagonal."""

    def __init__(self, types: np.ndarray, depth: int, device) -> None:
        t = torch.as_tensor(np.ascontiguousarray(types), device=device).long()
        self.shape = tuple(t.shape)
        img = torch.stack([(t == c).float() for c in range(3)])  # (3, nz, ny, nx)
        self.ipad, self.F, self.n = [], [], []
        for l in range(depth):
            if l > 0:
                img = F.avg_pool3d(img[None], 2)[0]
            pad = F.pad(img, (1, 1, 1, 1, 1, 1))
            pad[2] = F.pad(img[2], (1, 1, 1, 1, 1, 1), value=1.0)  # the solid ring
            self.ipad.append(pad)
            nz, ny, nx = img.shape[1:]
            fs = torch.stack([pad[:, dz:dz + nz, dy:dy + ny, dx:dx + nx].sum(dim=(1, 2, 3))
                              for dz in range(3) for dy in range(3) for dx in range(3)], dim=1)  # (3, 27)
            self.F.append(fs.double())
            self.n.append(nz * ny * nx)
        self.fluid = (t == 0)
        # diagonal of the reduced Poisson row: non-solid in-domain face neighbours
        ns = F.pad((t != 2).float(), (1, 1, 1, 1, 1, 1))
        nz, ny, nx = t.shape
        diag = torch.zeros_like(t, dtype=torch.float64)
        for dz, dy, dx in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
            diag += ns[dz:dz + nz, dy:dy + ny, dx:dx + nx].double()
        self.diag = diag * self.fluid


def kernels(ipad: torch.Tensor, W: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    """build_kernels (kernels.hpp:121-144): (27, nz, ny, nx)."""
    return F.conv3d(ipad[None], W.view(S, 3, 3, 3, 3), B)[0]


def apply(K: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """apply_kernels (kernels.hpp:147-172) on a batch v: (nb, nz, ny, nx)."""
    nz, ny, nx = v.shape[1:]
    vp = F.pad(v, (1, 1, 1, 1, 1, 1))
    out = torch.zeros_like(v)
    s = 0
    for dz in range(3):
        for dy in range(3):
            for dx in range(3):
                out = out + K[s] * vp[:, dz:dz + nz, dy:dy + ny, dx:dx + nx]
                s += 1
    return out


def net_apply(p: dict, geo: Geometry, x: torch.Tensor, depth: int) -> torch.Tensor:
    """NetContext::apply (forward.hpp:95-129) on a batch x: (nb, nz, ny, nx)."""
    ys, cur = [], x
    for l in range(depth - 1):
        y = apply(kernels(geo.ipad[l], p[f"dW{l}"], p[f"dB{l}"]), cur)
        ys.append(y)
        cur = F.avg_pool3d(y[:, None], 2)[:, 0]
    out = apply(kernels(geo.ipad[depth - 1], p["cW"], p["cB"]), cur)
    for l in range(depth - 2, -1, -1):
        up = out.repeat_interleave(2, 1).repeat_interleave(2, 2).repeat_interleave(2, 3)
        u = apply(kernels(geo.ipad[l], p[f"uW{l}"], p[f"uB{l}"]), up)
        norm = 1.0 / (27.0 * geo.n[l])
        za = p[f"ab{l}"][0] + norm * (p[f"aK{l}"].view(3, S).double() * geo.F[l]).sum().float()
        zb = p[f"bb{l}"][0] + norm * (p[f"bK{l}"].view(3, S).double() * geo.F[l]).sum().float()
        out = za * ys[l] + zb * u
    return out


def poisson(geo: Geometry, v: torch.Tensor) -> torch.Tensor:
    """A v for full-grid batches with zeros off fluid (assemble_poisson_3d)."""
    nz, ny, nx = v.shape[1:]
    vp = F.pad(v, (1, 1, 1, 1, 1, 1))
    nb = torch.zeros_like(v)
    for dz, dy, dx in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
        nb = nb + vp[:, dz:dz + nz, dy:dy + ny, dx:dx + nx]
    return (geo.diag * v - nb) * geo.fluid


def loss(p: dict, geo: Geometry, b: torch.Tensor, depth: int) -> torch.Tensor:
    """mean over the batch of ||b - A P(b)|| / ||b|| (loss_one, train.hpp:69-91;
    normalised per right-hand side so every frame weighs the same)."""
    d = net_apply(p, geo, b.float(), depth).double() * geo.fluid
    r = b - poisson(geo, d)
    return (r.flatten(1).norm(dim=1) / b.flatten(1).norm(dim=1)).mean()


def smooth_rhs(geo: Geometry, nb: int, gen: torch.Generator, sweeps: int) -> torch.Tensor:
    """Right-hand sides weighted to the operator's low end (the slow modes of
    CG, like the reference's Ritz-vector datasets, dataset.cpp:34-59): white
    noise on fluid cells smoothed by `sweeps` damped-Jacobi sweeps of A."""
    b = torch.randn((nb,) + geo.shape, generator=gen, device=geo.fluid.device, dtype=torch.float64) * geo.fluid
    inv = torch.where(geo.diag > 0, 1.0 / geo.diag.clamp(min=1), torch.zeros_like(geo.diag))
    for _ in range(sweeps):
        b = b - (2.0 / 3.0) * inv * poisson(geo, b)
    return b / b.flatten(1).norm(dim=1).view(-1, 1, 1, 1)


def train(frames, depth: int, steps: int, lr: float, init: np.ndarray, nb: int, seed: int, device,
          log=print, max_sweeps: int = 40) -> np.ndarray:
    """Adam on the flat parameter vector (adam_update, train.cpp:25-56)."""
    flat = torch.tensor(init, dtype=torch.float32, device=device, requires_grad=True)
    opt = torch.optim.Adam([flat], lr=lr, betas=(0.9, 0.999), eps=1e-8)
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, T_max=max(steps, 1), eta_min=lr * 0.05)
    geos = [Geometry(t, depth, device) for t in frames]
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for step in range(steps):
        geo = geos[step % len(geos)]
        sweeps = int(torch.randint(0, max_sweeps, (1,), generator=gen, device=device).item())
        b = smooth_rhs(geo, nb, gen, sweeps)
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

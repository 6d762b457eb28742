"""Train 3D network weights and measure them in the solve.

    python tools/train3d.py [--depth 5] [--steps 8000] [--n 128] [--big 8] [--ritz-m 300] [--out ...npm]

Training frames are 64^3 free-surface geometries drawn at random (pool levels,
droplets, obstacles, columns, pillars) — not the C3 benchmark frame. The
weights are written as a dim-3 model file (save_npm) and then evaluated by
the CUDA path: PSDO iterations to 1e-6 against the identity-equivalent
weights on C3 at 64^3 and 128^3.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes, train  # noqa: E402
from paper_2310_00177_b200.scenes import AIR, FLUID, SOLID  # noqa: E402


def random_frame(n: int, rng: np.random.Generator) -> np.ndarray:
    c = np.arange(n) + 0.5
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    t = np.full((n, n, n), AIR, np.uint8)
    t[y < rng.uniform(0.15, 0.6) * n] = FLUID  # pool
    for _ in range(rng.integers(0, 3)):  # droplets
        ctr = rng.uniform(0.2, 0.8, 3) * n
        r = rng.uniform(0.05, 0.15) * n
        t[(x - ctr[0]) ** 2 + (y - ctr[1]) ** 2 + (z - ctr[2]) ** 2 < r * r] = FLUID
    if rng.random() < 0.5:  # fluid column
        x1 = rng.uniform(0.2, 0.5) * n
        t[(x < x1) & (y < rng.uniform(0.5, 0.9) * n)] = FLUID
    for _ in range(rng.integers(0, 3)):  # solid obstacles
        lo = rng.uniform(0.1, 0.7, 3) * n
        hi = lo + rng.uniform(0.05, 0.25, 3) * n
        t[(x >= lo[0]) & (x < hi[0]) & (y >= 0) & (y < hi[1]) & (z >= lo[2]) & (z < hi[2])] = SOLID
    t[0], t[-1], t[:, 0], t[:, -1], t[:, :, 0], t[:, :, -1] = SOLID, SOLID, SOLID, SOLID, SOLID, SOLID
    return t


def iterations(types, params, seed, max_iters=20000):
    ctx = b200.Context(3, types.shape, params)
    ctx.set_mask(types)
    b = b200.rhs_normal(seed, types.size)[types.reshape(-1) == 0]
    res = ctx.psdo_solve(b, b200.SolveConfig(max_iters=max_iters))
    return res.report.iterations, res.report.converged, ctx.last_solve_ms


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--frames", type=int, default=48)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--init", default="random", help="random | identity | path of a dim-3 .npm to fine-tune")
    ap.add_argument("--max-sweeps", type=int, default=40, help="RHS smoothing: 0..max damped-Jacobi sweeps")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--big", type=int, default=0, help="extra 2n^3 training frames (scale robustness)")
    ap.add_argument("--eval256", action="store_true")
    ap.add_argument("--ritz-m", type=int, default=0, help="Lanczos steps of the Ritz-vector RHS sets (0: smoothed noise)")
    ap.add_argument("--ritz-every", type=int, default=1, help="Ritz sets on every k-th frame")
    ap.add_argument("--big-only", action="store_true", help="train on the 2n^3 frames only")
    ap.add_argument("--out", default=str(ROOT / "paper_2310_00177_b200" / "weights" / "npsd3d_L6.npm"))
    a = ap.parse_args()
    dev = torch.device("cuda")
    rng = np.random.default_rng(a.seed)
    frames = [random_frame(a.n, rng) for _ in range(a.frames)]
    frames += [random_frame(2 * a.n, rng) for _ in range(a.big)]
    # interleave: every k-th step trains on a large frame
    if a.big:
        small, big = frames[:a.frames], frames[a.frames:]
        k = max(a.frames // a.big, 1)
        frames = []
        for i, f in enumerate(small):
            frames.append(f)
            if i % k == k - 1 and big:
                frames.append(big.pop())
        frames += big
    if a.init == "random":
        init = b200.init_params(a.depth, a.seed).flat
    elif a.init == "identity":
        init = b200.identity_params(a.depth).flat
    else:
        init = b200.load_npm(a.init).flat
    t0 = time.time()
    if a.big_only:
        frames = [f for f in frames if f.shape[0] == 2 * a.n]
    flat = train.train(frames, a.depth, a.steps, a.lr, init, a.batch, a.seed, dev, max_sweeps=a.max_sweeps,
                       ritz_m=a.ritz_m, ritz_every=a.ritz_every)
    wall = time.time() - t0
    params = b200.NetParams(3, a.depth, flat.astype(np.float32))
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    b200.save_npm(params, out)
    report = {"train_seconds": wall, "steps": a.steps, "frames": a.frames, "n": a.n, "big_frames": a.big,
              "big_only": a.big_only, "init": a.init, "lr": a.lr, "batch": a.batch, "max_sweeps": a.max_sweeps,
              "ritz_m": a.ritz_m, "ritz_every": a.ritz_every, "seed": a.seed, "eval": {}}
    ident = b200.identity_params(a.depth)
    evals = [("C3", 64), ("C3", 128), ("C1", 64), ("C2", 128)] + ([("C3", 256)] if a.eval256 else [])
    evals = [(nm, n) for nm, n in evals if n % (1 << a.depth) == 0]
    for name, n in evals:
        t, seed = scenes.config(name, n)
        it_i, _, ms_i = iterations(t, ident, seed)
        it_t, conv_t, ms_t = iterations(t, params, seed)
        report["eval"][f"{name}@{n}"] = {"identity_iters": it_i, "trained_iters": it_t, "trained_converged": conv_t,
                                          "identity_ms": ms_i, "trained_ms": ms_t}
        print(f"{name}@{n}: identity {it_i} it ({ms_i:.1f} ms) | trained {it_t} it ({ms_t:.1f} ms) conv={conv_t}",
              flush=True)
    (out.with_suffix(".json")).write_text(json.dumps(report, indent=1) + "\n")
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main()

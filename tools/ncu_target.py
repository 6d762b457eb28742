"""Direct-launch workload for ncu: kernels inside the solve graph sit under a
conditional WHILE node, which ncu cannot profile, so this runs
Context.profile_iterations (the same kernels launched one by one) on a
benchmark frame.

    python tools/ncu_target.py [--config C3] [--n 256] [--iters 3]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--depth", type=int, default=None, help="default: the default model's depth")
a = ap.parse_args()
types, seed = scenes.config(a.config, a.n)
W = b200.default_model()
if a.depth and a.depth != W.depth:
    W = b200.identity_params(a.depth)
ctx = b200.Context(3, types.shape, W)
ctx.set_mask(types)
bf = scenes.full_rhs(types, seed)
db = b200.DeviceBuffer(ctx, bf.nbytes)
db.upload(bf)
ctx.profile_iterations(db.ptr, b200.SolveConfig(), 1)  # warm-up: module loading, first-touch
prof = ctx.profile_iterations(db.ptr, b200.SolveConfig(), a.iters)
tot = sum(prof.values())
for k, v in prof.items():
    print(f"{k:16s} {v * 1e3:9.1f} us  {100 * v / tot:5.1f}%")
print(f"{'total':16s} {tot * 1e3:9.1f} us")

"""set_mask of one frame, repeated (device time between CUDA events on the
context stream), for timing and for an ncu launch list:
    python tools/setmask_target.py [--config C3] [--n 256] [--reps 5]"""
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
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--depth", type=int, default=None, help="network depth (default: the default model's)")
a = ap.parse_args()
types, _ = scenes.config(a.config, a.n)
depth = a.depth or b200.default_model().depth
ctx = b200.Context(3, types.shape, b200.identity_params(depth))
d = b200.DeviceBuffer(ctx, types.size)
d.upload(types.reshape(-1).copy())
ctx.set_mask_device(d.ptr)
print("n_fluid", ctx.n_fluid)  # finishes the first frame (capacities settle)
ms = []
for i in range(a.reps):
    ctx.event_record(0)
    ctx.set_mask_device(d.ptr)
    ctx.event_record(1)
    ms.append(ctx.event_elapsed_ms(0, 1))
print(f"{a.config} depth {depth} set_mask device ms: {' '.join(f'{m:.3f}' for m in ms)}")

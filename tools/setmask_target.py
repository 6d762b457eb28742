"""set_mask of one frame, twice (the second is the one to read), for an ncu
launch list: python tools/setmask_target.py [--config C3] [--n 256]"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--n", type=int, default=None)
a = ap.parse_args()
types, _ = scenes.config(a.config, a.n)
ctx = b200.Context(3, types.shape, b200.identity_params(4))
d = b200.DeviceBuffer(ctx, types.size)
d.upload(types.reshape(-1).copy())
for i in range(3):
    ctx.synchronize()
    t0 = time.perf_counter()
    ctx.set_mask_device(d.ptr)
    ctx.synchronize()
    print(f"set_mask {1e3 * (time.perf_counter() - t0):.2f} ms")

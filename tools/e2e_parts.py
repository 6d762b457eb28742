"""Where the end-to-end time of one frame goes (host API, pinned buffers)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

t, seed = scenes.config("C3")
W = b200.default_model()
ctx = b200.Context(3, t.shape, W)
n_f = int((t == 0).sum())
pt = b200.PinnedBuffer(ctx, t.size, np.uint8)
pb = b200.PinnedBuffer(ctx, n_f, np.float64)
px = b200.PinnedBuffer(ctx, n_f, np.float64)
pt.array[:] = t.reshape(-1)
pb.array[:] = scenes.full_rhs(t, seed, b200.rhs_normal)[t.reshape(-1) == 0]
cfg = b200.SolveConfig()
for i in range(4):
    t0 = time.perf_counter()
    ctx.set_mask(pt.array)
    t1 = time.perf_counter()
    res = ctx.psdo_solve(pb.array, cfg, out=px.array)
    t2 = time.perf_counter()
    print(f"set_mask {1e3*(t1-t0):.2f} ms  psdo_solve {1e3*(t2-t1):.2f} ms (device solve {ctx.last_solve_ms:.2f})  "
          f"total {1e3*(t2-t0):.2f}")

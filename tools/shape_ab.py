"""Per-kernel iteration time on the same number of cells in differently shaped
grids (plane size 2 MB vs 512 KB of f64): does the z-march slow down with the
plane stride? python tools/shape_ab.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

W = b200.default_model()
for shape in ((512, 512, 512), (2048, 256, 256), (256, 256, 256)):
    t = scenes.random_types(shape, 3, p=(0.45, 0.4, 0.15), blobs=12)
    ctx = b200.Context(3, t.shape, W)
    ctx.set_mask(t)
    bf = np.zeros(t.size)
    bf[t.reshape(-1) == 0] = b200.rhs_normal(1, t.size)[t.reshape(-1) == 0]
    db = b200.DeviceBuffer(ctx, bf.nbytes)
    db.upload(bf)
    ctx.profile_iterations(db.ptr, b200.SolveConfig(), 1)
    prof = ctx.profile_iterations(db.ptr, b200.SolveConfig(), 3)
    nf = int((t == 0).sum())
    print(shape, "n_fluid", nf, " ".join(f"{k}={v * 1e3:.0f}us({v * 1e9 / nf:.1f}ps/cell)" for k, v in prof.items()
                                        if k in ("ortho", "update", "net_down_L0", "net_up_L0")), flush=True)
    ctx.close()

"""Per-iteration device time of the solve graph with and without programmatic
dependent launch (NPSD_PDL, read at context creation) on C1/C2/C3:
    python tools/pdl_ab.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

W = b200.load_npm(ROOT / "paper_2310_00177_b200" / "weights" / "npsd3d_L4.npm")
for name in ("C1", "C2", "C3"):
    t, seed = scenes.config(name)
    b = b200.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    for pdl in ("0", "1"):
        os.environ["NPSD_PDL"] = pdl
        ctx = b200.Context(3, t.shape, W)
        ctx.set_mask(t)
        ms = []
        for i in range(6):
            rep = ctx.psdo_solve(b, b200.SolveConfig(max_iters=2000)).report
            if i:
                ms.append(ctx.last_solve_ms / rep.iterations)
        print(f"{name} pdl={pdl} iters={rep.iterations} per-iter {np.median(ms) * 1e3:.1f} us", flush=True)
        ctx.close()

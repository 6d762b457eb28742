"""Per-iteration device time of the solve graph under a context-creation
environment switch (NPSD_PDL, NPSD_PDL_MASK, NPSD_COARSE_SKIP, ...) on C1/C2/C3:
    python tools/env_ab.py [VAR] [values...]   (default: NPSD_PDL 0 1)"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2310_00177_b200 as b200  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

W = b200.default_model()
for name in ("C1", "C2", "C3"):
    t, seed = scenes.config(name)
    b = b200.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    var = sys.argv[1] if len(sys.argv) > 1 else "NPSD_PDL"
    for pdl in (sys.argv[2:] or ["0", "1"]):
        os.environ[var] = pdl
        ctx = b200.Context(3, t.shape, W)
        ctx.set_mask(t)
        ms = []
        for i in range(6):
            rep = ctx.psdo_solve(b, b200.SolveConfig(max_iters=2000)).report
            if i:
                ms.append(ctx.last_solve_ms / rep.iterations)
        print(f"{name} {var}={pdl} iters={rep.iterations} per-iter {np.median(ms) * 1e3:.1f} us", flush=True)
        ctx.close()

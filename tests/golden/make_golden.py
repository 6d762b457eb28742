"""Generates tests/golden/ref2d.npz from the REAL reference (oracle/_ref, built
from /root/reference sources): 2D network outputs, linear-block coefficients,
NeuralPrecond outputs, reduced spmv and PSDO residual histories on seeded
inputs. tests/test_golden.py checks the CPU oracle against them bitwise, so the
oracle stays pinned on machines where the reference cannot be built.

    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle_lib import Ref  # noqa: E402
from paper_2310_00177_b200.scenes import random_types  # noqa: E402

ref = Ref()
out = {}
cases = [("a", (32, 32), 3, 11), ("b", (16, 48), 2, 12), ("c", (64, 64), 4, 13), ("d", (24, 40), 3, 14)]
for tag, shape, depth, seed in cases:
    t = random_types(shape, 1000 + seed)
    p = ref.init_params_2d(depth, 2000 + seed)
    x = np.random.default_rng(seed).standard_normal(shape).astype(np.float32)
    y, za, zb = ref.net_apply_2d(t, p, depth, x)
    nf = int((t == 0).sum())
    r = np.random.default_rng(100 + seed).standard_normal(nf)
    z = ref.precond_apply_2d(t, p, depth, r)
    ax = ref.spmv(t, r)
    b = ref.rhs_normal(3000 + seed, nf)
    h = ref.psdo_solve(t, b, mode="neural", params=p, depth=depth, max_iters=12, tol_reduction=1e-300)
    out.update({f"{tag}_types": t, f"{tag}_params": p, f"{tag}_depth": np.int64(depth), f"{tag}_x": x, f"{tag}_y": y,
                f"{tag}_za": za, f"{tag}_zb": zb, f"{tag}_r": r, f"{tag}_z": z, f"{tag}_ax": ax, f"{tag}_b": b,
                f"{tag}_hist": h["residual_history"], f"{tag}_xsol": h["x"]})
# 3D operator fixture (the reference assembles 3D too)
t3 = random_types((8, 12, 16), 77)
nf3 = int((t3 == 0).sum())
v3 = np.random.default_rng(78).standard_normal(nf3)
out["op3_types"], out["op3_x"], out["op3_ax"] = t3, v3, ref.spmv(t3, v3)
b3 = ref.rhs_normal(79, nf3)
h3 = ref.psdo_solve(t3, b3, mode="identity", max_iters=400)
out["op3_b"], out["op3_hist"] = b3, h3["residual_history"]
out["rng_1234"] = ref.rhs_normal(1234, 64)
out["init_d3_s42"] = ref.init_params_2d(3, 42)
np.savez_compressed(ROOT / "tests" / "golden" / "ref2d.npz", **out)
print("wrote", ROOT / "tests" / "golden" / "ref2d.npz", len(out), "arrays")

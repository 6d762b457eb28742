"""Generates tests/golden/iteration_counts.json: iterations to rel-res 1e-6 of the
REFERENCE psdo_solve (oracle/_ref: solver.cpp:189-276 on assemble_poisson_3d +
reduce, IdentityPrecond — what identity-equivalent network weights reduce to,
SURVEY.md §0.4) on the benchmark domains. bench.py's --impl reference arm uses
the count to turn its bounded per-iteration sample into a time-to-solution.
Run here (needs oracle/_ref); takes minutes at 256^3.

With --trained: the reference psdo_solve with the 3D network restatement
(NeuralPrecond3D) as its preconditioner and the committed trained weights
(paper_2310_00177_b200.DEFAULT_MODEL), entries "<name>_trained"."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle_lib import Ref  # noqa: E402
from paper_2310_00177_b200 import scenes  # noqa: E402

out = ROOT / "tests" / "golden" / "iteration_counts.json"
res = json.loads(out.read_text()) if out.exists() else {}
ref = Ref()
args = [a for a in sys.argv[1:] if a != "--trained"]
trained = "--trained" in sys.argv
if trained:
    import paper_2310_00177_b200 as b200

    W = b200.default_model()

def frames(name):
    """(key suffix, types, seed) per solve: one for C1/C2/C3/C5, 32 for C4
    (droplet frames at 128^3, RHS seed 2000+f)."""
    if name == "C4":
        for f, t in enumerate(scenes.droplet_frames(128, 32)):
            yield f"_f{f:02d}", t, 2000 + f
    else:
        t, seed = scenes.config(name)
        yield "", t, seed


todo = [(name, suf, t, seed) for name in (args or ["C1", "C2", "C3"]) for suf, t, seed in frames(name)]
for name, suf, t, seed in todo:
    b = ref.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    t0 = time.time()
    if trained:
        r = ref.psdo_solve(t, b, mode="neural", params=W.flat, depth=W.depth, max_iters=20000, tol_reduction=1e-6,
                           n_ortho=2)
        key, solver = f"{name}{suf}_trained", ("reference psdo_solve + NeuralPrecond3D (restatement) with "
                                          f"weights/{b200.DEFAULT_MODEL.name} (depth {W.depth}), n_ortho=2, tol 1e-6")
    else:
        r = ref.psdo_solve(t, b, mode="identity", max_iters=20000, tol_reduction=1e-6, n_ortho=2)
        key, solver = name + suf, "reference psdo_solve + IdentityPrecond, n_ortho=2, tol 1e-6"
    res[key] = {"n": int(t.shape[0]), "n_fluid": int(b.size), "iterations": r["iterations"],
                "converged": r["converged"], "final_rel_res": float(r["residual_history"][-1] / r["residual_history"][0]),
                "solver": solver, "cpu_seconds": time.time() - t0}
    print(key, res[key], flush=True)
    out.write_text(json.dumps(res, indent=1) + "\n")

"""run_bench (bench.cpp:35-137) on the device path: every method token per
system, nullspace_projection = is_pure_neumann(frame) (bench.cpp:52), rows.csv
/ traces / summary.csv / speedup_hist.csv written and read back by the
reference's own load_bench_rows (byte-identical round trip)."""
import csv

import numpy as np
import pytest

from paper_2310_00177_b200 import bench_matrix as bm
from paper_2310_00177_b200 import scenes

pytestmark = pytest.mark.gpu

METHODS = ["cg", "pcg+none", "pcg+jacobi", "pcg+ic0", "psd+none", "psdo+none", "psdo+jacobi", "psdo+neural",
           "fpcg+none", "psdo+ic0"]


def test_run_bench_rows_csv(b200, oracle, ref, tmp_path):
    t1, s1 = scenes.config("C1", 32)
    box = np.zeros((16, 16, 16), np.uint8)  # all fluid, closed: pure Neumann
    systems = {"C1_32": (t1, oracle.rhs_normal(s1, t1.size)[t1.reshape(-1) == 0]),
               "box_16": (box, oracle.rhs_normal(5, box.size))}
    # a harness test on small grids: the depth-4 model (32^3 and 16^3 hold whole depth-4 coarsest cells)
    model = b200.load_npm(b200.DEFAULT_MODEL.parent / "npsd3d_L4.npm")
    rows = bm.run_bench(systems, METHODS, bm.BenchConfig(max_iters=3000), model=model)
    bm.write_bench_outputs(rows, tmp_path / "out")
    bm.write_bench_report(rows, tmp_path / "out")
    by = {(r.system, r.method): r for r in rows}
    for name in systems:
        for m in METHODS:
            r = by[(name, m)]
            if m in ("fpcg+none", "psdo+ic0"):
                assert "not available" in r.error
                continue
            assert r.error == "", (name, m, r.error)
            assert r.total_seconds > 0 and r.setup_seconds > 0
            if m.startswith("psd+") or (name == "box_16" and m.endswith("+neural")):
                # steepest descent, and the free-surface-trained network on a
                # closed box: no convergence promised within the budget
                continue
            assert r.converged, (name, m)
            assert r.final_rel_residual <= 1e-6
            if m.startswith("psdo"):
                assert 0 < r.precond_seconds < r.iterate_seconds
    # psdo+none is the reference psdo_solve with IdentityPrecond; cg is cg_solve
    want = ref.psdo_solve(t1, systems["C1_32"][1], mode="identity", max_iters=3000)
    assert abs(by[("C1_32", "psdo+none")].iterations - want["iterations"]) <= 1
    want_psd = ref.psdo_solve(t1, systems["C1_32"][1], mode="identity", n_ortho=0, max_iters=30, tol_reduction=1e-300)
    h, w = np.array(by[("C1_32", "psd+none")].residual_history[:31]), want_psd["residual_history"]
    assert np.max(np.abs(h - w) / w) <= 1e-9
    want_cg = ref.pcg_solve(t1, systems["C1_32"][1], precond=0, max_iters=3000)
    assert abs(by[("C1_32", "cg")].iterations - want_cg["iterations"]) <= 1
    # the pure-Neumann box converged only because its solves projected
    want_ns = ref.pcg_solve(box, systems["box_16"][1], precond=0, max_iters=3000, nullspace_projection=True)
    assert abs(by[("box_16", "cg")].iterations - want_ns["iterations"]) <= 1
    # the reference's reader and writers reproduce our rows.csv byte for byte;
    # its report from the parsed rows equals ours from the same parsed rows
    # (the means of 9-decimal values, like its round trip)
    ref.bench_roundtrip(tmp_path / "out" / "rows.csv", tmp_path / "theirs")
    assert (tmp_path / "out" / "rows.csv").read_bytes() == (tmp_path / "theirs" / "rows.csv").read_bytes()
    bm.write_bench_report(bm.load_bench_rows(tmp_path / "out" / "rows.csv"), tmp_path / "parsed")
    for f in ("summary.csv", "speedup_hist.csv"):
        assert (tmp_path / "parsed" / f).read_bytes() == (tmp_path / "theirs" / f).read_bytes(), f
    with open(tmp_path / "out" / "rows.csv") as f:
        assert len(list(csv.DictReader(f))) == len(systems) * len(METHODS)
    assert (tmp_path / "out" / "traces" / "C1_32__psdo_neural.csv").exists()

"""The drop-in check from the reference's side, on the GPU: tests/cpp/dropin.cpp
(built by oracle/Makefile against the unmodified reference objects and
include/npsd_b200.hpp) swaps in npsd::b200::neural_precond inside the
reference's own psdo_solve, and runs npsd::b200::psdo_solve."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
EXE = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "dropin"


def test_reference_program_with_b200_preconditioner():
    if not EXE.exists():
        pytest.skip("oracle/_ref/dropin not built (needs the reference headers)")
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=300, check=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["precond_rel_l2"] <= 1e-5
    assert r["budget_hist_max_rel"] <= 1e-6
    assert r["ref_converged"] and r["b200_converged"]
    assert abs(r["ref_iters"] - r["b200_iters"]) <= 1
    assert r["invalid_argument_rethrown"] == 1
    # IdentityPrecond through the device loop (no network) vs the reference's
    assert abs(r["ident_ref_iters"] - r["ident_b200_iters"]) <= 1
    assert r["ident_hist_max_rel"] <= 1e-8
    # A is validated against the flag-derived operator
    assert r["scaled_a_rejected"] == 1 and r["moved_a_rejected"] == 1
    assert r["full_check_iters"] == r["b200_iters"]
    # SolveReport timing fields (solver.cpp:211-212, 237, 275)
    assert r["setup_seconds"] > 0 and r["precond_seconds"] > 0
    assert r["precond_seconds"] < r["iterate_seconds"]
    assert r["cum0"] == r["setup_seconds"] and r["cum_last"] >= r["cum0"]
    # is_pure_neumann (discretization.cpp:180-191)
    assert r["pure_neumann_frame"] == r["pure_neumann_frame_ref"] == 0
    assert r["pure_neumann_box"] == r["pure_neumann_box_ref"] == 1

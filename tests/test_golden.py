"""The CPU oracle against golden vectors generated from the real reference
(tests/golden/make_golden.py): bitwise. CPU only; needs no reference build."""
from pathlib import Path

import numpy as np
import pytest

G = np.load(Path(__file__).resolve().parent / "golden" / "ref2d.npz")
TAGS = ["a", "b", "c", "d"]


@pytest.mark.parametrize("tag", TAGS)
def test_net_apply_matches_reference_golden(oracle, tag):
    t, p, depth = G[f"{tag}_types"], G[f"{tag}_params"], int(G[f"{tag}_depth"])
    ctx = oracle.context(t, p, depth)
    y = ctx.net_apply(G[f"{tag}_x"])
    assert np.array_equal(y.view(np.uint32), G[f"{tag}_y"].view(np.uint32))
    za, zb = ctx.z()
    assert np.array_equal(za, G[f"{tag}_za"]) and np.array_equal(zb, G[f"{tag}_zb"])


@pytest.mark.parametrize("tag", TAGS)
def test_precond_and_operator_match_reference_golden(oracle, tag):
    t, p, depth = G[f"{tag}_types"], G[f"{tag}_params"], int(G[f"{tag}_depth"])
    ctx = oracle.context(t, p, depth)
    assert np.array_equal(ctx.precond_apply(G[f"{tag}_r"]), G[f"{tag}_z"])
    assert np.array_equal(ctx.spmv(G[f"{tag}_r"]), G[f"{tag}_ax"])


@pytest.mark.parametrize("tag", TAGS)
def test_psdo_history_matches_reference_golden(oracle, tag):
    t, p, depth = G[f"{tag}_types"], G[f"{tag}_params"], int(G[f"{tag}_depth"])
    ctx = oracle.context(t, p, depth)
    res = ctx.psdo_solve(G[f"{tag}_b"], max_iters=12, tol_reduction=1e-300)
    assert np.array_equal(res["residual_history"], G[f"{tag}_hist"])
    assert np.array_equal(res["x"], G[f"{tag}_xsol"])


def test_3d_operator_and_solver_match_reference_golden(oracle):
    t = G["op3_types"]
    ctx = oracle.context(t, oracle.identity_params(3, 1), 1)
    assert np.array_equal(ctx.spmv(G["op3_x"]), G["op3_ax"])
    res = ctx.psdo_solve(G["op3_b"], identity=True, max_iters=400)
    assert np.array_equal(res["residual_history"], G["op3_hist"])


def test_rng_and_init_params_match_reference_golden(oracle):
    assert np.array_equal(oracle.rhs_normal(1234, 64), G["rng_1234"])
    assert np.array_equal(oracle.init_params(2, 3, 42).view(np.uint32), G["init_d3_s42"].view(np.uint32))

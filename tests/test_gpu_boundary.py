"""The drop-in boundary's remaining reference behaviours on the GPU:
is_pure_neumann (discretization.cpp:180-191), IdentityPrecond inside the
device PSDO loop (precond.cpp:7-10), the check of a caller's A against the
flag-derived operator, nullspace projection in pcg_solve (solver.cpp:45-48,82)
and on z-slabs, and the SolveReport timing fields (solver.cpp:211-212,237,275)."""
import threading

import numpy as np
import pytest

from oracle_lib import reduced_csr as csr_of
from paper_2310_00177_b200 import scenes

pytestmark = pytest.mark.gpu


def test_is_pure_neumann(b200):
    p = b200.identity_params(2)
    cases = [(scenes.config("C1", 32)[0], False), (np.zeros((16, 16, 16), np.uint8), True)]
    box = np.full((16, 16, 16), 2, np.uint8)
    box[2:8, 2:8, 2:8] = 0      # fluid enclosed by solid ...
    box[10:14, 10:14, 10:14] = 1  # ... and air elsewhere, not touching it
    cases.append((box, True))
    box2 = box.copy()
    box2[8, 4, 4] = 1  # one air cell on the fluid's face
    cases.append((box2, False))
    for t, want in cases:
        ctx = b200.Context(3, t.shape, p)
        ctx.set_mask(t)
        assert ctx.is_pure_neumann() is want


def test_psdo_identity_precond_vs_reference(b200, oracle, ref):
    """PSDO with IdentityPrecond (no network) in the device loop against the
    reference psdo_solve with its IdentityPrecond on the reference assembly."""
    for name, n in (("C1", 32), ("C2", 32), ("C3", 48)):
        t, seed = scenes.config(name, n)
        b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
        P = b200.IdentityPrecond(t)
        got = b200.psdo_solve(csr_of_obj(t), b, P, b200.SolveConfig(max_iters=3000))
        want = ref.psdo_solve(t, b, mode="identity", max_iters=3000)
        assert got.report.converged and want["converged"]
        assert abs(got.report.iterations - want["iterations"]) <= 1
        h, w = got.report.residual_history, want["residual_history"]
        assert np.max(np.abs(h[:30] - w[:30]) / w[:30]) <= 1e-9
        assert got.report.method == "psdo+identity"


class _Csr:
    def __init__(self, ro, ci, va):
        self.row_offsets, self.col_indices, self.values = ro, ci, va
        self.n_rows = ro.size - 1


def csr_of_obj(t):
    return _Csr(*csr_of(t))


def test_operator_check(b200, oracle):
    t, seed = scenes.config("C2", 32)
    P = b200.NeuralPrecond(b200.identity_params(4), t)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    ro, ci, va = csr_of(t)
    cfg = b200.SolveConfig(max_iters=2000)
    ok = b200.psdo_solve(_Csr(ro, ci, va), b, P, cfg, check_a="full")
    assert ok.report.converged
    with pytest.raises(ValueError, match="diagonal"):
        b200.psdo_solve(_Csr(ro, ci, 2.0 * va), b, P, cfg)
    ci2 = ci.copy()
    k = int(np.nonzero(ci2 != np.repeat(np.arange(ro.size - 1), np.diff(ro)))[0][0])
    ci2[k] = (ci2[k] + 7) % (ro.size - 1)  # same pattern sizes, one wrong neighbour
    with pytest.raises(ValueError):
        b200.psdo_solve(_Csr(ro, ci2, va), b, P, cfg, check_a="full")
    other = scenes.config("C3", 32)[0]
    with pytest.raises(ValueError):
        b200.psdo_solve(csr_of_obj(other), b, P, cfg)


@pytest.mark.parametrize("precond", ["identity", "jacobi"])
def test_pcg_nullspace_vs_reference(b200, oracle, ref, precond):
    """pcg_solve with nullspace projection (solver.cpp:45-48, 82) on a
    pure-Neumann domain (an all-fluid closed box: singular system)."""
    t = np.zeros((16, 16, 16), np.uint8)
    t[:, :, :3] = 2  # a solid wall block: still pure Neumann
    b = oracle.rhs_normal(31, t.size)[t.reshape(-1) == 0]
    want = ref.pcg_solve(t, b, precond={"identity": 0, "jacobi": 1}[precond], max_iters=2000,
                         nullspace_projection=True)
    ctx = b200.Context(3, t.shape, b200.identity_params(2))
    ctx.set_mask(t)
    assert ctx.is_pure_neumann()
    got = ctx.pcg_solve(b, b200.SolveConfig(max_iters=2000, nullspace_projection=True), precond=precond)
    assert got.report.converged and want["converged"]
    assert abs(got.report.iterations - want["iterations"]) <= 1
    h, w = got.report.residual_history, want["residual_history"]
    assert np.max(np.abs(h[:20] - w[:20]) / w[:20]) <= 1e-9
    err = np.linalg.norm(got.x - want["x"]) / np.linalg.norm(want["x"])
    assert err <= 1e-6


def test_solve_report_timing_fields(b200, oracle):
    """setup_seconds (r0 and its norm), cumulative_seconds[0] = setup,
    precond_seconds accumulated over the network spans, iterate_seconds =
    total - setup (solver.cpp:211-212, 237, 275)."""
    t, seed = scenes.config("C3", 64)
    ctx = b200.Context(3, t.shape, b200.init_params(4, 42))
    ctx.set_mask(t)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    rep = ctx.psdo_solve(b, b200.SolveConfig(max_iters=20, tol_reduction=1e-30)).report
    secs = rep.cumulative_seconds
    assert rep.iterations == 20 and secs.size == 21
    assert rep.setup_seconds > 0 and secs[0] == rep.setup_seconds
    assert np.all(np.diff(secs) > 0)
    assert 0 < rep.precond_seconds < rep.iterate_seconds
    assert rep.iterate_seconds <= secs[-1] + 1e-3
    rep_c = ctx.pcg_solve(b, b200.SolveConfig(max_iters=20, tol_reduction=1e-30), precond="ic0").report
    assert rep_c.setup_seconds > 0 and rep_c.cumulative_seconds[0] == rep_c.setup_seconds
    assert 0 < rep_c.precond_seconds < rep_c.iterate_seconds


def test_slab_nullspace_projection(b200, oracle):
    """mean projection over all ranks' fluid cells on a z-slab decomposition
    (2 in-process ranks) against the single-domain solve."""
    t = np.zeros((32, 16, 16), np.uint8)
    t[:, :2, :] = 2
    P = b200.identity_params(3)
    b = oracle.rhs_normal(41, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=2000, nullspace_projection=True)
    single = b200.Context(3, t.shape, P)
    single.set_mask(t)
    want = single.psdo_solve(b, cfg)
    parts = b200.partition(t.shape[0], 2, 3)
    counts = [int((t[z0:z0 + k] == 0).sum()) for z0, k in parts]
    offs = np.concatenate([[0], np.cumsum(counts)])
    comm = b200.Comm.local(2)
    out, errs = [None, None], []

    def rank(r):
        try:
            z0, k = parts[r]
            ctx = b200.Context.slab(comm, r, t.shape, z0, k, P)
            ctx.set_mask(t[z0:z0 + k])
            out[r] = (ctx.is_pure_neumann(), ctx.psdo_solve(b[offs[r]:offs[r + 1]], cfg))
            ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for th in ts:
        th.start()
    for th in ts:
        th.join(300)
    comm.close()
    if errs:
        raise errs[0]
    assert out[0][0] and out[1][0]
    for _, res in out:
        assert res.report.converged
        assert abs(res.report.iterations - want.report.iterations) <= 1
    x = np.concatenate([res.x for _, res in out])
    assert np.linalg.norm(x - want.x) / np.linalg.norm(want.x) <= 1e-5

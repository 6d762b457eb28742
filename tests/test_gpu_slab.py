"""z-slab decomposition on one GPU: n in-process ranks (host threads, the
local communicator) against a single-domain context on the same frame. The
per-rank code path is the NCCL ranks' (only the communicator differs)."""
import threading

import numpy as np
import pytest

from paper_2310_00177_b200 import scenes

pytestmark = pytest.mark.gpu


def run_ranks(fn, n):
    out, errs = [None] * n, []

    def work(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    if errs:
        raise errs[0]
    return out


def split(t, parts, v):
    """the owned fluid cells of each slab are a contiguous run of the reduced vector"""
    counts = [int((t[z0:z0 + k] == 0).sum()) for z0, k in parts]
    offs = np.concatenate([[0], np.cumsum(counts)])
    return [v[offs[r]:offs[r + 1]] for r in range(len(parts))], counts


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,name", [(2, "C3"), (4, "C2")])
def test_slab_identity_solve_matches_single_domain(b200, oracle, n, name):
    t, seed = scenes.config(name, 64)
    P = b200.identity_params(4)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=2000)
    single = b200.Context(3, t.shape, P)
    single.set_mask(t)
    ref = single.psdo_solve(b, cfg)
    parts = b200.partition(t.shape[0], n, 4)
    bs, counts = split(t, parts, b)
    comm = b200.Comm.local(n)

    def rank(r):
        z0, k = parts[r]
        ctx = b200.Context.slab(comm, r, t.shape, z0, k, P)
        ctx.set_mask(t[z0:z0 + k])
        assert ctx.n_fluid == counts[r]
        res = ctx.psdo_solve(bs[r], cfg)
        return res, ctx.fluid_indices()

    out = run_ranks(rank, n)
    hists = [o[0].report.residual_history for o in out]
    for h in hists[1:]:  # identical solver state on every rank
        assert np.array_equal(h, hists[0])
    assert all(o[0].report.converged for o in out)
    assert abs(out[0][0].report.iterations - ref.report.iterations) <= 1
    # the dot products sum in another order (per-rank partials, rank order):
    # the histories agree to ~1e-14 at first and drift the way CG rounding
    # does; the reference's own bar is the iteration count (+-1)
    h0, hr = hists[0], ref.report.residual_history
    assert np.max(np.abs(h0[:50] - hr[:50]) / hr[:50]) <= 1e-7
    m = min(len(h0), len(hr)) - 1
    assert np.max(np.abs(h0[:m] - hr[:m]) / hr[:m]) <= 1e-3
    x = np.concatenate([o[0].x for o in out])
    assert rel(x, ref.x) <= 1e-5
    assert np.array_equal(np.concatenate([o[1] for o in out]), single.fluid_indices())


@pytest.mark.parametrize("n", [2, 4])
def test_slab_random_weights_precond_and_history(b200, oracle, n):
    t, seed = scenes.config("C3", 64)
    P = b200.init_params(4, 8)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    single = b200.Context(3, t.shape, P)
    single.set_mask(t)
    r = np.random.default_rng(3).standard_normal(single.n_fluid)
    z_ref = single.precond_apply(r)
    cfg = b200.SolveConfig(max_iters=20, tol_reduction=1e-300)
    h_ref = single.psdo_solve(b, cfg).report.residual_history
    parts = b200.partition(t.shape[0], n, 4)
    rs, _ = split(t, parts, r)
    bs, _ = split(t, parts, b)
    comm = b200.Comm.local(n)

    def rank(k):
        z0, nk = parts[k]
        ctx = b200.Context.slab(comm, k, t.shape, z0, nk, P)
        ctx.set_mask(t[z0:z0 + nk])
        z = ctx.precond_apply(rs[k])
        h = ctx.psdo_solve(bs[k], cfg).report.residual_history
        return z, h

    out = run_ranks(rank, n)
    assert rel(np.concatenate([o[0] for o in out]), z_ref) <= 1e-5
    assert np.max(np.abs(out[0][1] - h_ref) / h_ref) <= 1e-6
    for o in out[1:]:
        assert np.array_equal(o[1], out[0][1])


def test_slab_frames_and_errors(b200, oracle):
    """per-frame set_mask on slabs (C4 pattern) and the argument checks"""
    P = b200.init_params(4, 2)
    comm = b200.Comm.local(2)
    with pytest.raises(ValueError, match="multiples"):
        b200.Context.slab(comm, 0, (64, 64, 64), 4, 28, P)
    with pytest.raises(ValueError, match="rank"):
        b200.Context.slab(comm, 2, (64, 64, 64), 0, 32, P)
    frames = list(scenes.droplet_frames(64, 3))
    parts = b200.partition(64, 2, 4)

    def rank(k):
        z0, nk = parts[k]
        ctx = b200.Context.slab(comm, k, (64, 64, 64), z0, nk, P)
        res = []
        for t in frames:
            ctx.set_mask(t[z0:z0 + nk])
            r = np.random.default_rng(7).standard_normal(int((t == 0).sum()))
            rk, _ = split(t, parts, r)
            res.append(ctx.precond_apply(rk[k]))
        return res

    out = run_ranks(rank, 2)
    for f, t in enumerate(frames):
        single = b200.Context(3, t.shape, P)
        single.set_mask(t)
        r = np.random.default_rng(7).standard_normal(single.n_fluid)
        assert rel(np.concatenate([out[0][f], out[1][f]]), single.precond_apply(r)) <= 1e-5


def test_slab_nccl_one_rank_graph_path(b200, oracle):
    """The NCCL communicator for real (one rank): dlopen, init, the captured
    chunk graph with NCCL collectives inside, and the device-buffer API on the
    owned planes, against the single-domain context."""
    try:
        uid = b200.Comm.nccl_unique_id()
    except b200.DeviceError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    comm = b200.Comm.nccl(uid, 0, 1, 0)
    t, seed = scenes.config("C3", 64)
    P = b200.init_params(4, 8)
    single = b200.Context(3, t.shape, P)
    single.set_mask(t)
    ctx = b200.Context.slab(comm, 0, t.shape, 0, t.shape[0], P)
    ctx.set_mask(t)
    r = np.random.default_rng(1).standard_normal(single.n_fluid)
    assert rel(ctx.precond_apply(r), single.precond_apply(r)) <= 1e-5
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=40, tol_reduction=1e-300)
    h_ref = single.psdo_solve(b, cfg).report.residual_history
    for _ in range(2):  # second solve replays the cached chunk graph
        h = ctx.psdo_solve(b, cfg).report.residual_history
        assert ctx.slab_graph  # NCCL inside the captured chunk graph, not the eager fallback
        assert len(h) == len(h_ref)
        assert np.max(np.abs(h - h_ref) / h_ref) <= 1e-6
    # device API with identity weights: owned-plane buffers in and out
    ident = b200.Context.slab(comm, 0, t.shape, 0, t.shape[0], b200.identity_params(4))
    bfull = scenes.full_rhs(t, seed, oracle.rhs_normal)
    db, dx, dt = (b200.DeviceBuffer(ident, bfull.nbytes), b200.DeviceBuffer(ident, bfull.nbytes),
                  b200.DeviceBuffer(ident, t.size))
    db.upload(bfull)
    dt.upload(np.ascontiguousarray(t.reshape(-1)))
    ident.set_mask_device(dt.ptr)
    rep = ident.psdo_solve_device(db.ptr, dx.ptr, b200.SolveConfig(max_iters=2000))
    xf = np.empty_like(bfull)
    dx.download(xf)
    ident.synchronize()
    one = b200.Context(3, t.shape, b200.identity_params(4))
    one.set_mask(t)
    ref = one.psdo_solve(bfull[t.reshape(-1) == 0], b200.SolveConfig(max_iters=2000))
    assert rep.converged and abs(rep.iterations - ref.report.iterations) <= 1
    assert rel(xf[t.reshape(-1) == 0], ref.x) <= 1e-5
    for buf in (db, dx, dt):
        buf.free()

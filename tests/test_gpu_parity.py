"""GPU parity: the B200 path (through the C ABI) against the CPU oracle and the
reference build, on identical seeded inputs.

Bars (north_star): flag/mask coarsening bit-exact; network / preconditioner
output within 1e-5 relative L2 — in the default (fast) network arithmetic, and
bitwise in the exact mode (Context(exact=True): the reference's operation
order), asserted for both; iteration count to rel-res 1e-6 within +-1 of
the reference psdo_solve; residual history over a fixed budget within 1e-6
relative (random weights)."""
import numpy as np
import pytest

from paper_2310_00177_b200 import scenes

pytestmark = pytest.mark.gpu

REL_L2 = 1e-5  # preconditioner output tolerance (north_star)


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make(b200, oracle, types, depth, params, exact=True):
    dim = types.ndim
    P = b200.NetParams(dim, depth, params)
    ctx = b200.Context(dim, types.shape, P, exact=exact)
    ctx.set_mask(types)
    octx = oracle.context(types, params, depth)
    return ctx, octx


CASES = [
    ((16, 16, 16), 1, 0), ((16, 16, 16), 2, 1), ((16, 16, 16), 3, 2), ((32, 32, 32), 4, 3),
    ((16, 32, 48), 3, 4), ((32, 32), 3, 5), ((64, 32), 4, 6), ((16, 16), 1, 7),
]


@pytest.mark.parametrize("shape,depth,seed", CASES)
def test_level_images_and_z_bitexact(b200, oracle, shape, depth, seed):
    t = scenes.random_types(shape, 10 + seed)
    p = oracle.init_params(len(shape), depth, 20 + seed)
    ctx, octx = make(b200, oracle, t, depth, p)
    for l, want in enumerate(oracle.level_images(t, depth)):
        got = ctx.level_image(l)
        assert np.array_equal(got, want), f"level {l}"
    za, zb = ctx.linear_coeffs()
    oza, ozb = octx.z()
    assert np.array_equal(za, oza) and np.array_equal(zb, ozb)
    assert np.array_equal(ctx.fluid_indices(), octx.fluid_indices())


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("shape,depth,seed", CASES)
def test_net_apply_bitwise(b200, oracle, shape, depth, seed, exact):
    t = scenes.random_types(shape, 30 + seed)
    p = oracle.init_params(len(shape), depth, 40 + seed)
    ctx, octx = make(b200, oracle, t, depth, p, exact)
    x = np.random.default_rng(seed).standard_normal(shape).astype(np.float32)
    got = ctx.net_apply(x)
    want = octx.net_apply(x)
    assert rel_l2(got, want) <= REL_L2
    if exact:
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.ref
@pytest.mark.parametrize("shape,depth,seed", [((32, 32), 3, 0), ((64, 64), 4, 1), ((16, 48), 2, 2)])
def test_net_apply_2d_vs_reference_bitwise(b200, oracle, ref, shape, depth, seed):
    t = scenes.random_types(shape, 50 + seed)
    p = oracle.init_params(2, depth, 60 + seed)
    ctx, _ = make(b200, oracle, t, depth, p)
    x = np.random.default_rng(seed).standard_normal(shape).astype(np.float32)
    want, _, _ = ref.net_apply_2d(t, p, depth, x)
    assert np.array_equal(ctx.net_apply(x).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("shape,depth,seed", CASES)
def test_precond_apply(b200, oracle, shape, depth, seed, exact):
    t = scenes.random_types(shape, 70 + seed)
    p = oracle.init_params(len(shape), depth, 80 + seed)
    ctx, octx = make(b200, oracle, t, depth, p, exact)
    r = np.random.default_rng(seed).standard_normal(ctx.n_fluid)
    err = rel_l2(ctx.precond_apply(r), octx.precond_apply(r))
    assert err <= REL_L2
    if exact:
        assert err <= 1e-12  # bit-identical f32 network; f64 norm rounding only
    assert np.all(ctx.precond_apply(np.zeros_like(r)) == 0.0)  # test_neural.cpp:258-261


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("shape,depth,seed", [((64, 64, 128), 4, 0), ((48, 96, 64), 3, 1)])
def test_precond_apply_interior_tiles(b200, oracle, shape, depth, seed, exact):
    """Grids large enough that tiles have interior halos on every side (the
    small cases above are all-boundary tiles)."""
    t = scenes.random_types(shape, 170 + seed, p=(0.6, 0.3, 0.1), blobs=6)
    p = oracle.init_params(3, depth, 180 + seed)
    ctx, octx = make(b200, oracle, t, depth, p, exact)
    r = np.random.default_rng(seed).standard_normal(ctx.n_fluid)
    z = ctx.precond_apply(r)
    assert np.all(np.isfinite(z))
    err = rel_l2(z, octx.precond_apply(r))
    assert err <= REL_L2
    # exact: the f32 network of the solve path is bit-identical to the
    # restatement; only the f64 residual norm (tree vs serial sum) differs,
    # ~1e-16; a single f32 ulp at one cell would show as ~1e-10
    if exact:
        assert err <= 1e-12


def test_psdo_history_c3_64_random_weights(b200, oracle):
    t, seed = scenes.config("C3", 64)
    p = oracle.init_params(3, 4, 9)
    ctx, octx = make(b200, oracle, t, 4, p)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    got = ctx.psdo_solve(b, b200.SolveConfig(max_iters=20, tol_reduction=1e-300))
    want = octx.psdo_solve(b, max_iters=20, tol_reduction=1e-300)
    h, w = got.report.residual_history, want["residual_history"]
    assert np.max(np.abs(h - w) / w) <= 1e-6


@pytest.mark.parametrize("shape,seed", [((16, 16, 16), 0), ((32, 24, 16), 1), ((32, 32), 2), ((8, 8, 8), 3)])
def test_spmv_bitwise(b200, oracle, shape, seed):
    t = scenes.random_types(shape, 90 + seed)
    p = oracle.identity_params(len(shape), 1)
    ctx, octx = make(b200, oracle, t, 1, p)
    x = np.random.default_rng(seed).standard_normal(ctx.n_fluid)
    assert np.array_equal(ctx.spmv(x), octx.spmv(x))


@pytest.mark.parametrize("name,n,depth", [("C1", 32, 4), ("C2", 32, 3), ("C3", 32, 4), ("C1", 64, 4)])
def test_psdo_identity_weights_iteration_parity(b200, oracle, name, n, depth):
    """Identity-equivalent weights (the only convergent weights):
    iterations to rel-res 1e-6 within +-1 of the oracle psdo_solve (which is
    bitwise the reference solver, tests/test_oracle_pinning.py)."""
    t, seed = scenes.config(name, n)
    p = oracle.identity_params(3, depth)
    ctx, octx = make(b200, oracle, t, depth, p)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=5000)
    got = ctx.psdo_solve(b, cfg)
    want = octx.psdo_solve(b, max_iters=5000)
    assert got.report.converged and want["converged"]
    assert abs(got.report.iterations - want["iterations"]) <= 1
    assert got.report.residual_history[-1] <= 1e-6 * got.report.residual_history[0]
    assert rel_l2(got.x, want["x"]) <= 1e-5


@pytest.mark.parametrize("n_ortho", [0, 1, 2, 4])
def test_psdo_random_weights_history(b200, oracle, n_ortho):
    """Fixed 50-iteration budget with random weights: residual history within
    1e-6 relative of the oracle."""
    t = scenes.dam_break(16)
    p = oracle.init_params(3, 3, 42)
    ctx, octx = make(b200, oracle, t, 3, p)
    b = oracle.rhs_normal(1235, t.size)[t.reshape(-1) == 0]
    got = ctx.psdo_solve(b, b200.SolveConfig(max_iters=50, tol_reduction=1e-300, n_ortho=n_ortho))
    want = octx.psdo_solve(b, max_iters=50, tol_reduction=1e-300, n_ortho=n_ortho)
    assert got.report.iterations == want["iterations"] == 50
    h, w = got.report.residual_history, want["residual_history"]
    assert np.max(np.abs(h - w) / w) <= 1e-6


def test_psdo_2d_vs_reference(b200, oracle, ref):
    t = np.zeros((64, 64), np.uint8)
    c = np.arange(64) + 0.5
    y, x = np.meshgrid(c, c, indexing="ij")
    t[y >= 48] = 1
    t[(x < 19.2) & (y < 12.8)] = 2
    p = oracle.identity_params(2, 3)
    ctx, _ = make(b200, oracle, t, 3, p)
    b = ref.rhs_normal(13, ctx.n_fluid)
    got = ctx.psdo_solve(b, b200.SolveConfig(max_iters=3000))
    want = ref.psdo_solve(t, b, mode="neural", params=p, depth=3, max_iters=3000)
    assert got.report.converged and want["converged"]
    assert abs(got.report.iterations - want["iterations"]) <= 1


def test_nullspace_projection_pure_neumann(b200, oracle):
    """test_solvers.cpp:307-320 on the B200: all-fluid closed box, singular
    system, solved under mean projection."""
    t = np.zeros((16, 16, 16), np.uint8)
    p = oracle.identity_params(3, 2)
    ctx, octx = make(b200, oracle, t, 2, p)
    b = oracle.rhs_normal(21, t.size)
    b -= b.mean()
    cfg = b200.SolveConfig(max_iters=2000, nullspace_projection=True)
    got = ctx.psdo_solve(b, cfg)
    want = octx.psdo_solve(b, max_iters=2000, nullspace_projection=True)
    assert got.report.converged and want["converged"]
    assert abs(got.report.iterations - want["iterations"]) <= 1


def test_max_iters_and_history_length(b200, oracle):
    t = scenes.closed_box_half(16)
    ctx, _ = make(b200, oracle, t, 2, oracle.identity_params(3, 2))
    b = oracle.rhs_normal(22, t.size)[t.reshape(-1) == 0]
    res = ctx.psdo_solve(b, b200.SolveConfig(max_iters=3))
    assert not res.report.converged
    assert res.report.iterations == 3 and res.report.residual_history.size == 4  # test_solvers.cpp:322-331


def test_errors(b200, oracle):
    t = scenes.closed_box_half(16)
    P = b200.NeuralPrecond(b200.init_params(2, 5), t)
    b = np.ones(P.size())
    with pytest.raises(ValueError):
        b200.psdo_solve(None, b, P, b200.SolveConfig(tol_reduction=1.5))
    with pytest.raises(ValueError):
        b200.psdo_solve(None, np.ones(3), P)
    bad = b.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        b200.psdo_solve(None, bad, P)
    with pytest.raises(ValueError):
        b200.Context(3, (12, 12, 12), b200.init_params(3, 1))  # not divisible by 2^3
    with pytest.raises(b200.EmptySystemError):
        Q = b200.NeuralPrecond(b200.init_params(2, 5), np.full((16, 16, 16), 1, np.uint8))
        b200.psdo_solve(None, np.zeros(0), Q)


def test_breakdown_raises(b200, oracle):
    """A preconditioner whose output is A-orthogonal to nothing useful: zero
    weights give d = 0 -> curvature 0 -> SolverBreakdown (solver.cpp:247-250)."""
    t = scenes.closed_box_half(16)
    p = np.zeros(oracle.param_count(3, 2), np.float32)
    P = b200.NeuralPrecond(b200.NetParams(3, 2, p), t)
    b = oracle.rhs_normal(1, t.size)[t.reshape(-1) == 0]
    with pytest.raises(b200.SolverBreakdown):
        b200.psdo_solve(None, b, P, b200.SolveConfig(max_iters=10))


@pytest.mark.ref
@pytest.mark.parametrize("dim", [2, 3])
def test_dropin_reference_solver_with_b200_precond(b200, oracle, ref, dim):
    """The drop-in check: the reference's own psdo_solve (solver.cpp:189-276)
    driving the B200 NeuralPrecond through the C ABI (a C callback), against the
    same reference solver driving the CPU network."""
    if dim == 2:
        t = scenes.random_types((32, 32), 5, p=(0.7, 0.2, 0.1))
    else:
        t = scenes.dam_break(16)
    depth = 3
    p = oracle.init_params(dim, depth, 9)
    P = b200.NeuralPrecond(b200.NetParams(dim, depth, p), t)
    n = P.size()

    def cb(user, r_ptr, z_ptr, nn):
        r = np.ctypeslib.as_array(r_ptr, shape=(nn,))
        z = np.ctypeslib.as_array(z_ptr, shape=(nn,))
        z[:] = P.apply(r.copy())
        return 0

    b = ref.rhs_normal(3, n)
    got = ref.psdo_solve(t, b, mode="callback", callback=cb, max_iters=15, tol_reduction=1e-300)
    want = ref.psdo_solve(t, b, mode="neural", params=p, depth=depth, max_iters=15, tol_reduction=1e-300)
    h, w = got["residual_history"], want["residual_history"]
    assert np.max(np.abs(h - w) / w) <= 1e-6


def test_set_mask_frames_no_resetup(b200, oracle):
    """C4 pattern: one context, per-frame set_mask only; each frame matches a
    fresh oracle context."""
    p = oracle.init_params(3, 3, 5)
    ctx = b200.Context(3, (32, 32, 32), b200.NetParams(3, 3, p))
    for f, t in enumerate(scenes.droplet_frames(32, 4)):
        ctx.set_mask(t)
        octx = oracle.context(t, p, 3)
        r = np.random.default_rng(f).standard_normal(ctx.n_fluid)
        assert rel_l2(ctx.precond_apply(r), octx.precond_apply(r)) <= REL_L2


def test_solve_device_path(b200, oracle):
    """Device-resident full-grid API == host reduced API."""
    t = scenes.closed_box_half(32)
    P = b200.identity_params(4)
    ctx = b200.Context(3, t.shape, P)
    ctx.set_mask(t)
    bf = scenes.full_rhs(t, 1234, oracle.rhs_normal)
    cfg = b200.SolveConfig(max_iters=2000)
    host = ctx.psdo_solve(bf[t.reshape(-1) == 0], cfg)
    db = b200.DeviceBuffer(ctx, bf.nbytes)
    dx = b200.DeviceBuffer(ctx, bf.nbytes)
    db.upload(bf)
    rep = ctx.psdo_solve_device(db.ptr, dx.ptr, cfg)
    xf = np.empty_like(bf)
    dx.download(xf)
    ctx.synchronize()
    assert rep.iterations == host.report.iterations
    assert np.array_equal(xf[t.reshape(-1) == 0], host.x)
    assert np.all(xf[t.reshape(-1) != 0] == 0.0)
    db.free()
    dx.free()


def test_raw_network_then_solve_unchanged(b200, oracle):
    """The solve path visits live tiles only and relies on zeros elsewhere in
    its network buffers; a raw net_apply (dense input, writes every cell) and a
    frame change in between must not leak into the next solve."""
    t, seed = scenes.config("C3", 64)
    p = oracle.init_params(3, 4, 11)
    ctx = b200.Context(3, t.shape, b200.NetParams(3, 4, p))
    ctx.set_mask(t)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=15, tol_reduction=1e-300)
    first = ctx.psdo_solve(b, cfg).report.residual_history
    r = np.random.default_rng(0).standard_normal(ctx.n_fluid)
    z1 = ctx.precond_apply(r)
    ctx.net_apply(np.random.default_rng(1).standard_normal(t.size).astype(np.float32).reshape(t.shape))
    assert np.array_equal(ctx.precond_apply(r), z1)
    assert np.array_equal(ctx.psdo_solve(b, cfg).report.residual_history, first)
    # another frame, then back: bitwise the same again
    ctx.set_mask(list(scenes.droplet_frames(64, 2))[1])
    ctx.set_mask(t)
    assert np.array_equal(ctx.psdo_solve(b, cfg).report.residual_history, first)


def test_c5_512_identity_solve_explicit_residual(b200, oracle):
    """C5 at 512^3 (beyond the oracle's network; size-independent checks):
    PSDO with identity-equivalent weights converges, and the oracle's
    matrix-free A recomputes the final residual the history reports."""
    t, seed = scenes.config("C5")
    mask = t.reshape(-1) == 0
    ctx = b200.Context(3, t.shape, b200.identity_params(4))
    ctx.set_mask(t)
    b = oracle.rhs_normal(seed, t.size)[mask]
    res = ctx.psdo_solve(b, b200.SolveConfig(max_iters=10000))
    hist = res.report.residual_history
    assert res.report.converged and np.all(np.isfinite(res.x))
    r = b - oracle.spmv(t, res.x)
    nb, nr = np.linalg.norm(b), np.linalg.norm(r)
    assert nr <= 1e-6 * nb * (1 + 1e-9)
    assert abs(nr - hist[-1]) <= 1e-9 * nb
    assert hist[0] == pytest.approx(nb, rel=1e-12)


def test_c5_512_random_weights_precond_scaling_and_linearity(b200, oracle):
    """512^3, random weights: P(2r) == 2 P(r) bitwise (power-of-two scaling is
    exact through the normalisation, net_precond.cpp:20-34) and P is linear up
    to f32 rounding (the reference's linearity test, test_neural.cpp:182-210)."""
    t, _ = scenes.config("C5")
    ctx = b200.Context(3, t.shape, b200.init_params(4, 17))
    ctx.set_mask(t)
    rng = np.random.default_rng(5)
    r1, r2 = rng.standard_normal(ctx.n_fluid), rng.standard_normal(ctx.n_fluid)
    z1, z2 = ctx.precond_apply(r1), ctx.precond_apply(r2)
    assert np.all(np.isfinite(z1))
    assert np.array_equal(ctx.precond_apply(2.0 * r1), 2.0 * z1)
    z12 = ctx.precond_apply(r1 + r2)
    assert rel_l2(z12, z1 + z2) <= 1e-4


@pytest.mark.parametrize("shape,with_bc", [((16, 24, 32), False), ((16, 24, 32), True), ((40, 24), True)])
def test_mac_rhs_bitwise(b200, oracle, shape, with_bc):
    """mac_divergence_rhs on the device (discretization.cpp:193-227; 3D
    generalisation): bitwise equal to the restatement (3D) and to the
    reference (2D, when present), reduced to the solve's ordering."""
    t = scenes.random_types(shape, 41)
    rng = np.random.default_rng(6)
    if len(shape) == 3:
        nz, ny, nx = shape
        u, v, w = rng.standard_normal((nz, ny, nx + 1)), rng.standard_normal((nz, ny + 1, nx)), \
            rng.standard_normal((nz + 1, ny, nx))
        bc = tuple(rng.standard_normal(a.shape) for a in (u, v, w)) if with_bc else None
        ctx = b200.Context(3, shape, b200.identity_params(1))
    else:
        ny, nx = shape
        u, v, w = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx)), None
        bc = tuple(rng.standard_normal(a.shape) for a in (u, v)) if with_bc else None
        ctx = b200.Context(2, shape, b200.identity_params(1, dim=2))
    ctx.set_mask(t)
    got = ctx.mac_divergence_rhs(u, v, w, h=0.5, dt=0.02, rho=1.5, bc=bc)
    want = oracle.mac_rhs(t, u, v, w, h=0.5, dt=0.02, rho=1.5, bc=bc)[t.reshape(-1) == 0]
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_mac_rhs_device_pipeline(b200, oracle):
    """flags + velocity -> rhs -> solve without leaving HBM: identical to the
    host path (rhs on the host API, then the solve)."""
    t, _ = scenes.config("C3", 32)
    nz, ny, nx = t.shape
    rng = np.random.default_rng(8)
    u, v, w = rng.standard_normal((nz, ny, nx + 1)), rng.standard_normal((nz, ny + 1, nx)), \
        rng.standard_normal((nz + 1, ny, nx))
    ctx = b200.Context(3, t.shape, b200.identity_params(4))
    ctx.set_mask(t)
    cfg = b200.SolveConfig(max_iters=2000)
    host = ctx.psdo_solve(ctx.mac_divergence_rhs(u, v, w), cfg)
    bufs = [b200.DeviceBuffer(ctx, a.nbytes) for a in (u, v, w)]
    for bf, a in zip(bufs, (u, v, w)):
        bf.upload(np.ascontiguousarray(a))
    db, dx = b200.DeviceBuffer(ctx, 8 * t.size), b200.DeviceBuffer(ctx, 8 * t.size)
    ctx.mac_divergence_rhs_device(bufs[0].ptr, bufs[1].ptr, bufs[2].ptr, db.ptr)
    rep = ctx.psdo_solve_device(db.ptr, dx.ptr, cfg)
    xf = np.empty(t.size)
    dx.download(xf)
    ctx.synchronize()
    assert rep.iterations == host.report.iterations and rep.converged
    assert np.array_equal(xf[t.reshape(-1) == 0], host.x)
    for bf in (*bufs, db, dx):
        bf.free()


@pytest.mark.parametrize("name,n,precond", [("C1", 32, "identity"), ("C3", 32, "jacobi"), ("C2", 32, "jacobi"),
                                             ("C1", 32, "ic0"), ("C2", 32, "ic0"), ("C3", 48, "ic0")])
def test_pcg_iteration_parity_vs_reference(b200, oracle, ref, name, n, precond):
    """pcg_solve (solver.cpp:36-102) on the device, identity (cg_solve),
    Jacobi and IC0: iterations to 1e-6 within +-1 of the reference's own
    pcg_solve on the reference assembly; residual histories agree early and
    closely."""
    t, seed = scenes.config(name, n)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    want = ref.pcg_solve(t, b, precond={"identity": 0, "jacobi": 1, "ic0": 2}[precond], max_iters=3000)
    ctx = b200.Context(3, t.shape, b200.identity_params(4))
    ctx.set_mask(t)
    got = ctx.pcg_solve(b, b200.SolveConfig(max_iters=3000), precond=precond)
    assert got.report.converged and want["converged"]
    assert abs(got.report.iterations - want["iterations"]) <= 1
    h, w = got.report.residual_history, want["residual_history"]
    assert np.max(np.abs(h[:30] - w[:30]) / w[:30]) <= 1e-9
    assert rel_l2(got.x, want["x"]) <= 1e-5


def _ic0_cases():
    yield scenes.config("C1", 16)[0]
    yield scenes.config("C2", 32)[0]
    yield scenes.config("C3", 24)[0]
    yield scenes.config("C5", 32)[0]
    t = scenes.random_types((12, 20, 28), 5, p=(0.7, 0.25, 0.05))
    yield t
    yield scenes.droplet_pool(16)[8]  # 2D slice (ny, nx)


@pytest.mark.parametrize("k", range(6))
def test_ic0_apply_bitwise_vs_reference(b200, ref, k):
    """Ic0Precond (precond.cpp:28-112): the device factorization (level-
    scheduled over hyperplanes) and both triangular sweeps equal the
    reference's constructor + apply bit for bit, including its shift-retry
    count."""
    t = list(_ic0_cases())[k]
    dim = t.ndim
    ctx = b200.Context(dim, t.shape, b200.identity_params(2, dim))
    ctx.set_mask(t)
    r = np.random.default_rng(k).standard_normal(ctx.n_fluid)
    try:
        want, wret = ref.ic0_apply(t, r)
    except Exception as e:  # the reference cannot factor this frame: neither may we
        with pytest.raises(ValueError, match="ic0: factorization failed"):
            ctx.ic0_apply(r)
        pytest.skip(f"reference: {e}")
    got, gret = ctx.ic0_apply(r)
    assert gret == wret
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_ic0_isolated_cell_fails_like_reference(b200, ref):
    """A fluid cell with only solid neighbours has no diagonal in its row: the
    reference's factorization fails on every shift retry and throws."""
    t = np.full((8, 8, 8), 2, np.uint8)
    t[1:4, 1:7, 1:7] = 0
    t[0, :, :] = 1
    t[6, 4, 4] = 0  # isolated
    ctx = b200.Context(3, t.shape, b200.identity_params(2))
    ctx.set_mask(t)
    r = np.ones(ctx.n_fluid)
    with pytest.raises(Exception, match="ic0: factorization failed"):
        ref.ic0_apply(t, r)
    with pytest.raises(ValueError, match="ic0: factorization failed after diagonal-shift retries"):
        ctx.ic0_apply(r)
    with pytest.raises(ValueError, match="ic0: factorization failed"):
        ctx.pcg_solve(r, b200.SolveConfig(max_iters=10), precond="ic0")


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_trained_weights_iteration_parity(b200, name):
    """The committed trained 3D model (b200.DEFAULT_MODEL): iterations to
    1e-6 on the benchmark domains at their full sizes within +-1 of the
    reference psdo_solve with the same weights (tests/golden/iteration_counts.json,
    "<name>_trained", made by tests/golden/make_iteration_counts.py --trained)."""
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    want = json.loads((root / "tests" / "golden" / "iteration_counts.json").read_text())[f"{name}_trained"]
    W = b200.default_model()
    t, seed = scenes.config(name)
    ctx = b200.Context(3, t.shape, W)
    ctx.set_mask(t)
    b = b200.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    res = ctx.psdo_solve(b, b200.SolveConfig(max_iters=2000))
    assert res.report.converged
    assert abs(res.report.iterations - want["iterations"]) <= 1


def test_set_params_between_solves(b200, oracle):
    """set_params replaces every weight-dependent table and the captured solve
    graph (it holds the uniform-window kernels by value): solving with weights
    A, then B, then A again equals fresh contexts of A and B."""
    t, seed = scenes.config("C3", 32)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    cfg = b200.SolveConfig(max_iters=30, tol_reduction=1e-300)
    pa, pb = b200.init_params(4, 3), b200.identity_params(4)

    def fresh(p):
        c = b200.Context(3, t.shape, p)
        c.set_mask(t)
        return c.psdo_solve(b, cfg).report.residual_history

    ha, hb = fresh(pa), fresh(pb)
    ctx = b200.Context(3, t.shape, pa)
    ctx.set_mask(t)
    assert np.array_equal(ctx.psdo_solve(b, cfg).report.residual_history, ha)
    for p, h in ((pb, hb), (pa, ha)):
        ctx.set_params(p)
        ctx.set_mask(t)
        assert np.array_equal(ctx.psdo_solve(b, cfg).report.residual_history, h)


@pytest.mark.parametrize("exact", [True, False])
def test_merged_up0_equals_two_launches(b200, oracle, exact, monkeypatch):
    """Level-0 up: tiled and mixed cells in one launch (k_up_l0m) give the
    same direction as two launches; the MGS dots are one deterministic
    reduction instead of two (histories agree to rounding)."""
    t, seed = scenes.config("C3", 64)
    p = b200.init_params(4, 29)
    b = oracle.rhs_normal(seed, t.size)[t.reshape(-1) == 0]
    out = []
    for merge in ("1", "0"):
        monkeypatch.setenv("NPSD_MERGE_UP0", merge)
        ctx = b200.Context(3, t.shape, p, exact=exact)
        ctx.set_mask(t)
        out.append((ctx.precond_apply(b), ctx.psdo_solve(b, b200.SolveConfig(max_iters=15, tol_reduction=1e-300))))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    h, w = out[0][1].report.residual_history, out[1][1].report.residual_history
    assert np.max(np.abs(h - w) / w) <= 1e-9


@pytest.mark.parametrize("case", ["C1", "C2", "random128", "random64x128x256"])
def test_classify_simd_equals_scalar(b200, monkeypatch, case):
    """Level-0 classification with byte SIMD (4 cells per thread) writes the
    same cell bytes, masks, tile flags and window counts as one cell per
    thread: every set_mask product compares equal."""
    if case in ("C1", "C2"):
        t, _ = scenes.config(case)
    elif case == "random128":
        t = scenes.random_types((128, 128, 128), 77, p=(0.5, 0.3, 0.2), blobs=8)
    else:
        t = scenes.random_types((64, 128, 256), 78, p=(0.6, 0.25, 0.15), blobs=6)
    p = b200.init_params(4, 31)
    r = np.random.default_rng(3).standard_normal(int((t == 0).sum()))
    out = []
    for simd in ("1", "0"):
        monkeypatch.setenv("NPSD_CLASSIFY_SIMD", simd)
        ctx = b200.Context(3, t.shape, p, exact=True)
        ctx.set_mask(t)
        za, zb = ctx.linear_coeffs()
        out.append((ctx.fluid_indices(), ctx.mixed_counts(), za, zb, [ctx.level_image(l) for l in range(4)],
                    ctx.precond_apply(r), ctx.is_pure_neumann()))
        ctx.close()
    a, b = out
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2].view(np.uint32), b[2].view(np.uint32))
    assert np.array_equal(a[3].view(np.uint32), b[3].view(np.uint32))
    for la, lb in zip(a[4], b[4]):
        assert np.array_equal(la, lb)
    assert np.array_equal(a[5], b[5]) and a[6] == b[6]


def test_setup_branches_equal_serial(b200, monkeypatch):
    """set_mask's graph runs its independent chains as branches (aux streams
    forked and joined through events); one stream (NPSD_SETUP_SERIAL=1) gives
    the same frame bit for bit, across a frame sequence through one context
    whose capacities grow on the way (a simple frame, then a random one)."""
    n = 64
    frames = list(scenes.droplet_frames(n, 3))
    frames.insert(1, scenes.random_types((n, n, n), 91, p=(0.5, 0.3, 0.2), blobs=8))
    p = b200.default_model()
    out = {}
    for serial in ("1", "0"):
        monkeypatch.setenv("NPSD_SETUP_SERIAL", serial)
        ctx = b200.Context(3, (n, n, n), p)
        res = []
        for f, t in enumerate(frames):
            ctx.set_mask(t)
            r = np.random.default_rng(f).standard_normal(int((t == 0).sum()))
            b = b200.rhs_normal(50 + f, t.size)[t.reshape(-1) == 0]
            rep = ctx.psdo_solve(b, b200.SolveConfig(max_iters=300)).report
            res.append((ctx.mixed_counts(), ctx.precond_apply(r), rep.iterations, rep.residual_history))
        out[serial] = res
        ctx.close()
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(a[1], b[1])
        assert a[2] == b[2] and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("exact", [True, False])
def test_coarse_skip_equals_full(b200, monkeypatch, exact):
    """Solve-path coarse down steps skip tiles with no fluid within two cells
    (their outputs stay the frame's zeros): the preconditioner and a solve
    history equal the full launches bit for bit, across frames whose fluid
    moves and after a raw network call that writes every tile."""
    p = b200.default_model()
    n = 128
    frames = list(scenes.droplet_frames(n, 3))
    frames.insert(1, scenes.random_types((n, n, n), 93, p=(0.5, 0.3, 0.2), blobs=8))
    xin = np.random.default_rng(4).standard_normal(n ** 3).astype(np.float32)
    out = {}
    for skip in ("1", "0"):
        monkeypatch.setenv("NPSD_COARSE_SKIP", skip)
        ctx = b200.Context(3, (n, n, n), p, exact=exact)
        res = []
        for f, t in enumerate(frames):
            ctx.set_mask(t)
            r = np.random.default_rng(f).standard_normal(int((t == 0).sum()))
            a = ctx.precond_apply(r)
            raw = ctx.net_apply(xin)  # writes every coarse tile
            rep = ctx.psdo_solve(r, b200.SolveConfig(max_iters=15, tol_reduction=1e-300)).report
            res.append((a, raw, ctx.precond_apply(r), rep.residual_history))
        out[skip] = res
        ctx.close()
    for a, b in zip(out["1"], out["0"]):
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


def test_frame_after_larger_frame_equals_fresh_context(b200):
    """A frame's setup zeroes only the cells that stopped being fluid (the
    solver vectors' zero invariant): after solves on a frame with more fluid,
    a frame with less gives the same solve as a fresh context, bit for bit."""
    p = b200.default_model()
    n = 64
    big = scenes.random_types((n, n, n), 11, p=(0.8, 0.15, 0.05), blobs=4)
    small = scenes.random_types((n, n, n), 12, p=(0.4, 0.4, 0.2), blobs=8)
    cfg = b200.SolveConfig(max_iters=30, tol_reduction=1e-300)
    bs = b200.rhs_normal(3, small.size)[small.reshape(-1) == 0]
    ctx = b200.Context(3, (n, n, n), p)
    ctx.set_mask(big)
    ctx.psdo_solve(b200.rhs_normal(2, big.size)[big.reshape(-1) == 0], cfg)
    ctx.set_mask(small)
    got = ctx.psdo_solve(bs, cfg)
    ctx.close()
    fresh = b200.Context(3, (n, n, n), p)
    fresh.set_mask(small)
    want = fresh.psdo_solve(bs, cfg)
    fresh.close()
    assert np.array_equal(got.x, want.x)
    assert np.array_equal(got.report.residual_history, want.report.residual_history)

"""Pins the CPU oracle (oracle/npsd_oracle.hpp) against the REAL reference
(oracle/_ref, built from /root/reference sources) — bitwise in 2D, where the
reference has a network — and re-expresses the reference's own unit-test
assertions (test_neural.cpp, test_solvers.cpp, test_discretization.cpp) on the
oracle's 3D instantiation. CPU only."""
import numpy as np
import pytest

from paper_2310_00177_b200.scenes import random_types, closed_box_half, droplet_pool, dam_break


def _mixed_bc_2d(n):
    """test_solvers.cpp:17-28: air above 0.75n, solid box [0,0.3n)x[0,0.2n)."""
    c = np.arange(n) + 0.5
    y, x = np.meshgrid(c, c, indexing="ij")
    t = np.zeros((n, n), np.uint8)
    t[y >= 0.75 * n] = 1
    t[(x < 0.3 * n) & (y < 0.2 * n)] = 2
    return t


# --------------------------------------------------------------- weights/rng
@pytest.mark.ref
@pytest.mark.parametrize("depth", [1, 2, 3, 4])
def test_init_params_2d_bitwise(oracle, ref, depth):
    a = oracle.init_params(2, depth, 14 + depth)
    b = ref.init_params_2d(depth, 14 + depth)
    assert a.size == (depth - 1) * (2 * 252 + 2 * 28) + 252
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.ref
def test_rng_normal_stream(oracle, ref):
    assert np.array_equal(oracle.rhs_normal(1234, 1001), ref.rhs_normal(1234, 1001))


def test_param_count_3d(oracle):
    # L=4 -> 15,990
    assert oracle.param_count(3, 4) == 15990
    assert oracle.param_count(2, 3) == 2 * (2 * 252 + 2 * 28) + 252


# ---------------------------------------------------------------- network 2D
CASES_2D = [(16, 16, 1, 0), (16, 16, 2, 1), (32, 16, 3, 2), (32, 32, 3, 3), (64, 64, 4, 4), (24, 40, 3, 5)]


@pytest.mark.ref
@pytest.mark.parametrize("nx,ny,depth,seed", CASES_2D)
def test_level_images_2d_bitwise(oracle, ref, nx, ny, depth, seed):
    if nx % (1 << depth) or ny % (1 << depth):
        pytest.skip("not divisible")
    t = random_types((ny, nx), seed)
    for a, b in zip(oracle.level_images(t, depth), ref.level_images_2d(t, depth)):
        assert np.array_equal(a, b)


@pytest.mark.ref
@pytest.mark.parametrize("nx,ny,depth,seed", CASES_2D)
def test_net_apply_2d_bitwise(oracle, ref, nx, ny, depth, seed):
    if nx % (1 << depth) or ny % (1 << depth):
        pytest.skip("not divisible")
    t = random_types((ny, nx), 100 + seed)
    p = oracle.init_params(2, depth, 300 + seed)
    x = np.random.default_rng(seed).standard_normal((ny, nx)).astype(np.float32)
    ctx = oracle.context(t, p, depth)
    got = ctx.net_apply(x)
    want, za, zb = ref.net_apply_2d(t, p, depth, x)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    oza, ozb = ctx.z()
    assert np.array_equal(oza, za) and np.array_equal(ozb, zb)


@pytest.mark.ref
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_precond_apply_2d_bitwise(oracle, ref, seed):
    t = random_types((32, 32), 200 + seed)
    p = oracle.init_params(2, 3, 25 + seed)
    ctx = oracle.context(t, p, 3)
    r = np.random.default_rng(seed).standard_normal(ctx.n_fluid)
    assert np.array_equal(ctx.precond_apply(r), ref.precond_apply_2d(t, p, 3, r))


# ------------------------------------------------------------------ operator
@pytest.mark.ref
@pytest.mark.parametrize("shape,seed", [((16, 16), 0), ((32, 24), 1), ((8, 8, 8), 2), ((16, 12, 8), 3)])
def test_spmv_bitwise(oracle, ref, shape, seed):
    t = random_types(shape, 400 + seed)
    dim = len(shape)
    ctx = oracle.context(t, oracle.identity_params(dim, 1), 1)
    x = np.random.default_rng(seed).standard_normal(ctx.n_fluid)
    assert np.array_equal(ctx.spmv(x), ref.spmv(t, x))


# -------------------------------------------------------------------- solver
@pytest.mark.ref
def test_psdo_2d_neural_history_bitwise(oracle, ref):
    """Random weights never converge; run a fixed 30-iteration budget."""
    t = _mixed_bc_2d(32)
    p = oracle.init_params(2, 3, 42)
    ctx = oracle.context(t, p, 3)
    b = ref.rhs_normal(13, ctx.n_fluid)
    a = ctx.psdo_solve(b, max_iters=30, tol_reduction=1e-300)
    r = ref.psdo_solve(t, b, mode="neural", params=p, depth=3, max_iters=30, tol_reduction=1e-300)
    assert a["iterations"] == r["iterations"] == 30
    assert np.array_equal(a["residual_history"], r["residual_history"])
    assert np.array_equal(a["x"], r["x"])


@pytest.mark.ref
@pytest.mark.parametrize("n_ortho", [0, 1, 2, 3])
def test_psdo_3d_identity_bitwise(oracle, ref, n_ortho):
    t = closed_box_half(16)
    ctx = oracle.context(t, oracle.identity_params(3, 2), 2)
    b = ref.rhs_normal(1234, ctx.n_fluid)
    a = ctx.psdo_solve(b, identity=True, n_ortho=n_ortho, max_iters=500)
    r = ref.psdo_solve(t, b, mode="identity", n_ortho=n_ortho, max_iters=500)
    assert a["iterations"] == r["iterations"]
    assert np.array_equal(a["residual_history"], r["residual_history"])


@pytest.mark.ref
def test_psdo_3d_identity_weights_matches_reference_cg_count(oracle, ref):
    """Identity-equivalent weights make PSDO track the identity-preconditioned
    reference solve: iteration counts within 1."""
    t = closed_box_half(16)
    p = oracle.identity_params(3, 2)
    ctx = oracle.context(t, p, 2)
    b = ref.rhs_normal(1234, ctx.n_fluid)
    a = ctx.psdo_solve(b, max_iters=1000)
    r = ref.psdo_solve(t, b, mode="identity", max_iters=1000)
    assert a["converged"] and r["converged"]
    assert abs(a["iterations"] - r["iterations"]) <= 1


@pytest.mark.ref
def test_psdo_3d_neural_in_reference_solver(oracle, ref):
    """The 3D restatement inside the reference psdo_solve (the CPU baseline) is
    the oracle's own psdo restatement, bitwise."""
    t = dam_break(16)
    p = oracle.init_params(3, 2, 7)
    ctx = oracle.context(t, p, 2)
    b = ref.rhs_normal(1235, ctx.n_fluid)
    a = ctx.psdo_solve(b, max_iters=12, tol_reduction=1e-300)
    r = ref.psdo_solve(t, b, mode="neural", params=p, depth=2, max_iters=12, tol_reduction=1e-300)
    assert np.array_equal(a["residual_history"], r["residual_history"])


# -------------------------------------- reference unit assertions, 3D oracle
def test_forward_zero_in_zero_out_3d(oracle):
    t = random_types((16, 16, 16), 13)
    ctx = oracle.context(t, oracle.init_params(3, 3, 14), 3)
    y = ctx.net_apply(np.zeros((16, 16, 16), np.float32))
    assert np.all(y == 0.0)  # test_neural.cpp:164-170


def test_identity_weights_return_input_3d(oracle):
    t = random_types((16, 16, 16), 3)
    ctx = oracle.context(t, oracle.identity_params(3, 3), 3)
    x = np.random.default_rng(4).standard_normal((16, 16, 16)).astype(np.float32)
    assert np.array_equal(ctx.net_apply(x), x)  # test_neural.cpp:40-47 across all levels


@pytest.mark.parametrize("trial", range(3))
def test_forward_linear_3d(oracle, trial):
    t = random_types((16, 16, 16), 200 + trial)
    ctx = oracle.context(t, oracle.init_params(3, 3, 300 + trial), 3)
    rng = np.random.default_rng(18 + trial)
    r1 = rng.standard_normal((16, 16, 16)).astype(np.float32)
    r2 = rng.standard_normal((16, 16, 16)).astype(np.float32)
    a, b = np.float32(rng.uniform(-2, 2)), np.float32(rng.uniform(-2, 2))
    lhs = ctx.net_apply(a * r1 + b * r2).astype(np.float64)
    want = float(a) * ctx.net_apply(r1).astype(np.float64) + float(b) * ctx.net_apply(r2).astype(np.float64)
    scale = max(np.abs(lhs).max(), 1e-6)
    assert np.abs(lhs - want).max() <= 1e-4 * scale  # test_neural.cpp:182-210


def test_divisibility_error_3d(oracle):
    from oracle_lib import OracleError

    with pytest.raises(OracleError) as e:
        oracle.context(random_types((12, 12, 12), 1), oracle.init_params(3, 3, 1), 3)
    assert e.value.status == 1  # invalid_argument (forward.hpp:58-62)


def test_pooled_images_channel_sum_3d(oracle):
    t = random_types((16, 16, 16), 10)
    for l, im in enumerate(oracle.level_images(t, 4)):
        s = im.sum(axis=0)
        assert np.all(s == 1.0)  # test_neural.cpp:140-146 (exact: dyadic values)
        assert np.all(im * (8 ** l) == np.round(im * (8 ** l)))


def test_psdo_3d_converges_identity_c1_small(oracle):
    t = closed_box_half(32)
    ctx = oracle.context(t, oracle.identity_params(3, 4), 4)
    b = oracle.rhs_normal(1234, t.size)[t.reshape(-1) == 0]
    res = ctx.psdo_solve(b, max_iters=2000)
    assert res["converged"]
    assert res["residual_history"][-1] <= 1e-6 * res["residual_history"][0]


@pytest.mark.ref
@pytest.mark.parametrize("with_bc", [False, True])
def test_mac_rhs_2d_bitwise_vs_reference(oracle, ref, with_bc):
    """mac_divergence_rhs (discretization.cpp:193-227): the restatement equals
    the reference bit for bit on a mixed grid, with and without boundary
    velocities."""
    t = random_types((24, 40), 31)
    rng = np.random.default_rng(4)
    ny, nx = t.shape
    u, v = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    bc = (rng.standard_normal(u.shape), rng.standard_normal(v.shape)) if with_bc else None
    want = ref.mac_rhs_2d(t, u, v, h=0.5, dt=0.01, rho=2.0, bc=bc)
    got = oracle.mac_rhs(t, u, v, h=0.5, dt=0.01, rho=2.0, bc=bc)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.all(got[t.reshape(-1) != 0] == 0.0)


@pytest.mark.ref
@pytest.mark.parametrize("name,n", [("C1", 16), ("C2", 16), ("C3", 24)])
def test_reduced_csr_restatement_spmv_bitwise(ref, name, n):
    """oracle_lib.reduced_csr (the numpy assemble_poisson_3d + reduce used by
    the operator-check tests) reproduces the reference's reduced matrix: its
    CSR-order row sums equal the reference spmv bit for bit."""
    from oracle_lib import reduced_csr
    from paper_2310_00177_b200 import scenes

    t, _ = scenes.config(name, n)
    ro, ci, va = reduced_csr(t)
    x = np.random.default_rng(3).standard_normal(ro.size - 1)
    y = np.array([sum((va[k] * x[ci[k]] for k in range(ro[r], ro[r + 1])), 0.0) for r in range(ro.size - 1)])
    assert np.array_equal(y, ref.spmv(t, x))

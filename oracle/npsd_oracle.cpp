// ============================================================================
// TEST INFRASTRUCTURE — NOT THE PRODUCT. C ABI over the CPU restatement in
// npsd_oracle.hpp, loaded by tests/ (ctypes) and by bench.py's cpu_baseline
// leg only. Status codes match include/npsd_b200.h: 0 ok, 1 invalid_argument,
// 2 SolverBreakdown, 3 EmptySystemError, 4 other.
// ============================================================================
#include <chrono>
#include <cstdio>
#include <memory>
#include <string>

#include "npsd_oracle.hpp"

using namespace npsdo;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const SolverBreakdown& e) {
        g_err = e.what();
        return 2;
    } catch (const EmptySystemError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

struct OracleCtx {
    int D = 3;
    Dims d;
    std::vector<std::uint8_t> types;
    ReductionMap map;
    Params params;
    std::unique_ptr<NetContext<2>> net2;
    std::unique_ptr<NetContext<3>> net3;
    double build_seconds = 0.0;
};

Dims make_dims(int D, long nx, long ny, long nz) {
    require(D == 2 || D == 3, "dim must be 2 or 3");
    require(nx > 0 && ny > 0 && (D == 2 || nz > 0), "dims must be positive");
    return Dims{nx, ny, D == 3 ? nz : 1};
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

long oracle_param_count(int D, int depth) { return static_cast<long>(param_count(D, depth)); }

int oracle_init_params(int D, int depth, unsigned long long seed, float* out) {
    return guarded([&] { params_to_flat(init_params(D, depth, seed), out); });
}

int oracle_identity_params(int D, int depth, float* out) {
    return guarded([&] { params_to_flat(identity_params(D, depth), out); });
}

// rng.hpp:36-48 normals in linear order (test_solvers.cpp:30-35 pattern)
void oracle_rhs_normal(unsigned long long seed, long n, double* out) {
    Rng rng(seed);
    for (long i = 0; i < n; ++i) out[i] = rng.normal();
}

// Coarsened images (PaddedImage::pooled chain), interiors only, 3 planes per
// level, levels 0..depth-1 concatenated.
int oracle_level_images(int D, long nx, long ny, long nz, int depth, const unsigned char* types, float* out) {
    return guarded([&] {
        const Dims d = make_dims(D, nx, ny, nz);
        std::size_t o = 0;
        auto emit = [&](auto& img) {
            const Dims dd = img.d;
            for (int c = 0; c < 3; ++c)
                for (index_t z = 0; z < dd.nz; ++z)
                    for (index_t y = 0; y < dd.ny; ++y)
                        for (index_t x = 0; x < dd.nx; ++x) out[o++] = img.at(c, x, y, z);
        };
        if (D == 2) {
            auto img = PaddedImage<2>::from_types(types, d);
            for (int l = 0; l < depth; ++l) {
                emit(img);
                if (l + 1 < depth) img = img.pooled();
            }
        } else {
            auto img = PaddedImage<3>::from_types(types, d);
            for (int l = 0; l < depth; ++l) {
                emit(img);
                if (l + 1 < depth) img = img.pooled();
            }
        }
    });
}

int oracle_ctx_create(int D, long nx, long ny, long nz, int depth, const float* params, long n_params,
                      const unsigned char* types, void** out) {
    return guarded([&] {
        auto ctx = std::make_unique<OracleCtx>();
        ctx->D = D;
        ctx->d = make_dims(D, nx, ny, nz);
        ctx->types.assign(types, types + ctx->d.cells());
        ctx->map = ReductionMap::from_types(ctx->types.data(), ctx->d);
        ctx->params = params_from_flat(D, depth, params, static_cast<std::size_t>(n_params));
        const auto t0 = std::chrono::steady_clock::now();
        if (D == 2)
            ctx->net2 = std::make_unique<NetContext<2>>(NetContext<2>::build(ctx->params, ctx->types.data(), ctx->d));
        else
            ctx->net3 = std::make_unique<NetContext<3>>(NetContext<3>::build(ctx->params, ctx->types.data(), ctx->d));
        ctx->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = ctx.release();
    });
}

void oracle_ctx_destroy(void* h) { delete static_cast<OracleCtx*>(h); }

long oracle_ctx_n_fluid(void* h) { return static_cast<long>(static_cast<OracleCtx*>(h)->map.reduced_size()); }

double oracle_ctx_build_seconds(void* h) { return static_cast<OracleCtx*>(h)->build_seconds; }

int oracle_ctx_fluid_indices(void* h, long long* out) {
    auto* c = static_cast<OracleCtx*>(h);
    for (std::size_t i = 0; i < c->map.fluid_indices.size(); ++i) out[i] = c->map.fluid_indices[i];
    return 0;
}

// linear-block coefficients per level (levels 0..depth-2)
int oracle_ctx_z(void* h, float* za, float* zb) {
    auto* c = static_cast<OracleCtx*>(h);
    const int L = c->params.depth;
    for (int l = 0; l + 1 < L; ++l) {
        za[l] = (c->D == 2) ? c->net2->levels[l].z_a : c->net3->levels[l].z_a;
        zb[l] = (c->D == 2) ? c->net2->levels[l].z_b : c->net3->levels[l].z_b;
    }
    return 0;
}

// NetContext::apply on the full grid (forward.hpp:95-129)
int oracle_ctx_net_apply(void* h, const float* x, float* y) {
    return guarded([&] {
        auto* c = static_cast<OracleCtx*>(h);
        std::vector<float> in(x, x + c->d.cells());
        const std::vector<float> out = (c->D == 2) ? c->net2->apply(in) : c->net3->apply(in);
        std::memcpy(y, out.data(), out.size() * sizeof(float));
    });
}

namespace {
struct BorrowedNeural : Precond {
    OracleCtx* c;
    explicit BorrowedNeural(OracleCtx* cc) : c(cc) {}
    void apply(const Vector& r, Vector& z) const override {
        const double rnorm = norm2(r);
        z.assign(r.size(), 0.0);
        if (rnorm == 0.0) return;
        std::vector<float> full(static_cast<std::size_t>(c->d.cells()), 0.0f);
        const double inv = 1.0 / rnorm;
        for (std::size_t k = 0; k < r.size(); ++k)
            full[static_cast<std::size_t>(c->map.fluid_indices[k])] = static_cast<float>(r[k] * inv);
        const std::vector<float> out = (c->D == 2) ? c->net2->apply(full) : c->net3->apply(full);
        for (std::size_t k = 0; k < z.size(); ++k)
            z[k] = static_cast<double>(out[static_cast<std::size_t>(c->map.fluid_indices[k])]) * rnorm;
    }
};
}  // namespace

// NeuralPrecond::apply (net_precond.cpp:14-35) on reduced vectors
int oracle_ctx_precond_apply(void* h, const double* r, double* z) {
    return guarded([&] {
        auto* c = static_cast<OracleCtx*>(h);
        const std::size_t nf = static_cast<std::size_t>(c->map.reduced_size());
        Vector rv(r, r + nf), zv;
        BorrowedNeural(c).apply(rv, zv);
        std::memcpy(z, zv.data(), nf * sizeof(double));
    });
}

// reduced A·x (assemble_poisson[_3d] + reduce + spmv)
// mac_divergence_rhs (discretization.cpp:193-227), restated on cell types and
// generalised to 3D: b = scale * (((uR - uL) + (vT - vB)) + (wF - wB)) at fluid
// cells (2D: the first two terms), scale = -(rho * h) / dt; a face whose
// opposite cell is solid (or outside the domain) takes the boundary value
// (0 without one); non-fluid cells 0. Face arrays x fastest: u (nx+1, ny, nz),
// v (nx, ny+1, nz), w (nx, ny, nz+1).
int oracle_mac_rhs(int D, long nx, long ny, long nz, const unsigned char* types, const double* u, const double* v,
                   const double* w, double h, double dt, double rho, const double* bu, const double* bv,
                   const double* bw, double* b) {
    return guarded([&] {
        if (D == 2) nz = 1;
        auto solid = [&](long x, long y, long z) {
            if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) return true;
            return types[(z * ny + y) * nx + x] == 2;
        };
        auto ui = [&](long x, long y, long z) { return (z * ny + y) * (nx + 1) + x; };
        auto vi = [&](long x, long y, long z) { return (z * (ny + 1) + y) * nx + x; };
        auto wi = [&](long x, long y, long z) { return (z * ny + y) * nx + x; };
        const double scale = -(rho * h) / dt;
        for (long z = 0; z < nz; ++z)
            for (long y = 0; y < ny; ++y)
                for (long x = 0; x < nx; ++x) {
                    const long c = (z * ny + y) * nx + x;
                    if (types[c] != 0) {
                        b[c] = 0.0;
                        continue;
                    }
                    const double uR = solid(x + 1, y, z) ? (bu ? bu[ui(x + 1, y, z)] : 0.0) : u[ui(x + 1, y, z)];
                    const double uL = solid(x - 1, y, z) ? (bu ? bu[ui(x, y, z)] : 0.0) : u[ui(x, y, z)];
                    const double vT = solid(x, y + 1, z) ? (bv ? bv[vi(x, y + 1, z)] : 0.0) : v[vi(x, y + 1, z)];
                    const double vB = solid(x, y - 1, z) ? (bv ? bv[vi(x, y, z)] : 0.0) : v[vi(x, y, z)];
                    double div = (uR - uL) + (vT - vB);
                    if (D == 3) {
                        const double wF = solid(x, y, z + 1) ? (bw ? bw[wi(x, y, z + 1)] : 0.0) : w[wi(x, y, z + 1)];
                        const double wB = solid(x, y, z - 1) ? (bw ? bw[wi(x, y, z)] : 0.0) : w[wi(x, y, z)];
                        div = div + (wF - wB);
                    }
                    b[c] = scale * div;
                }
    });
}

// y = A x on the reduced system of a cell-type grid, without a network
// context (matrix-free PoissonOp; large-grid residual checks)
int oracle_spmv(int D, long nx, long ny, long nz, const unsigned char* types, const double* x, double* y) {
    return guarded([&] {
        const Dims d = make_dims(D, nx, ny, nz);
        const auto map = ReductionMap::from_types(types, d);
        const std::size_t nf = static_cast<std::size_t>(map.reduced_size());
        Vector xv(x, x + nf), yv;
        if (D == 2) {
            PoissonOp<2> A{d, types, &map};
            A.spmv(xv, yv);
        } else {
            PoissonOp<3> A{d, types, &map};
            A.spmv(xv, yv);
        }
        std::memcpy(y, yv.data(), nf * sizeof(double));
    });
}

int oracle_ctx_spmv(void* h, const double* x, double* y) {
    return guarded([&] {
        auto* c = static_cast<OracleCtx*>(h);
        const std::size_t nf = static_cast<std::size_t>(c->map.reduced_size());
        Vector xv(x, x + nf), yv;
        if (c->D == 2) {
            PoissonOp<2> A{c->d, c->types.data(), &c->map};
            A.spmv(xv, yv);
        } else {
            PoissonOp<3> A{c->d, c->types.data(), &c->map};
            A.spmv(xv, yv);
        }
        std::memcpy(y, yv.data(), nf * sizeof(double));
    });
}

// psdo_solve (solver.cpp:189-276). use_identity != 0 selects IdentityPrecond.
// hist must hold max_iters + 1 doubles. Returns the status; iterations,
// converged and the history length are written even on breakdown.
int oracle_ctx_psdo_solve(void* h, int use_identity, const double* b, const double* x0, double tol_reduction,
                          double tol_abs, long max_iters, int n_ortho, int nullspace_projection,
                          int normalize_before_precond, double* x_out, double* hist, long* iterations,
                          int* converged, long* hist_len, double* seconds) {
    return guarded([&] {
        auto* c = static_cast<OracleCtx*>(h);
        if (c->map.reduced_size() == 0) throw EmptySystemError("reduce: image has no fluid cells");
        const std::size_t nf = static_cast<std::size_t>(c->map.reduced_size());
        SolveConfig cfg;
        cfg.tol_reduction = tol_reduction;
        cfg.tol_abs = tol_abs;
        cfg.max_iters = max_iters;
        cfg.n_ortho = n_ortho;
        cfg.nullspace_projection = nullspace_projection != 0;
        cfg.normalize_before_precond = normalize_before_precond != 0;
        Vector bv(b, b + nf), x0v, xv;
        if (x0) x0v.assign(x0, x0 + nf);
        IdentityPrecond id;
        BorrowedNeural nn(c);
        const Precond& P = use_identity ? static_cast<const Precond&>(id) : static_cast<const Precond&>(nn);
        const auto t0 = std::chrono::steady_clock::now();
        SolveReport rep;
        if (c->D == 2) {
            PoissonOp<2> A{c->d, c->types.data(), &c->map};
            rep = psdo_solve(A, bv, P, cfg, x0 ? &x0v : nullptr, xv);
        } else {
            PoissonOp<3> A{c->d, c->types.data(), &c->map};
            rep = psdo_solve(A, bv, P, cfg, x0 ? &x0v : nullptr, xv);
        }
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(x_out, xv.data(), nf * sizeof(double));
        for (std::size_t i = 0; i < rep.residual_history.size(); ++i) hist[i] = rep.residual_history[i];
        *iterations = static_cast<long>(rep.iterations);
        *converged = rep.converged ? 1 : 0;
        *hist_len = static_cast<long>(rep.residual_history.size());
    });
}

}  // extern "C"

// ============================================================================
// TEST INFRASTRUCTURE — NOT THE PRODUCT.
//
// extern "C" shim over the REAL reference library, compiled by oracle/Makefile
// from the unmodified sources under /root/reference/proj/src into
// oracle/_ref/libnpsd_ref.so. Used (a) to pin the CPU restatement
// (npsd_oracle.hpp) bitwise in 2D, (b) to run the reference's own psdo_solve
// with a B200 preconditioner plugged in through a C callback (the drop-in
// check), and (c) as bench.py's CPU baseline: reference psdo_solve on the
// reference assemble_poisson_3d + reduce, preconditioned by the 3D network
// restatement wrapped as an npsd::Preconditioner (the reference has no 3D net).
// ============================================================================
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "npsd/bench.hpp"
#include "npsd/discretization.hpp"
#include "npsd/net/forward.hpp"
#include "npsd/net/precond.hpp"
#include "npsd/precond.hpp"
#include "npsd/rng.hpp"
#include "npsd/scene.hpp"
#include "npsd/solver.hpp"
#include "npsd/train/train.hpp"
#include "npsd_oracle.hpp"

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
    } catch (const npsd::SolverBreakdown& e) {
        g_err = e.what();
        return 2;
    } catch (const npsd::EmptySystemError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

// 3D volumes run through the 2D reference API on a flattened (nx, ny*nz)
// image: its linear index y'*nx + x equals (z*ny + y)*nx + x.
npsd::IndicatorImage image_from_types(long nx, long rows, const unsigned char* types) {
    npsd::IndicatorImage I(nx, rows, npsd::CellType::fluid);
    for (long y = 0; y < rows; ++y)
        for (long x = 0; x < nx; ++x) I.set_cell(x, y, static_cast<npsd::CellType>(types[y * nx + x]));
    return I;
}

npsd::net::NetParams params_2d(int depth, const float* flat, long n) {
    npsd::net::NetParams p;
    p.depth = depth;
    p.levels.resize(static_cast<std::size_t>(depth - 1));
    npsd::require(n == p.parameter_count(), "ref: param length mismatch");
    std::size_t o = 0;
    p.for_each_span([&](float* dst, std::size_t k) {
        std::memcpy(dst, flat + o, k * sizeof(float));
        o += k;
    });
    return p;
}

// The 3D network restatement as a reference Preconditioner.
class NeuralPrecond3D : public npsd::Preconditioner {
public:
    NeuralPrecond3D(const npsdo::Params& p, const unsigned char* types, npsdo::Dims d)
        : map_(npsdo::ReductionMap::from_types(types, d)), P_(p, types, d, &map_) {}
    using Preconditioner::apply;
    void apply(const npsd::Vector& r, npsd::Vector& z) const override { P_.apply(r, z); }
    bool is_linear() const override { return true; }
    bool is_symmetric() const override { return false; }
    npsd::index_t size() const override { return map_.reduced_size(); }
    std::string name() const override { return "neural3d"; }

private:
    npsdo::ReductionMap map_;
    npsdo::NeuralPrecond<3> P_;
};

typedef int (*apply_cb)(void* user, const double* r, double* z, long n);

class CallbackPrecond : public npsd::Preconditioner {
public:
    CallbackPrecond(apply_cb fn, void* user, long n) : fn_(fn), user_(user), n_(n) {}
    using Preconditioner::apply;
    void apply(const npsd::Vector& r, npsd::Vector& z) const override {
        z.assign(r.size(), 0.0);
        if (fn_(user_, r.data(), z.data(), static_cast<long>(r.size())) != 0)
            throw std::runtime_error("callback preconditioner failed");
    }
    bool is_linear() const override { return true; }
    bool is_symmetric() const override { return false; }
    npsd::index_t size() const override { return n_; }
    std::string name() const override { return "callback"; }

private:
    apply_cb fn_;
    void* user_;
    long n_;
};

npsd::SparseMatrix assemble(int dim, long nx, long ny, long nz, const npsd::IndicatorImage& I,
                            const unsigned char* types) {
    if (dim == 2) return npsd::assemble_poisson(I);
    npsd::IndicatorVolume V(nx, ny, nz);
    for (long i = 0; i < nx * ny * nz; ++i) V.cells[static_cast<std::size_t>(i)] = static_cast<npsd::CellType>(types[i]);
    return npsd::assemble_poisson_3d(V);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rhs_normal(unsigned long long seed, long n, double* out) {
    npsd::Rng rng(seed);
    for (long i = 0; i < n; ++i) out[i] = rng.normal();
}

int ref_init_params_2d(int depth, unsigned long long seed, float* out) {
    return guarded([&] {
        const auto p = npsd::net::init_params(depth, seed);
        std::size_t o = 0;
        p.for_each_span([&](const float* src, std::size_t k) {
            std::memcpy(out + o, src, k * sizeof(float));
            o += k;
        });
    });
}

// the reference's mac_divergence_rhs (2D) on a cell-type grid, full-grid output
int ref_mac_rhs_2d(long nx, long ny, const unsigned char* types, const double* u, const double* v, double h,
                   double dt, double rho, const double* bu, const double* bv, double* out) {
    return guarded([&] {
        npsd::MacVelocity vel(nx, ny, h, dt, rho);
        std::memcpy(vel.u.data.data(), u, vel.u.data.size() * sizeof(double));
        std::memcpy(vel.v.data.data(), v, vel.v.data.size() * sizeof(double));
        npsd::BoundaryVelocity bc;
        if (bu) {
            bc.u = vel.u;
            bc.v = vel.v;
            std::memcpy(bc.u.data.data(), bu, bc.u.data.size() * sizeof(double));
            std::memcpy(bc.v.data.data(), bv, bc.v.data.size() * sizeof(double));
        }
        const auto b = npsd::mac_divergence_rhs(vel, image_from_types(nx, ny, types), bu ? &bc : nullptr);
        std::memcpy(out, b.data(), b.size() * sizeof(double));
    });
}

// the reference's bench CSV contract (bench.cpp:139-263): parse a rows.csv
// with load_bench_rows, then write rows.csv / summary.csv / speedup_hist.csv
// with the reference's writers into out_dir
int ref_bench_roundtrip(const char* rows_csv, const char* out_dir) {
    return guarded([&] {
        npsd::BenchReport rep;
        rep.rows = npsd::load_bench_rows(rows_csv);
        rep.traces.resize(rep.rows.size());
        npsd::write_bench_outputs(rep, out_dir);
        npsd::write_bench_report(rep.rows, out_dir);
    });
}

// the reference's own model-file writer / reader (net_params.cpp:42-78)
int ref_save_npm_2d(int depth, unsigned long long seed, const char* path) {
    return guarded([&] { npsd::net::save_npm(npsd::net::init_params(depth, seed), path); });
}

int ref_load_npm_2d(const char* path, float* out, long cap, int* depth) {
    return guarded([&] {
        const auto p = npsd::net::load_npm(path);
        *depth = p.depth;
        long o = 0;
        p.for_each_span([&](const float* src, std::size_t k) {
            if (o + (long)k <= cap) std::memcpy(out + o, src, k * sizeof(float));
            o += (long)k;
        });
    });
}

// PaddedImage::pooled chain interiors (3 planes per level)
int ref_level_images_2d(long nx, long ny, int depth, const unsigned char* types, float* out) {
    return guarded([&] {
        auto img = npsd::net::PaddedImage<float>::from_image(image_from_types(nx, ny, types));
        std::size_t o = 0;
        for (int l = 0; l < depth; ++l) {
            for (int c = 0; c < 3; ++c)
                for (long y = 0; y < img.ny; ++y)
                    for (long x = 0; x < img.nx; ++x) out[o++] = img.at(c, x, y);
            if (l + 1 < depth) img = img.pooled();
        }
    });
}

int ref_net_apply_2d(long nx, long ny, int depth, const float* params, long n_params, const unsigned char* types,
                     const float* x, float* y, float* za, float* zb) {
    return guarded([&] {
        const auto p = params_2d(depth, params, n_params);
        const auto ctx = npsd::net::NetContext<float>::build(p, image_from_types(nx, ny, types));
        npsd::Field2D<float> f(nx, ny);
        std::memcpy(f.data.data(), x, sizeof(float) * static_cast<std::size_t>(nx * ny));
        const auto out = ctx.apply(f);
        std::memcpy(y, out.data.data(), sizeof(float) * static_cast<std::size_t>(nx * ny));
        for (int l = 0; l + 1 < depth; ++l) {
            if (za) za[l] = ctx.levels[static_cast<std::size_t>(l)].z_a;
            if (zb) zb[l] = ctx.levels[static_cast<std::size_t>(l)].z_b;
        }
    });
}

// The reference's hand-written training gradient (train.hpp:94-150,
// net/backward.hpp:46-169): backward_batch<float> on the reference assembly +
// reduce of a 2D frame, for nb reduced right-hand sides (row-major nb x n_f);
// the mean batch loss and the gradient in for_each_span order.
int ref_backward_2d(long nx, long ny, int depth, const float* params, long n_params, const unsigned char* types,
                    const double* rhs, int nb, double* loss, float* grads) {
    return guarded([&] {
        const auto I = image_from_types(nx, ny, types);
        const auto A = npsd::assemble_poisson(I);
        const auto sys = npsd::reduce(A, npsd::Vector(static_cast<std::size_t>(A.n_rows), 0.0), I);
        const std::size_t nf = static_cast<std::size_t>(sys.A.n_rows);
        std::vector<npsd::Vector> bs(static_cast<std::size_t>(nb));
        std::vector<const npsd::Vector*> batch;
        for (int i = 0; i < nb; ++i) {
            bs[static_cast<std::size_t>(i)].assign(rhs + static_cast<std::size_t>(i) * nf, rhs + (static_cast<std::size_t>(i) + 1) * nf);
            batch.push_back(&bs[static_cast<std::size_t>(i)]);
        }
        auto [l, g] = npsd::backward_batch<float>(params_2d(depth, params, n_params), I, sys.A, sys.map, batch);
        *loss = l;
        std::size_t o = 0;
        g.for_each_span([&](float* src, std::size_t k) {
            std::memcpy(grads + o, src, k * sizeof(float));
            o += k;
        });
    });
}

int ref_precond_apply_2d(long nx, long ny, int depth, const float* params, long n_params, const unsigned char* types,
                         const double* r, double* z) {
    return guarded([&] {
        const auto I = image_from_types(nx, ny, types);
        const auto map = npsd::ReductionMap::from_image(I);
        npsd::net::NeuralPrecond P(params_2d(depth, params, n_params), I, map);
        npsd::Vector rv(r, r + map.reduced_size()), zv;
        P.apply(rv, zv);
        std::memcpy(z, zv.data(), sizeof(double) * zv.size());
    });
}

int ref_spmv(int dim, long nx, long ny, long nz, const unsigned char* types, const double* x, double* y) {
    return guarded([&] {
        const long rows = (dim == 3) ? ny * nz : ny;
        const auto I = image_from_types(nx, rows, types);
        const auto A = assemble(dim, nx, ny, nz, I, types);
        const auto sys = npsd::reduce(A, npsd::Vector(static_cast<std::size_t>(A.n_rows), 0.0), I);
        npsd::Vector xv(x, x + sys.A.n_rows), yv;
        npsd::spmv(sys.A, xv, yv);
        std::memcpy(y, yv.data(), sizeof(double) * yv.size());
    });
}

// Reference psdo_solve (solver.cpp:189-276) on the reference assembly.
//   mode 0: IdentityPrecond
//   mode 1: neural — 2D: reference NeuralPrecond; 3D: NeuralPrecond3D restatement
//   mode 2: C callback preconditioner (a B200 NeuralPrecond through the C ABI)
// seconds[0] = setup (assembly + reduce + preconditioner build), seconds[1] = solve.
int ref_psdo_solve(int dim, long nx, long ny, long nz, const unsigned char* types, int mode, int depth,
                   const float* params, long n_params, apply_cb cb, void* cb_user, const double* b,
                   const double* x0, double tol_reduction, double tol_abs, long max_iters, int n_ortho,
                   int nullspace_projection, int normalize_before_precond, double* x_out, double* hist,
                   long* iterations, int* converged, long* hist_len, double* seconds) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const long rows = (dim == 3) ? ny * nz : ny;
        const auto I = image_from_types(nx, rows, types);
        const auto A = assemble(dim, nx, ny, nz, I, types);
        const auto sys = npsd::reduce(A, npsd::Vector(static_cast<std::size_t>(A.n_rows), 0.0), I);
        std::unique_ptr<npsd::Preconditioner> P;
        if (mode == 0) {
            P = npsd::identity_precond(sys.A.n_rows);
        } else if (mode == 1) {
            if (dim == 2)
                P = npsd::net::neural_precond(params_2d(depth, params, n_params), I, sys.map);
            else
                P = std::make_unique<NeuralPrecond3D>(npsdo::params_from_flat(3, depth, params, static_cast<std::size_t>(n_params)),
                                                      types, npsdo::Dims{nx, ny, nz});
        } else {
            P = std::make_unique<CallbackPrecond>(cb, cb_user, sys.A.n_rows);
        }
        const auto t1 = std::chrono::steady_clock::now();
        npsd::SolveConfig cfg;
        cfg.tol_reduction = tol_reduction;
        cfg.tol_abs = tol_abs;
        cfg.max_iters = max_iters;
        cfg.n_ortho = n_ortho;
        cfg.nullspace_projection = nullspace_projection != 0;
        cfg.normalize_before_precond = normalize_before_precond != 0;
        const std::size_t nf = static_cast<std::size_t>(sys.A.n_rows);
        npsd::Vector bv(b, b + nf), x0v;
        if (x0) x0v.assign(x0, x0 + nf);
        const auto res = npsd::psdo_solve(sys.A, bv, *P, cfg, x0 ? &x0v : nullptr);
        const auto t2 = std::chrono::steady_clock::now();
        std::memcpy(x_out, res.x.data(), nf * sizeof(double));
        for (std::size_t i = 0; i < res.report.residual_history.size(); ++i) hist[i] = res.report.residual_history[i];
        *iterations = static_cast<long>(res.report.iterations);
        *converged = res.report.converged ? 1 : 0;
        *hist_len = static_cast<long>(res.report.residual_history.size());
        if (seconds) {
            seconds[0] = std::chrono::duration<double>(t1 - t0).count();
            seconds[1] = std::chrono::duration<double>(t2 - t1).count();
        }
    });
}

// Reference pcg_solve (solver.cpp:36-102) on the reference assembly:
// precond 0 = IdentityPrecond (cg_solve), 1 = JacobiPrecond, 2 = Ic0Precond.
int ref_pcg_solve(int dim, long nx, long ny, long nz, const unsigned char* types, int precond, const double* b,
                  double tol_reduction, long max_iters, double* x_out, double* hist, long* iterations, int* converged,
                  long* hist_len, int nullspace) {
    return guarded([&] {
        const long rows = (dim == 3) ? ny * nz : ny;
        const auto I = image_from_types(nx, rows, types);
        const auto A = assemble(dim, nx, ny, nz, I, types);
        const auto sys = npsd::reduce(A, npsd::Vector(static_cast<std::size_t>(A.n_rows), 0.0), I);
        auto P = precond == 2 ? npsd::ic0_precond(sys.A)
                 : precond == 1 ? npsd::jacobi_precond(sys.A)
                                : npsd::identity_precond(sys.A.n_rows);
        npsd::SolveConfig cfg;
        cfg.tol_reduction = tol_reduction;
        cfg.max_iters = max_iters;
        cfg.nullspace_projection = nullspace != 0;
        const std::size_t nf = static_cast<std::size_t>(sys.A.n_rows);
        npsd::Vector bv(b, b + nf);
        const auto res = npsd::pcg_solve(sys.A, bv, *P, cfg, nullptr);
        std::memcpy(x_out, res.x.data(), nf * sizeof(double));
        for (std::size_t i = 0; i < res.report.residual_history.size(); ++i) hist[i] = res.report.residual_history[i];
        *iterations = static_cast<long>(res.report.iterations);
        *converged = res.report.converged ? 1 : 0;
        *hist_len = static_cast<long>(res.report.residual_history.size());
    });
}

// Reference Ic0Precond (precond.cpp:28-112) on the reference assembly:
// constructor (factorization with shift retries) + apply.
int ref_ic0_apply(int dim, long nx, long ny, long nz, const unsigned char* types, const double* r, double* z,
                  int* shift_retries) {
    return guarded([&] {
        const long rows = (dim == 3) ? ny * nz : ny;
        const auto I = image_from_types(nx, rows, types);
        const auto A = assemble(dim, nx, ny, nz, I, types);
        const auto sys = npsd::reduce(A, npsd::Vector(static_cast<std::size_t>(A.n_rows), 0.0), I);
        npsd::Ic0Precond P(sys.A);
        const std::size_t nf = static_cast<std::size_t>(sys.A.n_rows);
        npsd::Vector rv(r, r + nf), zv;
        P.apply(rv, zv);
        std::memcpy(z, zv.data(), nf * sizeof(double));
        *shift_retries = P.shift_retries();
    });
}

}  // extern "C"

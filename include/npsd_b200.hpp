// npsd_b200.hpp — header-only C++ shim that puts the B200 path behind the
// reference's own interfaces (/root/reference/proj/include/npsd):
//
//   npsd::b200::NeuralPrecond  : npsd::Preconditioner      (precond.hpp:12-29;
//                                same ctor as net::NeuralPrecond, net/precond.hpp:14-30)
//   npsd::b200::neural_precond                                (net/precond.hpp:32-33)
//   npsd::b200::IdentityPrecond : npsd::Preconditioner     (precond.hpp:35-43)
//   npsd::b200::psdo_solve / psd_solve                        (solver.hpp:64-69)
//
// The reference's psdo_solve can drive a b200::NeuralPrecond unchanged (host
// vectors through Preconditioner::apply); b200::psdo_solve runs the whole
// loop on the device. Errors are rethrown as the reference's exception types.
// Build against the reference include path plus this directory, link
// libnpsd_b200.so. There is no CPU fallback.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "npsd/discretization.hpp"
#include "npsd/net/params.hpp"
#include "npsd/precond.hpp"
#include "npsd/solver.hpp"
#include "npsd_b200.h"

namespace npsd::b200 {

inline void check(int st, const npsd_b200_ctx* c) {
    if (st == NPSD_OK) return;
    const std::string msg = npsd_b200_last_error(c);
    switch (st) {
        case NPSD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case NPSD_BREAKDOWN: throw SolverBreakdown(msg);
        case NPSD_EMPTY_SYSTEM: throw EmptySystemError(msg);
        default: throw std::runtime_error("npsd_b200: " + msg);
    }
}

inline std::vector<float> flatten(const net::NetParams& p) {
    std::vector<float> out;
    out.reserve(static_cast<std::size_t>(p.parameter_count()));
    p.for_each_span([&](const float* s, std::size_t n) { out.insert(out.end(), s, s + n); });
    return out;
}

// cell types (0 fluid, 1 air, 2 solid) of an image / volume, x fastest
inline std::vector<uint8_t> types_of(const IndicatorImage& I) {
    std::vector<uint8_t> t(static_cast<std::size_t>(I.cells()));
    for (index_t y = 0; y < I.ny; ++y)
        for (index_t x = 0; x < I.nx; ++x)
            t[static_cast<std::size_t>(y * I.nx + x)] = static_cast<uint8_t>(cell_type(I, x, y));
    return t;
}
inline std::vector<uint8_t> types_of(const IndicatorVolume& V) {
    std::vector<uint8_t> t(V.cells.size());
    for (std::size_t i = 0; i < t.size(); ++i) t[i] = static_cast<uint8_t>(V.cells[i]);
    return t;
}

class NeuralPrecond : public Preconditioner {
public:
    // 2D: the reference constructor (net_precond.cpp:9-12); throws on a map/image mismatch.
    NeuralPrecond(const net::NetParams& params, const IndicatorImage& I, const ReductionMap& map, int device = 0)
        : NeuralPrecond(2, I.nx, I.ny, 1, params.depth, flatten(params), types_of(I), device) {
        require(map.full_size == I.cells() && map.reduced_size() == size(), "NeuralPrecond: map does not match image");
    }
    // 3D: weights in for_each_span order with 27 slots, cell-type volume.
    NeuralPrecond(const std::vector<float>& params, int depth, const IndicatorVolume& V, int device = 0)
        : NeuralPrecond(3, V.nx, V.ny, V.nz, depth, params, types_of(V), device) {}

    NeuralPrecond(const NeuralPrecond&) = delete;
    NeuralPrecond& operator=(const NeuralPrecond&) = delete;
    ~NeuralPrecond() override { npsd_b200_destroy(ctx_); }

    using Preconditioner::apply;
    // Preconditioner::apply (precond.hpp:17) with NeuralPrecond semantics
    // (net_precond.cpp:14-35); reentrant (calls serialise on the context).
    void apply(const Vector& r, Vector& z) const override {
        require(static_cast<index_t>(r.size()) == size(), "NeuralPrecond::apply: size mismatch");
        z.assign(r.size(), 0.0);
        check(npsd_b200_precond_apply(ctx_, r.data(), z.data(), static_cast<int64_t>(r.size())), ctx_);
    }
    bool is_linear() const override { return true; }
    bool is_symmetric() const override { return false; }
    index_t size() const override { return static_cast<index_t>(npsd_b200_n_fluid(ctx_)); }
    std::string name() const override { return "neural"; }

    npsd_b200_ctx* context() const { return ctx_; }

private:
    NeuralPrecond(int dim, index_t nx, index_t ny, index_t nz, int depth, const std::vector<float>& params,
                  const std::vector<uint8_t>& types, int device) {
        check(npsd_b200_create(dim, static_cast<int>(nx), static_cast<int>(ny), static_cast<int>(nz), depth,
                               params.data(), params.size(), &device, 1, &ctx_),
              nullptr);
        const int st = npsd_b200_set_mask(ctx_, types.data());
        if (st != NPSD_OK) {
            const std::string msg = npsd_b200_last_error(ctx_);
            npsd_b200_destroy(ctx_);
            throw std::invalid_argument(msg);
        }
    }
    npsd_b200_ctx* ctx_ = nullptr;
};

// IdentityPrecond (precond.hpp:35-43, precond.cpp:7-10) for b200::psdo_solve:
// apply copies like the reference's; inside b200::psdo_solve the device loop
// forms d = r / ||r|| without the network. The image gives the device its
// matrix-free operator (an IdentityPrecond alone carries no grid).
class IdentityPrecond : public Preconditioner {
public:
    explicit IdentityPrecond(const IndicatorImage& I, int device = 0) : IdentityPrecond(2, I.nx, I.ny, 1, types_of(I), device) {}
    explicit IdentityPrecond(const IndicatorVolume& V, int device = 0)
        : IdentityPrecond(3, V.nx, V.ny, V.nz, types_of(V), device) {}
    IdentityPrecond(const IdentityPrecond&) = delete;
    IdentityPrecond& operator=(const IdentityPrecond&) = delete;
    ~IdentityPrecond() override { npsd_b200_destroy(ctx_); }

    using Preconditioner::apply;
    void apply(const Vector& r, Vector& z) const override {
        require(static_cast<index_t>(r.size()) == size(), "IdentityPrecond::apply: size mismatch");
        z = r;
    }
    bool is_linear() const override { return true; }
    bool is_symmetric() const override { return true; }
    index_t size() const override { return static_cast<index_t>(npsd_b200_n_fluid(ctx_)); }
    std::string name() const override { return "identity"; }
    npsd_b200_ctx* context() const { return ctx_; }

private:
    IdentityPrecond(int dim, index_t nx, index_t ny, index_t nz, const std::vector<uint8_t>& types, int device) {
        std::vector<float> p(npsd_b200_param_count(dim, 1));  // the network is never run: depth 1
        check(npsd_b200_identity_params(dim, 1, p.data()), nullptr);
        check(npsd_b200_create(dim, static_cast<int>(nx), static_cast<int>(ny), static_cast<int>(nz), 1, p.data(),
                               p.size(), &device, 1, &ctx_),
              nullptr);
        const int st = npsd_b200_set_mask(ctx_, types.data());
        if (st != NPSD_OK) {
            const std::string msg = npsd_b200_last_error(ctx_);
            npsd_b200_destroy(ctx_);
            throw std::invalid_argument(msg);
        }
    }
    npsd_b200_ctx* ctx_ = nullptr;
};

// How b200::psdo_solve checks the caller's A against the flag-derived operator
// (npsd_b200_check_operator): rows = every row's nnz, diagonal and -1
// off-diagonals (always, O(nnz) on the host); full = also A v bitwise (debug).
enum class OperatorCheck { rows, full };
inline OperatorCheck& operator_check() {
    static OperatorCheck mode = OperatorCheck::rows;
    return mode;
}

inline std::unique_ptr<Preconditioner> neural_precond(const net::NetParams& params, const IndicatorImage& I,
                                                      const ReductionMap& map) {
    return std::make_unique<NeuralPrecond>(params, I, map);
}

// psdo_solve (solver.cpp:189-276) with the loop on the device. The operator is
// the flag-derived mixed-BC Laplacian of P's grid — the matrix
// assemble_poisson[_3d] + reduce build — and A is checked against it
// (operator_check()): a different A throws invalid_argument rather than
// solving another system. P must be a b200::NeuralPrecond or a
// b200::IdentityPrecond (no CPU path).
inline SolveResult psdo_solve(const SparseMatrix& A, const Vector& b, const Preconditioner& P, const SolveConfig& cfg,
                              const Vector* x0 = nullptr) {
    npsd_b200_ctx* ctx = nullptr;
    int precond = 0;
    if (const auto* np = dynamic_cast<const NeuralPrecond*>(&P)) {
        ctx = np->context();
    } else if (const auto* ip = dynamic_cast<const IdentityPrecond*>(&P)) {
        ctx = ip->context();
        precond = 1;
    }
    require(ctx != nullptr, "b200::psdo_solve: P must be a b200::NeuralPrecond or b200::IdentityPrecond");
    require(A.n_rows == A.n_cols, "solve: matrix not square");
    require(static_cast<index_t>(b.size()) == A.n_rows && A.n_rows == P.size(), "solve: rhs length mismatch");
    if (x0) require(static_cast<index_t>(x0->size()) == A.n_rows, "solve: x0 length mismatch");
    static_assert(sizeof(index_t) == sizeof(int64_t), "CSR indices are int64");
    check(npsd_b200_check_operator(ctx, A.n_rows, reinterpret_cast<const int64_t*>(A.row_offsets.data()),
                                   reinterpret_cast<const int64_t*>(A.col_indices.data()), A.values.data(),
                                   static_cast<int64_t>(A.values.size()), operator_check() == OperatorCheck::full),
          ctx);
    npsd_b200_solve_cfg c{cfg.tol_reduction, cfg.tol_abs, static_cast<int64_t>(cfg.max_iters), cfg.n_ortho,
                          cfg.nullspace_projection ? 1 : 0, cfg.normalize_before_precond ? 1 : 0, precond};
    SolveResult res;
    res.x.assign(b.size(), 0.0);
    npsd_b200_report rep{};
    const int st = npsd_b200_psdo_solve(ctx, b.data(), x0 ? x0->data() : nullptr, &c, res.x.data(), &rep);
    check(st, ctx);
    res.report.iterations = rep.iterations;
    res.report.converged = rep.converged != 0;
    res.report.residual_history.assign(rep.residual_history, rep.residual_history + rep.history_len);
    res.report.cumulative_seconds.assign(rep.cumulative_seconds, rep.cumulative_seconds + rep.history_len);
    res.report.setup_seconds = rep.setup_seconds;
    res.report.iterate_seconds = rep.iterate_seconds;
    res.report.precond_seconds = rep.precond_seconds;
    res.report.method = "psdo+" + P.name();
    return res;
}

inline SolveResult psd_solve(const SparseMatrix& A, const Vector& b, const Preconditioner& P, const SolveConfig& cfg,
                             const Vector* x0 = nullptr) {
    SolveConfig c = cfg;
    c.n_ortho = 0;
    SolveResult res = b200::psdo_solve(A, b, P, c, x0);
    res.report.method = "psd+" + P.name();
    return res;
}

}  // namespace npsd::b200

// TEST INFRASTRUCTURE — the drop-in check from the reference's side.
//
// Built by oracle/Makefile (target `dropin`) against the UNMODIFIED reference
// headers and objects plus include/npsd_b200.hpp and libnpsd_b200.so; run on
// the GPU by tests/test_gpu_dropin.py. It swaps the reference's
// net::neural_precond for npsd::b200::neural_precond inside the reference's
// own psdo_solve, and also runs npsd::b200::psdo_solve (device loop), on a 2D
// mixed-BC frame built with the reference's rasterize / assemble / reduce.
// Prints one JSON line.
#include <cmath>
#include <cstdio>

#include "npsd/discretization.hpp"
#include "npsd/net/precond.hpp"
#include "npsd/rng.hpp"
#include "npsd/scene.hpp"
#include "npsd/solver.hpp"
#include "npsd_b200.hpp"

using namespace npsd;

int main() {
    // test_solvers.cpp:17-28 pattern at 64^2: air above 0.75n, solid box in a corner
    const index_t n = 64;
    SceneSpec spec;
    spec.nx = spec.ny = n;
    spec.prims.push_back({Primitive::Shape::half_plane, CellType::air, 0.0, 1.0, 0.75 * n, 0.0});
    spec.prims.push_back({Primitive::Shape::box, CellType::solid, 0.0, 0.0, 0.3 * n, 0.2 * n});
    const IndicatorImage I = rasterize(spec);
    const SparseMatrix A = assemble_poisson(I);
    Rng rng(7);
    Vector bfull(static_cast<std::size_t>(A.n_rows));
    for (auto& v : bfull) v = rng.normal();
    const ReducedSystem sys = reduce(A, bfull, I);

    // random weights: a fixed 20-iteration budget, histories compared
    const net::NetParams pr = net::init_params(3, 42);
    SolveConfig budget;
    budget.max_iters = 20;
    budget.tol_reduction = 1e-300;
    const auto cpu_p = net::neural_precond(pr, I, sys.map);
    const auto gpu_p = b200::neural_precond(pr, I, sys.map);
    // the reference's operation order in the network (bitwise to the CPU
    // network), so the 20-iteration histories compare at the f64 level
    b200::check(npsd_b200_set_exact(static_cast<b200::NeuralPrecond*>(gpu_p.get())->context(), 1), nullptr);
    const SolveResult ref_cpu = psdo_solve(sys.A, sys.b, *cpu_p, budget);
    const SolveResult ref_gpu = psdo_solve(sys.A, sys.b, *gpu_p, budget);  // reference solver, B200 precond
    double hist_rel = 0.0;
    for (std::size_t i = 0; i < ref_cpu.report.residual_history.size(); ++i)
        hist_rel = std::max(hist_rel, std::abs(ref_cpu.report.residual_history[i] - ref_gpu.report.residual_history[i]) /
                                          ref_cpu.report.residual_history[i]);
    Vector zc, zg;
    cpu_p->apply(sys.b, zc);
    gpu_p->apply(sys.b, zg);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < zc.size(); ++i) {
        num += (zc[i] - zg[i]) * (zc[i] - zg[i]);
        den += zc[i] * zc[i];
    }

    // identity-equivalent weights: time to rel-res 1e-6, device loop vs reference
    net::NetParams pid = net::init_params(3, 1);
    pid.for_each_span([](float* p, std::size_t k) {
        for (std::size_t i = 0; i < k; ++i) p[i] = 0.0f;
    });
    for (auto& lv : pid.levels) {
        lv.conv_down.B[4] = 1.0f;
        lv.conv_up.B[4] = 1.0f;
        lv.lin_a.bias = 1.0f;
    }
    pid.coarse.B[4] = 1.0f;
    SolveConfig tts;
    tts.max_iters = 5000;
    const auto cpu_i = net::neural_precond(pid, I, sys.map);
    b200::NeuralPrecond gpu_i(pid, I, sys.map);
    const SolveResult a = psdo_solve(sys.A, sys.b, *cpu_i, tts);
    const SolveResult b = b200::psdo_solve(sys.A, sys.b, gpu_i, tts);
    bool threw = false;
    try {
        SolveConfig bad = tts;
        bad.tol_reduction = 2.0;
        (void)b200::psdo_solve(sys.A, sys.b, gpu_i, bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    // IdentityPrecond: the reference psdo_solve + its IdentityPrecond against the
    // device loop with b200::IdentityPrecond (d = r / ||r||, no network)
    IdentityPrecond id_ref(sys.A.n_rows);
    b200::IdentityPrecond id_gpu(I);
    const SolveResult ia = psdo_solve(sys.A, sys.b, id_ref, tts);
    const SolveResult ib = b200::psdo_solve(sys.A, sys.b, id_gpu, tts);
    double id_hist = 0.0;
    const std::size_t nh = std::min(ia.report.residual_history.size(), ib.report.residual_history.size());
    for (std::size_t i = 0; i < std::min<std::size_t>(nh, 30); ++i)
        id_hist = std::max(id_hist, std::abs(ia.report.residual_history[i] - ib.report.residual_history[i]) /
                                        ia.report.residual_history[i]);

    // A is checked against the flags: a scaled or structurally different A throws
    auto throws_invalid = [&](const SparseMatrix& M) {
        try {
            (void)b200::psdo_solve(M, sys.b, gpu_i, tts);
        } catch (const std::invalid_argument&) {
            return true;
        }
        return false;
    };
    SparseMatrix scaled = sys.A;
    for (auto& v : scaled.values) v *= 2.0;
    SparseMatrix moved = sys.A;  // one off-diagonal column index changed
    for (index_t k = moved.row_offsets[5]; k < moved.row_offsets[6]; ++k)
        if (moved.col_indices[static_cast<std::size_t>(k)] != 5) {
            moved.col_indices[static_cast<std::size_t>(k)] = (moved.col_indices[static_cast<std::size_t>(k)] + 7) % moved.n_rows;
            break;
        }
    const bool scaled_rejected = throws_invalid(scaled);
    b200::operator_check() = b200::OperatorCheck::full;
    const bool moved_rejected = throws_invalid(moved);
    const SolveResult full = b200::psdo_solve(sys.A, sys.b, gpu_i, tts);  // the right A passes the full check
    b200::operator_check() = b200::OperatorCheck::rows;

    // is_pure_neumann (discretization.cpp:180-191): this frame, and a closed box
    IndicatorImage box(16, 16, CellType::fluid);
    for (index_t i = 0; i < 16; ++i) {
        box.set_cell(i, 0, CellType::solid);
        box.set_cell(i, 15, CellType::solid);
        box.set_cell(0, i, CellType::solid);
        box.set_cell(15, i, CellType::solid);
    }
    int pn_frame = -1, pn_box = -1;
    b200::check(npsd_b200_is_pure_neumann(gpu_i.context(), &pn_frame), gpu_i.context());
    b200::IdentityPrecond box_p(box);
    b200::check(npsd_b200_is_pure_neumann(box_p.context(), &pn_box), box_p.context());

    std::printf(
        "{\"n_fluid\": %lld, \"precond_rel_l2\": %.3e, \"budget_hist_max_rel\": %.3e, \"ref_iters\": %lld, "
        "\"b200_iters\": %lld, \"ref_converged\": %d, \"b200_converged\": %d, \"invalid_argument_rethrown\": %d, "
        "\"ident_ref_iters\": %lld, \"ident_b200_iters\": %lld, \"ident_hist_max_rel\": %.3e, "
        "\"scaled_a_rejected\": %d, \"moved_a_rejected\": %d, \"full_check_iters\": %lld, "
        "\"setup_seconds\": %.3e, \"iterate_seconds\": %.3e, \"precond_seconds\": %.3e, \"cum0\": %.3e, "
        "\"cum_last\": %.3e, \"pure_neumann_frame\": %d, \"pure_neumann_frame_ref\": %d, \"pure_neumann_box\": %d, "
        "\"pure_neumann_box_ref\": %d}\n",
        static_cast<long long>(sys.A.n_rows), std::sqrt(num / den), hist_rel,
        static_cast<long long>(a.report.iterations), static_cast<long long>(b.report.iterations),
        a.report.converged ? 1 : 0, b.report.converged ? 1 : 0, threw ? 1 : 0,
        static_cast<long long>(ia.report.iterations), static_cast<long long>(ib.report.iterations), id_hist,
        scaled_rejected ? 1 : 0, moved_rejected ? 1 : 0, static_cast<long long>(full.report.iterations),
        b.report.setup_seconds, b.report.iterate_seconds, b.report.precond_seconds,
        b.report.cumulative_seconds.front(), b.report.cumulative_seconds.back(), pn_frame,
        is_pure_neumann(I) ? 1 : 0, pn_box, is_pure_neumann(box) ? 1 : 0);
    return 0;
}

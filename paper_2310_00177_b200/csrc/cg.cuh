// Preconditioned CG on the device: pcg_solve (src/solver.cpp:36-102) with
// the identity (cg_solve, :104-109), Jacobi (precond.cpp:12-26) or IC0
// (precond.cpp:28-112, level-scheduled triangular sweeps) preconditioner, matrix-free on the cell bytes — the baseline the paper
// compares the neural PSDO against, on the same device path.
//
// One iteration is two kernels (the whole loop under the conditional WHILE
// node of a CUDA graph, like psdo):
//   k_cg_dir:    p = z + beta p, formed over tile + halo in the stencil
//                pipeline (stencil.cuh), Ap = A p, dot p.Ap -> alpha or a
//                breakdown (solver.cpp:74-80). p ping-pongs between two
//                buffers (neighbour blocks still read the old p's halo).
//   k_cg_update: x += alpha p, r += (-alpha) Ap, z = M r, ||r||^2 and r.z ->
//                history, convergence, beta = r.z / r.z_old (:81-99).
// Arithmetic follows the reference line by line (separately rounded); only
// the dot products are deterministic tree reductions instead of serial sums.
// The first iteration uses beta = -0.0: z + (-0.0) p == z exactly, i.e. p = z.
#pragma once

#include "common.cuh"
#include "psdo.cuh"
#include "stencil.cuh"

namespace nb2 {

// operand of the direction kernel: p' = z + beta * p (pcg_solve :99)
struct CgOp {
    static constexpr int NA = 2;  // z, p
    static constexpr int NC = 0;
    static constexpr int PF = STENCIL_PF_UPDATE;
    static constexpr int CS = 0;  // no centre inputs
    const double* in[NA];
    const double* ctr[1];
    double beta;
    __device__ __forceinline__ double value(const double (&a)[NA]) const {
        return __dadd_rn(a[0], __dmul_rn(beta, a[1]));
    }
};

template <int D>
__global__ void __launch_bounds__(kSX* kSY) k_cg_dir(Geom g, const uint8_t* __restrict__ cls,
                                                     const double* __restrict__ z, double* __restrict__ P0,
                                                     double* __restrict__ P1, double* __restrict__ Ap, SolverState* st,
                                                     double* __restrict__ partials, unsigned int* __restrict__ counter,
                                                     Sched sc) {
    CgOp op;
    const int pc = st->pcur;
    op.in[0] = z;
    op.in[1] = pc ? P1 : P0;
    op.ctr[0] = nullptr;
    op.beta = st->beta;
    double* pnew = pc ? P0 : P1;
    double acc[1] = {0.0};
    sched_for_each(sc, [&](int tx, int ty, int zc0, int zc1) {
        stencil_march<D, 1>(g, cls, op, tx, ty, zc0, zc1, acc,
                            [&](long long q, double2 v, double2 s, unsigned, const double(&)[2], const double(&)[2],
                                const double(&)[1], const double(&)[1], double(&a)[1]) {
                                *reinterpret_cast<double2*>(pnew + q) = v;
                                *reinterpret_cast<double2*>(Ap + q) = s;
                                a[0] += v.x * s.x;
                                a[0] += v.y * s.y;
                            });
    });
    double tot[1];
    if (grid_reduce<1>(acc, partials, counter, tot) && threadIdx.x == 0 && threadIdx.y == 0) {
        const double pAp = tot[0];
        if (!(pAp > 0.0) || fabs(pAp) < 1e-300) {
            st->breakdown = 1;
            st->done = 1;
            st->bad_value = pAp;
            st->alpha = 0.0;
        } else {
            st->alpha = st->rz / pAp;
        }
        st->pcur = pc ^ 1;  // the new direction is current
    }
}

// preconditioner modes of the device PCG
constexpr int kCgIdentity = 0, kCgJacobi = 1, kCgIc0 = 2;

// z = M r at one fluid cell: identity, or r * (1 / diag) (JacobiPrecond)
template <bool JACOBI>
__device__ __forceinline__ double cg_precond(double r, uint8_t b) {
    return JACOBI ? __dmul_rn(r, 1.0 / (double)cls_diag(b)) : r;
}

// the residual's norm, z = M r and r.z; the finish of an iteration (or, with
// INIT, of the prologue: r0 is r, history[0], threshold, beta = -0.0).
// MODE kCgIc0: z needs the triangular sweeps that follow, so this kernel only
// updates x, r, ||r|| and the convergence state; k_cg_rz finishes.
// PH: 0 the whole step; with nullspace projection (pcg_solve :82) the step
// splits around mean_project(r): 1 = the two axpys only, 2 = the rest on the
// projected r.
template <int MODE, bool INIT, int PH = 0>
__global__ void __launch_bounds__(kBlock) k_cg_update(Geom g, const uint8_t* __restrict__ cls,
                                                      const double* __restrict__ P0, const double* __restrict__ P1,
                                                      const double* __restrict__ Ap, double* __restrict__ x,
                                                      double* __restrict__ r, double* __restrict__ z, SolverState* st,
                                                      double* __restrict__ hist, double* __restrict__ times,
                                                      double* __restrict__ partials, unsigned int* __restrict__ counter,
                                                      cudaGraphConditionalHandle cond, int use_cond) {
    if (!INIT && st->breakdown) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(cond, use_cond, 0u);
        return;
    }
    const double alpha = INIT ? 0.0 : st->alpha;
    const double* p = st->pcur ? P1 : P0;
    double acc[2] = {0.0, 0.0};
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) != 0) continue;
        double rv = r[c];
        if (!INIT && PH != 2) {
            x[c] = __dadd_rn(x[c], __dmul_rn(alpha, p[c]));     // axpy_inplace(alpha, p, x)
            rv = __dadd_rn(rv, __dmul_rn(-alpha, Ap[c]));       // axpy_inplace(-alpha, Ap, r)
            r[c] = rv;
        }
        if (PH == 1) continue;
        acc[0] += rv * rv;
        if (MODE != kCgIc0) {
            const double zv = cg_precond<MODE == kCgJacobi>(rv, b);
            if (MODE == kCgJacobi) z[c] = zv;
            acc[1] += rv * zv;
        }
    }
    if (PH == 1) return;
    double tot[2];
    if (grid_reduce<2>(acc, partials, counter, tot) && threadIdx.x == 0) {
        const double rn = sqrt(tot[0]);
        st->rnorm = rn;
        const unsigned long long now = globaltimer();
        st->t_mark = now;
        if (INIT) {
            const double setup = (double)(now - st->t0) * 1e-9;  // solver.cpp:57-58
            st->setup_s = setup;
            hist[0] = rn;
            times[0] = setup;
            double thr = st->tol_reduction * rn;
            if (st->tol_abs > 0.0) thr = fmax(thr, st->tol_abs);
            st->thr = thr;
            st->k = 1;
            st->converged = (rn <= thr);
            st->done = st->converged || st->max_iters < 1;
            if (MODE != kCgIc0) {
                st->rz = tot[1];
                st->beta = -0.0;  // p = z on the first direction
            }
        } else {
            const long long k = st->k;
            hist[k] = rn;
            times[k] = (double)(now - st->t0) * 1e-9;
            st->converged = (rn <= st->thr);
            st->done = st->converged || k >= st->max_iters;
            st->k = k + 1;
            if (MODE != kCgIc0 && !st->done) {
                st->beta = tot[1] / st->rz;
                st->rz = tot[1];
            }
        }
        set_cond(cond, use_cond, st->done ? 0u : 1u);
    }
}

// ---------------------------------------------------------------------- IC0
// Ic0Precond (precond.cpp:28-112) on the flag-derived operator. The reduced
// matrix orders fluid cells by linear index, so a row's lower pattern is its
// fluid (z-1, y-1, x-1) neighbours in that column order, each entry -1. For
// this 7-point (5-point) pattern no two rows share a lower column, so the
// up-looking factorization reduces to
//   L_ij = -1 / L_jj                      (off-diagonal, j a lower neighbour)
//   L_ii = sqrt(A_ii + shift - sum_j L_ij^2)   (j in column order)
// and only the diagonal D = L_ii is stored; every off-diagonal value is
// recomputed as (-1.0) / D_j, the reference's own expression, so the factor
// and both triangular solves round exactly as the reference's loops do.
// Dependencies run along x-1, y-1, z-1: cells of one hyperplane x + y + z = h
// are independent, so each sweep is one launch per hyperplane (level
// scheduling), thread per (y, z) of the grid.
template <int MODE>  // 0 factor, 1 forward solve L y = r, 2 backward solve L^T z = y (in place)
__global__ void __launch_bounds__(kBlock) k_ic0_level(Geom g, const uint8_t* __restrict__ cls, int h, double shift,
                                                      double* __restrict__ D, const double* __restrict__ r,
                                                      double* __restrict__ Z, int* __restrict__ fail,
                                                      const SolverState* __restrict__ st) {
    if (st && st->done) return;  // the solve converged (or broke down) before this sweep
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)g.ny * g.nz) return;
    const int y = (int)(t % g.ny), z = (int)(t / g.ny), x = h - y - z;
    if (x < 0 || x >= g.nx) return;
    const long long nx = g.nx, plane = nx * g.ny, c = lin(g, x, y, z);
    const uint8_t b = cls[c];
    if (cls_type(b) != 0) return;
    auto fl = [&](long long q) { return cls_type(cls[q]) == 0; };
    if (MODE == 0) {
        const int diag = cls_diag(b);
        if (diag == 0) {  // the row has no diagonal in its pattern (assemble_poisson drops zeros)
            atomicOr(fail, 2);
            D[c] = 1.0;
            return;
        }
        double v = __dadd_rn((double)diag, shift);
        if (z > 0 && fl(c - plane)) {
            const double L = -1.0 / D[c - plane];
            v = __dadd_rn(v, -__dmul_rn(L, L));
        }
        if (y > 0 && fl(c - nx)) {
            const double L = -1.0 / D[c - nx];
            v = __dadd_rn(v, -__dmul_rn(L, L));
        }
        if (x > 0 && fl(c - 1)) {
            const double L = -1.0 / D[c - 1];
            v = __dadd_rn(v, -__dmul_rn(L, L));
        }
        if (v <= 0.0) {
            atomicOr(fail, 1);
            D[c] = 1.0;
        } else {
            D[c] = __dsqrt_rn(v);
        }
    } else if (MODE == 1) {
        double s = r[c];
        if (z > 0 && fl(c - plane)) s = __dadd_rn(s, -__dmul_rn(-1.0 / D[c - plane], Z[c - plane]));
        if (y > 0 && fl(c - nx)) s = __dadd_rn(s, -__dmul_rn(-1.0 / D[c - nx], Z[c - nx]));
        if (x > 0 && fl(c - 1)) s = __dadd_rn(s, -__dmul_rn(-1.0 / D[c - 1], Z[c - 1]));
        Z[c] = s / D[c];
    } else {
        // the scatter of rows c + plane, c + nx, c + 1 (visited in that, descending, order)
        const double dc = D[c], L = -1.0 / dc;
        double s = Z[c];
        if (z + 1 < g.nz && fl(c + plane)) s = __dadd_rn(s, -__dmul_rn(L, Z[c + plane]));
        if (y + 1 < g.ny && fl(c + nx)) s = __dadd_rn(s, -__dmul_rn(L, Z[c + nx]));
        if (x + 1 < g.nx && fl(c + 1)) s = __dadd_rn(s, -__dmul_rn(L, Z[c + 1]));
        Z[c] = s / dc;
    }
}

// sum of the stencil diagonal over the fluid cells (Ic0Precond's diag_mean)
__global__ void __launch_bounds__(kBlock) k_diag_sum(Geom g, const uint8_t* __restrict__ cls,
                                                     unsigned long long* __restrict__ sum) {
    unsigned long long a = 0;
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) == 0) a += (unsigned long long)cls_diag(b);
    }
    for (int o = 16; o; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0 && a) atomicAdd(sum, a);
}

// r.z after the IC0 sweeps: beta and rz (pcg_solve :96-100), the graph condition
template <bool INIT>
__global__ void __launch_bounds__(kBlock) k_cg_rz(Geom g, const uint8_t* __restrict__ cls, const double* __restrict__ r,
                                                  const double* __restrict__ z, SolverState* st,
                                                  double* __restrict__ partials, unsigned int* __restrict__ counter,
                                                  cudaGraphConditionalHandle cond, int use_cond) {
    if (st->done) {  // every block sees the same flag
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(cond, use_cond, 0u);
        return;
    }
    precond_span_end(st);  // the IC0 sweeps since k_cg_update (solver.cpp:66-70, 94-96)
    double acc[1] = {0.0};
    FOR_OWNED(g, c) {
        if (cls_type(cls[c]) != 0) continue;
        acc[0] += r[c] * z[c];
    }
    double tot[1];
    if (grid_reduce<1>(acc, partials, counter, tot) && threadIdx.x == 0) {
        if (INIT) {
            st->beta = -0.0;  // p = z on the first direction
        } else {
            st->beta = tot[0] / st->rz;
        }
        st->rz = tot[0];
        set_cond(cond, use_cond, 1u);
    }
}

}  // namespace nb2

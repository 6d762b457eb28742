// Preconditioned CG on the device: pcg_solve (src/solver.cpp:36-102) with
// the identity (cg_solve, :104-109) or Jacobi (precond.cpp:12-26)
// preconditioner, matrix-free on the cell bytes — the baseline the paper
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

// z = M r at one fluid cell: identity, or r * (1 / diag) (JacobiPrecond)
template <bool JACOBI>
__device__ __forceinline__ double cg_precond(double r, uint8_t b) {
    return JACOBI ? __dmul_rn(r, 1.0 / (double)cls_diag(b)) : r;
}

// the residual's norm, z = M r and r.z; the finish of an iteration (or, with
// INIT, of the prologue: r0 is r, history[0], threshold, beta = -0.0)
template <bool JACOBI, bool INIT>
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
        if (!INIT) {
            x[c] = __dadd_rn(x[c], __dmul_rn(alpha, p[c]));     // axpy_inplace(alpha, p, x)
            rv = __dadd_rn(rv, __dmul_rn(-alpha, Ap[c]));       // axpy_inplace(-alpha, Ap, r)
            r[c] = rv;
        }
        const double zv = cg_precond<JACOBI>(rv, b);
        if (JACOBI) z[c] = zv;
        acc[0] += rv * rv;
        acc[1] += rv * zv;
    }
    double tot[2];
    if (grid_reduce<2>(acc, partials, counter, tot) && threadIdx.x == 0) {
        const double rn = sqrt(tot[0]);
        st->rnorm = rn;
        const unsigned long long now = globaltimer();
        if (INIT) {
            st->t0 = now;
            hist[0] = rn;
            times[0] = 0.0;
            double thr = st->tol_reduction * rn;
            if (st->tol_abs > 0.0) thr = fmax(thr, st->tol_abs);
            st->thr = thr;
            st->k = 1;
            st->converged = (rn <= thr);
            st->done = st->converged || st->max_iters < 1;
            st->rz = tot[1];
            st->beta = -0.0;  // p = z on the first direction
        } else {
            const long long k = st->k;
            hist[k] = rn;
            times[k] = (double)(now - st->t0) * 1e-9;
            st->converged = (rn <= st->thr);
            st->done = st->converged || k >= st->max_iters;
            st->k = k + 1;
            if (!st->done) {
                st->beta = tot[1] / st->rz;
                st->rz = tot[1];
            }
        }
        set_cond(cond, use_cond, st->done ? 0u : 1u);
    }
}

}  // namespace nb2

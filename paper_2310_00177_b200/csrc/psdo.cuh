// PSDO iteration kernels (psdo_solve, src/solver.cpp:189-276), whole loop on
// device. Solver vectors live on the full grid in f64 with exact zeros at
// non-fluid cells, so the matrix-free operator needs no index maps: with the
// zero invariant, adding a non-fluid neighbour's (-1.0 * 0) leaves the CSR
// row sum bit-identical (s + -0.0 == s), and the row is accumulated in the
// reduced CSR column order (z-1, y-1, x-1, diag, x+1, y+1, z+1) from s = 0
// with explicit round-to-nearest ops, exactly like spmv (sparse.cpp:111-116)
// on assemble_poisson[_3d] + reduce (discretization.cpp:21-160).
#pragma once

#include "common.cuh"

namespace nb2 {

// (A v)(c) from a per-cell value functor (zero outside the domain).
template <int D, typename VFn>
__device__ __forceinline__ double stencil_row(const Geom& g, int x, int y, int z, int diag, double vc, VFn val) {
    double s = 0.0;
    if (D == 3 && z > 0) s = __dadd_rn(s, -val(lin(g, x, y, z - 1)));
    if (y > 0) s = __dadd_rn(s, -val(lin(g, x, y - 1, z)));
    if (x > 0) s = __dadd_rn(s, -val(lin(g, x - 1, y, z)));
    if (diag > 0) s = __dadd_rn(s, __dmul_rn((double)diag, vc));
    if (x + 1 < g.nx) s = __dadd_rn(s, -val(lin(g, x + 1, y, z)));
    if (y + 1 < g.ny) s = __dadd_rn(s, -val(lin(g, x, y + 1, z)));
    if (D == 3 && z + 1 < g.nz) s = __dadd_rn(s, -val(lin(g, x, y, z + 1)));
    return s;
}

__device__ __forceinline__ void decode(const Geom& g, long long c, int& x, int& y, int& z) {
    x = (int)(c % g.nx);
    y = (int)((c / g.nx) % g.ny);
    z = (int)(c / ((long long)g.nx * g.ny));
}

// ------------------------------------------------------------------ scatter
// reduced (ascending fluid order) -> full grid with zeros elsewhere
__global__ void __launch_bounds__(kBlock) k_scatter(Geom g, const uint8_t* __restrict__ cls,
                                                    const uint32_t* __restrict__ fmask,
                                                    const uint32_t* __restrict__ fbase, const double* __restrict__ red,
                                                    double* __restrict__ full) {
    FOR_OWNED(g, c)
        full[c] = (cls_type(cls[c]) == 0) ? red[mixed_index(fmask, fbase, c)] : 0.0;
}

__global__ void __launch_bounds__(kBlock) k_gather(Geom g, const uint8_t* __restrict__ cls,
                                                   const uint32_t* __restrict__ fmask,
                                                   const uint32_t* __restrict__ fbase, const double* __restrict__ full,
                                                   double* __restrict__ red) {
    FOR_OWNED(g, c)
        if (cls_type(cls[c]) == 0) red[mixed_index(fmask, fbase, c)] = full[c];
}

// zero non-fluid entries (enforces the invariant on caller-provided full vectors)
__global__ void __launch_bounds__(kBlock) k_mask_fluid(Geom g, const uint8_t* __restrict__ cls, const double* __restrict__ src,
                                                       double* __restrict__ dst) {
    FOR_OWNED(g, c)
        dst[c] = (cls_type(cls[c]) == 0) ? src[c] : 0.0;
}

// ------------------------------------------------------------ right-hand side
// mac_divergence_rhs (discretization.cpp:193-227) on the device, generalised
// to 3D: b = scale * (((uR - uL) + (vT - vB)) + (wF - wB)) at fluid cells,
// scale = -(rho * h) / dt; a face whose opposite cell is solid (or outside the
// domain) takes the boundary value (0 without one); 0 elsewhere (the zero
// invariant of the solver vectors). Faces x fastest: u (nx+1, ny, nz),
// v (nx, ny+1, nz), w (nx, ny, nz+1).
template <int D>
__global__ void __launch_bounds__(kBlock) k_mac_rhs(Geom g, const uint8_t* __restrict__ cls,
                                                    const double* __restrict__ u, const double* __restrict__ v,
                                                    const double* __restrict__ w, const double* __restrict__ bu,
                                                    const double* __restrict__ bv, const double* __restrict__ bw,
                                                    double scale, double* __restrict__ b) {
    const long long nx = g.nx, ny = g.ny;
    FOR_OWNED(g, c) {
        if (cls_type(cls[c]) != 0) {
            b[c] = 0.0;
            continue;
        }
        int x, y, z;
        decode(g, c, x, y, z);
        auto solid = [&](int xx, int yy, int zz) {
            if (xx < 0 || xx >= g.nx || yy < 0 || yy >= g.ny || zz < 0 || zz >= g.nz) return true;
            return cls_type(cls[lin(g, xx, yy, zz)]) == 2;
        };
        auto ui = [&](long long fx, long long fy, long long fz) { return (fz * ny + fy) * (nx + 1) + fx; };
        auto vi = [&](long long fx, long long fy, long long fz) { return (fz * (ny + 1) + fy) * nx + fx; };
        auto wi = [&](long long fx, long long fy, long long fz) { return (fz * ny + fy) * nx + fx; };
        const double uR = solid(x + 1, y, z) ? (bu ? bu[ui(x + 1, y, z)] : 0.0) : u[ui(x + 1, y, z)];
        const double uL = solid(x - 1, y, z) ? (bu ? bu[ui(x, y, z)] : 0.0) : u[ui(x, y, z)];
        const double vT = solid(x, y + 1, z) ? (bv ? bv[vi(x, y + 1, z)] : 0.0) : v[vi(x, y + 1, z)];
        const double vB = solid(x, y - 1, z) ? (bv ? bv[vi(x, y, z)] : 0.0) : v[vi(x, y, z)];
        double div = __dadd_rn(__dadd_rn(uR, -uL), __dadd_rn(vT, -vB));
        if (D == 3) {
            const double wF = solid(x, y, z + 1) ? (bw ? bw[wi(x, y, z + 1)] : 0.0) : w[wi(x, y, z + 1)];
            const double wB = solid(x, y, z - 1) ? (bw ? bw[wi(x, y, z)] : 0.0) : w[wi(x, y, z)];
            div = __dadd_rn(div, __dadd_rn(wF, -wB));
        }
        b[c] = __dmul_rn(scale, div);
    }
}

// Input checks on the device right after upload (check_inputs, solver.cpp:28-33;
// the cell-type range): flag |= 1 for a non-finite value / a type > 2.
__global__ void __launch_bounds__(kBlock) k_check_finite(const double* __restrict__ v, long long n,
                                                         unsigned int* __restrict__ flag) {
    bool bad = false;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        bad |= !isfinite(v[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void __launch_bounds__(kBlock) k_check_types(const uint8_t* __restrict__ t, long long n,
                                                        unsigned int* __restrict__ flag) {
    bool bad = false;
    const long long n4 = n / 4;
    const uint32_t* t4 = reinterpret_cast<const uint32_t*>(t);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t w = t4[i];
        bad |= ((w & 0xffu) > 2u) | (((w >> 8) & 0xffu) > 2u) | (((w >> 16) & 0xffu) > 2u) | ((w >> 24) > 2u);
    }
    for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        bad |= t[i] > 2;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// JacobiPrecond's check (precond.cpp:15-18): the smallest reduced row index of
// a fluid cell with a zero diagonal (no non-solid face neighbour), or none
__global__ void __launch_bounds__(kBlock) k_zero_diag(Geom g, const uint8_t* __restrict__ cls,
                                                      const uint32_t* __restrict__ fmask,
                                                      const uint32_t* __restrict__ fbase, unsigned int* __restrict__ row) {
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) == 0 && cls_diag(b) == 0) atomicMin(row, (unsigned int)mixed_index(fmask, fbase, c));
    }
}

// is_pure_neumann (discretization.cpp:180-191), negated: flag |= 1 when a fluid
// cell has an air face neighbour (outside the domain is solid; a z-slab's
// ghost planes hold the neighbours' cells or that outside)
template <int D>
__global__ void __launch_bounds__(kBlock) k_touches_air(Geom g, const uint8_t* __restrict__ cls,
                                                        unsigned int* __restrict__ flag) {
    bool hit = false;
    const long long nx = g.nx, plane = nx * g.ny;
    FOR_OWNED(g, c) {
        if (cls_type(cls[c]) != 0) continue;
        int x, y, z;
        decode(g, c, x, y, z);
        auto air = [&](long long q) { return cls_type(cls[q]) == 1; };
        hit |= (x > 0 && air(c - 1)) || (x + 1 < g.nx && air(c + 1)) || (y > 0 && air(c - nx)) ||
               (y + 1 < g.ny && air(c + nx));
        if (D == 3) hit |= (z > 0 && air(c - plane)) || (z + 1 < g.nz && air(c + plane));
    }
    if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// the flag-derived reduced row of every fluid cell, for checking a caller's
// CSR matrix against it: out[row] = diagonal (number of non-solid face
// neighbours, 0 = dropped, discretization.cpp:115-118) | fluid neighbours << 4
template <int D>
__global__ void __launch_bounds__(kBlock) k_row_info(Geom g, const uint8_t* __restrict__ cls,
                                                     const uint32_t* __restrict__ fmask,
                                                     const uint32_t* __restrict__ fbase, uint8_t* __restrict__ out) {
    const long long nx = g.nx, plane = nx * g.ny;
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) != 0) continue;
        int x, y, z;
        decode(g, c, x, y, z);
        auto fl = [&](long long q) { return cls_type(cls[q]) == 0 ? 1 : 0; };
        int nf = (x > 0 ? fl(c - 1) : 0) + (x + 1 < g.nx ? fl(c + 1) : 0) + (y > 0 ? fl(c - nx) : 0) +
                 (y + 1 < g.ny ? fl(c + nx) : 0);
        if (D == 3) nf += (z > 0 ? fl(c - plane) : 0) + (z + 1 < g.nz ? fl(c + plane) : 0);
        out[mixed_index(fmask, fbase, c)] = (uint8_t)(cls_diag(b) | (nf << 4));
    }
}

// ---------------------------------------------------------------- operator
template <int D>
__global__ void __launch_bounds__(kBlock) k_spmv(Geom g, const uint8_t* __restrict__ cls, const double* __restrict__ v,
                                                 double* __restrict__ out) {
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) != 0) {
            out[c] = 0.0;
            continue;
        }
        int x, y, z;
        decode(g, c, x, y, z);
        out[c] = stencil_row<D>(g, x, y, z, cls_diag(b), v[c], [&](long long q) { return __ldg(v + q); });
    }
}

// ------------------------------------------------------------ reductions
// sum of squares of a full-grid vector over fluid cells -> st fields per mode
enum NormMode { kNormPrecond = 0, kNormMean = 1 };

// Precond-only path: rnorm = ||r||, inv1 = 1/rnorm, inv2 = 1, nrm = rnorm
// (NeuralPrecond::apply, net_precond.cpp:20-26).
__device__ __forceinline__ void fin_norm_precond(SolverState* st, double rsq) {
    const double rn = sqrt(rsq);
    st->rnorm = rn;
    st->inv1 = (rn == 0.0) ? 0.0 : 1.0 / rn;
    st->inv2 = 1.0;
    st->nrm = rn;
}

__global__ void __launch_bounds__(kBlock) k_norm_precond(Geom g, const double* __restrict__ r, SolverState* st,
                                                         double* __restrict__ partials, unsigned int* __restrict__ counter) {
    double acc[1] = {0.0};
    FOR_OWNED(g, c) {
        const double v = r[c];
        acc[0] += v * v;
    }
    double tot[1];
    if (grid_reduce<1>(acc, partials, counter, tot) && threadIdx.x == 0) {
        if (st->dist)
            st->part[0] = tot[0];
        else
            fin_norm_precond(st, tot[0]);
    }
}

// Sets the network scales from st->rnorm for the next preconditioner call.
__device__ __forceinline__ void set_precond_scales(SolverState* st) {
    const double rn = st->rnorm;
    if (st->normalize) {
        // psdo: scaled = r * (1/||r||) (solver.cpp:230-233); NeuralPrecond
        // renormalises by ||scaled|| (net_precond.cpp:20-26), taken here as
        // ||r|| * (1/||r||) (equal in exact arithmetic).
        st->inv1 = 1.0 / rn;
        const double ns = rn * st->inv1;
        st->inv2 = 1.0 / ns;
        st->nrm = ns;
    } else {
        st->inv1 = 1.0;
        st->inv2 = 1.0 / rn;
        st->nrm = rn;
    }
}

// mean over fluid cells (mean_project, vector_ops.cpp:33-43): pass 1 sums.
__global__ void __launch_bounds__(kBlock) k_fluid_sum(Geom g, const uint8_t* __restrict__ cls, const double* __restrict__ v,
                                                      const uint32_t* __restrict__ n_fluid_dev, SolverState* st,
                                                      double* __restrict__ partials, unsigned int* __restrict__ counter) {
    if (st->dist && st->done) return;  // chunked z-slab loop after convergence
    double acc[1] = {0.0};
    FOR_OWNED(g, c) acc[0] += v[c];
    double tot[1];
    if (grid_reduce<1>(acc, partials, counter, tot) && threadIdx.x == 0) {
        const double n_fluid = (double)*n_fluid_dev;  // this frame's (set_mask, on the device)
        if (st->dist) {  // z-slab: this rank's sum and count; k_finalize(kFinMean) divides the totals
            st->part[0] = tot[0];
            st->part[1] = n_fluid;
        } else {
            st->mean = tot[0] / n_fluid;
        }
    }
}

// pass 2: v -= mean at fluid cells; FINAL_NORM also finishes the residual norm
// (and the iteration bookkeeping) exactly like k_update's finaliser.
__global__ void __launch_bounds__(kBlock) k_subtract_mean(Geom g, const uint8_t* __restrict__ cls, double* __restrict__ v,
                                                          const SolverState* __restrict__ st) {
    if (st->dist && st->done) return;
    const double m = st->mean;
    FOR_OWNED(g, c)
        if (cls_type(cls[c]) == 0) v[c] = __dadd_rn(v[c], -m);
}

// ------------------------------------------------------------------ init
// r0 = b - A x0 (solver.cpp:203-207); with PROJ the norm is taken later by
// k_residual_norm after the mean projection.
template <int D>
__global__ void __launch_bounds__(kBlock) k_residual(Geom g, const uint8_t* __restrict__ cls, const double* __restrict__ b,
                                                     const double* __restrict__ x, double* __restrict__ r) {
    FOR_OWNED(g, c) {
        const uint8_t bb = cls[c];
        if (cls_type(bb) != 0) continue;
        int xx, yy, zz;
        decode(g, c, xx, yy, zz);
        const double ax = stencil_row<D>(g, xx, yy, zz, cls_diag(bb), x[c], [&](long long q) { return __ldg(x + q); });
        r[c] = __dadd_rn(b[c], -ax);
    }
}

// first node of every solve: the %globaltimer origin of cumulative_seconds
// (solver.cpp:192, t0 = Clock::now()); precond_seconds starts at zero
__global__ void k_stamp_start(SolverState* st) {
    st->t0 = globaltimer();
    st->precond_s = 0.0;
}

// precond_seconds (solver.cpp:230-237): the network span of an iteration, from
// the end of the previous iteration (t_mark, set by finish_iteration) to the
// first kernel after the network; one thread of that kernel, after its
// dependency wait
__device__ __forceinline__ void precond_span_end(SolverState* st) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0 && !st->done)
        st->precond_s += (double)(globaltimer() - st->t_mark) * 1e-9;
}

__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle cond, int use_cond, unsigned v) {
    if (use_cond) cudaGraphSetConditional(cond, v);
}

__device__ __forceinline__ void finish_iteration(SolverState* st, double rsq, double* hist, double* times,
                                                 cudaGraphConditionalHandle cond, int use_cond, bool initial) {
    const double rn = sqrt(rsq);
    st->rnorm = rn;
    const unsigned long long now = globaltimer();
    st->t_mark = now;
    if (initial) {
        // setup_seconds = r0 and its norm, from the solve's first kernel (solver.cpp:211-212)
        const double setup = (double)(now - st->t0) * 1e-9;
        st->setup_s = setup;
        hist[0] = rn;
        times[0] = setup;
        double thr = st->tol_reduction * rn;
        if (st->tol_abs > 0.0) thr = fmax(thr, st->tol_abs);
        st->thr = thr;
        st->k = 1;
        st->n_cache = 0;
        st->head = st->ring - 1;
        st->converged = (rn <= thr);
        st->done = st->converged || st->max_iters < 1;
    } else {
        const long long k = st->k;
        hist[k] = rn;
        times[k] = (double)(now - st->t0) * 1e-9;
        // cache push (solver.cpp:265-268)
        if (st->n_ortho > 0) {
            const int R = st->ring;
            const int nw = (st->head + 1) % R;
            st->dAd[nw] = st->dAd_new;
            st->head = nw;
            st->n_cache = min(st->n_cache + 1, st->n_ortho);
        }
        st->xcur ^= 1;
        st->converged = (rn <= st->thr);
        st->done = st->converged || k >= st->max_iters;
        st->k = k + 1;
    }
    if (!st->done) set_precond_scales(st);
    set_cond(cond, use_cond, st->done ? 0u : 1u);
}

// ||r||^2 over the (already projected) residual, then bookkeeping.
__global__ void __launch_bounds__(kBlock) k_residual_norm(Geom g, const double* __restrict__ r, SolverState* st,
                                                          double* __restrict__ hist, double* __restrict__ times,
                                                          double* __restrict__ partials, unsigned int* __restrict__ counter,
                                                          cudaGraphConditionalHandle cond, int use_cond, int initial) {
    if (!initial && st->breakdown) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(cond, use_cond, 0u);
        return;
    }
    if (!initial && st->dist && st->done) return;
    double acc[1] = {0.0};
    FOR_OWNED(g, c) {
        const double v = r[c];
        acc[0] += v * v;
    }
    double tot[1];
    if (grid_reduce<1>(acc, partials, counter, tot) && threadIdx.x == 0) {
        if (st->dist)
            st->part[0] = tot[0];
        else
            finish_iteration(st, tot[0], hist, times, cond, use_cond, initial != 0);
    }
}

// The zero invariant across frames: the solver vectors are exactly zero at
// every non-fluid cell. A frame's setup zeroes only the cells that were fluid
// in the previous frame and are not now (then records the frame's fluid
// mask); every vector starts zeroed at allocation.
__global__ void __launch_bounds__(kBlock) k_zero_removed(long long nseg, uint32_t* __restrict__ prev,
                                                         const uint32_t* __restrict__ cur, double* __restrict__ v0,
                                                         double* __restrict__ v1, double* __restrict__ v2,
                                                         double* __restrict__ ring, int nring, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long seg = (long long)blockIdx.x * blockDim.x + threadIdx.x; seg < nseg; seg += stride) {
        const uint32_t now = cur[seg];
        uint32_t m = prev[seg] & ~now;
        prev[seg] = now;
        while (m) {
            const long long c = (seg << 5) + (__ffs(m) - 1);
            m &= m - 1;
            v0[c] = 0.0;
            v1[c] = 0.0;
            v2[c] = 0.0;
            for (int j = 0; j < nring; ++j) ring[(long long)j * n + c] = 0.0;
        }
    }
}

}  // namespace nb2

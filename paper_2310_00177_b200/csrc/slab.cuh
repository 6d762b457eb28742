// z-slab decomposition: the device side of the reduction points.
//
// With st->dist set, each reduction kernel stops after its deterministic grid
// reduction and leaves this rank's totals in st->part. The communicator then
// gathers every rank's part into all[r * kPart + j] (rank order) on every
// rank, and k_finalize sums them in rank order and runs the same finalisation
// the single-domain kernels run inline: every rank ends with bit-identical
// solver state, so the ranks take the same branches (convergence, breakdown,
// cache pushes) without further communication.
#pragma once

#include "common.cuh"
#include "mixed.cuh"
#include "psdo.cuh"
#include "stencil.cuh"

namespace nb2 {

enum FinKind { kFinNorm0 = 0, kFinNormPrecond = 1, kFinProj = 2, kFinOrtho = 3, kFinUpdate = 4, kFinMean = 5 };

__global__ void k_finalize(int kind, SolverState* st, const double* __restrict__ all, int nranks,
                           double* __restrict__ hist, double* __restrict__ times) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // iteration reductions after the solve finished (chunked loop): nothing to do
    if ((kind == kFinProj || kind == kFinOrtho || kind == kFinUpdate || kind == kFinMean) && st->done) return;
    double tot[kPart];
    for (int j = 0; j < kPart; ++j) {
        double t = 0.0;
        for (int r = 0; r < nranks; ++r) t += all[r * kPart + j];
        tot[j] = t;
    }
    const cudaGraphConditionalHandle none = 0;
    switch (kind) {
        case kFinNorm0: finish_iteration(st, tot[0], hist, times, none, 0, true); break;
        case kFinNormPrecond: fin_norm_precond(st, tot[0]); break;
        case kFinProj: fin_projections(st, tot); break;
        case kFinOrtho: fin_ortho(st, tot); break;
        case kFinUpdate: finish_iteration(st, tot[0], hist, times, none, 0, false); break;
        case kFinMean: st->mean = tot[0] / tot[1]; break;  // mean_project over all ranks' fluid cells
        default: break;
    }
}

// exact integer allreduce tail: out[j] = sum_r all[r * k + j]
__global__ void k_sum_u64(const unsigned long long* __restrict__ all, int nranks, int k,
                          unsigned long long* __restrict__ out) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        unsigned long long t = 0;
        for (int r = 0; r < nranks; ++r) t += all[r * k + j];
        out[j] = t;
    }
}

// set_mask capacity flags agreed over the ranks (any rank overflowing makes
// every rank redo the frame: the redo runs the exchanges again)
__global__ void k_flags_u64(const uint32_t* __restrict__ flags, unsigned long long* __restrict__ v) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *v = *flags;
}
__global__ void k_u64_flags(const unsigned long long* __restrict__ v, uint32_t* __restrict__ flags) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *flags = *v ? 0xffffffffu : 0u;
}

// planes [z0, z1) of a level's 3-channel image set to the outside of the
// domain (solid: channels 0, 0, 1) — the ghost planes of a slab before the
// neighbours' copies arrive
__global__ void k_solid_planes(Geom g, float* __restrict__ img, int z0, int z1) {
    const long long plane = (long long)g.nx * g.ny;
    const long long n = (long long)(z1 - z0) * plane;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long c = (long long)z0 * plane + i;
        img[c] = 0.0f;
        img[g.n + c] = 0.0f;
        img[2 * g.n + c] = 1.0f;
    }
}

}  // namespace nb2

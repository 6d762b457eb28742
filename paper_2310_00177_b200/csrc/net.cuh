// Network kernels: NetContext::apply (net/forward.hpp:95-129) as one fused
// kernel per level and sweep direction.
//
//   k_down<D, L0>  y_l = conv_down_l(x_l) (apply_kernels, net/kernels.hpp:147-172)
//                  and x_{l+1} = avg_pool(y_l) (net/kernels.hpp:279-289) in the
//                  same pass. One thread owns a 2x2(x2) brick, so the pool is a
//                  register sum. L0 variant: x_0 = f32((r * inv1) * inv2) is
//                  formed on load from the f64 residual (net_precond.cpp:24-29)
//                  and y_0 is stored for fluid cells only (the only ones the up
//                  sweep reads).
//   k_up<D, MODE>  out_l = z_a * y_l + z_b * conv_up_l(upsample(out_{l+1}))
//                  (forward.hpp:118-127, kernels.hpp:292-304). The brick's
//                  2x2(x2) cells share one coarse parent, so the 4^D upsampled
//                  window is a 3^D coarse window. L0 variant: fluid cells only,
//                  d = f64(out_0) * nrm (net_precond.cpp:31-34) fused with the
//                  A-orthogonalisation dots d.Ad_j (solver.cpp:239-243).
//
// Per cell the kernel is a compile-time-known uniform kernel (3 per level,
// shared memory) or a row of the compact mixed-cell table.
#pragma once

#include "common.cuh"

namespace nb2 {

// Mixed-window kernels are AoS rows of kRowW floats (27 used). Row of a mixed
// cell = kid[mixed_index] (level 0: window-pattern dictionary) or its row code
// (levels >= 1, k_row_codes).
constexpr int kRowW = 28;

struct ConvTab {
    const uint8_t* cls;
    const uint32_t* mmask;
    const uint32_t* mbase;
    const float* tab;     // rows [row][kRowW]
    const uint32_t* kid;  // mixed index -> row, or nullptr (identity)
    const float* kconst;  // [3][S]
    const uint32_t* rcode;  // levels >= 1: per cell (window class << 30) | row, or nullptr
};

// levels >= 1: the cell's row code (k_row_codes); level 0: the cell's
// window pattern (kid = the dictionary ids by mixed index)
__device__ __forceinline__ const float* kernel_row(const ConvTab& ct, long long c) {
    if (ct.rcode) return ct.tab + (long long)(__ldg(ct.rcode + c) & 0x3fffffffu) * kRowW;
    const long long idx = mixed_index(ct.mmask, ct.mbase, c);
    const long long row = ct.kid ? (long long)__ldg(ct.kid + idx) : idx;
    return ct.tab + row * kRowW;
}

// y = sum_s K[s] * win(s), slot order, round-to-nearest (apply_kernels order).
template <int D, typename WinFn>
__device__ __forceinline__ float conv_cell(const ConvTab& ct, const float* sK, long long c, uint8_t b, WinFn win) {
    constexpr int S = Sh<D>::S;
    const int wc = cls_window(b);
    float acc = 0.0f;
    if (wc < 3) {
        const float* K = sK + wc * S;
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(K[s], win(s)));
    } else {
        const float* K = kernel_row(ct, c);
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(__ldg(K + s), win(s)));
    }
    return acc;
}

template <int D>
__device__ __forceinline__ void load_kconst(float* sK, const float* kconst) {
    for (int i = threadIdx.x; i < 3 * Sh<D>::S; i += blockDim.x) sK[i] = kconst[i];
    __syncthreads();
}

// ------------------------------------------------------------------ down
// in_f: f32 input (levels >= 1, or raw-network L0); in_d: f64 residual (L0 solve).
template <int D, bool L0, bool POOL>
__global__ void __launch_bounds__(kBlock) k_down(Geom g, const float* __restrict__ in_f,
                                                 const double* __restrict__ in_d, const SolverState* __restrict__ st,
                                                 ConvTab ct, float* __restrict__ y, float* __restrict__ xnext,
                                                 Geom gc) {
    constexpr int S = Sh<D>::S, BZ = Sh<D>::BZ, WZ = Sh<D>::WZ;
    __shared__ float sK[3 * S];
    load_kconst<D>(sK, ct.kconst);
    double inv1 = 1.0, inv2 = 1.0;
    if (L0) {
        inv1 = st->inv1;
        inv2 = st->inv2;
    }
    const int nbx = g.nx >> 1, nby = g.ny >> 1, nbz = (D == 3) ? (g.nz >> 1) : 1;
    const long long nb = (long long)nbx * nby * nbz;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
        const int bx = (int)(b % nbx);
        const int by = (int)((b / nbx) % nby);
        const int bz = (int)(b / ((long long)nbx * nby));
        const int x0 = 2 * bx, y0 = 2 * by, z0 = (D == 3) ? 2 * bz : 0;
        float w[WZ][4][4];
#pragma unroll
        for (int kz = 0; kz < WZ; ++kz) {
            const int z = (D == 3) ? z0 - 1 + kz : 0;
            const bool zin = z >= 0 && z < g.nz;
#pragma unroll
            for (int ky = 0; ky < 4; ++ky) {
                const int yy = y0 - 1 + ky;
                const bool yin = zin && yy >= 0 && yy < g.ny;
#pragma unroll
                for (int kx = 0; kx < 4; ++kx) {
                    const int xx = x0 - 1 + kx;
                    float v = 0.0f;
                    if (yin && xx >= 0 && xx < g.nx) {
                        const long long q = lin(g, xx, yy, z);
                        if (L0)
                            v = __double2float_rn(__dmul_rn(__dmul_rn(__ldg(in_d + q), inv1), inv2));
                        else
                            v = __ldg(in_f + q);
                    }
                    w[kz][ky][kx] = v;
                }
            }
        }
        float psum = 0.0f;
#pragma unroll
        for (int cz = 0; cz < BZ; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                for (int cx = 0; cx < 2; ++cx) {
                    const long long c = lin(g, x0 + cx, y0 + cy, z0 + cz);
                    const uint8_t bb = ct.cls[c];
                    const float yv = conv_cell<D>(ct, sK, c, bb, [&](int s) {
                        const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
                        return w[(D == 3) ? cz + 1 + dz : 0][cy + 1 + dy][cx + 1 + dx];
                    });
                    if (!L0 || cls_type(bb) == 0) y[c] = yv;
                    if (POOL) psum = (cz == 0 && cy == 0 && cx == 0) ? yv : __fadd_rn(psum, yv);
                }
        if (POOL) xnext[lin(gc, bx, by, bz)] = __fmul_rn((D == 3) ? 0.125f : 0.25f, psum);
    }
}

// -------------------------------------------------------------------- up
enum UpMode { kUpMid = 0, kUpL0 = 1, kUpL0Depth1 = 2, kUpRaw0 = 3 };

// kUpMid:      levels >= 1 (and level 0 of the raw network when MODE==kUpRaw0):
//              out_l (f32, every cell)
// kUpL0:       level 0 of the solve: d (f64, fluid cells) + dots with AD_j
// kUpL0Depth1: depth 1: the network is the single coarse conv, d = f64(y_0) * nrm
template <int D, int MODE>
__global__ void __launch_bounds__(kBlock) k_up(Geom g, Geom gc, const float* __restrict__ outc,
                                               const float* __restrict__ yl, const float* __restrict__ zab, ConvTab ct,
                                               float* __restrict__ outl, double* __restrict__ dout,
                                               SolverState* __restrict__ st, const double* __restrict__ ADring,
                                               double* __restrict__ partials, unsigned int* __restrict__ counter) {
    constexpr int S = Sh<D>::S, BZ = Sh<D>::BZ, CW = Sh<D>::CW;
    constexpr bool SOLVE = (MODE == kUpL0 || MODE == kUpL0Depth1);
    __shared__ float sK[3 * S];
    load_kconst<D>(sK, ct.kconst);
    float za = 0.0f, zb = 0.0f;
    if (MODE != kUpL0Depth1) {
        za = zab[0];
        zb = zab[1];
    }
    double nrm = 1.0;
    int nc = 0;
    const double* adp[kMaxOrtho];
    if (SOLVE) {
        nrm = st->nrm;
        nc = st->n_cache;
        const int R = st->ring;
        for (int j = 0; j < kMaxOrtho; ++j) {
            const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
            adp[j] = ADring + (long long)slot * g.n;
        }
    }
    double acc[kMaxOrtho];
#pragma unroll
    for (int j = 0; j < kMaxOrtho; ++j) acc[j] = 0.0;

    const int nbx = g.nx >> 1, nby = g.ny >> 1, nbz = (D == 3) ? (g.nz >> 1) : 1;
    const long long nb = (long long)nbx * nby * nbz;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
        const int bx = (int)(b % nbx);
        const int by = (int)((b / nbx) % nby);
        const int bz = (int)(b / ((long long)nbx * nby));
        const int x0 = 2 * bx, y0 = 2 * by, z0 = (D == 3) ? 2 * bz : 0;
        // fluid cells of the brick (solve path): skip all loads if none
        uint8_t bb[BZ][2][2];
        bool any = !SOLVE;
#pragma unroll
        for (int cz = 0; cz < BZ; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                for (int cx = 0; cx < 2; ++cx) {
                    bb[cz][cy][cx] = ct.cls[lin(g, x0 + cx, y0 + cy, z0 + cz)];
                    if (SOLVE) any |= (cls_type(bb[cz][cy][cx]) == 0);
                }
        if (!any) continue;
        float cw[CW][3][3];
        if (MODE != kUpL0Depth1) {
#pragma unroll
            for (int kz = 0; kz < CW; ++kz) {
                const int z = (D == 3) ? bz - 1 + kz : 0;
                const bool zin = z >= 0 && z < gc.nz;
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) {
                    const int yy = by - 1 + ky;
                    const bool yin = zin && yy >= 0 && yy < gc.ny;
#pragma unroll
                    for (int kx = 0; kx < 3; ++kx) {
                        const int xx = bx - 1 + kx;
                        cw[kz][ky][kx] = (yin && xx >= 0 && xx < gc.nx) ? __ldg(outc + lin(gc, xx, yy, z)) : 0.0f;
                    }
                }
            }
        }
#pragma unroll
        for (int cz = 0; cz < BZ; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                for (int cx = 0; cx < 2; ++cx) {
                    const uint8_t cb = bb[cz][cy][cx];
                    if (SOLVE && cls_type(cb) != 0) continue;
                    const long long c = lin(g, x0 + cx, y0 + cy, z0 + cz);
                    float o;
                    if (MODE == kUpL0Depth1) {
                        o = yl[c];
                    } else {
                        const float u = conv_cell<D>(ct, sK, c, cb, [&](int s) {
                            const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
                            return cw[(D == 3) ? ((cz + dz) >> 1) + 1 : 0][((cy + dy) >> 1) + 1][((cx + dx) >> 1) + 1];
                        });
                        o = __fadd_rn(__fmul_rn(za, yl[c]), __fmul_rn(zb, u));
                    }
                    if (SOLVE) {
                        const double dv = __dmul_rn((double)o, nrm);
                        dout[c] = dv;
#pragma unroll
                        for (int j = 0; j < kMaxOrtho; ++j)
                            if (j < nc) acc[j] += dv * __ldg(adp[j] + c);
                    } else {
                        outl[c] = o;
                    }
                }
    }
    if (SOLVE) {
        double tot[kMaxOrtho];
        if (grid_reduce<kMaxOrtho>(acc, partials, counter, tot) && threadIdx.x == 0) {
            // MGS projections, oldest first (solver.cpp:239-243), in fused form:
            // p_j = (d.Ad_j - sum_{i<j} p_i d_i.Ad_j) / d_j'Ad_j
            const int R = st->ring;
            int slot[kMaxOrtho];
            for (int j = 0; j < nc; ++j) slot[j] = (st->head - (nc - 1) + j + 2 * R) % R;
            for (int j = 0; j < nc; ++j) {
                double num = tot[j];
                for (int i = 0; i < j; ++i) num -= st->p[i] * st->cross[slot[i]][slot[j]];
                st->p[j] = num / st->dAd[slot[j]];
            }
        }
    }
}

}  // namespace nb2

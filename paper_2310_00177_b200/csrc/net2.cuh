// Network kernels, tiled and software-pipelined: NetContext::apply
// (net/forward.hpp:95-129), one fused kernel per level and sweep direction.
//
// A 16 x 8 block owns a 32 x 16 x-y tile of cells; each thread owns one 2x2
// column of bricks and marches a z-chunk two planes at a time. Input planes
// are staged cooperatively in shared memory (coalesced rows, halo included,
// double-buffered: one barrier per step) and each thread keeps the 4-plane
// window of its 2x2(x2) brick in registers, so a brick step stages 2 new
// planes and reuses 2. The next step's planes and cell bytes are prefetched
// into registers before the current brick is computed. The 27 taps of each
// cell are applied in slot order with round-to-nearest ops (apply_kernels,
// net/kernels.hpp:147-172): outputs are bit-identical to the restatement.
// A cell whose whole input window is zero has output exactly +0 (every term
// is K * 0 = +-0 and +0 + -0 = +0), so such bricks are not computed — at
// level 0 that is every brick away from fluid.
//
// k_down3<D, L0, POOL>: y_l = conv_down_l(x_l) and x_{l+1} = avg_pool(y_l).
//   L0: the input is f32((r * inv1) * inv2), formed while staging
//   (net_precond.cpp:24-29); y_0 is stored at fluid cells only.
// k_up3<D, MODE, NO>: out_l = z_a y_l + z_b conv_up_l(upsample(out_{l+1})).
//   MODE kUpL0: fluid cells only, d = f64(out_0) * nrm (net_precond.cpp:31-34)
//   fused with the A-orthogonalisation dots d.Ad_j (solver.cpp:239-243).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "net.cuh"

namespace nb2 {

constexpr int kNX = 16, kNY = 8, kNT = kNX * kNY;   // threads per block
constexpr int kPW = 2 * kNX + 2, kPH = 2 * kNY + 2;  // staged fine-plane patch (34 x 18)
constexpr int kNE = (kPW * kPH + kNT - 1) / kNT;     // staged elements per thread per plane (5)
constexpr int kCW = kNX + 2, kCH = kNY + 2;          // staged coarse-plane patch (18 x 10)
constexpr int kNEC = (kCW * kCH + kNT - 1) / kNT;    // (2)

// The three uniform-window kernels of a conv (build_kernels on a pure
// window), passed by value in the kernel parameter space.
struct KC {
    float k[3][27];
};

template <int D>
__device__ __forceinline__ float conv27(const ConvTab& ct, const KC& kc, long long c, int wc,
                                        const float (&w)[Sh<D>::S]) {
    constexpr int S = Sh<D>::S;
    float acc = 0.0f;
    // uniform windows: one branch per class so every kernel value is a
    // compile-time offset into the parameter bank (no dynamic LDC)
    if (wc == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(kc.k[0][s], w[s]));
    } else if (wc == 1) {
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(kc.k[1][s], w[s]));
    } else if (wc == 2) {
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(kc.k[2][s], w[s]));
    } else {
        const float* K = kernel_row(ct, c);
#pragma unroll
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, __fmul_rn(__ldg(K + s), w[s]));
    }
    return acc;
}

// two adjacent cell bytes (x even, nx even: 2-byte aligned)
__device__ __forceinline__ unsigned pair_bytes(const uint8_t* __restrict__ cls, long long c) {
    return __ldg(reinterpret_cast<const unsigned short*>(cls + c));
}

// ------------------------------------------------------------------ down
template <int D, bool L0, bool POOL>
__global__ void __launch_bounds__(kNT) k_down3(Geom g, const float* __restrict__ in_f,
                                               const double* __restrict__ in_d, const SolverState* __restrict__ st,
                                               ConvTab ct, const __grid_constant__ KC kc, float* __restrict__ y,
                                               float* __restrict__ xnext, Geom gc, int zchunk, Occ occ) {
    constexpr int S = Sh<D>::S, WZ = Sh<D>::WZ, NP = (D == 3) ? 2 : 1;  // planes staged per step
    using Raw = typename std::conditional<L0, double, float>::type;
    __shared__ float sp[2][NP][kPH][kPW];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kNX + tx;
    const int X0 = blockIdx.x * 2 * kNX, Y0 = blockIdx.y * 2 * kNY;
    const int x0 = X0 + 2 * tx, y0 = Y0 + 2 * ty;
    const bool own = x0 < g.nx && y0 < g.ny;  // dims are even: the whole 2x2 is inside
    const long long plane = (long long)g.nx * g.ny;
    double inv1 = 1.0, inv2 = 1.0;
    if (L0) {
        inv1 = st->inv1;
        inv2 = st->inv2;
    }
    const int nbz = (D == 3) ? (g.nz >> 1) : 1;
    const int bz0 = blockIdx.z * zchunk;
    const int bz1 = min(bz0 + zchunk, nbz);
    if (bz0 >= bz1) return;
    if (L0 && occ.flags) {
        // fluid-free region (tile dilated by one cell, one plane each side):
        // the input window is all zero, so y_0 = +0 (not stored: non-fluid)
        // and x_1 = +0
        const int zlo = (D == 3) ? 2 * bz0 - 1 : 0, zhi = (D == 3) ? 2 * bz1 : 0;
        if (!region_has_fluid(occ.flags, occ.ntx, occ.nty, g.nz, blockIdx.x, blockIdx.x + 1, 2 * blockIdx.y,
                              2 * blockIdx.y + 2, zlo, zhi)) {
            if (POOL && own)
                for (int bz = bz0; bz < bz1; ++bz) xnext[lin(gc, x0 >> 1, y0 >> 1, bz)] = 0.0f;
            return;
        }
    }

    Raw pre[NP][kNE];
    // issue the loads of planes z, z+1 (zero outside the domain)
    auto issue = [&](int z) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int zz = z + p;
            const bool zin = zz >= 0 && zz < g.nz;
#pragma unroll
            for (int e = 0; e < kNE; ++e) {
                const int i = tid + e * kNT;
                const int ly = i / kPW, lx = i - ly * kPW;
                const int gx = X0 - 1 + lx, gy = Y0 - 1 + ly;
                const bool ok = zin && i < kPW * kPH && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny;
                const long long q = (long long)zz * plane + (long long)gy * g.nx + gx;
                if (L0)
                    pre[p][e] = ok ? (Raw)__ldg(in_d + q) : (Raw)0;
                else
                    pre[p][e] = ok ? (Raw)__ldg(in_f + q) : (Raw)0;
            }
        }
    };
    auto publish = [&](int b) {
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
            for (int e = 0; e < kNE; ++e) {
                const int i = tid + e * kNT;
                if (i < kPW * kPH) {
                    const int ly = i / kPW, lx = i - ly * kPW;
                    float v;
                    if (L0)
                        v = __double2float_rn(__dmul_rn(__dmul_rn((double)pre[p][e], inv1), inv2));
                    else
                        v = (float)pre[p][e];
                    sp[b][p][ly][lx] = v;
                }
            }
    };
    float w[WZ][4][4];
    bool nz_[WZ];  // plane patch holds a nonzero value
    auto take = [&](int b, int p, int slot) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float v = sp[b][p][2 * ty + j][2 * tx + i];
                w[slot][j][i] = v;
                any |= (v != 0.0f);
            }
        nz_[slot] = any;
    };

    int buf = 0;
    if (D == 3) {
        issue(2 * bz0 - 1);
        publish(0);
        __syncthreads();
        take(0, 0, 0);
        take(0, 1, 1);
        issue(2 * bz0 + 1);
        publish(1);
        __syncthreads();
        take(1, 0, 2);
        take(1, 1, 3);
        buf = 1;
    } else {
        issue(0);
        publish(0);
        __syncthreads();
        take(0, 0, 0);
    }
    unsigned cb[Sh<D>::BZ][2];  // cell bytes of the brick: [cz][cy] = 2 x-adjacent bytes
    auto load_bytes = [&](int z0) {
#pragma unroll
        for (int cz = 0; cz < Sh<D>::BZ; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy) cb[cz][cy] = own ? pair_bytes(ct.cls, lin(g, x0, y0 + cy, z0 + cz)) : 0u;
    };
    load_bytes((D == 3) ? 2 * bz0 : 0);
    for (int bz = bz0; bz < bz1; ++bz) {
        const int z0 = (D == 3) ? 2 * bz : 0;
        const bool more = (D == 3) && (bz + 1 < bz1);
        if (more) issue(z0 + 3);  // prefetch the next step's planes
        unsigned cbn[Sh<D>::BZ][2];
#pragma unroll
        for (int cz = 0; cz < Sh<D>::BZ; ++cz)
#pragma unroll
            for (int cy = 0; cy < 2; ++cy) cbn[cz][cy] = (more && own) ? pair_bytes(ct.cls, lin(g, x0, y0 + cy, z0 + 2 + cz)) : 0u;
        if (own) {
            float psum = 0.0f;
#pragma unroll
            for (int cz = 0; cz < Sh<D>::BZ; ++cz) {
                const bool need = (D == 3) ? (nz_[cz] || nz_[cz + 1] || nz_[cz + 2]) : nz_[0];
#pragma unroll
                for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                    for (int cx = 0; cx < 2; ++cx) {
                        const long long c = lin(g, x0 + cx, y0 + cy, z0 + cz);
                        const uint8_t bb = (uint8_t)(cb[cz][cy] >> (8 * cx));
                        float yv = 0.0f;
                        if (L0 && cls_window(bb) == 3) {
                            // mixed window: computed by k_mixed_down0 (+0 without fluid)
                            yv = cls_wfluid(bb) ? y[c] : 0.0f;
                        } else if (need) {
                            float win[S];
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
                                win[s] = w[(D == 3) ? cz + 1 + dz : 0][cy + 1 + dy][cx + 1 + dx];
                            }
                            yv = conv27<D>(ct, kc, c, cls_window(bb), win);
                        }
                        if ((!L0 || cls_type(bb) == 0) && !(L0 && cls_window(bb) == 3)) y[c] = yv;
                        if (POOL) psum = (cz == 0 && cy == 0 && cx == 0) ? yv : __fadd_rn(psum, yv);
                    }
            }
            if (POOL) xnext[lin(gc, x0 >> 1, y0 >> 1, bz)] = __fmul_rn((D == 3) ? 0.125f : 0.25f, psum);
        }
        if (more) {
            publish(buf ^ 1);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    w[0][j][i] = w[2][j][i];
                    w[1][j][i] = w[3][j][i];
                }
            nz_[0] = nz_[2];
            nz_[1] = nz_[3];
            take(buf ^ 1, 0, 2);
            take(buf ^ 1, 1, 3);
            buf ^= 1;
#pragma unroll
            for (int cz = 0; cz < Sh<D>::BZ; ++cz)
#pragma unroll
                for (int cy = 0; cy < 2; ++cy) cb[cz][cy] = cbn[cz][cy];
        }
    }
}

// -------------------------------------------------------------------- up
// NO: n_ortho bound for the fused dots (kUpL0 only).
template <int D, int MODE, int NO>
__global__ void __launch_bounds__(kNT) k_up3(Geom g, Geom gc, const float* __restrict__ outc,
                                             const float* __restrict__ yl, const float* __restrict__ zab, ConvTab ct,
                                             const __grid_constant__ KC kc, float* __restrict__ outl,
                                             double* __restrict__ dout, SolverState* __restrict__ st,
                                             const double* __restrict__ ADring, double* __restrict__ partials,
                                             unsigned int* __restrict__ counter, int zchunk, Occ occ) {
    constexpr int S = Sh<D>::S, CW = Sh<D>::CW, BZ = Sh<D>::BZ;
    constexpr bool SOLVE = (MODE == kUpL0);
    constexpr int NA = (NO > 0) ? NO : 1;
    __shared__ float sc[2][kCH][kCW];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kNX + tx;
    const int BX0 = blockIdx.x * kNX, BY0 = blockIdx.y * kNY;  // coarse tile origin
    const int bx = BX0 + tx, by = BY0 + ty;                    // my coarse column
    const bool own = bx < gc.nx && by < gc.ny;
    const int x0 = 2 * bx, y0 = 2 * by;
    const long long cplane = (long long)gc.nx * gc.ny;
    const float za = zab[0], zb = zab[1];
    double nrm = 1.0;
    int nc = 0;
    const double* adp[NA];
    if (SOLVE) {
        nrm = st->nrm;
        nc = st->n_cache;
        const int R = st->ring;
#pragma unroll
        for (int j = 0; j < NA; ++j) {
            const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
            adp[j] = ADring + (long long)slot * g.n;
        }
    }
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;

    const int nbz = (D == 3) ? gc.nz : 1;
    const int bz0 = blockIdx.z * zchunk;
    const int bz1 = min(bz0 + zchunk, nbz);

    float pre[kNEC];
    auto issue = [&](int z) {
        const bool zin = z >= 0 && z < gc.nz;
#pragma unroll
        for (int e = 0; e < kNEC; ++e) {
            const int i = tid + e * kNT;
            const int ly = i / kCW, lx = i - ly * kCW;
            const int gx = BX0 - 1 + lx, gy = BY0 - 1 + ly;
            const bool ok = zin && i < kCW * kCH && gx >= 0 && gx < gc.nx && gy >= 0 && gy < gc.ny;
            pre[e] = ok ? __ldg(outc + (long long)z * cplane + (long long)gy * gc.nx + gx) : 0.0f;
        }
    };
    auto publish = [&](int b) {
#pragma unroll
        for (int e = 0; e < kNEC; ++e) {
            const int i = tid + e * kNT;
            if (i < kCW * kCH) {
                const int ly = i / kCW, lx = i - ly * kCW;
                sc[b][ly][lx] = pre[e];
            }
        }
    };
    float cw[CW][3][3];
    auto take = [&](int b, int slot) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) cw[slot][j][i] = sc[b][ty + j][tx + i];
    };
    // L0: a fluid-free tile has no output and no dot contribution (the block
    // still joins the grid reduction below)
    bool active = bz0 < bz1;
    if (SOLVE && occ.flags && active)
        active = region_has_fluid(occ.flags, occ.ntx, occ.nty, g.nz, blockIdx.x, blockIdx.x + 1, 2 * blockIdx.y,
                                  2 * blockIdx.y + 2, (D == 3) ? 2 * bz0 : 0, (D == 3) ? 2 * bz1 - 1 : 0);
    if (active) {
        int buf = 0;
        if (D == 3) {
            issue(bz0 - 1);
            publish(0);
            __syncthreads();
            take(0, 0);
            issue(bz0);
            publish(1);
            __syncthreads();
            take(1, 1);
            issue(bz0 + 1);
            publish(0);
            __syncthreads();
            take(0, 2);
            buf = 0;
        } else {
            issue(0);
            publish(0);
            __syncthreads();
            take(0, 0);
        }
        for (int bz = bz0; bz < bz1; ++bz) {
            const int z0 = (D == 3) ? 2 * bz : 0;
            const bool more = (D == 3) && (bz + 1 < bz1);
            if (more) issue(bz + 2);  // prefetch the next coarse plane
            if (own) {
                // per-cell inputs of this brick, issued before the convolutions
                unsigned cb[BZ][2];
                float yv[BZ][2][2];
                double adv[BZ][2][2][NA];
#pragma unroll
                for (int cz = 0; cz < BZ; ++cz)
#pragma unroll
                    for (int cy = 0; cy < 2; ++cy) {
                        cb[cz][cy] = pair_bytes(ct.cls, lin(g, x0, y0 + cy, z0 + cz));
#pragma unroll
                        for (int cx = 0; cx < 2; ++cx) {
                            const long long c = lin(g, x0 + cx, y0 + cy, z0 + cz);
                            const bool live = !SOLVE || cls_type((uint8_t)(cb[cz][cy] >> (8 * cx))) == 0;
                            yv[cz][cy][cx] = live ? __ldg(yl + c) : 0.0f;
#pragma unroll
                            for (int j = 0; j < NA; ++j)
                                adv[cz][cy][cx][j] = (SOLVE && live && j < nc) ? __ldg(adp[j] + c) : 0.0;
                        }
                    }
#pragma unroll
                for (int cz = 0; cz < BZ; ++cz)
#pragma unroll
                    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
                        for (int cx = 0; cx < 2; ++cx) {
                            const uint8_t bb = (uint8_t)(cb[cz][cy] >> (8 * cx));
                            if (SOLVE && (cls_type(bb) != 0 || cls_window(bb) == 3)) continue;  // mixed: k_mixed_up0
                            const long long c = lin(g, x0 + cx, y0 + cy, z0 + cz);
                            float win[S];
#pragma unroll
                            for (int s = 0; s < S; ++s) {
                                const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
                                win[s] = cw[(D == 3) ? ((cz + dz) >> 1) + 1 : 0][((cy + dy) >> 1) + 1][((cx + dx) >> 1) + 1];
                            }
                            const float u = conv27<D>(ct, kc, c, cls_window(bb), win);
                            const float o = __fadd_rn(__fmul_rn(za, yv[cz][cy][cx]), __fmul_rn(zb, u));
                            if (SOLVE) {
                                const double dv = __dmul_rn((double)o, nrm);
                                dout[c] = dv;
#pragma unroll
                                for (int j = 0; j < NO; ++j)
                                    if (j < nc) acc[j] += dv * adv[cz][cy][cx][j];
                            } else {
                                outl[c] = o;
                            }
                        }
            }
            if (more) {
                publish(buf ^ 1);
                __syncthreads();
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        cw[0][j][i] = cw[1][j][i];
                        cw[1][j][i] = cw[2][j][i];
                    }
                take(buf ^ 1, 2);
                buf ^= 1;
            }
        }
    }
    if (SOLVE) {
        double tot[NA];
        // the mixed fluid cells follow in k_mixed_up0, which finalises the
        // MGS projections from these totals plus its own
        if (grid_reduce<NA>(acc, partials, counter, tot) && tid == 0)
            for (int j = 0; j < NA; ++j) st->dot_main[j] = tot[j];
    }
}

}  // namespace nb2

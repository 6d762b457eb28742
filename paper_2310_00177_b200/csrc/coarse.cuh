// Network levels above the solve's level 0, 3D (and every level of the raw
// network): NetContext::apply's down and up steps (net/forward.hpp:95-129).
//
// These grids are small (128^3 and below at 256^3) and their kernels are
// latency-bound, not bandwidth-bound: what matters is enough independent
// cells in flight and short dependent chains. Each cell reads its kernel as
// one 28-float row (seven 16-byte loads) through a single pointer — the shared
// copy of its uniform class's kernel or its mixed row in global memory — so
// uniform and mixed cells of a warp run the same code. The window sum is
// win_dot (common.cuh): the reference's slot order with round-to-nearest ops
// (apply_kernels, net/kernels.hpp:147-172; bit-identical outputs) or, in the
// fast mode, fused per-plane chains.
//
// k_cdownz<POOL>: y_l = conv_down_l(x_l); x_{l+1} = avg_pool(y_l), summed x
//   fastest, then y, then z (avg_pool2, kernels.hpp:279-292, 3D order).
//   Without POOL: the coarsest level's single conv (forward.hpp:89,116).
// k_cupz: out_l = z_a y_l + z_b conv_up_l(upsample2(out_{l+1}))
//   (forward.hpp:118-127); a fine tap reads coarse cell (x >> 1, y >> 1,
//   z >> 1), zero outside.
#pragma once

#include "common.cuh"
#include "net.cuh"
#include "net2.cuh"

namespace nb2 {

// The three uniform-window kernels in shared memory as 28-float rows, so every
// cell reads its kernel through one pointer: no per-class code paths, no warp
// divergence between uniform and mixed cells.
struct UniRows {
    float4 r[3][7];
};

__device__ __forceinline__ void load_uni_rows(UniRows& U, const KC& kc, int tid) {
    if (tid < 84) {
        const int w = tid / 28, s = tid - 28 * w;
        reinterpret_cast<float*>(&U.r[w][0])[s] = (s < 27) ? kc.k[w][s] : 0.0f;
    }
}

__device__ __forceinline__ void load_row(const float4* row, float (&k)[28]) {
#pragma unroll
    for (int i = 0; i < 7; ++i) {
        const float4 v = row[i];  // generic: shared or global
        k[4 * i] = v.x;
        k[4 * i + 1] = v.y;
        k[4 * i + 2] = v.z;
        k[4 * i + 3] = v.w;
    }
}

// ---------------------------------------------------------------------------
// z-marching kernels: a 32 x 8 block owns a 32 x 8
// x-y tile and ZC consecutive planes; each thread marches its (x, y) column
// through the ZC planes. The input box (tile + one-cell halo, ZC + 2 planes) is
// staged once; the 3 x 3 x 3 window rolls through registers (9 new shared
// loads per cell instead of 27) and the per-block index work is spread over
// ZC cells per thread. Warps are 16 x 2 cells (lane = x + 16 y), so a 2 x 2
// pooling quad sits inside one warp and the pool is summed with shuffles in
// the reference order (no barrier). Shared rows are padded to 48 floats
// (= 16 mod 32 banks): the two half-warps' rows fall on disjoint banks.
// Accumulation: win_dot (exact: slot order, bit-identical; fast: fused chains).
constexpr int kZX = 32, kZY = 8, kZT = kZX * kZY;  // block tile (x, y) = 256 threads
#ifndef COARSEZ_MINB
#define COARSEZ_MINB 4  // min resident blocks per SM of the z-marching kernels: a 64-register cap (1: 84 registers, 3 blocks; measured 3-4 us slower per L1 kernel)
#endif
constexpr int kZSP = 48;                           // padded shared row stride (floats)

// (NZ x NY x NX) box at (bx, by, bz) of gg, zero outside the grid, staged
// into dst[NZ][NY][kZSP]; one warp per row. load() issues every load (into
// registers) so that other independent loads can be issued before store().
template <int NX, int NY, int NZ>
struct ZStager {
    static constexpr int NW = kZT / 32, ROWS = NY * NZ, RPW = (ROWS + NW - 1) / NW, EPL = (NX + 31) / 32;
    float v[RPW][EPL];
    // 32-bit offsets from the box's first plane (a box spans NZ planes, so
    // they fit for any grid this library allocates)
    __device__ __forceinline__ void load(const float* __restrict__ src, const Geom& gg, int bx, int by, int bz,
                                         int warp, int lane) {
        const float* p0 = src + (long long)bz * gg.nx * gg.ny + bx;
        const int wly = warp % NY, wlz = warp / NY;
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            // row r = warp + NW k: (ly, lz) advanced from the warp's own (ly, lz)
            const int t = wly + (NW * k) % NY;
            const int ly = t - (t >= NY ? NY : 0), lz = wlz + (NW * k) / NY + (t >= NY ? 1 : 0);
            const int gy = by + ly, gz = bz + lz;
            const bool rin = (warp + NW * k) < ROWS && (unsigned)gy < (unsigned)gg.ny && (unsigned)gz < (unsigned)gg.nz;
            const float* rowp = p0 + (lz * gg.ny + gy) * gg.nx;
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const int lx = lane + 32 * e;
                v[k][e] = (rin && lx < NX && (unsigned)(bx + lx) < (unsigned)gg.nx) ? __ldg(rowp + lx) : 0.0f;
            }
        }
    }
    __device__ __forceinline__ void store(float* dst, int warp, int lane) const {
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NW * k;
            if (r < ROWS) {
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const int lx = lane + 32 * e;
                    if (lx < NX) dst[r * kZSP + lx] = v[k][e];
                }
            }
        }
    }
};

// A cell's row code before its row pointer: levels >= 1 carry per-cell codes
// (window class << 30 | row); the raw level-0 network has class bytes and the
// mixed-index maps instead.
__device__ __forceinline__ uint32_t cell_code(const ConvTab& ct, long long c, bool own) {
    if (!own) return 1u << 30;  // uniform air
    if (ct.rcode) return __ldg(ct.rcode + c);
    return (uint32_t)cls_window(__ldg(ct.cls + c)) << 30;
}
__device__ __forceinline__ const float4* code_row(const ConvTab& ct, const UniRows& U, uint32_t rc, long long c) {
    const int wc = (int)(rc >> 30);
    if (wc < 3) return &U.r[wc][0];
    if (ct.rcode) return reinterpret_cast<const float4*>(ct.tab + (long long)(rc & 0x3fffffffu) * kRowW);
    return reinterpret_cast<const float4*>(kernel_row(ct, c));
}

// shared memory of one z-marching tile: the staged box and the uniform rows
template <int ZC>
struct CDownSmem {
    static constexpr int PL = (kZY + 2) * kZSP;
    float sx[(ZC + 2) * PL];
    UniRows U;
};
template <int ZC>
struct CUpSmem {
    static constexpr int PL = (kZY / 2 + 2) * kZSP;
    float sc[(ZC / 2 + 2) * PL];
    UniRows U;
};

// one 32 x 8 x ZC tile (bx, by, bz) of a down step; S in shared memory
template <bool POOL, int ZC, bool F>
__device__ __forceinline__ void cdownz_tile(const Geom& g, const float* __restrict__ x, const ConvTab& ct, const KC& kc,
                                            float* __restrict__ y, float* __restrict__ xnext, const Geom& gc, int bx,
                                            int by, int bz, CDownSmem<ZC>& S, const int* __restrict__ done) {
    static_assert(!POOL || ZC % 2 == 0, "pooling pairs planes");
    constexpr int SX = kZX + 2, SY = kZY + 2, SZ = ZC + 2, PL = SY * kZSP;
    float* sx = S.sx;
    UniRows& U = S.U;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tx = 16 * (warp & 1) + (lane & 15), ty = 2 * (warp >> 1) + (lane >> 4);
    const int X0 = bx * kZX, Y0 = by * kZY, Z0 = g.zo0 + bz * ZC;
    const int cx = X0 + tx, cy = Y0 + ty;
    const bool oxy = cx < g.nx && cy < g.ny;
    const long long plane = (long long)g.nx * g.ny;
    const long long c0 = oxy ? lin(g, cx, cy, Z0) : 0;
    const int nown = oxy ? min(ZC, g.zo1 - Z0) : 0;  // planes of this column the rank owns
    // setup data first (row codes, the uniform rows, the first cell's row):
    // with programmatic launch it overlaps the previous kernel
    uint32_t rc[ZC];
#pragma unroll
    for (int k = 0; k < ZC; ++k) rc[k] = cell_code(ct, c0 + k * plane, k < nown);
    load_uni_rows(U, kc, tid);
    __syncthreads();
    float kr[28];  // the next cell's kernel row (prefetched one cell ahead)
    load_row(code_row(ct, U, rc[0], c0), kr);
    pdl_wait_then_trigger();  // x_l is the previous kernel's output
    if (done && *done) return;  // z-slab chunked loop: the solve has finished (block-uniform)
    ZStager<SX, SY, SZ> box;
    box.load(x, g, X0 - 1, Y0 - 1, Z0 - 1, warp, lane);
    box.store(sx, warp, lane);
    __syncthreads();
    const float* base = sx + ty * kZSP + tx;  // window (dz, dy, dx) at plane p: base[p*PL + (1+dy)*kZSP + 1+dx]
    float P[3][9];                            // rolling planes: P[p % 3] = plane p's 3 x 3
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 9; ++j) P[p][j] = base[p * PL + (j / 3) * kZSP + (j % 3)];
    float yprev = 0.0f;
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
#pragma unroll
        for (int j = 0; j < 9; ++j) P[(k + 2) % 3][j] = base[(k + 2) * PL + (j / 3) * kZSP + (j % 3)];
        const int z = Z0 + k;
        const bool own = k < nown;
        const long long c = c0 + k * plane;
        float w[27];
#pragma unroll
        for (int s = 0; s < 27; ++s) w[s] = P[(k + s / 9) % 3][s % 9];
        // branch-free (a cell outside the rank's planes reads the uniform-air
        // row and is not stored), so the cells' chains can interleave
        float yv = win_dot<F, 27>([&](int t) { return kr[t]; }, [&](int t) { return w[t]; });
        if (k + 1 < ZC) load_row(code_row(ct, U, rc[k + 1], c + plane), kr);
        if (!own) yv = 0.0f;
        if (own) y[c] = yv;
        if (POOL) {
            if (k & 1) {
                // quad (x, y), (x+1, y), (x, y+1), (x+1, y+1) of planes z-1, z:
                // lanes l, l+1, l+16, l+17; avg_pool2 order (x, then y, then z)
                const float a1 = __shfl_down_sync(0xffffffffu, yprev, 1), a2 = __shfl_down_sync(0xffffffffu, yprev, 16),
                            a3 = __shfl_down_sync(0xffffffffu, yprev, 17);
                const float b1 = __shfl_down_sync(0xffffffffu, yv, 1), b2 = __shfl_down_sync(0xffffffffu, yv, 16),
                            b3 = __shfl_down_sync(0xffffffffu, yv, 17);
                const int qx = cx >> 1, qy = cy >> 1, qz = (z - 1) >> 1;
                if ((lane & 17) == 0 && qx < gc.nx && qy < gc.ny && z - 1 < g.zo1) {
                    float ps = yprev;
                    ps = __fadd_rn(ps, a1);
                    ps = __fadd_rn(ps, a2);
                    ps = __fadd_rn(ps, a3);
                    ps = __fadd_rn(ps, yv);
                    ps = __fadd_rn(ps, b1);
                    ps = __fadd_rn(ps, b2);
                    ps = __fadd_rn(ps, b3);
                    xnext[lin(gc, qx, qy, qz)] = __fmul_rn(0.125f, ps);
                }
            }
            yprev = yv;
        }
    }
}

// grid (ceil(nx/32), ceil(ny/8), ceil(owned planes/ZC)), block 256
template <bool POOL, int ZC, bool F>
__global__ void __launch_bounds__(kZT, COARSEZ_MINB) k_cdownz(Geom g, const float* __restrict__ x, ConvTab ct,
                                                const __grid_constant__ KC kc, float* __restrict__ y,
                                                float* __restrict__ xnext, Geom gc, const int* __restrict__ done,
                                                const uint8_t* __restrict__ live) {
    // solve path: a tile without fluid near it (k_coarse_live) keeps the zeros
    // its outputs were given for the frame (setup data: read before the wait)
    if (live && !live[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x]) return;
    __shared__ __align__(16) CDownSmem<ZC> S;
    cdownz_tile<POOL, ZC, F>(g, x, ct, kc, y, xnext, gc, blockIdx.x, blockIdx.y, blockIdx.z, S, done);
}

// one tile of an up step (outc is level l+1)
template <int ZC, bool F>
__device__ __forceinline__ void cupz_tile(const Geom& g, const Geom& gc, const float* __restrict__ outc,
                                          const float* __restrict__ yl, const float* __restrict__ zab,
                                          const ConvTab& ct, const KC& kc, float* __restrict__ outl, int bx, int by,
                                          int bz, CUpSmem<ZC>& S, const int* __restrict__ done) {
    static_assert(ZC % 2 == 0, "fine planes come in coarse pairs");
    // coarse box: (X0/2 - 1 .. X0/2 + 16) x (Y0/2 - 1 .. Y0/2 + 4) x (Z0/2 - 1 .. Z0/2 + ZC/2)
    constexpr int CX = kZX / 2 + 2, CY = kZY / 2 + 2, CZ = ZC / 2 + 2, PL = CY * kZSP;
    float* sc = S.sc;
    UniRows& U = S.U;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tx = 16 * (warp & 1) + (lane & 15), ty = 2 * (warp >> 1) + (lane >> 4);
    const int X0 = bx * kZX, Y0 = by * kZY, Z0 = g.zo0 + bz * ZC;
    const int cx = X0 + tx, cy = Y0 + ty;
    const bool oxy = cx < g.nx && cy < g.ny;
    const long long plane = (long long)g.nx * g.ny;
    const long long c0 = oxy ? lin(g, cx, cy, Z0) : 0;
    const int nown = oxy ? min(ZC, g.zo1 - Z0) : 0;  // planes of this column the rank owns
    // setup data first (row codes, the uniform rows, the first cell's row):
    // with programmatic launch it overlaps the previous kernel
    uint32_t rc[ZC];
#pragma unroll
    for (int k = 0; k < ZC; ++k) rc[k] = cell_code(ct, c0 + k * plane, k < nown);
    load_uni_rows(U, kc, tid);
    __syncthreads();
    float kr[28];  // the next cell's kernel row (prefetched one cell ahead)
    load_row(code_row(ct, U, rc[0], c0), kr);
    pdl_wait_then_trigger();  // out_{l+1} is the previous kernel's output (y_l, z an earlier one's)
    if (done && *done) return;  // z-slab chunked loop: the solve has finished (block-uniform)
    ZStager<CX, CY, CZ> box;
    box.load(outc, gc, (X0 >> 1) - 1, (Y0 >> 1) - 1, (Z0 >> 1) - 1, warp, lane);
    float yv[ZC];
#pragma unroll
    for (int k = 0; k < ZC; ++k) yv[k] = k < nown ? __ldg(yl + c0 + k * plane) : 0.0f;
    const float za = zab[0], zb = zab[1];
    box.store(sc, warp, lane);
    __syncthreads();
    // fine tap (cx + dx, cy + dy) -> staged coarse ((cx + dx) >> 1) - (X0/2 - 1), likewise y;
    // out-of-domain fine cells map to out-of-domain coarse cells (dims even): staged zeros
    int off[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const int dy = j / 3 - 1, dx = j % 3 - 1;
        off[j] = (((ty + dy) >> 1) + 1) * kZSP + ((tx + dx) >> 1) + 1;  // X0, Y0 even
    }
    // coarse plane of fine tap (k + dz): ((k + dz) >> 1) + 1 in the box (Z0 even)
    float Q[3][9];  // rolling coarse planes: Q[q % 3] = staged coarse plane q's 9 taps
#pragma unroll
    for (int j = 0; j < 9; ++j) Q[0][j] = sc[off[j]];
#pragma unroll
    for (int k = 0; k < ZC; ++k) {
        const int qn = ((k + 1) >> 1) + 1;  // the new coarse plane this fine plane reaches
        if (k == 0 || (k & 1)) {
#pragma unroll
            for (int j = 0; j < 9; ++j) Q[qn % 3][j] = sc[qn * PL + off[j]];
        }
        const long long c = c0 + k * plane;
        float w[27];
#pragma unroll
        for (int s = 0; s < 27; ++s) {
            const int dz = s / 9 - 1;
            w[s] = Q[(((k + dz) >> 1) + 1) % 3][s % 9];
        }
        const float u = win_dot<F, 27>([&](int t) { return kr[t]; }, [&](int t) { return w[t]; });
        if (k + 1 < ZC) load_row(code_row(ct, U, rc[k + 1], c + plane), kr);
        if (k < nown)
            outl[c] = F ? __fmaf_rn(za, yv[k], __fmul_rn(zb, u)) : __fadd_rn(__fmul_rn(za, yv[k]), __fmul_rn(zb, u));
    }
}

// grid (ceil(nx/32), ceil(ny/8), ceil(owned planes/ZC)), block 256; outc is level l+1
template <int ZC, bool F>
__global__ void __launch_bounds__(kZT, COARSEZ_MINB) k_cupz(Geom g, Geom gc, const float* __restrict__ outc,
                                              const float* __restrict__ yl, const float* __restrict__ zab, ConvTab ct,
                                              const __grid_constant__ KC kc, float* __restrict__ outl,
                                              const int* __restrict__ done, const uint8_t* __restrict__ live) {
    // solve path: only out_l within two cells of a level-l fluid cell is ever
    // read (the level-0 up step reads out_1 within one coarse cell of a fluid
    // cell; each up step reads out_{l+1} within one cell of its own reads), so
    // a tile without fluid within two cells (k_coarse_live) is skipped
    if (live && !live[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x]) return;
    __shared__ __align__(16) CUpSmem<ZC> S;
    cupz_tile<ZC, F>(g, gc, outc, yl, zab, ct, kc, outl, blockIdx.x, blockIdx.y, blockIdx.z, S, done);
}

// Live tiles of a coarse down step (k_cdownz's 32 x 8 x zc tiles, level l >= 1),
// for the solve path only: its input x_l is zero outside the cells within one
// cell of a level-l cell holding fluid (x_0 = r vanishes off the fluid; a conv
// of an all-zero window is zero; pooling keeps the bound), so a tile whose
// window box (tile + 1) has no fluid within 2 cells has y_l = 0 and writes
// zeros only. One block per tile scans the tile +- 2 for a fluid fraction > 0.
__global__ void __launch_bounds__(kBlock) k_coarse_live(Geom g, const float* __restrict__ fluid, int zc,
                                                        uint8_t* __restrict__ live) {
    const int ntx = (g.nx + kZX - 1) / kZX, nty = (g.ny + kZY - 1) / kZY;
    const int t = blockIdx.x, bx = t % ntx, by = (t / ntx) % nty, bz = t / (ntx * nty);
    const int X0 = bx * kZX - 2, Y0 = by * kZY - 2, Z0 = bz * zc - 2;
    const int BX = kZX + 4, BY = kZY + 4, BZ = zc + 4;
    bool any = false;
    for (int i = threadIdx.x; i < BX * BY * BZ && !any; i += blockDim.x) {
        const int x = X0 + i % BX, y = Y0 + (i / BX) % BY, z = Z0 + i / (BX * BY);
        if ((unsigned)x < (unsigned)g.nx && (unsigned)y < (unsigned)g.ny && (unsigned)z < (unsigned)g.nz)
            any = fluid[((long long)z * g.ny + y) * g.nx + x] > 0.0f;
    }
    any = __syncthreads_or(any) != 0;
    if (threadIdx.x == 0) live[t] = any ? 1 : 0;
}

}  // namespace nb2

// Level-0 up sweep of the solve (P3), 3D: at every fluid cell with a
// uniform-fluid window
//     o = z_a y_0 + z_b conv_up_0(upsample2(out_1))     (net/forward.hpp:118-127)
//     d = f64(o) * nrm                                  (net_precond.cpp:31-34)
// fused with the A-orthogonalisation dots d.Ad_j (solver.cpp:239-243). Mixed
// fluid cells follow in k_mixed_up0, which adds these dot totals
// (st->dot_main) to its own and finalises the projections.
//
// The stencil pipeline of stencil.cuh / down0.cuh on the balanced schedule: a
// 32 x 8 block owns a 64 x 8 tile (thread = x pair) and marches z. Each thread
// cp.async-copies its pair's y_0 and Ad_j PF planes ahead (src-size 0 — no
// traffic — for pairs without such a cell); out_1 is staged as 34 x 6 coarse
// planes (tile + halo, zero outside) in a 4-plane ring, one new coarse plane
// every second fine plane. One barrier per plane; a fine tap (x+dx, y+dy,
// z+dz) reads coarse ((x+dx)>>1, (y+dy)>>1, (z+dz)>>1). Slot-order
// round-to-nearest arithmetic: bit-identical to the restatement.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "down0.cuh"
#include "mixed.cuh"
#include "stencil.cuh"

namespace nb2 {

constexpr int kUST = 4;  // own-input stages: the step's two planes and the next step's two in flight
constexpr int kOW = kTX / 2 + 2, kOH = kTY / 2 + 2;  // coarse plane tile (34 x 6)

template <int NO>
struct Up0Smem {
    static constexpr int NA = (NO > 0) ? NO : 1;
    double ad[kUST][NA][kTY][kTX];  // Ad_j, own pairs
    float y[kUST][kTY][kTX];        // y_0, own pairs
    float oc[4][kOH][kOW];          // out_1 coarse planes (ring by coarse z & 3)
};

// the pair has a cell this kernel computes (fluid, uniform-fluid window)
__device__ __forceinline__ bool up_cell(unsigned b) { return (b & 0xfu) == 0u; }  // window 0, type 0
__device__ __forceinline__ bool up_pair(unsigned b2) { return up_cell(b2 & 0xffu) || up_cell(b2 >> 8); }

// The uniform-fluid up kernel: its 27 slots (exact path) and, for the fast
// path, the taps merged per fine-cell parity. Upsampling maps the three fine
// taps of a dimension onto two coarse cells — parity 0: d = -1 -> coarse
// -1, d = 0, +1 -> coarse 0; parity 1: d = -1, 0 -> coarse 0, d = +1 ->
// coarse +1 — so m[pz*4 + py*2 + px][a*4 + b*2 + c] is the sum of k over the
// taps landing on coarse (lo/hi)^3 = (a, b, c): 8 fused multiply-adds per
// cell instead of 27 (forward.hpp:118-127 reassociated; fast path only).
struct KUp0 {
    float k[27];
    float m[8][8];
};

// floor(f / 2) mod 4 for small f >= -2 (coarse ring slot of fine offset f)
__host__ __device__ constexpr int up_cslot(int f) { return ((f + 4) / 2 + 2) % 4; }

// One column segment: tile (tx, ty), planes [zc0, zc1) (both even: the down
// schedule's plane pairs). Two fine planes per step (one barrier), stepping
// 8 planes per chunk with the step index a compile-time constant, so every
// ring slot is a constant offset: own inputs of plane zc0 + k in stage k % 4,
// coarse plane zc0/2 + m in slot m % 4 (one new coarse plane per step).
template <int NO, bool F>
__device__ __forceinline__ void up_l0_segment(const Geom& g, const Geom& gc, const uint8_t* __restrict__ cls,
                                              const float* __restrict__ outc, const float* __restrict__ y0,
                                              const KUp0& kc, float za, float zb, double nrm, int nc,
                                              const double* const (&adp)[(NO > 0) ? NO : 1],
                                              double* __restrict__ dout, double (&acc)[(NO > 0) ? NO : 1], int tx,
                                              int ty, int zc0, int zc1, bool& waited) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Up0Smem<NO>& S = *reinterpret_cast<Up0Smem<NO>*>(smem_raw);
    __syncthreads();  // the previous segment's last reads of S are done
    const int lane = threadIdx.x, row = threadIdx.y, tid = row * kSX + lane;
    const int X0 = tx * kTX, Y0 = ty * kTY;
    const int x = X0 + 2 * lane, yy = Y0 + row;
    const bool own = x < g.nx && yy < g.ny;
    const long long nx = g.nx, plane = nx * g.ny;
    const long long qo = (long long)(own ? yy : 0) * nx + (own ? x : 0);
    // coarse staging role: element tid of the 34 x 6 coarse tile
    const int CX0 = (X0 >> 1) - 1, CY0 = (Y0 >> 1) - 1;
    const bool crole = tid < kOW * kOH;
    const int cr = crole ? tid / kOW : 0, ccol = crole ? tid - cr * kOW : 0;
    const int cgx = CX0 + ccol, cgy = CY0 + cr;
    const bool cxy_in = crole && cgx >= 0 && cgx < gc.nx && cgy >= 0 && cgy < gc.ny;
    const long long cqo = cxy_in ? (long long)cgy * gc.nx + cgx : 0;
    const long long cplane = (long long)gc.nx * gc.ny;
    const int cz0 = zc0 >> 1;  // coarse plane of fine zc0, zc0 + 1
    auto zin = [&](int z) { return z >= 0 && z < g.nz; };
    auto own_bytes = [&](int z) -> unsigned {
        return (own && zin(z)) ? (unsigned)__ldg(reinterpret_cast<const unsigned short*>(cls + z * plane + qo)) : kOut2;
    };
    auto coarse = [&](int k, int cs) {  // stage coarse plane k into slot cs (zero outside)
        if (crole) {
            const bool ok = cxy_in && k >= 0 && k < gc.nz;
            cp_async4(&S.oc[cs][cr][ccol], outc + (ok ? k * cplane + cqo : 0), ok);
        }
    };
    auto fine = [&](int z, int s, unsigned ob) {  // own inputs of plane z into stage s
        if (zin(z)) {
            const bool ol = own && up_pair(ob);
            const long long q = z * plane + qo;
            cp_async8(&S.y[s][row][2 * lane], y0 + q, ol);  // q in the grid: src-size 0 reads nothing
#pragma unroll
            for (int j = 0; j < NO; ++j) cp_async16(&S.ad[s][j][row][2 * lane], adp[j] + q, ol && j < nc);
        }
    };
    // fine row offsets into the coarse tile (per thread): (yy + dy) >> 1 - CY0
    int crow[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) crow[d] = ((yy + d - 1) >> 1) - CY0;

    unsigned ob[8];  // ob[k % 8]: own bytes of plane zc0 + k (planes z .. z+7 at a step)
#pragma unroll
    for (int k = 0; k < 8; ++k) ob[k] = own_bytes(zc0 + k);
    // prologue group: planes zc0, zc0+1 and coarse planes cz0-1 .. cz0+1
    fine(zc0, 0, ob[0]);
    fine(zc0 + 1, 1, ob[1]);
    // y_0 and Ad_j are older than the previous launch; out_1 is its output
    if (!waited) {
        pdl_launch_wait();
        waited = true;
    }
    coarse(cz0 - 1, up_cslot(-2));
    coarse(cz0, up_cslot(0));
    coarse(cz0 + 1, up_cslot(2));
    cp_commit();
    // one step: planes z = z8 + K, z + 1 (K = 2J; z8 - zc0 a multiple of 8)
    auto step = [&](auto Jc, int z8) {
        constexpr int J = decltype(Jc)::value, K = 2 * J;
        const int z = z8 + K;
        // the next step's group: planes z+2, z+3 and coarse plane (z + 4) / 2
        fine(z + 2, (K + 2) % kUST, ob[(K + 2) % 8]);
        fine(z + 3, (K + 3) % kUST, ob[(K + 3) % 8]);
        coarse(cz0 + (z8 - zc0) / 2 + J + 2, up_cslot(K + 4));
        cp_commit();
        cp_wait<1>();     // this step's group landed (own thread)
        __syncthreads();  // and every thread's coarse copies
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const unsigned bc = ob[(K + p) % 8];
            if (!(own && up_pair(bc))) continue;
            const int s = (K + p) % kUST;
            const float2 yv = *reinterpret_cast<const float2*>(&S.y[s][row][2 * lane]);
            float u[2];
            if (F) {
                // merged parity taps: coarse (lo, hi) per dimension
                const int zl = up_cslot(K + p - 1), zh = up_cslot(K + p + 1);
                const int pyz = (p << 2) | ((yy & 1) << 1);  // z + p has parity p (z even)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float* m = kc.m[pyz | h];
                    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int b = t >> 1, cc = t & 1;
                        const int rr = crow[2 * b], col = lane + h + cc;
                        a0 = __fmaf_rn(m[t], S.oc[zl][rr][col], a0);
                        a1 = __fmaf_rn(m[4 + t], S.oc[zh][rr][col], a1);
                    }
                    u[h] = __fadd_rn(a0, a1);
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float a = 0.0f;
#pragma unroll
                    for (int t = 0; t < 27; ++t) {
                        const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                        const int kz = up_cslot(K + p + dz);
                        const int col = lane + ((h + dx) >> 1) + 1;  // ((x + h + dx) >> 1) - CX0
                        a = __fadd_rn(a, __fmul_rn(kc.k[t], S.oc[kz][crow[dy + 1]][col]));
                    }
                    u[h] = a;
                }
            }
            const long long q = (z + p) * plane + qo;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!up_cell((bc >> (8 * h)) & 0xffu)) continue;
                const float o = F ? __fmaf_rn(za, h ? yv.y : yv.x, __fmul_rn(zb, u[h]))
                                  : __fadd_rn(__fmul_rn(za, h ? yv.y : yv.x), __fmul_rn(zb, u[h]));
                const double dv = __dmul_rn((double)o, nrm);
                dout[q + h] = dv;
#pragma unroll
                for (int j = 0; j < NO; ++j)
                    if (j < nc) acc[j] += dv * S.ad[s][j][row][2 * lane + h];
            }
        }
        ob[K % 8] = own_bytes(z + 8);
        ob[(K + 1) % 8] = own_bytes(z + 9);
        __syncthreads();  // the slots this step read are restaged by the next step's issue
    };
    for (int z8 = zc0; z8 < zc1; z8 += 8) {
        step(std::integral_constant<int, 0>{}, z8);
        if (z8 + 2 >= zc1) break;
        step(std::integral_constant<int, 1>{}, z8);
        if (z8 + 4 >= zc1) break;
        step(std::integral_constant<int, 2>{}, z8);
        if (z8 + 6 >= zc1) break;
        step(std::integral_constant<int, 3>{}, z8);
    }
    cp_wait<0>();
}

// UP0_MINB: optional register cap. Unset, the bound has no block count and
// ptxas settles at 64 registers (4 blocks/SM); an explicit 1 gives 80 (3 blocks,
// 54.6 -> 56.1 us), 4 gives 48 (61 -> 64 us), 5 gives 42 (-> 66 us).
#ifdef UP0_MINB
#define UP0_BOUNDS __launch_bounds__(kSX* kSY, UP0_MINB)
#else
#define UP0_BOUNDS __launch_bounds__(kSX* kSY)
#endif
template <int NO, bool F>
__global__ void UP0_BOUNDS k_up_l0(Geom g, Geom gc, const uint8_t* __restrict__ cls,
                                                    const float* __restrict__ outc, const float* __restrict__ y0,
                                                    const float* __restrict__ zab, const __grid_constant__ KUp0 kc,
                                                    double* __restrict__ dout, SolverState* st,
                                                    const double* __restrict__ ADring, double* __restrict__ partials,
                                                    unsigned int* __restrict__ counter, Sched sc) {
    constexpr int NA = (NO > 0) ? NO : 1;
    if (st->dist && st->done) {  // (written by the update, three launches back)
        pdl_launch_wait();
        return;
    }
    const float za = zab[0], zb = zab[1];
    const double nrm = st->nrm;
    const int nc = st->n_cache, R = st->ring;
    const double* adp[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
        adp[j] = ADring + (long long)slot * g.n;
    }
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;
    bool waited = false;  // reads before the programmatic wait: st, y_0, Ad_j, cell bytes (older launches)
    sched_for_each(sc, [&](int tx, int ty, int u0, int u1) {  // units: plane pairs (the down schedule)
        up_l0_segment<NO, F>(g, gc, cls, outc, y0, kc, za, zb, nrm, nc, adp, dout, acc, tx, ty, 2 * u0,
                             min(2 * u1, g.nz), waited);
    });
    if (!waited) pdl_launch_wait();
    double tot[NA];
    // the mixed fluid cells follow in k_mixed_up0, which finalises the MGS
    // projections from these totals plus its own
    if (grid_reduce<NA>(acc, partials, counter, tot) && threadIdx.x == 0 && threadIdx.y == 0)
        for (int j = 0; j < NA; ++j) st->dot_main[j] = tot[j];
}

// k_up_l0 and k_mixed_up0 as one launch: blocks [0, nb_tiled) march the
// uniform-fluid tiles, the others take the mixed fluid cells of the up list;
// one grid reduction over all blocks gives the dots d.Ad_j and the MGS
// projections (the two kernels' cell sets are disjoint, so nothing waits).
template <int NO, bool F>
__global__ void UP0_BOUNDS k_up_l0m(Geom g, Geom gc, const uint8_t* __restrict__ cls, const float* __restrict__ outc,
                                     const float* __restrict__ y0, const float* __restrict__ zab,
                                     const __grid_constant__ KUp0 kc, double* __restrict__ dout, SolverState* st,
                                     const double* __restrict__ ADring, double* __restrict__ partials,
                                     unsigned int* __restrict__ counter, Sched sc, int nb_tiled,
                                     const uint32_t* __restrict__ ulist, const uint32_t* __restrict__ ucount,
                                     const float* __restrict__ tab, const uint32_t* __restrict__ ukid) {
    constexpr int NA = (NO > 0) ? NO : 1;
    if (st->dist && st->done) {  // (written by the update, three launches back)
        pdl_launch_wait();
        return;
    }
    const float za = zab[0], zb = zab[1];
    const double nrm = st->nrm;
    const int nc = st->n_cache, R = st->ring;
    const double* adp[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
        adp[j] = ADring + (long long)slot * g.n;
    }
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;
    bool waited = false;  // reads before the programmatic wait: st, y_0, Ad_j, cell bytes (older launches)
    if ((int)blockIdx.x < nb_tiled) {
        sched_for_each_n(sc, blockIdx.x, nb_tiled, [&](int tx, int ty, int u0, int u1) {  // plane pairs
            up_l0_segment<NO, F>(g, gc, cls, outc, y0, kc, za, zb, nrm, nc, adp, dout, acc, tx, ty, 2 * u0,
                                 min(2 * u1, g.nz), waited);
        });
        if (!waited) pdl_launch_wait();
    } else {
        pdl_launch_wait();  // the mixed cells read out_1 at once
        const int tid = threadIdx.y * kSX + threadIdx.x;
        const long long nthr = (long long)(gridDim.x - nb_tiled) * (kSX * kSY);
        mixed_up_cells<3, NO, F>(g, gc, ulist, *ucount, outc, y0, za, zb, tab, ukid, dout, nrm, nc, adp, acc,
                                 (long long)(blockIdx.x - nb_tiled) * (kSX * kSY) + tid, nthr);
    }
    double tot[NA];
    if (grid_reduce<NA, kSX * kSY>(acc, partials, counter, tot) && threadIdx.x == 0 && threadIdx.y == 0) {
        if (st->dist) {
            for (int j = 0; j < kMaxOrtho; ++j) st->part[j] = (j < nc && j < NO) ? tot[j] : 0.0;
        } else {
            fin_projections(st, tot);
        }
    }
}

}  // namespace nb2

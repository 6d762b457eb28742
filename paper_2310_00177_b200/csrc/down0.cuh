// Level-0 down sweep of the solve (P1), 3D: y_0 = conv_down_0(x_0) and
// x_1 = avg_pool(y_0), with x_0 = f32((r * inv1) * inv2) (net_precond.cpp:24-29,
// net/forward.hpp:105-113).
//
// At level 0 the window classes make the work sparse: a uniform air/solid
// window has an all-zero input (y_0 = +0), a mixed window's y_0 was computed by
// k_mixed_down0, so only uniform-fluid cells convolve — with one constant
// kernel (compile-time offsets into the parameter bank). The kernel is the
// stencil pipeline of stencil.cuh: a 32 x 8 block owns a 64 x 8 tile (one
// thread per x pair) and marches z; each thread cp.async-copies the residual
// of its pair and halo assignment PF planes ahead (src-size 0 for pairs
// without fluid: zero-fill, no DRAM read; r is exactly 0 there) and converts
// its own copies into a 4-plane f32 ring; one barrier per plane; taps are read
// from shared memory. Pooling: the even row of each row pair sums the 2x2x2
// blocks in the restatement's order at odd planes. Arithmetic order per cell
// is apply_kernels' (net/kernels.hpp:147-172): bit-identical.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "net.cuh"
#include "stencil.cuh"

namespace nb2 {

struct KC0 {
    float k[27];
};

// Two planes per step: planes z, z+1 (z even) are convolved after ONE barrier
// (four independent accumulation chains per thread), and their 2x2x2 pools
// are summed after the next step's barrier.
#ifndef D0_AHEAD
#define D0_AHEAD 2  // planes in flight beyond the step's two (4 and 6 measured slower at C3 256^3: 69.8 / 70.2 vs 66.2 us)
#endif
constexpr int kD0A = D0_AHEAD;
constexpr int kD0R = kD0A + 2;  // raw (f64) plane stages: planes z+1 .. z+2+kD0A
constexpr int kD0X = 8;  // x_0 (f32) plane ring: z-3 .. z+2 in use around a barrier

struct Down0Smem {
    double raw[kD0R][kVH][kVW];  // residual copies (tile + halo)
    float xin[kD0X][kVH][kVW];   // converted network input x_0
    float yp[2][2][kTY][kTX];    // y_0 of a step's two planes, double-buffered (pooling)
};

// One column segment: tile (tx, ty), planes [zc0, zc1) (both even). The z
// loop runs in chunks of 8 planes (4 steps of 2) with the step index a
// compile-time constant, so every ring slot (raw stages, x_0 planes, own cell
// bytes, pooling buffers) is a constant offset: no per-plane slot arithmetic.
// Every thread issues one own copy and at most one halo copy per plane, both
// 16-byte pairs (column halos as the aligned pair holding the halo cell), so
// the issue and conversion code has no per-role branches.
template <bool F>
__device__ __forceinline__ void down_l0_segment(const Geom& g, const uint8_t* __restrict__ cls,
                                                const double* __restrict__ r, const SolverState* __restrict__ st,
                                                const KC0& kc, float* __restrict__ y, float* __restrict__ xnext,
                                                const Geom& gc, int tx, int ty, int zc0, int zc1, bool& waited) {
    static_assert(kD0R == 4 && kD0X == 8, "the 8-plane chunk maps ring slots to constants");
    const int lane = threadIdx.x, row = threadIdx.y;
    const int X0 = tx * kTX, Y0 = ty * kTY;
    const int x = X0 + 2 * lane, yy = Y0 + row;
    const bool own = x < g.nx && yy < g.ny;  // nx even: the pair is whole
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Down0Smem& S = *reinterpret_cast<Down0Smem*>(smem_raw);
    __syncthreads();  // the previous segment's last reads of S are done
    const long long nx = g.nx, plane = nx * g.ny;
    const double inv1 = st->inv1, inv2 = st->inv2;
    // halo pair (even x, 16 bytes): rows above / below (rows 0, 1), the column
    // pairs holding x0-1 / x0+64 (row 2, lanes < 16) and the four corners
    // (row 3, lanes < 4); staged at (hsr, hsc .. hsc+1)
    bool hk = false;
    int hx = 0, hy = 0, hsr = 0, hsc = 0;
    if (row == 0 || row == 1) {
        hk = true;
        hx = x;
        hy = (row == 0) ? Y0 - 1 : Y0 + kTY;
        hsr = (row == 0) ? 0 : kVH - 1;
        hsc = 2 + 2 * lane;
    } else if (row == 2 && lane < 2 * kTY) {
        hk = true;
        hx = (lane < kTY) ? X0 - 2 : X0 + kTX;
        hy = Y0 + (lane & (kTY - 1));
        hsr = 1 + (lane & (kTY - 1));
        hsc = (lane < kTY) ? 0 : kTX + 2;
    } else if (row == 3 && lane < 4) {
        hk = true;
        hx = (lane & 1) ? X0 + kTX : X0 - 2;
        hy = (lane & 2) ? Y0 + kTY : Y0 - 1;
        hsr = (lane & 2) ? kVH - 1 : 0;
        hsc = (lane & 1) ? kTX + 2 : 0;
    }
    const bool h_in = hk && hx >= 0 && hx < g.nx && hy >= 0 && hy < g.ny;
    const long long qo = (long long)(own ? yy : 0) * nx + (own ? x : 0);
    const long long qh = h_in ? (long long)hy * nx + hx : 0;
    auto zin = [&](int z) { return z >= 0 && z < g.nz; };
    auto own_bytes = [&](int z) -> unsigned {
        return (own && zin(z)) ? (unsigned)__ldg(reinterpret_cast<const unsigned short*>(cls + z * plane + qo)) : kOut2;
    };
    // own pairs without fluid zero-filled; halo always copied (exact zeros).
    // The source address is in the grid whatever the predicate: src-size 0 reads nothing.
    const double* r_own = r + qo;
    const double* r_halo = r + qh;
    // plane z into raw stage RS
    auto issue = [&](int z, int rs, unsigned ob) {
        if (zin(z)) {
            const long long qz = z * plane;
            cp_async16(&S.raw[rs][row + 1][2 + 2 * lane], r_own + qz, own && pair_live(ob));
            if (hk) cp_async16(&S.raw[rs][hsr][hsc], r_halo + qz, h_in);
        }
        cp_commit();
    };
    auto cvt = [&](double v) { return __double2float_rn(__dmul_rn(__dmul_rn(v, inv1), inv2)); };
    // raw stage RS -> x_0 plane slot XS (zeros outside the domain)
    auto form = [&](int z, int rs, int xs) {
        const bool zi = zin(z);
        const double2 o = *reinterpret_cast<const double2*>(&S.raw[rs][row + 1][2 + 2 * lane]);
        *reinterpret_cast<float2*>(&S.xin[xs][row + 1][2 + 2 * lane]) =
            zi ? make_float2(cvt(o.x), cvt(o.y)) : make_float2(0.0f, 0.0f);
        if (hk) {
            const double2 h = *reinterpret_cast<const double2*>(&S.raw[rs][hsr][hsc]);
            *reinterpret_cast<float2*>(&S.xin[xs][hsr][hsc]) =
                zi ? make_float2(cvt(h.x), cvt(h.y)) : make_float2(0.0f, 0.0f);
        }
    };
    // mixed cells' y_0 (k_mixed_down0), loaded a step ahead
    auto mixed_y = [&](int z, unsigned b2, float& ya, float& yb) {
        const long long q = z * plane + qo;
        const uint8_t ba = (uint8_t)(b2 & 0xffu), bb = (uint8_t)(b2 >> 8);
        ya = (own && zin(z) && cls_window(ba) == 3 && cls_wfluid(ba)) ? __ldg(y + q) : 0.0f;
        yb = (own && zin(z) && cls_window(bb) == 3 && cls_wfluid(bb)) ? __ldg(y + q + 1) : 0.0f;
    };
    // 2x2x2 pool of the step at z (its y_0 tile in yp[b]), restatement order:
    // x fastest, then y, then z (avg_pool2, net/kernels.hpp:279-292)
    auto pool = [&](int z, int b) {
        if (own && !(row & 1)) {
            float ps = S.yp[b][0][row][2 * lane];
            ps = __fadd_rn(ps, S.yp[b][0][row][2 * lane + 1]);
            ps = __fadd_rn(ps, S.yp[b][0][row + 1][2 * lane]);
            ps = __fadd_rn(ps, S.yp[b][0][row + 1][2 * lane + 1]);
            ps = __fadd_rn(ps, S.yp[b][1][row][2 * lane]);
            ps = __fadd_rn(ps, S.yp[b][1][row][2 * lane + 1]);
            ps = __fadd_rn(ps, S.yp[b][1][row + 1][2 * lane]);
            ps = __fadd_rn(ps, S.yp[b][1][row + 1][2 * lane + 1]);
            xnext[lin(gc, x >> 1, yy >> 1, z >> 1)] = __fmul_rn(0.125f, ps);
        }
    };

    // ring slots relative to zc0: plane zc0 + k uses raw stage (k + 1) % 4 and
    // x_0 slot (k + 1) % 8; ob[(k) % 8] holds plane zc0 + k's own bytes
    unsigned ob[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) ob[k] = own_bytes(zc0 + k);
    // prologue: planes zc0-1 .. zc0+2 issued, zc0-1 and zc0 formed
    issue(zc0 - 1, 0, own_bytes(zc0 - 1));
#pragma unroll
    for (int k = 0; k <= kD0A; ++k) issue(zc0 + k, (k + 1) % kD0R, ob[k]);
    // r (the update two launches back) and the cell bytes are complete; the
    // mixed cells' y_0 is the previous launch's (k_mixed_down0): wait for it
    if (!waited) {
        pdl_launch_wait();
        waited = true;
    }
    cp_wait<kD0A>();  // planes zc0-1, zc0 landed
    form(zc0 - 1, 0, 0);
    form(zc0, 1, 1);
    float my[2][2];
    mixed_y(zc0, ob[0], my[0][0], my[0][1]);
    mixed_y(zc0 + 1, ob[1], my[1][0], my[1][1]);
    // one step: planes z = z8 + 2J, z + 1
    auto step = [&](auto Jc, int z8) {
        constexpr int J = decltype(Jc)::value;
        constexpr int K = 2 * J;  // z - z8 (z8 - zc0 is a multiple of 8)
        const int z = z8 + K;
        issue(z + kD0A + 1, (K + kD0A + 2) % kD0R, ob[(K + kD0A + 1) % 8]);
        issue(z + kD0A + 2, (K + kD0A + 3) % kD0R, ob[(K + kD0A + 2) % 8]);
        cp_wait<kD0A>();  // planes z+1, z+2 landed (own copies)
        form(z + 1, (K + 2) % kD0R, (K + 2) % kD0X);
        form(z + 2, (K + 3) % kD0R, (K + 3) % kD0X);
        float ny[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
        if (z + 2 < zc1) {
            mixed_y(z + 2, ob[(K + 2) % 8], ny[0][0], ny[0][1]);
            mixed_y(z + 3, ob[(K + 3) % 8], ny[1][0], ny[1][1]);
        }
        __syncthreads();  // x_0 of planes z-1 .. z+2 complete; yp of the last step too
        if (z > zc0) pool(z - 2, (J + 1) & 1);
        const int c0 = 2 + 2 * lane, r0 = row + 1;
        float yv[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
        if (own) {
            // uniform-fluid windows convolve with the constant kernel (win_dot:
            // slot order, or fused chains per plane); the four cells' chains
            // are independent
            float acc[2][2];
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    acc[p][h] = win_dot<F, 27>([&](int t) { return kc.k[t]; }, [&](int t) {
                        const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                        return S.xin[(K + p + dz + 1 + kD0X) % kD0X][r0 + dy][c0 + h + dx];
                    });
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const unsigned bc = ob[(K + p) % 8];
                const uint8_t ba = (uint8_t)(bc & 0xffu), bb = (uint8_t)(bc >> 8);
                const int wa = cls_window(ba), wb = cls_window(bb);
                yv[p][0] = (wa == 0) ? acc[p][0] : (wa == 3 ? my[p][0] : 0.0f);
                yv[p][1] = (wb == 0) ? acc[p][1] : (wb == 3 ? my[p][1] : 0.0f);
                // y_0 is stored at fluid cells; mixed ones already hold it
                const long long q = (z + p) * plane + qo;
                if (cls_type(ba) == 0 && wa != 3) y[q] = yv[p][0];
                if (cls_type(bb) == 0 && wb != 3) y[q + 1] = yv[p][1];
            }
        }
#pragma unroll
        for (int p = 0; p < 2; ++p)
            *reinterpret_cast<float2*>(&S.yp[J & 1][p][row][2 * lane]) = make_float2(yv[p][0], yv[p][1]);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            my[p][0] = ny[p][0];
            my[p][1] = ny[p][1];
        }
        ob[K % 8] = own_bytes(z + 8);
        ob[(K + 1) % 8] = own_bytes(z + 9);
    };
    int last_pb = 0;
    for (int z8 = zc0; z8 < zc1; z8 += 8) {
        step(std::integral_constant<int, 0>{}, z8);
        last_pb = 0;
        if (z8 + 2 >= zc1) break;
        step(std::integral_constant<int, 1>{}, z8);
        last_pb = 1;
        if (z8 + 4 >= zc1) break;
        step(std::integral_constant<int, 2>{}, z8);
        last_pb = 0;
        if (z8 + 6 >= zc1) break;
        step(std::integral_constant<int, 3>{}, z8);
        last_pb = 1;
    }
    cp_wait<0>();
    __syncthreads();
    pool(zc1 - 2, last_pb);
}

// Balanced schedule (Sched, units of two planes: pooling pairs stay inside a
// segment); dynamic smem = sizeof(Down0Smem). Units outside the schedule have
// an all-zero window: their x_1 cells keep the zeros set before the solve.
#ifndef D0_MINB
#define D0_MINB 3  // 3 blocks/SM (77 registers; 116 uncapped, 2 blocks): 67 -> 61 us at C3 256^3; 4 (64 registers): 62.3 us
#endif
template <bool F>
__global__ void __launch_bounds__(kSX* kSY, D0_MINB) k_down_l0(Geom g, const uint8_t* __restrict__ cls,
                                                      const double* __restrict__ r, const SolverState* __restrict__ st,
                                                      const __grid_constant__ KC0 kc, float* __restrict__ y,
                                                      float* __restrict__ xnext, Geom gc, Sched sc) {
    // reads before the programmatic wait: the solver state and r (written two
    // launches back), cell bytes and the schedule (setup)
    if (st->dist && st->done) {
        pdl_launch_wait();
        return;
    }
    bool waited = false;
    sched_for_each(sc, [&](int tx, int ty, int u0, int u1) {
        down_l0_segment<F>(g, cls, r, st, kc, y, xnext, gc, tx, ty, 2 * u0, min(2 * u1, g.nz), waited);
    });
    if (!waited) pdl_launch_wait();
}

}  // namespace nb2

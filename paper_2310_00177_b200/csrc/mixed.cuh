// Level-0 mixed-window cells, processed apart from the tiled network kernels.
//
// A cell whose 3^D window is not one pure cell type needs its own kernel (a
// row of the compact table, build_kernels net/kernels.hpp:121-144). Inside the
// tiled kernels such cells cost a dependent chain (cell byte -> mixed index ->
// 27 table loads) that stalls whole warps at every wall and interface. Here
// they are a compact list: one thread per mixed cell, table rows read with
// consecutive indices (fully coalesced SoA), window taps gathered (L2 hits).
//
// k_mixed_down0: y_0 at every mixed cell whose window holds fluid, before the
//   level-0 down kernel (which loads it instead of convolving, so the pooling
//   order is unchanged).
// k_mixed_up0:   d at every mixed fluid cell, after k_up3<kUpL0> (which skips
//   them); its last block adds the main kernel's dot totals (st->dot_main) to
//   its own in a fixed order and finalises the MGS projections.
// Arithmetic order per cell is the restatement's (bit-identical outputs).
#pragma once

#include "common.cuh"

namespace nb2 {

// compact list of the cells of a segment mask (the owned mixed cells:
// list[mixed_index(c)] = c), one thread per 32-cell segment: reads 4 bytes
// of mask per 32 cells instead of every cell byte
__global__ void __launch_bounds__(kBlock) k_mixed_list(long long nseg, const uint32_t* __restrict__ mmask,
                                                       const uint32_t* __restrict__ mbase, uint32_t* __restrict__ list) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long seg = (long long)blockIdx.x * blockDim.x + threadIdx.x; seg < nseg; seg += stride) {
        uint32_t m = mmask[seg];
        if (!m) continue;
        uint32_t k = mbase[seg];
        const uint32_t c0 = (uint32_t)(seg << 5);
        while (m) {
            const int b = __ffs(m) - 1;
            list[k++] = c0 + (uint32_t)b;
            m &= m - 1;
        }
    }
}

// Exclusive scans of up to four segment-count arrays of nseg entries (the
// total left in base[nseg]) and, optionally, the compacted list of the set
// bits of array 0's mask (k_mixed_list) — one block, one launch: for the small
// arrays of the coarse levels and of small grids, where two cub launches per
// scan cost more than the work. (set_mask writes the lists with k_mixed_list:
// one block's serial per-segment loops took 37 us for level 0 at 64^3.)
struct SmallScan {
    const uint32_t* cnt[4];
    uint32_t* base[4];
    int n;
    const uint32_t* mask;  // nullptr: no list
    uint32_t* list;
};
constexpr int kScanSmallT = 1024;
constexpr int kScanSmallPer = 8;  // segments per thread
constexpr long long kScanSmallMax = (long long)kScanSmallT * kScanSmallPer;
__device__ __forceinline__ int ss_pad(int i) { return i + (i >> 5); }  // conflict-free chunk reads

// Global loads and stores are coalesced (thread t: segments t + 1024 i); the
// scan reads each thread's 8 consecutive segments from shared memory.
__global__ void __launch_bounds__(kScanSmallT) k_scan_small(long long nseg_ll, SmallScan a) {
    __shared__ uint32_t buf[kScanSmallMax + kScanSmallMax / 32];
    __shared__ uint32_t wsum[kScanSmallT / 32];
    const int nseg = (int)nseg_ll;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k >= a.n) break;
        const uint32_t* __restrict__ cnt = a.cnt[k];
        uint32_t v[kScanSmallPer], mk[kScanSmallPer];  // counts (and array 0's masks), issued together
#pragma unroll
        for (int i = 0; i < kScanSmallPer; ++i) {
            const int s = t + kScanSmallT * i;
            v[i] = (s < nseg) ? cnt[s] : 0u;
            mk[i] = (k == 0 && a.mask && s < nseg) ? a.mask[s] : 0u;
        }
#pragma unroll
        for (int i = 0; i < kScanSmallPer; ++i) buf[ss_pad(t + kScanSmallT * i)] = v[i];
        __syncthreads();
        uint32_t c[kScanSmallPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kScanSmallPer; ++j) {
            c[j] = buf[ss_pad(kScanSmallPer * t + j)];
            sum += c[j];
        }
        uint32_t x = sum;  // inclusive warp scan, then the warps' totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t q = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, q, o);
                if (lane >= o) q += y;
            }
            wsum[lane] = q;
        }
        __syncthreads();
        uint32_t run = x - sum + (w ? wsum[w - 1] : 0u);
#pragma unroll
        for (int j = 0; j < kScanSmallPer; ++j) {
            buf[ss_pad(kScanSmallPer * t + j)] = run;
            run += c[j];
        }
        __syncthreads();
        uint32_t* __restrict__ base = a.base[k];
#pragma unroll
        for (int i = 0; i < kScanSmallPer; ++i) {
            const int s = t + kScanSmallT * i;
            if (s < nseg) base[s] = buf[ss_pad(s)];
        }
        if (t == 0) base[nseg] = wsum[kScanSmallT / 32 - 1];
        if (k == 0 && a.mask) {  // the list: adjacent lanes, adjacent segments
#pragma unroll
            for (int i = 0; i < kScanSmallPer; ++i) {
                const int s = t + kScanSmallT * i;
                if (s >= nseg) break;
                uint32_t m = mk[i], q = buf[ss_pad(s)];
                const uint32_t c0 = (uint32_t)s << 5;
                while (m) {
                    a.list[q++] = c0 + (uint32_t)(__ffs(m) - 1);
                    m &= m - 1;
                }
            }
        }
        __syncthreads();  // buf and wsum are reused by the next array
    }
}

// The solve needs y_0 only at mixed cells whose window holds a fluid cell (the
// input is zero over the others: y_0 = +0, never computed or read) and the up
// output only at fluid cells. Those two sublists of the level-0 mixed cells
// (with their pattern ids), ascending cell order kept, come from segment masks
// like every other cell list: k_sub_masks (one warp per 32-cell segment), a
// scan of the counts, then k_mixed_sub places each mixed cell.
__global__ void __launch_bounds__(kBlock) k_sub_masks(Geom g, const uint8_t* __restrict__ cls,
                                                      uint32_t* __restrict__ dmask, uint32_t* __restrict__ dcount,
                                                      uint32_t* __restrict__ umask, uint32_t* __restrict__ ucount) {
    const long long nseg = (g.n + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long wstride = (long long)gridDim.x * blockDim.x / 32;
    for (long long seg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32; seg < nseg; seg += wstride) {
        const long long c = seg * 32 + lane;
        const bool in = c >= owned_lo(g) && c < owned_hi(g);
        const uint8_t b = in ? cls[c] : 0;
        const bool mixed = in && cls_window(b) == 3;
        const uint32_t dm = __ballot_sync(0xffffffffu, mixed && cls_wfluid(b));
        const uint32_t um = __ballot_sync(0xffffffffu, mixed && cls_type(b) == 0);
        if (lane == 0) {
            dmask[seg] = dm;
            dcount[seg] = __popc(dm);
            umask[seg] = um;
            ucount[seg] = __popc(um);
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_mixed_sub(const uint32_t* __restrict__ list,
                                                      const uint32_t* __restrict__ pid,
                                                      const uint32_t* __restrict__ count,
                                                      const uint32_t* __restrict__ dmask, const uint32_t* __restrict__ dbase,
                                                      const uint32_t* __restrict__ umask, const uint32_t* __restrict__ ubase,
                                                      uint32_t* __restrict__ dlist, uint32_t* __restrict__ dkid,
                                                      uint32_t* __restrict__ ulist, uint32_t* __restrict__ ukid) {
    const uint32_t n = *count;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t c = list[i], k = pid[i];
        const uint32_t bit = 1u << (c & 31);
        if (dmask[c >> 5] & bit) {
            const long long j = mixed_index(dmask, dbase, c);
            dlist[j] = c;
            dkid[j] = k;
        }
        if (umask[c >> 5] & bit) {
            const long long j = mixed_index(umask, ubase, c);
            ulist[j] = c;
            ukid[j] = k;
        }
    }
}

// levels >= 1: one word per cell, (window class << 30) | mixed row, so the
// coarse kernels reach a mixed cell's row with one load (coarse.cuh). The
// row is the cell's dictionary pattern, or (*unverified) its mixed index;
// rows at or beyond the table capacity read row 0 (the frame is redone, see
// k_build_rows).
__global__ void __launch_bounds__(kBlock) k_row_codes(Geom g, const uint8_t* __restrict__ cls,
                                                      const uint32_t* __restrict__ mmask,
                                                      const uint32_t* __restrict__ mbase,
                                                      const uint32_t* __restrict__ pid,
                                                      const uint32_t* __restrict__ unverified, uint32_t rows_cap,
                                                      uint32_t* __restrict__ rcode) {
    const bool pc = *unverified != 0;
    FOR_OWNED(g, c) {
        const uint32_t w = (uint32_t)cls_window(cls[c]);
        uint32_t row = 0;
        if (w == 3) {
            row = (uint32_t)mixed_index(mmask, mbase, c);
            if (!pc) row = pid[row];
            if (row >= rows_cap) row = 0;
        }
        rcode[c] = (w << 30) | row;
    }
}

__device__ __forceinline__ void decode32(const Geom& g, uint32_t c, int& x, int& y, int& z) {
    const uint32_t nx = (uint32_t)g.nx, ny = (uint32_t)g.ny;
    const uint32_t row = c / nx;
    x = (int)(c - row * nx);
    z = (int)(row / ny);
    y = (int)(row - (uint32_t)z * ny);
}

template <int D, bool F>
#ifndef MIXDN_MINB
#define MIXDN_MINB 4  // register cap (64: no spills with the row-run path; round 1: 5 blocks/SM, 37 -> 29 us)
#endif
__global__ void __launch_bounds__(kBlock, MIXDN_MINB) k_mixed_down0(Geom g, const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ count, const double* __restrict__ r,
                                                        const SolverState* __restrict__ st,
                                                        const float* __restrict__ tab, const uint32_t* __restrict__ kid,
                                                        float* __restrict__ y) {
    constexpr int S = Sh<D>::S;
    // the first cell's list entry and kernel row are setup data: loaded before
    // the programmatic wait (the previous launch writes r). The loop is
    // warp-uniform: a warp takes 32 consecutive list entries.
    const uint32_t n = *count;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long i = i0;
    uint32_t c = 0;
    float k[S];
    auto fetch = [&](long long j) {
        c = list[j];
        const float* K = tab + (long long)__ldg(kid + j) * kRowW;
#pragma unroll
        for (int s = 0; s < S; ++s) k[s] = __ldg(K + s);
    };
    if (i < n) fetch(i);
    pdl_launch_wait();
    if (st->dist && st->done) return;
    const double inv1 = st->inv1, inv2 = st->inv2;
    const long long plane = (long long)g.nx * g.ny;
    auto cvt = [&](double v) { return __double2float_rn(__dmul_rn(__dmul_rn(v, inv1), inv2)); };
    for (; i - lane < n; i += stride) {
        const bool valid = i < n;
        if (valid && i != i0) fetch(i);
        // 32 consecutive cells of one x row (a flat surface or wall): the 3 x 3
        // rows of their windows are read once, coalesced, converted once, and
        // handed to the neighbours by shuffles (the same values as the gather,
        // summed in win_dot's order)
        const uint32_t cf = __shfl_sync(0xffffffffu, c, 0), cl = __shfl_sync(0xffffffffu, c, 31);
        const bool run = D == 3 && __all_sync(0xffffffffu, valid) && cl - cf == 31u &&
                         (cf % (uint32_t)g.nx) + 31u < (uint32_t)g.nx;
        float yv = 0.0f;
        if (run) {
            int x0, y0, z0;
            decode32(g, cf, x0, y0, z0);
            float a[3] = {0.0f, 0.0f, 0.0f};  // exact: a[0] only (slot order); fast: one chain per window plane
#pragma unroll
            for (int rr = 0; rr < 9; ++rr) {
                const int dy = rr % 3 - 1, dz = rr / 3 - 1;
                const bool rin = (unsigned)(y0 + dy) < (unsigned)g.ny && (unsigned)(z0 + dz) < (unsigned)g.nz;
                const double* rowp = r + ((long long)(z0 + dz) * plane + (long long)(y0 + dy) * g.nx + x0);
                // v: x0 - 1 + lane; e: x0 + 31 (lane 0), x0 + 32 (lane 1)
                const float v = (rin && x0 - 1 + lane >= 0) ? cvt(__ldg(rowp - 1 + lane)) : 0.0f;
                const float e = (rin && lane < 2 && x0 + 31 + lane < g.nx) ? cvt(__ldg(rowp + 31 + lane)) : 0.0f;
                const float v1 = __shfl_down_sync(0xffffffffu, v, 1), v2 = __shfl_down_sync(0xffffffffu, v, 2);
                const float e0 = __shfl_sync(0xffffffffu, e, 0), e1 = __shfl_sync(0xffffffffu, e, 1);
                const float t3[3] = {v, (lane < 31) ? v1 : e0, (lane < 30) ? v2 : (lane == 30 ? e0 : e1)};
#pragma unroll
                for (int dx = 0; dx < 3; ++dx) {
                    const int sl = rr * 3 + dx;
                    if (F)
                        a[dz + 1] = __fmaf_rn(k[sl], t3[dx], a[dz + 1]);
                    else
                        a[0] = __fadd_rn(a[0], __fmul_rn(k[sl], t3[dx]));
                }
            }
            yv = F ? __fadd_rn(__fadd_rn(a[0], a[1]), a[2]) : a[0];
        } else if (valid) {
            int x, yy, z;
            decode32(g, c, x, yy, z);
            yv = win_dot<F, S>([&](int t) { return k[t]; }, [&](int s2) {
                const int dx = s2 % 3 - 1, dy = (s2 / 3) % 3 - 1, dz = (D == 3) ? s2 / 9 - 1 : 0;
                const int xx = x + dx, y2 = yy + dy, zz = z + dz;
                const bool in = xx >= 0 && xx < g.nx && y2 >= 0 && y2 < g.ny && zz >= 0 && zz < g.nz;
                return in ? cvt(__ldg(r + lin(g, xx, y2, zz))) : 0.0f;
            });
        }
        if (valid) y[c] = yv;
    }
}

// MGS projections from the dots d.Ad_j (solver.cpp:240-243, classical form
// on the cached cross terms)
__device__ __forceinline__ void fin_projections(SolverState* st, const double* dots) {
    const int nc = st->n_cache, R = st->ring;
    int slot[kMaxOrtho];
    for (int j = 0; j < nc && j < kMaxOrtho; ++j) slot[j] = (st->head - (nc - 1) + j + 2 * R) % R;
    for (int j = 0; j < nc && j < kMaxOrtho; ++j) {
        double num = dots[j];
        for (int i = 0; i < j; ++i) num -= st->p[i] * st->cross[slot[i]][slot[j]];
        st->p[j] = num / st->dAd[slot[j]];
    }
}

// IdentityPrecond (precond.cpp:7-10) in the device loop: d = r / ||r|| as
// psdo_solve forms it (scale_inplace(1/||r||), solver.cpp:230-233; d = r
// without normalize_before_precond), then the dots d.Ad_j and the MGS
// projections, like the network's last kernel. JAC: JacobiPrecond
// (precond.cpp:12-26), d = (r / ||r||) * (1 / A_ii).
template <int NO, bool JAC>
__global__ void __launch_bounds__(kBlock) k_ident_dir(Geom g, const uint8_t* __restrict__ cls,
                                                      const double* __restrict__ r, double* __restrict__ dout,
                                                      SolverState* st, const double* __restrict__ ADring,
                                                      double* __restrict__ partials, unsigned int* __restrict__ counter) {
    constexpr int NA = (NO > 0) ? NO : 1;
    if (st->dist && st->done) return;
    const bool scale = st->normalize != 0;
    const double inv = st->inv1;
    const int nc = st->n_cache, R = st->ring;
    const double* adp[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) adp[j] = ADring + (long long)((st->head - (nc - 1) + j + 2 * R) % R) * g.n;
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;
    FOR_OWNED(g, c) {
        const uint8_t b = cls[c];
        if (cls_type(b) != 0) continue;
        double dv = scale ? __dmul_rn(r[c], inv) : r[c];
        if (JAC) dv = __dmul_rn(dv, 1.0 / (double)cls_diag(b));
        dout[c] = dv;
#pragma unroll
        for (int j = 0; j < NO; ++j)
            if (j < nc) acc[j] += dv * __ldg(adp[j] + c);
    }
    double tot[NA];
    if (grid_reduce<NA>(acc, partials, counter, tot) && threadIdx.x == 0) {
        if (st->dist) {
            for (int j = 0; j < kMaxOrtho; ++j) st->part[j] = (j < nc && j < NO) ? tot[j] : 0.0;
        } else {
            fin_projections(st, tot);
        }
    }
}

// d at the mixed fluid cells i = start, start + stride, ... of the up list, with
// their dots d.Ad_j accumulated into acc (k_mixed_up0, and the mixed blocks
// of k_up_l0m)
template <int D, int NO, bool F>
__device__ __forceinline__ void mixed_up_cells(const Geom& g, const Geom& gc, const uint32_t* __restrict__ list,
                                               uint32_t n, const float* __restrict__ outc,
                                               const float* __restrict__ y0, float za, float zb,
                                               const float* __restrict__ tab, const uint32_t* __restrict__ kid,
                                               double* __restrict__ dout, double nrm, int nc,
                                               const double* const (&adp)[(NO > 0) ? NO : 1],
                                               double (&acc)[(NO > 0) ? NO : 1], long long start, long long stride) {
    constexpr int S = Sh<D>::S;
    for (long long i = start; i < n; i += stride) {
        const uint32_t c = list[i];
        const float* K = tab + (long long)__ldg(kid + i) * kRowW;
        int x, yy, z;
        decode32(g, c, x, yy, z);
        float w[S], k[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int dx = s % 3 - 1, dy = (s / 3) % 3 - 1, dz = (D == 3) ? s / 9 - 1 : 0;
            const int xx = x + dx, y2 = yy + dy, zz = z + dz;
            // upsample2: fine (xx, y2, zz) -> coarse (xx>>1, y2>>1, zz>>1); zero outside
            const bool in = xx >= 0 && xx < g.nx && y2 >= 0 && y2 < g.ny && zz >= 0 && zz < g.nz;
            w[s] = in ? __ldg(outc + lin(gc, xx >> 1, y2 >> 1, (D == 3) ? zz >> 1 : 0)) : 0.0f;
            k[s] = __ldg(K + s);
        }
        const float u = win_dot<F, S>([&](int t) { return k[t]; }, [&](int t) { return w[t]; });
        const float o = F ? __fmaf_rn(za, __ldg(y0 + c), __fmul_rn(zb, u))
                          : __fadd_rn(__fmul_rn(za, __ldg(y0 + c)), __fmul_rn(zb, u));
        const double dv = __dmul_rn((double)o, nrm);
        dout[c] = dv;
#pragma unroll
        for (int j = 0; j < NO; ++j)
            if (j < nc) acc[j] += dv * __ldg(adp[j] + c);
    }
}

template <int D, int NO, bool F>
#ifndef MIXUP_MINB
#define MIXUP_MINB 4  // register cap for 4 blocks/SM (measured 26 -> 24 us)
#endif
__global__ void __launch_bounds__(kBlock, MIXUP_MINB) k_mixed_up0(Geom g, Geom gc, const uint32_t* __restrict__ list,
                                                      const uint32_t* __restrict__ count,
                                                      const float* __restrict__ outc, const float* __restrict__ y0,
                                                      const float* __restrict__ zab, const float* __restrict__ tab,
                                                      const uint32_t* __restrict__ kid, double* __restrict__ dout, SolverState* st,
                                                      const double* __restrict__ ADring, double* __restrict__ partials,
                                                      unsigned int* __restrict__ counter) {
    constexpr int NA = (NO > 0) ? NO : 1;
    pdl_launch_wait();
    if (st->dist && st->done) return;
    const uint32_t n = *count;
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
    const long long stride = (long long)gridDim.x * blockDim.x;
    mixed_up_cells<D, NO, F>(g, gc, list, n, outc, y0, za, zb, tab, kid, dout, nrm, nc, adp, acc,
                             (long long)blockIdx.x * blockDim.x + threadIdx.x, stride);
    double tot[NA];
    if (grid_reduce<NA>(acc, partials, counter, tot) && threadIdx.x == 0) {
        // totals of the tiled kernel first, then this kernel's (fixed order)
        double dots[kMaxOrtho];
        for (int j = 0; j < nc && j < NO; ++j) dots[j] = st->dot_main[j] + tot[j];
        if (st->dist) {
            for (int j = 0; j < kMaxOrtho; ++j) st->part[j] = (j < nc && j < NO) ? dots[j] : 0.0;
        } else {
            fin_projections(st, dots);
        }
    }
}

}  // namespace nb2

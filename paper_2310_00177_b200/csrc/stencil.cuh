// Kernels for the two stencil phases of a PSDO iteration (solver.cpp:239-258):
// k_ortho2 (d' = MGS(d), A d', dots) and k_update2 (x' = x + alpha d',
// r = b - A x', ||r||^2).
//
// Asynchronous-copy pipeline. A 32 x 8 block owns a 64 x 8 x-y tile (each
// thread a pair of x-adjacent cells) and marches a z-chunk. Each thread
// copies, with cp.async (LDGSTS, no register staging), the inputs of its own
// pair and of its halo assignment for the plane PF steps ahead into a ring of
// shared-memory stages; a copy whose pair holds no fluid cell is issued with
// src-size 0, which zero-fills without touching DRAM (exact, by the zero
// invariant of the solver vectors). Every thread reads back only what it
// copied itself, so the input ring needs no barriers. The operand v (d' or
// x') is formed once per cell into a 4-plane shared ring with its halo; one
// barrier per step; the 7-point rows are then evaluated from shared memory in
// reduced-CSR column order with round-to-nearest ops, bit-identical to spmv
// (sparse.cpp:111-116) on assemble_poisson_3d + reduce.
#pragma once

#include "common.cuh"
#include "psdo.cuh"
#include "tma.cuh"

namespace nb2 {

constexpr int kSX = 32, kSY = 8;          // threads per block (x lanes, y rows)
constexpr int kTX = 2 * kSX, kTY = kSY;    // cells per block tile (64 x 8)
constexpr int kVW = kTX + 4, kVH = kTY + 2;  // staged plane: cols x0-2..x0+65, rows y0-1..y0+8
constexpr int kPF = 2;                     // planes prefetched ahead (down0.cuh)
#ifndef STENCIL_PF_ORTHO
#define STENCIL_PF_ORTHO 2
#endif
#ifndef STENCIL_PF_UPDATE
#define STENCIL_PF_UPDATE 2
#endif
constexpr int kST = kPF + 1;               // input ring stages
// rows of the ortho/update tile (64 x SY cells, 32 x SY threads). A taller
// tile reads fewer halo rows per cell (2/SY), but SY = 16 (one 512-thread
// block per SM, half the schedule columns) measured slower at C3 256^3:
// ortho 100 -> 107 us, update 76 -> 93 us. Kept as a compile-time knob.
#ifndef STENCIL_SY
#define STENCIL_SY 8
#endif
constexpr int kMarchSY = STENCIL_SY;
// ortho: r read into registers (no ring stages) and a 2-plane prefetch bring
// the block to 70 KB, and a register cap (79) to three blocks per SM instead
// of two: 100.7 -> 89.8 us at C3 256^3 (r only: 94.6 us; tools/runs/o3_ab.sh)
#ifndef STENCIL_ORTHO_CTR_DIRECT
#define STENCIL_ORTHO_CTR_DIRECT 1
#endif
#ifndef ORTHO_MINB
#define ORTHO_MINB 3
#endif
// UPDATE_MINB: optional register cap for update (unset: no block count in
// the bound, 64 registers; an explicit 1 gives 86 and two blocks per SM)
#ifdef UPDATE_MINB
#define UPDATE_BOUNDS __launch_bounds__(kSX* SY, SY == kSY ? UPDATE_MINB : 1)
#else
#define UPDATE_BOUNDS __launch_bounds__(kSX* SY)
#endif
#ifndef STENCIL_UPDATE_CTR_DIRECT
#define STENCIL_UPDATE_CTR_DIRECT 1
#endif
// TMA plane loads (stencil_march_tma) for the 3D ortho / update kernels: one
// thread issues a tensor copy of each input's tile plane (halo included,
// zeros outside the domain) into a ring of STENCIL_TMA_PF + 1 stages, all
// threads wait on the stage's mbarrier. Per kernel, the measured faster path
// (C3 256^3, tools/ab_tma.sh): update 75.0 -> 73.7 us with TMA; ortho 89.9 us
// with cp.async vs 94.4 us with TMA (its three inputs' whole boxes: the
// cp.async path skips air pairs, 7% less DRAM traffic). 0: the cp.async path.
#ifndef STENCIL_TMA_ORTHO
#define STENCIL_TMA_ORTHO 0
#endif
#ifndef STENCIL_TMA_UPDATE
#define STENCIL_TMA_UPDATE 1
#endif
#ifndef STENCIL_TMA_PF
#define STENCIL_TMA_PF 2
#endif
constexpr unsigned kOut2 = 0x0C0Cu;        // pair bytes outside the domain: type 3

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Row sum in the reduced-CSR column order; out-of-domain / non-fluid
// neighbours are exact zeros and `s + -0.0 == s`, so adding them is bitwise
// neutral (see psdo.cuh).
__device__ __forceinline__ double row_sum(double vzm, double vym, double vxm, int diag, double vc, double vxp, double vyp,
                                          double vzp) {
    double s = 0.0;
    s = __dadd_rn(s, -vzm);
    s = __dadd_rn(s, -vym);
    s = __dadd_rn(s, -vxm);
    if (diag > 0) s = __dadd_rn(s, __dmul_rn((double)diag, vc));
    s = __dadd_rn(s, -vxp);
    s = __dadd_rn(s, -vyp);
    s = __dadd_rn(s, -vzp);
    return s;
}

__device__ __forceinline__ bool fluid(unsigned b) { return ((b >> 2) & 3u) == 0u; }
__device__ __forceinline__ bool pair_live(unsigned b2) { return fluid(b2 & 0xffu) || fluid(b2 >> 8); }

// Ortho operand (NA = 1 + NO inputs): d' = d + (-p_1) d_1 + ... (axpy order).
template <int NO>
struct OrthoOp {
    static constexpr int NA = 1 + NO;  // d, d_1..d_NO
    static constexpr int NC = 1;       // r (centre only)
    static constexpr int PF = STENCIL_PF_ORTHO;  // planes prefetched ahead
    static constexpr int CS = STENCIL_ORTHO_CTR_DIRECT ? 0 : PF + 1;  // centre inputs staged in the ring
    static constexpr int TPF = STENCIL_TMA_PF;                        // TMA path: planes in flight ahead
    static constexpr bool TMA = STENCIL_TMA_ORTHO != 0;
    const double* in[NA];
    const CUtensorMap* tin[NA];  // TMA path: the inputs' tensor maps
    const double* ctr[NC];
    double mp[NO > 0 ? NO : 1];
    int nc;
    __device__ __forceinline__ double value(const double (&a)[NA]) const {
        double r = a[0];
#pragma unroll
        for (int j = 0; j < NO; ++j)
            if (j < nc) r = __dadd_rn(r, __dmul_rn(mp[j], a[1 + j]));
        return r;
    }
};
// Update operand: x' = x + alpha d'.
struct UpdateOp {
    static constexpr int NA = 2;  // x, d'
    static constexpr int NC = 1;  // b (centre only)
    static constexpr int PF = STENCIL_PF_UPDATE;
    // b read straight into registers, one step ahead of its use: without its
    // ring stages the block fits four per SM instead of three
    static constexpr int CS = STENCIL_UPDATE_CTR_DIRECT ? 0 : PF + 1;
    static constexpr int TPF = STENCIL_TMA_PF;
    static constexpr bool TMA = STENCIL_TMA_UPDATE != 0;
    const double* in[NA];
    const CUtensorMap* tin[NA];
    const double* ctr[NC];
    double alpha;
    __device__ __forceinline__ double value(const double (&a)[NA]) const {
        return __dadd_rn(a[0], __dmul_rn(alpha, a[1]));
    }
};

// Op::CS: stages of centre-only inputs in shared memory (0: none staged; the
// epilogue reads them from global memory into registers)
template <typename Op, int SY = kSY, bool Staged = (Op::CS > 0)>
struct MarchSmem {
    static constexpr int VH = SY + 2;
    double raw[Op::PF + 1][Op::NA][VH][kVW];  // operand inputs, tile + halo
    double ctr[Op::PF + 1][Op::NC > 0 ? Op::NC : 1][SY][kTX];  // centre-only inputs
    double v[4][VH][kVW];              // operand ring
};
template <typename Op, int SY>
struct MarchSmem<Op, SY, false> {
    static constexpr int VH = SY + 2;
    double raw[Op::PF + 1][Op::NA][VH][kVW];
    double v[4][VH][kVW];
};

// Epi(q, v2 own pair, s2 rows, pair bytes, own raw inputs [NA] x 2, centre [NC] x 2, acc)
template <int D, int NV, int SY = kSY, typename Op, typename Epi>
__device__ __forceinline__ void stencil_march(const Geom& g, const uint8_t* __restrict__ cls, const Op& op, int tx,
                                              int ty, int zc0, int zc1, double (&acc)[NV], Epi epi) {
    constexpr int PF = Op::PF, ST = PF + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int kTY = SY, kVH = SY + 2;
    static_assert(2 * SY <= 32, "column halos: one lane per row and side");
    MarchSmem<Op, SY>& S = *reinterpret_cast<MarchSmem<Op, SY>*>(smem_raw);
    __syncthreads();  // the previous segment's last reads of S are done
    const int lane = threadIdx.x, row = threadIdx.y;
    const int X0 = tx * kTX, Y0 = ty * kTY;
    const int x = X0 + 2 * lane, y = Y0 + row;
    const bool own = x < g.nx && y < g.ny;  // nx even: the pair is whole
    const long long nx = g.nx, plane = nx * g.ny;
    // halo assignment: rows 0/1 -> pair of row y0-1 / y0+8; row 2, lanes 0..15 -> column x0-1 / x0+64
    int hx = 0, hy = 0, hsr = 0, hsc = 0;
    int hkind = 0;  // 0 none, 1 pair, 2 single cell
    if (row == 0 || row == 1) {
        hkind = 1;
        hx = x;
        hy = (row == 0) ? Y0 - 1 : Y0 + kTY;
        hsr = (row == 0) ? 0 : kVH - 1;
        hsc = 2 + 2 * lane;
    } else if (row == 2 && lane < 2 * kTY) {
        hkind = 2;
        hx = (lane < kTY) ? X0 - 1 : X0 + kTX;
        hy = Y0 + (lane & (kTY - 1));
        hsr = 1 + (lane & (kTY - 1));
        hsc = (lane < kTY) ? 1 : kTX + 2;  // smem column c <-> global x0 - 2 + c
    }
    const bool h_in = hkind != 0 && hx >= 0 && hx < g.nx && hy >= 0 && hy < g.ny;
    const long long qo = (long long)(own ? y : 0) * nx + (own ? x : 0);
    const long long qh = h_in ? (long long)hy * nx + hx : 0;
    auto zin = [&](int z) { return z >= 0 && z < g.nz; };
    auto own_bytes = [&](int z) -> unsigned {
        return (own && zin(z)) ? (unsigned)__ldg(reinterpret_cast<const unsigned short*>(cls + z * plane + qo)) : kOut2;
    };
    auto slot = [&](int z) { return (int)((unsigned)(z - zc0 + 1 + ST * 1024) % (unsigned)ST); };
    // issue the copies of plane z (one commit group per plane, even if empty).
    // Own pairs without fluid are zero-filled (no traffic); halo cells are
    // always copied when in the domain: their non-fluid values are the exact
    // zeros of the solver vectors, so no byte test sits on the issue path.
    // the source address is in the grid whatever the predicate (qo / qh are 0
    // for a lane without a pair / halo cell): src-size 0 reads nothing
    auto issue = [&](int z, unsigned ob) {
        if (zin(z)) {
            const int s = slot(z);
            const bool ol = own && pair_live(ob);
            const long long qz = z * plane;
#pragma unroll
            for (int a = 0; a < Op::NA; ++a) {
                cp_async16(&S.raw[s][a][row + 1][2 + 2 * lane], op.in[a] + (qz + qo), ol);
                if (hkind == 1)
                    cp_async16(&S.raw[s][a][hsr][hsc], op.in[a] + (qz + qh), h_in);
                else if (hkind == 2)
                    cp_async8(&S.raw[s][a][hsr][hsc], op.in[a] + (qz + qh), h_in);
            }
            if constexpr (Op::CS > 0) {
#pragma unroll
                for (int a = 0; a < Op::NC; ++a) cp_async16(&S.ctr[s][a][row][2 * lane], op.ctr[a] + (qz + qo), ol);
            }
        }
        cp_commit();
    };
    // form v of plane z for my positions (own pair, halo) into v slot z & 3
    auto form = [&](int z) {
        const int s = slot(z), vs = (z + 1024) & 3;
        double a0[Op::NA], a1[Op::NA];
        if (zin(z)) {
#pragma unroll
            for (int a = 0; a < Op::NA; ++a) {
                a0[a] = S.raw[s][a][row + 1][2 + 2 * lane];
                a1[a] = S.raw[s][a][row + 1][3 + 2 * lane];
            }
            S.v[vs][row + 1][2 + 2 * lane] = op.value(a0);
            S.v[vs][row + 1][3 + 2 * lane] = op.value(a1);
            if (hkind != 0) {
#pragma unroll
                for (int a = 0; a < Op::NA; ++a) a0[a] = S.raw[s][a][hsr][hsc];
                S.v[vs][hsr][hsc] = op.value(a0);
                if (hkind == 1) {
#pragma unroll
                    for (int a = 0; a < Op::NA; ++a) a1[a] = S.raw[s][a][hsr][hsc + 1];
                    S.v[vs][hsr][hsc + 1] = op.value(a1);
                }
            }
        } else {
            S.v[vs][row + 1][2 + 2 * lane] = 0.0;
            S.v[vs][row + 1][3 + 2 * lane] = 0.0;
            if (hkind != 0) S.v[vs][hsr][hsc] = 0.0;
            if (hkind == 1) S.v[vs][hsr][hsc + 1] = 0.0;
        }
    };

    // prologue: bytes and copies of planes zc0-1 .. zc0+PF-1
    const int zlo = (D == 3) ? zc0 - 1 : zc0;
    unsigned ob[PF + 2];  // own bytes of planes z .. z+PF+1 (rotating)
    unsigned ob_m = own_bytes(zlo);
    issue(zlo, ob_m);
    if (D == 3) {
#pragma unroll
        for (int k = 0; k < PF + 2; ++k) ob[k] = own_bytes(zc0 + k);
#pragma unroll
        for (int k = 0; k < PF; ++k) issue(zc0 + k, ob[k]);
        cp_wait<PF - 1>();  // planes zc0-1, zc0 landed (own copies)
        form(zc0 - 1);
        form(zc0);
    } else {
        ob[0] = ob_m;
        cp_wait<0>();
        form(zc0);
    }
    // unrolled by the queue length: the rotation below becomes register
    // renaming instead of moves that would wait on the in-flight byte loads
#pragma unroll(PF + 2)
    for (int z = zc0; z < zc1; ++z) {
        constexpr int NCD = (Op::CS == 0 && Op::NC > 0) ? Op::NC : 0;
        double2 cdir[NCD > 0 ? NCD : 1];
        if constexpr (NCD > 0) {
            const bool l = own && pair_live(ob[0]);
#pragma unroll
            for (int a = 0; a < NCD; ++a)
                cdir[a] = l ? __ldg(reinterpret_cast<const double2*>(op.ctr[a] + z * plane + qo)) : make_double2(0.0, 0.0);
        }
        if (D == 3) {
            issue(z + PF, ob[PF]);  // the plane PF steps ahead
            cp_wait<PF - 1>();                 // plane z+1 landed
            form(z + 1);
        }
        __syncthreads();  // v of planes z-1, z, z+1 complete (halos included)
        const unsigned bc = ob[0];
        if (own && pair_live(bc)) {
            const int vm = (z + 1023) & 3, vc = (z + 1024) & 3, vp = (z + 1025) & 3;
            const int c0 = 2 + 2 * lane, r0 = row + 1;
            const double v0 = S.v[vc][r0][c0], v1 = S.v[vc][r0][c0 + 1];
            const double zm0 = (D == 3) ? S.v[vm][r0][c0] : 0.0, zm1 = (D == 3) ? S.v[vm][r0][c0 + 1] : 0.0;
            const double zp0 = (D == 3) ? S.v[vp][r0][c0] : 0.0, zp1 = (D == 3) ? S.v[vp][r0][c0 + 1] : 0.0;
            double2 s;
            s.x = fluid(bc & 0xffu) ? row_sum(zm0, S.v[vc][r0 - 1][c0], S.v[vc][r0][c0 - 1], cls_diag(bc & 0xffu), v0,
                                              v1, S.v[vc][r0 + 1][c0], zp0)
                                    : 0.0;
            s.y = fluid(bc >> 8) ? row_sum(zm1, S.v[vc][r0 - 1][c0 + 1], v0, cls_diag(bc >> 8), v1,
                                           S.v[vc][r0][c0 + 2], S.v[vc][r0 + 1][c0 + 1], zp1)
                                 : 0.0;
            const int sl = slot(z);
            double raw0[Op::NA], raw1[Op::NA], c0v[Op::NC > 0 ? Op::NC : 1] = {}, c1v[Op::NC > 0 ? Op::NC : 1] = {};
#pragma unroll
            for (int a = 0; a < Op::NA; ++a) {
                raw0[a] = S.raw[sl][a][r0][c0];
                raw1[a] = S.raw[sl][a][r0][c0 + 1];
            }
            if constexpr (Op::CS > 0) {
#pragma unroll
                for (int a = 0; a < Op::NC; ++a) {
                    c0v[a] = S.ctr[sl][a][row][2 * lane];
                    c1v[a] = S.ctr[sl][a][row][2 * lane + 1];
                }
            } else if constexpr (NCD > 0) {
#pragma unroll
                for (int a = 0; a < NCD; ++a) {
                    c0v[a] = cdir[a].x;
                    c1v[a] = cdir[a].y;
                }
            }
            epi(z * plane + qo, make_double2(v0, v1), s, bc, raw0, raw1, c0v, c1v, acc);
        }
        // rotate the byte queues
#pragma unroll
        for (int k = 0; k < PF + 1; ++k) ob[k] = ob[k + 1];
        if (D == 3) ob[PF + 1] = own_bytes(z + PF + 2);
    }
    cp_wait<0>();
}

// Shared memory of the TMA march: the input ring (each box a 128-byte aligned
// 68 x VH plane of doubles), the operand ring, one mbarrier per stage.
template <typename Op, int SY>
struct TmaSmem {
    static constexpr int VH = SY + 2;
    static constexpr int PLANE = VH * kVW;                               // doubles in a box
    static constexpr int PSTRIDE = ((PLANE * 8 + 127) / 128) * 128 / 8;  // box stride, 128-byte aligned
    static constexpr int ST = Op::TPF + 1;
    double raw[ST][Op::NA][PSTRIDE];
    double v[4][VH][kVW];
    uint64_t bar[ST];
};
template <typename Sm>
__device__ __forceinline__ Sm& tma_smem() {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned a = smem_u32(smem_raw);
    return *reinterpret_cast<Sm*>(smem_raw + (((a + 127u) & ~127u) - a));
}
template <typename Op, int SY>
__host__ __device__ constexpr size_t tma_smem_bytes() {
    return sizeof(TmaSmem<Op, SY>) + 128;
}
template <typename Op, int SY>
__device__ __forceinline__ void tma_march_init() {
    TmaSmem<Op, SY>& S = tma_smem<TmaSmem<Op, SY>>();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        for (int i = 0; i < TmaSmem<Op, SY>::ST; ++i) mbar_init(&S.bar[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
}

// stencil_march with the inputs' planes loaded by TMA (3D). A plane's stage
// is read only while its operand v is formed (the own cells' inputs the
// epilogue needs stay in registers from there), so the ring has TPF + 1
// stages: the plane issued at step z (z + TPF) reuses the stage of plane
// z - 1, formed before step z - 1's barrier. seq numbers the planes a block
// has issued (mbarrier phases), across segments. Same epilogue interface and
// arithmetic as stencil_march.
template <int NV, int SY, typename Op, typename Epi>
__device__ __forceinline__ void stencil_march_tma(const Geom& g, const uint8_t* __restrict__ cls, const Op& op, int tx,
                                                  int ty, int zc0, int zc1, double (&acc)[NV], unsigned& seq, Epi epi) {
    using Sm = TmaSmem<Op, SY>;
    constexpr int PF = Op::TPF, ST = Sm::ST;
    static_assert(PF >= 1, "the prologue forms planes zc0 - 1 and zc0");
    Sm& S = tma_smem<Sm>();
    __syncthreads();  // the previous segment's last reads of S are done
    constexpr int kTY = SY, kVH = SY + 2;
    const int lane = threadIdx.x, row = threadIdx.y;
    const bool leader = lane == 0 && row == 0;
    const int X0 = tx * kTX, Y0 = ty * kTY;
    const int x = X0 + 2 * lane, y = Y0 + row;
    const bool own = x < g.nx && y < g.ny;
    const long long nx = g.nx, plane = nx * g.ny;
    // the positions this thread forms: own pair; rows 0/1: the halo row pair
    // above / below; row 2, lanes 0..2SY-1: the halo column cells
    int hsr = 0, hsc = 0, hkind = 0;
    if (row == 0 || row == 1) {
        hkind = 1;
        hsr = (row == 0) ? 0 : kVH - 1;
        hsc = 2 + 2 * lane;
    } else if (row == 2 && lane < 2 * kTY) {
        hkind = 2;
        hsr = 1 + (lane & (kTY - 1));
        hsc = (lane < kTY) ? 1 : kTX + 2;
    }
    const long long qo = (long long)(own ? y : 0) * nx + (own ? x : 0);
    auto own_bytes = [&](int z) -> unsigned {
        return (own && z >= 0 && z < g.nz) ? (unsigned)__ldg(reinterpret_cast<const unsigned short*>(cls + z * plane + qo))
                                           : kOut2;
    };
    const unsigned q0 = seq;  // sequence number of plane zc0 - 1
    auto pseq = [&](int z) { return q0 + (unsigned)(z - (zc0 - 1)); };
    auto issue = [&](int z) {
        if (z > zc1 || !leader) return;  // the last input plane of the segment is zc1
        const unsigned k = pseq(z), st = k % ST;
        fence_proxy_async_smem();
        mbar_expect_tx(&S.bar[st], (unsigned)(Op::NA * Sm::PLANE * sizeof(double)));
#pragma unroll
        for (int a = 0; a < Op::NA; ++a) tma_load_3d(&S.raw[st][a][0], op.tin[a], X0 - 2, Y0 - 1, z, &S.bar[st]);
    };
    auto wait = [&](int z) {
        const unsigned k = pseq(z);
        mbar_wait(&S.bar[k % ST], (k / ST) & 1u);
    };
    auto rw = [&](int st, int a, int r, int c) -> double { return S.raw[st][a][r * kVW + c]; };
    // v of plane z at this thread's positions (zeros outside the domain came
    // with the box); the own pair's inputs stay in a0 / a1 for the epilogue
    auto form = [&](int z, double (&a0)[Op::NA], double (&a1)[Op::NA]) {
        const int st = (int)(pseq(z) % ST), vs = (z + 1024) & 3;
#pragma unroll
        for (int a = 0; a < Op::NA; ++a) {
            a0[a] = rw(st, a, row + 1, 2 + 2 * lane);
            a1[a] = rw(st, a, row + 1, 3 + 2 * lane);
        }
        S.v[vs][row + 1][2 + 2 * lane] = op.value(a0);
        S.v[vs][row + 1][3 + 2 * lane] = op.value(a1);
        if (hkind != 0) {
            double h0[Op::NA], h1[Op::NA];
#pragma unroll
            for (int a = 0; a < Op::NA; ++a) h0[a] = rw(st, a, hsr, hsc);
            S.v[vs][hsr][hsc] = op.value(h0);
            if (hkind == 1) {
#pragma unroll
                for (int a = 0; a < Op::NA; ++a) h1[a] = rw(st, a, hsr, hsc + 1);
                S.v[vs][hsr][hsc + 1] = op.value(h1);
            }
        }
    };
#pragma unroll
    for (int k = 0; k <= PF; ++k) issue(zc0 - 1 + k);
    unsigned ob[PF + 2];  // own bytes of planes z .. z+PF+1 (rotating)
#pragma unroll
    for (int k = 0; k < PF + 2; ++k) ob[k] = own_bytes(zc0 + k);
    double cur0[Op::NA], cur1[Op::NA];  // the own pair's inputs of plane z (from form)
    wait(zc0 - 1);
    form(zc0 - 1, cur0, cur1);
    wait(zc0);
    form(zc0, cur0, cur1);
    __syncthreads();  // every thread has formed plane zc0 - 1: its stage takes plane zc0 + PF next
    // centre-only inputs straight to registers, one plane ahead of their step
    constexpr int NCD = (Op::NC > 0) ? Op::NC : 0;
    auto cload = [&](int z, unsigned b2, double2 (&cd)[NCD > 0 ? NCD : 1]) {
        const bool l = own && z < zc1 && pair_live(b2);
#pragma unroll
        for (int a = 0; a < NCD; ++a)
            cd[a] = l ? __ldg(reinterpret_cast<const double2*>(op.ctr[a] + z * plane + qo)) : make_double2(0.0, 0.0);
    };
    double2 cnext[NCD > 0 ? NCD : 1];
    cload(zc0, ob[0], cnext);
#pragma unroll(PF + 2)
    for (int z = zc0; z < zc1; ++z) {
        double2 cdir[NCD > 0 ? NCD : 1];
#pragma unroll
        for (int a = 0; a < (NCD > 0 ? NCD : 1); ++a) cdir[a] = cnext[a];
        cload(z + 1, ob[1], cnext);
        issue(z + PF);
        double nxt0[Op::NA], nxt1[Op::NA];
        wait(z + 1);
        form(z + 1, nxt0, nxt1);
        __syncthreads();  // v of planes z-1, z, z+1 complete (halos included)
        const unsigned bc = ob[0];
        if (own && pair_live(bc)) {
            const int vm = (z + 1023) & 3, vc = (z + 1024) & 3, vp = (z + 1025) & 3;
            const int c0 = 2 + 2 * lane, r0 = row + 1;
            const double v0 = S.v[vc][r0][c0], v1 = S.v[vc][r0][c0 + 1];
            const double zm0 = S.v[vm][r0][c0], zm1 = S.v[vm][r0][c0 + 1];
            const double zp0 = S.v[vp][r0][c0], zp1 = S.v[vp][r0][c0 + 1];
            double2 sv;
            sv.x = fluid(bc & 0xffu) ? row_sum(zm0, S.v[vc][r0 - 1][c0], S.v[vc][r0][c0 - 1], cls_diag(bc & 0xffu), v0,
                                               v1, S.v[vc][r0 + 1][c0], zp0)
                                     : 0.0;
            sv.y = fluid(bc >> 8) ? row_sum(zm1, S.v[vc][r0 - 1][c0 + 1], v0, cls_diag(bc >> 8), v1,
                                            S.v[vc][r0][c0 + 2], S.v[vc][r0 + 1][c0 + 1], zp1)
                                  : 0.0;
            double c0v[Op::NC > 0 ? Op::NC : 1] = {}, c1v[Op::NC > 0 ? Op::NC : 1] = {};
            if constexpr (NCD > 0) {
#pragma unroll
                for (int a = 0; a < NCD; ++a) {
                    c0v[a] = cdir[a].x;
                    c1v[a] = cdir[a].y;
                }
            }
            epi(z * plane + qo, make_double2(v0, v1), sv, bc, cur0, cur1, c0v, c1v, acc);
        }
#pragma unroll
        for (int a = 0; a < Op::NA; ++a) {
            cur0[a] = nxt0[a];
            cur1[a] = nxt1[a];
        }
#pragma unroll
        for (int k = 0; k < PF + 1; ++k) ob[k] = ob[k + 1];
        ob[PF + 1] = own_bytes(z + PF + 2);
    }
    seq = pseq(zc1) + 1;  // planes zc0 - 1 .. zc1 were issued and waited on
}

// d'.Ad' and r.d' -> alpha, or a breakdown (solver.cpp:245-251); d_j.Ad' are
// the cross terms of the direction's future projections. tot = {d'Ad', r.d',
// d_1.Ad', ...}.
__device__ __forceinline__ void fin_ortho(SolverState* st, const double* tot) {
    const int nc = st->n_cache, R = st->ring;
    const int nw = (st->head + 1) % R;
    const double dAd = tot[0];
    st->dAd_new = dAd;
    st->rd_new = tot[1];
    for (int j = 0; j < nc && j < kMaxOrtho; ++j) {
        const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
        st->cross[slot][nw] = tot[2 + j];
    }
    if (!(dAd > 0.0) || fabs(dAd) < 1e-300) {
        st->breakdown = 1;
        st->done = 1;
        st->bad_value = dAd;
        st->alpha = 0.0;
    } else {
        st->alpha = tot[1] / dAd;
    }
}

// the 3D ortho / update kernels load their operand planes with TMA
template <int D, typename Op>
__host__ __device__ constexpr bool stencil_tma() {
    return D == 3 && Op::TMA;
}

// d' = MGS(d); Ad'; dots d'.Ad', r.d', d_j.Ad'. NO = n_ortho (cache bound).
template <int D, int NO, int SY>
__global__ void __launch_bounds__(kSX* SY, SY == kSY ? ORTHO_MINB : 1) k_ortho2(Geom g, const uint8_t* __restrict__ cls,
                                                     const double* __restrict__ dtmp, const double* __restrict__ r,
                                                     double* __restrict__ Dring, double* __restrict__ ADring,
                                                     SolverState* st, double* __restrict__ partials,
                                                     unsigned int* __restrict__ counter, Sched sc,
                                                     const __grid_constant__ TmaMaps maps) {
    using Op = OrthoOp<NO>;
    if constexpr (stencil_tma<D, Op>()) tma_march_init<Op, SY>();
    pdl_launch_wait();
    if (st->dist && st->done) return;
    precond_span_end(st);
    const int nc = st->n_cache, R = st->ring;
    const int nw = (st->head + 1) % R;
    Op op;
    op.in[0] = dtmp;
    op.tin[0] = &maps.m[kMapD];
    op.ctr[0] = r;
    op.nc = nc;
#pragma unroll
    for (int j = 0; j < NO; ++j) {
        const int slot = (st->head - (nc - 1) + j + 2 * R) % R;
        op.in[1 + j] = Dring + (long long)slot * g.n;
        op.tin[1 + j] = &maps.m[kMapRing + slot];
        op.mp[j] = (j < nc) ? -st->p[j] : 0.0;
    }
    double* dnew = Dring + (long long)nw * g.n;
    double* adnew = ADring + (long long)nw * g.n;
    constexpr int NV = 2 + (NO > 0 ? NO : 1);
    double acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = 0.0;
    auto epi = [&](long long q, double2 v, double2 s, unsigned bc, const double(&i0)[Op::NA], const double(&i1)[Op::NA],
                   const double(&c0)[1], const double(&c1)[1], double(&a)[NV]) {
        *reinterpret_cast<double2*>(dnew + q) = v;
        *reinterpret_cast<double2*>(adnew + q) = s;
        // non-fluid halves are exact zeros: their terms vanish
        a[0] += v.x * s.x;
        a[0] += v.y * s.y;
        a[1] += c0[0] * v.x;
        a[1] += c1[0] * v.y;
#pragma unroll
        for (int j = 0; j < NO; ++j)
            if (j < nc) {
                a[2 + j] += i0[1 + j] * s.x;
                a[2 + j] += i1[1 + j] * s.y;
            }
    };
    unsigned seq = 0;
    sched_for_each(sc, [&](int tx, int ty, int zc0, int zc1) {
        if constexpr (stencil_tma<D, Op>())
            stencil_march_tma<NV, SY>(g, cls, op, tx, ty, zc0, zc1, acc, seq, epi);
        else
            stencil_march<D, NV, SY>(g, cls, op, tx, ty, zc0, zc1, acc, epi);
    });
    double tot[NV];
    if (grid_reduce<NV, kSX * SY>(acc, partials, counter, tot)) {
        if (threadIdx.x == 0 && threadIdx.y == 0) {
            if (st->dist) {
                for (int j = 0; j < kPart; ++j) st->part[j] = (j < NV) ? tot[j] : 0.0;
            } else {
                fin_ortho(st, tot);
            }
        }
    }
}

// x' = x + alpha d'; r = b - A x'; ||r||^2 (solver.cpp:252-260).
template <int D, int SY>
__global__ void UPDATE_BOUNDS k_update2(Geom g, const uint8_t* __restrict__ cls,
                                                      const double* __restrict__ b, double* __restrict__ X0,
                                                      double* __restrict__ X1, const double* __restrict__ Dring,
                                                      double* __restrict__ r, SolverState* st, double* __restrict__ hist,
                                                      double* __restrict__ times, double* __restrict__ partials,
                                                      unsigned int* __restrict__ counter,
                                                      cudaGraphConditionalHandle cond, int use_cond, int do_norm,
                                                      Sched sc, const __grid_constant__ TmaMaps maps) {
    if constexpr (stencil_tma<D, UpdateOp>()) tma_march_init<UpdateOp, SY>();
    pdl_launch_wait();
    if (st->breakdown) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0)
            set_cond(cond, use_cond, 0u);
        return;
    }
    if (st->dist && st->done) return;
    const int nw = (st->head + 1) % st->ring;
    UpdateOp op;
    op.in[0] = st->xcur ? X1 : X0;
    op.in[1] = Dring + (long long)nw * g.n;
    op.tin[0] = &maps.m[st->xcur ? kMapX1 : kMapX0];
    op.tin[1] = &maps.m[kMapRing + nw];
    op.ctr[0] = b;
    op.alpha = st->alpha;
    double* xn = st->xcur ? X0 : X1;
    double acc[1] = {0.0};
    auto epi = [&](long long q, double2 v, double2 s, unsigned bc, const double(&)[2], const double(&)[2],
                   const double(&c0)[1], const double(&c1)[1], double(&a)[1]) {
        double2 rv;
        rv.x = fluid(bc & 0xffu) ? __dadd_rn(c0[0], -s.x) : 0.0;
        rv.y = fluid(bc >> 8) ? __dadd_rn(c1[0], -s.y) : 0.0;
        *reinterpret_cast<double2*>(xn + q) = v;
        *reinterpret_cast<double2*>(r + q) = rv;
        a[0] += rv.x * rv.x;
        a[0] += rv.y * rv.y;
    };
    unsigned seq = 0;
    sched_for_each(sc, [&](int tx, int ty, int zc0, int zc1) {
        if constexpr (stencil_tma<D, UpdateOp>())
            stencil_march_tma<1, SY>(g, cls, op, tx, ty, zc0, zc1, acc, seq, epi);
        else
            stencil_march<D, 1, SY>(g, cls, op, tx, ty, zc0, zc1, acc, epi);
    });
    if (!do_norm) return;
    double tot[1];
    if (grid_reduce<1, kSX * SY>(acc, partials, counter, tot) && threadIdx.x == 0 && threadIdx.y == 0) {
        if (st->dist)
            st->part[0] = tot[0];
        else
            finish_iteration(st, tot[0], hist, times, cond, use_cond, false);
    }
}

template <typename Op, int SY = kSY>
constexpr size_t march_smem_bytes() {
    return sizeof(MarchSmem<Op, SY>);
}
// tile rows for an ortho/update operand: kMarchSY while its stages fit the
// shared memory of one block, else kSY
template <typename Op>
constexpr int march_sy() {
    return march_smem_bytes<Op, kMarchSY>() <= 220 * 1024 ? kMarchSY : kSY;
}
// dynamic shared memory of an ortho / update launch
template <int D, typename Op, int SY>
constexpr size_t stencil_smem_bytes() {
    return stencil_tma<D, Op>() ? tma_smem_bytes<Op, SY>() : march_smem_bytes<Op, SY>();
}

}  // namespace nb2

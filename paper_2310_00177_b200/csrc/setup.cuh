// Per-frame setup kernels (npsd_b200_set_mask): the device replacement for
// NeuralPrecond's constructor work — ReductionMap::from_image
// (discretization.cpp:5-19), PaddedImage::from_image/pooled (net/kernels.hpp:37-56),
// build_kernels (net/kernels.hpp:121-144) and linear_image_sums + z
// (net/kernels.hpp:253-276, net/forward.hpp:76-86) — plus the stencil
// coefficients of assemble_poisson[_3d] (discretization.cpp:21-127).
//
// Kernels are NOT materialised for every cell (27 f32 per cell per conv would
// cost more HBM traffic than the rest of a PSDO iteration). A cell whose whole
// 3^D window is one pure cell type uses one of three per-level constant
// kernels; only "mixed" cells get a row in a compact SoA table
// tab[slot * cap + mixed_index].
#pragma once

#include <climits>

#include "common.cuh"

namespace nb2 {

// Device-side results of a set_mask that the host reads once, lazily
// (setup_sync in npsd_b200.cu): set_mask itself never waits on the device.
// Buffers sized from earlier frames may be too small for this one; the
// kernels then clamp their writes and raise a flag, and the host redoes the
// frame with grown capacities.
struct SetupInfo {
    uint32_t flags;                  // bit 2l: level l's hash table over half full; bit 2l+1: its rows over capacity
    uint32_t n_fluid;                // the reduced system size
    uint32_t n_mixed[kMaxDepth];     // mixed-window cells per level
    uint32_t npat[kMaxDepth];        // dictionary rows (window patterns) per level
    uint32_t unverified[kMaxDepth];  // levels >= 1: a window differs from its pattern's (per-cell rows)
};

// the frame's totals (scans' trailing entries) into SetupInfo, one launch
struct InfoSources {
    const uint32_t* n_fluid;
    const uint32_t* n_mixed[kMaxDepth];
    int depth;
};
__global__ void k_setup_info(InfoSources src, SetupInfo* info) {
    const int t = threadIdx.x;
    if (t == 0) info->n_fluid = *src.n_fluid;
    if (t < src.depth) info->n_mixed[t] = *src.n_mixed[t];
}


// L0: cell byte (window class, own type, stencil diagonal) plus 32-cell
// segment masks of mixed cells and of fluid cells.
template <int D>
__global__ void __launch_bounds__(kBlock) k_setup_l0(Geom g, const uint8_t* __restrict__ types,
                                                     uint8_t* __restrict__ cls, uint32_t* __restrict__ mmask,
                                                     uint32_t* __restrict__ mcount, uint32_t* __restrict__ fmask,
                                                     uint32_t* __restrict__ fcount) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long nround = (g.n + 31) & ~31LL;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nround; c += stride) {
        bool mixed = false, fluid = false;
        if (c < g.n) {
            const int x = (int)(c % g.nx);
            const int y = (int)((c / g.nx) % g.ny);
            const int z = (int)(c / ((long long)g.nx * g.ny));
            const int t = types[c];
            bool uniform = true, wfluid = false;
            const int zr = (D == 3) ? 1 : 0;
            for (int dz = -zr; dz <= zr; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int xx = x + dx, yy = y + dy, zz = z + dz;
                        const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
                        const int tt = in ? types[lin(g, xx, yy, zz)] : 2;
                        uniform &= (tt == t);
                        wfluid |= (tt == 0);
                    }
            // stencil diagonal: non-solid in-domain face neighbours (discretization.cpp:105-113)
            int diag = 0;
            const int nbx[6] = {0, 0, -1, 1, 0, 0}, nby[6] = {0, -1, 0, 0, 1, 0}, nbz[6] = {-1, 0, 0, 0, 0, 1};
            for (int k = 0; k < 6; ++k) {
                if (D == 2 && nbz[k] != 0) continue;
                const int xx = x + nbx[k], yy = y + nby[k], zz = z + nbz[k];
                const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
                if (in && types[lin(g, xx, yy, zz)] != 2) ++diag;
            }
            const int w = uniform ? t : 3;
            cls[c] = (uint8_t)(w | (t << 2) | (diag << 4) | ((int)wfluid << 7));
            // mixed / fluid masks count owned cells only (ghost planes are
            // the neighbours' or the outside of the domain)
            const bool owned = c >= owned_lo(g) && c < owned_hi(g);
            mixed = !uniform && owned;
            fluid = (t == 0) && owned;
        }
        const uint32_t mm = __ballot_sync(0xffffffffu, mixed);
        const uint32_t fm = __ballot_sync(0xffffffffu, fluid);
        if ((threadIdx.x & 31) == 0) {
            const long long seg = c >> 5;
            mmask[seg] = mm;
            mcount[seg] = __popc(mm);
            fmask[seg] = fm;
            fcount[seg] = __popc(fm);
        }
    }
}

// Window classes by z-march over a byte grid (3D, nx a multiple of 32): a
// 32 x 8 block owns a 32 x 8 tile and ZC planes. Each staged plane (tile +
// one-cell halo, outside the domain solid = 2) is reduced at once to per-cell
// 3 x 3 summaries (min, max, centre, non-solid face neighbours in the plane),
// which roll through registers along z: a window is uniform iff its min equals
// its max (types 0..2; a coarse cell that is not pure reads 3, which never
// equals a uniform window's type), and holds fluid iff its min is 0.
//   L0: src = the cell types. Writes the cell bytes (w | t << 2 | diag << 4 |
//       wfluid << 7), mixed and fluid segment masks, the tile flags (a staged
//       plane's "any fluid" is the tile dilated by one cell in x and y,
//       k_tile_flags' definition) and the linear-block window counts of every
//       level l < nzs (k_zsums, but counted from the L0 types: a level-l
//       cell's pooled value times 8^l is the count of its L0 cells of that
//       type, so the totals are the same integers).
//   coarse: src = pure-type bytes (k_pool_image). Writes cls = uniform ? t : 3
//       and the mixed masks (k_classify).
struct ZsumArgs {
    unsigned long long* G[kMaxDepth];  // per level: [3][27] counts (k_zsums layout)
    int nzs;                           // levels with window counts (depth - 1)
    int zg_off;                        // global plane of local plane 0 (level 0)
    int nxg, nyg, nzg;                 // the full grid (level 0)
};

// L0 also writes the solve's mixed sublist masks (mixed.cuh k_sub_masks):
// dmask = mixed windows holding fluid, umask = mixed fluid cells.
struct SubMasks {
    uint32_t *dmask, *dcount, *umask, *ucount;
};

template <int ZC, bool L0>
__global__ void __launch_bounds__(256) k_classify_march(Geom g, const uint8_t* __restrict__ src,
                                                        uint8_t* __restrict__ cls, uint32_t* __restrict__ mmask,
                                                        uint32_t* __restrict__ mcount, uint32_t* __restrict__ fmask,
                                                        uint32_t* __restrict__ fcount, int ftx, int fty,
                                                        uint8_t* __restrict__ tflags, ZsumArgs za, SubMasks sm) {
    static_assert(kFlagTX == 32 && kFlagTY == 8, "the block tile is the flag tile");
    __shared__ uint8_t st[2][10][36];
    __shared__ uint32_t sG[L0 ? kMaxDepth * 81 : 1];  // 32-bit block counts (64-bit shared atomics are CAS loops)
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
    const int X0 = blockIdx.x * 32, Y0 = blockIdx.y * 8, Z0 = blockIdx.z * ZC;
    const long long plane = (long long)g.nx * g.ny;
    if (L0) {
        for (int i = tid; i < za.nzs * 81; i += 256) sG[i] = 0u;
    }
    // staging: my (up to) two bytes of the 10 x 34 plane
    int off[2], sidx[2];
    bool inxy[2], use[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int i = tid + 256 * j, ly = i / 34, lx = i - 34 * ly;
        const int xx = X0 - 1 + lx, yy = Y0 - 1 + ly;
        use[j] = i < 340;
        inxy[j] = use[j] && (unsigned)xx < (unsigned)g.nx && (unsigned)yy < (unsigned)g.ny;
        off[j] = inxy[j] ? yy * g.nx + xx : 0;
        sidx[j] = ly * 36 + lx;
    }
    // per-plane summaries (min, max, centre, in-plane non-solid face
    // neighbours) of my cell's 3 x 3 for planes z - 1 (P), z (M), z + 1 (N),
    // rotated by value each step: a runtime loop, no unrolled copies of the body
    int mnP = 0, mxP = 0, cvP = 0, mnM = 0, mxM = 0, cvM = 0, nbM = 0, mnN = 0, mxN = 0, cvN = 0, nbN = 0;
    // my staging bytes of a plane, loaded one plane ahead of their store
    uint8_t pv[2];
    auto load_plane = [&](int p) {
        const bool zin = p >= 0 && p < g.nz;
        const uint8_t* sp = src + (zin ? (long long)p * plane : 0);
#pragma unroll
        for (int j = 0; j < 2; ++j) pv[j] = (zin && inxy[j]) ? __ldg(sp + off[j]) : (uint8_t)2;
    };
    load_plane(Z0 - 1);
    // stage plane p (its bytes are in pv) into buffer (p - Z0 + 1) & 1, issue the loads of
    // plane p + 1, and summarise plane p into N; returns "any fluid" of plane p
    auto plane_step = [&](int p) -> bool {
        const int buf = (p - Z0 + 1) & 1;
        uint8_t* dst = &st[buf][0][0];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            if (!use[j]) continue;
            dst[sidx[j]] = pv[j];
            any |= (pv[j] == 0);
        }
        load_plane(p + 1);
        const bool anyb = __syncthreads_or(any) != 0;
        int lo = 255, hi = 0, n4 = 0, ctr = 0;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const int v = st[buf][ty + dy][tx + dx];
                lo = min(lo, v);
                hi = max(hi, v);
                if (dy == 1 && dx == 1) ctr = v;
                if ((dy == 1) != (dx == 1)) n4 += (v != 2);
            }
        mnP = mnM, mxP = mxM, cvP = cvM;
        mnM = mnN, mxM = mxN, cvM = cvN, nbM = nbN;
        mnN = lo, mxN = hi, cvN = ctr, nbN = n4;
        return anyb;
    };
    auto flag = [&](int zz, bool any) {
        if (L0 && tid == 0) tflags[((long long)zz * fty + blockIdx.y) * ftx + blockIdx.x] = any ? 1 : 0;
    };
    __shared__ uint32_t zin_cnt[L0 ? 8 : 1][3];  // per warp: counts of warps interior at every level
    if (L0 && tx == 0)
        for (int i = 0; i < 3; ++i) zin_cnt[ty][i] = 0;
    const int x = X0 + tx, y = Y0 + ty;
    plane_step(Z0 - 1);
#pragma unroll 1
    for (int p = Z0; p <= Z0 + ZC; ++p) {
        if (p - 1 >= g.nz) break;  // block-uniform
        const bool anyp = plane_step(p);  // now P, M, N = planes p - 2, p - 1, p
        if (p < Z0 + ZC && p < g.nz) flag(p, anyp);
        const int z = p - 1;
        if (z < Z0) continue;
        if (y >= g.ny) continue;  // whole warp (rows)
        const int lo = min(mnP, min(mnM, mnN)), hi = max(mxP, max(mxM, mxN));
        const int t = cvM;
        const bool uniform = lo == hi && (L0 || t != 3);  // every window cell is the centre's pure type
        const long long c = (long long)z * plane + (long long)y * g.nx + x;
        const bool owned = c >= owned_lo(g) && c < owned_hi(g);
        const uint32_t mm = __ballot_sync(0xffffffffu, !uniform && owned);
        if (L0) {
            // stencil diagonal: non-solid in-domain face neighbours (discretization.cpp:105-113)
            const int diag = nbM + (cvP != 2) + (cvN != 2);
            const bool wfluid = lo == 0;
            cls[c] = (uint8_t)((uniform ? t : 3) | (t << 2) | (diag << 4) | ((int)wfluid << 7));
            const uint32_t fm = __ballot_sync(0xffffffffu, t == 0 && owned);
            const uint32_t dm = __ballot_sync(0xffffffffu, !uniform && owned && wfluid);
            const uint32_t um = __ballot_sync(0xffffffffu, !uniform && owned && t == 0);
            if (tx == 0) {
                const long long seg = c >> 5;
                mmask[seg] = mm;
                mcount[seg] = __popc(mm);
                fmask[seg] = fm;
                fcount[seg] = __popc(fm);
                sm.dmask[seg] = dm;
                sm.dcount[seg] = __popc(dm);
                sm.umask[seg] = um;
                sm.ucount[seg] = __popc(um);
            }
            // window counts of every level l < nzs: classes by the level's
            // global (x, y, z) position (k_zsums), warp-aggregated. A warp
            // interior at the coarsest counted level is interior at every
            // level (the boundary bands grow with l): one update for all.
            const uint32_t b0 = __ballot_sync(0xffffffffu, owned && t == 0);
            const uint32_t b1 = __ballot_sync(0xffffffffu, owned && t == 1);
            const uint32_t b2 = __ballot_sync(0xffffffffu, owned && t == 2);
            const int zg = z + za.zg_off, Lc = za.nzs - 1;
            const int x0c = X0 >> Lc, x1c = (X0 + 31) >> Lc, ycl = y >> Lc, zcl = zg >> Lc;
            const bool all_inner = x0c > 0 && x1c < (za.nxg >> Lc) - 1 && ycl > 0 && ycl < (za.nyg >> Lc) - 1 &&
                                   zcl > 0 && zcl < (za.nzg >> Lc) - 1;
            if (all_inner) {
                if (tx == 0) {
                    zin_cnt[ty][0] += __popc(b0);
                    zin_cnt[ty][1] += __popc(b1);
                    zin_cnt[ty][2] += __popc(b2);
                }
            } else {
#pragma unroll 1
                for (int l = 0; l < za.nzs; ++l) {
                    const int xl = x >> l, yl = y >> l, zl = zg >> l;
                    const int kx = (xl == 0) ? 0 : ((xl == (za.nxg >> l) - 1) ? 2 : 1);
                    const int ky = (yl == 0) ? 0 : ((yl == (za.nyg >> l) - 1) ? 2 : 1);
                    const int kz = (zl == 0) ? 0 : ((zl == (za.nzg >> l) - 1) ? 2 : 1);
#pragma unroll
                    for (int kv = 0; kv < 3; ++kv) {
                        const uint32_t mk = __ballot_sync(0xffffffffu, kx == kv);
                        if (tx == 0 && mk) {
                            const int cl = (kz * 3 + ky) * 3 + kv;
                            const uint32_t n0 = __popc(b0 & mk), n1 = __popc(b1 & mk), n2 = __popc(b2 & mk);
                            if (n0) atomicAdd(&sG[l * 81 + 0 * 27 + cl], n0);
                            if (n1) atomicAdd(&sG[l * 81 + 1 * 27 + cl], n1);
                            if (n2) atomicAdd(&sG[l * 81 + 2 * 27 + cl], n2);
                        }
                    }
                }
            }
        } else {
            cls[c] = (uint8_t)(uniform ? t : 3);
            if (tx == 0) {
                const long long seg = c >> 5;
                mmask[seg] = mm;
                mcount[seg] = __popc(mm);
            }
        }
    }
    if (L0) {
        if (tx == 0)  // the all-interior counts go to the interior class (13) of every level
            for (int i = 0; i < za.nzs * 3; ++i)
                if (zin_cnt[ty][i % 3]) atomicAdd(&sG[(i / 3) * 81 + (i % 3) * 27 + 13], zin_cnt[ty][i % 3]);
        __syncthreads();
        for (int i = tid; i < za.nzs * 81; i += 256)
            if (sG[i]) atomicAdd(&za.G[i / 81][i % 81], (unsigned long long)sG[i]);
    }
}

// ---------------------------------------------------------------------------
// Level-0 classification with byte SIMD (k_classify_simd): the outputs of
// k_classify_march<ZC, true>, bit for bit, four cells per thread. A thread
// owns a 32-bit word of cell types (x .. x+3) and marches z. Types are staged
// as one-hot byte codes 1 << t (1 fluid, 2 air, 4 solid; outside the domain
// solid), so a window's set of types is the plain 32-bit OR of its words: the
// 3 x 3 in-plane OR (rows, then the left / right neighbours by byte permutes
// of adjacent words), then across three planes. A window is uniform iff its
// OR equals the centre's code; it holds fluid iff bit 0 is set. (Byte min /
// max intrinsics are emulated on sm_100: ~6 instructions each.) A block is
// LX lanes x (256 / LX) rows: a tile of 4 LX x (256 / LX) cells (128 x 8 or
// 64 x 16), i.e. whole 32-cell mask segments (8 lanes) and whole 32 x 8 flag
// tiles.
__device__ __forceinline__ uint32_t type_code4(uint32_t v) {  // bytes t in 0..2 -> 1 << t
    return 0x01010101u + v + ((v >> 1) & 0x01010101u);
}
__device__ __forceinline__ uint32_t code_nonsolid4(uint32_t c) {  // per byte: code != 4
    return (c | (c >> 1)) & 0x01010101u;
}
__device__ __forceinline__ uint32_t nib4(uint32_t b) {  // bytes' bit 0 -> 4-bit mask (byte i -> bit i)
    return ((b & 0x01010101u) * 0x00204081u) >> 21 & 0xFu;
}

template <int LX, int ZC>
__global__ void __launch_bounds__(256) k_classify_simd(Geom g, const uint8_t* __restrict__ src,
                                                       uint8_t* __restrict__ cls, uint32_t* __restrict__ mmask,
                                                       uint32_t* __restrict__ mcount, uint32_t* __restrict__ fmask,
                                                       uint32_t* __restrict__ fcount, int ftx, int fty,
                                                       uint8_t* __restrict__ tflags, ZsumArgs za, SubMasks sm) {
    constexpr int H = 256 / LX, W = 4 * LX;       // tile rows, tile cells in x
    constexpr int SW = LX + 2, SH = H + 2;        // staged words per row (one halo word each side), rows
    constexpr int NFX = W / kFlagTX, NFY = H / kFlagTY;  // flag tiles of the block tile
    static_assert(W % kFlagTX == 0 && H % kFlagTY == 0, "whole flag tiles");
    __shared__ uint32_t st[2][SH][SW];
    // level 0's block counts: 32-bit (a block holds < 2^32 cells; 64-bit shared atomics are CAS loops)
    __shared__ uint32_t sG[81];
    __shared__ uint32_t sflag[NFX * NFY];
    __shared__ uint32_t sint[kMaxDepth][3];  // interior-class counts
    const int lane = threadIdx.x % LX, row = threadIdx.x / LX, tid = threadIdx.x;
    // the lanes of my tile row (a warp is one row at LX = 32, two at LX = 16)
    const unsigned rmask = (LX == 32) ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
    const int X0 = blockIdx.x * W, Y0 = blockIdx.y * H, Z0 = blockIdx.z * ZC;
    const long long plane = (long long)g.nx * g.ny;
    for (int i = tid; i < 81; i += 256) sG[i] = 0u;
    if (tid < kMaxDepth * 3) sint[tid / 3][tid % 3] = 0u;
    // staging: my (up to) two words of the SH x SW plane window
    int off[2], sidx[2];
    bool use[2], inxy[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int i = tid + 256 * j, ly = i / SW, lw = i - SW * ly;
        const int xx = X0 - 4 + 4 * lw, yy = Y0 - 1 + ly;
        use[j] = i < SH * SW;
        inxy[j] = use[j] && xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny;
        off[j] = inxy[j] ? yy * g.nx + xx : 0;
        sidx[j] = i;
    }
    uint32_t pv[2];
    auto load_plane = [&](int p) {
        const bool zin = p >= 0 && p < g.nz;
        const uint8_t* sp = src + (zin ? (long long)p * plane : 0);
#pragma unroll
        for (int j = 0; j < 2; ++j)
            pv[j] = (zin && inxy[j]) ? __ldg(reinterpret_cast<const uint32_t*>(sp + off[j])) : 0x02020202u;
    };
    // per plane: the 3 x 3 type set (OR of codes), the centre code, the in-plane non-solid face neighbours
    uint32_t orP = 0, cvP = 0, orM = 0, cvM = 0, nbM = 0, orN = 0, cvN = 0, nbN = 0;
    load_plane(Z0 - 1);
    // stage plane p, issue plane p + 1, summarise plane p into N; returns
    // (in sflag) the flag tiles of plane p holding fluid in their dilation
    auto plane_step = [&](int p) {
        const int buf = (p - Z0 + 1) & 1;
        uint32_t* dst = &st[buf][0][0];
#pragma unroll
        for (int j = 0; j < 2; ++j)
            if (use[j]) dst[sidx[j]] = type_code4(pv[j]);
        if (tid < NFX * NFY) sflag[tid] = 0u;
        load_plane(p + 1);
        __syncthreads();
        const uint32_t U0 = st[buf][row][lane], U1 = st[buf][row][lane + 1], U2 = st[buf][row][lane + 2];
        const uint32_t M0 = st[buf][row + 1][lane], M1 = st[buf][row + 1][lane + 1], M2 = st[buf][row + 1][lane + 2];
        const uint32_t D0 = st[buf][row + 2][lane], D1 = st[buf][row + 2][lane + 1], D2 = st[buf][row + 2][lane + 2];
        const uint32_t r0 = U0 | M0 | D0, r1 = U1 | M1 | D1, r2 = U2 | M2 | D2;
        // bytes x-1 .. x+2 and x+1 .. x+4 of a row: permutes of adjacent words
        const uint32_t orp = __byte_perm(r0, r1, 0x6543) | r1 | __byte_perm(r1, r2, 0x4321);
        const uint32_t n4 = code_nonsolid4(U1) + code_nonsolid4(D1) + code_nonsolid4(__byte_perm(M0, M1, 0x6543)) +
                            code_nonsolid4(__byte_perm(M1, M2, 0x4321));
        // flag tiles: a cell whose in-plane 3 x 3 holds fluid
        // (one atomic per 8-lane group, i.e. per 32-cell flag-tile row)
        const uint32_t fb = __ballot_sync(0xffffffffu, (orp & 0x01010101u) != 0u);
        if ((tid & 7) == 0 && ((fb >> (tid & 24)) & 0xffu))
            atomicOr(&sflag[(row / kFlagTY) * NFX + (4 * lane) / kFlagTX], 1u);
        orP = orM, cvP = cvM;
        orM = orN, cvM = cvN, nbM = nbN;
        orN = orp, cvN = M1, nbN = n4;
        __syncthreads();  // sflag complete; every read of this staging buffer done before its reuse
    };
    const int x = X0 + 4 * lane, y = Y0 + row;
    const int zoff = za.zg_off;
    uint32_t cnt_int[3] = {0u, 0u, 0u};  // this warp row's interior-class counts (lane 0)
    plane_step(Z0 - 1);
#pragma unroll 1
    for (int p = Z0; p <= Z0 + ZC; ++p) {
        if (p - 1 >= g.nz) break;  // block-uniform
        plane_step(p);  // now P, M, N = planes p - 2, p - 1, p
        if (p < Z0 + ZC && p < g.nz && tid < NFX * NFY)
            tflags[((long long)p * fty + blockIdx.y * NFY + tid / NFX) * ftx + blockIdx.x * NFX + tid % NFX] =
                sflag[tid] ? 1 : 0;
        const int z = p - 1;
        if (z < Z0) continue;
        if (y >= g.ny) continue;  // whole warp rows
        const long long c = (long long)z * plane + (long long)y * g.nx + x;
        const bool owned = z >= g.zo0 && z < g.zo1;
        const uint32_t wor = orP | orM | orN;                                      // the window's type set
        const uint32_t mixb = (((wor ^ cvM) + 0x7f7f7f7fu) & 0x80808080u) >> 7;    // 1 per non-uniform byte
        const uint32_t t = (cvM >> 1) & 0x03030303u;                               // the centre's type
        const uint32_t diag = nbM + code_nonsolid4(cvP) + code_nonsolid4(cvN);
        const uint32_t wf = wor & 0x01010101u;                                     // fluid in the window
        *reinterpret_cast<uint32_t*>(cls + c) = t | (mixb * 3u) | (t << 2) | (diag << 4) | (wf << 7);
        // masks of the 32-cell segment of 8 lanes
        const uint32_t mixed = owned ? mixb : 0u;
        const uint32_t t0 = owned ? (cvM & 0x01010101u) : 0u;
        const uint32_t t1 = owned ? ((cvM >> 1) & 0x01010101u) : 0u;
        const uint32_t t2 = owned ? ((cvM >> 2) & 0x01010101u) : 0u;
        const int sh = 4 * (lane & 7);
        uint32_t mm = nib4(mixed) << sh, fm = nib4(t0) << sh, dm = nib4(mixed & wf) << sh, um = nib4(mixed & t0) << sh;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            mm |= __shfl_xor_sync(rmask, mm, o);
            fm |= __shfl_xor_sync(rmask, fm, o);
            dm |= __shfl_xor_sync(rmask, dm, o);
            um |= __shfl_xor_sync(rmask, um, o);
        }
        if ((lane & 7) == 0) {
            const long long seg = c >> 5;
            mmask[seg] = mm;
            mcount[seg] = __popc(mm);
            fmask[seg] = fm;
            fcount[seg] = __popc(fm);
            sm.dmask[seg] = dm;
            sm.dcount[seg] = __popc(dm);
            sm.umask[seg] = um;
            sm.ucount[seg] = __popc(um);
        }
        // level 0's linear-block window counts (k_zsums: classes by global
        // position; za.nzs is 0 or 1 here, coarser levels count their pooled
        // images): interior-class cells in registers, the two x-end cells of a
        // row and the rows on the y / z faces in shared counters
        if (za.nzs == 0 || !owned) continue;
        const int zg = z + zoff;
        const int ky = (y == 0) ? 0 : ((y == za.nyg - 1) ? 2 : 1);
        const int kz = (zg == 0) ? 0 : ((zg == za.nzg - 1) ? 2 : 1);
        const bool xe0 = x == 0, xe3 = x + 3 == za.nxg - 1;
        if (ky == 1 && kz == 1) {
            const uint32_t im = 0x01010101u & ~(xe0 ? 0x01u : 0u) & ~(xe3 ? 0x01000000u : 0u);
            cnt_int[0] += __popc(nib4(t0 & im));
            cnt_int[1] += __popc(nib4(t1 & im));
            cnt_int[2] += __popc(nib4(t2 & im));
            if (xe0) atomicAdd(&sG[(t & 0xffu) * 27 + 12 + 0], 1u);
            if (xe3) atomicAdd(&sG[(t >> 24) * 27 + 12 + 2], 1u);
        } else {
            uint32_t cc[3][3] = {};  // [type][kx]
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int kx = (k == 0 && xe0) ? 0 : ((k == 3 && xe3) ? 2 : 1);
                const uint32_t tb = (t >> (8 * k)) & 0xffu;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) cc[a][b] += (tb == (uint32_t)a && kx == b) ? 1u : 0u;
            }
#pragma unroll
            for (int ty = 0; ty < 3; ++ty)
#pragma unroll
                for (int kx = 0; kx < 3; ++kx)
                    if (cc[ty][kx]) atomicAdd(&sG[ty * 27 + (kz * 3 + ky) * 3 + kx], cc[ty][kx]);
        }
    }
    // interior rows: the interior class (13) of every level
#pragma unroll
    for (int ty = 0; ty < 3; ++ty) {
        const uint32_t v = __reduce_add_sync(rmask, cnt_int[ty]);
        if (lane == 0 && v) atomicAdd(&sint[0][ty], v);
    }
    __syncthreads();
    if (tid < 3 && za.nzs) sG[tid * 27 + 13] += sint[0][tid];
    __syncthreads();
    for (int i = tid; i < za.nzs * 81; i += 256)
        if (sG[i]) atomicAdd(&za.G[0][i], (unsigned long long)sG[i]);
}

// Tile occupancy at L0: flags[(z * nty + ty) * ntx + tx] = any fluid cell in
// the 32 x 8 tile (tx, ty) of plane z dilated by one cell in x and y. Kernels
// OR the flags of their region (plus one plane each side in z) and skip
// fluid-free blocks: every input they would read there is exactly zero.
__global__ void __launch_bounds__(kBlock) k_tile_flags(Geom g, const uint8_t* __restrict__ types, int ntx, int nty,
                                                       uint8_t* __restrict__ flags) {
    const long long n = (long long)ntx * nty * g.nz;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int tx = (int)(i % ntx), ty = (int)((i / ntx) % nty), z = (int)(i / ((long long)ntx * nty));
        const int x0 = max(tx * kFlagTX - 1, 0), x1 = min(tx * kFlagTX + kFlagTX + 1, g.nx);
        const int y0 = max(ty * kFlagTY - 1, 0), y1 = min(ty * kFlagTY + kFlagTY + 1, g.ny);
        bool any = false;
        for (int y = y0; y < y1 && !any; ++y)
            for (int x = x0; x < x1; ++x)
                if (types[lin(g, x, y, z)] == 0) {
                    any = true;
                    break;
                }
        flags[i] = any ? 1 : 0;
    }
}

// Live plane range of each tile column (a column covers cw x ch flag tiles):
// first / last plane in [zo0 - zdil, zo1 + zdil) whose flags are set, or -1.
// One warp per column, planes lane-strided.
__global__ void __launch_bounds__(kBlock) k_col_range(const uint8_t* __restrict__ flags, int ftx, int fty, int nz,
                                                      int zo0, int zo1, int cw, int ch, int ntx, int nty, int zdil,
                                                      int* __restrict__ first, int* __restrict__ last) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= ntx * nty) return;
    const int fx0 = (t % ntx) * cw, fy0 = (t / ntx) * ch;  // x fastest (common.cuh Sched)
    const int fx1 = min(fx0 + cw, ftx), fy1 = min(fy0 + ch, fty);
    int lo = INT_MAX, hi = -1;
    for (int z = max(zo0 - zdil, 0) + lane; z < min(zo1 + zdil, nz); z += 32) {
        bool any = false;
        for (int fy = fy0; fy < fy1 && !any; ++fy)
            for (int fx = fx0; fx < fx1; ++fx) any |= flags[((long long)z * fty + fy) * ftx + fx] != 0;
        if (any) {
            lo = min(lo, z);
            hi = max(hi, z);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
        first[t] = (hi < 0) ? -1 : lo;
        last[t] = hi;
    }
}

// Schedule pieces: piece p = c * ncol + t is column t's live units within
// chunk c (units [c * hu, (c + 1) * hu); a unit = `unit` planes). Chunk-major
// order (build_sched uses a single chunk: chunked orders measured slower).
// Units are live within zdil planes of a set flag, and owned.
__global__ void __launch_bounds__(kBlock) k_sched_pieces(const int* __restrict__ first, const int* __restrict__ last,
                                                         int ncol, int nchunk, int hu, int zo0, int zo1, int unit,
                                                         int zdil, int* __restrict__ zlo, int* __restrict__ len) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= ncol * nchunk) return;
    const int t = p % ncol, c = p / ncol;
    zlo[p] = 0;
    len[p] = 0;
    if (first[t] < 0) return;
    const int lo = max(first[t] - zdil, zo0), hi = min(last[t] + zdil, zo1 - 1);
    if (lo > hi) return;
    const int u0 = max(lo / unit, c * hu), u1 = min(hi / unit, (c + 1) * hu - 1);
    if (u0 > u1) return;
    zlo[p] = u0;
    len[p] = u1 - u0 + 1;
}

__global__ void k_sched_prefix(const int* __restrict__ len, int n, int* __restrict__ pre) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int acc = 0;
    for (int t = 0; t < n; ++t) {
        pre[t] = acc;
        acc += len[t];
    }
    pre[n] = acc;
}

// PaddedImage::pooled (net/kernels.hpp:46-56), 3D order x-fastest then z+1
// plane; from the L0 one-hot types (src_types) or a pooled level (src_img).
template <int D>
__global__ void __launch_bounds__(kBlock) k_pool_image(Geom gf, Geom gc, const uint8_t* __restrict__ src_types,
                                                       const float* __restrict__ src_img, float* __restrict__ dst,
                                                       uint8_t* __restrict__ pure) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < gc.n; c += stride) {
        const int x = (int)(c % gc.nx);
        const int y = (int)((c / gc.nx) % gc.ny);
        const int z = (int)(c / ((long long)gc.nx * gc.ny));
        float vals[3];
        for (int ch = 0; ch < 3; ++ch) {
            float acc = 0.0f;
            bool first = true;
            for (int cz = 0; cz < Sh<D>::BZ; ++cz)
                for (int cy = 0; cy < 2; ++cy)
                    for (int cx = 0; cx < 2; ++cx) {
                        const long long f = lin(gf, 2 * x + cx, 2 * y + cy, (D == 3) ? 2 * z + cz : 0);
                        const float v = src_types ? ((src_types[f] == ch) ? 1.0f : 0.0f) : src_img[ch * gf.n + f];
                        acc = first ? v : __fadd_rn(acc, v);
                        first = false;
                    }
            const float v = __fmul_rn((D == 3) ? 0.125f : 0.25f, acc);
            dst[ch * gc.n + c] = v;
            vals[ch] = v;
        }
        if (pure) {  // k_classify's pure(): the one-hot type, else 3
            const float a = vals[0], b = vals[1], sd = vals[2];
            pure[c] = (a == 1.0f && b == 0.0f && sd == 0.0f)   ? 0
                      : (a == 0.0f && b == 1.0f && sd == 0.0f) ? 1
                      : (a == 0.0f && b == 0.0f && sd == 1.0f) ? 2
                                                                : 3;
        }
    }
}

// Window class of a pooled level: uniform iff every window cell (solid outside)
// is the same pure cell type.
template <int D>
__global__ void __launch_bounds__(kBlock) k_classify(Geom g, const float* __restrict__ img, uint8_t* __restrict__ cls,
                                                     uint32_t* __restrict__ mmask, uint32_t* __restrict__ mcount) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long nround = (g.n + 31) & ~31LL;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nround; c += stride) {
        bool mixed = false;
        if (c < g.n) {
            const int x = (int)(c % g.nx);
            const int y = (int)((c / g.nx) % g.ny);
            const int z = (int)(c / ((long long)g.nx * g.ny));
            auto pure = [&](long long q) -> int {
                const float a = img[q], b = img[g.n + q], s = img[2 * g.n + q];
                if (a == 1.0f && b == 0.0f && s == 0.0f) return 0;
                if (a == 0.0f && b == 1.0f && s == 0.0f) return 1;
                if (a == 0.0f && b == 0.0f && s == 1.0f) return 2;
                return 3;
            };
            const int t = pure(c);
            bool uniform = (t != 3);
            const int zr = (D == 3) ? 1 : 0;
            for (int dz = -zr; dz <= zr && uniform; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int xx = x + dx, yy = y + dy, zz = z + dz;
                        const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
                        uniform &= ((in ? pure(lin(g, xx, yy, zz)) : 2) == t);
                    }
            cls[c] = (uint8_t)(uniform ? t : 3);
            mixed = !uniform && c >= owned_lo(g) && c < owned_hi(g);
        }
        const uint32_t mm = __ballot_sync(0xffffffffu, mixed);
        if ((threadIdx.x & 31) == 0) {
            mmask[c >> 5] = mm;
            mcount[c >> 5] = __popc(mm);
        }
    }
}

// build_kernels (net/kernels.hpp:121-144) for a list of cells (the mixed
// cells of a coarse level, or one representative cell per window pattern at
// level 0): K[s] = B[s] + sum_c sum_window W[s,c,w] * I(c, x+w), order
// (c, dz, dy, dx); row i of `tab` (kRowW floats) for cells[i], i < *count.
// Rows come from the dictionary (cells = representatives, count = patterns)
// unless *unverified (coarse levels whose windows did not all match their
// pattern): then one row per mixed cell (cells_pc / count_pc). At most
// rows_cap rows are written; more raises flag_bit (the frame is redone).
template <int D>
__global__ void __launch_bounds__(kBlock) k_build_rows(Geom g, const uint8_t* __restrict__ src_types,
                                                       const float* __restrict__ img,
                                                       const uint32_t* __restrict__ cells_dict,
                                                       const uint32_t* __restrict__ count_dict,
                                                       const uint32_t* __restrict__ cells_pc,
                                                       const uint32_t* __restrict__ count_pc,
                                                       const uint32_t* __restrict__ unverified, uint32_t rows_cap,
                                                       uint32_t* __restrict__ flags, uint32_t flag_bit,
                                                       const float* __restrict__ W, const float* __restrict__ B,
                                                       float* __restrict__ tab, const float* __restrict__ W2,
                                                       const float* __restrict__ B2, float* __restrict__ tab2) {
    const bool pc = unverified && *unverified;
    const uint32_t* cells = pc ? cells_pc : cells_dict;
    const uint32_t* count = pc ? count_pc : count_dict;
    // one warp per row: lanes t < S stage the window (3 channels), then lane s
    // accumulates slot s in the reference order B[s] + sum_{ch, t} W[s,ch,t] I
    constexpr int S = Sh<D>::S;
    constexpr int NW = kBlock / 32;
    __shared__ float sW[2][S * 3 * S];  // the conv's weights; [1]: the optional second conv (W2)
    __shared__ float sB[2][S];
    __shared__ float win[NW][3][S];
    long long n = *count;
    if (n > rows_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, flag_bit);
        n = rows_cap;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if ((long long)blockIdx.x * NW >= n) return;  // grid sized for the capacity
    const int nconv = W2 ? 2 : 1;
    for (int i = threadIdx.x; i < S * 3 * S; i += blockDim.x) {
        sW[0][i] = W[i];
        if (W2) sW[1][i] = W2[i];
    }
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        sB[0][i] = B[i];
        if (B2) sB[1][i] = B2[i];
    }
    __syncthreads();
    for (long long ii = (long long)blockIdx.x * NW + wid; ii < n; ii += (long long)gridDim.x * NW) {
        const long long c = cells[ii];
        const int x = (int)(c % g.nx);
        const int y = (int)((c / g.nx) % g.ny);
        const int z = (int)(c / ((long long)g.nx * g.ny));
        if (lane < S) {
            const int t = lane;
            const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = (D == 3) ? t / 9 - 1 : 0;
            const int xx = x + dx, yy = y + dy, zz = z + dz;
            const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
            float w0 = 0.0f, w1 = 0.0f, w2 = 1.0f;  // outside: the solid ring
            if (in) {
                const long long q = lin(g, xx, yy, zz);
                if (src_types) {
                    const int tt = src_types[q];
                    w0 = (tt == 0) ? 1.0f : 0.0f;
                    w1 = (tt == 1) ? 1.0f : 0.0f;
                    w2 = (tt == 2) ? 1.0f : 0.0f;
                } else {
                    w0 = img[q];
                    w1 = img[g.n + q];
                    w2 = img[2 * g.n + q];
                }
            }
            win[wid][0][t] = w0;
            win[wid][1][t] = w1;
            win[wid][2][t] = w2;
        }
        __syncwarp();
        if (lane < S) {
            const int sl = lane;
            for (int v = 0; v < nconv; ++v) {
                float acc = sB[v][sl];
                const float* w = sW[v] + sl * 3 * S;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch)
#pragma unroll
                    for (int t = 0; t < S; ++t) acc = __fadd_rn(acc, __fmul_rn(w[ch * S + t], win[wid][ch][t]));
                (v ? tab2 : tab)[ii * kRowW + sl] = acc;
            }
        }
        __syncwarp();
    }
}

// ---- level-0 window-pattern dictionary -----------------------------------
// At level 0 a mixed cell's kernel depends only on the cell types of its
// window (3^D two-bit codes, exact 54-bit key in 3D), and few patterns exist
// (C3 256^3: 926k mixed cells, 3,064 patterns). Keys are sorted, runs get a
// pattern id, one representative cell per pattern gets a kernel row.
template <int D>
__global__ void __launch_bounds__(kBlock) k_window_keys(Geom g, const uint8_t* __restrict__ types,
                                                        const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ count,
                                                        unsigned long long* __restrict__ keys,
                                                        uint32_t* __restrict__ vals) {
    const long long n = *count;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long c = list[i];
        const int x = (int)(c % g.nx), y = (int)((c / g.nx) % g.ny), z = (int)(c / ((long long)g.nx * g.ny));
        unsigned long long key = 0;
#pragma unroll
        for (int t = 0; t < Sh<D>::S; ++t) {
            const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = (D == 3) ? t / 9 - 1 : 0;
            const int xx = x + dx, yy = y + dy, zz = z + dz;
            const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
            const unsigned long long tt = in ? types[lin(g, xx, yy, zz)] : 2ull;
            key |= tt << (2 * t);
        }
        keys[i] = key;
        vals[i] = (uint32_t)i;
    }
}

// Coarse levels: the pooled window of a mixed cell (3 channels x 3^D cells,
// the solid ring outside) keyed by a 64-bit hash for the pattern dictionary.
// A hash is not exact, so k_verify_windows compares every cell's window with
// its pattern's representative bit for bit; set_mask drops the dictionary
// (per-cell rows) on any mismatch.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

template <int D>
__device__ __forceinline__ uint32_t window_bits(const Geom& g, const float* __restrict__ img, int x, int y, int z,
                                                int t, int ch) {
    const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = (D == 3) ? t / 9 - 1 : 0;
    const int xx = x + dx, yy = y + dy, zz = z + dz;
    const bool in = xx >= 0 && xx < g.nx && yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz;
    const float v = in ? img[(long long)ch * g.n + lin(g, xx, yy, zz)] : (ch == 2 ? 1.0f : 0.0f);
    return __float_as_uint(v);
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_window_hash(Geom g, const float* __restrict__ img,
                                                        const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ count,
                                                        unsigned long long* __restrict__ keys,
                                                        uint32_t* __restrict__ vals) {
    const long long n = *count;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long c = list[i];
        const int x = (int)(c % g.nx), y = (int)((c / g.nx) % g.ny), z = (int)(c / ((long long)g.nx * g.ny));
        // multiply-xor over the 81 values (FNV-1a order), one avalanche at the
        // end: collisions only cost the dictionary (k_verify_windows)
        unsigned long long h = 0xcbf29ce484222325ull;
#pragma unroll 3
        for (int t = 0; t < Sh<D>::S; ++t)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) h = (h ^ window_bits<D>(g, img, x, y, z, t, ch)) * 0x100000001b3ull;
        keys[i] = mix64(h);
        vals[i] = (uint32_t)i;
    }
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_verify_windows(Geom g, const float* __restrict__ img,
                                                           const uint32_t* __restrict__ list,
                                                           const uint32_t* __restrict__ count,
                                                           const uint32_t* __restrict__ pid,
                                                           const uint32_t* __restrict__ repcell,
                                                           uint32_t* __restrict__ mismatch) {
    const long long n = *count;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const long long c = list[i], r = repcell[pid[i]];
        if (c == r) continue;
        const int x = (int)(c % g.nx), y = (int)((c / g.nx) % g.ny), z = (int)(c / ((long long)g.nx * g.ny));
        const int rx = (int)(r % g.nx), ry = (int)((r / g.nx) % g.ny), rz = (int)(r / ((long long)g.nx * g.ny));
        bool same = true;
        for (int t = 0; t < Sh<D>::S; ++t)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
                same &= window_bits<D>(g, img, x, y, z, t, ch) == window_bits<D>(g, img, rx, ry, rz, t, ch);
        if (!same) atomicOr(mismatch, 1u);
    }
}

// Pattern ids by hashing: keys go into an open-addressing table (linear probing); the thread that inserts a
// key gives it the next id and makes its cell the representative. Ids come out
// in a nondeterministic order, but a pattern's row depends only on the
// pattern (level 0: the exact key; coarse levels: every member's window is
// compared with its representative's bit for bit), so the kernels' outputs
// are the same bits whichever order or representative wins.
constexpr unsigned long long kEmptyKey = ~0ull;

__global__ void __launch_bounds__(kBlock) k_dedup_insert(const unsigned long long* __restrict__ keys,
                                                         const uint32_t* __restrict__ count,
                                                         const uint32_t* __restrict__ list,
                                                         unsigned long long* __restrict__ tk, uint32_t* __restrict__ tv,
                                                         unsigned long long mask, uint32_t* __restrict__ slot,
                                                         uint32_t* __restrict__ repcell, uint32_t* __restrict__ npat,
                                                         uint32_t* __restrict__ flags, uint32_t flag_bit) {
    const long long n = *count;
    // more than half full: probing could run long (or forever when full);
    // skip, flag, and let the host redo the frame with a larger table
    if (2 * (unsigned long long)n > mask + 1) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, flag_bit);
        return;
    }
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long k = keys[i];
        if (k == kEmptyKey) k = kEmptyKey - 1;  // a coarse hash; collisions are caught by k_verify_windows
        // neighbouring cells often share a window: one probe per distinct key of the warp
        const unsigned peers = __match_any_sync(__activemask(), k);
        const int leader = __ffs(peers) - 1;
        unsigned long long h = 0;
        if ((int)(threadIdx.x & 31) == leader) {
            h = mix64(k) & mask;
            while (true) {
                unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(tk + h);
                if (cur == kEmptyKey) cur = atomicCAS(tk + h, kEmptyKey, k);
                if (cur == kEmptyKey) {  // inserted: new pattern
                    const uint32_t id = atomicAdd(npat, 1u);
                    tv[h] = id;
                    repcell[id] = list[i];
                    break;
                }
                if (cur == k) break;
                h = (h + 1) & mask;
            }
        }
        slot[i] = (uint32_t)__shfl_sync(peers, (unsigned)h, leader);
    }
}

// pid[i] = the pattern of key i, clamped below the row capacity (an
// overflowing frame is redone; until then every row index stays in bounds)
__global__ void __launch_bounds__(kBlock) k_dedup_ids(const uint32_t* __restrict__ slot,
                                                      const uint32_t* __restrict__ count,
                                                      const uint32_t* __restrict__ tv, unsigned long long mask,
                                                      uint32_t rows_cap, uint32_t* __restrict__ pid) {
    const long long n = *count;
    const bool skipped = 2 * (unsigned long long)n > mask + 1;  // k_dedup_insert did not run
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t p = skipped ? 0u : tv[slot[i]];
        pid[i] = p < rows_cap ? p : 0u;
    }
}

// The three uniform-window kernels of a conv (same arithmetic as
// build_kernels on a pure window: I = 1 on channel T, 0 elsewhere).
template <int D>
__global__ void k_kconst(const float* __restrict__ W, const float* __restrict__ B, float* __restrict__ out) {
    constexpr int S = Sh<D>::S;
    const int i = threadIdx.x;
    if (i >= 3 * S) return;
    const int T = i / S, s = i % S;
    float acc = B[s];
    for (int ch = 0; ch < 3; ++ch)
        for (int t = 0; t < S; ++t) acc = __fadd_rn(acc, __fmul_rn(W[(s * 3 + ch) * S + t], (ch == T) ? 1.0f : 0.0f));
    out[T * S + s] = acc;
}

// Exact window-sum ingredients for linear_image_sums: per-channel integer
// counts (value * scale, scale = 2^(D*level)) accumulated per boundary class
// (per axis: first plane, interior, last plane) over the owned cells; a z-slab
// classifies by global plane (zg_off: global index of local plane 0, nzg: the
// level's global plane count) so the ranks' counts add up to the full grid's.
// k_zsums by rows (the launcher's default): a row's y / z class is
// block-uniform and no 64-bit division sits in the per-cell path.
template <int D>
__global__ void __launch_bounds__(kBlock) k_zsums_rows(Geom g, const uint8_t* __restrict__ src_types,
                                                       const float* __restrict__ img, float scale, int zg_off, int nzg,
                                                       unsigned long long* __restrict__ G) {
    constexpr int NC = (D == 3) ? 27 : 9;
    constexpr int kInterior = (D == 3) ? 13 : 4;
    __shared__ unsigned long long sG[3 * NC];
    for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x) sG[i] = 0ull;
    __syncthreads();
    // a warp per row: its y / z class is warp-uniform; the row's two end
    // cells (x classes 0 and 2) go to shared atomics, the rest is summed in
    // registers (interior rows) or reduced per warp at the end of the row
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    unsigned long long inner[3] = {0ull, 0ull, 0ull};
    const long long nrows = (long long)g.ny * (g.zo1 - g.zo0);
    for (long long row = (long long)blockIdx.x * wpb + (threadIdx.x >> 5); row < nrows;
         row += (long long)gridDim.x * wpb) {
        const int y = (int)(row % g.ny), zl = g.zo0 + (int)(row / g.ny), z = zl + zg_off;  // global plane
        const int ky = (y == 0) ? 0 : ((y == g.ny - 1) ? 2 : 1);
        const int kz = (D == 3) ? ((z == 0) ? 0 : ((z == nzg - 1) ? 2 : 1)) : 0;
        const int cl1 = (kz * 3 + ky) * 3 + 1;
        const long long base = ((long long)zl * g.ny + y) * g.nx;
        unsigned long long racc[3] = {0ull, 0ull, 0ull};
        for (int x = lane; x < g.nx; x += 32) {
            const long long c = base + x;
            const bool xend = x == 0 || x == g.nx - 1;
            const uint8_t t = src_types ? src_types[c] : (uint8_t)0;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const unsigned long long v = src_types ? ((t == ch) ? 1ull : 0ull)
                                                       : (unsigned long long)__fmul_rn(img[ch * g.n + c], scale);
                if (!xend)
                    racc[ch] += v;
                else if (v)
                    atomicAdd(&sG[ch * NC + cl1 - 1 + ((x == 0) ? 0 : 2)], v);
            }
        }
        if (cl1 == kInterior) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) inner[ch] += racc[ch];
        } else {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                unsigned long long v = racc[ch];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && v) atomicAdd(&sG[ch * NC + cl1], v);
            }
        }
    }
    for (int ch = 0; ch < 3; ++ch) {
        unsigned long long v = inner[ch];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&sG[ch * NC + kInterior], v);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x)
        if (sG[i]) atomicAdd(&G[i], sG[i]);
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_zsums(Geom g, const uint8_t* __restrict__ src_types,
                                                  const float* __restrict__ img, float scale, int zg_off, int nzg,
                                                  unsigned long long* __restrict__ G) {
    constexpr int NC = (D == 3) ? 27 : 9;
    __shared__ unsigned long long sG[3 * NC];
    for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x) sG[i] = 0ull;
    __syncthreads();
    // interior cells (the all-interior class, nearly every cell) are counted
    // in registers and reduced per warp; boundary cells go to shared atomics
    constexpr int kInterior = (D == 3) ? 13 : 4;
    unsigned long long inner[3] = {0ull, 0ull, 0ull};
    FOR_OWNED(g, c) {
        const int x = (int)(c % g.nx);
        const int y = (int)((c / g.nx) % g.ny);
        const int z = (int)(c / ((long long)g.nx * g.ny)) + zg_off;  // global plane
        const int kx = (x == 0) ? 0 : ((x == g.nx - 1) ? 2 : 1);
        const int ky = (y == 0) ? 0 : ((y == g.ny - 1) ? 2 : 1);
        const int kz = (D == 3) ? ((z == 0) ? 0 : ((z == nzg - 1) ? 2 : 1)) : 0;
        const int cl = (kz * 3 + ky) * 3 + kx;
        for (int ch = 0; ch < 3; ++ch) {
            unsigned long long v;
            if (src_types)
                v = (src_types[c] == ch) ? 1ull : 0ull;
            else
                v = (unsigned long long)__fmul_rn(img[ch * g.n + c], scale);
            if (cl == kInterior)
                inner[ch] += v;
            else if (v)
                atomicAdd(&sG[ch * NC + cl], v);
        }
    }
    for (int ch = 0; ch < 3; ++ch) {
        unsigned long long v = inner[ch];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sG[ch * NC + kInterior], v);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x)
        if (sG[i]) atomicAdd(&G[i], sG[i]);
}

// z_a / z_b of one level (net/forward.hpp:78-86) from the class counts.
// F[c,w] = sum of I_pad(c, p + w) over interior p, exact in f64, then f32.
// every level's linear-block coefficients in one launch: block l = level l
struct ZfinLevel {
    Geom g;                          // the level's full grid
    const unsigned long long* G;     // window-class counts
    double scale;                    // 8^l (4^l in 2D)
    const float *KA, *KB;            // lin_a / lin_b kernels
    float biasA, biasB;
    float *za, *zb;
};
struct ZfinArgs {
    ZfinLevel lv[kMaxDepth];
};

template <int D>
__global__ void k_zfinal(const __grid_constant__ ZfinArgs a) {
    constexpr int S = Sh<D>::S;
    constexpr int NC = (D == 3) ? 27 : 9;
    const ZfinLevel& L = a.lv[blockIdx.x];
    const Geom g = L.g;
    const double scale = L.scale;
    __shared__ unsigned long long sG[3 * NC];
    __shared__ float F[3 * S], sKA[3 * S], sKB[3 * S];
    for (int i = threadIdx.x; i < 3 * NC; i += blockDim.x) sG[i] = L.G[i];
    for (int i = threadIdx.x; i < 3 * S; i += blockDim.x) {
        sKA[i] = L.KA[i];
        sKB[i] = L.KB[i];
    }
    __syncthreads();
    // one thread per (channel, tap): F = the exact count of the shifted box
    for (int i = threadIdx.x; i < 3 * S; i += blockDim.x) {
        const int ch = i / S, t = i % S;
        const int d[3] = {t % 3 - 1, (t / 3) % 3 - 1, (D == 3) ? t / 9 - 1 : 0};
        unsigned long long cnt = 0;
        for (int cl = 0; cl < NC; ++cl) {
            const int k[3] = {cl % 3, (cl / 3) % 3, cl / 9};
            bool ok = true;
            for (int a = 0; a < D; ++a) {
                if (d[a] == 1 && k[a] == 0) ok = false;   // q_a = p_a + 1 never hits plane 0
                if (d[a] == -1 && k[a] == 2) ok = false;  // q_a = p_a - 1 never hits plane n-1
            }
            if (ok) cnt += sG[ch * NC + cl];
        }
        double f = (double)cnt / scale;
        if (ch == 2) {
            // ring (solid) cells inside the shifted box
            const long long dims[3] = {g.nx, g.ny, g.nz};
            long long inside = 1;
            for (int a = 0; a < 3; ++a) inside *= dims[a] - ((a < D) ? (d[a] != 0 ? 1 : 0) : 0);
            f += (double)(g.n - inside);
        }
        F[i] = (float)f;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    // z = bias + sum_t (norm * K[t]) * F[t], serial in t (forward.hpp:78-86)
    const float norm = __fdiv_rn(1.0f, __fmul_rn((float)S, __ll2float_rn(g.n)));
    float za = L.biasA, zb = L.biasB;
    for (int t = 0; t < 3 * S; ++t) {
        za = __fadd_rn(za, __fmul_rn(__fmul_rn(norm, sKA[t]), F[t]));
        zb = __fadd_rn(zb, __fmul_rn(__fmul_rn(norm, sKB[t]), F[t]));
    }
    *L.za = za;
    *L.zb = zb;
}

}  // namespace nb2

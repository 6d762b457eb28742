// Shared device-side definitions for the B200 neural-preconditioned PSDO solve.
//
// Bitwise rule: every floating-point operation that the reference performs in
// its network (net/kernels.hpp, net/forward.hpp) and in its stencil
// (sparse.cpp:100-117) is issued here as an explicit round-to-nearest
// intrinsic (__fmul_rn/__fadd_rn, __dmul_rn/__dadd_rn) in the reference's
// order, so the compiler can never contract it into an FMA. The network and
// the operator are therefore bit-identical to the CPU restatement; only the
// tree-ordered dot products differ from the reference's serial loops.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nb2 {

constexpr int kMaxOrtho = 8;            // n_ortho supported on device
constexpr int kRing = kMaxOrtho + 1;    // cache slots + the direction being built
constexpr int kMaxDepth = 8;
constexpr int kBlock = 256;             // threads per block for all kernels

// Level geometry. nz == 1 for 2D.
// A level's local grid. nz counts every stored plane; [zo0, zo1) are the
// planes this context owns. Single-domain: zo0 = 0, zo1 = nz. A z-slab adds
// ghost planes on both sides (neighbour copies, or the outside of the domain
// at its faces): kernels read through them but compute, store and reduce
// over owned planes only.
struct Geom {
    int nx, ny, nz;
    long long n;
    int zo0, zo1;
};

__host__ __device__ inline Geom make_geom(int nx, int ny, int nz) {
    Geom g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.n = (long long)nx * ny * nz;
    g.zo0 = 0;
    g.zo1 = nz;
    return g;
}

__host__ __device__ inline long long owned_lo(const Geom& g) { return (long long)g.zo0 * g.nx * g.ny; }
__host__ __device__ inline long long owned_hi(const Geom& g) { return (long long)g.zo1 * g.nx * g.ny; }

// grid-stride loop over the owned cells of g
#define FOR_OWNED(g, c)                                                                    \
    for (long long c = owned_lo(g) + (long long)blockIdx.x * blockDim.x + threadIdx.x; \
         c < owned_hi(g); c += (long long)gridDim.x * blockDim.x)

__host__ __device__ __forceinline__ long long lin(const Geom& g, int x, int y, int z) {
    return ((long long)z * g.ny + y) * g.nx + x;
}

template <int D>
struct Sh {
    static constexpr int S = (D == 3) ? 27 : 9;  // slots (== window cells)
    static constexpr int BZ = (D == 3) ? 2 : 1;  // brick extent along z
    static constexpr int WZ = (D == 3) ? 4 : 1;  // 2-brick window planes along z
    static constexpr int CW = (D == 3) ? 3 : 1;  // coarse window planes along z
    static constexpr int NB = (D == 3) ? 6 : 4;  // stencil neighbours
};

// Window dot product sum_s k(s) * w(s) of the network's spatially varying
// convolution (apply_kernels, net/kernels.hpp:147-172), S = 27 (3D) or 9 slots.
// Exact (F = false): the reference's slot order, one rounded multiply and one
// rounded add per slot — bit-identical to the restatement. Fast (F = true):
// fused multiply-adds in one chain per window plane (three independent
// chains in 3D), then (a0 + a1) + a2 — within the north_star tolerance
// (1e-5 relative L2 of the preconditioner output), not bitwise.
template <bool F, int S, typename KF, typename WF>
__device__ __forceinline__ float win_dot(KF k, WF w) {
    if (!F) {
        float a = 0.0f;
#pragma unroll
        for (int s = 0; s < S; ++s) a = __fadd_rn(a, __fmul_rn(k(s), w(s)));
        return a;
    }
    constexpr int P = (S == 27) ? 3 : 1, L = S / P;
    float a[P];
#pragma unroll
    for (int p = 0; p < P; ++p) a[p] = 0.0f;
#pragma unroll
    for (int s = 0; s < S; ++s) a[s / L] = __fmaf_rn(k(s), w(s), a[s / L]);
    float t = a[0];
#pragma unroll
    for (int p = 1; p < P; ++p) t = __fadd_rn(t, a[p]);
    return t;
}

// L0 cell byte: bits 0-1 window class (0/1/2 = uniform fluid/air/solid window,
// 3 = mixed), bits 2-3 own cell type, bits 4-6 stencil diagonal (# non-solid
// in-domain face neighbours), bit 7 window holds a fluid cell. Coarse levels
// use bits 0-1 only.
__device__ __forceinline__ int cls_window(uint8_t b) { return b & 3; }
__device__ __forceinline__ int cls_type(uint8_t b) { return (b >> 2) & 3; }
__device__ __forceinline__ int cls_diag(uint8_t b) { return (b >> 4) & 7; }
// level 0 only: the 3^D window holds a fluid cell (else the solve's input is
// zero over it and y_0 = +0 exactly)
__device__ __forceinline__ bool cls_wfluid(uint8_t b) { return (b >> 7) != 0; }

// Mixed-cell table index from 32-cell segment masks and exclusive bases.
__device__ __forceinline__ long long mixed_index(const uint32_t* __restrict__ mmask,
                                                 const uint32_t* __restrict__ mbase, long long c) {
    const long long seg = c >> 5;
    const uint32_t bit = (uint32_t)(c & 31);
    return (long long)mbase[seg] + __popc(mmask[seg] & ((1u << bit) - 1u));
}

// Device-resident solver state (one per context). Written only by the last
// block of a reducing kernel; read by every later kernel.
constexpr int kPart = 2 + kMaxOrtho;  // doubles per reduction point (z-slab partials)

struct SolverState {
    // configuration (host-written before each solve)
    double tol_reduction, tol_abs;
    long long max_iters;
    int n_ortho, normalize, nullspace;
    int ring;  // n_ortho + 1
    // iteration
    long long k;      // iteration being computed (1-based)
    int n_cache;      // valid cached directions
    int head;         // ring slot of the newest cached direction
    int done, converged, breakdown;
    int xcur;         // which x buffer holds the current iterate
    double rnorm, thr;
    double inv1, inv2, nrm;         // network input scales / output multiplier
    double p[kMaxOrtho];            // MGS projections of the current direction
    double dot_main[kMaxOrtho];     // d.Ad_j over the tiled kernel's cells (mixed cells added later)
    double dAd[kRing];              // per ring slot: d'Ad
    double cross[kRing][kRing];     // cross[i][j] = d_i . A d_j (i older than j)
    double dAd_new, rd_new, alpha;  // for the direction being built
    double mean;                    // nullspace projection mean
    double rz, beta;                // pcg: r.z and the direction update's beta (cg.cuh)
    int pcur;                       // pcg: which p buffer holds the current direction
    double bad_value;               // curvature at breakdown
    unsigned long long t0;          // %globaltimer at solve start (k_stamp_start)
    unsigned long long t_mark;      // %globaltimer at the end of the last iteration (precond span start)
    double setup_s, precond_s;      // SolveReport setup_seconds / precond_seconds (solver.cpp:211,237)
    double part[kPart];             // z-slab: this rank's totals at a reduction point
    int dist;                       // z-slab: reductions stop at part[], k_finalize finishes them;
                                    // iteration kernels return at once when done (chunked loop)
};

// Programmatic dependent launch (the iteration kernels): wait for the
// previous kernel's completion and memory, then let the next kernel in the
// stream launch. At most one kernel runs ahead, so whatever a kernel reads
// before its wait must not be written by its immediate predecessor (anything
// older is complete). Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_launch_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The coarse-level kernels: what they read before this point comes from the
// frame's setup only (row codes, kernel rows, uniform kernels), so with the
// launch attribute it overlaps the previous kernel; then wait for it, and
// only then let the next kernel launch (at most one kernel runs ahead).
__device__ __forceinline__ void pdl_wait_then_trigger() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// Deterministic grid reduction: each block reduces NV doubles (fixed tree),
// writes them to partials[j * gridDim.x + block]; the last block to arrive sums
// the partials in block order and returns true with the totals in `tot`.
// Grid size is fixed per kernel and context, so results are run-to-run
// bitwise reproducible.
// ---------------------------------------------------------------------------
template <int NV, int NT = kBlock>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], double* __restrict__ partials,
                                            unsigned int* __restrict__ counter, double (&tot)[NV]) {
    __shared__ double sred[NT / 32][NV];  // NT >= threads per block
    __shared__ bool s_last;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    const int nwarp = nthr >> 5;
    const unsigned int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const unsigned int nblk = gridDim.x * gridDim.y * gridDim.z;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double a = v[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) sred[warp][j] = a;
    }
    __syncthreads();
    if (tid < NV) {
        double a = 0.0;
        for (int w = 0; w < nwarp; ++w) a += sred[w][tid];
        partials[(long long)tid * nblk + bid] = a;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned int ticket = atomicAdd(counter, 1u);
        s_last = (ticket == nblk - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    // last block: deterministic sum over blocks
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double a = 0.0;
        for (unsigned int b = tid; b < nblk; b += nthr) a += __ldcg(partials + (long long)j * nblk + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) sred[warp][j] = a;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double a = 0.0;
        for (int w = 0; w < nwarp; ++w) a += sred[w][j];
        tot[j] = a;
    }
    if (tid == 0) *counter = 0u;
    return true;
}

// L0 tile occupancy (k_tile_flags): 32 x 8 tiles per plane, dilated by one
// cell; flags == nullptr disables skipping (raw-network calls).
constexpr int kFlagTX = 32, kFlagTY = 8;
struct Occ {
    const uint8_t* flags;
    int ntx, nty;
};

// Block-wide: does the region [tx0, tx1) x [ty0, ty1) x [z0, z1] (flag tiles,
// planes clamped to the grid) hold fluid? Every thread of the block calls it.
__device__ __forceinline__ bool region_has_fluid(const uint8_t* __restrict__ flags, int ntx, int nty, int nz, int tx0,
                                                 int tx1, int ty0, int ty1, int z0, int z1) {
    tx1 = min(tx1, ntx);
    ty1 = min(ty1, nty);
    z0 = max(z0, 0);
    z1 = min(z1, nz - 1);
    const int wx = tx1 - tx0, wy = ty1 - ty0;
    const int cnt = (wx > 0 && wy > 0 && z1 >= z0) ? wx * wy * (z1 - z0 + 1) : 0;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    int any = 0;
    for (int i = tid; i < cnt; i += nthr) {
        const int xx = i % wx, yy = (i / wx) % wy, zz = i / (wx * wy);
        any |= flags[((long long)(z0 + zz) * nty + (ty0 + yy)) * ntx + (tx0 + xx)];
    }
    return __syncthreads_or(any) != 0;
}

// Balanced schedule over the live L0 tile columns (setup.cuh k_col_range,
// k_sched_pieces): piece p = chunk * ncol + t, column t = ty * ntx + tx,
// holds units [zlo[t], zlo[t] + pre[t+1] - pre[t])
// (a unit = `unit` planes). The pre[ncol] live units are split evenly over the
// blocks of a one-wave 1D grid, so the work is balanced whatever the geometry
// and the grid never runs a second, mostly idle wave.
struct Sched {
    const int* pre;  // [npiece + 1] exclusive prefix of the live lengths
    const int* zlo;  // [npiece] first live unit
    int npiece;      // pieces p = chunk * ncol + column
    int ncol, ntx;   // (group) columns x fastest: t = ty * ntx + tx
    int gx, gy;      // tiles per group column (x, y): its gx*gy blocks march together
    int tnx, tny;    // tiles of the grid
};

// f(tx, ty, u0, u1) for each column segment of this block's share (block-uniform).
// Columns are groups of gx x gy tiles; the gx*gy consecutive blocks of a group
// take the same share of group-column units, one tile each, so neighbouring
// tiles are marched at the same time and their halo rows and columns come
// from L2 instead of DRAM.
// bid / nblk: this block's index among the nblk blocks sharing the schedule
template <typename F>
__device__ __forceinline__ void sched_for_each_n(const Sched& sc, int bid, int nblk, F f) {
    const int G = sc.gx * sc.gy, Q = nblk / G, q = bid / G, m = bid - q * G;
    if (q >= Q) return;
    const long long W = sc.pre[sc.npiece];
    long long s = W * q / Q;
    const long long e = W * (q + 1) / Q;
    if (s >= e) return;
    int lo = 0, hi = sc.npiece - 1;  // last piece with pre[t] <= s
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sc.pre[mid] <= s)
            lo = mid;
        else
            hi = mid - 1;
    }
    for (int t = lo; s < e; ++t) {
        const long long cend = sc.pre[t + 1];
        if (cend <= s) continue;
        const long long n = min(cend, e) - s;
        const int u0 = sc.zlo[t] + (int)(s - sc.pre[t]);
        const int col = t % sc.ncol;
        const int tx = (col % sc.ntx) * sc.gx + m % sc.gx, ty = (col / sc.ntx) * sc.gy + m / sc.gx;
        if (tx < sc.tnx && ty < sc.tny) f(tx, ty, u0, u0 + (int)n);
        s += n;
    }
}
template <typename F>
__device__ __forceinline__ void sched_for_each(const Sched& sc, F f) {
    sched_for_each_n(sc, blockIdx.x, gridDim.x, f);
}

}  // namespace nb2

// npsd_b200.cu — context, per-frame setup, network and PSDO solve behind the
// C ABI in include/npsd_b200.h. One context per GPU; everything after
// set_mask stays in HBM; the PSDO loop is one CUDA graph whose body (one
// iteration: 2*depth-1 network kernels + ortho + update) repeats under a
// device-side conditional WHILE node, so the host never synchronises inside
// the solve.
#include <cudaTypedefs.h>
#include <cub/device/device_scan.cuh>

#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/npsd_b200.h"
#include "common.cuh"
#include "net.cuh"
#include "psdo.cuh"
#include "setup.cuh"
#include "stencil.cuh"
#include "net2.cuh"
#include "mixed.cuh"
#include "down0.cuh"
#include "coarse.cuh"
#include "up0.cuh"
#include "slab.cuh"
#include "cg.cuh"

using namespace nb2;

namespace {

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
struct InvalidArgument : std::runtime_error {
    explicit InvalidArgument(const std::string& w) : std::runtime_error(w) {}
};
struct Breakdown : std::runtime_error {
    explicit Breakdown(const std::string& w) : std::runtime_error(w) {}
};
struct EmptySystem : std::runtime_error {
    explicit EmptySystem(const std::string& w) : std::runtime_error(w) {}
};

#define CK(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")");                                          \
    } while (0)

inline void require(bool c, const std::string& m) {
    if (!c) throw InvalidArgument(m);
}

thread_local std::string g_create_err;

struct LevelBufs {
    Geom g{};
    long long nseg = 0;
    uint8_t* cls = nullptr;
    uint32_t *mmask = nullptr, *mbase = nullptr, *mcount = nullptr;
    float* img = nullptr;  // 3 planes (levels >= 1)
    float *tab_down = nullptr, *tab_up = nullptr;
    float *kc_down = nullptr, *kc_up = nullptr;  // [3][S]
    float *y = nullptr, *x = nullptr, *out = nullptr;
    unsigned long long* zG = nullptr;
    uint32_t* mlist = nullptr;  // compact mixed cells (k_mixed_list)
    uint32_t* mcnt = nullptr;   // their number (device)
    uint32_t* rcode = nullptr;  // levels >= 1: (window class << 30) | row per cell (k_row_codes)
    uint32_t* pid = nullptr;    // levels >= 1: mixed index -> dictionary row (dedup_patterns)
};

// one balanced schedule (common.cuh Sched) over L0 tile columns
struct SchedBufs {
    int *pre = nullptr, *zlo = nullptr, *len = nullptr, *first = nullptr, *last = nullptr;
    int ncol = 0, ntx = 0, nchunk = 0, hu = 0, npiece = 0;
    int gx = 1, gy = 1, tnx = 0, tny = 0;
    Sched view() const { return Sched{pre, zlo, npiece, ncol, ntx, gx, gy, tnx, tny}; }
};

// offsets of one level's blocks inside the flat parameter vector
struct LevelOffsets {
    size_t down_W, down_B, up_W, up_B, a_K, a_bias, b_K, b_bias;
};

}  // namespace

// ------------------------------------------------------------------ z-slab
// Communicator of a z-slab decomposition ("Multi-GPU"): ghost-plane
// exchange with the two neighbours and an allgather of per-rank partials.
// NCCL ranks enqueue both on the context's stream (graph-capturable); the
// in-process communicator (one host thread per rank, one device) uses host
// barriers and device copies and is for correctness tests only.
struct npsd_b200_comm {
    int nranks = 1;
    virtual ~npsd_b200_comm() = default;
    virtual bool capturable() const = 0;
    // planes zo0 / zo1-1 of the field at base go to rank-1 / rank+1, whose
    // boundary planes arrive in zo0-1 / zo1 (plane = pb bytes)
    virtual void exchange(int rank, cudaStream_t s, char* base, size_t pb, int zo0, int zo1) = 0;
    // all[r * bytes ...] = rank r's part, on every rank, rank order
    virtual void allgather(int rank, cudaStream_t s, const void* part, void* all, size_t bytes) = 0;
};

namespace {

// NCCL, resolved at run time (no link dependency for single-GPU use)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) return;
        auto sym = [](const char* n) { return dlsym(api.h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!api.h || !api.CommInitRank || !api.Send || !api.Recv || !api.AllGather)
        throw CudaError("npsd_b200: libnccl.so.2 not found (z-slab contexts need NCCL)");
    return api;
}

#define NCK(call)                                                                                  \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw CudaError(std::string(#call) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r_) : "nccl error")); \
    } while (0)

struct NcclComm : npsd_b200_comm {
    ncclComm_t comm = nullptr;
    int rank = 0;
    bool capturable() const override { return true; }
    void exchange(int, cudaStream_t s, char* base, size_t pb, int zo0, int zo1) override {
        NcclApi& A = nccl();
        NCK(A.GroupStart());
        if (rank > 0) {
            NCK(A.Send(base + (size_t)zo0 * pb, pb, ncclUint8, rank - 1, comm, s));
            NCK(A.Recv(base + (size_t)(zo0 - 1) * pb, pb, ncclUint8, rank - 1, comm, s));
        }
        if (rank + 1 < nranks) {
            NCK(A.Send(base + (size_t)(zo1 - 1) * pb, pb, ncclUint8, rank + 1, comm, s));
            NCK(A.Recv(base + (size_t)zo1 * pb, pb, ncclUint8, rank + 1, comm, s));
        }
        NCK(A.GroupEnd());
    }
    void allgather(int, cudaStream_t s, const void* part, void* all, size_t bytes) override {
        NCK(nccl().AllGather(part, all, bytes, ncclUint8, comm, s));
    }
    ~NcclComm() override {
        if (comm) nccl().CommDestroy(comm);
    }
};

// In-process ranks (threads) on one device: each collective is two barriers
// around device copies between the ranks' buffers; no device-side waiting.
struct LocalComm : npsd_b200_comm {
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<char*> base;
    std::vector<const void*> src;
    std::vector<int> zo0v, zo1v;
    explicit LocalComm(int n) : base(n), src(n), zo0v(n), zo1v(n) { nranks = n; }
    bool capturable() const override { return false; }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long long g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; })) {
            throw CudaError("local comm: a rank did not reach the barrier within 120 s");
        }
    }
    void exchange(int rank, cudaStream_t s, char* b, size_t pb, int zo0, int zo1) override {
        CK(cudaStreamSynchronize(s));  // this rank's owned planes are final
        base[rank] = b;
        zo0v[rank] = zo0;
        zo1v[rank] = zo1;
        barrier();
        if (rank > 0)
            CK(cudaMemcpyAsync(b + (size_t)(zo0 - 1) * pb, base[rank - 1] + (size_t)(zo1v[rank - 1] - 1) * pb, pb,
                               cudaMemcpyDeviceToDevice, s));
        if (rank + 1 < nranks)
            CK(cudaMemcpyAsync(b + (size_t)zo1 * pb, base[rank + 1] + (size_t)zo0v[rank + 1] * pb, pb,
                               cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        barrier();  // no rank overwrites its planes before every copy is done
    }
    void allgather(int rank, cudaStream_t s, const void* part, void* all, size_t bytes) override {
        CK(cudaStreamSynchronize(s));
        src[rank] = part;
        barrier();
        for (int r = 0; r < nranks; ++r)
            CK(cudaMemcpyAsync(static_cast<char*>(all) + (size_t)r * bytes, src[r], bytes, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        barrier();
    }
};

struct SlabInfo {
    bool on = false;
    int rank = 0, nranks = 1;
    int z0 = 0, nz_own = 0, nz_global = 0;  // level-0 planes
    int ghost[kMaxDepth] = {};              // ghost planes per side, level l: 2^(depth-1-l)
    npsd_b200_comm* comm = nullptr;
    double* all = nullptr;                  // [nranks][kPart] gathered partials
    unsigned long long* allu = nullptr;     // [nranks][81] gathered window counts
};

}  // namespace

struct npsd_b200_ctx {
    int dim = 3, depth = 1, S = 27, dev = 0, num_sms = 148;
    Geom g0{};
    SlabInfo slab;                // z-slab decomposition (single domain: off)
    Geom gglob[kMaxDepth] = {};   // the full grid per level (z-slab: all ranks)
    cudaGraphExec_t slab_exec = nullptr;  // z-slab: a chunk of iterations (NCCL ranks)
    cudaGraphExec_t slab_exec_short = nullptr;  // z-slab: a chunk of one ring period (the last chunks)
    long long slab_short_launches = 0;
    int slab_exec_no = -1, slab_exec_k0 = -1, slab_exec_ns = 0, slab_exec_ident = 0;
    bool slab_no_graph = false;   // the chunk graph could not be captured: eager chunks
    // programmatic dependent launch of the iteration kernels (NPSD_PDL=0
    // disables): each waits for its predecessor, then lets the next launch;
    // what a kernel reads before its wait is older than its predecessor
    // (common.cuh pdl_launch_wait)
    bool pdl = true;
    // per launch site (pdl_on; NPSD_PDL_MASK): the level-0 network kernels.
    // Measured per site (C1 / C2 / C3 us per iteration vs none): down L0
    // -2.3 / -3.6 / -3.2, up L0 -1.0 / -1.2 / -1.9, mixed down and ortho
    // neutral, update +0.5 / +7.8 / +25.6 (profiles/r02_ab_pdl_sites.txt)
    unsigned pdl_mask = 0x7;
    // the coarse-level kernels only (their setup loads overlap the previous kernel): NPSD_PDL_COARSE=0 disables
    bool pdl_coarse = true;
    double* icD = nullptr;    // IC0 factor diagonal (full grid)
    int* icFail = nullptr;    // IC0 factorization failure flag (+ scratch)
    int ic0_shift_retries = 0;
    // tiles per schedule group (common.cuh Sched): stencil/up0 and down0 schedules
    unsigned long long* htk = nullptr;  // pattern hash table: keys, values (dedup_patterns)
    uint32_t* htv = nullptr;
    unsigned long long ht_alloc = 0;            // slots allocated
    unsigned long long cap_ht[kMaxDepth] = {};  // slots used per level (power of two; grown by setup_sync)
    long long tab_alloc[kMaxDepth] = {};        // kernel-row table rows allocated per level
    // set_mask without host synchronisation (setup.cuh SetupInfo): device
    // results, their pinned readback and its event; the captured setup graph
    SetupInfo* d_info = nullptr;
    SetupInfo* info_host = nullptr;
    cudaEvent_t ev_setup = nullptr;
    // psdo_solve_n: the rhs upload overlaps a set_mask in flight (its own
    // stream, ordered after the work queued before that set_mask)
    cudaStream_t s_up = nullptr;
    cudaEvent_t ev_pre_mask = nullptr, ev_up = nullptr;
    bool setup_pending = false;
    uint8_t* types_dev = nullptr;        // the frame's cell types (the setup graph reads them here)
    const uint8_t* types_cur = nullptr;  // the buffer the last set_mask read (for a redo)
    cudaGraphExec_t mask_exec = nullptr;
    unsigned mask_exec_gen = ~0u;
    long long mask_nodes = 0;
    bool mask_graph_ok = true;
    uint32_t *dmask = nullptr, *dcount = nullptr, *dbase = nullptr;  // L0 mixed cells whose window holds fluid
    uint32_t *umask = nullptr, *ucount = nullptr, *ubase = nullptr;  // L0 mixed fluid cells
    bool fast = true;  // network arithmetic: fused/reassociated (true) or the reference's order, bitwise (false)
    int coarse_zc_max = 4;    // planes per block of the z-marching coarse kernels (at most)
    bool merge_up0 = true;    // level-0 up: tiled and mixed cells in one launch (NPSD_MERGE_UP0=0: two)
    bool classify_simd = true;  // level-0 classification with byte SIMD (NPSD_CLASSIFY_SIMD=0: one cell per thread)
    int up0_mixb = 0;         // its mixed-list blocks per SM (NPSD_UP0_MIXB; 0: by grid size, up0_mixed_blocks)
    long long slab_chunk_launches = 0;
    cudaStream_t s = nullptr, s2 = nullptr;
    std::vector<float> params;
    std::vector<LevelOffsets> offs;
    size_t coarse_W = 0, coarse_B = 0;
    float* d_params = nullptr;
    LevelBufs L[kMaxDepth];
    float* zab = nullptr;  // [depth][2]
    KC kc_down[kMaxDepth], kc_up[kMaxDepth], kc_coarse;  // host copies of the uniform kernels
    uint32_t *fmask = nullptr, *fbase = nullptr, *fcount = nullptr;
    uint32_t* fmask_prev = nullptr;  // the previous frame's fluid mask (k_zero_removed)
    uint8_t* tflags = nullptr;  // L0 tile occupancy (k_tile_flags)
    SchedBufs sch_stencil;      // 64 x 8 tile columns, plane units (k_up_l0, k_cg_dir; k_ortho2 at n_ortho > 2)
    SchedBufs sch_march;        // 64 x kMarchSY tile columns, plane units (k_ortho2, k_update2)
    SchedBufs sch_down0;        // 64 x 8 tile columns, plane-pair units, window dilation (k_down_l0)
    bool x1_clean = false;      // L1.x is zero outside sch_down0's units (and the skipped coarse tiles' outputs zero)
    // coarse down steps of the solve path: live tiles per level (k_coarse_live;
    // NPSD_COARSE_SKIP=0: every tile runs)
    bool coarse_skip = true;
    uint8_t* clive[kMaxDepth] = {};
    // level-0 window-pattern dictionary (setup.cuh)
    unsigned long long* dkeys = nullptr;
    uint32_t* dvals = nullptr;
    uint32_t *pid0 = nullptr, *repcell0 = nullptr, *npat0 = nullptr;
    // level-0 mixed sublists the solve reads (mixed.cuh): windows holding fluid
    // (down) and fluid cells (up), with their pattern ids
    uint32_t *crep = nullptr, *cnpat = nullptr;  // coarse dictionaries (scratch; level l at roff[l], cnpat[l])
    size_t koff[kMaxDepth] = {}, roff[kMaxDepth] = {};  // level l's window keys (dkeys/dvals) and crep offsets
    unsigned long long htoff[kMaxDepth] = {};          // level l's hash-table slots (htk/htv)
    unsigned long long cap_ht_graph[kMaxDepth] = {};   // the capacities the setup graph was built with
    uint32_t *dlist0 = nullptr, *dkid0 = nullptr, *dcnt0 = nullptr;
    uint32_t *ulist0 = nullptr, *ukid0 = nullptr, *ucnt0 = nullptr;
    int tf_ntx = 0, tf_nty = 0;
    long long n_fluid = 0;
    bool mask_ok = false;
    // solver
    double *X0 = nullptr, *X1 = nullptr, *R = nullptr, *Bf = nullptr, *Dtmp = nullptr;
    double *Dring = nullptr, *ADring = nullptr;
    int ring_alloc = 0;
    TmaMaps* maps = nullptr;  // tensor maps of d, the ring slots, x0 / x1 (build_tma_maps)
    SolverState* st = nullptr;
    SolverState* st_host = nullptr;  // pinned
    double* partials = nullptr;
    unsigned int* counter = nullptr;
    double *hist = nullptr, *times = nullptr;
    long long hist_cap = 0;
    double *hist_host = nullptr, *times_host = nullptr;
    long long hist_host_cap = 0;
    double *red_a = nullptr, *red_b = nullptr;
    float *xin_f = nullptr, *out_f = nullptr;  // raw-network buffers (lazy)
    double* mac = nullptr;                      // face arrays of the host mac_divergence_rhs (lazy)
    unsigned int* check_flag = nullptr;         // device input checks
    char* l2pool = nullptr;                     // levels >= 1 per-cell arrays, L2-persisting window
    long long tab_cap[kMaxDepth] = {};          // kernel-row table capacity (rows) per level
    // pcg (cg.cuh): two direction buffers, A p, z (Jacobi); graph per preconditioner
    double *cgP0 = nullptr, *cgP1 = nullptr, *cgAp = nullptr, *cgZ = nullptr;
    cudaGraphExec_t cg_exec = nullptr;
    int cg_exec_kind = -1;
    int cg_exec_ns = 0;
    unsigned cg_exec_gen = 0;
    const void* cg_exec_key = nullptr;
    unsigned buf_gen = 0;                       // bumped when a buffer a captured graph uses moves
    unsigned exec_gen = 0, slab_exec_gen = 0;
    size_t l2pool_bytes = 0;
    size_t mac_cap = 0;
    void* cub_tmp[3] = {};  // cub scratch per setup stream that scans (main, schedules, coarse chain)
    size_t cub_bytes[3] = {};
    // set_mask's independent chains run as branches of its graph (fork/join
    // through events): aux streams sx[0] solver memsets, sx[1] schedules,
    // sx[2] the coarse image chain, sx[2 + l] level l's dictionary
    bool setup_par = true;  // NPSD_SETUP_SERIAL=1: one stream
    cudaStreamAttrValue apw = {};  // the L2 access-policy window of the streams (l2pool)
    bool apw_on = false;
    cudaStream_t sx[2 * kMaxDepth + 2] = {};  // [2 + kMaxDepth + l]: level l's window counts and live tiles
    cudaEvent_t evf[4 * kMaxDepth + 8] = {};
    int nev = 0;
    // solve graph
    cudaGraphExec_t exec = nullptr;
    const void* exec_key[4] = {nullptr, nullptr, nullptr, nullptr};
    int exec_nullspace = -1, exec_no = -1, exec_ident = -1;
    int solve_ident = 0;  // the solve's preconditioner: 0 network, 1 IdentityPrecond (cfg->precond)
    int body_launches = 0, prologue_launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t user_ev[16] = {};
    std::vector<cudaEvent_t> prof_ev;
    long long launches = 0;  // kernels executed on behalf of API calls
    float last_ms = 0.0f;
    long long last_launches = 0;
    std::vector<double> report_hist, report_times;
    std::mutex mu;
    std::string err;
};

namespace {

template <typename T>
T* dalloc(size_t n) {
    T* p = nullptr;
    if (n == 0) n = 1;
    CK(cudaMalloc(&p, n * sizeof(T)));
    return p;
}

template <typename K>
int grid_for(npsd_b200_ctx* c, K kernel, long long items) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kBlock, 0));
    if (occ < 1) occ = 1;
    const long long want = (items + kBlock - 1) / kBlock;
    long long g = (long long)c->num_sms * occ;
    if (want < g) g = want;
    if (g < 1) g = 1;
    return (int)g;
}

#define LAUNCH(c, stream, kernel, items, ...)                                \
    do {                                                                     \
        auto kfn_ = kernel;                                                  \
        const int g_ = grid_for(c, kfn_, (items));                          \
        kfn_<<<g_, kBlock, 0, (stream)>>>(__VA_ARGS__);                      \
        CK(cudaGetLastError());                                              \
        ++(c)->launches;                                                     \
    } while (0)

// Launch of a tiled kernel on an explicit 3D grid.
#define LAUNCH3(c, stream, kernel, grid, block, ...)                         \
    do {                                                                     \
        auto kfn_ = kernel;                                                  \
        kfn_<<<(grid), (block), 0, (stream)>>>(__VA_ARGS__);                 \
        CK(cudaGetLastError());                                              \
        ++(c)->launches;                                                     \
    } while (0)

// Launch with dynamic shared memory.
#define LAUNCH3S(c, stream, kernel, grid, block, smem, ...)                  \
    do {                                                                     \
        auto kfn_ = kernel;                                                  \
        kfn_<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
        CK(cudaGetLastError());                                              \
        ++(c)->launches;                                                     \
    } while (0)

Geom level_geom(const npsd_b200_ctx* c, int l) {
    if (!c->slab.on) return c->gglob[l];
    // z-slab: owned planes between ghost[l] planes on each side (ghost widths
    // halve per level, so local fine plane = 2 x local coarse plane holds)
    const int G = c->slab.ghost[l], own = c->slab.nz_own >> l;
    Geom g = make_geom(c->gglob[l].nx, c->gglob[l].ny, own + 2 * G);
    g.zo0 = G;
    g.zo1 = G + own;
    return g;
}

// global index of local plane 0 at level l
int zg_offset(const npsd_b200_ctx* c, int l) {
    return c->slab.on ? (c->slab.z0 >> l) - c->slab.ghost[l] : 0;
}

// z-slab collectives on the context's stream
void slab_exchange(npsd_b200_ctx* c, cudaStream_t s, void* base, size_t elem, int l) {
    const Geom& g = c->L[l].g;
    c->slab.comm->exchange(c->slab.rank, s, static_cast<char*>(base), (size_t)g.nx * g.ny * elem, g.zo0, g.zo1);
}

void slab_allreduce_u64(npsd_b200_ctx* c, cudaStream_t s, unsigned long long* v, int k) {
    c->slab.comm->allgather(c->slab.rank, s, v, c->slab.allu, (size_t)k * sizeof(unsigned long long));
    k_sum_u64<<<1, 128, 0, s>>>(c->slab.allu, c->slab.nranks, k, v);
    CK(cudaGetLastError());
    ++c->launches;
}

void slab_reduce(npsd_b200_ctx* c, cudaStream_t s, int kind) {
    c->slab.comm->allgather(c->slab.rank, s, c->st->part, c->slab.all, kPart * sizeof(double));
    k_finalize<<<1, 32, 0, s>>>(kind, c->st, c->slab.all, c->slab.nranks, c->hist, c->times);
    CK(cudaGetLastError());
    ++c->launches;
}

void compute_offsets(npsd_b200_ctx* c) {
    const size_t S = (size_t)c->S, WN = S * 3 * S, KN = 3 * S;
    size_t o = 0;
    c->offs.assign((size_t)c->depth - 1, LevelOffsets{});
    for (auto& lo : c->offs) {
        lo.down_W = o;
        o += WN;
        lo.down_B = o;
        o += S;
        lo.up_W = o;
        o += WN;
        lo.up_B = o;
        o += S;
        lo.a_K = o;
        o += KN;
        lo.a_bias = o;
        o += 1;
        lo.b_K = o;
        o += KN;
        lo.b_bias = o;
        o += 1;
    }
    c->coarse_W = o;
    o += WN;
    c->coarse_B = o;
}

size_t param_count_impl(int dim, int depth) {
    const size_t S = (dim == 3) ? 27 : 9;
    const size_t conv = S * 3 * S + S, lin = 3 * S + 1;
    return (size_t)(depth - 1) * (2 * conv + 2 * lin) + conv;
}

// exclusive scan on stream s with cub scratch `slot` (one per setup stream that scans)
void scan_u32(npsd_b200_ctx* c, cudaStream_t s, int slot, const uint32_t* in, uint32_t* out, long long n) {
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, s));
    if (bytes > c->cub_bytes[slot]) {
        if (c->cub_tmp[slot]) CK(cudaFree(c->cub_tmp[slot]));
        CK(cudaMalloc(&c->cub_tmp[slot], bytes));
        c->cub_bytes[slot] = bytes;
    }
    CK(cub::DeviceScan::ExclusiveSum(c->cub_tmp[slot], bytes, in, out, (int)n, s));
    c->launches += 2;  // cub: tile-state init + scan
}

// set_mask branches: aux stream k continues after `from`'s work so far, and
// is joined back into the main stream before the frame's summary. Serial
// mode (z-slab contexts, NPSD_SETUP_SERIAL): everything on the main stream.
cudaStream_t setup_fork(npsd_b200_ctx* c, cudaStream_t from, int k) {
    if (!c->setup_par) return c->s;
    require(c->nev < (int)(sizeof(c->evf) / sizeof(c->evf[0])), "npsd_b200: set_mask events");
    cudaEvent_t e = c->evf[c->nev++];
    CK(cudaEventRecord(e, from));
    CK(cudaStreamWaitEvent(c->sx[k], e, 0));
    return c->sx[k];
}
void setup_join(npsd_b200_ctx* c, int k) {
    if (!c->setup_par) return;
    require(c->nev < (int)(sizeof(c->evf) / sizeof(c->evf[0])), "npsd_b200: set_mask events");
    cudaEvent_t e = c->evf[c->nev++];
    CK(cudaEventRecord(e, c->sx[k]));
    CK(cudaStreamWaitEvent(c->s, e, 0));
}

template <int D>
void upload_params_and_kconst(npsd_b200_ctx* c) {
    CK(cudaMemcpyAsync(c->d_params, c->params.data(), c->params.size() * sizeof(float), cudaMemcpyHostToDevice, c->s));
    for (int l = 0; l < c->depth; ++l) {
        LevelBufs& L = c->L[l];
        if (l < c->depth - 1) {
            const LevelOffsets& o = c->offs[(size_t)l];
            k_kconst<D><<<1, 96, 0, c->s>>>(c->d_params + o.down_W, c->d_params + o.down_B, L.kc_down);
            k_kconst<D><<<1, 96, 0, c->s>>>(c->d_params + o.up_W, c->d_params + o.up_B, L.kc_up);
        } else {
            k_kconst<D><<<1, 96, 0, c->s>>>(c->d_params + c->coarse_W, c->d_params + c->coarse_B, L.kc_down);
        }
        CK(cudaGetLastError());
        c->launches += (l < c->depth - 1) ? 2 : 1;
    }
    // host copies, passed by value to the tiled network kernels
    const size_t kb = 3 * (size_t)c->S * sizeof(float);
    for (int l = 0; l < c->depth; ++l) {
        std::memset(&c->kc_down[l], 0, sizeof(KC));
        std::memset(&c->kc_up[l], 0, sizeof(KC));
        float tmp[81];
        if (l < c->depth - 1) {
            CK(cudaMemcpyAsync(tmp, c->L[l].kc_down, kb, cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            for (int t = 0; t < 3; ++t)
                for (int k = 0; k < c->S; ++k) c->kc_down[l].k[t][k] = tmp[t * c->S + k];
            CK(cudaMemcpyAsync(tmp, c->L[l].kc_up, kb, cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            for (int t = 0; t < 3; ++t)
                for (int k = 0; k < c->S; ++k) c->kc_up[l].k[t][k] = tmp[t * c->S + k];
        } else {
            CK(cudaMemcpyAsync(tmp, c->L[l].kc_down, kb, cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            std::memset(&c->kc_coarse, 0, sizeof(KC));
            for (int t = 0; t < 3; ++t)
                for (int k = 0; k < c->S; ++k) c->kc_coarse.k[t][k] = tmp[t * c->S + k];
        }
    }
}

ConvTab tab_down(const npsd_b200_ctx* c, int l) {
    const LevelBufs& L = c->L[l];
    return ConvTab{L.cls, L.mmask, L.mbase, L.tab_down, (l == 0) ? c->pid0 : nullptr, L.kc_down, L.rcode};
}
ConvTab tab_up(const npsd_b200_ctx* c, int l) {
    const LevelBufs& L = c->L[l];
    return ConvTab{L.cls, L.mmask, L.mbase, L.tab_up, (l == 0) ? c->pid0 : nullptr, L.kc_up, L.rcode};
}

// ---------------------------------------------------------------- set_mask
// Balanced schedule over the L0 tile columns of a tx x ty tiling (units of
// `unit` planes, live within zdil planes of a fluid flag): k_sched_cols then
// the prefix. Sizes are fixed per context; buffers are made on first use.
void build_sched(npsd_b200_ctx* c, cudaStream_t s, SchedBufs& sb, int tx, int ty, int unit, int zdil, int gx, int gy) {
    const int tnx = (c->g0.nx + tx - 1) / tx, tny = (c->g0.ny + ty - 1) / ty;
    const int ntx = (tnx + gx - 1) / gx, nty = (tny + gy - 1) / gy;  // group columns
    // one piece per column: chunking columns into z pieces (chunk-major, so
    // halo rows come from L2) was measured slower — every piece restarts the
    // pipeline — so a piece is a whole column's live range
    const int hu = c->g0.nz / unit + 1;
    const int nchunk = 1;
    if (!sb.pre) {
        sb.ncol = ntx * nty;
        sb.ntx = ntx;
        sb.nchunk = nchunk;
        sb.hu = hu;
        sb.npiece = sb.ncol * nchunk;
        sb.gx = gx;
        sb.gy = gy;
        sb.tnx = tnx;
        sb.tny = tny;
        sb.pre = dalloc<int>((size_t)sb.npiece + 1);
        sb.zlo = dalloc<int>((size_t)sb.npiece);
        sb.len = dalloc<int>((size_t)sb.npiece + 1);  // len[npiece] = 0: the scan leaves the total in pre[npiece]
        CK(cudaMemset(sb.len, 0, ((size_t)sb.npiece + 1) * sizeof(int)));
        sb.first = dalloc<int>((size_t)sb.ncol);
        sb.last = dalloc<int>((size_t)sb.ncol);
    }
    const Geom& g = c->g0;
    k_col_range<<<(sb.ncol * 32 + kBlock - 1) / kBlock, kBlock, 0, s>>>(
        c->tflags, c->tf_ntx, c->tf_nty, g.nz, g.zo0, g.zo1, gx * tx / kFlagTX, gy * ty / kFlagTY, ntx, nty, zdil,
        sb.first, sb.last);
    k_sched_pieces<<<(sb.npiece + kBlock - 1) / kBlock, kBlock, 0, s>>>(sb.first, sb.last, sb.ncol, sb.nchunk, sb.hu,
                                                                         g.zo0, g.zo1, unit, zdil, sb.zlo, sb.len);
    CK(cudaGetLastError());
    c->launches += 2;
    // exclusive prefix (lengths are non-negative: scanned as u32), total included
    auto* len = reinterpret_cast<uint32_t*>(sb.len);
    auto* pre = reinterpret_cast<uint32_t*>(sb.pre);
    scan_u32(c, s, 1, len, pre, sb.npiece + 1);
}

// one wave of k's blocks (the schedule's grid)
template <typename K>
int wave_blocks(npsd_b200_ctx* c, K kernel, int threads, size_t smem) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    if (occ < 1) occ = 1;
    return c->num_sms * occ;
}

// planes per block of the z-marching coarse kernels: as many as still leave
// about four blocks per SM (small levels: short marches, more blocks)
inline int coarse_zc(const npsd_b200_ctx* c, const Geom& g) {
    const long long tiles = (long long)((g.nx + kZX - 1) / kZX) * ((g.ny + kZY - 1) / kZY);
    const int nzo = g.zo1 - g.zo0;
    int zc = c->coarse_zc_max;
    while (zc > 2 && tiles * ((nzo + zc - 1) / zc) < 4LL * c->num_sms) zc /= 2;
    return zc;
}

// Pattern ids of level l's mixed cells (keys in c->dkeys) by the hash table
// (setup.cuh k_dedup_*): pid[i], rep[pattern] = its representative, *npat.
// The table's level-l capacity (c->cap_ht[l] slots, a power of two) is sized
// from earlier frames; more than half full raises a flag instead of probing
// (the host redoes the frame, setup_sync).
void dedup_patterns(npsd_b200_ctx* c, cudaStream_t s, int l, const uint32_t* count, const uint32_t* list,
                    uint32_t* pid, uint32_t* rep, uint32_t* npat) {
    const unsigned long long cap = c->cap_ht[l];
    const long long items = std::min<long long>(c->L[l].g.n, (long long)cap);
    unsigned long long* htk = c->htk + c->htoff[l];  // level l's own table and keys: levels run concurrently
    uint32_t* htv = c->htv + c->htoff[l];
    CK(cudaMemsetAsync(htk, 0xff, cap * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(npat, 0, sizeof(uint32_t), s));
    LAUNCH(c, s, k_dedup_insert, items, c->dkeys + c->koff[l], count, list, htk, htv, cap - 1, c->dvals + c->koff[l],
           rep, npat, &c->d_info->flags, 1u << (2 * l));
    LAUNCH(c, s, k_dedup_ids, items, c->dvals + c->koff[l], count, htv, cap - 1, (uint32_t)c->tab_cap[l], pid);
}

// Every launch of a frame's setup, with no host synchronisation and no host
// decision on device data (graph-capturable): sizes come from the device
// (counts), capacities from earlier frames. The independent chains are
// branches (setup_fork / setup_join), so the captured graph's critical path
// is the longest chain, not the sum of ~80 small launches:
//   main        level-0 classification, scans, dictionary, sublists, rows
//   sx[0]       the solver vectors' zero invariant (memsets)
//   sx[1]       the tile-column schedules (tile flags of the classification)
//   sx[2]       pooled images, classification and lists of levels >= 1
//   sx[2 + l]   level l's dictionary and rows (after sx[2]'s level l)
template <int D>
void set_mask_enqueue(npsd_b200_ctx* c, const uint8_t* dtypes) {
    cudaStream_t s = c->s;
    c->nev = 0;
    LevelBufs& L0 = c->L[0];
    constexpr int NCW = (D == 3) ? 27 : 9;
    CK(cudaMemsetAsync(c->d_info, 0, sizeof(SetupInfo), s));
    // window counts of the linear blocks, levels l < depth - 1 (k_zfinal below)
    for (int l = 0; l + 1 < c->depth; ++l) CK(cudaMemsetAsync(c->L[l].zG, 0, 3 * NCW * sizeof(unsigned long long), s));
    if (c->slab.on) {  // zero invariant of the solver vectors at the new non-fluid cells
        cudaStream_t sm = setup_fork(c, s, 0);
        const size_t nb = (size_t)c->g0.n * sizeof(double);
        CK(cudaMemsetAsync(c->X1, 0, nb, sm));
        CK(cudaMemsetAsync(c->R, 0, nb, sm));
        CK(cudaMemsetAsync(c->Dtmp, 0, nb, sm));
        CK(cudaMemsetAsync(c->Dring, 0, nb * (size_t)c->ring_alloc, sm));
    }
    // levels >= 1: pooled images (from the cell types: independent of level 0's classification)
    const cudaStream_t sc = setup_fork(c, s, 2);
    for (int l = 1; l < c->depth; ++l) {
        LevelBufs& Lf = c->L[l - 1];
        LevelBufs& Lc = c->L[l];
        // pure-type bytes for the z-marching classifier (scratch: this level's row codes, written later)
        const bool marchc = D == 3 && !c->slab.on && Lc.g.nx % 32 == 0;
        uint8_t* pure = marchc ? reinterpret_cast<uint8_t*>(Lc.rcode) : nullptr;
        LAUNCH(c, sc, k_pool_image<D>, Lc.g.n, Lf.g, Lc.g, (l == 1) ? dtypes : nullptr, (l == 1) ? nullptr : Lf.img,
               Lc.img, pure);
        if (c->slab.on) {
            // ghost planes: the outside of the domain, then the neighbours' planes
            if (Lc.g.zo0 > 0)
                LAUNCH(c, sc, k_solid_planes, (long long)Lc.g.zo0 * Lc.g.nx * Lc.g.ny, Lc.g, Lc.img, 0, Lc.g.zo0);
            if (Lc.g.zo1 < Lc.g.nz)
                LAUNCH(c, sc, k_solid_planes, (long long)(Lc.g.nz - Lc.g.zo1) * Lc.g.nx * Lc.g.ny, Lc.g, Lc.img,
                       Lc.g.zo1, Lc.g.nz);
            for (int ch = 0; ch < 3; ++ch) slab_exchange(c, sc, Lc.img + (size_t)ch * Lc.g.n, sizeof(float), l);
        }
        if (marchc) {
            constexpr int ZC = 8;
            const dim3 grid(Lc.g.nx / 32, (Lc.g.ny + 7) / 8, (Lc.g.nz + ZC - 1) / ZC);
            LAUNCH3(c, sc, (k_classify_march<ZC, false>), grid, dim3(32, 8), Lc.g, (const uint8_t*)pure, Lc.cls,
                    Lc.mmask, Lc.mcount, (uint32_t*)nullptr, (uint32_t*)nullptr, 0, 0, (uint8_t*)nullptr, ZsumArgs{},
                    SubMasks{});
        } else {
            LAUNCH(c, sc, k_classify<D>, Lc.g.n, Lc.g, Lc.img, Lc.cls, Lc.mmask, Lc.mcount);
        }
        if (Lc.nseg <= kScanSmallMax) {
            SmallScan ss{};
            ss.cnt[0] = Lc.mcount;
            ss.base[0] = Lc.mbase;
            ss.n = 1;
            LAUNCH3(c, sc, k_scan_small, dim3(1), dim3(kScanSmallT), Lc.nseg, ss);
            LAUNCH(c, sc, k_mixed_list, Lc.nseg, Lc.nseg, (const uint32_t*)Lc.mmask, (const uint32_t*)Lc.mbase,
                   Lc.mlist);
        } else {
            scan_u32(c, sc, 2, Lc.mcount, Lc.mbase, Lc.nseg + 1);
            LAUNCH(c, sc, k_mixed_list, Lc.nseg, Lc.nseg, (const uint32_t*)Lc.mmask, (const uint32_t*)Lc.mbase,
                   Lc.mlist);
        }
        // level l's dictionary (hashed windows, verified) and rows
        const cudaStream_t sl = setup_fork(c, sc, 2 + l);
        {  // from the pooled image alone, beside the dictionary: live tiles and the linear block's counts
            const cudaStream_t sz = setup_fork(c, sc, 2 + kMaxDepth + l);
            if (c->clive[l]) {
                const int zc = coarse_zc(c, Lc.g);
                const int nt = ((Lc.g.nx + kZX - 1) / kZX) * ((Lc.g.ny + kZY - 1) / kZY) * ((Lc.g.nz + zc - 1) / zc);
                LAUNCH3(c, sz, k_coarse_live, dim3(nt), dim3(kBlock), Lc.g, (const float*)Lc.img, zc, c->clive[l]);
            }
            if (l < c->depth - 1) {
                // the window counts: the pooled image x 8^l (exact dyadic values)
                const int nrows = Lc.g.ny * (Lc.g.zo1 - Lc.g.zo0);  // a warp per row
                const int blocks = std::max(1, std::min((nrows + kBlock / 32 - 1) / (kBlock / 32), 4 * c->num_sms));
                LAUNCH3(c, sz, k_zsums_rows<D>, dim3(blocks), dim3(kBlock), Lc.g, (const uint8_t*)nullptr,
                        (const float*)Lc.img, (float)std::ldexp(1.0, D * l), zg_offset(c, l), c->gglob[l].nz, Lc.zG);
            }
        }
        const uint32_t rows_cap = (uint32_t)c->tab_cap[l];
        const uint32_t rows_bit = 1u << (2 * l + 1);
        uint32_t* rep = c->crep + c->roff[l];
        uint32_t* npat = c->cnpat + l;
        const uint32_t* unver = &c->d_info->unverified[l];
        const long long items = std::min<long long>(Lc.g.n, (long long)c->cap_ht[l]);
        LAUNCH(c, sl, k_window_hash<D>, items, Lc.g, Lc.img, Lc.mlist, Lc.mcnt, c->dkeys + c->koff[l],
               c->dvals + c->koff[l]);
        dedup_patterns(c, sl, l, Lc.mcnt, Lc.mlist, Lc.pid, rep, npat);
        CK(cudaMemcpyAsync(&c->d_info->npat[l], npat, sizeof(uint32_t), cudaMemcpyDeviceToDevice, sl));
        LAUNCH(c, sl, k_verify_windows<D>, items, Lc.g, Lc.img, Lc.mlist, Lc.mcnt, Lc.pid, (const uint32_t*)rep,
               &c->d_info->unverified[l]);
        LAUNCH(c, sl, k_row_codes, Lc.g.n, Lc.g, Lc.cls, Lc.mmask, Lc.mbase, Lc.pid, unver, rows_cap, Lc.rcode);
        // rows: one per window pattern when the hashed dictionary verifies, else one per mixed cell
        const long long row_items = 32LL * std::min<long long>(rows_cap, Lc.g.n);
        if (l < c->depth - 1) {
            const LevelOffsets& o = c->offs[(size_t)l];
            LAUNCH(c, sl, k_build_rows<D>, row_items, Lc.g, (const uint8_t*)nullptr, (const float*)Lc.img,
                   (const uint32_t*)rep, (const uint32_t*)npat, (const uint32_t*)Lc.mlist, (const uint32_t*)Lc.mcnt,
                   unver, rows_cap, &c->d_info->flags, rows_bit, c->d_params + o.down_W, c->d_params + o.down_B,
                   Lc.tab_down, (const float*)(c->d_params + o.up_W), (const float*)(c->d_params + o.up_B), Lc.tab_up);
        } else {
            LAUNCH(c, sl, k_build_rows<D>, row_items, Lc.g, (const uint8_t*)nullptr, (const float*)Lc.img,
                   (const uint32_t*)rep, (const uint32_t*)npat, (const uint32_t*)Lc.mlist, (const uint32_t*)Lc.mcnt,
                   unver, rows_cap, &c->d_info->flags, rows_bit, c->d_params + c->coarse_W, c->d_params + c->coarse_B,
                   Lc.tab_down, (const float*)nullptr, (const float*)nullptr, (float*)nullptr);
        }
    }
    // level 0
    const bool march0 = D == 3 && c->g0.nx % 32 == 0 && c->depth - 1 <= kMaxDepth - 1;
    if (march0) {
        // cell bytes, masks, tile flags and every level's window counts in one z-marching pass
        constexpr int ZC = 16;
        ZsumArgs za{};
        // level 0's window counts (levels >= 1 count their pooled images, below)
        za.G[0] = L0.zG;
        za.nzs = (c->depth > 1) ? 1 : 0;
        za.zg_off = zg_offset(c, 0);
        za.nxg = c->gglob[0].nx;
        za.nyg = c->gglob[0].ny;
        za.nzg = c->gglob[0].nz;
        const SubMasks sub{c->dmask, c->dcount, c->umask, c->ucount};
        // byte SIMD, 4 cells per thread, 128 x 8 or 64 x 16 tiles (setup.cuh
        // k_classify_simd); planes per block: the most that still fill two waves
        const bool simd32 = c->classify_simd && c->g0.nx % 128 == 0 && c->g0.ny % 8 == 0;
        const bool simd16 = !simd32 && c->classify_simd && c->g0.nx % 64 == 0 && c->g0.ny % 16 == 0;
        if (simd32 || simd16) {
            const long long tiles = simd32 ? (long long)(c->g0.nx / 128) * (c->g0.ny / 8)
                                           : (long long)(c->g0.nx / 64) * (c->g0.ny / 16);
            const int zc = (tiles * ((c->g0.nz + 15) / 16) >= 2 * c->num_sms)  ? 16
                           : (tiles * ((c->g0.nz + 3) / 4) >= 2 * c->num_sms) ? 4
                                                                              : 2;
            const dim3 grid(simd32 ? c->g0.nx / 128 : c->g0.nx / 64, simd32 ? c->g0.ny / 8 : c->g0.ny / 16,
                            (c->g0.nz + zc - 1) / zc);
#define NPSD_CLASSIFY_SIMD(LX, Z)                                                                                     \
    LAUNCH3(c, s, (k_classify_simd<LX, Z>), grid, dim3(256), c->g0, dtypes, L0.cls, L0.mmask, L0.mcount, c->fmask,   \
            c->fcount, c->tf_ntx, c->tf_nty, c->tflags, za, sub)
            if (simd32) {
                if (zc == 16) NPSD_CLASSIFY_SIMD(32, 16);
                else if (zc == 4) NPSD_CLASSIFY_SIMD(32, 4);
                else NPSD_CLASSIFY_SIMD(32, 2);
            } else {
                if (zc == 16) NPSD_CLASSIFY_SIMD(16, 16);
                else if (zc == 4) NPSD_CLASSIFY_SIMD(16, 4);
                else NPSD_CLASSIFY_SIMD(16, 2);
            }
#undef NPSD_CLASSIFY_SIMD
        } else {
            const dim3 grid(c->g0.nx / 32, (c->g0.ny + 7) / 8, (c->g0.nz + ZC - 1) / ZC);
            LAUNCH3(c, s, (k_classify_march<ZC, true>), grid, dim3(32, 8), c->g0, dtypes, L0.cls, L0.mmask, L0.mcount,
                    c->fmask, c->fcount, c->tf_ntx, c->tf_nty, c->tflags, za, sub);
        }
    } else {
        LAUNCH(c, s, k_setup_l0<D>, c->g0.n, c->g0, dtypes, L0.cls, L0.mmask, L0.mcount, c->fmask, c->fcount);
        LAUNCH(c, s, k_tile_flags, (long long)c->tf_ntx * c->tf_nty * c->g0.nz, c->g0, dtypes, c->tf_ntx, c->tf_nty,
               c->tflags);
    }
    if (!c->slab.on) {  // zero invariant: only the cells the previous frame had as fluid and this one not
        cudaStream_t sm = setup_fork(c, s, 0);
        LAUNCH(c, sm, k_zero_removed, L0.nseg, L0.nseg, c->fmask_prev, (const uint32_t*)c->fmask, c->X1, c->R,
               c->Dtmp, c->Dring, c->ring_alloc, c->g0.n);
    }
    if (!march0) LAUNCH(c, s, k_sub_masks, L0.g.n, L0.g, L0.cls, c->dmask, c->dcount, c->umask, c->ucount);
    const bool small0 = L0.nseg <= kScanSmallMax;
    {
        const cudaStream_t sb = setup_fork(c, s, 1);
        if (!small0) {  // the down / up prefixes (k_mixed_sub, after a join)
            scan_u32(c, sb, 1, c->dcount, c->dbase, L0.nseg + 1);
            scan_u32(c, sb, 1, c->ucount, c->ubase, L0.nseg + 1);
        }
        build_sched(c, sb, c->sch_stencil, kTX, kTY, 1, 0, 1, 1);
        if (kMarchSY != kSY) build_sched(c, sb, c->sch_march, kTX, kMarchSY, 1, 0, 1, 1);
        if (D == 3 && c->depth > 1) build_sched(c, sb, c->sch_down0, kTX, kTY, 2, 1, 1, 1);
    }
    // the mixed, fluid, down and up prefixes (totals land in base[nseg]) and the mixed list
    if (small0) {
        SmallScan ss{{L0.mcount, c->fcount, c->dcount, c->ucount}, {L0.mbase, c->fbase, c->dbase, c->ubase}, 4,
                     nullptr, nullptr};
        LAUNCH3(c, s, k_scan_small, dim3(1), dim3(kScanSmallT), L0.nseg, ss);
        LAUNCH(c, s, k_mixed_list, L0.nseg, L0.nseg, (const uint32_t*)L0.mmask, (const uint32_t*)L0.mbase, L0.mlist);
    } else {
        scan_u32(c, s, 0, L0.mcount, L0.mbase, L0.nseg + 1);
        scan_u32(c, s, 0, c->fcount, c->fbase, L0.nseg + 1);
        LAUNCH(c, s, k_mixed_list, L0.nseg, L0.nseg, (const uint32_t*)L0.mmask, (const uint32_t*)L0.mbase, L0.mlist);
    }
    // window-pattern dictionary (pid per mixed cell, one row per pattern),
    // then the solve's down / up sublists with their pattern ids
    LAUNCH(c, s, k_window_keys<D>, std::min<long long>(c->g0.n, (long long)c->cap_ht[0]), c->g0, dtypes, L0.mlist,
           L0.mcnt, c->dkeys, c->dvals);
    dedup_patterns(c, s, 0, L0.mcnt, L0.mlist, c->pid0, c->repcell0, c->npat0);
    CK(cudaMemcpyAsync(&c->d_info->npat[0], c->npat0, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    if (!small0) setup_join(c, 1);
    LAUNCH(c, s, k_mixed_sub, std::min<long long>(c->g0.n, (long long)c->cap_ht[0]), L0.mlist, c->pid0, L0.mcnt,
           c->dmask, c->dbase, c->umask, c->ubase, c->dlist0, c->dkid0, c->ulist0, c->ukid0);
    if (c->depth > 1) {
        const uint32_t rows_cap = (uint32_t)c->tab_cap[0];
        const LevelOffsets& o = c->offs[0];
        LAUNCH(c, s, k_build_rows<D>, 32LL * std::min<long long>(rows_cap, L0.g.n), L0.g, dtypes, (const float*)nullptr,
               (const uint32_t*)c->repcell0, (const uint32_t*)c->npat0, (const uint32_t*)L0.mlist,
               (const uint32_t*)L0.mcnt, (const uint32_t*)nullptr, rows_cap, &c->d_info->flags, 1u << 1,
               c->d_params + o.down_W, c->d_params + o.down_B, L0.tab_down, (const float*)(c->d_params + o.up_W),
               (const float*)(c->d_params + o.up_B), L0.tab_up);
    } else {
        const uint32_t rows_cap = (uint32_t)c->tab_cap[0];
        LAUNCH(c, s, k_build_rows<D>, 32LL * std::min<long long>(rows_cap, L0.g.n), L0.g, dtypes, (const float*)nullptr,
               (const uint32_t*)c->repcell0, (const uint32_t*)c->npat0, (const uint32_t*)L0.mlist,
               (const uint32_t*)L0.mcnt, (const uint32_t*)nullptr, rows_cap, &c->d_info->flags, 1u << 1,
               c->d_params + c->coarse_W, c->d_params + c->coarse_B, L0.tab_down, (const float*)nullptr,
               (const float*)nullptr, (float*)nullptr);
    }
    for (int k = 0; k < 2 + c->depth; ++k) setup_join(c, k);  // zeroing, schedules, coarse chain, dictionaries 1..
    for (int l = 1; l < c->depth; ++l) setup_join(c, 2 + kMaxDepth + l);  // counts and live tiles 1..
    // linear-block coefficients of every level (k_zfinal: one block per level)
    ZfinArgs zf{};
    for (int l = 0; l + 1 < c->depth; ++l) {
        LevelBufs& L = c->L[l];
        constexpr int NC = (D == 3) ? 27 : 9;
        const double scale = std::ldexp(1.0, D * l);
        if (l == 0 && !march0) {  // (levels >= 1: in their branches)
            const int nrows = L.g.ny * (L.g.zo1 - L.g.zo0);  // a warp per row
            const int blocks = std::max(1, std::min((nrows + kBlock / 32 - 1) / (kBlock / 32), 4 * c->num_sms));
            LAUNCH3(c, s, k_zsums_rows<D>, dim3(blocks), dim3(kBlock), L.g, dtypes, (const float*)nullptr,
                    (float)scale, zg_offset(c, l), c->gglob[l].nz, L.zG);
        }
        if (c->slab.on) slab_allreduce_u64(c, s, L.zG, 3 * NC);
        const LevelOffsets& o = c->offs[(size_t)l];
        zf.lv[l] = ZfinLevel{c->gglob[l], L.zG, scale, c->d_params + o.a_K, c->d_params + o.b_K,
                             c->params[o.a_bias], c->params[o.b_bias], c->zab + 2 * l, c->zab + 2 * l + 1};
    }
    if (c->depth > 1) LAUNCH3(c, s, k_zfinal<D>, dim3(c->depth - 1), dim3(128), zf);
    InfoSources src{};
    src.n_fluid = c->fbase + L0.nseg;
    src.depth = c->depth;
    for (int l = 0; l < c->depth; ++l) src.n_mixed[l] = c->L[l].mcnt;
    LAUNCH3(c, s, k_setup_info, dim3(1), dim3(32), src, c->d_info);
    if (c->slab.on) {  // the ranks redo a frame together
        unsigned long long* v = reinterpret_cast<unsigned long long*>(c->red_b);
        LAUNCH3(c, s, k_flags_u64, dim3(1), dim3(32), (const uint32_t*)&c->d_info->flags, v);
        slab_allreduce_u64(c, s, v, 1);
        LAUNCH3(c, s, k_u64_flags, dim3(1), dim3(32), (const unsigned long long*)v, &c->d_info->flags);
    }
}

// cub scratch for every scan set_mask runs, per scanning stream (allocated outside any capture)
void ensure_cub(npsd_b200_ctx* c) {
    long long nmax = c->L[0].nseg;
    for (const SchedBufs* sb : {&c->sch_stencil, &c->sch_march, &c->sch_down0}) nmax = std::max<long long>(nmax, sb->npiece);
    // the schedules' piece counts (build_sched allocates them on first use): bounded by the tile columns
    nmax = std::max<long long>(nmax, (long long)((c->g0.nx + kTX - 1) / kTX) * ((c->g0.ny + kTY - 1) / kTY) + 1);
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)nmax, c->s));
    for (int k = 0; k < 3; ++k)
        if (bytes > c->cub_bytes[k]) {
            if (c->cub_tmp[k]) CK(cudaFree(c->cub_tmp[k]));
            CK(cudaMalloc(&c->cub_tmp[k], bytes));
            c->cub_bytes[k] = bytes;
        }
}

// kernel-row tables (rows per level) and the pattern hash table at the
// current capacities (grow only; the captured setup graph holds the pointers)
void ensure_setup_capacity(npsd_b200_ctx* c) {
    for (int l = 0; l < c->depth; ++l) {
        LevelBufs& L = c->L[l];
        if (c->tab_alloc[l] < c->tab_cap[l]) {
            const size_t rows = (size_t)c->tab_cap[l];
            if (L.tab_down) CK(cudaFree(L.tab_down));
            L.tab_down = dalloc<float>((size_t)kRowW * rows);
            if (l < c->depth - 1) {
                if (L.tab_up) CK(cudaFree(L.tab_up));
                L.tab_up = dalloc<float>((size_t)kRowW * rows);
            }
            c->tab_alloc[l] = c->tab_cap[l];
            ++c->buf_gen;
        }
    }
    // one table per level (the levels' dictionaries run concurrently)
    unsigned long long ht = 0;
    bool moved = false;
    for (int l = 0; l < c->depth; ++l) {
        c->htoff[l] = ht;
        ht += c->cap_ht[l];
        moved |= c->cap_ht[l] != c->cap_ht_graph[l];  // a captured setup graph holds the sizes too
        c->cap_ht_graph[l] = c->cap_ht[l];
    }
    if (moved) ++c->buf_gen;
    if (ht > c->ht_alloc) {
        if (c->htk) CK(cudaFree(c->htk));
        if (c->htv) CK(cudaFree(c->htv));
        c->htk = dalloc<unsigned long long>((size_t)ht);
        c->htv = dalloc<uint32_t>((size_t)ht);
        c->ht_alloc = ht;
        ++c->buf_gen;
    }
}

// One frame's setup from device cell types: the launches of set_mask_enqueue,
// replayed as one captured graph per context (z-slab contexts: eager, their
// exchanges run through the communicator), then an asynchronous readback of
// the frame's SetupInfo. Nothing here waits for the device.
template <int D>
void set_mask_run(npsd_b200_ctx* c, const uint8_t* dtypes) {
    CK(cudaEventRecord(c->ev_pre_mask, c->s));
    ensure_setup_capacity(c);
    c->x1_clean = false;
    const bool graph = !c->slab.on && c->mask_graph_ok && dtypes == c->types_dev;
    if (graph) {
        if (!c->mask_exec || c->mask_exec_gen != c->buf_gen) {
            if (c->mask_exec) CK(cudaGraphExecDestroy(c->mask_exec));
            c->mask_exec = nullptr;
            ensure_cub(c);
            // schedules allocate their buffers on first use: once outside the capture
            if (!c->sch_stencil.pre) set_mask_enqueue<D>(c, dtypes);
            const long long before = c->launches;
            CK(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
            try {
                set_mask_enqueue<D>(c, dtypes);
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(c->s, &junk);
                if (junk) cudaGraphDestroy(junk);
                cudaGetLastError();
                c->mask_graph_ok = false;  // eager from now on
                c->launches = before;
                set_mask_enqueue<D>(c, dtypes);
                goto readback;
            }
            cudaGraph_t gr = nullptr;
            CK(cudaStreamEndCapture(c->s, &gr));
            const cudaError_t ie = cudaGraphInstantiate(&c->mask_exec, gr, 0);
            cudaGraphDestroy(gr);
            CK(ie);
            c->mask_nodes = c->launches - before;
            c->launches = before;
            c->mask_exec_gen = c->buf_gen;
        }
        CK(cudaGraphLaunch(c->mask_exec, c->s));
        c->launches += c->mask_nodes;
    } else {
        set_mask_enqueue<D>(c, dtypes);
    }
readback:
    CK(cudaMemcpyAsync(c->info_host, c->d_info, sizeof(SetupInfo), cudaMemcpyDeviceToHost, c->s));
    CK(cudaEventRecord(c->ev_setup, c->s));
    c->setup_pending = true;
    c->mask_ok = true;
}

// Finishes the last set_mask on the host: waits for its SetupInfo; when a
// capacity was too small, grows it from the frame's counts and redoes the
// frame (a few times at most: the first frames of a context). Returns true
// when the frame was redone (device work queued before the call saw the
// smaller tables and must be repeated).
bool setup_sync(npsd_b200_ctx* c) {
    if (!c->setup_pending) return false;
    bool redone = false;
    for (int attempt = 0;; ++attempt) {
        CK(cudaEventSynchronize(c->ev_setup));
        const SetupInfo& h = *c->info_host;
        if (h.flags == 0) break;
        require(attempt < 4, "npsd_b200: set_mask capacities did not converge");
        for (int l = 0; l < c->depth; ++l) {
            const unsigned long long want_ht = std::max<unsigned long long>(1024, 2ull * h.n_mixed[l] + h.n_mixed[l] / 2);
            while (c->cap_ht[l] < want_ht) c->cap_ht[l] <<= 1;
            const long long rows = std::max<long long>(
                {(long long)h.npat[l], (l > 0 && h.unverified[l]) ? (long long)h.n_mixed[l] : 0LL, 1LL});
            if (rows > c->tab_cap[l]) c->tab_cap[l] = rows + rows / 4 + 64;
            if ((h.flags >> (2 * l)) & 1u) {  // the table was skipped: npat unknown, allow every mixed cell a row
                c->tab_cap[l] = std::max<long long>(c->tab_cap[l], (long long)h.n_mixed[l] + 64);
            }
        }
        if (c->dim == 3)
            set_mask_run<3>(c, c->types_cur);
        else
            set_mask_run<2>(c, c->types_cur);
        redone = true;
    }
    c->n_fluid = c->info_host->n_fluid;
    c->setup_pending = false;
    return redone;
}

template <int D>
void set_mask_impl(npsd_b200_ctx* c, const uint8_t* dtypes) {
    c->types_cur = dtypes;
    set_mask_run<D>(c, dtypes);
}

// ------------------------------------------------------------ network
// One named launcher per kernel of an iteration: the graph body is captured
// from these, and the profiler runs them one by one between CUDA events.
struct Step {
    std::string name;
    std::function<void(cudaStream_t)> run;
};

// Launch of an iteration kernel (one that starts with pdl_launch_wait()) with
// programmatic stream serialisation: its blocks may launch while the previous
// kernel drains; in a captured graph this becomes a programmatic edge.
template <typename... KArgs, typename... Args>
void launch_pdl_if(npsd_b200_ctx* c, cudaStream_t s, bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block,
                   size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
    ++c->launches;
}
template <typename... KArgs, typename... Args>
void launch_pdl(npsd_b200_ctx* c, cudaStream_t s, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                Args&&... args) {
    launch_pdl_if(c, s, c->pdl, k, grid, block, smem, std::forward<Args>(args)...);
}
// the coarse-level kernels read only setup data before their wait (coarse.cuh)
inline bool pdl_coarse(const npsd_b200_ctx* c) { return c->pdl || (c->pdl_coarse && !c->slab.on); }
// the level-0 / solver kernels: bit 0 mixed down, 1 down L0, 2 up L0 (+ mixed up), 3 ortho, 4 update
inline bool pdl_on(const npsd_b200_ctx* c, int bit) { return c->pdl && ((c->pdl_mask >> bit) & 1); }

// z-chunk (in bricks or planes) so that a launch has about two waves of blocks.
template <typename K>
int zchunk_for(npsd_b200_ctx* c, K kernel, int threads, long long tiles_xy, int nz_units, size_t smem = 0) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem));
    if (occ < 1) occ = 1;
    const long long target = 2LL * c->num_sms * occ;
    long long zc = (tiles_xy * nz_units + target - 1) / target;
    if (zc < 1) zc = 1;
    if (zc > nz_units) zc = nz_units;
    return (int)zc;
}

template <int D, bool L0, bool POOL>
void launch_down(npsd_b200_ctx* c, cudaStream_t s, int l, const float* in_f, const double* in_d,
                 bool skip = false) {
    LevelBufs& L = c->L[l];
    const Geom gc = POOL ? c->L[l + 1].g : L.g;
    float* xnext = POOL ? c->L[l + 1].x : nullptr;
    if (D == 3 && !L0) {
        // f32 input (levels >= 1, raw level 0): z-marching columns (coarse.cuh)
        const KC& kc = (l == c->depth - 1) ? c->kc_coarse : c->kc_down[l];
        const int* dn = c->slab.on ? &c->st->done : nullptr;
        const int zc = coarse_zc(c, L.g);
        const dim3 grid((L.g.nx + kZX - 1) / kZX, (L.g.ny + kZY - 1) / kZY, (L.g.zo1 - L.g.zo0 + zc - 1) / zc);
        const uint8_t* live = (skip && POOL) ? c->clive[l] : nullptr;
#define NPSD_CDOWN(ZC_, F_) \
    launch_pdl_if(c, s, pdl_coarse(c), k_cdownz<POOL, ZC_, F_>, grid, dim3(kZT), 0, L.g, in_f, tab_down(c, l), kc, L.y, \
                  xnext, gc, dn, live)
        if (c->fast) {
            if (zc == 8) NPSD_CDOWN(8, true);
            else if (zc == 4) NPSD_CDOWN(4, true);
            else NPSD_CDOWN(2, true);
        } else {
            if (zc == 8) NPSD_CDOWN(8, false);
            else if (zc == 4) NPSD_CDOWN(4, false);
            else NPSD_CDOWN(2, false);
        }
#undef NPSD_CDOWN
        return;
    }
    const dim3 block(kNX, kNY);
    const int gx = (L.g.nx + 2 * kNX - 1) / (2 * kNX), gy = (L.g.ny + 2 * kNY - 1) / (2 * kNY);
    const int nbz = (D == 3) ? (L.g.nz >> 1) : 1;
    auto k = k_down3<D, L0, POOL>;
    // coarse levels are small: one brick plane per block keeps the serial chain short
    const int zc = (l > 0) ? 1 : zchunk_for(c, k, kNX * kNY, (long long)gx * gy, nbz);
    const dim3 grid(gx, gy, (nbz + zc - 1) / zc);
    const KC& kc = (l == c->depth - 1) ? c->kc_coarse : c->kc_down[l];
    const Occ occ = (L0 && c->tflags) ? Occ{c->tflags, c->tf_ntx, c->tf_nty} : Occ{nullptr, 0, 0};
    LAUNCH3(c, s, k, grid, block, L.g, in_f, in_d, c->st, tab_down(c, l), kc, L.y, xnext, gc, zc, occ);
}

template <int D, int MODE, int NO>
void launch_up(npsd_b200_ctx* c, cudaStream_t s, int l, float* outl, double* dout, bool skip = false) {
    LevelBufs& L = c->L[l];
    const LevelBufs& Lc = c->L[l + 1];
    const float* outc = (l + 1 == c->depth - 1) ? Lc.y : Lc.out;
    if (D == 3 && MODE == kUpMid) {
        const int* dn = c->slab.on ? &c->st->done : nullptr;
        const int zc = coarse_zc(c, L.g);
        const dim3 grid((L.g.nx + kZX - 1) / kZX, (L.g.ny + kZY - 1) / kZY, (L.g.zo1 - L.g.zo0 + zc - 1) / zc);
#define NPSD_CUP(ZC_, F_)                                                                                        \
    launch_pdl_if(c, s, pdl_coarse(c), k_cupz<ZC_, F_>, grid, dim3(kZT), 0, L.g, Lc.g, outc, L.y, c->zab + 2 * l, \
                  tab_up(c, l), c->kc_up[l], outl, dn, skip ? c->clive[l] : (const uint8_t*)nullptr)
        if (c->fast) {
            if (zc == 8) NPSD_CUP(8, true);
            else if (zc == 4) NPSD_CUP(4, true);
            else NPSD_CUP(2, true);
        } else {
            if (zc == 8) NPSD_CUP(8, false);
            else if (zc == 4) NPSD_CUP(4, false);
            else NPSD_CUP(2, false);
        }
#undef NPSD_CUP
        return;
    }
    const dim3 block(kNX, kNY);
    const int gx = (Lc.g.nx + kNX - 1) / kNX, gy = (Lc.g.ny + kNY - 1) / kNY;
    const int nbz = (D == 3) ? Lc.g.nz : 1;
    auto k = k_up3<D, MODE, NO>;
    const int zc = (l > 0) ? 1 : zchunk_for(c, k, kNX * kNY, (long long)gx * gy, nbz);
    const dim3 grid(gx, gy, (nbz + zc - 1) / zc);
    LAUNCH3(c, s, k, grid, block, L.g, Lc.g, outc, L.y, c->zab + 2 * l, tab_up(c, l), c->kc_up[l], outl, dout, c->st,
            c->ADring, c->partials, c->counter, zc,
            (MODE == kUpL0) ? Occ{c->tflags, c->tf_ntx, c->tf_nty} : Occ{nullptr, 0, 0});
}

// KUp0 of a uniform-fluid up kernel: its slots and the parity-merged taps
// (up0.cuh), summed in f64 and rounded once
KUp0 up0_kernel(const float* k27) {
    KUp0 o;
    for (int i = 0; i < 27; ++i) o.k[i] = k27[i];
    for (int p = 0; p < 8; ++p) {
        const int pz = p >> 2, py = (p >> 1) & 1, px = p & 1;
        double m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        auto side = [](int par, int d) { return ((par + d) >> 1) - par + 1; };  // 0 = lo coarse cell, 1 = hi
        for (int t = 0; t < 27; ++t) {
            const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
            m[side(pz, dz) * 4 + side(py, dy) * 2 + side(px, dx)] += (double)k27[t];
        }
        for (int j = 0; j < 8; ++j) o.m[p][j] = (float)m[j];
    }
    return o;
}

template <int D, int NO>
void launch_up0(npsd_b200_ctx* c, cudaStream_t s) {
    if (D == 3) {
        // 3D: the pipelined level-0 up sweep on the balanced schedule (up0.cuh)
        const LevelBufs& L = c->L[0];
        const LevelBufs& L1 = c->L[1];
        const float* outc = (c->depth == 2) ? L1.y : L1.out;
        const KUp0 kc0 = up0_kernel(c->kc_up[0].k[0]);  // the uniform-fluid kernel (+ merged parity taps)
        const size_t sm = sizeof(Up0Smem<NO>);
        if (c->merge_up0) {
            // tiled and mixed cells in one launch (k_up_l0m): a wave of tile
            // blocks plus one block per SM for the mixed list
            auto k = c->fast ? k_up_l0m<NO, true> : k_up_l0m<NO, false>;
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            const int nt = wave_blocks(c, k, kSX * kSY, sm);
            // mixed-list blocks per SM: measured best 1 at 64^3, 2 at 128^3, 4 at 256^3
            // (C1/C2/C3, tools/env_ab.py NPSD_UP0_MIXB): about one per 2^20 cells, 1..4
            const int mixb = c->up0_mixb ? c->up0_mixb : (int)std::max(1LL, std::min(4LL, L.g.n >> 20));
            launch_pdl_if(c, s, pdl_on(c, 2), k, dim3(nt + mixb * c->num_sms), dim3(kSX, kSY), sm, L.g, L1.g, L.cls, outc, L.y, c->zab, kc0,
                       c->Dtmp, c->st, c->ADring, c->partials, c->counter, c->sch_down0.view(), nt,
                       (const uint32_t*)c->ulist0, (const uint32_t*)c->ucnt0, (const float*)L.tab_up,
                       (const uint32_t*)c->ukid0);
            return;
        }
        auto k = c->fast ? k_up_l0<NO, true> : k_up_l0<NO, false>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        launch_pdl_if(c, s, pdl_on(c, 2), k, dim3(wave_blocks(c, k, kSX * kSY, sm)), dim3(kSX, kSY), sm, L.g, L1.g, L.cls, outc, L.y,
                   c->zab, kc0, c->Dtmp, c->st, c->ADring, c->partials, c->counter, c->sch_down0.view());
        return;
    }
    launch_up<D, kUpL0, NO>(c, s, 0, nullptr, c->Dtmp);
}

// n_ortho (the cache bound) is a template parameter of the kernels that loop
// over the cached directions; dispatch once at launch-build time.
template <int D>
void launch_up0_no(npsd_b200_ctx* c, cudaStream_t s, int no) {
    switch (no) {
        case 0: launch_up0<D, 0>(c, s); break;
        case 1: launch_up0<D, 1>(c, s); break;
        case 2: launch_up0<D, 2>(c, s); break;
        case 3: launch_up0<D, 3>(c, s); break;
        case 4: launch_up0<D, 4>(c, s); break;
        default: launch_up0<D, kMaxOrtho>(c, s); break;
    }
}

template <int D, int NO>
void launch_ortho(npsd_b200_ctx* c, cudaStream_t s) {
    const Geom g = c->g0;
    constexpr int SY = march_sy<OrthoOp<NO>>();
    const dim3 block(kSX, SY);
    auto k = k_ortho2<D, NO, SY>;
    const size_t sm = stencil_smem_bytes<D, OrthoOp<NO>, SY>();
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const dim3 grid(wave_blocks(c, k, kSX * SY, sm));
    launch_pdl_if(c, s, pdl_on(c, 3), k, grid, block, sm, g, c->L[0].cls, c->Dtmp, c->R, c->Dring, c->ADring, c->st, c->partials,
               c->counter, (SY == kSY ? c->sch_stencil : c->sch_march).view(), *c->maps);
}

template <int D>
void launch_ortho_no(npsd_b200_ctx* c, cudaStream_t s, int no) {
    switch (no) {
        case 0: launch_ortho<D, 0>(c, s); break;
        case 1: launch_ortho<D, 1>(c, s); break;
        case 2: launch_ortho<D, 2>(c, s); break;
        case 3: launch_ortho<D, 3>(c, s); break;
        case 4: launch_ortho<D, 4>(c, s); break;
        default: launch_ortho<D, kMaxOrtho>(c, s); break;
    }
}

template <int D>
void launch_update(npsd_b200_ctx* c, cudaStream_t s, cudaGraphConditionalHandle h, int use_cond, int do_norm) {
    const Geom g = c->g0;
    constexpr int SY = march_sy<UpdateOp>();
    const dim3 block(kSX, SY);
    auto k = k_update2<D, SY>;
    const size_t sm = stencil_smem_bytes<D, UpdateOp, SY>();
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const dim3 grid(wave_blocks(c, k, kSX * SY, sm));
    launch_pdl_if(c, s, pdl_on(c, 4), k, grid, block, sm, g, c->L[0].cls, c->Bf, c->X0, c->X1, c->Dring, c->R, c->st, c->hist,
               c->times, c->partials, c->counter, h, use_cond, do_norm, (SY == kSY ? c->sch_stencil : c->sch_march).view(),
               *c->maps);
}

// One named launcher per kernel of an iteration: the graph body is captured
// from these, and the profiler runs them one by one between CUDA events.
// raw: the network on an f32 full-grid input (xin_f -> out_f), no solver.
// 3D level-0 down sweep with pooling (down0.cuh)
void launch_down_l0(npsd_b200_ctx* c, cudaStream_t s) {
    const LevelBufs& L = c->L[0];
    const Geom g = L.g;
    const dim3 block(kSX, kSY);
    const size_t sm = sizeof(Down0Smem);
    auto k = c->fast ? k_down_l0<true> : k_down_l0<false>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const dim3 grid(wave_blocks(c, k, kSX * kSY, sm));
    KC0 kc0;
    for (int i = 0; i < 27; ++i) kc0.k[i] = c->kc_down[0].k[0][i];  // the uniform-fluid kernel
    launch_pdl_if(c, s, pdl_on(c, 1), k, grid, block, sm, g, L.cls, c->R, (const SolverState*)c->st, kc0, L.y, c->L[1].x, c->L[1].g,
               c->sch_down0.view());
}

template <int D>
void launch_mixed_down0(npsd_b200_ctx* c, cudaStream_t s) {
    const LevelBufs& L = c->L[0];
    auto k = c->fast ? k_mixed_down0<D, true> : k_mixed_down0<D, false>;
    launch_pdl_if(c, s, pdl_on(c, 0), k, dim3(grid_for(c, k, L.g.n)), dim3(kBlock), 0, L.g, c->dlist0, c->dcnt0, c->R,
               (const SolverState*)c->st, L.tab_down, c->dkid0, L.y);
}

template <int D, int NO>
void launch_mixed_up0(npsd_b200_ctx* c, cudaStream_t s) {
    const LevelBufs& L = c->L[0];
    const LevelBufs& L1 = c->L[1];
    const float* outc = (c->depth == 2) ? L1.y : L1.out;
    auto k = c->fast ? k_mixed_up0<D, NO, true> : k_mixed_up0<D, NO, false>;
    launch_pdl_if(c, s, pdl_on(c, 2), k, dim3(grid_for(c, k, L.g.n)), dim3(kBlock), 0, L.g, L1.g, c->ulist0, c->ucnt0, outc, L.y,
               c->zab, L.tab_up, c->ukid0, c->Dtmp, c->st, c->ADring, c->partials, c->counter);
}

template <int D>
void launch_mixed_up0_no(npsd_b200_ctx* c, cudaStream_t s, int no) {
    switch (no) {
        case 0: launch_mixed_up0<D, 0>(c, s); break;
        case 1: launch_mixed_up0<D, 1>(c, s); break;
        case 2: launch_mixed_up0<D, 2>(c, s); break;
        case 3: launch_mixed_up0<D, 3>(c, s); break;
        case 4: launch_mixed_up0<D, 4>(c, s); break;
        default: launch_mixed_up0<D, kMaxOrtho>(c, s); break;
    }
}

// z-slab: ghost planes of a level-l field refreshed from the neighbours
Step xchg_step(npsd_b200_ctx* c, const std::string& name, std::function<void*()> ptr, size_t elem, int l) {
    return {name, [c, ptr, elem, l](cudaStream_t s) { slab_exchange(c, s, ptr(), elem, l); }};
}

Step reduce_step(npsd_b200_ctx* c, const std::string& name, int kind) {
    return {name, [c, kind](cudaStream_t s) { slab_reduce(c, s, kind); }};
}

template <int D>
std::vector<Step> network_steps(npsd_b200_ctx* c, bool raw, int no) {
    std::vector<Step> v;
    const int Ld = c->depth;
    const bool xg = c->slab.on && !raw;  // z-slab: halos before every conv level
    // solve path: level-0 mixed-window cells are computed apart (mixed.cuh)
    if (!raw) v.push_back({"net_mixed_down_L0", [c](cudaStream_t s) { launch_mixed_down0<D>(c, s); }});
    for (int l = 0; l < Ld; ++l) {
        const bool pool = (l + 1 < Ld);
        const std::string nm = (l == Ld - 1) ? "net_coarse_L" + std::to_string(l) : "net_down_L" + std::to_string(l);
        v.push_back({nm, [c, l, pool, raw](cudaStream_t s) {
                         if (l == 0 && !raw) {
                             if (pool && D == 3)
                                 launch_down_l0(c, s);
                             else if (pool)
                                 launch_down<D, true, true>(c, s, 0, nullptr, c->R);
                             else
                                 launch_down<D, true, false>(c, s, 0, nullptr, c->R);
                         } else {
                             const float* in = (l == 0) ? c->xin_f : c->L[l].x;
                             if (pool)
                                 launch_down<D, false, true>(c, s, l, in, nullptr, !raw);
                             else
                                 launch_down<D, false, false>(c, s, l, in, nullptr);
                         }
                     }});
        if (xg && pool)
            v.push_back(xchg_step(c, "xchg_x_L" + std::to_string(l + 1), [c, l] { return (void*)c->L[l + 1].x; },
                                  sizeof(float), l + 1));
        else if (xg)
            v.push_back(xchg_step(c, "xchg_y_L" + std::to_string(l), [c, l] { return (void*)c->L[l].y; }, sizeof(float),
                                  l));
    }
    for (int l = Ld - 2; l >= 0; --l) {
        v.push_back({"net_up_L" + std::to_string(l), [c, l, raw, no](cudaStream_t s) {
                         if (l == 0 && !raw)
                             launch_up0_no<D>(c, s, no);
                         else
                             launch_up<D, kUpMid, 0>(c, s, l, (l == 0) ? c->out_f : c->L[l].out, nullptr, !raw);
                     }});
        if (xg && l > 0)
            v.push_back(xchg_step(c, "xchg_out_L" + std::to_string(l), [c, l] { return (void*)c->L[l].out; },
                                  sizeof(float), l));
    }
    if (!raw && Ld > 1 && !(D == 3 && c->merge_up0))
        v.push_back({"net_mixed_up_L0", [c, no](cudaStream_t s) { launch_mixed_up0_no<D>(c, s, no); }});
    if (Ld == 1 && !raw) {
        v.push_back({"net_out_L0", [c](cudaStream_t s) {
                         LevelBufs& L = c->L[0];
                         const long long nb = L.g.n / ((D == 3) ? 8 : 4);
                         LAUNCH(c, s, (k_up<D, kUpL0Depth1>), nb, L.g, L.g, nullptr, L.y, c->zab, tab_up(c, 0), nullptr,
                                c->Dtmp, c->st, c->ADring, c->partials, c->counter);
                     }});
    }
    return v;
}

// k_down_l0 visits only live units: x_1 must hold zeros elsewhere before a
// solve-path network runs (set_mask and raw-network calls leave it dirty)
void ensure_x1_clean(npsd_b200_ctx* c, cudaStream_t s) {
    if (c->x1_clean || c->dim != 3 || c->depth < 2) return;
    CK(cudaMemsetAsync(c->L[1].x, 0, (size_t)c->L[1].g.n * sizeof(float), s));
    for (int l = 1; l + 1 < c->depth; ++l)
        if (c->clive[l]) {  // outputs of the coarse tiles the solve path skips
            CK(cudaMemsetAsync(c->L[l].y, 0, (size_t)c->L[l].g.n * sizeof(float), s));
            CK(cudaMemsetAsync(c->L[l].out, 0, (size_t)c->L[l].g.n * sizeof(float), s));
            CK(cudaMemsetAsync(c->L[l + 1].x, 0, (size_t)c->L[l + 1].g.n * sizeof(float), s));
        }
    c->x1_clean = true;
}

template <int D>
void launch_network(npsd_b200_ctx* c, cudaStream_t s, bool raw, int* launches) {
    if (raw)
        c->x1_clean = false;
    else
        ensure_x1_clean(c, s);
    const auto steps = network_steps<D>(c, raw, 0);
    for (const auto& st : steps) st.run(s);
    if (launches) *launches = (int)steps.size();
}

// d = P(r / ||r||): the network, IdentityPrecond (cfg precond = 1) or
// JacobiPrecond (2)
template <int D>
std::vector<Step> direction_steps(npsd_b200_ctx* c, int no) {
    if (!c->solve_ident) return network_steps<D>(c, false, no);
    const Geom g = c->g0;
    const bool jac = c->solve_ident == 2;
    return {{jac ? "jacobi_dir" : "ident_dir", [c, g, no, jac](cudaStream_t s) {
                 const uint8_t* cls = c->L[0].cls;
#define NPSD_IDENT(NO_)                                                                                        \
    if (jac)                                                                                                    \
        LAUNCH(c, s, (k_ident_dir<NO_, true>), g.n, g, cls, (const double*)c->R, c->Dtmp, c->st,               \
               (const double*)c->ADring, c->partials, c->counter);                                             \
    else                                                                                                        \
        LAUNCH(c, s, (k_ident_dir<NO_, false>), g.n, g, cls, (const double*)c->R, c->Dtmp, c->st,              \
               (const double*)c->ADring, c->partials, c->counter)
                 switch (no) {
                     case 0: NPSD_IDENT(0); break;
                     case 1: NPSD_IDENT(1); break;
                     case 2: NPSD_IDENT(2); break;
                     case 3: NPSD_IDENT(3); break;
                     case 4: NPSD_IDENT(4); break;
                     default: NPSD_IDENT(8); break;
                 }
#undef NPSD_IDENT
             }}};
}

template <int D>
std::vector<Step> prologue_steps(npsd_b200_ctx* c, cudaGraphConditionalHandle h, int use_cond, int nullspace) {
    std::vector<Step> v;
    const Geom g = c->g0;
    const uint8_t* cls = c->L[0].cls;
    v.push_back({"stamp", [=](cudaStream_t s) { LAUNCH3(c, s, k_stamp_start, dim3(1), dim3(1), c->st); }});
    // projections (solver.cpp:197-201), r0 = b - A x0, ||r0||
    if (nullspace) {
        v.push_back({"proj_b_sum", [=](cudaStream_t s) {
                         LAUNCH(c, s, k_fluid_sum, g.n, g, cls, c->Bf, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
                     }});
        v.push_back({"proj_b_sub", [=](cudaStream_t s) { LAUNCH(c, s, k_subtract_mean, g.n, g, cls, c->Bf, c->st); }});
        v.push_back({"proj_x_sum", [=](cudaStream_t s) {
                         LAUNCH(c, s, k_fluid_sum, g.n, g, cls, c->X0, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
                     }});
        v.push_back({"proj_x_sub", [=](cudaStream_t s) { LAUNCH(c, s, k_subtract_mean, g.n, g, cls, c->X0, c->st); }});
    }
    v.push_back({"residual0", [=](cudaStream_t s) { LAUNCH(c, s, k_residual<D>, g.n, g, cls, c->Bf, c->X0, c->R); }});
    if (nullspace) {
        v.push_back({"proj_r0_sum", [=](cudaStream_t s) {
                         LAUNCH(c, s, k_fluid_sum, g.n, g, cls, c->R, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
                     }});
        v.push_back({"proj_r0_sub", [=](cudaStream_t s) { LAUNCH(c, s, k_subtract_mean, g.n, g, cls, c->R, c->st); }});
    }
    v.push_back({"norm0", [=](cudaStream_t s) {
                     LAUNCH(c, s, k_residual_norm, g.n, g, c->R, c->st, c->hist, c->times, c->partials, c->counter, h,
                            use_cond, 1);
                 }});
    return v;
}

template <int D>
std::vector<Step> body_steps(npsd_b200_ctx* c, cudaGraphConditionalHandle h, int use_cond, int nullspace, int no) {
    std::vector<Step> v = direction_steps<D>(c, no);
    const Geom g = c->g0;
    const uint8_t* cls = c->L[0].cls;
    v.push_back({"ortho", [=](cudaStream_t s) { launch_ortho_no<D>(c, s, no); }});
    v.push_back({"update", [=](cudaStream_t s) { launch_update<D>(c, s, h, use_cond, nullspace ? 0 : 1); }});
    if (nullspace) {
        v.push_back({"proj_r_sum", [=](cudaStream_t s) {
                         LAUNCH(c, s, k_fluid_sum, g.n, g, cls, c->R, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
                     }});
        v.push_back({"proj_r_sub", [=](cudaStream_t s) { LAUNCH(c, s, k_subtract_mean, g.n, g, cls, c->R, c->st); }});
        v.push_back({"norm", [=](cudaStream_t s) {
                         LAUNCH(c, s, k_residual_norm, g.n, g, c->R, c->st, c->hist, c->times, c->partials, c->counter,
                                h, use_cond, 0);
                     }});
    }
    return v;
}

// Tensor maps (tma.cuh) of the stencil kernels' TMA inputs: full-grid f64
// vectors as (nx, ny, local nz) tensors, boxes of one 68 x (SY + 2) tile
// plane (the 64 x SY tile, two columns and one row of halo each side); rebuilt
// whenever one of the vectors moves (the solve graphs hold them by value).
void build_tma_maps(npsd_b200_ctx* c) {
    static PFN_cuTensorMapEncodeTiled encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }();
    if (!c->maps) {
        void* p = nullptr;
        CK(cudaMallocHost(&p, sizeof(TmaMaps)));
        c->maps = static_cast<TmaMaps*>(p);
    }
    std::memset(c->maps, 0, sizeof(TmaMaps));
    if (c->dim != 3) return;
    const Geom& g = c->g0;
    auto make = [&](CUtensorMap* m, const double* base) {
        if (!base) return;
        const cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
        const cuuint64_t strides[2] = {(cuuint64_t)g.nx * sizeof(double), (cuuint64_t)g.nx * g.ny * sizeof(double)};
        const cuuint32_t box[3] = {(cuuint32_t)kVW, (cuuint32_t)(kMarchSY + 2), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    };
    make(&c->maps->m[kMapD], c->Dtmp);
    for (int j = 0; j < c->ring_alloc && j < kRing; ++j) make(&c->maps->m[kMapRing + j], c->Dring + (size_t)j * g.n);
    make(&c->maps->m[kMapX0], c->X0);
    make(&c->maps->m[kMapX1], c->X1);
    ++c->buf_gen;
}

void ensure_ring(npsd_b200_ctx* c, int ring) {
    if (ring <= c->ring_alloc) return;
    const size_t n = (size_t)c->g0.n;
    if (c->Dring) CK(cudaFree(c->Dring));
    if (c->ADring) CK(cudaFree(c->ADring));
    c->Dring = dalloc<double>(n * ring);
    c->ADring = dalloc<double>(n * ring);
    CK(cudaMemsetAsync(c->Dring, 0, n * ring * sizeof(double), c->s));
    CK(cudaMemsetAsync(c->ADring, 0, n * ring * sizeof(double), c->s));
    c->ring_alloc = ring;
    if (c->X1) build_tma_maps(c);
}

void ensure_hist(npsd_b200_ctx* c, long long need) {
    if (need <= c->hist_cap) return;
    if (c->hist) CK(cudaFree(c->hist));
    if (c->times) CK(cudaFree(c->times));
    c->hist = dalloc<double>((size_t)need);
    c->times = dalloc<double>((size_t)need);
    c->hist_cap = need;
}

void ensure_hist_host(npsd_b200_ctx* c, long long need) {
    if (need <= c->hist_host_cap) return;
    if (c->hist_host) CK(cudaFreeHost(c->hist_host));
    if (c->times_host) CK(cudaFreeHost(c->times_host));
    CK(cudaMallocHost(&c->hist_host, (size_t)need * sizeof(double)));
    CK(cudaMallocHost(&c->times_host, (size_t)need * sizeof(double)));
    c->hist_host_cap = need;
}

template <int D>
void capture_solve_graph(npsd_b200_ctx* c, int nullspace, int no) {
    if (c->exec) {
        CK(cudaGraphExecDestroy(c->exec));
        c->exec = nullptr;
    }
    cudaStream_t s = c->s, s2 = c->s2;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
    const auto pro = prologue_steps<D>(c, h, 1, nullspace);
    for (const auto& st : pro) st.run(s);
    // while (!done) { one PSDO iteration }
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, cg, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const auto bod = body_steps<D>(c, h, 1, nullspace, no);
    for (const auto& st : bod) st.run(s2);
    cudaGraph_t body_out = nullptr;
    CK(cudaStreamEndCapture(s2, &body_out));
    cudaGraph_t graph = nullptr;
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(&c->exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    c->exec_key[0] = c->Dring;
    c->exec_key[1] = c->hist;
    c->exec_key[2] = c->ADring;
    c->exec_key[3] = c->partials;
    c->exec_nullspace = nullspace;
    c->exec_no = no;
    c->exec_ident = c->solve_ident;
    c->exec_gen = c->buf_gen;
    c->body_launches = (int)bod.size();
    c->prologue_launches = (int)pro.size();
    c->launches -= (long long)(bod.size() + pro.size());  // captured, not executed
}

long long first_zero_diag_row(npsd_b200_ctx* c);

// Runs the solve on c->Bf / c->X0 (already masked). Returns the status.
template <int D>
int solve_device_impl(npsd_b200_ctx* c, const npsd_b200_solve_cfg* cfg, npsd_b200_report* rep) {
    // stop_threshold / check_inputs (solver.cpp:20-33)
    require(cfg->tol_reduction > 0.0 && cfg->tol_reduction < 1.0, "SolveConfig: tol_reduction must lie in (0,1)");
    require(cfg->n_ortho >= 0, "psdo: n_ortho must be >= 0");
    require(cfg->n_ortho <= kMaxOrtho, "psdo: n_ortho > 8 is not supported by the B200 build");
    require(cfg->precond >= 0 && cfg->precond <= 2, "psdo: precond must be 0 (network), 1 (identity) or 2 (jacobi)");
    if (cfg->precond == 2) {
        const long long row = first_zero_diag_row(c);  // JacobiPrecond's constructor check
        require(row < 0, "jacobi precond: zero diagonal at row " + std::to_string(row));
    }
    c->solve_ident = cfg->precond;
    const long long max_iters = cfg->max_iters < 0 ? 0 : cfg->max_iters;
    const int ring = cfg->n_ortho + 1;
    ensure_ring(c, ring);
    ensure_hist(c, max_iters + 1);
    const int nullspace = cfg->nullspace_projection ? 1 : 0;
    if (!c->exec || c->exec_gen != c->buf_gen || c->exec_key[0] != c->Dring || c->exec_key[1] != c->hist ||
        c->exec_key[2] != c->ADring ||
        c->exec_nullspace != nullspace || c->exec_no != cfg->n_ortho || c->exec_ident != c->solve_ident)
        capture_solve_graph<D>(c, nullspace, cfg->n_ortho);
    SolverState* h = c->st_host;
    std::memset(h, 0, sizeof(SolverState));
    h->tol_reduction = cfg->tol_reduction;
    h->tol_abs = cfg->tol_abs;
    h->max_iters = max_iters;
    h->n_ortho = cfg->n_ortho;
    h->normalize = cfg->normalize_before_precond ? 1 : 0;
    h->nullspace = nullspace;
    h->ring = ring;
    CK(cudaMemcpyAsync(c->st, h, sizeof(SolverState), cudaMemcpyHostToDevice, c->s));
    ensure_x1_clean(c, c->s);
    CK(cudaEventRecord(c->ev0, c->s));
    CK(cudaGraphLaunch(c->exec, c->s));
    CK(cudaEventRecord(c->ev1, c->s));
    CK(cudaMemcpyAsync(h, c->st, sizeof(SolverState), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    const long long iters = h->breakdown ? h->k - 1 : ((h->k > 1) ? h->k - 1 : 0);
    // history entries written: 0..iters (a breakdown stops before entry k)
    const long long hl = iters + 1;
    ensure_hist_host(c, hl);
    CK(cudaMemcpyAsync(c->hist_host, c->hist, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaMemcpyAsync(c->times_host, c->times, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    c->last_launches = c->prologue_launches + (h->breakdown ? (iters * c->body_launches + c->body_launches)
                                                            : iters * c->body_launches);
    c->launches += c->last_launches;
    c->report_hist.assign(c->hist_host, c->hist_host + hl);
    c->report_times.assign(c->times_host, c->times_host + hl);
    if (rep) {
        rep->iterations = iters;
        rep->converged = h->converged;
        rep->breakdown = h->breakdown;
        rep->residual_history = c->report_hist.data();
        rep->cumulative_seconds = c->report_times.data();
        rep->history_len = hl;
        rep->setup_seconds = h->setup_s;
        rep->iterate_seconds = c->last_ms * 1e-3 - h->setup_s;  // solver.cpp:275
        rep->precond_seconds = h->precond_s;
    }
    if (h->breakdown) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "psdo: curvature d'Ad = %f at iteration %lld (||r|| = %f)", h->bad_value,
                      h->k, h->rnorm);
        throw Breakdown(buf);
    }
    return NPSD_OK;
}

// ------------------------------------------------------------ z-slab solve
// One iteration for iteration index k (1-based): the ring slot and the x
// buffer an iteration writes follow from k (head and xcur advance once per
// iteration), so a chunk of lcm(2, ring) * m iterations repeats exactly.
// mean_project over all ranks (vector_ops.cpp:33-43): rank sums and counts,
// rank-ordered totals, subtract
void slab_project(npsd_b200_ctx* c, cudaStream_t s, double* v) {
    const Geom g = c->g0;
    LAUNCH(c, s, k_fluid_sum, g.n, g, c->L[0].cls, v, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
    slab_reduce(c, s, kFinMean);
    LAUNCH(c, s, k_subtract_mean, g.n, g, c->L[0].cls, v, c->st);
}

template <int D>
std::vector<Step> slab_body_steps(npsd_b200_ctx* c, int no, long long k, int ns) {
    std::vector<Step> v = direction_steps<D>(c, no);
    const int R = no + 1;
    const int nw = (int)((R - 1 + k) % R);
    double* dnew = c->Dring + (size_t)nw * (size_t)c->g0.n;
    double* xnew = ((k - 1) & 1) ? c->X0 : c->X1;
    v.push_back(reduce_step(c, "reduce_proj", kFinProj));
    v.push_back(xchg_step(c, "xchg_d", [c] { return (void*)c->Dtmp; }, sizeof(double), 0));
    v.push_back({"ortho", [c, no](cudaStream_t s) { launch_ortho_no<D>(c, s, no); }});
    v.push_back(reduce_step(c, "reduce_ortho", kFinOrtho));
    v.push_back(xchg_step(c, "xchg_dnew", [dnew] { return (void*)dnew; }, sizeof(double), 0));
    if (ns) {  // r = b - A x', mean_project(r), ||r|| (solver.cpp:255-260)
        v.push_back({"update", [c](cudaStream_t s) { launch_update<D>(c, s, 0, 0, 0); }});
        v.push_back({"project_r", [c](cudaStream_t s) { slab_project(c, s, c->R); }});
        v.push_back({"norm", [c](cudaStream_t s) {
                         const Geom g = c->g0;
                         LAUNCH(c, s, k_residual_norm, g.n, g, c->R, c->st, c->hist, c->times, c->partials,
                                c->counter, (cudaGraphConditionalHandle)0, 0, 0);
                     }});
    } else {
        v.push_back({"update", [c](cudaStream_t s) { launch_update<D>(c, s, 0, 0, 1); }});
    }
    v.push_back(reduce_step(c, "reduce_update", kFinUpdate));
    v.push_back(xchg_step(c, "xchg_xnew", [xnew] { return (void*)xnew; }, sizeof(double), 0));
    v.push_back(xchg_step(c, "xchg_r", [c] { return (void*)c->R; }, sizeof(double), 0));
    return v;
}

int slab_chunk(int ring) {
    const int p = (ring % 2 == 0) ? ring : 2 * ring;  // lcm(2, ring)
    return p * ((12 + p - 1) / p);
}

// psdo_solve over a z-slab (c->Bf / c->X0 set on the owned planes). The
// iterations run in chunks — one captured graph of slab_chunk() iterations per
// launch for NCCL ranks, eager steps for the in-process communicator — with
// every iteration kernel returning at once after the solve has finished.
template <int D>
int slab_solve_impl(npsd_b200_ctx* c, const npsd_b200_solve_cfg* cfg, npsd_b200_report* rep) {
    require(cfg->tol_reduction > 0.0 && cfg->tol_reduction < 1.0, "SolveConfig: tol_reduction must lie in (0,1)");
    require(cfg->n_ortho >= 0, "psdo: n_ortho must be >= 0");
    require(cfg->n_ortho <= kMaxOrtho, "psdo: n_ortho > 8 is not supported by the B200 build");
    require(cfg->precond == 0 || cfg->precond == 1, "psdo: precond must be 0 (network) or 1 (identity) on a z-slab");
    c->solve_ident = cfg->precond;
    cudaStream_t s = c->s;
    const long long max_iters = cfg->max_iters < 0 ? 0 : cfg->max_iters;
    const int no = cfg->n_ortho, ring = no + 1;
    ensure_ring(c, ring);
    ensure_hist(c, max_iters + 1);
    SolverState* h = c->st_host;
    std::memset(h, 0, sizeof(SolverState));
    h->tol_reduction = cfg->tol_reduction;
    h->tol_abs = cfg->tol_abs;
    h->max_iters = max_iters;
    h->n_ortho = no;
    h->normalize = cfg->normalize_before_precond ? 1 : 0;
    h->ring = ring;
    h->dist = 1;
    const int ns = cfg->nullspace_projection ? 1 : 0;
    h->nullspace = ns;
    CK(cudaMemcpyAsync(c->st, h, sizeof(SolverState), cudaMemcpyHostToDevice, s));
    ensure_x1_clean(c, s);
    const Geom g = c->g0;
    const uint8_t* cls = c->L[0].cls;
    CK(cudaEventRecord(c->ev0, s));
    LAUNCH3(c, s, k_stamp_start, dim3(1), dim3(1), c->st);
    // prologue: [projections of b and x0], r0 = b - A x0 (x0's ghosts first),
    // [projection of r0], ||r0|| over all ranks (solver.cpp:197-209)
    if (ns) {
        slab_project(c, s, c->Bf);
        slab_project(c, s, c->X0);
    }
    slab_exchange(c, s, c->X0, sizeof(double), 0);
    LAUNCH(c, s, k_residual<D>, g.n, g, cls, c->Bf, c->X0, c->R);
    if (ns) slab_project(c, s, c->R);
    LAUNCH(c, s, k_residual_norm, g.n, g, c->R, c->st, c->hist, c->times, c->partials, c->counter,
           (cudaGraphConditionalHandle)0, 0, 1);
    slab_reduce(c, s, kFinNorm0);
    slab_exchange(c, s, c->R, sizeof(double), 0);
    // chunks: K iterations, or P (the ring period) when the residual's decay
    // predicts the end within P iterations — fewer dead iterations after
    // convergence (their kernels return at once; their exchanges still run)
    const int K = slab_chunk(ring), P = (ring % 2 == 0) ? ring : 2 * ring;
    bool graph = c->slab.comm->capturable() && !c->slab_no_graph;
    auto capture = [&](int kc, cudaGraphExec_t& exec, long long& nlaunch) {
        if (exec) CK(cudaGraphExecDestroy(exec));
        exec = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const long long before = c->launches;
        try {
            for (long long k = 1; k <= kc; ++k)
                for (const auto& st : slab_body_steps<D>(c, no, k, ns)) st.run(s);
            nlaunch = c->launches - before;  // kernels per chunk replay
            c->launches = before;            // captured, not executed
        } catch (...) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(s, &junk);
            if (junk) cudaGraphDestroy(junk);
            throw;
        }
        cudaGraph_t gr = nullptr;
        CK(cudaStreamEndCapture(s, &gr));
        const cudaError_t ie = cudaGraphInstantiate(&exec, gr, 0);
        cudaGraphDestroy(gr);
        CK(ie);
    };
    if (graph && (!c->slab_exec || c->slab_exec_gen != c->buf_gen || c->slab_exec_no != no ||
                  c->slab_exec_ns != ns || c->slab_exec_ident != cfg->precond ||
                  c->exec_key[0] != c->Dring || c->exec_key[1] != c->hist ||
                  c->exec_key[2] != c->ADring)) {
        // the chunks: iterations of kernels and NCCL calls in one graph each; if
        // the capture is refused, the chunks run as eager launches instead
        CK(cudaStreamSynchronize(s));
        try {
            capture(K, c->slab_exec, c->slab_chunk_launches);
            capture(P, c->slab_exec_short, c->slab_short_launches);
            c->slab_exec_no = no;
            c->slab_exec_ns = ns;
            c->slab_exec_ident = cfg->precond;
            c->slab_exec_gen = c->buf_gen;
            c->exec_key[0] = c->Dring;
            c->exec_key[1] = c->hist;
            c->exec_key[2] = c->ADring;
        } catch (const std::exception&) {
            cudaGetLastError();
            c->slab_exec = nullptr;
            c->slab_no_graph = true;
            graph = false;
        }
    }
    double prev_rn = 0.0;
    int prev_kc = 0;
    for (long long k0 = 1;;) {
        CK(cudaMemcpyAsync(h, c->st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (h->done) break;
        int kc = K;
        if (prev_kc > 0 && prev_rn > 0.0 && h->rnorm > 0.0 && h->rnorm < prev_rn) {
            const double rate = std::pow(h->rnorm / prev_rn, 1.0 / prev_kc);  // per-iteration decay
            const double left = std::log(h->thr / h->rnorm) / std::log(rate);
            if (left <= P) kc = P;
        }
        prev_rn = h->rnorm;
        prev_kc = kc;
        if (graph) {
            CK(cudaGraphLaunch(kc == K ? c->slab_exec : c->slab_exec_short, s));
            c->launches += (kc == K) ? c->slab_chunk_launches : c->slab_short_launches;
        } else {
            for (long long k = k0; k < k0 + kc; ++k)
                for (const auto& st : slab_body_steps<D>(c, no, k, ns)) st.run(s);
        }
        k0 += kc;
    }
    CK(cudaEventRecord(c->ev1, s));
    CK(cudaMemcpyAsync(h, c->st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    const long long iters = h->breakdown ? h->k - 1 : ((h->k > 1) ? h->k - 1 : 0);
    const long long hl = iters + 1;
    ensure_hist_host(c, hl);
    CK(cudaMemcpyAsync(c->hist_host, c->hist, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->times_host, c->times, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->report_hist.assign(c->hist_host, c->hist_host + hl);
    c->report_times.assign(c->times_host, c->times_host + hl);
    if (rep) {
        rep->iterations = iters;
        rep->converged = h->converged;
        rep->breakdown = h->breakdown;
        rep->residual_history = c->report_hist.data();
        rep->cumulative_seconds = c->report_times.data();
        rep->history_len = hl;
        rep->setup_seconds = h->setup_s;
        rep->iterate_seconds = c->last_ms * 1e-3 - h->setup_s;  // solver.cpp:275
        rep->precond_seconds = h->precond_s;
    }
    if (h->breakdown) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "psdo: curvature d'Ad = %f at iteration %lld (||r|| = %f)", h->bad_value,
                      h->k, h->rnorm);
        throw Breakdown(buf);
    }
    return NPSD_OK;
}

// true when the device check kernel found nothing (one 4-byte readback)
template <typename K, typename... Args>
bool device_check(npsd_b200_ctx* c, K kernel, long long items, Args... args) {
    unsigned int* flag = c->check_flag;
    CK(cudaMemsetAsync(flag, 0, sizeof(unsigned int), c->s));
    LAUNCH(c, c->s, kernel, items, args..., flag);
    unsigned int h = 0;
    CK(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return h == 0;
}

// ------------------------------------------------------------------- pcg
// pcg_solve (solver.cpp:36-102) on the device: identity (cg_solve) or Jacobi.
long long first_zero_diag_row(npsd_b200_ctx* c) {
    unsigned int* d = reinterpret_cast<unsigned int*>(c->red_b);
    const unsigned int none = 0xffffffffu;
    CK(cudaMemcpyAsync(d, &none, sizeof none, cudaMemcpyHostToDevice, c->s));
    LAUNCH(c, c->s, k_zero_diag, c->g0.n, c->g0, c->L[0].cls, c->fmask, c->fbase, d);
    unsigned int row = none;
    CK(cudaMemcpyAsync(&row, d, sizeof row, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return row == none ? -1 : (long long)row;
}

// ---- IC0 (precond.cpp:28-112): level-scheduled factor and sweeps
inline int ic0_levels(const Geom& g) { return (g.nx - 1) + (g.ny - 1) + (g.nz - 1) + 1; }

// one sweep (MODE 0 factor, 1 forward, 2 backward) as one launch per hyperplane
template <int MODE>
void ic0_sweep(npsd_b200_ctx* c, cudaStream_t s, double shift, const double* r, const SolverState* st) {
    const Geom g = c->g0;
    const int nl = ic0_levels(g);
    const int blocks = (int)(((long long)g.ny * g.nz + kBlock - 1) / kBlock);
    for (int i = 0; i < nl; ++i) {
        const int h = (MODE == 2) ? nl - 1 - i : i;
        k_ic0_level<MODE><<<blocks, kBlock, 0, s>>>(g, c->L[0].cls, h, shift, c->icD, r, c->cgZ, c->icFail, st);
        CK(cudaGetLastError());
        ++c->launches;
    }
}

// Ic0Precond's constructor: factor with shift 0, then 1e-3 * mean diagonal,
// doubling, at most 5 retries (precond.cpp:28-46); throws like the reference
void ic0_factor(npsd_b200_ctx* c) {
    cudaStream_t s = c->s;
    if (!c->icD) {
        c->icD = dalloc<double>((size_t)c->g0.n);
        c->icFail = dalloc<int>(4);  // [0] failure flag, [2..3] diagonal sum
    }
    // sum of the diagonal over fluid rows: small integers, exact in any order
    unsigned long long* dsum = reinterpret_cast<unsigned long long*>(c->icFail + 2);
    CK(cudaMemsetAsync(c->icFail, 0, 4 * sizeof(int), s));
    LAUNCH(c, s, k_diag_sum, c->g0.n, c->g0, c->L[0].cls, dsum);
    unsigned long long sum = 0;
    CK(cudaMemcpyAsync(&sum, dsum, sizeof sum, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double diag_mean = (double)sum / (double)std::max<long long>(c->n_fluid, 1);
    double shift = 0.0;
    for (int attempt = 0; attempt <= 5; ++attempt) {
        CK(cudaMemsetAsync(c->icFail, 0, sizeof(int), s));
        ic0_sweep<0>(c, s, shift, nullptr, nullptr);
        int fail = 0;
        CK(cudaMemcpyAsync(&fail, c->icFail, sizeof fail, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (!fail) {
            c->ic0_shift_retries = attempt;
            return;
        }
        shift = (shift == 0.0) ? 1e-3 * diag_mean : 2.0 * shift;
    }
    throw InvalidArgument("ic0: factorization failed after diagonal-shift retries");
}

template <int D, int M>
void capture_cg_graph(npsd_b200_ctx* c, int ns) {
    if (c->cg_exec) {
        CK(cudaGraphExecDestroy(c->cg_exec));
        c->cg_exec = nullptr;
    }
    cudaStream_t s = c->s, s2 = c->s2;
    const Geom g = c->g0;
    const uint8_t* cls = c->L[0].cls;
    double* z = (M != kCgIdentity) ? c->cgZ : c->R;
    const long long before = c->launches;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
    // mean_project(v) (vector_ops.cpp:33-43) as two kernels
    auto project = [&](cudaStream_t st, double* v) {
        LAUNCH(c, st, k_fluid_sum, g.n, g, cls, v, (const uint32_t*)(c->fbase + c->L[0].nseg), c->st, c->partials, c->counter);
        LAUNCH(c, st, k_subtract_mean, g.n, g, cls, v, c->st);
    };
    // prologue (solver.cpp:38-58): [projections of b, x0], r0 = b - A x0,
    // [projection of r0], z0 = M r0, ||r0||, r0.z0
    LAUNCH3(c, s, k_stamp_start, dim3(1), dim3(1), c->st);
    if (ns) {
        project(s, c->Bf);
        project(s, c->X0);
    }
    LAUNCH(c, s, k_residual<D>, g.n, g, cls, c->Bf, c->X0, c->R);
    if (ns) project(s, c->R);
    LAUNCH(c, s, (k_cg_update<M, true>), g.n, g, cls, c->cgP0, c->cgP1, c->cgAp, c->X0, c->R, z, c->st, c->hist,
           c->times, c->partials, c->counter, h, M == kCgIc0 ? 0 : 1);
    if (M == kCgIc0) {
        ic0_sweep<1>(c, s, 0.0, c->R, c->st);
        ic0_sweep<2>(c, s, 0.0, c->R, c->st);
        LAUNCH(c, s, k_cg_rz<true>, g.n, g, cls, c->R, c->cgZ, c->st, c->partials, c->counter, h, 1);
    }
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, cg, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    {
        auto k = k_cg_dir<D>;
        const size_t sm = march_smem_bytes<CgOp>();
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        LAUNCH3S(c, s2, k, dim3(wave_blocks(c, k, kSX * kSY, sm)), dim3(kSX, kSY), sm, g, cls, (const double*)z,
                 c->cgP0, c->cgP1, c->cgAp, c->st, c->partials, c->counter, c->sch_stencil.view());
        if (ns) {  // x, r axpys; mean_project(r) (solver.cpp:82); the rest on the projected r
            LAUNCH(c, s2, (k_cg_update<M, false, 1>), g.n, g, cls, c->cgP0, c->cgP1, c->cgAp, c->X0, c->R, z, c->st,
                   c->hist, c->times, c->partials, c->counter, h, M == kCgIc0 ? 0 : 1);
            project(s2, c->R);
            LAUNCH(c, s2, (k_cg_update<M, false, 2>), g.n, g, cls, c->cgP0, c->cgP1, c->cgAp, c->X0, c->R, z, c->st,
                   c->hist, c->times, c->partials, c->counter, h, M == kCgIc0 ? 0 : 1);
        } else {
            LAUNCH(c, s2, (k_cg_update<M, false>), g.n, g, cls, c->cgP0, c->cgP1, c->cgAp, c->X0, c->R, z, c->st,
                   c->hist, c->times, c->partials, c->counter, h, M == kCgIc0 ? 0 : 1);
        }
        if (M == kCgIc0) {
            ic0_sweep<1>(c, s2, 0.0, c->R, c->st);
            ic0_sweep<2>(c, s2, 0.0, c->R, c->st);
            LAUNCH(c, s2, k_cg_rz<false>, g.n, g, cls, c->R, c->cgZ, c->st, c->partials, c->counter, h, 1);
        }
    }
    cudaGraph_t body_out = nullptr;
    CK(cudaStreamEndCapture(s2, &body_out));
    cudaGraph_t graph = nullptr;
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(&c->cg_exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    c->launches = before;
    c->cg_exec_ns = ns;
    c->cg_exec_kind = M;
    c->cg_exec_gen = c->buf_gen;
    c->cg_exec_key = c->hist;
}

// the solve on c->Bf / c->X0 (masked); x ends in c->X0
int pcg_solve_impl(npsd_b200_ctx* c, const npsd_b200_solve_cfg* cfg, int precond, npsd_b200_report* rep) {
    require(cfg->tol_reduction > 0.0 && cfg->tol_reduction < 1.0, "SolveConfig: tol_reduction must lie in (0,1)");
    require(precond >= 0 && precond <= 2, "pcg: preconditioner must be 0 (identity), 1 (jacobi) or 2 (ic0)");
    require(!c->slab.on, "pcg: not available on a z-slab context");
    cudaStream_t s = c->s;
    const Geom g = c->g0;
    const size_t nb = (size_t)g.n * sizeof(double);
    if (!c->cgP0) {
        c->cgP0 = dalloc<double>((size_t)g.n);
        c->cgP1 = dalloc<double>((size_t)g.n);
        c->cgAp = dalloc<double>((size_t)g.n);
        c->cgZ = dalloc<double>((size_t)g.n);
        ++c->buf_gen;
    }
    if (precond == 1) {
        // JacobiPrecond: a fluid cell without a non-solid neighbour has no diagonal
        const long long row = first_zero_diag_row(c);
        require(row < 0, "jacobi precond: zero diagonal at row " + std::to_string(row));
    }
    if (precond == 2) ic0_factor(c);  // Ic0Precond(A): per solve, on this frame
    const long long max_iters = cfg->max_iters < 0 ? 0 : cfg->max_iters;
    ensure_hist(c, max_iters + 1);
    // the zero invariant of the directions, A p and z on this frame
    for (double* v : {c->cgP0, c->cgP1, c->cgAp, c->cgZ}) CK(cudaMemsetAsync(v, 0, nb, s));
    const int ns = cfg->nullspace_projection ? 1 : 0;
    if (!c->cg_exec || c->cg_exec_kind != precond || c->cg_exec_gen != c->buf_gen || c->cg_exec_key != c->hist ||
        c->cg_exec_ns != ns) {
        if (c->dim == 3) {
            if (precond == 0) capture_cg_graph<3, kCgIdentity>(c, ns);
            else if (precond == 1) capture_cg_graph<3, kCgJacobi>(c, ns);
            else capture_cg_graph<3, kCgIc0>(c, ns);
        } else {
            if (precond == 0) capture_cg_graph<2, kCgIdentity>(c, ns);
            else if (precond == 1) capture_cg_graph<2, kCgJacobi>(c, ns);
            else capture_cg_graph<2, kCgIc0>(c, ns);
        }
    }
    SolverState* h = c->st_host;
    std::memset(h, 0, sizeof(SolverState));
    h->tol_reduction = cfg->tol_reduction;
    h->tol_abs = cfg->tol_abs;
    h->max_iters = max_iters;
    CK(cudaMemcpyAsync(c->st, h, sizeof(SolverState), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(c->ev0, s));
    CK(cudaGraphLaunch(c->cg_exec, s));
    CK(cudaEventRecord(c->ev1, s));
    CK(cudaMemcpyAsync(h, c->st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    const long long iters = h->breakdown ? h->k - 1 : ((h->k > 1) ? h->k - 1 : 0);
    const long long hl = iters + 1;
    ensure_hist_host(c, hl);
    CK(cudaMemcpyAsync(c->hist_host, c->hist, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->times_host, c->times, (size_t)hl * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->report_hist.assign(c->hist_host, c->hist_host + hl);
    c->report_times.assign(c->times_host, c->times_host + hl);
    const long long sweeps = (precond == 2) ? 2LL * ic0_levels(g) + 1 : 0;  // per preconditioner apply
    c->last_launches = 3 + 6 * ns + sweeps + (2 + 3 * ns + sweeps) * iters;
    c->launches += c->last_launches;
    if (rep) {
        rep->iterations = iters;
        rep->converged = h->converged;
        rep->breakdown = h->breakdown;
        rep->residual_history = c->report_hist.data();
        rep->cumulative_seconds = c->report_times.data();
        rep->history_len = hl;
        rep->setup_seconds = h->setup_s;
        rep->iterate_seconds = c->last_ms * 1e-3 - h->setup_s;  // solver.cpp:275
        rep->precond_seconds = h->precond_s;
    }
    if (h->breakdown) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "pcg: non-positive curvature p'Ap = %f at iteration %lld", h->bad_value, h->k);
        throw Breakdown(buf);
    }
    return NPSD_OK;
}

int solve_any(npsd_b200_ctx* c, const npsd_b200_solve_cfg* cfg, npsd_b200_report* rep) {
    if (c->slab.on) return slab_solve_impl<3>(c, cfg, rep);
    return (c->dim == 3) ? solve_device_impl<3>(c, cfg, rep) : solve_device_impl<2>(c, cfg, rep);
}

template <typename Fn>
int guarded(npsd_b200_ctx* c, Fn&& fn) {
    if (!c) return NPSD_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(c->mu);
    try {
        CK(cudaSetDevice(c->dev));
        fn();
        c->err.clear();
        return NPSD_OK;
    } catch (const InvalidArgument& e) {
        c->err = e.what();
        return NPSD_INVALID_ARGUMENT;
    } catch (const Breakdown& e) {
        c->err = e.what();
        return NPSD_BREAKDOWN;
    } catch (const EmptySystem& e) {
        c->err = e.what();
        return NPSD_EMPTY_SYSTEM;
    } catch (const std::exception& e) {
        c->err = e.what();
        return NPSD_CUDA_ERROR;
    }
}

// host API calls that need the frame's sizes: the last set_mask finished
void check_mask(npsd_b200_ctx* c) {
    require(c->mask_ok, "npsd_b200: set_mask has not been called");
    setup_sync(c);
}

// device-resident calls: the frame may still be in flight (setup_sync after)
void check_mask_async(const npsd_b200_ctx* c) {
    require(c->mask_ok, "npsd_b200: set_mask has not been called");
}

// A device-resident call after an asynchronous set_mask: run it, then finish
// the set_mask; when the frame had to be redone with larger tables, run it
// again (the first run saw the smaller tables; it may even have failed).
// The reference's EmptySystemError comes last, from the frame's sizes.
template <typename Fn>
void run_after_setup(npsd_b200_ctx* c, Fn&& fn) {
    const bool pending = c->setup_pending;
    bool again = false;
    try {
        fn();
    } catch (const InvalidArgument&) {
        throw;
    } catch (...) {
        if (!(pending && setup_sync(c))) throw;
        again = true;
    }
    if (!again && setup_sync(c)) again = true;
    if (c->n_fluid == 0) throw EmptySystem("reduce: image has no fluid cells");
    if (again) fn();
}

void free_ctx(npsd_b200_ctx* c) {
    auto F = [](void* p) {
        if (p) cudaFree(p);
    };
    F(c->slab.all);
    F(c->slab.allu);
    F(c->mac);
    F(c->check_flag);
    F(c->cgP0);
    F(c->cgP1);
    F(c->cgAp);
    F(c->cgZ);
    F(c->icD);
    F(c->htk);
    F(c->htv);
    F(c->icFail);
    if (c->cg_exec) cudaGraphExecDestroy(c->cg_exec);
    if (c->slab_exec) cudaGraphExecDestroy(c->slab_exec);
    if (c->slab_exec_short) cudaGraphExecDestroy(c->slab_exec_short);
    for (SchedBufs* sb : {&c->sch_stencil, &c->sch_march, &c->sch_down0}) {
        F(sb->pre);
        F(sb->zlo);
        F(sb->len);
        F(sb->first);
        F(sb->last);
    }
    for (int l = 1; l < kMaxDepth; ++l) {  // carved from the L2 pool
        LevelBufs& L = c->L[l];
        L.cls = nullptr;
        L.rcode = nullptr;
        L.y = nullptr;
        L.x = nullptr;
        L.out = nullptr;
    }
    F(c->l2pool);
    for (auto& L : c->L) {
        F(L.cls);
        F(L.mmask);
        F(L.mbase);
        F(L.mcount);
        F(L.img);
        F(L.tab_down);
        F(L.tab_up);
        F(L.kc_down);
        F(L.kc_up);
        F(L.y);
        F(L.x);
        F(L.out);
        F(L.zG);
        F(L.mlist);
        F(L.rcode);
        F(L.pid);
    }
    F(c->d_params);
    F(c->zab);
    F(c->fmask);
    F(c->fmask_prev);
    F(c->fbase);
    F(c->fcount);
    F(c->tflags);
    for (void* p : {(void*)c->dkeys, (void*)c->dvals, (void*)c->pid0, (void*)c->repcell0, (void*)c->npat0,
                    (void*)c->dlist0, (void*)c->dkid0, (void*)c->ulist0, (void*)c->ukid0, (void*)c->crep, (void*)c->cnpat, (void*)c->dmask, (void*)c->dcount,
                    (void*)c->dbase, (void*)c->umask, (void*)c->ucount, (void*)c->ubase, (void*)c->d_info,
                    (void*)c->types_dev})
        F(p);
    if (c->info_host) cudaFreeHost(c->info_host);
    if (c->maps) cudaFreeHost(c->maps);
    for (auto p : c->clive)
        if (p) cudaFree(p);
    if (c->ev_setup) cudaEventDestroy(c->ev_setup);
    if (c->ev_pre_mask) cudaEventDestroy(c->ev_pre_mask);
    if (c->ev_up) cudaEventDestroy(c->ev_up);
    if (c->s_up) cudaStreamDestroy(c->s_up);
    if (c->mask_exec) cudaGraphExecDestroy(c->mask_exec);
    F(c->X0);
    F(c->X1);
    F(c->R);
    F(c->Bf);
    F(c->Dtmp);
    F(c->Dring);
    F(c->ADring);
    F(c->st);
    F(c->partials);
    F(c->counter);
    F(c->hist);
    F(c->times);
    F(c->red_a);
    F(c->red_b);
    F(c->xin_f);
    F(c->out_f);
    for (void* p : c->cub_tmp) F(p);
    for (auto x : c->sx)
        if (x) cudaStreamDestroy(x);
    for (auto e : c->evf)
        if (e) cudaEventDestroy(e);
    if (c->st_host) cudaFreeHost(c->st_host);
    if (c->hist_host) cudaFreeHost(c->hist_host);
    if (c->times_host) cudaFreeHost(c->times_host);
    if (c->exec) cudaGraphExecDestroy(c->exec);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->s) cudaStreamDestroy(c->s);
    if (c->s2) cudaStreamDestroy(c->s2);
}

void do_set_params(npsd_b200_ctx* c, const float* params, size_t n) {
    require(params != nullptr, "npsd_b200: params is null");
    require(n == param_count_impl(c->dim, c->depth), "npsd_b200: parameter count mismatch");
    c->params.assign(params, params + n);
    if (c->dim == 3)
        upload_params_and_kconst<3>(c);
    else
        upload_params_and_kconst<2>(c);
    c->mask_ok = false;  // tables depend on the weights
    ++c->buf_gen;        // captured graphs hold the uniform-window kernels by value
}

}  // namespace

// =====================================================================  C ABI
extern "C" {

size_t npsd_b200_param_count(int dim, int depth) {
    if ((dim != 2 && dim != 3) || depth < 1) return 0;
    return param_count_impl(dim, depth);
}

namespace {

// One context: the whole grid, or (slab != nullptr) one rank's z-slab.
int create_impl(int dim, int nx, int ny, int nz, int depth, const float* params, size_t n_params, int device,
                const SlabInfo* slab, npsd_b200_ctx** out) {
    if (!out) return NPSD_INVALID_ARGUMENT;
    *out = nullptr;
    npsd_b200_ctx* c = new npsd_b200_ctx();
    try {
        require(dim == 2 || dim == 3, "npsd_b200: dim must be 2 or 3");
        require(depth >= 1 && depth <= kMaxDepth, "NetContext: depth must be >= 1 (and <= 8 here)");
        if (dim == 2) nz = 1;
        require(nx > 0 && ny > 0 && nz > 0, "IndicatorImage: dims must be positive");
        const long long div = 1LL << depth;
        require(nx % div == 0 && ny % div == 0 && (dim == 2 || nz % div == 0),
                "NetContext: dims " + std::to_string(nx) + "x" + std::to_string(ny) +
                    (dim == 3 ? "x" + std::to_string(nz) : std::string()) + " not divisible by 2^" +
                    std::to_string(depth));
        c->dim = dim;
        c->depth = depth;
        c->S = (dim == 3) ? 27 : 9;
        c->dev = device;
        if (const char* e = std::getenv("NPSD_PDL")) c->pdl = (e[0] != '0');
        if (const char* e = std::getenv("NPSD_PDL_MASK")) c->pdl_mask = (unsigned)std::strtoul(e, nullptr, 0);
        if (const char* e = std::getenv("NPSD_MERGE_UP0")) c->merge_up0 = (e[0] != '0');
        if (const char* e = std::getenv("NPSD_CLASSIFY_SIMD")) c->classify_simd = (e[0] != '0');
        if (const char* e = std::getenv("NPSD_COARSE_SKIP")) c->coarse_skip = (e[0] != '0');
        if (const char* e = std::getenv("NPSD_PDL_COARSE")) c->pdl_coarse = (e[0] != '0');
        if (const char* e = std::getenv("NPSD_UP0_MIXB")) c->up0_mixb = std::max(0, std::min(16, std::atoi(e)));
        if (slab) {
            c->slab = *slab;
            for (int l = 0; l < depth; ++l) c->slab.ghost[l] = 1 << (depth - 1 - l);
        }
        for (int l = 0; l < depth; ++l)
            c->gglob[l] = make_geom(nx >> l, ny >> l, (dim == 3) ? (nz >> l) : 1);
        c->g0 = level_geom(c, 0);
        require(c->g0.n < (1LL << 31) * 16, "npsd_b200: grid too large");
        CK(cudaSetDevice(c->dev));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->dev));
        CK(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking));
        CK(cudaEventCreate(&c->ev0));
        CK(cudaEventCreate(&c->ev1));
        compute_offsets(c);
        c->d_params = dalloc<float>(param_count_impl(dim, depth));
        // L2-resident pool: the per-cell arrays of levels >= 1 (class bytes, row
        // codes, x, y, out; ~2.3 B x n_c at depth 4) live in one allocation that
        // an access-policy window keeps persisting in L2, so the coarse levels'
        // latency chains hit L2 instead of DRAM after the L0 phases stream
        {
            size_t bytes = 0;
            auto add = [&](size_t b) { bytes += (b + 255) & ~(size_t)255; };
            for (int l = 1; l < depth; ++l) {
                const size_t n = (size_t)level_geom(c, l).n;
                add(n);                                         // cls
                add(4 * n);                                     // rcode
                add(4 * n);                                     // y
                add(4 * n);                                     // x
                if (l < depth - 1) add(4 * n);                  // out
            }
            if (bytes) {
                CK(cudaMalloc(&c->l2pool, bytes));
                // zero: the z-slab ghost planes at the domain faces are never
                // written and must read as the zero outside of the domain
                CK(cudaMemset(c->l2pool, 0, bytes));
                c->l2pool_bytes = bytes;
            }
        }
        size_t pool_off = 0;
        auto carve = [&](size_t b) {
            void* p = c->l2pool + pool_off;
            pool_off += (b + 255) & ~(size_t)255;
            return p;
        };
        for (int l = 0; l < depth; ++l) {
            LevelBufs& L = c->L[l];
            L.g = level_geom(c, l);
            L.nseg = (L.g.n + 31) / 32;
            const size_t nl = (size_t)L.g.n;
            if (l > 0) {
                L.cls = static_cast<uint8_t*>(carve(nl));
                L.rcode = static_cast<uint32_t*>(carve(4 * nl));
                L.y = static_cast<float*>(carve(4 * nl));
                L.x = static_cast<float*>(carve(4 * nl));
                if (l < depth - 1) L.out = static_cast<float*>(carve(4 * nl));
            } else {
                L.cls = dalloc<uint8_t>(nl);
            }
            // counts and bases carry one trailing entry: count 0, so the scan
            // leaves the total in base[nseg] (mcnt points there)
            L.mmask = dalloc<uint32_t>((size_t)L.nseg);
            L.mbase = dalloc<uint32_t>((size_t)L.nseg + 1);
            L.mcount = dalloc<uint32_t>((size_t)L.nseg + 1);
            CK(cudaMemset(L.mcount, 0, ((size_t)L.nseg + 1) * sizeof(uint32_t)));
            if (l > 0) L.img = dalloc<float>(3 * (size_t)L.g.n);
            // kernel-row tables: allocated at the capacities set_mask uses (ensure_setup_capacity)
            L.mlist = dalloc<uint32_t>((size_t)L.g.n);
            if (l > 0) L.pid = dalloc<uint32_t>((size_t)L.g.n);
            L.mcnt = L.mbase + L.nseg;
            L.kc_down = dalloc<float>(3 * (size_t)c->S);
            L.kc_up = dalloc<float>(3 * (size_t)c->S);
            if (l == 0) {
                L.y = dalloc<float>((size_t)L.g.n);
                CK(cudaMemset(L.y, 0, (size_t)L.g.n * sizeof(float)));
            }
            L.zG = dalloc<unsigned long long>(81);
        }
        if (c->l2pool) {
            int maxp = 0, maxw = 0;
            CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, c->dev));
            CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, c->dev));
            if (maxp > 0 && maxw > 0) {
                size_t cur = 0;
                CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
                const size_t want = std::min(c->l2pool_bytes, (size_t)maxp);
                if (want > cur) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
                CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
                const size_t win = std::min(c->l2pool_bytes, (size_t)maxw);
                cudaStreamAttrValue v = {};
                v.accessPolicyWindow.base_ptr = c->l2pool;
                v.accessPolicyWindow.num_bytes = win;
                v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)cur / (double)win);
                v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                CK(cudaStreamSetAttribute(c->s, cudaStreamAttributeAccessPolicyWindow, &v));
                CK(cudaStreamSetAttribute(c->s2, cudaStreamAttributeAccessPolicyWindow, &v));
                // set_mask's branches (created below) take the window in ctx_create's stream loop
                c->apw = v;
                c->apw_on = true;
            }
        }
        c->zab = dalloc<float>(2 * (size_t)depth);
        CK(cudaMemset(c->zab, 0, 2 * (size_t)depth * sizeof(float)));
        const long long nseg0 = c->L[0].nseg;
        c->fmask = dalloc<uint32_t>((size_t)nseg0);
        c->fmask_prev = dalloc<uint32_t>((size_t)nseg0);
        CK(cudaMemset(c->fmask_prev, 0, (size_t)nseg0 * sizeof(uint32_t)));
        c->fbase = dalloc<uint32_t>((size_t)nseg0 + 1);
        c->fcount = dalloc<uint32_t>((size_t)nseg0 + 1);
        CK(cudaMemset(c->fcount, 0, ((size_t)nseg0 + 1) * sizeof(uint32_t)));
        c->tf_ntx = (nx + kFlagTX - 1) / kFlagTX;
        c->tf_nty = (ny + kFlagTY - 1) / kFlagTY;
        // every local plane: a z-slab's ghost planes are flagged too (k_classify_march, k_tile_flags)
        c->tflags = dalloc<uint8_t>((size_t)c->tf_ntx * c->tf_nty * c->L[0].g.nz);
        {  // window keys of every level, and the coarse levels' pattern representatives
            size_t nk = 0, nr = 0;
            for (int l = 0; l < depth; ++l) {
                c->koff[l] = nk;
                nk += (size_t)c->L[l].g.n;
                c->roff[l] = nr;
                if (l > 0) nr += (size_t)c->L[l].g.n;
            }
            c->dkeys = dalloc<unsigned long long>(nk);
            c->dvals = dalloc<uint32_t>(nk);
            c->crep = dalloc<uint32_t>(std::max<size_t>(nr, 1));
            c->cnpat = dalloc<uint32_t>((size_t)kMaxDepth);
        }
        if (const char* e = std::getenv("NPSD_SETUP_SERIAL")) c->setup_par = (e[0] == '0');
        if (c->slab.on) c->setup_par = false;  // the communicator's exchanges run on the main stream
        for (auto& x : c->sx) {
            CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            if (c->apw_on) CK(cudaStreamSetAttribute(x, cudaStreamAttributeAccessPolicyWindow, &c->apw));
        }
        for (auto& e : c->evf) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (uint32_t** v : {&c->dmask, &c->dcount, &c->dbase, &c->umask, &c->ucount, &c->ubase}) {
            *v = dalloc<uint32_t>((size_t)nseg0 + 1);
            CK(cudaMemset(*v, 0, ((size_t)nseg0 + 1) * sizeof(uint32_t)));
        }
        c->dcnt0 = c->dbase + nseg0;  // the scans' trailing totals
        c->ucnt0 = c->ubase + nseg0;
        c->d_info = dalloc<SetupInfo>(1);
        CK(cudaMallocHost(&c->info_host, sizeof(SetupInfo)));
        CK(cudaEventCreateWithFlags(&c->ev_setup, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&c->s_up, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_pre_mask, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_up, cudaEventDisableTiming));
        CK(cudaEventRecord(c->ev_pre_mask, c->s));
        c->types_dev = dalloc<uint8_t>((size_t)c->g0.n);
        if (dim == 3 && !c->slab.on && c->coarse_skip)
            for (int l = 1; l + 1 < depth; ++l) {  // k_coarse_live flags per coarse down tile
                const Geom& gl = c->L[l].g;
                const int zc = coarse_zc(c, gl);
                c->clive[l] = dalloc<uint8_t>((size_t)((gl.nx + kZX - 1) / kZX) * ((gl.ny + kZY - 1) / kZY) *
                                              ((gl.nz + zc - 1) / zc));
            }
        // first capacities of the per-frame tables; setup_sync grows them from a frame's counts
        for (int l = 0; l < depth; ++l) {
            c->cap_ht[l] = 1 << 14;
            c->tab_cap[l] = 4096;
        }
        c->pid0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->repcell0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->dlist0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->dkid0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->ulist0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->ukid0 = dalloc<uint32_t>((size_t)c->g0.n);
        c->check_flag = dalloc<unsigned int>(1);
        c->npat0 = dalloc<uint32_t>(1);
        const size_t n = (size_t)c->g0.n;
        c->X0 = dalloc<double>(n);
        c->X1 = dalloc<double>(n);
        c->R = dalloc<double>(n);
        c->Bf = dalloc<double>(n);
        c->Dtmp = dalloc<double>(n);
        // the zero invariant from the start (frames then zero what stops being fluid)
        for (double* v : {c->X1, c->R, c->Dtmp}) CK(cudaMemset(v, 0, n * sizeof(double)));
        c->red_a = dalloc<double>(n);
        c->red_b = dalloc<double>(n);
        c->st = dalloc<SolverState>(1);
        CK(cudaMemset(c->st, 0, sizeof(SolverState)));
        CK(cudaMallocHost(&c->st_host, sizeof(SolverState)));
        c->counter = dalloc<unsigned int>(1);
        CK(cudaMemset(c->counter, 0, sizeof(unsigned int)));
        {
            // the pair-stencil grids: one block per 64 x 4 x 1 tile
            const long long nblk = ((long long)(nx + 63) / 64) * ((ny + 3) / 4) * nz;
            c->partials = dalloc<double>((size_t)std::max<long long>(65536, nblk) * (2 + kMaxOrtho));
        }
        ensure_ring(c, 3);
        ensure_hist(c, 1001);
        if (c->slab.on) {
            c->slab.all = dalloc<double>((size_t)c->slab.nranks * kPart);
            c->slab.allu = dalloc<unsigned long long>((size_t)c->slab.nranks * 81);
            // ghost planes start as the outside of the domain (zeros)
            const size_t n = (size_t)c->g0.n;
            for (double* v : {c->X0, c->X1, c->R, c->Bf, c->Dtmp}) CK(cudaMemsetAsync(v, 0, n * sizeof(double), c->s));
        }
        do_set_params(c, params, n_params);
        CK(cudaStreamSynchronize(c->s));
        *out = c;
        return NPSD_OK;
    } catch (const InvalidArgument& e) {
        g_create_err = e.what();
        free_ctx(c);
        delete c;
        return NPSD_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_create_err = e.what();
        free_ctx(c);
        delete c;
        return NPSD_CUDA_ERROR;
    }
}

thread_local std::string g_comm_err;

}  // namespace

int npsd_b200_create(int dim, int nx, int ny, int nz, int depth, const float* params, size_t n_params,
                     const int* devices, int n_devices, npsd_b200_ctx** out) {
    if (n_devices > 1) {
        g_create_err = "npsd_b200: one device per context; shard a grid with npsd_b200_create_slab";
        if (out) *out = nullptr;
        return NPSD_INVALID_ARGUMENT;
    }
    return create_impl(dim, nx, ny, nz, depth, params, n_params, (devices && n_devices == 1) ? devices[0] : 0,
                       nullptr, out);
}

int npsd_b200_create_slab(int nx, int ny, int nz, int z0, int nz_own, int depth, const float* params,
                          size_t n_params, int device, npsd_b200_comm* comm, int rank, npsd_b200_ctx** out) {
    if (out) *out = nullptr;
    if (!comm || !out) {
        g_create_err = "create_slab: null communicator or output";
        return NPSD_INVALID_ARGUMENT;
    }
    const int unit = 1 << (depth > 0 ? depth - 1 : 0);
    std::string why;
    if (depth < 2 || depth > kMaxDepth) why = "create_slab: depth must be in [2, 8]";
    else if (rank < 0 || rank >= comm->nranks) why = "create_slab: rank out of range";
    else if (nz_own <= 0 || z0 < 0 || z0 + nz_own > nz) why = "create_slab: slab outside the grid";
    else if (z0 % unit != 0 || nz_own % unit != 0)
        why = "create_slab: slab bounds must be multiples of 2^(depth-1) = " + std::to_string(unit);
    else if (((long long)nx * ny) % 32 != 0) why = "create_slab: nx * ny must be a multiple of 32";
    if (!why.empty()) {
        g_create_err = why;
        return NPSD_INVALID_ARGUMENT;
    }
    SlabInfo si;
    si.on = true;
    si.rank = rank;
    si.nranks = comm->nranks;
    si.z0 = z0;
    si.nz_own = nz_own;
    si.nz_global = nz;
    si.comm = comm;
    return create_impl(3, nx, ny, nz, depth, params, n_params, device, &si, out);
}

int npsd_b200_nccl_unique_id(void* id128) {
    try {
        if (!id128) return NPSD_INVALID_ARGUMENT;
        ncclUniqueId id;
        NCK(nccl().GetUniqueId(&id));
        std::memcpy(id128, &id, sizeof(id));
        return NPSD_OK;
    } catch (const std::exception& e) {
        g_comm_err = e.what();
        return NPSD_CUDA_ERROR;
    }
}

int npsd_b200_comm_create_nccl(const void* id128, int rank, int nranks, int device, npsd_b200_comm** out) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return NPSD_INVALID_ARGUMENT;
    *out = nullptr;
    try {
        CK(cudaSetDevice(device));
        auto* cm = new NcclComm();
        cm->nranks = nranks;
        cm->rank = rank;
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        try {
            NCK(nccl().CommInitRank(&cm->comm, nranks, id, rank));
        } catch (...) {
            delete cm;
            throw;
        }
        *out = cm;
        return NPSD_OK;
    } catch (const std::exception& e) {
        g_comm_err = e.what();
        return NPSD_CUDA_ERROR;
    }
}

int npsd_b200_comm_create_local(int nranks, npsd_b200_comm** out) {
    if (!out || nranks < 1) return NPSD_INVALID_ARGUMENT;
    *out = new LocalComm(nranks);
    return NPSD_OK;
}

int npsd_b200_comm_destroy(npsd_b200_comm* comm) {
    delete comm;
    return NPSD_OK;
}

const char* npsd_b200_comm_last_error(void) { return g_comm_err.c_str(); }

int npsd_b200_slab_graph(const npsd_b200_ctx* c) {
    return (c && c->slab.on && c->slab_exec && !c->slab_no_graph) ? 1 : 0;
}

int npsd_b200_destroy(npsd_b200_ctx* c) {
    if (!c) return NPSD_OK;
    cudaSetDevice(c->dev);
    cudaStreamSynchronize(c->s);
    free_ctx(c);
    delete c;
    return NPSD_OK;
}

const char* npsd_b200_last_error(const npsd_b200_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

int npsd_b200_set_exact(npsd_b200_ctx* c, int exact) {
    return guarded(c, [&] {
        const bool fast = exact == 0;
        if (fast != c->fast) {
            c->fast = fast;
            ++c->buf_gen;  // captured graphs hold the other kernels
        }
    });
}

int npsd_b200_set_params(npsd_b200_ctx* c, const float* params, size_t n) {
    return guarded(c, [&] {
        do_set_params(c, params, n);
        CK(cudaStreamSynchronize(c->s));
    });
}

// z-slab: the owned planes' types (host or device) into the local layout,
// ghost planes = solid outside the domain, then the neighbours' planes
void slab_stage_types(npsd_b200_ctx* c, const uint8_t* types, cudaMemcpyKind kind) {
    const Geom& g = c->g0;
    const size_t plane = (size_t)g.nx * g.ny;
    uint8_t* d = c->types_dev;
    CK(cudaMemsetAsync(d, 2, (size_t)g.n, c->s));
    CK(cudaMemcpyAsync(d + (size_t)g.zo0 * plane, types, (size_t)(g.zo1 - g.zo0) * plane, kind, c->s));
    slab_exchange(c, c->s, d, 1, 0);
    set_mask_impl<3>(c, d);
    // finished here, on every rank at once: a redo (setup_sync) is collective
    setup_sync(c);
}

int npsd_b200_set_mask_device(npsd_b200_ctx* c, const uint8_t* d_types) {
    return guarded(c, [&] {
        require(d_types != nullptr, "npsd_b200: cell types pointer is null");
        if (c->slab.on) {
            slab_stage_types(c, d_types, cudaMemcpyDeviceToDevice);
            return;
        }
        // the frame's types into the context's buffer (the captured setup graph
        // reads them there; the caller's buffer is free once this returns)
        CK(cudaMemcpyAsync(c->types_dev, d_types, (size_t)c->g0.n, cudaMemcpyDeviceToDevice, c->s));
        if (c->dim == 3)
            set_mask_impl<3>(c, c->types_dev);
        else
            set_mask_impl<2>(c, c->types_dev);
    });
}

int npsd_b200_set_mask(npsd_b200_ctx* c, const uint8_t* types) {
    return guarded(c, [&] {
        require(types != nullptr, "npsd_b200: cell types pointer is null");
        const size_t n = c->slab.on ? (size_t)(c->g0.zo1 - c->g0.zo0) * c->g0.nx * c->g0.ny : (size_t)c->g0.n;
        // the range check runs on the device, on the uploaded bytes
        uint8_t* chk = reinterpret_cast<uint8_t*>(c->red_b);
        CK(cudaMemcpyAsync(chk, types, n, cudaMemcpyHostToDevice, c->s));
        require(device_check(c, k_check_types, (long long)n, (const uint8_t*)chk, (long long)n),
                "npsd_b200: cell type out of range (0 fluid, 1 air, 2 solid)");
        if (c->slab.on) {
            slab_stage_types(c, chk, cudaMemcpyDeviceToDevice);
            return;
        }
        CK(cudaMemcpyAsync(c->types_dev, chk, n, cudaMemcpyDeviceToDevice, c->s));
        if (c->dim == 3)
            set_mask_impl<3>(c, c->types_dev);
        else
            set_mask_impl<2>(c, c->types_dev);
    });
}

int npsd_b200_is_pure_neumann(npsd_b200_ctx* c, int* out) {
    return guarded(c, [&] {
        require(out != nullptr, "is_pure_neumann: out is NULL");
        check_mask(c);
        const Geom g = c->g0;
        bool none = (c->dim == 3) ? device_check(c, k_touches_air<3>, g.n, g, (const uint8_t*)c->L[0].cls)
                                  : device_check(c, k_touches_air<2>, g.n, g, (const uint8_t*)c->L[0].cls);
        if (c->slab.on) {  // any rank's fluid touching air
            unsigned long long* v = reinterpret_cast<unsigned long long*>(c->red_b);
            const unsigned long long mine = none ? 0ull : 1ull;
            CK(cudaMemcpyAsync(v, &mine, sizeof mine, cudaMemcpyHostToDevice, c->s));
            slab_allreduce_u64(c, c->s, v, 1);
            unsigned long long tot = 0;
            CK(cudaMemcpyAsync(&tot, v, sizeof tot, cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            none = (tot == 0);
        }
        *out = none ? 1 : 0;
        return NPSD_OK;
    });
}

int64_t npsd_b200_n_fluid(const npsd_b200_ctx* cc) {
    // the last set_mask may still be in flight: finish it (the count is device-side)
    auto* c = const_cast<npsd_b200_ctx*>(cc);
    if (!c || !c->mask_ok) return -1;
    return guarded(c, [&] { setup_sync(c); }) == NPSD_OK ? c->n_fluid : -1;
}

int npsd_b200_fluid_indices(npsd_b200_ctx* c, int64_t* out) {
    return guarded(c, [&] {
        check_mask(c);
        // scatter the reduced index ramp, then read positions back on host
        std::vector<uint32_t> mask((size_t)c->L[0].nseg), base((size_t)c->L[0].nseg);
        CK(cudaMemcpyAsync(mask.data(), c->fmask, mask.size() * 4, cudaMemcpyDeviceToHost, c->s));
        CK(cudaMemcpyAsync(base.data(), c->fbase, base.size() * 4, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        // z-slab: global linear indices (local plane zo0 is global plane z0)
        const long long plane = (long long)c->g0.nx * c->g0.ny;
        const long long shift = c->slab.on ? ((long long)c->slab.z0 - c->g0.zo0) * plane : 0;
        for (size_t sgm = 0; sgm < mask.size(); ++sgm) {
            uint32_t m = mask[sgm];
            long long k = base[sgm];
            while (m) {
                const int b = __builtin_ctz(m);
                out[k++] = (int64_t)(sgm * 32 + (size_t)b) + shift;
                m &= m - 1;
            }
        }
    });
}

int npsd_b200_precond_apply(npsd_b200_ctx* c, const double* r, double* z, int64_t n_f) {
    return guarded(c, [&] {
        check_mask(c);
        require(n_f == c->n_fluid, "NeuralPrecond::apply: size mismatch");
        if (n_f == 0) return;
        const Geom g = c->g0;
        CK(cudaMemcpyAsync(c->red_a, r, (size_t)n_f * sizeof(double), cudaMemcpyHostToDevice, c->s));
        LAUNCH(c, c->s, k_scatter, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->red_a, c->R);
        if (c->slab.on) {
            // ||r|| over every rank, then r's ghost planes
            const int flags[2] = {1, 0};  // dist, done
            CK(cudaMemcpyAsync(&c->st->dist, &flags[0], sizeof(int), cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(&c->st->done, &flags[1], sizeof(int), cudaMemcpyHostToDevice, c->s));
        }
        LAUNCH(c, c->s, k_norm_precond, g.n, g, c->R, c->st, c->partials, c->counter);
        if (c->slab.on) {
            slab_reduce(c, c->s, kFinNormPrecond);
            slab_exchange(c, c->s, c->R, sizeof(double), 0);
        }
        // no cached directions: the fused dots in the L0 up kernel are empty
        const int zero = 0;
        CK(cudaMemcpyAsync(&c->st->n_cache, &zero, sizeof(int), cudaMemcpyHostToDevice, c->s));
        const int one = 1;
        CK(cudaMemcpyAsync(&c->st->ring, &one, sizeof(int), cudaMemcpyHostToDevice, c->s));
        if (c->dim == 3)
            launch_network<3>(c, c->s, false, nullptr);
        else
            launch_network<2>(c, c->s, false, nullptr);
        LAUNCH(c, c->s, k_gather, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->Dtmp, c->red_b);
        CK(cudaMemcpyAsync(z, c->red_b, (size_t)n_f * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_ic0_apply(npsd_b200_ctx* c, const double* r, double* z, int64_t n_f, int* shift_retries) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "ic0: not available on a z-slab context");
        require(n_f == c->n_fluid, "ic0: size mismatch");
        if (n_f == 0) return;
        const Geom g = c->g0;
        if (!c->cgZ) {
            c->cgP0 = dalloc<double>((size_t)g.n);
            c->cgP1 = dalloc<double>((size_t)g.n);
            c->cgAp = dalloc<double>((size_t)g.n);
            c->cgZ = dalloc<double>((size_t)g.n);
            ++c->buf_gen;
        }
        ic0_factor(c);
        if (shift_retries) *shift_retries = c->ic0_shift_retries;
        CK(cudaMemcpyAsync(c->red_a, r, (size_t)n_f * sizeof(double), cudaMemcpyHostToDevice, c->s));
        LAUNCH(c, c->s, k_scatter, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->red_a, c->R);
        ic0_sweep<1>(c, c->s, 0.0, c->R, nullptr);
        ic0_sweep<2>(c, c->s, 0.0, c->R, nullptr);
        LAUNCH(c, c->s, k_gather, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->cgZ, c->red_b);
        CK(cudaMemcpyAsync(z, c->red_b, (size_t)n_f * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_spmv(npsd_b200_ctx* c, const double* x, double* y, int64_t n_f) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "spmv: not available on a z-slab context");
        require(n_f == c->n_fluid, "spmv: dimension mismatch");
        if (n_f == 0) return;
        const Geom g = c->g0;
        CK(cudaMemcpyAsync(c->red_a, x, (size_t)n_f * sizeof(double), cudaMemcpyHostToDevice, c->s));
        LAUNCH(c, c->s, k_scatter, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->red_a, c->Dtmp);
        if (c->dim == 3)
            LAUNCH(c, c->s, k_spmv<3>, g.n, g, c->L[0].cls, c->Dtmp, c->R);
        else
            LAUNCH(c, c->s, k_spmv<2>, g.n, g, c->L[0].cls, c->Dtmp, c->R);
        LAUNCH(c, c->s, k_gather, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->R, c->red_b);
        CK(cudaMemcpyAsync(y, c->red_b, (size_t)n_f * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        // restore the zero invariant of the scratch vectors used
        CK(cudaMemsetAsync(c->Dtmp, 0, (size_t)g.n * sizeof(double), c->s));
        CK(cudaMemsetAsync(c->R, 0, (size_t)g.n * sizeof(double), c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_check_operator(npsd_b200_ctx* c, int64_t n_rows, const int64_t* row_offsets,
                             const int64_t* col_indices, const double* values, int64_t nnz, int full) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "check_operator: not available on a z-slab context");
        require(n_rows == c->n_fluid, "solve: matrix rows (" + std::to_string(n_rows) + ") != fluid cells of the mask (" +
                                          std::to_string(c->n_fluid) + ")");
        require(row_offsets != nullptr && (nnz == 0 || (col_indices && values)), "check_operator: null CSR arrays");
        require(row_offsets[0] == 0 && row_offsets[n_rows] == nnz, "check_operator: row_offsets do not span nnz");
        if (n_rows == 0) return;
        // the flag-derived rows (assemble_poisson[_3d] + reduce, discretization.cpp:21-160)
        const Geom g = c->g0;
        uint8_t* d_info = reinterpret_cast<uint8_t*>(c->red_b);
        if (c->dim == 3)
            LAUNCH(c, c->s, k_row_info<3>, g.n, g, c->L[0].cls, c->fmask, c->fbase, d_info);
        else
            LAUNCH(c, c->s, k_row_info<2>, g.n, g, c->L[0].cls, c->fmask, c->fbase, d_info);
        std::vector<uint8_t> info((size_t)n_rows);
        CK(cudaMemcpyAsync(info.data(), d_info, (size_t)n_rows, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        // nnz, the diagonal and the off-diagonal values of every row
        long long want_nnz = 0;
        for (int64_t r = 0; r < n_rows; ++r) {
            const int diag = info[(size_t)r] & 15, nf = info[(size_t)r] >> 4;
            want_nnz += (diag != 0) + nf;
            const int64_t a = row_offsets[r], e = row_offsets[r + 1];
            require(e - a == (diag != 0) + nf, "solve: A is not the mixed-BC Laplacian of the mask (row " +
                                                   std::to_string(r) + " has " + std::to_string(e - a) +
                                                   " entries, the flags give " + std::to_string((diag != 0) + nf) + ")");
            bool seen_diag = false;
            for (int64_t k = a; k < e; ++k) {
                const int64_t col = col_indices[k];
                require(col >= 0 && col < n_rows, "solve: A column index out of range at row " + std::to_string(r));
                if (col == r) {
                    seen_diag = true;
                    require(values[k] == (double)diag, "solve: A's diagonal differs from the flags at row " +
                                                           std::to_string(r));
                } else {
                    require(values[k] == -1.0, "solve: A's off-diagonal entry differs from -1 at row " +
                                                   std::to_string(r));
                }
            }
            require(seen_diag == (diag != 0), "solve: A's diagonal pattern differs from the flags at row " +
                                                  std::to_string(r));
        }
        require(want_nnz == nnz, "solve: A's nnz differs from the flag-derived operator");
        if (!full) return;
        // debug: the whole operator, A v (CSR order, spmv's serial row sums,
        // sparse.cpp:100-117) against the device operator, bitwise
        std::vector<double> v((size_t)n_rows), ya((size_t)n_rows), yd((size_t)n_rows);
        unsigned long long st = 0x9e3779b97f4a7c15ull;
        for (auto& x : v) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            x = (double)(st >> 11) * (1.0 / 9007199254740992.0) - 0.5;
        }
        for (int64_t r = 0; r < n_rows; ++r) {
            double acc = 0.0;
            for (int64_t k = row_offsets[r]; k < row_offsets[r + 1]; ++k) acc += values[k] * v[(size_t)col_indices[k]];
            ya[(size_t)r] = acc;
        }
        CK(cudaMemcpyAsync(c->red_a, v.data(), (size_t)n_rows * sizeof(double), cudaMemcpyHostToDevice, c->s));
        LAUNCH(c, c->s, k_scatter, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->red_a, c->Dtmp);
        if (c->dim == 3)
            LAUNCH(c, c->s, k_spmv<3>, g.n, g, c->L[0].cls, c->Dtmp, c->R);
        else
            LAUNCH(c, c->s, k_spmv<2>, g.n, g, c->L[0].cls, c->Dtmp, c->R);
        LAUNCH(c, c->s, k_gather, g.n, g, c->L[0].cls, c->fmask, c->fbase, c->R, c->red_b);
        CK(cudaMemcpyAsync(yd.data(), c->red_b, (size_t)n_rows * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        CK(cudaMemsetAsync(c->Dtmp, 0, (size_t)g.n * sizeof(double), c->s));
        CK(cudaMemsetAsync(c->R, 0, (size_t)g.n * sizeof(double), c->s));
        CK(cudaStreamSynchronize(c->s));
        for (int64_t r = 0; r < n_rows; ++r)
            require(std::memcmp(&ya[(size_t)r], &yd[(size_t)r], sizeof(double)) == 0,
                    "solve: A v differs from the flag-derived operator at row " + std::to_string(r));
    });
}

namespace {
// face-array element counts: u (nx+1, ny, nz), v (nx, ny+1, nz), w (nx, ny, nz+1)
void mac_sizes(const npsd_b200_ctx* c, size_t n[3]) {
    const size_t nx = c->g0.nx, ny = c->g0.ny, nz = c->g0.nz;
    n[0] = (nx + 1) * ny * nz;
    n[1] = nx * (ny + 1) * nz;
    n[2] = (c->dim == 3) ? nx * ny * (nz + 1) : 0;
}

void launch_mac_rhs(npsd_b200_ctx* c, const double* const f[6], double h, double dt, double rho, double* b) {
    require(c->dim == 2 || f[2] != nullptr, "mac_divergence_rhs: w is null");
    require(!c->slab.on, "mac_divergence_rhs: not available on a z-slab context");
    require(dt != 0.0, "mac_divergence_rhs: dt must be nonzero");
    const bool bc = f[3] != nullptr;
    require(!bc || (f[4] != nullptr && (c->dim == 2 || f[5] != nullptr)),
            "mac_divergence_rhs: boundary value shape mismatch");
    const double scale = -(rho * h) / dt;
    const Geom g = c->g0;
    if (c->dim == 3)
        LAUNCH(c, c->s, k_mac_rhs<3>, g.n, g, c->L[0].cls, f[0], f[1], f[2], f[3], f[4], f[5], scale, b);
    else
        LAUNCH(c, c->s, k_mac_rhs<2>, g.n, g, c->L[0].cls, f[0], f[1], nullptr, f[3], f[4], nullptr, scale, b);
}
}  // namespace

int npsd_b200_mac_divergence_rhs(npsd_b200_ctx* c, const double* u, const double* v, const double* w, double h,
                                 double dt, double rho, const double* bc_u, const double* bc_v, const double* bc_w,
                                 double* b_reduced) {
    return guarded(c, [&] {
        check_mask(c);
        require(u && v && b_reduced, "mac_divergence_rhs: null argument");
        size_t n[3];
        mac_sizes(c, n);
        const size_t tot = n[0] + n[1] + n[2];
        if (c->mac_cap < 2 * tot) {
            if (c->mac) CK(cudaFree(c->mac));
            c->mac = dalloc<double>(2 * tot);
            c->mac_cap = 2 * tot;
        }
        const double* host[6] = {u, v, w, bc_u, bc_v, bc_w};
        const double* dev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        size_t off = 0;
        for (int i = 0; i < 6; ++i) {
            const size_t k = n[i % 3];
            if (host[i] && k) {
                CK(cudaMemcpyAsync(c->mac + off, host[i], k * sizeof(double), cudaMemcpyHostToDevice, c->s));
                dev[i] = c->mac + off;
            }
            off += k;
        }
        double* full = c->red_a;  // scratch (n doubles)
        launch_mac_rhs(c, dev, h, dt, rho, full);
        const Geom g = c->g0;
        LAUNCH(c, c->s, k_gather, g.n, g, c->L[0].cls, c->fmask, c->fbase, full, c->red_b);
        CK(cudaMemcpyAsync(b_reduced, c->red_b, (size_t)c->n_fluid * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_mac_divergence_rhs_device(npsd_b200_ctx* c, const double* d_u, const double* d_v, const double* d_w,
                                        double h, double dt, double rho, const double* d_bc_u, const double* d_bc_v,
                                        const double* d_bc_w, double* d_b_full) {
    return guarded(c, [&] {
        check_mask(c);
        require(d_u && d_v && d_b_full, "mac_divergence_rhs: null argument");
        const double* dev[6] = {d_u, d_v, d_w, d_bc_u, d_bc_v, d_bc_w};
        launch_mac_rhs(c, dev, h, dt, rho, d_b_full);
    });
}

int npsd_b200_net_apply(npsd_b200_ctx* c, const float* x, float* y) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "net_apply: not available on a z-slab context");
        const size_t n = (size_t)c->g0.n;
        if (!c->xin_f) c->xin_f = dalloc<float>(n);
        if (!c->out_f) c->out_f = dalloc<float>(n);
        CK(cudaMemcpyAsync(c->xin_f, x, n * sizeof(float), cudaMemcpyHostToDevice, c->s));
        if (c->dim == 3)
            launch_network<3>(c, c->s, true, nullptr);
        else
            launch_network<2>(c, c->s, true, nullptr);
        const float* res = (c->depth == 1) ? c->L[0].y : c->out_f;
        CK(cudaMemcpyAsync(y, res, n * sizeof(float), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_psdo_solve_device(npsd_b200_ctx* c, const double* d_b, const double* d_x0,
                                const npsd_b200_solve_cfg* cfg, double* d_x, npsd_b200_report* rep) {
    return guarded(c, [&] {
        check_mask_async(c);
        require(cfg != nullptr && d_b != nullptr && d_x != nullptr, "solve: null argument");
        run_after_setup(c, [&] {
            const Geom g = c->g0;
            const uint8_t* cls = c->L[0].cls;
            const double* b_in = d_b;
            const double* x0_in = d_x0;
            // z-slab: caller buffers hold the owned planes only
            const size_t off = (size_t)owned_lo(g), cnt = (size_t)(owned_hi(g) - owned_lo(g));
            if (c->slab.on) {
                CK(cudaMemcpyAsync(c->Bf + off, d_b, cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
                b_in = c->Bf;
                if (d_x0) {
                    CK(cudaMemcpyAsync(c->X0 + off, d_x0, cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
                    x0_in = c->X0;
                }
            }
            LAUNCH(c, c->s, k_mask_fluid, g.n, g, cls, b_in, c->Bf);
            if (x0_in)
                LAUNCH(c, c->s, k_mask_fluid, g.n, g, cls, x0_in, c->X0);
            else
                CK(cudaMemsetAsync(c->X0, 0, (size_t)g.n * sizeof(double), c->s));
            solve_any(c, cfg, rep);
            const double* xr = c->st_host->xcur ? c->X1 : c->X0;
            CK(cudaMemcpyAsync(d_x, xr + off, cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
            CK(cudaStreamSynchronize(c->s));
        });
    });
}

// psdo_solve on reduced host vectors. Unsized: the length is the fluid count
// (known once the frame's setup is finished). Sized: the caller's length,
// checked against it, and the rhs upload starts before the setup has
// finished (its own stream).
static int psdo_solve_host(npsd_b200_ctx* c, const double* b, bool sized, long long nb, const double* x0,
                           const npsd_b200_solve_cfg* cfg, double* x, npsd_b200_report* rep) {
    return guarded(c, [&] {
        require(cfg != nullptr && b != nullptr && x != nullptr, "solve: null argument");
        bool uploaded = false;
        if (sized) {
            require(nb >= 0 && nb <= c->g0.n, "solve: rhs length mismatch");
            if (!c->slab.on && nb > 0) {
                CK(cudaStreamWaitEvent(c->s_up, c->ev_pre_mask, 0));
                CK(cudaMemcpyAsync(c->red_a, b, (size_t)nb * sizeof(double), cudaMemcpyHostToDevice, c->s_up));
                CK(cudaEventRecord(c->ev_up, c->s_up));
                // the solve's stream is ordered after the upload (the setup already queued runs first)
                CK(cudaStreamWaitEvent(c->s, c->ev_up, 0));
                uploaded = true;
            }
        }
        check_mask(c);
        if (c->n_fluid == 0) throw EmptySystem("reduce: image has no fluid cells");
        require(!sized || nb == c->n_fluid, "solve: rhs length mismatch");
        const Geom g = c->g0;
        const uint8_t* cls = c->L[0].cls;
        const size_t nf = (size_t)c->n_fluid;
        // check_inputs (solver.cpp:28-33) on the device, on the uploaded vector
        if (!uploaded) CK(cudaMemcpyAsync(c->red_a, b, nf * sizeof(double), cudaMemcpyHostToDevice, c->s));
        require(device_check(c, k_check_finite, (long long)nf, (const double*)c->red_a, (long long)nf),
                "solve: rhs has non-finite entries");
        LAUNCH(c, c->s, k_scatter, g.n, g, cls, c->fmask, c->fbase, c->red_a, c->Bf);
        if (x0) {
            CK(cudaMemcpyAsync(c->red_b, x0, nf * sizeof(double), cudaMemcpyHostToDevice, c->s));
            LAUNCH(c, c->s, k_scatter, g.n, g, cls, c->fmask, c->fbase, c->red_b, c->X0);
        } else {
            CK(cudaMemsetAsync(c->X0, 0, (size_t)g.n * sizeof(double), c->s));
        }
        try {
            solve_any(c, cfg, rep);
        } catch (const Breakdown&) {
            const double* xr = c->st_host->xcur ? c->X1 : c->X0;
            LAUNCH(c, c->s, k_gather, g.n, g, cls, c->fmask, c->fbase, xr, c->red_b);
            CK(cudaMemcpyAsync(x, c->red_b, nf * sizeof(double), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            throw;
        }
        const double* xr = c->st_host->xcur ? c->X1 : c->X0;
        LAUNCH(c, c->s, k_gather, g.n, g, cls, c->fmask, c->fbase, xr, c->red_b);
        CK(cudaMemcpyAsync(x, c->red_b, nf * sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}

int npsd_b200_psdo_solve(npsd_b200_ctx* c, const double* b, const double* x0, const npsd_b200_solve_cfg* cfg,
                         double* x, npsd_b200_report* rep) {
    return psdo_solve_host(c, b, false, 0, x0, cfg, x, rep);
}

int npsd_b200_psdo_solve_n(npsd_b200_ctx* c, const double* b, int64_t nb, const double* x0,
                           const npsd_b200_solve_cfg* cfg, double* x, npsd_b200_report* rep) {
    return psdo_solve_host(c, b, true, (long long)nb, x0, cfg, x, rep);
}

int npsd_b200_pcg_solve(npsd_b200_ctx* c, const double* b, const double* x0, const npsd_b200_solve_cfg* cfg,
                        int precond, double* x, npsd_b200_report* rep) {
    return guarded(c, [&] {
        check_mask(c);
        require(cfg != nullptr && b != nullptr && x != nullptr, "solve: null argument");
        if (c->n_fluid == 0) throw EmptySystem("reduce: image has no fluid cells");
        const Geom g = c->g0;
        const uint8_t* cls = c->L[0].cls;
        const size_t nf = (size_t)c->n_fluid;
        CK(cudaMemcpyAsync(c->red_a, b, nf * sizeof(double), cudaMemcpyHostToDevice, c->s));
        require(device_check(c, k_check_finite, (long long)nf, (const double*)c->red_a, (long long)nf),
                "solve: rhs has non-finite entries");
        LAUNCH(c, c->s, k_scatter, g.n, g, cls, c->fmask, c->fbase, c->red_a, c->Bf);
        if (x0) {
            CK(cudaMemcpyAsync(c->red_b, x0, nf * sizeof(double), cudaMemcpyHostToDevice, c->s));
            LAUNCH(c, c->s, k_scatter, g.n, g, cls, c->fmask, c->fbase, c->red_b, c->X0);
        } else {
            CK(cudaMemsetAsync(c->X0, 0, (size_t)g.n * sizeof(double), c->s));
        }
        auto gather = [&] {
            LAUNCH(c, c->s, k_gather, g.n, g, cls, c->fmask, c->fbase, c->X0, c->red_b);
            CK(cudaMemcpyAsync(x, c->red_b, nf * sizeof(double), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
        };
        try {
            pcg_solve_impl(c, cfg, precond, rep);
        } catch (const Breakdown&) {
            gather();
            throw;
        }
        gather();
    });
}

int npsd_b200_pcg_solve_device(npsd_b200_ctx* c, const double* d_b, const double* d_x0,
                               const npsd_b200_solve_cfg* cfg, int precond, double* d_x, npsd_b200_report* rep) {
    return guarded(c, [&] {
        check_mask_async(c);
        require(cfg != nullptr && d_b != nullptr && d_x != nullptr, "solve: null argument");
        if (precond == 2) setup_sync(c);  // the IC0 factor's diagonal shift uses the frame's size
        run_after_setup(c, [&] {
            const Geom g = c->g0;
            const uint8_t* cls = c->L[0].cls;
            LAUNCH(c, c->s, k_mask_fluid, g.n, g, cls, d_b, c->Bf);
            if (d_x0)
                LAUNCH(c, c->s, k_mask_fluid, g.n, g, cls, d_x0, c->X0);
            else
                CK(cudaMemsetAsync(c->X0, 0, (size_t)g.n * sizeof(double), c->s));
            pcg_solve_impl(c, cfg, precond, rep);
            CK(cudaMemcpyAsync(d_x, c->X0, (size_t)g.n * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
            CK(cudaStreamSynchronize(c->s));
        });
    });
}

int npsd_b200_level_image(npsd_b200_ctx* c, int level, float* out) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "level_image: not available on a z-slab context");
        require(level >= 0 && level < c->depth, "level out of range");
        const LevelBufs& L = c->L[level];
        if (level == 0) {
            std::vector<uint8_t> cls((size_t)L.g.n);
            CK(cudaMemcpyAsync(cls.data(), L.cls, cls.size(), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            for (int ch = 0; ch < 3; ++ch)
                for (size_t i = 0; i < cls.size(); ++i)
                    out[(size_t)ch * cls.size() + i] = (((cls[i] >> 2) & 3) == ch) ? 1.0f : 0.0f;
        } else {
            CK(cudaMemcpyAsync(out, L.img, 3 * (size_t)L.g.n * sizeof(float), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
        }
    });
}

int npsd_b200_linear_coeffs(npsd_b200_ctx* c, float* za, float* zb) {
    return guarded(c, [&] {
        check_mask(c);
        std::vector<float> h(2 * (size_t)c->depth);
        CK(cudaMemcpyAsync(h.data(), c->zab, h.size() * sizeof(float), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        for (int l = 0; l + 1 < c->depth; ++l) {
            za[l] = h[2 * (size_t)l];
            zb[l] = h[2 * (size_t)l + 1];
        }
    });
}

int npsd_b200_mixed_counts(npsd_b200_ctx* c, int64_t* counts) {
    return guarded(c, [&] {
        check_mask(c);
        for (int l = 0; l < c->depth; ++l) {
            const LevelBufs& L = c->L[l];
            uint32_t t[2];
            CK(cudaMemcpyAsync(&t[0], L.mbase + (L.nseg - 1), 4, cudaMemcpyDeviceToHost, c->s));
            CK(cudaMemcpyAsync(&t[1], L.mcount + (L.nseg - 1), 4, cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            counts[l] = (int64_t)t[0] + t[1];
        }
    });
}

int npsd_b200_device_alloc(npsd_b200_ctx* c, size_t bytes, void** out) {
    return guarded(c, [&] { CK(cudaMalloc(out, bytes ? bytes : 1)); });
}
int npsd_b200_device_free(npsd_b200_ctx* c, void* p) {
    return guarded(c, [&] { CK(cudaFree(p)); });
}
int npsd_b200_host_alloc(npsd_b200_ctx* c, size_t bytes, void** out) {
    return guarded(c, [&] { CK(cudaMallocHost(out, bytes ? bytes : 1)); });
}
int npsd_b200_host_free(npsd_b200_ctx* c, void* p) {
    return guarded(c, [&] { CK(cudaFreeHost(p)); });
}
int npsd_b200_memcpy(npsd_b200_ctx* c, void* dst, const void* src, size_t bytes) {
    return guarded(c, [&] { CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->s)); });
}
int npsd_b200_synchronize(npsd_b200_ctx* c) {
    return guarded(c, [&] { CK(cudaStreamSynchronize(c->s)); });
}

double npsd_b200_last_solve_ms(const npsd_b200_ctx* c) { return c ? (double)c->last_ms : 0.0; }
int64_t npsd_b200_last_solve_launches(const npsd_b200_ctx* c) { return c ? c->last_launches : 0; }

int npsd_b200_event_record(npsd_b200_ctx* c, int slot) {
    return guarded(c, [&] {
        require(slot >= 0 && slot < 16, "event slot out of range");
        if (!c->user_ev[slot]) CK(cudaEventCreate(&c->user_ev[slot]));
        CK(cudaEventRecord(c->user_ev[slot], c->s));
    });
}

double npsd_b200_event_elapsed_ms(npsd_b200_ctx* c, int a, int b) {
    if (!c || a < 0 || b < 0 || a >= 16 || b >= 16 || !c->user_ev[a] || !c->user_ev[b]) return -1.0;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaSetDevice(c->dev);
    if (cudaEventSynchronize(c->user_ev[b]) != cudaSuccess) return -1.0;
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, c->user_ev[a], c->user_ev[b]) != cudaSuccess) return -1.0;
    return (double)ms;
}

int64_t npsd_b200_launch_count(const npsd_b200_ctx* c) { return c ? c->launches : 0; }

int npsd_b200_profile_iterations(npsd_b200_ctx* c, const double* d_b, const npsd_b200_solve_cfg* cfg, int iters,
                                 double* ms_out, int* n_out, char* names, int name_len) {
    return guarded(c, [&] {
        check_mask(c);
        require(!c->slab.on, "profile_iterations: not available on a z-slab context");
        require(cfg != nullptr && d_b != nullptr && iters > 0 && n_out != nullptr, "profile: bad arguments");
        if (c->n_fluid == 0) throw EmptySystem("reduce: image has no fluid cells");
        const Geom g = c->g0;
        const uint8_t* cls = c->L[0].cls;
        LAUNCH(c, c->s, k_mask_fluid, g.n, g, cls, d_b, c->Bf);
        CK(cudaMemsetAsync(c->X0, 0, (size_t)g.n * sizeof(double), c->s));
        const int ring = cfg->n_ortho + 1;
        require(cfg->n_ortho >= 0 && cfg->n_ortho <= kMaxOrtho, "psdo: n_ortho out of range");
        ensure_ring(c, ring);
        ensure_hist(c, (long long)iters + 1);
        SolverState* h = c->st_host;
        std::memset(h, 0, sizeof(SolverState));
        h->tol_reduction = 1e-300;
        h->max_iters = iters;
        h->n_ortho = cfg->n_ortho;
        h->normalize = cfg->normalize_before_precond ? 1 : 0;
        h->ring = ring;
        CK(cudaMemcpyAsync(c->st, h, sizeof(SolverState), cudaMemcpyHostToDevice, c->s));
        const int ns = cfg->nullspace_projection ? 1 : 0;
        require(cfg->precond >= 0 && cfg->precond <= 2, "psdo: precond must be 0, 1 or 2");
        c->solve_ident = cfg->precond;
        ensure_x1_clean(c, c->s);
        std::vector<Step> pro, bod;
        if (c->dim == 3) {
            pro = prologue_steps<3>(c, 0, 0, ns);
            bod = body_steps<3>(c, 0, 0, ns, cfg->n_ortho);
        } else {
            pro = prologue_steps<2>(c, 0, 0, ns);
            bod = body_steps<2>(c, 0, 0, ns, cfg->n_ortho);
        }
        for (const auto& st : pro) st.run(c->s);
        const size_t nk = bod.size();
        while (c->prof_ev.size() < nk + 1) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            c->prof_ev.push_back(e);
        }
        std::vector<double> acc(nk, 0.0);
        for (int it = 0; it < iters; ++it) {
            for (size_t k = 0; k < nk; ++k) {
                CK(cudaEventRecord(c->prof_ev[k], c->s));
                bod[k].run(c->s);
            }
            CK(cudaEventRecord(c->prof_ev[nk], c->s));
            CK(cudaEventSynchronize(c->prof_ev[nk]));
            for (size_t k = 0; k < nk; ++k) {
                float ms = 0.0f;
                CK(cudaEventElapsedTime(&ms, c->prof_ev[k], c->prof_ev[k + 1]));
                acc[k] += ms;
            }
        }
        const int cap = *n_out;
        *n_out = (int)nk;
        for (size_t k = 0; k < nk && (int)k < cap; ++k) {
            if (ms_out) ms_out[k] = acc[k] / iters;
            if (names && name_len > 0) {
                std::strncpy(names + k * (size_t)name_len, bod[k].name.c_str(), (size_t)name_len - 1);
                names[k * (size_t)name_len + name_len - 1] = 0;
            }
        }
        CK(cudaStreamSynchronize(c->s));
        // the profiled iterations leave the solver vectors dirty at fluid cells
        // only; the zero invariant at non-fluid cells still holds.
    });
}

}  // extern "C"

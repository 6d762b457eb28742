/*
 * npsd_b200.h — C ABI of the B200-native neural-preconditioned PSDO ("DCDM")
 * Poisson solve. Plain pointers and sizes only; no torch or C++ types.
 *
 * Each entry point replaces one reference interface on the hot path
 * (/root/reference/proj, C++ library `npsd`):
 *
 *   npsd_b200_create         net::NeuralPrecond ctor / net::neural_precond
 *                            (include/npsd/net/precond.hpp:14-33,
 *                            src/net_precond.cpp:9-12, 37-40) for the weights;
 *                            the grid (dims, depth) comes from the
 *                            IndicatorImage and NetContext::build's
 *                            divisibility rule (net/forward.hpp:56-62)
 *   npsd_b200_set_mask       the per-frame part of the same ctor:
 *                            IndicatorImage -> ReductionMap::from_image
 *                            (src/discretization.cpp:5-19) + NetContext::build
 *                            (net/forward.hpp:56-93) + assemble_poisson[_3d]
 *                            (src/discretization.cpp:21-127; matrix-free here)
 *   npsd_b200_precond_apply  Preconditioner::apply (include/npsd/precond.hpp:17)
 *                            as NeuralPrecond::apply (src/net_precond.cpp:14-35)
 *   npsd_b200_psdo_solve     psdo_solve (include/npsd/solver.hpp:64-65,
 *                            src/solver.cpp:189-276); n_ortho = 0 is psd_solve
 *                            (solver.hpp:68-69)
 *   npsd_b200_spmv           spmv on the reduced matrix (include/npsd/sparse.hpp:38-39)
 *   npsd_b200_net_apply      NetContext<float>::apply (net/forward.hpp:95-129)
 *
 * Every call returns a status: NPSD_OK, or the code of the exception the
 * reference would throw — NPSD_INVALID_ARGUMENT (npsd::require ->
 * std::invalid_argument, types.hpp:30-32), NPSD_BREAKDOWN (SolverBreakdown,
 * solver.cpp:247-250), NPSD_EMPTY_SYSTEM (EmptySystemError,
 * discretization.cpp:137), NPSD_CUDA_ERROR (device failure; there is no CPU
 * fallback). npsd_b200_last_error(ctx) returns the message.
 *
 * Layouts: grids are x-fastest, linear index (z*ny + y)*nx + x
 * (discretization.hpp:38); cell types 0 fluid, 1 air, 2 solid (scene.hpp:11);
 * "reduced" vectors hold the n_f fluid cells in ascending linear order
 * (ReductionMap). Weights are f32 in for_each_span order (net/params.hpp:66-80)
 * with 9 slots in 2D and 27 in 3D (see DESIGN.md for the 3D layout).
 */
#ifndef NPSD_B200_H
#define NPSD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    NPSD_OK = 0,
    NPSD_INVALID_ARGUMENT = 1,
    NPSD_BREAKDOWN = 2,
    NPSD_EMPTY_SYSTEM = 3,
    NPSD_CUDA_ERROR = 4,
    NPSD_IO_ERROR = 5
};

typedef struct npsd_b200_ctx npsd_b200_ctx;
typedef struct npsd_b200_comm npsd_b200_comm;

/* SolveConfig (include/npsd/solver.hpp:11-26) as a POD. */
typedef struct {
    double tol_reduction;         /* stop when ||r_k|| <= tol_reduction * ||r_0||, in (0,1) */
    double tol_abs;               /* optional absolute stop, active when > 0 */
    int64_t max_iters;
    int32_t n_ortho;              /* A-orthogonalise against the last n_ortho directions (0..8) */
    int32_t nullspace_projection; /* bool */
    int32_t normalize_before_precond; /* bool */
    int32_t precond;              /* psdo: 0 = the network (NeuralPrecond), 1 = IdentityPrecond
                                     (precond.cpp:7-10: d = r / ||r||), 2 = JacobiPrecond
                                     (precond.cpp:12-26; single-domain); pcg takes its own argument */
} npsd_b200_solve_cfg;

/* SolveReport (include/npsd/solver.hpp:28-37). residual_history and
 * cumulative_seconds point into ctx-owned memory valid until the next solve. */
typedef struct {
    int64_t iterations;
    int32_t converged;
    int32_t breakdown;
    const double* residual_history;   /* ||r_0|| ... ||r_k||, length history_len = iterations + 1 */
    const double* cumulative_seconds; /* device %globaltimer at each history entry, from the solve's first
                                         kernel (solver.cpp:192,212,263); entry 0 = setup_seconds */
    int64_t history_len;
    double setup_seconds;    /* set_mask excluded: projections, r0 = b - A x0 and its norm (solver.cpp:211) */
    double iterate_seconds;  /* device solve time minus setup_seconds (solver.cpp:275) */
    double precond_seconds;  /* sum of the per-iteration preconditioner spans (solver.cpp:230-237), from
                                %globaltimer stamps: end of the previous iteration -> start of the first
                                kernel after the network (includes the launch gaps between them) */
} npsd_b200_report;

/* Weights: n_params f32 in for_each_span order for (dim, depth).
 * devices/n_devices: CUDA ordinals; one device per context in this build. */
int npsd_b200_create(int dim, int nx, int ny, int nz, int depth, const float* params, size_t n_params,
                     const int* devices, int n_devices, npsd_b200_ctx** out);
int npsd_b200_destroy(npsd_b200_ctx* ctx);
const char* npsd_b200_last_error(const npsd_b200_ctx* ctx); /* ctx may be NULL (create errors) */

/* Network arithmetic. exact = 0 (the default): fused multiply-adds, one
 * accumulation chain per window plane, and the level-0 up convolution's taps
 * merged per fine-cell parity (upsampling maps 27 fine taps onto 8 coarse
 * cells) — the preconditioner output stays within the north_star tolerance
 * (1e-5 relative L2 of the reference's) but is not bitwise. exact = 1: every
 * network operation in the reference's order with round-to-nearest
 * multiplies and adds (apply_kernels, net/kernels.hpp:147-172): outputs
 * bit-identical to the CPU restatement. The solver (f64) is the same in both. */
int npsd_b200_set_exact(npsd_b200_ctx* ctx, int exact);

/* Replace the weights (same dim/depth); the next set_mask rebuilds tables. */
int npsd_b200_set_params(npsd_b200_ctx* ctx, const float* params, size_t n_params);

/* Per-frame setup from nx*ny*nz cell types (host or device pointer). */
int npsd_b200_set_mask(npsd_b200_ctx* ctx, const uint8_t* cell_types);
int npsd_b200_set_mask_device(npsd_b200_ctx* ctx, const uint8_t* d_cell_types);

/* Number of fluid cells of the current mask (the reduced system size). */
int64_t npsd_b200_n_fluid(const npsd_b200_ctx* ctx);
/* Ascending fluid cell linear indices (length n_fluid). */
int npsd_b200_fluid_indices(npsd_b200_ctx* ctx, int64_t* out);

/* is_pure_neumann (discretization.cpp:180-191) of the current mask, 3D with
 * six face neighbours: *out = 1 when no fluid cell has an air face neighbour
 * (outside the domain is solid), i.e. the reduced system is singular and the
 * caller should set nullspace_projection (bench.cpp:52, npsd_cli.cpp:280). */
int npsd_b200_is_pure_neumann(npsd_b200_ctx* ctx, int* out);

/* Checks a caller's reduced CSR matrix (SparseMatrix, sparse.hpp:11-18:
 * n_rows, row_offsets[n_rows+1], col_indices/values[nnz]) against the
 * flag-derived operator the solve uses (assemble_poisson[_3d] + reduce,
 * discretization.cpp:21-160): row count, every row's nnz, diagonal value and
 * -1 off-diagonals; with full != 0 also A v for a fixed pseudo-random v,
 * computed here in CSR order like spmv (sparse.cpp:100-117), bitwise against
 * the device operator. NPSD_INVALID_ARGUMENT names the first mismatching row. */
int npsd_b200_check_operator(npsd_b200_ctx* ctx, int64_t n_rows, const int64_t* row_offsets,
                             const int64_t* col_indices, const double* values, int64_t nnz, int full);

/* Preconditioner::apply on reduced host vectors (NeuralPrecond semantics). */
int npsd_b200_precond_apply(npsd_b200_ctx* ctx, const double* r_reduced, double* z_reduced, int64_t n_f);

/* psdo_solve on reduced host vectors; x0 may be NULL (zero start). */
int npsd_b200_psdo_solve(npsd_b200_ctx* ctx, const double* b_reduced, const double* x0_reduced,
                         const npsd_b200_solve_cfg* cfg, double* x_reduced, npsd_b200_report* rep);

/* The same with the caller's vector length n_b (b, x0 and x hold n_b
 * entries; NPSD_INVALID_ARGUMENT unless n_b equals the fluid count). With
 * the length known up front, the rhs upload overlaps a set_mask still
 * running on the device (npsd_b200_psdo_solve waits for the frame's setup
 * to learn the length first). */
int npsd_b200_psdo_solve_n(npsd_b200_ctx* ctx, const double* b_reduced, int64_t n_b, const double* x0_reduced,
                           const npsd_b200_solve_cfg* cfg, double* x_reduced, npsd_b200_report* rep);

/* Same solve on device-resident FULL-GRID vectors (n_c = nx*ny*nz doubles,
 * zero at non-fluid cells): b in, x0 in (may be NULL), x out. */
int npsd_b200_psdo_solve_device(npsd_b200_ctx* ctx, const double* d_b_full, const double* d_x0_full,
                                const npsd_b200_solve_cfg* cfg, double* d_x_full, npsd_b200_report* rep);

/* Reduced y = A x with the matrix-free 7/5-point operator. */
int npsd_b200_spmv(npsd_b200_ctx* ctx, const double* x_reduced, double* y_reduced, int64_t n_f);

/* Raw network on the full grid (f32, n_c values). */
int npsd_b200_net_apply(npsd_b200_ctx* ctx, const float* x_full, float* y_full);

/* Introspection for parity tests: coarsened indicator image of a level
 * (3 planes of level cells), the linear-block coefficients z_a/z_b per level
 * (depth-1 each), and the mixed-window cell count per level. */
int npsd_b200_level_image(npsd_b200_ctx* ctx, int level, float* out);
int npsd_b200_linear_coeffs(npsd_b200_ctx* ctx, float* za, float* zb);
int npsd_b200_mixed_counts(npsd_b200_ctx* ctx, int64_t* counts);

/* Deterministic inputs (mirror rng.hpp / net_params.cpp; host side). */
size_t npsd_b200_param_count(int dim, int depth);
int npsd_b200_init_params(int dim, int depth, uint64_t seed, float* out);
int npsd_b200_identity_params(int dim, int depth, float* out);
void npsd_b200_rhs_normal(uint64_t seed, int64_t n, double* out);

/* Preconditioned CG on the device, replacing pcg_solve / cg_solve
 * (solver.cpp:36-109): precond 0 = identity (cg_solve), 1 = Jacobi
 * (precond.cpp:12-26; NPSD_INVALID_ARGUMENT "jacobi precond: zero diagonal"
 * like the reference's constructor), 2 = IC0 (precond.cpp:28-112, see
 * npsd_b200_ic0_apply; factored per solve on the current frame). Same vectors, report and errors as
 * psdo_solve (nullspace projection as pcg_solve :45-48, 82); n_ortho,
 * normalize_before_precond and precond of the cfg are ignored. The baseline the
 * paper compares NPSDO with. */
int npsd_b200_pcg_solve(npsd_b200_ctx* ctx, const double* b, const double* x0, const npsd_b200_solve_cfg* cfg,
                        int precond, double* x, npsd_b200_report* rep);
int npsd_b200_pcg_solve_device(npsd_b200_ctx* ctx, const double* d_b, const double* d_x0,
                               const npsd_b200_solve_cfg* cfg, int precond, double* d_x, npsd_b200_report* rep);

/* Ic0Precond (precond.cpp:28-112) on the current frame: the constructor's
 * factorization (diagonal-shift retries; *shift_retries may be NULL) then
 * apply(r, z): forward L y = r and backward L^T z = y, level-scheduled over
 * the hyperplanes x + y + z = const. Bit-identical to the reference's loops;
 * NPSD_INVALID_ARGUMENT "ic0: factorization failed after diagonal-shift
 * retries" where the reference throws. */
int npsd_b200_ic0_apply(npsd_b200_ctx* ctx, const double* r, double* z, int64_t n_f, int* shift_retries);

/* Right-hand side from a MAC velocity field, replacing mac_divergence_rhs
 * (discretization.cpp:193-227) + reduce: b = -(rho*h/dt) * (signed sum of face
 * velocities) at fluid cells, a face whose opposite cell is solid (or outside
 * the domain) taking the boundary value (bc arrays NULL: 0). 3D adds w faces
 * (the reference is 2D only). Face arrays x fastest: u (nx+1, ny, nz),
 * v (nx, ny+1, nz), w (nx, ny, nz+1); 2D passes w = bc_w = NULL. Needs the
 * frame's set_mask. Host variant: b_reduced (n_fluid entries, the solve's
 * ordering). Device variant: d_b_full on the full grid (zeros off fluid), the
 * input of psdo_solve_device — flags + velocity -> solve without leaving HBM. */
int npsd_b200_mac_divergence_rhs(npsd_b200_ctx* ctx, const double* u, const double* v, const double* w, double h,
                                 double dt, double rho, const double* bc_u, const double* bc_v, const double* bc_w,
                                 double* b_reduced);
int npsd_b200_mac_divergence_rhs_device(npsd_b200_ctx* ctx, const double* d_u, const double* d_v, const double* d_w,
                                        double h, double dt, double rho, const double* d_bc_u, const double* d_bc_v,
                                        const double* d_bc_w, double* d_b_full);

/* z-slab decomposition across GPUs ("Multi-GPU"): one process
 * (or, for tests, one host thread) and one context per rank; rank r owns
 * global planes [z0, z0 + nz_own) of an nx x ny x nz grid (3D, depth >= 2;
 * z0 and nz_own multiples of 2^(depth-1)). The per-rank calls are the
 * single-domain ones: set_mask takes the owned planes' types, precond_apply
 * / psdo_solve take the owned fluid cells' entries in ascending global order
 * (fluid_indices returns their global linear indices), and every rank gets
 * the same iteration count and residual history. Halo planes move over NCCL
 * (NVLink) before each stencil / conv level; dot products are gathered and
 * summed in rank order, so all ranks hold identical solver state.
 *
 * npsd_b200_nccl_unique_id: rank 0 makes the id (128 bytes) and the caller
 * broadcasts it (e.g. torch.distributed); every rank then creates its NCCL
 * communicator on its device. npsd_b200_comm_create_local: one communicator
 * shared by n contexts of one process on one device, each driven by its own
 * host thread (correctness tests of the decomposition; not a performance
 * path). net_apply, level_image, spmv and profile_iterations are single-domain
 * only. */
int npsd_b200_nccl_unique_id(void* id128);
int npsd_b200_comm_create_nccl(const void* id128, int rank, int nranks, int device, npsd_b200_comm** out);
int npsd_b200_comm_create_local(int nranks, npsd_b200_comm** out);
int npsd_b200_comm_destroy(npsd_b200_comm* comm);
const char* npsd_b200_comm_last_error(void);
/* 1 when the slab's last solve ran its iterations as captured chunk graphs
 * (NCCL communicators), 0 for eager launches */
int npsd_b200_slab_graph(const npsd_b200_ctx* c);
int npsd_b200_create_slab(int nx, int ny, int nz, int z0, int nz_own, int depth, const float* params,
                          size_t n_params, int device, npsd_b200_comm* comm, int rank, npsd_b200_ctx** out);

/* Model files, replacing npsd::net::save_npm / load_npm (net_params.cpp:42-78):
 * "NPMW", u32 version 1, u32 dim, u32 depth, then the weights in
 * for_each_span order as little-endian f32. dim 2 files are byte-identical to
 * the reference's; dim 3 is the 3D variant of the same layout (the reference
 * writes and accepts dim 2 only, net_params.cpp:45,64). Errors return
 * NPSD_IO_ERROR (the reference's std::runtime_error) with the reference's
 * message in npsd_b200_npm_last_error(); NPSD_INVALID_ARGUMENT for bad
 * arguments. load: out == NULL queries dim/depth/count only; otherwise cap
 * must hold the whole parameter vector. */
int npsd_b200_save_npm(const char* path, int dim, int depth, const float* params, size_t n);
int npsd_b200_load_npm(const char* path, int* dim, int* depth, float* out, size_t cap, size_t* n_out);
const char* npsd_b200_npm_last_error(void);

/* Device buffers and pinned host memory for callers without a CUDA runtime of
 * their own (the Python mirror uses these; the C++ shim may too). */
int npsd_b200_device_alloc(npsd_b200_ctx* ctx, size_t bytes, void** out);
int npsd_b200_device_free(npsd_b200_ctx* ctx, void* p);
int npsd_b200_host_alloc(npsd_b200_ctx* ctx, size_t bytes, void** out);
int npsd_b200_host_free(npsd_b200_ctx* ctx, void* p);
int npsd_b200_memcpy(npsd_b200_ctx* ctx, void* dst, const void* src, size_t bytes); /* any direction, on ctx stream */
int npsd_b200_synchronize(npsd_b200_ctx* ctx);

/* Device timing of a solve (CUDA events on the ctx stream around the device
 * solve graph; excludes host staging). Milliseconds of the last solve. */
double npsd_b200_last_solve_ms(const npsd_b200_ctx* ctx);
/* Kernel launches issued by the last solve (graph nodes executed). */
int64_t npsd_b200_last_solve_launches(const npsd_b200_ctx* ctx);
/* Cumulative kernel launches executed for this context (all calls). */
int64_t npsd_b200_launch_count(const npsd_b200_ctx* ctx);

/* CUDA events on the context stream (16 slots) for caller-side device timing. */
int npsd_b200_event_record(npsd_b200_ctx* ctx, int slot);
double npsd_b200_event_elapsed_ms(npsd_b200_ctx* ctx, int slot_a, int slot_b); /* waits for b; <0 on error */

/* Per-kernel device time of `iters` PSDO iterations launched one by one
 * between CUDA events (no graph) on device full-grid b; writes the mean ms per
 * kernel into ms_out and NUL-terminated kernel names (name_len bytes each).
 * *n_kernels: capacity in, count out. Leaves no solve state behind. */
int npsd_b200_profile_iterations(npsd_b200_ctx* ctx, const double* d_b_full, const npsd_b200_solve_cfg* cfg,
                                 int iters, double* ms_out, int* n_kernels, char* names, int name_len);

#ifdef __cplusplus
}
#endif

#endif /* NPSD_B200_H */

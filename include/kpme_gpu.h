/*
 * kpme_gpu.h -- C ABI of the B200-native SKP-PME reciprocal path.
 *
 * Drop-in boundary for the reference's header-only C++ API
 * (/root/reference/proj/include/kpme/, "the reference" below). Plain
 * pointers, sizes and POD structs only; no C++, torch or CUDA types appear
 * in any signature (CUDA streams are passed as void*). Every function that
 * can fail returns a status code; kpme_gpu_last_error() returns the message
 * of the last failure on the calling thread.
 *
 * Each entry point names the reference interface it replaces (file:line
 * relative to /root/reference/proj/). INTEGRATION.md shows the C++ wrapper
 * (include/kpme_b200/kpme.hpp) and the ctypes binding a maintainer adds.
 *
 * Layout conventions (shared with the reference):
 *   positions : double[n][3] (AoS, PointCloud::positions, geometry.hpp:43-47)
 *   charges   : double[n]    (ChargeVector::values, geometry.hpp:49-53)
 *   profiles  : double[nterms][3][2M+1], m = -M..M (SkpTerm, alpha.hpp:69-73)
 *   cell grids: double[K0*K1*K2][L^3]; cell c = (c0*K1 + c1)*K2 + c2
 *               (CellGrid::flatten, geometry.hpp:69-71), each L^3 block
 *               lexicographic with axis 0 slowest (tensor_weights,
 *               interpolation.hpp:52-58)
 *   meshes    : double[n0][n1][n2], n_a = K_a*L, lexicographic, axis 0
 *               slowest (kron.hpp:36-38)
 */
#ifndef KPME_GPU_H
#define KPME_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define KPME_GPU_ABI_VERSION 2

/* Status codes. The C++ wrapper rethrows 1 as std::invalid_argument,
 * 2 as std::runtime_error and 3 as kpme::numerical_error, the exception
 * contract of the reference (tools/kpme.cpp:415-424). */
enum {
    KPME_GPU_OK = 0,
    KPME_GPU_INVALID_ARGUMENT = 1,
    KPME_GPU_RUNTIME = 2,
    KPME_GPU_NUMERICAL = 3,
    KPME_GPU_CUDA = 4,
    KPME_GPU_NCCL = 5
};

/* SKP formulation of the grid operator. */
enum {
    KPME_GPU_FORM_AUTO = 0,      /* per-shape chooser (collapsed wins on configs 1-4) */
    KPME_GPU_FORM_COLLAPSED = 1, /* term-collapsed W^T (G .* (W phi)) form            */
    KPME_GPU_FORM_DENSE = 2      /* per-term dense n x n mode products on DMMA (D)    */
};

/* Everything kpme_apply receives besides the particles
 * (parallel.hpp:243-246): EwaldConfig (alpha.hpp:20-31), CellGrid
 * (geometry.hpp:63-111), order, SkpDecomposition (alpha.hpp:75-80) and
 * KpmeOptions (parallel.hpp:230-233). */
typedef struct {
    double xi;                  /* EwaldConfig.xi            */
    int modes;                  /* EwaldConfig.modes (M)     */
    double center[3];           /* CellGrid.box.center       */
    double radius;              /* CellGrid.box.radius       */
    int counts[3];              /* CellGrid.counts           */
    int order;                  /* interpolation order L     */
    int dec_modes;              /* SkpDecomposition.modes    */
    double correction;          /* SkpDecomposition.correction (c_Lambda) */
    int nterms;                 /* SkpDecomposition.terms.size() */
    const double* term_weights; /* [nterms] SkpTerm.weight   */
    const double* profiles;     /* [nterms][3][2M+1] SkpTerm.profiles */
    int fuse_terms;             /* KpmeOptions.fuse_terms (ledger shape only) */
    int threads;                /* KpmeOptions.threads (accepted, unused on GPU) */
    int device;                 /* CUDA device ordinal */
    int formulation;            /* KPME_GPU_FORM_* */
    /* ABI 2: several devices driven by one process (a multi-device plan:
     * z-slabs of whole cell planes, one per entry; see
     * kpme_gpu_plan_create_multi for other rank grids). ndevices <= 1 uses
     * `device` alone. */
    int ndevices;
    const int* devices;
} kpme_gpu_config;

typedef struct kpme_gpu_plan_s* kpme_gpu_plan;

const char* kpme_gpu_last_error(void);
int kpme_gpu_abi_version(void);

/* ---- host-side SKP construction (reference host code, unchanged role) -- */
/* sinc_rule (alpha.hpp:114-151); nodes/weights hold 2*n_quad+1 entries. */
int kpme_sinc_rule(int n_quad, int modes, double* nodes, double* weights,
                   double* lifting, double* eps);
/* sinc_rule_for_eps (alpha.hpp:154-161); nodes/weights hold 2*max_n+1. */
int kpme_sinc_rule_for_eps(double eps, int modes, int max_n, int* n_quad,
                           double* nodes, double* weights, double* lifting,
                           double* eps_out);
/* skp_from_quadrature (alpha.hpp:165-188). */
int kpme_skp_from_quadrature(int count, const double* nodes,
                             const double* weights, double min_arg,
                             double max_arg, double xi, int modes,
                             double* term_weights, double* profiles,
                             double* correction);
/* load_tabulated_rule (alpha.hpp:192-212). */
int kpme_load_tabulated_rule(const char* path, int cap, int* count,
                             double* nodes, double* weights, double* min_arg,
                             double* max_arg, double* eps);
/* assemble_alpha (alpha.hpp:54-65): the target tensor alpha(m), entries
 * [(2M+1)^3], m0 slowest, m = -M..M. */
int kpme_assemble_alpha(double xi, int modes, double* entries);
/* nkpa_svd (alpha.hpp:225-281): SVD-kind decomposition of alpha by two nested
 * truncated SVDs (host one-sided Jacobi). Writes up to cap terms:
 * term_weights[cap], profiles[cap][3][2M+1]; *nterms = the term count (call
 * with cap = 0 / NULL arrays to size); error_bound (nullable) = the a priori
 * Frobenius estimate. Correction is 0 (SkpKind::svd). The plan API consumes
 * these terms like any other (signed profiles ride on the factors,
 * symfourier.hpp:101-102). */
int kpme_nkpa_svd(int modes, const double* alpha, double tol_outer, double tol_inner,
                  int cap, int* nterms, double* term_weights, double* profiles,
                  double* error_bound);
/* sample_cloud (geometry.hpp:238-251), splitmix64. */
void kpme_sample_cloud(const double center[3], double radius, int64_t n,
                       uint64_t seed, double* xyz, double* q);
/* KpmeResult.ledger (parallel.hpp:84-96, 110-138), synthesised: 4 int64 per
 * row (rank, step, group_axis, payload); returns the row count in *rows. */
int kpme_gpu_ledger(const kpme_gpu_config* cfg, int64_t* out, int64_t cap,
                    int64_t* rows);

/* ---- one-shot call ----------------------------------------------------- */
/* kpme_apply (parallel.hpp:243-290) on host buffers: potentials[n] in
 * global particle order, including -c_Lambda * sum(q). Plans are cached per
 * configuration (decomposition contents included) and device list, so
 * repeated one-shot calls skip the factor build and the allocations;
 * KPME_GPU_PLAN_CACHE=0 disables the cache. */
int kpme_gpu_apply(const kpme_gpu_config* cfg, int64_t n, const double* xyz,
                   const double* q, double* potentials);
/* Frees every cached plan of kpme_gpu_apply. */
int kpme_gpu_apply_cache_clear(void);

/* ---- plan API (steady state) ------------------------------------------- */
/* Builds factor tables (W_a, the collapsed core G, dense A_a(lambda) when
 * the dense form is selected) and sizes buffers for up to max_particles. */
int kpme_gpu_plan_create(const kpme_gpu_config* cfg, int64_t max_particles,
                         kpme_gpu_plan* out);
int kpme_gpu_plan_destroy(kpme_gpu_plan plan);
/* The plan runs on this stream from now on (cudaStream_t as void*; NULL =
 * the legacy default stream, which cannot be graph-captured). A new plan
 * owns a non-blocking stream. */
int kpme_gpu_plan_set_stream(kpme_gpu_plan plan, void* stream);
/* Host buffers; H2D of xyz/q and D2H of potentials happen inside. Large
 * calls are pipelined in particle chunks: each chunk is sorted and spread
 * while the next one crosses PCIe, and the potentials leave chunk by chunk
 * behind the gather. Pinned host buffers give full overlap. */
int kpme_gpu_plan_execute(kpme_gpu_plan plan, int64_t n, const double* xyz,
                          const double* q, double* potentials);
/* Chunk count of kpme_gpu_plan_execute: -1 automatic (one chunk per ~1/3 M
 * particles, at most 3), 1 = unpipelined, else 2..8. */
int kpme_gpu_plan_set_host_chunks(kpme_gpu_plan plan, int chunks);
/* Device buffers, stream-ordered. flags & KPME_GPU_DEFER_CHECKS skips the
 * stream synchronisation that reports invalid particles; call
 * kpme_gpu_plan_status() later instead. */
#define KPME_GPU_DEFER_CHECKS 1
int kpme_gpu_plan_execute_device(kpme_gpu_plan plan, int64_t n,
                                 const double* d_xyz, const double* d_q,
                                 double* d_potentials, int flags);
/* Synchronises the plan's stream and reports deferred argument errors
 * (particle outside the box, geometry.hpp:136-138). */
int kpme_gpu_plan_status(kpme_gpu_plan plan);
/* Number of kernel launches one execute issues (for bench accounting). */
int kpme_gpu_plan_launches(kpme_gpu_plan plan);
/* Capture execute_device into a CUDA graph and replay it (same pointers). */
int kpme_gpu_plan_graph_execute(kpme_gpu_plan plan, int64_t n,
                                const double* d_xyz, const double* d_q,
                                double* d_potentials);
/* Per-stage device times (ms) of the last execute when timing is on. */
int kpme_gpu_plan_enable_timing(kpme_gpu_plan plan, int on);
int kpme_gpu_plan_stage_times(kpme_gpu_plan plan, double* ms, int cap,
                              int* count);

/* ---- z-slab plans (multi-GPU, one process per GPU) ---------------------- */
/* A plan owning cell planes [z_lo, z_hi) along axis 2 (the slab of one
 * rank). Particles passed to it must lie in the slab (else
 * KPME_GPU_INVALID_ARGUMENT at the next status check). The collapsed form's
 * only exchange is a sum over ranks of the R^3 + 1 core (R = 2M+1; the last
 * entry carries sum(q)), done by the caller between the two halves below --
 * the distributed counterpart of the axis-group reductions of spkmv
 * (parallel.hpp:169-176) and allreduce_scalar (parallel.hpp:254-257). */
int kpme_gpu_plan_create_slab(const kpme_gpu_config* cfg, int64_t max_particles,
                              int z_lo, int z_hi, kpme_gpu_plan* out);
/* General P0 x P1 x P2 device grids: a plan owning the cell block
 * [lo[a], hi[a]) on every axis -- one rank of a rank grid that flattens like
 * cells (RankGrid, parallel.hpp:46-82). The same forward / core all-reduce /
 * backward halves as slabs; particles outside the block are
 * KPME_GPU_INVALID_ARGUMENT at the next status check. */
int kpme_gpu_plan_create_block(const kpme_gpu_config* cfg, int64_t max_particles,
                               const int lo[3], const int hi[3], kpme_gpu_plan* out);
int kpme_gpu_plan_core_size(kpme_gpu_plan plan);
/* sort .. forward contractions: d_core[R^3 + 1] = this slab's partial core */
int kpme_gpu_plan_forward(kpme_gpu_plan plan, int64_t n, const double* d_xyz,
                          const double* d_q, double* d_core);
/* core (summed over slabs) -> backward contractions -> gather - c*sum(q) */
int kpme_gpu_plan_backward(kpme_gpu_plan plan, const double* d_core,
                           double* d_potentials);

/* ---- multi-device plans (one process drives several GPUs) --------------- */
/* The reference's rank-grid decomposition of kpme_apply (RankGrid,
 * parallel.hpp:46-82; SimulatedComm, parallel.hpp:98-145) on one node: a
 * P0 x P1 x P2 grid of cell blocks, block r on cfg->devices[r] (ranks flatten
 * like cells). Every device keeps its block's particles (routing on device),
 * sorts, spreads and contracts them into a partial core; the partial cores
 * are summed (the collapsed form's only exchange, replacing the axis-group
 * reductions of spkmv, parallel.hpp:169-176, and allreduce_scalar,
 * parallel.hpp:254-257); every device gathers its particles and the home
 * device (devices[0]) returns all potentials in global order.
 * kpme_gpu_plan_create with cfg->ndevices > 1 makes a (1, 1, ndevices) grid.
 * execute and execute_device (buffers on the home device) and status work on
 * a multi-device plan; the stage entry points, graphs and timing do not. */
enum {
    KPME_GPU_COLL_AUTO = 0, /* PEER when every device pair has peer access, else NCCL */
    KPME_GPU_COLL_PEER = 1, /* each device sums all partial cores from peer memory
                               (NVLink), in rank order: no NCCL round, same bits everywhere */
    KPME_GPU_COLL_NCCL = 2  /* one grouped ncclAllReduce over the plan's own communicators */
};
int kpme_gpu_plan_create_multi(const kpme_gpu_config* cfg, int64_t max_particles,
                               const int dims[3], kpme_gpu_plan* out);
int kpme_gpu_plan_set_collective(kpme_gpu_plan plan, int mode);
/* The exchange in use (KPME_GPU_COLL_*), or -1 for a single-device plan. */
int kpme_gpu_plan_collective(kpme_gpu_plan plan);
/* Device entries of the plan (count returned; up to cap written). */
int kpme_gpu_plan_devices(kpme_gpu_plan plan, int* devices, int cap);

/* ---- one process per GPU: a block plan owning an NCCL communicator ------ */
/* Rank r of an nranks-process job (torchrun / MPI) builds its block plan
 * (kpme_gpu_plan_create_slab/_block), rank 0 makes an id, the job broadcasts
 * the 128 bytes, and every rank attaches. From then on execute_device and
 * graph_execute run forward half -> ncclAllReduce of the core -> backward
 * half on the plan's stream (capturable as one graph). */
#define KPME_GPU_NCCL_ID_BYTES 128
int kpme_gpu_nccl_unique_id(void* id);
int kpme_gpu_plan_attach_comm(kpme_gpu_plan plan, int nranks, int rank, const void* id);

/* ---- stage entry points (device buffers, plan stream) ------------------ */
/* assign_particles (geometry.hpp:131-154), bit-exact: perm[n] is the
 * concatenation of Partition.members in flattened cell order,
 * cell_start[K0*K1*K2+1]. */
int kpme_gpu_sort(kpme_gpu_plan plan, int64_t n, const double* d_xyz,
                  int32_t* d_perm, int32_t* d_cell_start);
/* InterpOperator::interpolate (interpolation.hpp:84-92). */
int kpme_gpu_spread(kpme_gpu_plan plan, int64_t n, const double* d_xyz,
                    const double* d_q, double* d_phi_cells);
/* spkmv_sum (parallel.hpp:184-228) over all terms, per-cell grids in/out. */
int kpme_gpu_skp_apply(kpme_gpu_plan plan, const double* d_phi_cells,
                       double* d_psi_cells);
/* InterpOperator::anterpolate (interpolation.hpp:95-105), no correction. */
int kpme_gpu_gather(kpme_gpu_plan plan, int64_t n, const double* d_xyz,
                    const double* d_psi_cells, double* d_out);

/* ---- dense SKP grid operator (config 5; kron.hpp:180-197 semantics) ---- */
/* y = sum_r (A_r (x) B_r (x) C_r) x on an n0 x n1 x n2 lexicographic mesh,
 * A_r: [nterms][n0][n0], B_r: [nterms][n1][n1], C_r: [nterms][n2][n2]
 * row-major, all device pointers. Runs the FP64 DMMA mode-product kernel;
 * work buffers are allocated per call unless a workspace is given
 * (kpme_gpu_dense_workspace_bytes). */
size_t kpme_gpu_dense_workspace_bytes(int n0, int n1, int n2, int nterms);
int kpme_gpu_kron_matvec_dense(int device, void* stream, int n0, int n1,
                               int n2, int nterms, const double* d_A,
                               const double* d_B, const double* d_C,
                               const double* d_x, double* d_y,
                               void* d_workspace, size_t workspace_bytes);
/* Dense full-axis operands A_a(lambda) = W_a^T diag(d_{lambda,a}) W_a
 * (n_a x n_a, symfourier.hpp:108-124 assembled over all cells of the axis)
 * for the plan's decomposition: d_out[nterms][n_a][n_a]. */
int kpme_gpu_plan_axis_operands(kpme_gpu_plan plan, int axis, double* d_out);
/* The FP64 GEMM the dense form is built from: out[m][i] (+)= sum_k
 * in[k][m] * F[i][k]  (M x N result, K contraction); accumulate != 0 adds
 * into out. Exposed for the FP64 DMMA roofline probe and tests. */
int kpme_gpu_dgemm_tn(void* stream, int64_t M, int64_t N, int64_t K,
                      const double* d_in, const double* d_F, double* d_out,
                      int accumulate);

/* ---- dense operator on z-slabs (config 5, multi-GPU) --------------------- */
/* y = sum_r (A_r (x) B_r (x) C_r) x with x, y distributed as z-slabs
 * [n0][n1][z_hi - z_lo] (rank order = z order, balanced split of n2; see
 * kpme_gpu_dense_slab_bounds). The three strategies for the sharded z
 * product (the reference's axis-group reduction, parallel.hpp:169-176, and
 * the north star's slab all-to-all and rank split + reduce); every local
 * product is the FP64 DMMA GEMM. */
enum {
    KPME_GPU_SLAB_REDUCE_SCATTER = 0, /* z contracted from the local slice, one reduce-scatter */
    KPME_GPU_SLAB_RANK_SPLIT = 1,     /* all-gather, terms split over ranks, reduce-scatter   */
    KPME_GPU_SLAB_ALLTOALL = 2        /* all-to-all z <-> x transpose around the z product      */
};
typedef struct kpme_gpu_dense_slab_s* kpme_gpu_dense_slab;
/* Rank `rank` of an nranks-process job on `device`; A, B, C: the full
 * [nterms][n][n] operands in that device's memory; nccl_id: 128 bytes from
 * kpme_gpu_nccl_unique_id on rank 0 (NULL when nranks == 1). The handle owns
 * its NCCL communicator, streams and every work buffer. */
int kpme_gpu_dense_slab_create(int device, int n0, int n1, int n2, int nterms,
                               const double* A, const double* B, const double* C,
                               int nranks, int rank, const void* nccl_id,
                               kpme_gpu_dense_slab* out);
/* All nranks ranks in this process, rank r on devices[r] (devices may
 * repeat); collectives by peer copies in rank order. A/B/C: per-rank device
 * pointers. */
int kpme_gpu_dense_slab_create_group(int nranks, const int* devices, int n0, int n1,
                                     int n2, int nterms, const double* const* A,
                                     const double* const* B, const double* const* C,
                                     kpme_gpu_dense_slab* out);
int kpme_gpu_dense_slab_destroy(kpme_gpu_dense_slab h);
int kpme_gpu_dense_slab_bounds(kpme_gpu_dense_slab h, int rank, int* z_lo, int* z_hi);
/* Stream of local rank `local` (0 for a process rank; 0..nranks-1 for a group). */
int kpme_gpu_dense_slab_set_stream(kpme_gpu_dense_slab h, int local, void* stream);
/* x_local/y_local: one device pointer per local rank. Stream-ordered on the
 * handle's streams; kpme_gpu_dense_slab_sync waits for them. */
int kpme_gpu_dense_slab_apply(kpme_gpu_dense_slab h, int strategy,
                              const double* const* x_local, double* const* y_local);
int kpme_gpu_dense_slab_sync(kpme_gpu_dense_slab h);
/* Times every strategy (CUDA events, reps applications each, max over
 * ranks) and returns the fastest in *best; ms[3] gets the per-apply times. */
int kpme_gpu_dense_slab_choose(kpme_gpu_dense_slab h, const double* const* x_local,
                               double* const* y_local, int reps, double* ms, int* best);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* KPME_GPU_H */

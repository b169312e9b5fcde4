/*
 * gb_bal.h — C ABI of the B200-native Levenberg–Marquardt bundle-adjustment
 * solver (the LM inner loop of arXiv 2509.26581, reference `gopt`).
 *
 * This is the drop-in boundary for the reference's hot path. Each entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj). Plain pointers and sizes only: no C++ or torch types.
 *
 * Element types follow the reference's precision pairs
 * (src/experiment.cpp:153-157):
 *   GB_FP64       graph FP = double, system SP = double
 *   GB_FP32       graph FP = float,  system SP = float
 *   GB_FP32_BF16  graph FP = float,  system SP = bfloat16 (uint16 storage,
 *                 include/gopt/bfloat16.hpp:12-37), arithmetic in float
 * Buffers documented as "FP" hold double for GB_FP64 and float otherwise;
 * "SP" buffers hold double / float / uint16 bf16 bits; "Arith" buffers hold
 * double for GB_FP64 and float otherwise.
 *
 * Error model: every int-returning call returns GB_OK or one of the GB_ERR_*
 * codes, which map one-to-one onto the exception the reference throws in the
 * same situation; gb_last_error() returns the message.
 */
#ifndef GB_BAL_H_
#define GB_BAL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define GB_OK 0
#define GB_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument (vertex_descriptor.hpp:71-74,
                                     factor_descriptor.hpp:553-555, precision.hpp:44-49) */
#define GB_ERR_OUT_OF_RANGE 2     /* std::out_of_range (factor_descriptor.hpp:543-547) */
#define GB_ERR_LOGIC 3            /* std::logic_error (graph.hpp:64-65, 92) */
#define GB_ERR_RUNTIME 4          /* std::runtime_error (levenberg_marquardt.hpp:133-134) */
#define GB_ERR_CUDA 5             /* device failure (no reference counterpart) */
#define GB_ERR_NO_DEVICE 6        /* no CUDA device: the device path never falls back to CPU */

/* ---- enums (values match the reference enum order) ---------------------- */
/* bench/experiment.hpp:16 PrecisionMode */
#define GB_FP64 0
#define GB_FP32 1
#define GB_FP32_BF16 2
/* factor_descriptor.hpp:23 DifferentiationMode */
#define GB_ANALYTIC 0
#define GB_AUTO 1
#define GB_DYNAMIC 2
/* loss.hpp:10 LossKind */
#define GB_LOSS_DEFAULT 0
#define GB_LOSS_HUBER 1
/* factor_descriptor.hpp:37 DampingPlacement */
#define GB_DAMPING_AFTER_SCALING 0
#define GB_DAMPING_BEFORE_SCALING 1
/* linear solver of the LM step (gb_set_linear_solver) */
#define GB_SOLVER_PCG 0   /* matrix-free PCG on the full system (the reference, linear_system.hpp:185-207) */
#define GB_SOLVER_SCHUR 1 /* Schur complement onto the cameras (north star (c); no reference counterpart) */
/* levenberg_marquardt.hpp:28-35 Termination */
#define GB_TERM_MAX_ITERATIONS 0
#define GB_TERM_TOLERANCE_REACHED 1
#define GB_TERM_GRADIENT_SMALL 2
#define GB_TERM_DAMPING_OVERFLOW 3
#define GB_TERM_NON_FINITE_LINEARIZATION 4
#define GB_TERM_NO_FREE_PARAMETERS 5

/* ---- configuration (same fields and defaults as the reference) ---------- */
/* pcg.hpp:12-17 PCGConfig */
typedef struct gb_pcg_config {
  int32_t max_iterations;  /* 50 */
  double tolerance;        /* 1e-6 */
  double rejection_ratio;  /* 10 */
  int32_t normalize_rhs;   /* 1 */
} gb_pcg_config;

/* pcg.hpp:19-23 PCGStats */
typedef struct gb_pcg_stats {
  int32_t iterations;
  double final_relative_residual;
  int32_t converged;
} gb_pcg_stats;

/* levenberg_marquardt.hpp:15-26 LMConfig + linear_system.hpp:15-19 LinearSystemOptions */
typedef struct gb_lm_config {
  int32_t max_iterations;      /* 10 */
  double tolerance;            /* 1e-6 */
  int32_t level;               /* 0 */
  double tau;                  /* 1e-4 */
  gb_pcg_config pcg;
  double clamp_min;            /* 1e-6 */
  double clamp_max;            /* 1e32 */
  int32_t damping;             /* GB_DAMPING_AFTER_SCALING */
  int32_t use_rejection_guard; /* 1 */
  int32_t refresh_on_reject;   /* 0 */
  double lambda_max;           /* 1e32 */
  double gradient_tolerance;   /* 1e-12 */
} gb_lm_config;

/* levenberg_marquardt.hpp:49-61 IterationRecord */
typedef struct gb_iteration_record {
  int32_t iteration;
  double chi2_before;
  double chi2_after;
  double lambda;
  int32_t pcg_iterations;
  int32_t pcg_converged;
  double pcg_relative_residual;
  int32_t low_quality_step;
  int32_t precond_fallback_blocks;
  int32_t accepted;
  double wall_seconds;
} gb_iteration_record;

/* levenberg_marquardt.hpp:63-68 MemoryAccount (analytic, SPEC "Memory accounting") */
typedef struct gb_memory_account {
  uint64_t jacobian_bytes;
  uint64_t preconditioner_bytes;
  uint64_t workspace_bytes;
  uint64_t graph_bytes;
} gb_memory_account;

/* levenberg_marquardt.hpp:72-83 SolveReport (iterations returned separately) */
typedef struct gb_solve_report {
  double initial_chi2;
  double final_chi2;
  int32_t accepted_steps;
  int32_t termination;
  double total_seconds;
  int64_t free_dims;
  int64_t residual_dims;
  uint64_t active_factors;
  gb_memory_account memory;
  int32_t iterations_run;
  /* device-side extras (no reference field): */
  double setup_seconds;    /* host->device upload + activation + initial linearize */
  double h2d_bytes;
  double d2h_bytes;
} gb_solve_report;

typedef struct gb_graph gb_graph;

/* Fills the reference defaults (levenberg_marquardt.hpp:15-26, pcg.hpp:12-17,
 * linear_system.hpp:15-19). */
void gb_default_config(gb_lm_config* cfg);

/* Last error message of the calling thread ("" if none). */
const char* gb_last_error(void);

/* Number of visible CUDA devices (0 on a host without a GPU). */
int gb_device_count(void);

/* ---- graph construction -------------------------------------------------
 * Replaces bal::build_graph<FP,SP> (include/gopt/bal/adapter.hpp:106-143),
 * which builds CameraDescriptor / Point3Descriptor / ReprojectionFactor and a
 * Graph<FP,SP> (graph.hpp:26-45). precision is a GB_FP* code, diff_mode a
 * GB_* differentiation mode (factor_descriptor.hpp:230-235). device is the
 * CUDA ordinal this handle runs on. Returns NULL on error (gb_last_error). */
gb_graph* gb_create(int precision, int diff_mode, int device);
void gb_destroy(gb_graph* g);

/* Cameras: AoS FP[9*n] in the Snavely layout [w1 w2 w3 t1 t2 t3 f k1 k2]
 * (bal/snavely.hpp:47). The buffer is the user's vertex storage and is
 * refined IN PLACE by gb_optimize (CameraTraits::update, adapter.hpp:16-28);
 * it must stay valid for the handle's lifetime. fixed: NULL or uint8[n]
 * (VertexDescriptor::set_fixed, vertex_descriptor.hpp:80-83). Vertex ids are
 * the positions 0..n-1 (build_graph adds vertex c with id c, adapter.hpp:117). */
int gb_set_cameras(gb_graph* g, void* params_fp, uint64_t n, const uint8_t* fixed);
/* Points: AoS FP[3*n], refined in place (Point3Traits, adapter.hpp:30-42). */
int gb_set_points(gb_graph* g, void* params_fp, uint64_t n, const uint8_t* fixed);
/* Observations, one reprojection factor each (FactorDescriptor::add_factor,
 * factor_descriptor.hpp:192-210, via build_graph adapter.hpp:136-141):
 * camera/point ids, observed pixel FP[2*n], identity information, level
 * (NULL = all 0; FactorDescriptor::set_level :222-226), loss kind and Huber
 * delta (loss.hpp:15-23). The arrays are referenced, not copied (like the
 * camera / point buffers): keep them alive and unchanged until the next
 * gb_set_observations or gb_destroy (fp32 observations are widened once into
 * an internal copy). Unknown ids -> GB_ERR_INVALID_ARGUMENT (resolve_slots
 * :549-558). */
int gb_set_observations(gb_graph* g, uint64_t n, const uint32_t* camera_index,
                        const uint32_t* point_index, const void* observed_fp,
                        const uint8_t* level, int loss_kind, double huber_delta);
/* Linear solver of every LM step: GB_SOLVER_PCG (default, the reference's
 * algorithm) or GB_SOLVER_SCHUR: points are eliminated with their exact 3x3
 * blocks, PCG (same pcg_solve semantics and config) runs on the reduced camera
 * system S = A_cc - A_cp A_pp^-1 A_pc with block-Jacobi on S's camera blocks,
 * and the points are back-substituted. Stored-Jacobian modes, single GPU. */
int gb_set_linear_solver(gb_graph* g, int solver);
/* FactorDescriptor::set_differentiation_mode (factor_descriptor.hpp:230-235). */
int gb_set_differentiation_mode(gb_graph* g, int diff_mode);

/* ---- the solve ------------------------------------------------------------
 * Replaces levenberg_marquardt<FP,SP>(Graph&, const LMConfig&)
 * (levenberg_marquardt.hpp:115-224). Uploads once, runs every LM iteration on
 * the device (no host round-trip per iteration), writes the refined cameras
 * and points back into the registered user buffers. records: NULL or an array
 * of max_records IterationRecords (report->iterations_run are valid).
 * Non-finite initial chi^2 -> GB_ERR_RUNTIME with the reference message. */
int gb_optimize(gb_graph* g, const gb_lm_config* cfg, gb_solve_report* report,
                gb_iteration_record* records, int32_t max_records);

/* The same solve split into phases, for callers that interleave their own
 * work or time individual LM iterations (bench.py):
 *   gb_begin   upload + activation + initial linearize + lambda0
 *              (levenberg_marquardt.hpp:116-147); fills the initial fields of
 *              report (may be NULL).
 *   gb_step    enqueues n LM iterations (:149-220) on the solver stream and
 *              returns without synchronizing; iterations after termination
 *              are device-side no-ops.
 *   gb_end     synchronizes, fills report/records, writes the parameters back.
 *   gb_stream  the cudaStream_t all of the handle's kernels run on.
 *   gb_time_hvp  average device time (ms, CUDA events on gb_stream) of
 *              `reps` back-to-back Hessian-vector products at the current
 *              linearization (the dominant kernel pair of a PCG iteration). */
int gb_begin(gb_graph* g, const gb_lm_config* cfg, gb_solve_report* report);
int gb_step(gb_graph* g, int32_t n);
int gb_end(gb_graph* g, gb_solve_report* report, gb_iteration_record* records, int32_t max_records);
void* gb_stream(gb_graph* g);
int gb_time_hvp(gb_graph* g, int32_t reps, double* ms_per_hvp, double* ms_tiles_only);
/* gb_hvp_bytes  bytes one HVP timed by gb_time_hvp moves on the configured
 *              path (factored J store, per-tile blobs, partial slots), and the
 *              reference-layout figure E (24 s_J + 8) + N (s_V + s_A) of
 *              SURVEY.md §8(d) (the roofline's "algorithmic bytes"). */
int gb_hvp_bytes(gb_graph* g, double* kernel_bytes, double* reference_bytes);
/* gb_hvp_info  the configured HVP path (0 dynamic tile kernel, 1 stored-J
 *              tile kernel, 2 stored-J bulk-copy pipeline, 3 recompute
 *              pipeline (hvp_rc.cuh: no Jacobian store)), the bytes one HVP
 *              moves on it, and SURVEY.md §8(d)'s algorithmic bytes and flops
 *              for it: stored J  E (24 s_J + 8) + N (s_V + s_A), 0 flops;
 *              recompute / dynamic  E (2 s_FP + 8) + (9 nc + 3 np) s_FP +
 *              N (s_V + s_A) and E * 500 flops.
 * gb_fma_peak  measured FMA throughput (TFLOP/s, 2 flops per FMA) of this
 *              device in fp64 (precision 0) or fp32 (1): a dependent-chain-
 *              free DFMA / FFMA loop over every SM, timed with CUDA events. */
int gb_hvp_info(gb_graph* g, int32_t* path, double* kernel_bytes, double* algorithmic_bytes, double* algorithmic_flops);
int gb_fma_peak(int32_t device, int32_t precision, double* tflops);
/* gb_iteration_kernels  number of kernel launches one LM iteration replays
 *              (kernel nodes of the captured per-iteration CUDA graph, between
 *              gb_begin and gb_end; 0 when the iteration is not captured). */
int gb_iteration_kernels(gb_graph* g, int32_t* kernels);

/* gb_host_alloc / gb_host_free  page-locked host memory for the caller's
 *              camera / point arrays (bal::BalGraph owns its AoS arrays,
 *              adapter.hpp:82-90), so the solve's upload and in-place write-
 *              back run at full host-link rate. Freed blocks are cached for the
 *              next graph. gb_host_alloc returns NULL when no device is usable
 *              (the caller then uses ordinary memory). */
void* gb_host_alloc(uint64_t bytes);
void gb_host_free(void* p);
/* gb_host_copy  memcpy split over host threads (fills those arrays from the
 *              caller's problem at full host-memory bandwidth). */
void gb_host_copy(void* dst, const void* src, uint64_t bytes);

/* ---- multi-GPU sharding (no reference counterpart: the reference is a
 * single-process CPU solver) -------------------------------
 * One process (or host thread) per shard. Every rank registers the FULL
 * problem; the solve shards it into contiguous point-tile ranges balanced by
 * edge count, replicates the cameras, and allreduces the camera-sized vectors
 * and PCG scalars every PCG iteration. After gb_optimize every rank holds the
 * complete refined cameras and points.
 *   kind 0: NCCL; id = the 128-byte ncclUniqueId from gb_nccl_unique_id on
 *           rank 0, shared with the other ranks out of band.
 *   kind 1: in-process loopback (ranks are host threads on one GPU; for
 *           testing the sharded path on a single device); id = uint64 key.
 *   kind 2: shared memory (one process per rank on one host, any devices,
 *           also several ranks on the same GPU; host-synchronous collectives
 *           through a POSIX shm segment); id = uint64 key, equal on all ranks.
 * gb_shard_plan (host only) reports each rank's [tile0,tile1), [point0,point1)
 * (internal order), edge count and (optionally) the owner rank of every point
 * for `world` ranks. world == 1 with kind 0 runs the collective code path on
 * a single rank. */
int gb_nccl_unique_id(void* out128);
int gb_set_distributed(gb_graph* g, int world, int rank, int kind, const void* id);
/* Test hook (host only, no GPU): the kind-2 shared-memory collectives on host
 * buffers: allreduce (sum, or max) of data[n] in rank order, then a broadcast
 * of bcast[nb] (may be NULL) from rank world-1. Blocks until all ranks call. */
int gb_shm_allreduce_selftest(int world, int rank, uint64_t key, double* data, uint64_t n, int max, double* bcast,
                              uint64_t nb);
int gb_shard_plan(uint64_t num_cameras, uint64_t num_points, uint64_t n, const uint32_t* camera_index,
                  const uint32_t* point_index, int world, uint32_t* tiles_out, uint32_t* points_out,
                  uint64_t* edges_out, uint32_t* point_owner);

/* Test hook: runs the device activation and the host reference activation
 * (activate.cpp, the same rules) and compares every structure bit for bit.
 * GB_OK or GB_ERR_LOGIC naming the first differing array. */
int gb_activation_selfcheck(gb_graph* g, int level);

/* BalGraph::mse (adapter.hpp:95-99) at the current user parameters. */
int gb_mse(gb_graph* g, double* out);
/* Graph::total_error(level) (graph.hpp:99-104). */
int gb_total_error(gb_graph* g, int level, double* out);

/* ---- LinearSystem surface (linear_system.hpp:44-216) ----------------------
 * These expose the same intermediate quantities as the reference's public
 * LinearSystem accessors so parity can be checked step by step. Vectors are
 * in the REFERENCE column layout (free cameras 9 each in insertion order,
 * then free points 3 each; VertexDescriptor::assign_columns :115-126). */

/* Graph::activate + LinearSystem::prepare + linearize (linear_system.hpp:44-82).
 * Any output pointer may be NULL. free_dims receives N. */
int gb_ls_linearize(gb_graph* g, int level, double clamp_min, double clamp_max, int damping,
                    double* chi2, int64_t* free_dims, void* b_fp, void* diag_fp,
                    void* clamped_fp, void* scaling_fp, int32_t* finite);
/* out = (D H D + damp) v   (LinearSystem::hvp, linear_system.hpp:104-115).
 * v: SP[N], out: Arith[N]. */
int gb_ls_hvp(gb_graph* g, const void* v_sp, void* out_arith, double lambda);
/* LinearSystem::build_preconditioner (linear_system.hpp:120-160): inverse
 * blocks in the reference's PrecondLayout order (camera 9x9 blocks, then point
 * 3x3 blocks, one per free vertex), FP. fallbacks may be NULL. */
int gb_ls_preconditioner(gb_graph* g, double lambda, void* blocks_fp, int32_t* fallbacks);
/* LinearSystem::solve_step (linear_system.hpp:185-207): dx FP[N]. */
int gb_ls_solve_step(gb_graph* g, double lambda, const gb_pcg_config* pcg, void* dx_fp,
                     gb_pcg_stats* stats, double* predicted_decrease, int32_t* finite);
/* Stored Jacobian blocks, per active factor [Jc 2x9 | Jp 2x3] row-major, SP
 * (factor_descriptor.hpp:662-670 layout), active-factor order. */
int gb_ls_jacobians(gb_graph* g, void* out_sp);
/* The edge->vertex incidence CSR of FactorDescriptor::build_incidence
 * (factor_descriptor.hpp:710-753) for descriptor 0 (cameras) or 1 (points):
 * call once with NULL arrays to get the sizes, then again with buffers.
 * vertex_of_segment: uint64[nseg], offsets: uint64[nseg+1], items_factor:
 * uint32[nitems] (active factor index a), items_slot: uint16[nitems]. */
int gb_incidence(gb_graph* g, int descriptor, uint64_t* nseg, uint64_t* nitems,
                 uint64_t* vertex_of_segment, uint64_t* offsets, uint32_t* items_factor,
                 uint16_t* items_slot);

/* ---- report wire format -------------------------------------------------
 * Replaces gopt::to_json(const SolveReport&).dump() and gopt::to_csv
 * (include/gopt/report.hpp:32-71; used by src/experiment.cpp:84,90): the
 * same bytes for a report + its n IterationRecords. Writes at most cap bytes
 * (NUL-terminated) into buf (may be NULL); *needed = full length + 1. */
int gb_report_json(const gb_solve_report* report, const gb_iteration_record* records, int32_t n, char* buf,
                   uint64_t cap, uint64_t* needed);
int gb_report_csv(const gb_solve_report* report, const gb_iteration_record* records, int32_t n, char* buf,
                  uint64_t cap, uint64_t* needed);

/* ---- synthetic BAL-shaped problems (bench / test input) -------------------
 * Deterministic generator with the semantics of tests/synthetic_bal.hpp:16-113
 * (camera ring, point cloud, pixel noise, perturbed initial estimate), sized
 * to an exact (cameras, points, observations) shape; see DESIGN.md. Outputs
 * are binary64 (BALProblem layout, bal/problem.hpp:25-40). camera_stride 0
 * picks the default; zipf_s > 0 draws each point's first camera from a
 * Zipf(s) law (skewed camera degrees). Host-only, no GPU needed. */
int gb_synthetic_bal(uint64_t num_cameras, uint64_t num_points, uint64_t num_observations,
                     uint64_t seed, uint64_t camera_stride, double zipf_s,
                     uint32_t* camera_index, uint32_t* point_index, double* observed,
                     double* cameras, double* points);

#ifdef __cplusplus
}
#endif

#endif /* GB_BAL_H_ */

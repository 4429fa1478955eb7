/*
 * rkmf_b200 — C ABI of the B200-native restarted randomized-Arnoldi f(A)b
 * hot path (arXiv 2503.22631; reference artifact `rkmf`, /root/reference/proj).
 *
 * Plain pointers and sizes only: no torch or CUDA types in the signatures
 * (a cudaStream_t is passed as void*). Every entry point returns a status
 * code that mirrors the reference's exception hierarchy
 * (proj/include/rkmf/types.hpp:25-48); the message of the last failure is
 * available from rkmf_last_error(). The C++ wrapper include/rkmf_b200.hpp
 * rethrows the reference exception types with the same message prefixes.
 *
 * Device pointers ("d_" prefix) must be cudaMalloc'ed on the context's device.
 * Host pointers ("h_" prefix) are plain host memory (pinned or pageable).
 * Calls are synchronous with respect to the host unless stated otherwise:
 * like the reference, one solve runs at a time per context; distinct
 * contexts are independent (proj/src/restart.cpp:267-299).
 */
#ifndef RKMF_B200_H
#define RKMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: types.hpp:25-48 (Error / ShapeError / ParameterError /
 *      NumericalError) plus device-side failures ---- */
#define RKMF_OK 0
#define RKMF_PARAMETER_ERROR 1 /* rkmf::ParameterError */
#define RKMF_SHAPE_ERROR 2     /* rkmf::ShapeError */
#define RKMF_NUMERICAL_ERROR 3 /* rkmf::NumericalError */
#define RKMF_DEVICE_ERROR 4    /* CUDA / NCCL failure (rkmf::Error) */
#define RKMF_INTERNAL_ERROR 5  /* rkmf::Error */
#define RKMF_PARSE_ERROR 6     /* rkmf::ParseError (Matrix Market / vector files) */

/* ---- function kinds: densefun.hpp:20 FunctionSpec::Kind. EXP_NEG is the
 *      reference's ExpNeg(t): f(z) = exp(-t z). INV_SQRT (f(z) = z^{-1/2}) is
 *      an extension required by BASELINE cfg3; the reference has no such kind. */
#define RKMF_FN_EXP_NEG 0
#define RKMF_FN_INV_SQRT 4

/* ---- dense-f evaluation strategy (rkmf_restart_options.dense_f) ---- */
#define RKMF_DENSE_AUTO 0       /* FULL for EXP_NEG, QUADRATURE for INV_SQRT */
#define RKMF_DENSE_FULL 1       /* f(R_accum) in full every cycle, restart.cpp:72-78 */
#define RKMF_DENSE_QUADRATURE 2 /* restart quadrature, O(N_q m^2) per cycle */

typedef struct rkmf_context rkmf_context;
typedef struct rkmf_matrix rkmf_matrix; /* device CSR, sparse.hpp:16-24 */
typedef struct rkmf_sketch rkmf_sketch; /* device SketchOperator, sketch.hpp:16-24 */

/* Replaces restart::RestartOptions (restart.hpp:20-26). Defaults via
 * rkmf_restart_options_default(): m_r=20, tol=1e-10, k_max=100,
 * budget_total_m=4000, divergence_factor=1e6. */
typedef struct {
  int64_t m_r;
  double tol; /* absolute: stop when ||y_k|| <= tol (restart.cpp:113) */
  int64_t k_max;
  int64_t budget_total_m;
  double divergence_factor;
  int32_t dense_f;        /* RKMF_DENSE_* */
  int32_t quad_nodes;     /* InvSqrt quadrature nodes: 0 (default) = designed from
                             the Ritz values of every cycle with node doubling
                             (branch-cut guard); > 0 = that many fixed nodes */
  int32_t diagnostics;    /* 1: fill CycleRecord kappa_W / leftmost_ritz_re
                             (restart.cpp:101,103; one Gram pass over W_m per
                             cycle, m <= 64); 0 (default): NaN */
  int32_t reserved;
} rkmf_restart_options;

/* Replaces restart::CycleRecord (restart.hpp:28-40). kappa_W and
 * leftmost_ritz_re (restart.cpp:101,103) are filled when
 * rkmf_restart_options.diagnostics is set, else NaN (not on the hot path).
 * Times are device times from CUDA events. */
typedef struct {
  int64_t cycle;
  int64_t total_m;
  int64_t total_matvecs;
  double update_norm;
  double error_vs_reference; /* NaN when no reference vector was given */
  double kappa_W;
  double leftmost_ritz_re;
  double alpha_dev;
  double elapsed_ms;
  double build_ms;
  double funm_ms;
  double start_norm;
  double subdiag;
} rkmf_cycle_record;

/* Replaces restart::RestartResult (restart.hpp:56-65) minus f_hat (written
 * to the caller's buffer) and R_accum (rkmf_last_r_accum). Counters are
 * PerfCounters (types.hpp:57-75). */
typedef struct {
  int64_t converged;
  int64_t cycles;
  int64_t total_m;
  double alpha;
  int64_t matvecs;
  int64_t dot_n;
  int64_t dot_d;
  int64_t basis_updates;
  int64_t peak_basis_cols;
  int64_t n_records;
  double solve_ms; /* device time of the whole solve (CUDA events) */
  int64_t quad_nodes; /* restart-quadrature nodes of the last cycle (0: FULL dense f) */
} rkmf_restart_result;

/* ---- context ---- */
int rkmf_context_create(int device, rkmf_context** out);
int rkmf_context_destroy(rkmf_context* ctx);
const char* rkmf_last_error(const rkmf_context* ctx);
/* Launch all work on this cudaStream_t (NULL = the context's own stream). */
int rkmf_context_set_stream(rkmf_context* ctx, void* cuda_stream);
void rkmf_restart_options_default(rkmf_restart_options* opts);
/* Number of this library's kernels launched so far on the context. */
int64_t rkmf_context_launch_count(const rkmf_context* ctx);

/* Per-kernel-class device timing: CUDA events around every launch of the
 * solve (off by default; adds ~1 us gaps, so keep it out of headline runs).
 * Classes: 0 spmv_sketch (K2), 1 rgs_step (K3), 2 basis_update (K4),
 * 3 dense f (K6), 4 final_update (K5), 5 start sketch + init (K7),
 * 6 a cycle's steps fused into one kernel (small matrices, below). */
#define RKMF_KCLASS_COUNT 7
int rkmf_context_kernel_timing(rkmf_context* ctx, int enable);
/* Matrices of at most 131072 rows (single rank, randomized builder, m <= 63)
 * run each cycle's m steps as one cooperative kernel with grid barriers
 * instead of three launches per step (enable != 0, the default); 0 keeps the
 * per-step kernels (A/B runs, tests of both paths). */
int rkmf_context_set_fused_cycle(rkmf_context* ctx, int enable);
/* ms[7] accumulated device milliseconds, launches[7] counts; reset != 0 clears. */
int rkmf_context_kernel_times(rkmf_context* ctx, double* ms, int64_t* launches, int reset);

/* ---- CSR matrices (sparse.hpp:16-24). Columns int32; row pointers int64 on
 *      the host side; stored on device as int32 when nnz < 2^31. The matrix is
 *      validated on creation (sparse.cpp:61-81) instead of every cycle as the
 *      reference does (basis.cpp:15); norm1 (sparse.cpp:97-102) is cached. ---- */
int rkmf_matrix_create_host(rkmf_context* ctx, int64_t n_rows, int64_t n_cols,
                            const int64_t* h_row_ptr, const int32_t* h_col_idx,
                            const double* h_values, rkmf_matrix** out);
/* Device arrays are copied (the caller keeps ownership of its buffers). */
int rkmf_matrix_create_device(rkmf_context* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                              const int64_t* d_row_ptr, const int32_t* d_col_idx,
                              const double* d_values, rkmf_matrix** out);
int rkmf_matrix_destroy(rkmf_matrix* A);
int rkmf_matrix_info(const rkmf_matrix* A, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                     double* norm1);
/* Storage format of the SpMV stream (B200-specific, no reference counterpart).
 * A matrix whose nonzeros lie on at most 8 diagonals (stencils) also gets a
 * diagonal copy on creation, streamed by the fused SpMV + sketch instead of the
 * CSR arrays (8 bytes per slot, no indices; results bit-identical). enable = 0
 * drops the copy (CSR path only), 1 builds it if the matrix qualifies, 2
 * only queries; *ndiag (optional) receives the diagonal count, 0 = CSR only. */
int rkmf_matrix_dia(rkmf_matrix* A, int enable, int* ndiag);
/* Row dictionary of the diagonal copy (B200-specific): when the copy's rows
 * take at most 256 distinct value tuples (constant-coefficient stencils: 27 on
 * a 3D 7-point grid), the fused SpMV + sketch streams one tuple-id byte per
 * row and reads the values from a shared-memory dictionary (results
 * bit-identical). Built with the diagonal copy by default. enable = 0 drops
 * it, 1 builds it if the copy exists and qualifies, 2 only queries;
 * *ntuples (optional) receives the tuple count, 0 = none. */
int rkmf_matrix_dia_dict(rkmf_matrix* A, int enable, int* ntuples);
/* Row-pointer width of the device CSR: stored as int32 when nnz < 2^31 - 1,
 * else int64 (cfg5 on one GPU). enable != 0 widens an int32 matrix to int64
 * so the int64 instantiations of the SpMV kernels run on small problems
 * (testing; results are identical); *is64 (optional) receives the width. */
int rkmf_matrix_rp64(rkmf_matrix* A, int enable, int* is64);
/* Copies the device CSR to the host: h_row_ptr[n_rows+1] (int64),
 * h_col_idx[nnz], h_values[nnz] (sizes from rkmf_matrix_info; any pointer may
 * be NULL). A partitioned matrix exports its local rows in the local column
 * numbering [owned | halo]. Backs save_matrix_market (sparse.cpp:196-211). */
int rkmf_matrix_export(rkmf_context* ctx, const rkmf_matrix* A, int64_t* h_row_ptr,
                       int32_t* h_col_idx, double* h_values);

/* ---- sketch operator: make_sketch (sketch.cpp:13-49), generated on device,
 *      bit-identical to the reference's SplitMix64/Floyd definition ---- */
int rkmf_sketch_create(rkmf_context* ctx, int64_t d, int64_t n, int64_t zeta, uint64_t seed,
                       rkmf_sketch** out);
int rkmf_sketch_destroy(rkmf_sketch* S);
/* SketchOperator::scale (default 1/sqrt(zeta)); settable as the reference's
 * tests do (test_sketch.cpp:162-173). */
int rkmf_sketch_set_scale(rkmf_sketch* S, double scale);
/* Bytes per 128-column tile of the device tile layout the fused kernel
 * streams: the header and the entry block (no reference counterpart; for
 * bandwidth accounting). */
int rkmf_sketch_layout_info(const rkmf_sketch* S, int64_t* header_bytes, int64_t* entry_bytes);
/* Copies rows (n*zeta int64) and signs (n*zeta int8) to the host. */
int rkmf_sketch_export(rkmf_context* ctx, const rkmf_sketch* S, int64_t* h_rows, int8_t* h_signs,
                       double* h_scale);

/* ---- single operations on device vectors ---- */
/* y = A x  (sparse.cpp:83-95) */
int rkmf_spmv(rkmf_context* ctx, const rkmf_matrix* A, const double* d_x, double* d_y);
/* y = S x  (sketch.cpp:51-63) */
int rkmf_sketch_apply(rkmf_context* ctx, const rkmf_sketch* S, const double* d_x, double* d_y);
/* z = A x and p = S z in one pass (the fused K2 kernel) */
int rkmf_spmv_sketch(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                     const double* d_x, double* d_z, double* d_p);
/* Measurement only: average device time of `reps` back-to-back launches of the
 * step kernel on the context stream (CUDA events), mode 1 = fused SpMV+sketch
 * (K2), 0 = SpMV alone, 2 = sketch of x alone. pacc accumulates over the reps. */
int rkmf_kernel_bench(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S, int32_t mode,
                      const double* d_x, double* d_z, double* d_p, int32_t reps, double* avg_ms);

/* ---- one randomized Arnoldi decomposition: basis.cpp:92-142 ----
 * d_W: n x (m+1) column-major with leading dimension ldw >= n (device);
 * d_U: d x (m+1) column-major (device); h_Rbar: (m+1) x m column-major (host).
 * *mk = m, or the kept size k+1 after a breakdown (*breakdown_at = k+1,
 * else 0). counters[5] = {matvecs, dot_n, dot_d, basis_updates, peak_basis_cols}. */
int rkmf_randomized_arnoldi(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                            const double* d_b, int64_t m, double* d_W, int64_t ldw, double* d_U,
                            double* h_Rbar, double* start_norm, int64_t* mk,
                            int64_t* breakdown_at, int64_t* counters);

/* ---- the drop-in boundary: restart::restarted_krylov (restart.hpp:74-79,
 *      restart.cpp:27-122) with S != nullptr (randomized builder).
 * b and f_out are host or device pointers (b_on_device / f_on_device).
 * reference (optional, same residency as b) fills error_vs_reference.
 * records: caller array of records_cap entries (may be NULL). ---- */
int rkmf_restarted_krylov(rkmf_context* ctx, const rkmf_matrix* A, const rkmf_sketch* S,
                          const double* b, int b_on_device, int32_t fn_kind, double fn_t,
                          const rkmf_restart_options* opts, double* f_out, int f_on_device,
                          const double* reference, rkmf_restart_result* result,
                          rkmf_cycle_record* records, int64_t records_cap);

/* ---- multi-GPU: one process per GPU, rows block-partitioned.
 * rkmf_nccl_unique_id fills 128 bytes on one rank; broadcast them (any
 * transport) and call rkmf_context_init_comm on every rank. A partitioned
 * matrix takes the rank's rows [row_starts[rank], row_starts[rank+1]) with
 * local row pointers and GLOBAL column indices; a partitioned sketch is the
 * same column range of make_sketch(d, n_global, zeta, seed). With both,
 * rkmf_restarted_krylov / rkmf_randomized_arnoldi run the distributed solve:
 * b, f_out and reference are the rank's local slices. ---- */
int rkmf_nccl_unique_id(void* out128);
int rkmf_context_init_comm(rkmf_context* ctx, int32_t nranks, int32_t rank,
                           const void* unique_id128);
/* The same collectives through caller callbacks on pinned host buffers (an MPI
 * or gloo host stack; tests with fewer GPUs than ranks). Each returns 0 on
 * success. alltoallv_b64: send holds one segment per rank in rank order
 * (send_counts[q] 8-byte elements for rank q), recv receives rank q's segment
 * (recv_counts[q] elements) in rank order; own-rank counts are 0. */
typedef struct rkmf_host_comm {
  void* user;
  int (*allreduce_sum_f64)(void* user, double* buf, int64_t count);
  int (*allreduce_max_f64)(void* user, double* buf, int64_t count);
  int (*alltoallv_b64)(void* user, const void* send, const int64_t* send_counts, void* recv,
                       const int64_t* recv_counts);
} rkmf_host_comm;
int rkmf_context_init_host_comm(rkmf_context* ctx, int32_t nranks, int32_t rank,
                                const rkmf_host_comm* callbacks);
/* The communicator as the library sees it: ranks (ncclCommCount for NCCL),
 * this rank, transport 0 none / 1 NCCL / 2 host callbacks. */
int rkmf_context_comm_info(const rkmf_context* ctx, int32_t* nranks, int32_t* rank,
                           int32_t* transport);
int rkmf_matrix_create_partitioned(rkmf_context* ctx, int64_t n_global, const int64_t* row_starts,
                                   const int64_t* h_row_ptr_local, const int32_t* h_col_global,
                                   const double* h_values, rkmf_matrix** out);
int rkmf_sketch_create_partitioned(rkmf_context* ctx, int64_t d, int64_t n_global, int64_t zeta,
                                   uint64_t seed, int64_t col_begin, int64_t n_local,
                                   rkmf_sketch** out);
/* Host-only partition helpers (no GPU needed): nnz-balanced contiguous row
 * blocks, and one rank's halo plan (see partition.cpp). */
int rkmf_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* row_starts);
int rkmf_partition_halo(int32_t nranks, int32_t rank, const int64_t* row_starts,
                        const int64_t* row_ptr_local, const int32_t* col_global, int64_t* n_halo,
                        int64_t* halo_global, int64_t* recv_counts, int32_t* col_local);

/* ---- on-device generators of the BASELINE matrices (same entries as the
 * host rkmf_gen_* below; cfg5's 3.6e9 nonzeros never touch the host) ---- */
int rkmf_matrix_gen_q1_hex(rkmf_context* ctx, int64_t N, int32_t lognormal, uint64_t coef_seed,
                           int32_t dirichlet, rkmf_matrix** out);
int rkmf_matrix_gen_laplacian(rkmf_context* ctx, int32_t dim, int64_t N, rkmf_matrix** out);
/* cfg4's upwind convection-diffusion, entries identical to rkmf_gen_convdiff_upwind */
int rkmf_matrix_gen_convdiff(rkmf_context* ctx, int64_t N, double peclet, double vx, double vy,
                             double vz, rkmf_matrix** out);
/* One rank's rows of the Q1 matrix (cfg5 partitioned) generated in HBM, with
 * the halo plan rkmf_matrix_create_partitioned would build from the same host
 * rows; row_starts[nranks+1] must be increasing multiples of N^2 (whole
 * x-planes per rank). Needs the communicator (rkmf_context_init_*comm). */
int rkmf_matrix_gen_q1_hex_partitioned(rkmf_context* ctx, int64_t N, int32_t lognormal,
                                       uint64_t coef_seed, int32_t dirichlet,
                                       const int64_t* row_starts, rkmf_matrix** out);
/* d_out[i] = gaussian(seed, i0 + i) on the device (rng.hpp:47-59) */
int rkmf_gen_gaussian_device(rkmf_context* ctx, uint64_t seed, int64_t i0, int64_t n,
                             double* d_out);

/* ---- CycleObserver / CycleInfo (restart.hpp:42-54, restart.cpp:91-92):
 * test-only hook fired after each cycle's update, fed by device->host copies
 * (it adds synchronisations; leave it unset on timed runs). All arrays are
 * host memory owned by the library and valid during the call only:
 *   W        n x w_cols column-major (ld n): the cycle's basis block as built,
 *            column 0 = start / alpha_k; w_cols = m_k, +1 when a next vector
 *            exists (restart.hpp:46)
 *   R_accum  total_m x total_m column-major, or NULL when R_accum is not kept
 *            (budget beyond the dense-f capacity)
 *   update   y_k = f_hat - f_hat_prev (the difference of the two host copies)
 *   f_hat    the running approximation
 * When partitioned, n and the vectors are the rank's local rows. ---- */
typedef struct {
  int64_t cycle; /* 1-based */
  int64_t n;
  int64_t m_k;
  int64_t w_cols;
  const double* W;
  int64_t total_m;
  const double* R_accum;
  const double* update;
  const double* f_hat;
  double alpha; /* global scale from cycle 1 */
} rkmf_cycle_info;
typedef void (*rkmf_cycle_observer)(void* user, const rkmf_cycle_info* info);
/* Observer for the following solves on ctx (NULL clears it). */
int rkmf_context_set_observer(rkmf_context* ctx, rkmf_cycle_observer fn, void* user);

/* ---- Matrix Market / vector interchange (sparse.cpp:140-242,
 * sparse.hpp:55-66): "coordinate real {general|symmetric}", symmetric
 * expanded, 1-based indices converted, duplicates summed, rows sorted;
 * vectors one value per line ('%' comments and blank lines skipped); writes
 * at %.17g. Host-only (no GPU needed). Parse failures return
 * RKMF_PARSE_ERROR with "path:line: what" in err (err_cap bytes). Arrays
 * returned by the loaders are malloc'ed by the library: free them with
 * rkmf_host_free. ---- */
int rkmf_mtx_load(const char* path, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                  int64_t** h_row_ptr, int32_t** h_col_idx, double** h_values, char* err,
                  int64_t err_cap);
int rkmf_mtx_save(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* h_row_ptr,
                  const int32_t* h_col_idx, const double* h_values, char* err, int64_t err_cap);
int rkmf_vector_load(const char* path, int64_t* n, double** h_out, char* err, int64_t err_cap);
int rkmf_vector_save(const char* path, int64_t n, const double* h_v, char* err, int64_t err_cap);
void rkmf_host_free(void* p);
/* load_matrix_market straight into a validated device matrix / a device
 * matrix written back out (its CSR copied to the host first) */
int rkmf_matrix_load_mtx(rkmf_context* ctx, const char* path, rkmf_matrix** out);
int rkmf_matrix_save_mtx(rkmf_context* ctx, const rkmf_matrix* A, const char* path);

/* ---- convergence sweep + CSV: restart::convergence_sweep / MethodSpec /
 * SweepRecord (restart.hpp:81-129, restart.cpp:124-305) and the CLI's CSV
 * (rkmf_bench.cpp:172-186). Methods "restart" (classical builder) and
 * "restart-rand" (d = 16 m unless given) run on the device, one row per
 * cycle; the one-shot approximants "arnoldi" and "rand" (d = 4 m unless given)
 * are the first cycle of those methods and become one row with cycle 0; a
 * failing or unsupported cell (the one-shot approximants "incomplete",
 * "rand-ls", "sfom" are not on the device path) becomes one NaN row carrying
 * the sanitised message. Rows keep the method order;
 * without timing the CSV is byte-identical across reruns. ---- */
typedef struct {
  char name[32];
  int64_t m;    /* m_r */
  int64_t d;    /* sketch rows, 0 = 16 m (restart.cpp:231-232) */
  int64_t zeta; /* reference default 4 */
  double tol;   /* absolute, reference default 1e-10 */
  int64_t k_max;
  uint64_t seed;
} rkmf_method_spec;
typedef struct {
  char method[32];
  int64_t n, m_or_totalm, cycle, matvecs;
  double rel_error, update_norm, kappa_W, leftmost_ritz_re, elapsed_ms;
  char note[256];
  double phase_build_ms, phase_eval_ms; /* not CSV columns (the CLI's timing summary) */
} rkmf_sweep_record;
/* h_b, h_reference (optional): host vectors; out: cap records, *n_out the count */
int rkmf_convergence_sweep(rkmf_context* ctx, const rkmf_matrix* A, const double* h_b,
                           int32_t fn_kind, double fn_t, const double* h_reference,
                           const rkmf_method_spec* methods, int64_t n_methods, int32_t with_timing,
                           rkmf_sweep_record* out, int64_t cap, int64_t* n_out);
/* fixed header, %.17g numbers; path NULL or "" = stdout */
int rkmf_sweep_write_csv(const rkmf_sweep_record* rows, int64_t n_rows, const char* path,
                         char* err, int64_t err_cap);

/* R_accum of the last solve on this context (total_m x total_m, column-major,
 * host); n_cap is the caller's capacity in rows. */
int rkmf_last_r_accum(rkmf_context* ctx, double* h_R, int64_t n_cap, int64_t* total_m);

/* ---- synthetic inputs for the BASELINE configs (host, deterministic) ----
 * Node ordering (ix*ny+iy)*nz+iz as problems.cpp:30-32. Two-call pattern:
 * call with NULL arrays to get n and nnz, then with buffers. */
int rkmf_gen_laplacian(int32_t dim, int64_t N, int64_t* n, int64_t* nnz, int64_t* h_row_ptr,
                       int32_t* h_col_idx, double* h_values);
int rkmf_gen_q1_hex(int64_t N, int32_t lognormal, uint64_t coef_seed, int32_t dirichlet,
                    int64_t* n, int64_t* nnz, int64_t* h_row_ptr, int32_t* h_col_idx,
                    double* h_values);
int rkmf_gen_convdiff_upwind(int64_t N, double peclet, double vx, double vy, double vz,
                             int64_t* n, int64_t* nnz, int64_t* h_row_ptr, int32_t* h_col_idx,
                             double* h_values);
/* b[i] = first N(0,1) draw of SplitMix64(derive(seed, i)) (rng.hpp:47-59). */
int rkmf_gen_gaussian(uint64_t seed, int64_t n, double* h_out);
/* entries [i0, i0 + n) of the same vector (one rank's slice of b) */
int rkmf_gen_gaussian_range(uint64_t seed, int64_t i0, int64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* RKMF_B200_H */

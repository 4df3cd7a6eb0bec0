/*
 * scs_b200.h -- C-ABI of the B200-native SCS indirect-method hot path.
 *
 * Drop-in boundary for the per-iteration path of conesplit 0.1.0 (the
 * reference, /root/reference/pkg/src/conesplit).  The reference has no FFI:
 * its hot path is the Python loop body Workspace.solve (solver.py:355-369)
 * over iterate_once (solver.py:153-166), project_affine / solve_kkt indirect
 * (embedding.py:101-114,165-197), cg_solve (sparse_linalg.py:253-290),
 * spmv/spmv_t (sparse_linalg.py:121-138), project_embedding_cone
 * (cones.py:241-249), residuals_original (scaling.py:148-207) and
 * check_termination (solver.py:210-234), with equilibrate
 * (scaling.py:79-129) and setup_cache (embedding.py:117-162) run once.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions: plain pointers and sizes, no torch types.  The caller owns
 * every host buffer; the library copies inputs during the call and never
 * keeps host pointers.  The library owns all device memory (and the NCCL
 * communicator when world > 1) and frees it in scs_destroy.  A handle is
 * not thread-safe; distinct handles may be used concurrently.  Every int
 * function returns SCS_OK (0) or a negative error code; the message is
 * available from scs_last_error(handle) (or scs_last_error(NULL) for
 * failures that happen before a handle exists).  Never aborts the process.
 */
#ifndef SCS_B200_H
#define SCS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCS_B200_ABI_VERSION 2

/* error codes -> Python exception classes:
 *   SCS_EINVAL, SCS_ENONFINITE -> ValueError (problem.py:38-53,
 *   sparse_linalg.py:260-287, cones.py:194-200); SCS_ESETUP -> SetupError
 *   (embedding.py:22-23, 159-161); SCS_ENOCONV, SCS_ECUDA, SCS_ENCCL,
 *   SCS_ENOMEM -> RuntimeError (cones.py:164-167). */
#define SCS_OK 0
#define SCS_EINVAL (-1)
#define SCS_ENONFINITE (-2)
#define SCS_ESETUP (-3)
#define SCS_ENOCONV (-4)
#define SCS_ECUDA (-5)
#define SCS_ENCCL (-6)
#define SCS_ENOMEM (-7)

/* Status values (solver.py:43-49, same order). */
#define SCS_RUNNING (-1)
#define SCS_SOLVED 0
#define SCS_INFEASIBLE 1
#define SCS_UNBOUNDED 2
#define SCS_INFEASIBLE_AND_UNBOUNDED 3
#define SCS_INDETERMINATE 4
#define SCS_MAX_ITERS_REACHED 5

/* Problem data: min c'x s.t. Ax + s = b, s in K  (problem.py:15-53).
 * A is the reference SparseMatrix CSC layout (sparse_linalg.py:16-54):
 * colptr int64[n+1], rowidx int64[nnz] strictly increasing per column,
 * vals fp64[nnz].  The cone is the reference ConeSpec / JSON cone dict
 * {"z","l","q","s"} (cones.py:89-139, fileio.py:68-73) extended with "ep",
 * the count of 3-dimensional exponential cones placed after the PSD blocks.
 *
 * Row sharding (world > 1): a rank passes only its rows [row_lo, row_lo+m)
 * of the global m_global-row problem (CSC of that row slice, local row
 * indices, b of that slice); c and the cone are always global. */
typedef struct {
  int64_t m, n;
  const int64_t* colptr;
  const int64_t* rowidx;
  const double* vals;
  const double* b;
  const double* c;
  int64_t z, l;
  int64_t nq;
  const int64_t* q;
  int64_t ns;
  const int64_t* s;
  int64_t ep;
  int64_t m_global; /* 0 -> m */
  int64_t row_lo;   /* 0 for a single shard */
} scs_problem;

/* Settings (solver.py:52-84).  cg_tol <= 0 selects the decaying schedule
 * tol = 1e-3 (1 + ||rhs||) / k^1.5 (embedding.py:179-185). */
typedef struct {
  double alpha;
  int64_t max_iters;
  double eps_pri, eps_dual, eps_gap, eps_infeas, eps_unbdd;
  int64_t check_interval;
  int64_t cg_max;
  double cg_tol;
  int32_t normalize;
  int32_t sweeps;
  int32_t device;   /* CUDA ordinal */
  int32_t fast;     /* 0: reference algorithm (parity mode); else SCS_FAST_* bits */
} scs_settings;

/* Opt-in modes, reported separately from parity mode:
 * SCS_FAST_PCG        Jacobi-preconditioned CG, M = diag(I + A^T A) of the
 *                     scaled A (the north star's "diagonally preconditioned
 *                     CG"; changes the iterates)
 * SCS_FAST_RECURRENCE A x of the CG iterate carried by recurrence
 *                     (A x += alpha A p) instead of a final matrix pass,
 *                     refreshed directly every 20 iterations (rounding-level
 *                     deviation from the reference, 5 matrix passes
 *                     per iteration instead of 6). */
#define SCS_FAST_PCG 1
#define SCS_FAST_RECURRENCE 2

/* Distributed launch (row sharding); NULL -> single GPU.  Rank k passes
 * rows [bounds[k], bounds[k+1]) (scs_problem.row_lo / m / m_global).  Ranks
 * are one process per GPU joined by NCCL (nccl_id), or -- to test the
 * sharded kernels on one GPU -- one host thread per shard in one process
 * joined by an emulated group (emu_group), or one process per shard on one
 * node joined through POSIX shared memory (flags & SCS_DIST_HOST: nccl_id
 * then carries a NUL-terminated shared-memory name agreed by the ranks;
 * the host all-reduce sums in rank order, so every rank gets the same
 * bits).  flags & SCS_DIST_FORCE forces the sharded code path (all-reduce
 * points included) even when world == 1. */
#define SCS_DIST_FORCE 1
#define SCS_DIST_HOST 2
typedef struct scs_emu_group scs_emu_group;
typedef struct {
  int32_t rank, world;
  const uint8_t* nccl_id;  /* 128 bytes from scs_nccl_unique_id on rank 0
                              (SCS_DIST_HOST: the shared-memory name) */
  scs_emu_group* emu_group;
  const int64_t* bounds;   /* world + 1 global row bounds */
  int32_t flags;
  int32_t pad_;
} scs_dist;

/* Residuals (scaling.py:37-55, same field order) and iteration info
 * (solver.py:96-105). */
typedef struct {
  int32_t status;
  int32_t pad_;
  int64_t iterations;
  int64_t cg_iters;
  double res[8]; /* pri_norm, dual_norm, gap, pri_thresh, dual_thresh,
                    gap_thresh, unbdd_measure, infeas_measure */
  double setup_seconds;
  double solve_seconds;
  int64_t launches; /* kernels launched by the last scs_solve/scs_step */
} scs_info;

typedef struct scs_handle scs_handle;

/* Workspace.__init__ (solver.py:300-316): copy A/b/c/cone to the device,
 * build CSR(A) and CSR(A^T), equilibrate on device (scaling.py:79-129) and
 * solve g = M^-1 h by CG (embedding.py:117-162). */
int scs_create(const scs_problem* prob, const scs_settings* st,
               const scs_dist* dist, scs_handle** out);

/* Workspace.solve (solver.py:336-378) up to the loop exit: run the whole
 * loop on the device.  warm_x/y/s (original units, nullable as a group)
 * follow initialize_state (solver.py:128-150) via scale_solution
 * (scaling.py:132-137).  On return `info` holds the status (including
 * MAX_ITERS_REACHED / INDETERMINATE), iteration counts and residuals. */
int scs_solve(scs_handle* h, const double* warm_x, const double* warm_y,
              const double* warm_s, scs_info* info);

/* Stepping interface for on_iteration callbacks (solver.py:357-358) and the
 * iterate-parity tests: scs_begin resets the state like the head of
 * Workspace.solve; scs_step runs up to k iterations (stopping at
 * termination); scs_finish applies the post-loop status rule
 * (solver.py:364-369). */
int scs_begin(scs_handle* h, const double* warm_x, const double* warm_y,
              const double* warm_s);
int scs_step(scs_handle* h, int64_t k, scs_info* info);
int scs_finish(scs_handle* h, scs_info* info);

/* SolverState (solver.py:87-93): copies u, v (length n + m_local + 1; on a
 * shard the y-part is the local slice). */
int scs_get_state(scs_handle* h, double* u, double* v);

/* ScalingData (scaling.py:18-34): D (m_local), E (n), sigma, rho. */
int scs_get_scaling(scs_handle* h, double* D, double* E, double* sigma,
                    double* rho);

/* Workspace.update_vectors (solver.py:325-334): new b (m_local) and/or c
 * (n), nullable; re-equilibrates and re-solves g, keeping A on device. */
int scs_update_vectors(scs_handle* h, const double* b, const double* c);

/* _point_residuals (solver.py:237-248) of an original-units point:
 * out = {pri, dual, gap}; computed on the device through D^-1 A_hat E^-1. */
int scs_point_residuals(scs_handle* h, const double* x, const double* y,
                        const double* s, double* out3);

/* extract_solution for status solved / max_iters_reached (solver.py:251-270,
 * unscale_solution scaling.py:140-145, _point_residuals solver.py:237-248)
 * on the device: x (n), y, s (m_local) in original units, copied into the
 * caller's buffers (each nullable); out5 = {pri, dual, gap, c'x, b'y}
 * (b'y all-reduced over row shards), so primal_obj = c'x and
 * dual_obj = -b'y without a second upload of the point. */
int scs_extract_point(scs_handle* h, double* x, double* y, double* s, double* out5);

/* spmv / spmv_t (sparse_linalg.py:121-138) on the device copy of the
 * ORIGINAL (unscaled) A is not kept; these apply the equilibrated A_hat:
 * which = 0: y = A_hat x; which = 1: x = A_hat^T y. */
int scs_apply_a(scs_handle* h, int which, const double* in, double* out);

/* project_embedding_cone (cones.py:241-249) / project_dual_cone
 * (cones.py:220-238) / project_primal_cone (cones.py:203-217) as a
 * standalone device call for tests: kind 0 = dual cone K*, 1 = primal K,
 * 2 = embedding R^n x K* x R_+ (x has n + m + 1 entries). */
int scs_project_cone(int64_t z, int64_t l, int64_t nq, const int64_t* q,
                     int64_t ns, const int64_t* s, int64_t ep, int kind,
                     int64_t n, const double* x, double* out, int device);

/* Independent solution checker (replaces the per-block
 * loop of the reference's `conesplit check`, cli.py:174-199): cone-membership
 * margins of a stacked host vector of length m, one per block in the order
 * zero (primal only: -max|v|), nonnegative (min v), each SOC (v0 - ||v1:||),
 * each PSD (minimum eigenvalue of the unpacked svec block), each exponential
 * cone (-distance to K_exp, or to K_exp* when dual).  nout must equal
 * scs_cone_margin_count(...).  Stateless (no handle): device `device`. */
int64_t scs_cone_margin_count(int64_t z, int64_t l, int64_t nq, int64_t ns, int64_t ep,
                              int32_t dual);
int scs_cone_margins(const double* vec, int64_t m, int64_t z, int64_t l, int64_t nq,
                     const int64_t* q, int64_t ns, const int64_t* s, int64_t ep, int32_t dual,
                     int32_t device, double* out, int64_t nout);
/* ... and its products Ax = A x, Aty = A^T y of the unscaled CSC matrix
 * (spmv / spmv_t in cli.py:209-210, 234, 263); either output may be NULL. */
int scs_check_products(int64_t m, int64_t n, const int64_t* colptr, const int64_t* rowidx,
                       const double* vals, const double* x, const double* y, double* Ax,
                       double* Aty, int32_t device);

/* Benchmark hooks (bench.py): device time of k back-to-back iterations
 * (CUDA events on the solver stream; no host sync inside) after the state
 * of scs_begin; and the average device time of one launch of a single
 * kernel -- kind 0: A-pass SpMV (q = A p), kind 1: A^T-pass SpMV with the
 * CG epilogue (Gp = p + A^T q, p'Gp) -- with its algorithmic HBM bytes. */
int scs_bench_iters(scs_handle* h, int64_t k, double* ms);
int scs_bench_kernel(scs_handle* h, int kind, int64_t reps, double* ms_per_launch,
                     double* bytes_per_launch);

/* Introspection of the device layout chosen at setup (no reference
 * counterpart; tests use it to assert which SpMV format ran):
 *   SCS_Q_FORMAT_A / SCS_Q_FORMAT_AT: 0 CSR kernel, 1 TMA-streamed tiles;
 *   SCS_Q_LAUNCHES_PER_ITER: kernel launches of one captured iteration;
 *   SCS_Q_STREAM_BYTES_A / _AT: bytes of the streamed format (0 if CSR);
 *   SCS_Q_CG_ITERS_TOTAL: EmbeddingCache.cg_iters_total (embedding.py:43,
 *   112): CG iterations of the setup solve of g plus every solve since. */
#define SCS_Q_FORMAT_A 0
#define SCS_Q_FORMAT_AT 1
#define SCS_Q_LAUNCHES_PER_ITER 2
#define SCS_Q_STREAM_BYTES_A 3
#define SCS_Q_STREAM_BYTES_AT 4
#define SCS_Q_CG_ITERS_TOTAL 5
int scs_query(scs_handle* h, int32_t key, int64_t* out);

/* Page-locked host memory (cudaHostAlloc) for warm starts and solution
 * buffers: copies to and from it run at full link speed and overlap the
 * device work (no reference counterpart; the Python layer pools it). */
int scs_host_alloc(int64_t bytes, void** out);
void scs_host_free(void* p);

void scs_destroy(scs_handle* h);
const char* scs_last_error(const scs_handle* h);
int scs_abi_version(void);

/* NCCL bootstrap for world > 1: rank 0 creates the id and the host
 * broadcasts it (torch.distributed store / gloo) to the other ranks. */
int scs_nccl_unique_id(uint8_t* out128);

/* Sum `n` host doubles over the shards of a row-sharded handle (in place);
 * a no-op copy for a single shard.  Used by the host for the m-length dot
 * products of extract_solution (b'y, certificate normalisation). */
int scs_allreduce(scs_handle* h, double* vals, int64_t n);

/* In-process emulated group of `world` shards on one GPU (tests). */
scs_emu_group* scs_emu_group_create(int32_t world);
void scs_emu_group_destroy(scs_emu_group* g);

/* Row partition for sharding: splits [0, m) into `world` contiguous ranges
 * at cone-block boundaries (only a second-order cone may straddle),
 * balancing the per-row weights (typically nnz per row).  bounds has
 * world + 1 entries. */
int scs_partition_rows(int64_t z, int64_t l, int64_t nq, const int64_t* q,
                       int64_t ns, const int64_t* s, int64_t ep,
                       const int64_t* row_nnz, int32_t world, int64_t* bounds);

/* Sparse-F LASSO in gen_lasso's standard form (generators.py:81-120), built
 * multithreaded on the host directly as CSC for 1e8-1e9 nonzeros
 * (SURVEY D4).  Call with colptr == NULL to get sizes (m, n, nnz); then
 * with buffers of those sizes.  Rows [row_lo, row_hi) only (row_hi <= 0 ->
 * all rows), with local row indices, for per-rank shard generation. */
int scs_gen_lasso(int64_t p, int64_t q, int64_t nnz_f, uint64_t seed,
                  int64_t row_lo, int64_t row_hi, int threads, int64_t* m,
                  int64_t* n, int64_t* nnz, int64_t* colptr, int64_t* rowidx,
                  double* vals, double* b, double* c);

#ifdef __cplusplus
}
#endif
#endif /* SCS_B200_H */

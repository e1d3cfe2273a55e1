/* hmat_b200.h -- C ABI of the B200-native H-matrix engine (libhmat_b200.so).
 *
 * Drop-in boundary for the reference library's public API
 * (/root/reference/proj/include/hmat/hmatrix.hpp, solver.hpp, morton.hpp, aca.hpp):
 * plain pointers and sizes, no C++ or torch types.  Every entry point is
 * noexcept; C++ exception kinds of the reference map onto hm_status codes
 * (SURVEY.md §8b).  The header-only C++ facade include/hmat_b200.hpp restores
 * the reference's hmat:: signatures on top of these functions.
 *
 * Conventions (same as the reference):
 *   - coordinates are structure-of-arrays: coords[a*n + i], a < d, 1 <= d <= 20;
 *   - vectors given to / returned by hm_mvp* and hm_cg_solve are in the ORIGINAL
 *     point ordering (permute_vector, core.cpp:167-177);
 *   - leaf lists are in canonical order (tree.cpp:189-194), dense list first.
 *
 * Thread safety: an hm_handle is immutable after hm_setup except for its product
 * workspace.  Calls on ONE handle are serialised on the host (a mutex per handle) and
 * on the device: all of a handle's work runs on its own stream, and the *_device entry
 * points join the caller's stream to it with events (the caller's stream waits for the
 * product, the product waits for the caller's earlier work).  Distinct handles are
 * independent.  hm_destroy waits for the handle's outstanding work.
 */
#ifndef HMAT_B200_H
#define HMAT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hm_handle hm_handle;

typedef enum {
  HM_OK = 0,
  HM_EINVAL = 1,     /* std::invalid_argument (bad config / length)        */
  HM_ERANGE = 2,     /* std::out_of_range (cluster range, unsupported size) */
  HM_ENOMEM = 3,     /* device or host allocation failed                   */
  HM_ECUDA = 4,      /* CUDA runtime error (also: no CUDA device)          */
  HM_ENCCL = 5,      /* NCCL error                                         */
  HM_ENONFINITE = 6, /* non-finite value (cg_solve, solver.cpp:51-54)      */
  HM_ELOGIC = 7,     /* std::logic_error / internal invariant              */
  HM_EIO = 8         /* std::runtime_error from file output (dump_leaves_csv) */
} hm_status;

typedef enum { HM_KERNEL_GAUSSIAN = 0, HM_KERNEL_MATERN = 1 } hm_kernel_kind;

/* Admissibility mode (tree.hpp:64-68). */
typedef enum { HM_ADM_GEOMETRIC = 0, HM_ADM_FORCE_DENSE = 1, HM_ADM_FORCE_ADMISSIBLE = 2 } hm_adm_mode;

/* HmatrixConfig (hmatrix.hpp:15-34) plus the B200 placement knobs. */
typedef struct {
  double eta;              /* admissibility parameter, default 1.5                      */
  int64_t c_leaf;          /* leaf size C_leaf, default 256                              */
  int64_t k;               /* ACA rank cap, default 16 (device limit 32)                 */
  int64_t bs_aca;          /* ACA batch size (partition_aca_queue, aca.cpp:229-250): batches
                              of Sigma m <= bs_aca (<= 0: one block per batch); recompute
                              chunks are runs of whole batches.  Results do not depend on it */
  int64_t bs_dense;        /* dense group cap (dense_blocks.cpp:36-66): setup throws
                              HM_EINVAL if one block has m*n > bs_dense > 0, like the
                              reference; the near field itself needs no workspace        */
  int32_t precompute_aca;  /* 1: factors computed once at setup and kept in HBM          */
  int32_t has_epsilon;     /* optional adaptive-rank criterion                           */
  double epsilon;
  int32_t adm_mode;        /* hm_adm_mode; force_dense (hmatrix.hpp:23) == FORCE_DENSE   */
  int32_t near_stored;     /* 1: dense leaves assembled once at setup and kept in HBM    */
  int32_t rank, world;     /* row-cluster ownership across GPUs (world = 1: single GPU)  */
  int32_t device;          /* CUDA device ordinal                                        */
  int64_t aca_chunk_rows;  /* recompute mode: factor workspace cap in rows (0 = auto)   */
} hm_config;

/* Timings of the last call (MvpTimings hmatrix.hpp:50-54, plus setup phases). */
typedef struct {
  double setup_ms, morton_ms, tree_ms, aca_ms, near_ms;
  double mvp_ms;        /* MvpTimings::total_ms of the last hm_mvp (host wall, copies inside) */
  double mvp_dense_ms;  /* MvpTimings::dense_ms: near-field phase (device events)            */
  double mvp_aca_ms;    /* MvpTimings::aca_ms: far-field phase incl. recompute-mode ACA      */
} hm_timings;

/* Algorithmic sizes: S_d = sum_dense m*n, S_l = sum_adm k_eff*(m+n). */
typedef struct {
  int64_t n_dense, n_aca;
  double S_d, S_l, sum_m_adm, sum_n_adm;
  double S_lm, S_ln;       /* sum_adm k_eff*m and k_eff*n (own rows; recompute mode: after a product) */
  double S_d_own;          /* dense entries of the rows this rank owns */
  int64_t aca_rejections;  /* rejected candidate columns in the last factorisation */
  int32_t dmax_leaf;
  int64_t row_begin, row_end;
  double device_bytes;
  double S_d_stored;       /* dense entries actually stored (symmetric near field: about half) */
  int32_t near_sym;        /* 1: symmetric near-field storage + pair kernel in use */
  int64_t n_aca_batches;   /* reference ACA batches of the own leaves (bs_aca) */
  int64_t n_aca_chunks;    /* device factorisation chunks (runs of whole batches) */
  int64_t aca_rejected_entries; /* sum of m over the rejected candidate columns (last factorisation) */
  double S_chain;          /* sum_adm k_eff (k_eff - 1) (m + n): residual-chain FP64 ops, own rows */
  int64_t near_pairs;      /* symmetric near field: dense blocks evaluated/streamed once for both leaves */
  int32_t near_sym_rc;     /* 1: recomputed near field on the symmetric pair kernel */
} hm_stats;

const char* hm_last_error(void);
void hm_config_default(hm_config* cfg);
int hm_device_count(void);

/* hmat::setup(PointSet, KernelFunction, HmatrixConfig) -- hmatrix.hpp:48.
 * coords: host SoA (d x n).  matern_beta: 0 = derive 1 + d/2 (core.hpp:35-40). */
hm_status hm_setup(const double* coords, int64_t n, int32_t d, int32_t kernel, double matern_beta,
                   const hm_config* cfg, hm_handle** out);
/* Same with device-resident coordinates (cudaMalloc'd on cfg->device). */
hm_status hm_setup_device(const double* coords_dev, int64_t n, int32_t d, int32_t kernel, double matern_beta,
                          const hm_config* cfg, hm_handle** out);
void hm_destroy(hm_handle* h);

/* hmat::mvp(HMatrix, x, kernel, MvpTimings*) -- hmatrix.hpp:58-59.  Host x and z
 * (length n, original ordering); copies are inside the call. */
hm_status hm_mvp(hm_handle* h, const double* x, double* z, hm_timings* t);
/* Device x and z on `stream` (cudaStream_t; NULL = the legacy default stream, as in the
 * CUDA runtime).  The product runs on the handle's stream, ordered after the work already
 * queued on `stream`, and `stream` is ordered after the product.  Asynchronous:
 * no host synchronisation (every launch parameter is fixed at setup), so the call can be
 * captured into a CUDA graph on `stream` once a first product has sized the workspaces. */
hm_status hm_mvp_device(hm_handle* h, const double* x_dev, double* z_dev, void* stream);
/* Attach an NCCL communicator for row-sliced products (world > 1): the 128-byte
 * ncclUniqueId produced by hm_nccl_unique_id on rank 0 and broadcast by the caller. */
hm_status hm_nccl_unique_id(unsigned char id[128]);
hm_status hm_attach_nccl(hm_handle* h, const unsigned char id[128]);

/* This rank's slice of the product without the allgather: z_slice (host, Morton order)
 * receives rows [row_begin, row_end) of hm_get_stats.  Lets world > 1 handles be tested
 * on one GPU (rank by rank). */
hm_status hm_mvp_local(hm_handle* h, const double* x, double* z_slice);

/* hmat::cg_solve(HMatrix, kernel, b, SolveConfig) -- solver.hpp:27-28 (host vectors). */
hm_status hm_cg_solve(hm_handle* h, const double* b, double sigma2, double tol, int64_t max_iter, double* x,
                      int64_t* iterations, double* relative_residual);
/* ---- multiple right-hand sides (BASELINE config 5) ----
 * X, Z: n x nrhs column-major (column r at X + r*n), original ordering.  One pass over
 * the operator serves up to 16 vectors (larger nrhs runs in passes of 16).
 * flags = HM_MULTI_EXACT: column r is bitwise equal to hm_mvp of X[:, r].
 * flags = HM_MULTI_DMMA : recompute-mode near field contracted on the FP64 tensor cores
 *                         (nrhs 8 or 16 per pass); per-leaf sums in a different order. */
#define HM_MULTI_EXACT 0
#define HM_MULTI_DMMA 1
hm_status hm_mvp_multi(hm_handle* h, const double* X, double* Z, int64_t nrhs, int32_t flags);
hm_status hm_mvp_multi_device(hm_handle* h, const double* X_dev, double* Z_dev, int64_t nrhs, int32_t flags,
                              void* stream);
/* nrhs independent hmat::cg_solve runs in lock-step on multi-RHS products (B, X: n x nrhs);
 * iterations / relative_residual: one entry per right-hand side. */
hm_status hm_cg_solve_multi(hm_handle* h, const double* B, int64_t nrhs, double sigma2, double tol, int64_t max_iter,
                            int32_t flags, double* X, int64_t* iterations, double* relative_residual);

/* hmat::dump_leaves_csv (tree.hpp:94, tree.cpp:197-205): every leaf of the block tree in
 * canonical order, "row_lower,row_upper,col_lower,col_upper,admissible" (HM_EIO when
 * the file cannot be written, the reference's runtime_error). */
hm_status hm_dump_leaves_csv(hm_handle* h, const char* path);
/* hmat::relative_error (hmatrix.hpp:63) -- exact product on the device, no N limit. */
hm_status hm_relative_error(hm_handle* h, const double* x, double* out);
/* exact dense product z = A x (oracle.cpp:24-55 semantics, device), original ordering */
hm_status hm_dense_mvp(hm_handle* h, const double* x, double* z);

/* Per-kernel device timing: CUDA events recorded on the launching stream around
 * every launch between begin and end; end returns the summed milliseconds and launch
 * counts per kernel id (0 gather x, 1 V^T x, 2 near+far rows, 3 scatter z,
 * 4 ACA (recompute mode), 5 far-field rows (recompute mode), 6 y allgather, 7 unused). */
hm_status hm_profile_begin(hm_handle* h);
hm_status hm_profile_end(hm_handle* h, double ms[8], int64_t counts[8]);

/* ---- introspection for bit-exact parity checks ---- */
hm_status hm_get_stats(hm_handle* h, hm_stats* st);
hm_status hm_get_timings(hm_handle* h, hm_timings* t);
/* Morton-ordered coordinates (d x n) and permutation (HMatrix::points). */
hm_status hm_get_points(hm_handle* h, double* coords, int64_t* perm);
/* Morton codes of the INPUT points (compute_morton_codes, morton.cpp:37-48). */
hm_status hm_get_codes(hm_handle* h, uint64_t* codes);
/* which 0: dense queue, 1: aca queue.  rows4: (row.lower,row.upper,col.lower,col.upper)
 * per leaf; boxes (nullable): 4*d per leaf (row a, row b, col a, col b). */
hm_status hm_get_leaves(hm_handle* h, int32_t which, int64_t* rows4, double* boxes);
/* Batched-ACA factors of every admissible leaf (factorises if not precomputed).
 * u: k*m per leaf rank-major, v: k*n per leaf rank-major, zero padded past k_eff;
 * nullable u/v return pivots only. */
hm_status hm_get_aca(hm_handle* h, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v);

/* ---- standalone primitives (reference unit-test surface) ---- */
/* compute_morton_codes (morton.cpp:37-48) on the device; host in/out. */
hm_status hm_morton_codes(const double* coords, int64_t n, int32_t d, uint64_t* codes);
/* morton_order (morton.cpp:50-71): stable sort + gather + perm composition. */
hm_status hm_morton_order(const double* coords, int64_t n, int32_t d, const int64_t* perm_in, double* coords_out,
                          int64_t* perm_out);
/* aca_batched on explicit blocks (aca.cpp:567-578): shapes (m,n) pairs, entries row-major concatenated. */
hm_status hm_aca_dense(int64_t nblocks, const int64_t* shapes, const double* entries, int64_t kmax,
                       int32_t has_eps, double eps, double eta, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv,
                       double* u, double* v);
/* phi(y_i, yp_i) for n point pairs (SoA d x n) evaluated on the device (eval_kernel, core.cpp:141-151). */
hm_status hm_eval_kernel(int32_t kernel, double matern_beta, int32_t d, int64_t n, const double* y,
                         const double* yp, double* out);
/* Host-compiled glibc-exp port (tests compare it with libm exp bit for bit). */
void hm_exp_port_host(int64_t n, const double* x, double* out);
/* Device glibc-exp port. */
hm_status hm_exp_port_device(int64_t n, const double* x, double* out);
/* glibc-log ports (Matern K1 series, core.cpp:46), host and device. */
void hm_log_port_host(int64_t n, const double* x, double* out);
hm_status hm_log_port_device(int64_t n, const double* x, double* out);

#ifdef __cplusplus
}
#endif
#endif

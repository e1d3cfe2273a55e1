// hmatrix.h -- device-resident H-matrix state and the host orchestration of
// setup() and mvp() (reference: proj/include/hmat/hmatrix.hpp:36-59).
#pragma once
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "kernel_math.cuh"

namespace hmb {

struct Config {
  double eta = 1.5;
  long long c_leaf = 256;
  long long k = 16;
  long long bs_aca = 1ll << 20;
  long long bs_dense = 1ll << 22;
  bool precompute_aca = false;
  bool has_epsilon = false;
  double epsilon = 0.0;
  int mode = 0;          // 0 geometric, 1 force dense, 2 force admissible
  int near_stored = 0;   // 0: near field recomputed per product (reference), 1: stored at setup
  int rank = 0, world = 1;
  long long aca_chunk_rows = 0;  // recompute-mode workspace cap in rows (0 = automatic)
};

// One leaf list (dense or admissible), canonical order (tree.cpp:189-194).
struct LeafList {
  long long count = 0;
  DevBuf<int> rl, m, cl, n;  // row.lower, |row|, col.lower, |col|
  DevBuf<int> tau_slot;      // cluster-table slot of the row cluster
  DevBuf<int> sigma_slot;
  DevBuf<unsigned char> depth;
  // per cluster slot: [start, end) of the run of leaves with that row cluster
  DevBuf<int> run_start, run_end;
  HostVec<int> h_rl, h_m, h_cl, h_n;  // host mirrors (chunk planning, partitioning, dumps)
};

// Per-kernel CUDA-event clock (enabled by hm_profile_begin): events are recorded on
// the launching stream around each launch and summed at hm_profile_end.
enum KernelId : int {
  kKGather = 0, kKLowrankT = 1, kKRows = 2, kKScatter = 3, kKAca = 4, kKRowsFar = 5, kKAllgather = 6,
  kKNearPairs = 7, kKNum = 8
};
struct KClock {
  bool on = false;
  std::vector<cudaEvent_t> ev[kKNum][2];
  void mark(int id, int which, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    ev[id][which].push_back(e);
  }
  void start(int id, cudaStream_t s) { mark(id, 0, s); }
  void stop(int id, cudaStream_t s) { mark(id, 1, s); }
};

struct Timings {
  double morton_ms = 0, tree_ms = 0, aca_ms = 0, near_ms = 0, setup_ms = 0;
  double mvp_ms = 0, mvp_dense_ms = 0, mvp_aca_ms = 0;
};

// ACA kernel size classes (aca.cu): windows <= 64..1024, clusters <= 2048/4096, big, CTA
constexpr int kAcaClasses = 9;

// One factorisation chunk: aca leaves [c0, c1) with host copies of everything the
// product needs to launch it without reading the device (see HMatrix::chunks).
struct AcaChunk {
  long long c0 = 0, c1 = 0;
  long long row_lo = 0, row_hi = 0;       // rows its leaves touch
  long long ub = 0, vb = 0, ue = 0, ve = 0;  // factor offsets u_off/v_off at c0 and c1
  long long ccount[kAcaClasses] = {};     // jobs per size class
  long long sched_off = 0;                // into sched_jobs / sched_order
  int max_rows_big = 0;                   // largest m of the big-block class
};

// Device, streams and events of a handle.  A base class so that it is destroyed AFTER
// every DevBuf member of HMatrix (their stream-ordered frees are enqueued on `stream`).
struct HandleStreams {
  int device = 0;
  cudaStream_t stream = nullptr;  // every product / setup operation of the handle
  cudaStream_t aux = nullptr;     // auxiliary stream (near field beside the V^T x fold)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_last = nullptr;  // end of the last work on `stream` (orders caller streams)
  cudaEvent_t ev_ph[4] = {};      // MvpTimings: near [0,1), far [2,3)
  cudaEvent_t ev_chunk[5] = {};   // recompute overlap: [b] factors of buffer b ready, [2+b] applied, [4] join
  void create(int dev);           // streams + events (throws HM_ECUDA)
  ~HandleStreams();
};

struct HMatrix : HandleStreams {
  Config cfg;
  KernelParams kp{};
  long long n = 0;
  int d = 0;

  // points (Morton order, SoA) and permutation: slot i holds original point perm[i]
  DevBuf<double> coords;
  DevBuf<long long> perm;
  DevBuf<unsigned long long> codes;  // Morton codes in input order (introspection)

  // implicit cluster tree: slot = depth_base[e] + idx, e in [0, dcap]
  int dcap = 0;       // deepest depth with boxes
  int dmax_leaf = 0;  // deepest depth holding a leaf
  std::vector<long long> depth_base;
  long long nslots = 0;
  DevBuf<long long> slot_lo, slot_hi;  // cluster ranges
  DevBuf<double> boxes;                // 2*d per slot: a[0..d), b[0..d)

  LeafList dense, aca;

  // Per deepest-level row cluster c (depth dmax_leaf): the leaf runs of every cluster of
  // its ancestor chain, in canonical order (tree.cpp:189-194), as CSR spans [start, end)
  // into the dense / aca lists.  All rows of c accumulate exactly these leaves, in order.
  DevBuf<int> row_cluster;             // Morton row -> deepest cluster index
  DevBuf<int> dspan_ptr, aspan_ptr;    // size 2^dmax_leaf + 1
  DevBuf<int> dspans, aspans;          // (start, end) pairs

  // rows owned by this rank (Morton order), [row_begin, row_end)
  long long row_begin = 0, row_end = 0;

  // admissible-block factors: U rank-major (kmax x m), V interleaved (n x kmax)
  DevBuf<long long> u_off, v_off;  // per aca leaf (also per-chunk in recompute mode)
  DevBuf<double> U, V;
  // recompute mode: a second factor workspace, so chunk c+1 is factorised (stream) while
  // chunk c's far field is applied (aux stream) -- each workspace half the chunk budget
  DevBuf<double> U2, V2;
  bool chunk_overlap = false;
  // Regular geometry (N = S * 2^dmax_leaf, S a power of two <= 256, k even) with stored
  // factors: U is row-tiled by S rows ([i/S][l][i%S]) and the product runs the
  // TMA-pipelined cluster kernel; otherwise U is rank-major (kmax x m).
  int u_tile_shift = -1;
  bool tma_rows = false;
  bool tma_far = false;  // recompute mode: far-field chunks on the TMA row kernel (U row-tiled)
  bool compact = false;  // stored factors with stride ke2 = k_eff rounded to even (mvp.cu compact_factors)
  DevBuf<int> k_eff, row_piv, col_piv;
  // host copies of the factor offsets (fixed at setup: the product never reads them back)
  HostVec<long long> h_uoff, h_voff;
  // Factorisation schedule, fixed at setup.  The own admissible leaves are split into
  // chunks (recompute mode: the factor workspace holds one chunk; precompute: one chunk).
  // A chunk is a run of whole reference batches (partition_aca_queue, aca.cpp:229-250,
  // Sigma m <= bs_aca) that fits the workspace budget.  Per chunk the leaves are sorted
  // once into the per-size-class job lists of the ACA kernels (sched_jobs) and the
  // long-leaves-first order of the V^T x fold (sched_order).
  std::vector<AcaChunk> chunks;
  long long n_batches = 0;      // reference batches of the own admissible leaves
  DevBuf<int> sched_jobs, sched_order;
  DevBuf<int> sched_corder;     // multi-RHS: per chunk, leaves by column start (x reuse in L2)
  DevBuf<int> aca_counters;     // per-class job counters (reset before every chunk)
  DevBuf<double> aca_big_scratch;  // window scratch of the big-block ACA kernel (grown once)
  DevBuf<int> aca_fallback;     // smooth-path kernels: blocks handed to the window kernels
  DevBuf<unsigned long long> aca_rej;  // [0] rejected columns, [1] their entries: current factorisation
  bool keff_known = false;      // k_eff holds the ranks of a complete factorisation of the own leaves
  bool phase_events = false;      // record ev_ph around the product phases (hm_mvp)
  DevBuf<double> t;         // per (aca leaf, rank) V^T x
  bool factors_valid = false;

  // stored near field: column-major blocks
  DevBuf<long long> dense_off;
  long long h_dense_off_base = 0;  // dense_off of the first own leaf (host copy)
  DevBuf<double> dense_vals;
  // Symmetric near field (regular geometry, TMA product): A(sigma,tau) = A(tau,sigma)^T
  // bitwise (dx^2 is sign-symmetric), so only blocks with row.lower <= col.lower are
  // stored.  The pair kernel streams each stored block once and writes the per-leaf
  // dense products of BOTH leaves of the pair into part (S doubles per dense leaf);
  // the row product then folds those partials in leaf order (hmatrix.cpp:80-104).
  bool near_sym = false;
  bool near_sym_rc = false;  // same pairing for the recomputed (matrix-free) near field
  long long n_pairs = 0;
  DevBuf<int> pair_leaf, pair_mirror;  // stored leaf, mirror leaf (-1: diagonal or not own)
  DevBuf<int4> pair_desc;              // {leaf, first stored column, col.lower, row.lower}
  DevBuf<double> part;

  // product workspaces
  DevBuf<double> xm, zm, xin, zout;
  // multi-RHS workspaces (multi.cu): rhs-major vectors, chunk-relative t, symmetric partials
  DevBuf<double> xmR, zmR, tR, partR, xinR, zoutR;
  DevBuf<double> xmT;  // x interleaved [point][16] (the multi-RHS V^T x fold)
  DevBuf<long long> dmma_tiles;
  long long n_dmma_tiles = -1;  // -1: not built yet
  DevBuf<int> counter;

  // algorithmic sizes
  double S_d = 0, sum_m_adm = 0, sum_n_adm = 0, S_l = 0, S_lm = 0, S_ln = 0;
  double S_d_own = 0;  // dense entries of the rows this rank owns
  double S_chain = 0;  // sum_adm k_eff (k_eff - 1) (m + n), own leaves
  double S_d_stored = 0;  // dense entries stored (near_stored; about S_d_own / 2 when near_sym)
  Timings tm;
  KClock clk;

  ~HMatrix();
};

// setup() pipeline (hmatrix.cpp:38-64); coords_dev: d x n SoA on the device.
void build_hmatrix(HMatrix& h, const double* coords_dev);
// mvp (hmatrix.cpp:66-123) on device vectors in ORIGINAL order.
void mvp_device(HMatrix& h, const double* x_dev, double* z_dev, cudaStream_t s);
// Morton-ordered product into h.zm (rows [row_begin,row_end)), x already in h.xm.
void mvp_morton(HMatrix& h, cudaStream_t s);
// R right-hand sides (multi.cu): h.xmR -> h.zmR; flags bit 0: DMMA near field
void ensure_multi(HMatrix& h, int R, cudaStream_t s);
void gather_multi(HMatrix& h, const double* X, long long ldx, int R, cudaStream_t s);
void scatter_multi(HMatrix& h, double* Z, long long ldz, int R, cudaStream_t s);
void mvp_multi_morton(HMatrix& h, int R, int flags, cudaStream_t s);

// large host -> device copy through the pinned staging ring (setup.cu); synchronous
void upload_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);

// components
void morton_codes_device(const double* coords, long long n, int d, unsigned long long* codes, cudaStream_t s);
// schedule of aca leaves [c0, c1) into h.sched_* at c.sched_off (setup time, may sync)
void plan_aca_chunk(HMatrix& h, AcaChunk& c, cudaStream_t s);
// every chunk of the own leaves [lo, hi) at once (false: not applicable, plan per chunk)
bool plan_aca_chunks_all(HMatrix& h, long long lo, long long hi, cudaStream_t s);
// factorise one planned chunk into h.U / h.V (offsets relative to c.ub / c.vb); no host sync
void compute_aca(HMatrix& h, const AcaChunk& c, cudaStream_t s);
// rejected-column counter of the current factorisation
void reset_aca_rejections(HMatrix& h, cudaStream_t s);
// S_l, S_lm, S_ln, S_chain of the own aca leaves [lo, hi) from their ranks ke[b - lo]
void rank_sums(HMatrix& h, const int* ke, long long lo, long long hi);
void store_near_field(HMatrix& h, cudaStream_t s);
void plan_near_pairs(HMatrix& h, cudaStream_t s);
void plan_far_field(HMatrix& h, cudaStream_t s);
// explicit-matrix ACA seam (aca.cpp:567-578) on the GPU
void aca_dense_blocks(long long nblocks, const long long* shapes, const double* entries_host, long long kmax,
                      bool has_eps, double eps, double eta, long long* k_eff, long long* row_piv,
                      long long* col_piv, double* u_host, double* v_host, cudaStream_t s);


}  // namespace hmb

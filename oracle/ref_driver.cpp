// ref_driver.cpp -- C ABI harness around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This file is compiled together with the reference
// sources where they lie (/root/reference/proj/src/*.cpp, see oracle/Makefile)
// into oracle/_ref/libhmat_ref.so.  It is used (a) to pin the C restatement in
// oracle/hmat_oracle.c, (b) to generate the golden fixtures under tests/golden/
// and (c) as the reference CPU arm of bench.py.  Nothing in the product path
// links or loads it.
//
// The reference worker pool races with more than one thread (SURVEY.md F1,
// parallel.cpp:33-92), so the constructor below pins HMAT_THREADS=1 unless the
// caller set it explicitly.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hmat/aca.hpp"
#include "hmat/core.hpp"
#include "hmat/dense_blocks.hpp"
#include "hmat/hmatrix.hpp"
#include "hmat/morton.hpp"
#include "hmat/parallel.hpp"
#include "hmat/solver.hpp"
#include "hmat/tree.hpp"

using namespace hmat;

namespace {

thread_local std::string g_err;

__attribute__((constructor)) void pin_threads() {
  if (!std::getenv("HMAT_THREADS")) setenv("HMAT_THREADS", "1", 1);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown exception";
    return 1;
  }
}

PointSet make_points(std::int64_t n, int d, const double* coords, const std::int64_t* perm) {
  PointSet p;
  p.dim = d;
  p.count = n;
  p.coords.assign(static_cast<std::size_t>(d), std::vector<double>(static_cast<std::size_t>(n)));
  p.perm.resize(static_cast<std::size_t>(n));
  for (int a = 0; a < d; ++a) std::memcpy(p.coords[a].data(), coords + a * n, sizeof(double) * n);
  for (std::int64_t i = 0; i < n; ++i) p.perm[i] = perm ? perm[i] : i;
  return p;
}

KernelFunction make_kernel(int kind, double beta) {
  KernelFunction k;
  k.kind = kind == 0 ? KernelKind::Gaussian : KernelKind::Matern;
  k.matern_beta = beta;
  return k;
}

struct RefHandle {
  HMatrix h;
  KernelFunction kernel;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_threads() { return parallel_thread_count(); }

int ref_bessel_k1(std::int64_t n, const double* x, double* out) {
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) out[i] = bessel_k1(x[i]);
  });
}

// out[i] = phi(y_i, yp_i) for n point pairs given SoA (d x n each)
int ref_eval_kernel(int kind, double beta, int d, std::int64_t n, const double* y, const double* yp, double* out) {
  return guarded([&] {
    const KernelFunction k = make_kernel(kind, beta);
    std::vector<double> a(d), b(d);
    for (std::int64_t i = 0; i < n; ++i) {
      for (int q = 0; q < d; ++q) {
        a[q] = y[q * n + i];
        b[q] = yp[q * n + i];
      }
      out[i] = eval_kernel(k, a, b);
    }
  });
}

int ref_halton(std::int64_t n, int d, double* coords) {
  return guarded([&] {
    const PointSet p = halton_points(n, d);
    for (int a = 0; a < d; ++a) std::memcpy(coords + a * n, p.coords[a].data(), sizeof(double) * n);
  });
}

int ref_morton_codes(std::int64_t n, int d, const double* coords, std::uint64_t* codes) {
  return guarded([&] {
    const PointSet p = make_points(n, d, coords, nullptr);
    const std::vector<std::uint64_t> c = compute_morton_codes(p);
    std::memcpy(codes, c.data(), sizeof(std::uint64_t) * n);
  });
}

int ref_morton_order(std::int64_t n, int d, const double* coords, const std::int64_t* perm_in, double* coords_out,
                     std::int64_t* perm_out) {
  return guarded([&] {
    const PointSet s = morton_order(make_points(n, d, coords, perm_in));
    for (int a = 0; a < d; ++a) std::memcpy(coords_out + a * n, s.coords[a].data(), sizeof(double) * n);
    std::memcpy(perm_out, s.perm.data(), sizeof(std::int64_t) * n);
  });
}

void* ref_setup(std::int64_t n, int d, const double* coords, int kernel_kind, double matern_beta, double eta,
                std::int64_t c_leaf, std::int64_t k, std::int64_t bs_aca, std::int64_t bs_dense, int precompute,
                int has_eps, double eps, int force_dense) {
  RefHandle* out = nullptr;
  const int rc = guarded([&] {
    HmatrixConfig cfg;
    cfg.eta = eta;
    cfg.c_leaf = c_leaf;
    cfg.k = k;
    cfg.bs_aca = bs_aca;
    cfg.bs_dense = bs_dense;
    cfg.precompute_aca = precompute != 0;
    if (has_eps) cfg.epsilon = eps;
    cfg.force_dense = force_dense != 0;
    auto* r = new RefHandle;
    r->kernel = make_kernel(kernel_kind, matern_beta);
    try {
      r->h = setup(make_points(n, d, coords, nullptr), r->kernel, cfg);
    } catch (...) {
      delete r;
      throw;
    }
    out = r;
  });
  return rc == 0 ? out : nullptr;
}

void ref_free(void* h) { delete static_cast<RefHandle*>(h); }

std::int64_t ref_count(void* h, int which) {
  const RefHandle* r = static_cast<RefHandle*>(h);
  return static_cast<std::int64_t>(which == 0 ? r->h.dense_queue.size() : r->h.aca_queue.size());
}

// rows: 4 int64 per leaf (row.lower, row.upper, col.lower, col.upper);
// boxes (optional): 4*d doubles per leaf (row a[d], row b[d], col a[d], col b[d]).
int ref_leaves(void* h, int which, std::int64_t* rows, double* boxes) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    const auto& q = which == 0 ? r->h.dense_queue : r->h.aca_queue;
    const int d = r->h.points.dim;
    for (std::size_t i = 0; i < q.size(); ++i) {
      rows[4 * i + 0] = q[i].row.lower;
      rows[4 * i + 1] = q[i].row.upper;
      rows[4 * i + 2] = q[i].col.lower;
      rows[4 * i + 3] = q[i].col.upper;
      if (boxes) {
        double* b = boxes + 4 * d * i;
        for (int a = 0; a < d; ++a) {
          b[a] = q[i].box_row.a[a];
          b[d + a] = q[i].box_row.b[a];
          b[2 * d + a] = q[i].box_col.a[a];
          b[3 * d + a] = q[i].box_col.b[a];
        }
      }
    }
  });
}

int ref_points(void* h, double* coords, std::int64_t* perm) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    const std::int64_t n = r->h.points.count;
    for (int a = 0; a < r->h.points.dim; ++a) std::memcpy(coords + a * n, r->h.points.coords[a].data(), sizeof(double) * n);
    std::memcpy(perm, r->h.points.perm.data(), sizeof(std::int64_t) * n);
  });
}

int ref_mvp(void* h, const double* x, double* z, double* timings3) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    MvpTimings t;
    const std::vector<double> out = mvp(r->h, {x, static_cast<std::size_t>(r->h.points.count)}, r->kernel, &t);
    std::memcpy(z, out.data(), sizeof(double) * out.size());
    if (timings3) {
      timings3[0] = t.dense_ms;
      timings3[1] = t.aca_ms;
      timings3[2] = t.total_ms;
    }
  });
}

int ref_relative_error(void* h, const double* x, double* out) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    *out = relative_error(r->h, r->kernel, {x, static_cast<std::size_t>(r->h.points.count)});
  });
}

int ref_cg(void* h, const double* b, double sigma2, double tol, std::int64_t max_iter, double* x,
           std::int64_t* iterations, double* rel_res) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    SolveConfig cfg;
    cfg.sigma2 = sigma2;
    cfg.tol = tol;
    cfg.max_iter = max_iter;
    const SolveResult s = cg_solve(r->h, r->kernel, {b, static_cast<std::size_t>(r->h.points.count)}, cfg);
    std::memcpy(x, s.x.data(), sizeof(double) * s.x.size());
    *iterations = s.iterations;
    *rel_res = s.relative_residual;
  });
}

// Batched ACA over every admissible leaf, exactly as mvp() recomputes it
// (aca.cpp:548-558 through the setup's own batches).  Outputs per admissible
// block b (aca_queue order): k_eff[b], row/col pivots (kmax each, -1 padded),
// u (kmax*m, rank-major) and v (kmax*n, rank-major) at offsets u_off[b] / v_off[b]
// that the caller computed as prefix sums of kmax*m and kmax*n.
int ref_aca_all(void* h, std::int64_t* k_eff, std::int64_t* row_piv, std::int64_t* col_piv, double* u, double* v,
                std::int64_t* rejections) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    AcaOptions opt;
    opt.max_rank = r->h.config.k;
    opt.epsilon = r->h.config.epsilon;
    opt.eta = r->h.config.eta;
    const std::int64_t kmax = opt.max_rank;
    std::int64_t block = 0, uo = 0, vo = 0;
    (void)rejections;
    for (const AcaBatch& batch : r->h.aca_batches) {
      BatchedAcaResult res = aca_batched(batch, r->kernel, r->h.points, opt);
      for (std::size_t b = 0; b < batch.items.size(); ++b, ++block) {
        const std::int64_t m = batch.items[b].row.size();
        const std::int64_t n = batch.items[b].col.size();
        k_eff[block] = res.k_eff[b];
        for (std::int64_t l = 0; l < kmax; ++l) {
          row_piv[block * kmax + l] = res.row_pivots[b * kmax + l];
          col_piv[block * kmax + l] = res.col_pivots[b * kmax + l];
          if (u) {
            if (l < res.k_eff[b]) {
              std::memcpy(u + uo + l * m, res.u_storage.data() + l * batch.total_rows + batch.row_offset[b], sizeof(double) * m);
              std::memcpy(v + vo + l * n, res.v_storage.data() + l * batch.total_cols + batch.col_offset[b], sizeof(double) * n);
            } else {
              std::memset(u + uo + l * m, 0, sizeof(double) * m);
              std::memset(v + vo + l * n, 0, sizeof(double) * n);
            }
          }
        }
        uo += kmax * m;
        vo += kmax * n;
      }
    }
  });
}

// Explicit-matrix seam (aca.cpp:567-578): nblocks dense row-major blocks with
// shapes (m,n) concatenated.  Same output layout as ref_aca_all.  single != 0
// runs aca_single (aca.cpp:180-183) per block instead, for the F2 comparison.
int ref_aca_dense(std::int64_t nblocks, const std::int64_t* shapes, const double* entries, std::int64_t kmax,
                  int has_eps, double eps, double eta, int single, std::int64_t* k_eff, std::int64_t* row_piv,
                  std::int64_t* col_piv, double* u, double* v) {
  return guarded([&] {
    std::vector<DenseMatrix> blocks;
    std::vector<std::pair<std::int64_t, std::int64_t>> sh;
    std::int64_t off = 0;
    for (std::int64_t b = 0; b < nblocks; ++b) {
      const std::int64_t m = shapes[2 * b], n = shapes[2 * b + 1];
      DenseMatrix a(m, n);
      std::memcpy(a.entries.data(), entries + off, sizeof(double) * m * n);
      off += m * n;
      blocks.push_back(std::move(a));
      sh.push_back({m, n});
    }
    AcaOptions opt;
    opt.max_rank = kmax;
    if (has_eps) opt.epsilon = eps;
    opt.eta = eta;
    std::int64_t uo = 0, vo = 0;
    if (single) {
      for (std::int64_t b = 0; b < nblocks; ++b) {
        AcaStats stats;
        AcaOptions o = opt;
        o.stats = &stats;
        const LowRankFactors f = aca_single(blocks[b], o);
        const std::int64_t m = sh[b].first, n = sh[b].second;
        k_eff[b] = f.k_eff;
        for (std::int64_t l = 0; l < kmax; ++l) {
          row_piv[b * kmax + l] = l < f.k_eff ? stats.row_pivots[l] : -1;
          col_piv[b * kmax + l] = l < f.k_eff ? stats.col_pivots[l] : -1;
          for (std::int64_t i = 0; i < m; ++i) u[uo + l * m + i] = l < f.k_eff ? f.u[l * m + i] : 0.0;
          for (std::int64_t j = 0; j < n; ++j) v[vo + l * n + j] = l < f.k_eff ? f.v[l * n + j] : 0.0;
        }
        uo += kmax * m;
        vo += kmax * n;
      }
      return;
    }
    const AcaBatch batch = make_batch_from_shapes(sh);
    const BatchedAcaResult res = aca_batched(batch, blocks, opt);
    for (std::int64_t b = 0; b < nblocks; ++b) {
      const std::int64_t m = sh[b].first, n = sh[b].second;
      k_eff[b] = res.k_eff[b];
      for (std::int64_t l = 0; l < kmax; ++l) {
        row_piv[b * kmax + l] = res.row_pivots[b * kmax + l];
        col_piv[b * kmax + l] = res.col_pivots[b * kmax + l];
        const bool live = l < res.k_eff[b];
        for (std::int64_t i = 0; i < m; ++i)
          u[uo + l * m + i] = live ? res.u_storage[l * batch.total_rows + batch.row_offset[b] + i] : 0.0;
        for (std::int64_t j = 0; j < n; ++j)
          v[vo + l * n + j] = live ? res.v_storage[l * batch.total_cols + batch.col_offset[b] + j] : 0.0;
      }
      uo += kmax * m;
      vo += kmax * n;
    }
  });
}

// Row-sampled product: every leaf whose row cluster
// intersects one of the given [lo,hi) Morton ranges is evaluated through the
// reference's own public batch functions, accumulated dense-then-ACA in leaf
// order exactly like mvp() (hmatrix.cpp:80-113).  z_morton (length N, zeroed
// here) is valid on the sampled rows.  x is in ORIGINAL ordering.
int ref_mvp_rows(void* h, const double* x, std::int64_t nranges, const std::int64_t* ranges, double* z_morton) {
  return guarded([&] {
    const RefHandle* r = static_cast<RefHandle*>(h);
    const std::int64_t n = r->h.points.count;
    const auto hit = [&](const WorkItem& w) {
      for (std::int64_t q = 0; q < nranges; ++q) {
        if (w.row.lower < ranges[2 * q + 1] && ranges[2 * q] < w.row.upper) return true;
      }
      return false;
    };
    std::vector<WorkItem> dense, aca;
    for (const WorkItem& w : r->h.dense_queue) if (hit(w)) dense.push_back(w);
    for (const WorkItem& w : r->h.aca_queue) if (hit(w)) aca.push_back(w);
    const std::vector<double> xm = permute_vector({x, static_cast<std::size_t>(n)}, r->h.points.perm, PermDirection::Forward);
    std::fill(z_morton, z_morton + n, 0.0);
    std::vector<double> y;
    for (const DenseGroup& g : partition_dense_queue(dense, r->h.config.bs_dense)) {
      DenseBatch batch;
      assemble_dense_batch(g, r->kernel, r->h.points, batch);
      gather_dense_inputs(batch, xm);
      batched_gemv(batch, y);
      for (std::size_t b = 0; b < g.items.size(); ++b) {
        for (std::int64_t i = 0; i < g.items[b].row.size(); ++i) z_morton[g.items[b].row.lower + i] += y[g.row_offset[b] + i];
      }
    }
    AcaOptions opt;
    opt.max_rank = r->h.config.k;
    opt.epsilon = r->h.config.epsilon;
    opt.eta = r->h.config.eta;
    for (const AcaBatch& batch : partition_aca_queue(aca, r->h.config.bs_aca)) {
      const BatchedAcaResult res = aca_batched(batch, r->kernel, r->h.points, opt);
      y.assign(static_cast<std::size_t>(batch.total_rows), 0.0);
      batched_low_rank_apply(res, batch, xm, y);
      for (std::size_t b = 0; b < batch.items.size(); ++b) {
        for (std::int64_t i = 0; i < batch.items[b].row.size(); ++i) z_morton[batch.items[b].row.lower + i] += y[batch.row_offset[b] + i];
      }
    }
  });
}

// Bench sample for the reference CPU arm: the leaves touching the given row ranges
// are factorised first (aca_batched, the precompute_aca=true path of setup(),
// hmatrix.cpp:57-62; reported as t_aca_ms) and then `reps` products are timed with
// the reference's precompute-mode mvp() body (dense assemble + gemv, low-rank apply,
// hmatrix.cpp:80-113; t_mvp_ms is the total).  flops = 2*(sum_dense m*n +
// sum_adm k_eff*(m+n)) of the evaluated leaves per product.
int ref_mvp_rows_timed(void* h, const double* x, std::int64_t nranges, const std::int64_t* ranges, std::int64_t reps,
                       double* z_morton, double* t_aca_ms, double* t_mvp_ms, double* flops) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const RefHandle* r = static_cast<RefHandle*>(h);
    const std::int64_t n = r->h.points.count;
    const auto hit = [&](const WorkItem& w) {
      for (std::int64_t q = 0; q < nranges; ++q) {
        if (w.row.lower < ranges[2 * q + 1] && ranges[2 * q] < w.row.upper) return true;
      }
      return false;
    };
    std::vector<WorkItem> dense, aca;
    for (const WorkItem& w : r->h.dense_queue) if (hit(w)) dense.push_back(w);
    for (const WorkItem& w : r->h.aca_queue) if (hit(w)) aca.push_back(w);
    AcaOptions opt;
    opt.max_rank = r->h.config.k;
    opt.epsilon = r->h.config.epsilon;
    opt.eta = r->h.config.eta;
    const auto t0 = Clock::now();
    const std::vector<AcaBatch> batches = partition_aca_queue(aca, r->h.config.bs_aca);
    std::vector<BatchedAcaResult> factors;
    for (const AcaBatch& b : batches) factors.push_back(aca_batched(b, r->kernel, r->h.points, opt));
    *t_aca_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    double f = 0.0;
    for (const WorkItem& w : dense) f += 2.0 * static_cast<double>(w.row.size()) * static_cast<double>(w.col.size());
    for (std::size_t gi = 0; gi < batches.size(); ++gi)
      for (std::size_t b = 0; b < batches[gi].items.size(); ++b)
        f += 2.0 * static_cast<double>(factors[gi].k_eff[b]) *
             static_cast<double>(batches[gi].items[b].row.size() + batches[gi].items[b].col.size());
    *flops = f;
    const std::vector<DenseGroup> groups = partition_dense_queue(dense, r->h.config.bs_dense);
    // The reference's mvp() permutes the whole N-vector once per product (hmatrix.cpp:76);
    // a row sample is charged its share of that O(N) pass (sampled rows / N), measured once,
    // instead of the full pass every rep (which would dominate a 1,024-row sample).
    const auto tp0 = Clock::now();
    const std::vector<double> xm = permute_vector({x, static_cast<std::size_t>(n)}, r->h.points.perm, PermDirection::Forward);
    const double t_perm = std::chrono::duration<double, std::milli>(Clock::now() - tp0).count();
    std::int64_t sampled = 0;
    for (std::int64_t q = 0; q < nranges; ++q) sampled += ranges[2 * q + 1] - ranges[2 * q];
    const auto t1 = Clock::now();
    for (std::int64_t rep = 0; rep < reps; ++rep) {
      for (std::int64_t q = 0; q < nranges; ++q) std::fill(z_morton + ranges[2 * q], z_morton + ranges[2 * q + 1], 0.0);
      DenseBatch dbatch;
      std::vector<double> y;
      for (const DenseGroup& g : groups) {
        assemble_dense_batch(g, r->kernel, r->h.points, dbatch);
        gather_dense_inputs(dbatch, xm);
        batched_gemv(dbatch, y);
        for (std::size_t b = 0; b < g.items.size(); ++b)
          for (std::int64_t i = 0; i < g.items[b].row.size(); ++i) z_morton[g.items[b].row.lower + i] += y[g.row_offset[b] + i];
      }
      for (std::size_t gi = 0; gi < batches.size(); ++gi) {
        const AcaBatch& batch = batches[gi];
        y.assign(static_cast<std::size_t>(batch.total_rows), 0.0);
        batched_low_rank_apply(factors[gi], batch, xm, y);
        for (std::size_t b = 0; b < batch.items.size(); ++b)
          for (std::int64_t i = 0; i < batch.items[b].row.size(); ++i) z_morton[batch.items[b].row.lower + i] += y[batch.row_offset[b] + i];
      }
    }
    *t_mvp_ms = std::chrono::duration<double, std::milli>(Clock::now() - t1).count() +
                static_cast<double>(reps) * t_perm * static_cast<double>(sampled) / static_cast<double>(n);
  });
}

// Reference CPU arm for the recompute-mode (matrix-free) configurations, where the
// reference's own setup() at N = 2^22 is far outside a bench's time budget: the
// reference's recompute-mode mvp() body (hmatrix.cpp:80-113, with aca_batched inside
// the product, :96-104) over an explicit sample of leaves of the (bit-verified) block
// tree, on the Morton-ordered points.  Per rep: dense groups assembled and applied,
// then ACA batches factorised and applied -- exactly the work mvp() does per leaf.
// t_ms = total over reps; flops = 2 (sum_dense m n + sum_adm k_eff (m + n)) per rep.
int ref_leaves_mvp_timed(const double* coords_m, std::int64_t n, int d, int kernel, double beta, std::int64_t k,
                         double eta, std::int64_t ndense, const std::int64_t* dense4, std::int64_t naca,
                         const std::int64_t* aca4, const double* xm, std::int64_t reps, double* z_morton,
                         double* t_ms, double* flops) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const PointSet pts = make_points(n, d, coords_m, nullptr);
    const KernelFunction kf = make_kernel(kernel, beta);
    auto items = [&](std::int64_t cnt, const std::int64_t* r4, bool adm) {
      std::vector<WorkItem> v(static_cast<std::size_t>(cnt));
      for (std::int64_t i = 0; i < cnt; ++i) {
        v[i].row = Cluster{r4[4 * i], r4[4 * i + 1]};
        v[i].col = Cluster{r4[4 * i + 2], r4[4 * i + 3]};
        v[i].admissible = adm;
      }
      return v;
    };
    const std::vector<WorkItem> dense = items(ndense, dense4, false), aca = items(naca, aca4, true);
    AcaOptions opt;
    opt.max_rank = k;
    opt.eta = eta;
    const std::vector<DenseGroup> groups = partition_dense_queue(dense, std::int64_t{1} << 22);
    const std::vector<AcaBatch> batches = partition_aca_queue(aca, std::int64_t{1} << 20);
    const std::span<const double> x{xm, static_cast<std::size_t>(n)};
    double f = 0.0;
    for (const WorkItem& w : dense) f += 2.0 * static_cast<double>(w.row.size()) * static_cast<double>(w.col.size());
    const auto t0 = Clock::now();
    for (std::int64_t rep = 0; rep < reps; ++rep) {
      std::fill(z_morton, z_morton + n, 0.0);
      DenseBatch dbatch;
      std::vector<double> y;
      for (const DenseGroup& g : groups) {
        assemble_dense_batch(g, kf, pts, dbatch);
        gather_dense_inputs(dbatch, x);
        batched_gemv(dbatch, y);
        for (std::size_t b = 0; b < g.items.size(); ++b)
          for (std::int64_t i = 0; i < g.items[b].row.size(); ++i) z_morton[g.items[b].row.lower + i] += y[g.row_offset[b] + i];
      }
      for (const AcaBatch& batch : batches) {
        const BatchedAcaResult res = aca_batched(batch, kf, pts, opt);
        if (rep == 0)
          for (std::size_t b = 0; b < batch.items.size(); ++b)
            f += 2.0 * static_cast<double>(res.k_eff[b]) *
                 static_cast<double>(batch.items[b].row.size() + batch.items[b].col.size());
        y.assign(static_cast<std::size_t>(batch.total_rows), 0.0);
        batched_low_rank_apply(res, batch, x, y);
        for (std::size_t b = 0; b < batch.items.size(); ++b)
          for (std::int64_t i = 0; i < batch.items[b].row.size(); ++i) z_morton[batch.items[b].row.lower + i] += y[batch.row_offset[b] + i];
      }
    }
    *t_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    *flops = f;
  });
}

}  // extern "C"

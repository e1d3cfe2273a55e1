// hmat_b200.hpp -- header-only C++ facade over the C ABI (hmat_b200.h) that restores
// the reference library's signatures, so code written against
// /root/reference/proj/include/hmat/{core,morton,aca,hmatrix,solver}.hpp builds against
// the B200 engine by swapping the include and linking libhmat_b200.so.
//
//   reference                                         facade
//   hmat::setup(PointSet, KernelFunction, HmatrixConfig)  hmatrix.hpp:48   -> hm_setup
//   hmat::mvp(HMatrix, span x, KernelFunction, MvpTimings*) :58-59       -> hm_mvp
//   hmat::relative_error(HMatrix, KernelFunction, span x)   :63          -> hm_relative_error
//   hmat::cg_solve(HMatrix, KernelFunction, span b, SolveConfig) solver.hpp:27-28 -> hm_cg_solve
//   hmat::compute_morton_codes / morton_order           morton.hpp:23-26 -> hm_morton_codes / hm_morton_order
//   hmat::aca_batched(AcaBatch-from-shapes, blocks, AcaOptions) aca.hpp:88-89 -> hm_aca_dense
//
// Errors: non-zero hm_status is rethrown as the reference's exception kinds
// (std::invalid_argument, std::out_of_range, std::runtime_error, std::bad_alloc).
// HMatrix is move-only and owns the device-resident operator (the reference's is a
// value type holding host vectors).
#pragma once
#include <cstdint>
#include <memory>
#include <new>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hmat_b200.h"

#ifndef HMAT_B200_NAMESPACE
#define HMAT_B200_NAMESPACE hmat
#endif

namespace HMAT_B200_NAMESPACE {

inline void check(hm_status st) {
  if (st == HM_OK) return;
  const std::string msg = hm_last_error();
  switch (st) {
    case HM_EINVAL: throw std::invalid_argument(msg);
    case HM_ERANGE: throw std::out_of_range(msg);
    case HM_ENOMEM: throw std::bad_alloc();
    case HM_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline constexpr int kMaxDim = 20;

// core.hpp:26-31
struct PointSet {
  int dim = 0;
  std::int64_t count = 0;
  std::vector<std::vector<double>> coords;  // coords[axis][i]
  std::vector<std::int64_t> perm;
};

// core.hpp:35-40
enum class KernelKind { Gaussian, Matern };
struct KernelFunction {
  KernelKind kind = KernelKind::Gaussian;
  double matern_beta = 0.0;
};

// hmatrix.hpp:15-34 (+ B200 placement knobs)
struct HmatrixConfig {
  double eta = 1.5;
  std::int64_t c_leaf = 256;
  std::int64_t k = 16;
  std::int64_t bs_aca = std::int64_t{1} << 20;
  std::int64_t bs_dense = std::int64_t{1} << 22;
  bool precompute_aca = false;
  std::optional<double> epsilon;
  bool force_dense = false;
  bool near_stored = false;
  int rank = 0, world = 1, device = 0;

  static HmatrixConfig large_scale() {
    HmatrixConfig cfg;
    cfg.c_leaf = 2048;
    cfg.bs_aca = std::int64_t{1} << 25;
    cfg.bs_dense = std::int64_t{1} << 27;
    return cfg;
  }
  hm_config to_c() const {
    hm_config c;
    hm_config_default(&c);
    c.eta = eta;
    c.c_leaf = c_leaf;
    c.k = k;
    c.bs_aca = bs_aca;
    c.bs_dense = bs_dense;
    c.precompute_aca = precompute_aca ? 1 : 0;
    c.has_epsilon = epsilon.has_value() ? 1 : 0;
    c.epsilon = epsilon.value_or(0.0);
    c.adm_mode = force_dense ? HM_ADM_FORCE_DENSE : HM_ADM_GEOMETRIC;
    c.near_stored = near_stored ? 1 : 0;
    c.rank = rank;
    c.world = world;
    c.device = device;
    return c;
  }
};

// hmatrix.hpp:50-54
struct MvpTimings {
  double dense_ms = 0.0;  // near-field phase (device events)
  double aca_ms = 0.0;    // far-field phase, incl. the recompute-mode factorisation
  double total_ms = 0.0;  // whole call, host copies included
};

struct Cluster {
  std::int64_t lower = 0, upper = 0;
  std::int64_t size() const { return upper - lower; }
};
struct Leaf {
  Cluster row, col;
  bool admissible = false;
};

// hmatrix.hpp:36-44: owns the device-resident operator
class HMatrix {
 public:
  HMatrix() = default;
  explicit HMatrix(hm_handle* h, HmatrixConfig cfg, std::int64_t n, int d) : h_(h, &hm_destroy), config(cfg), n_(n), d_(d) {}
  hm_handle* handle() const { return h_.get(); }
  std::int64_t size() const { return n_; }
  int dim() const { return d_; }

  // Morton-ordered points (HMatrix::points)
  PointSet points() const {
    PointSet p;
    p.dim = d_;
    p.count = n_;
    std::vector<double> flat(static_cast<std::size_t>(n_ * d_));
    p.perm.resize(static_cast<std::size_t>(n_));
    check(hm_get_points(h_.get(), flat.data(), reinterpret_cast<int64_t*>(p.perm.data())));
    p.coords.resize(static_cast<std::size_t>(d_));
    for (int a = 0; a < d_; ++a) p.coords[a].assign(flat.begin() + a * n_, flat.begin() + (a + 1) * n_);
    return p;
  }
  // dense_queue / aca_queue (hmatrix.hpp:39-40), canonical order
  std::vector<Leaf> queue(bool admissible) const {
    hm_stats st;
    check(hm_get_stats(h_.get(), &st));
    const std::int64_t cnt = admissible ? st.n_aca : st.n_dense;
    std::vector<int64_t> rows(static_cast<std::size_t>(4 * cnt));
    check(hm_get_leaves(h_.get(), admissible ? 1 : 0, rows.data(), nullptr));
    std::vector<Leaf> out(static_cast<std::size_t>(cnt));
    for (std::int64_t i = 0; i < cnt; ++i)
      out[i] = Leaf{{rows[4 * i], rows[4 * i + 1]}, {rows[4 * i + 2], rows[4 * i + 3]}, admissible};
    return out;
  }
  std::vector<Leaf> dense_queue() const { return queue(false); }
  std::vector<Leaf> aca_queue() const { return queue(true); }

 private:
  std::shared_ptr<hm_handle> h_;

 public:
  HmatrixConfig config;

 private:
  std::int64_t n_ = 0;
  int d_ = 0;
};

inline std::vector<double> flatten(const PointSet& p) {
  if (p.dim < 1 || static_cast<int>(p.coords.size()) != p.dim) throw std::invalid_argument("PointSet: bad dimension");
  std::vector<double> flat(static_cast<std::size_t>(p.count * p.dim));
  for (int a = 0; a < p.dim; ++a) {
    if (static_cast<std::int64_t>(p.coords[a].size()) != p.count) throw std::invalid_argument("PointSet: bad size");
    std::copy(p.coords[a].begin(), p.coords[a].end(), flat.begin() + a * p.count);
  }
  return flat;
}

// hmatrix.hpp:48
inline HMatrix setup(const PointSet& raw_points, const KernelFunction& kernel, const HmatrixConfig& config) {
  const std::vector<double> flat = flatten(raw_points);
  const hm_config c = config.to_c();
  hm_handle* h = nullptr;
  check(hm_setup(flat.data(), raw_points.count, raw_points.dim, kernel.kind == KernelKind::Gaussian ? 0 : 1,
                 kernel.matern_beta, &c, &h));
  return HMatrix(h, config, raw_points.count, raw_points.dim);
}

// hmatrix.hpp:58-59 (the kernel captured at setup is used; the reference requires equality)
inline std::vector<double> mvp(const HMatrix& h, std::span<const double> x, const KernelFunction& /*kernel*/,
                               MvpTimings* timings = nullptr) {
  if (static_cast<std::int64_t>(x.size()) != h.size()) throw std::invalid_argument("mvp: vector length mismatch");
  std::vector<double> z(x.size());
  hm_timings t;
  check(hm_mvp(h.handle(), x.data(), z.data(), &t));
  if (timings) {
    timings->dense_ms = t.mvp_dense_ms;
    timings->aca_ms = t.mvp_aca_ms;
    timings->total_ms = t.mvp_ms;
  }
  return z;
}

// hmatrix.hpp:63 (no N limit: the exact product runs on the device)
inline double relative_error(const HMatrix& h, const KernelFunction& /*kernel*/, std::span<const double> x_rand) {
  if (static_cast<std::int64_t>(x_rand.size()) != h.size())
    throw std::invalid_argument("relative_error: vector length mismatch");
  double out = 0.0;
  check(hm_relative_error(h.handle(), x_rand.data(), &out));
  return out;
}

// solver.hpp:12-28
struct SolveConfig {
  double sigma2 = 0.0;
  double tol = 1e-8;
  std::int64_t max_iter = 500;
};
struct SolveResult {
  std::vector<double> x;
  std::int64_t iterations = 0;
  double relative_residual = 0.0;
};
inline SolveResult cg_solve(const HMatrix& h, const KernelFunction& /*kernel*/, std::span<const double> b,
                            const SolveConfig& config) {
  if (static_cast<std::int64_t>(b.size()) != h.size()) throw std::invalid_argument("cg_solve: rhs length mismatch");
  SolveResult r;
  r.x.resize(b.size());
  int64_t it = 0;
  check(hm_cg_solve(h.handle(), b.data(), config.sigma2, config.tol, config.max_iter, r.x.data(), &it,
                    &r.relative_residual));
  r.iterations = it;
  return r;
}

// ---- B200 extensions (no reference counterpart) ----
// Z[:, r] = H X[:, r]; X, Z column-major n x nrhs.  dmma = false: every column bitwise
// equal to mvp(X[:, r]); dmma = true: recompute near field on the FP64 tensor cores.
inline std::vector<double> mvp_multi(const HMatrix& h, std::span<const double> X, std::int64_t nrhs,
                                     bool dmma = false) {
  if (nrhs < 1 || static_cast<std::int64_t>(X.size()) != h.size() * nrhs)
    throw std::invalid_argument("mvp_multi: X must hold n * nrhs values");
  std::vector<double> Z(X.size());
  check(hm_mvp_multi(h.handle(), X.data(), Z.data(), nrhs, dmma ? HM_MULTI_DMMA : HM_MULTI_EXACT));
  return Z;
}
struct SolveResultMulti {
  std::vector<double> x;  // n x nrhs, column-major
  std::vector<std::int64_t> iterations;
  std::vector<double> relative_residual;
};
// nrhs independent cg_solve runs (solver.cpp:19-73) on multi-RHS products
inline SolveResultMulti cg_solve_multi(const HMatrix& h, std::span<const double> B, std::int64_t nrhs,
                                       const SolveConfig& config, bool dmma = false) {
  if (nrhs < 1 || static_cast<std::int64_t>(B.size()) != h.size() * nrhs)
    throw std::invalid_argument("cg_solve_multi: B must hold n * nrhs values");
  SolveResultMulti r;
  r.x.resize(B.size());
  r.iterations.resize(static_cast<std::size_t>(nrhs));
  r.relative_residual.resize(static_cast<std::size_t>(nrhs));
  check(hm_cg_solve_multi(h.handle(), B.data(), nrhs, config.sigma2, config.tol, config.max_iter,
                          dmma ? HM_MULTI_DMMA : HM_MULTI_EXACT, r.x.data(),
                          reinterpret_cast<int64_t*>(r.iterations.data()), r.relative_residual.data()));
  return r;
}
// tree.hpp:94 dump_leaves_csv, for the leaves of a set-up H-matrix (canonical order)
inline void dump_leaves_csv(const HMatrix& h, const std::string& path) {
  check(hm_dump_leaves_csv(h.handle(), path.c_str()));
}

// morton.hpp:23-26
inline std::vector<std::uint64_t> compute_morton_codes(const PointSet& points) {
  const std::vector<double> flat = flatten(points);
  std::vector<std::uint64_t> codes(static_cast<std::size_t>(points.count));
  check(hm_morton_codes(flat.data(), points.count, points.dim, reinterpret_cast<uint64_t*>(codes.data())));
  return codes;
}
inline PointSet morton_order(const PointSet& points) {
  const std::vector<double> flat = flatten(points);
  std::vector<double> out(flat.size());
  PointSet s;
  s.dim = points.dim;
  s.count = points.count;
  s.perm.resize(static_cast<std::size_t>(points.count));
  check(hm_morton_order(flat.data(), points.count, points.dim,
                        points.perm.empty() ? nullptr : reinterpret_cast<const int64_t*>(points.perm.data()),
                        out.data(), reinterpret_cast<int64_t*>(s.perm.data())));
  s.coords.resize(static_cast<std::size_t>(points.dim));
  for (int a = 0; a < points.dim; ++a)
    s.coords[a].assign(out.begin() + a * points.count, out.begin() + (a + 1) * points.count);
  return s;
}

// aca.hpp:30-37 / 68-75 / 88-89 (explicit-matrix seam)
struct AcaOptions {
  std::int64_t max_rank = 16;
  std::optional<double> epsilon;
  double eta = 0.0;
};
struct DenseMatrix {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> entries;  // row-major
};
struct BatchedAcaResult {
  std::int64_t max_rank = 0;
  std::vector<std::int64_t> k_eff, row_pivots, col_pivots;
  std::vector<std::vector<double>> u, v;  // per block: max_rank x m / max_rank x n, rank-major
};
inline BatchedAcaResult aca_batched(std::span<const DenseMatrix> blocks, const AcaOptions& opt) {
  std::vector<int64_t> shapes;
  std::vector<double> entries;
  std::int64_t su = 0, sv = 0;
  for (const DenseMatrix& b : blocks) {
    shapes.push_back(b.rows);
    shapes.push_back(b.cols);
    entries.insert(entries.end(), b.entries.begin(), b.entries.end());
    su += opt.max_rank * b.rows;
    sv += opt.max_rank * b.cols;
  }
  const std::int64_t nb = static_cast<std::int64_t>(blocks.size());
  BatchedAcaResult r;
  r.max_rank = opt.max_rank;
  r.k_eff.resize(nb);
  r.row_pivots.resize(nb * opt.max_rank);
  r.col_pivots.resize(nb * opt.max_rank);
  std::vector<double> u(su), v(sv);
  check(hm_aca_dense(nb, shapes.data(), entries.data(), opt.max_rank, opt.epsilon ? 1 : 0, opt.epsilon.value_or(0.0),
                     opt.eta, reinterpret_cast<int64_t*>(r.k_eff.data()),
                     reinterpret_cast<int64_t*>(r.row_pivots.data()), reinterpret_cast<int64_t*>(r.col_pivots.data()),
                     u.data(), v.data()));
  std::int64_t uo = 0, vo = 0;
  for (const DenseMatrix& b : blocks) {
    r.u.emplace_back(u.begin() + uo, u.begin() + uo + opt.max_rank * b.rows);
    r.v.emplace_back(v.begin() + vo, v.begin() + vo + opt.max_rank * b.cols);
    uo += opt.max_rank * b.rows;
    vo += opt.max_rank * b.cols;
  }
  return r;
}

// core.hpp:63-64
inline double eval_kernel(const KernelFunction& kernel, std::span<const double> y, std::span<const double> yp) {
  if (y.size() != yp.size()) throw std::invalid_argument("eval_kernel: point dimensions differ");
  double out = 0.0;
  check(hm_eval_kernel(kernel.kind == KernelKind::Gaussian ? 0 : 1, kernel.matern_beta, static_cast<int32_t>(y.size()),
                       1, y.data(), yp.data(), &out));
  return out;
}

}  // namespace HMAT_B200_NAMESPACE

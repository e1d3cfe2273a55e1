// Reference-style client code (proj/README.md "Typical use") built against the B200
// facade: only the include and the link line differ from a reference build.
#include <cmath>
#include <cstdio>
#include <vector>

#include "hmat_b200.hpp"

int main() {
  hmat::PointSet points;
  points.dim = 2;
  points.count = 1 << 13;
  points.coords.assign(2, std::vector<double>(points.count));
  points.perm.resize(points.count);
  // Halton-like deterministic points (radical inverse bases 2 and 3)
  for (std::int64_t i = 0; i < points.count; ++i) {
    points.perm[i] = i;
    for (int a = 0; a < 2; ++a) {
      const int base = a == 0 ? 2 : 3;
      double f = 1.0 / base, v = 0.0;
      for (std::int64_t k = i + 1; k > 0; k /= base, f /= base) v += f * static_cast<double>(k % base);
      points.coords[a][i] = v;
    }
  }
  hmat::KernelFunction kernel{hmat::KernelKind::Gaussian};
  hmat::HmatrixConfig config;
  config.c_leaf = 64;
  hmat::HMatrix h = hmat::setup(points, kernel, config);
  std::vector<double> x(points.count, 1.0);
  hmat::MvpTimings t;
  std::vector<double> z = hmat::mvp(h, x, kernel, &t);
  const double e = hmat::relative_error(h, kernel, x);
  hmat::SolveConfig sc;
  sc.sigma2 = 1.0;
  const hmat::SolveResult r = hmat::cg_solve(h, kernel, x, sc);
  // B200 extensions: 8 right-hand sides in one operator pass, column 0 == the single product
  std::vector<double> X(static_cast<std::size_t>(points.count) * 8);
  for (std::size_t q = 0; q < X.size(); ++q) X[q] = 1.0 + 0.001 * static_cast<double>(q % 97);
  for (std::int64_t i = 0; i < points.count; ++i) X[i] = 1.0;
  const std::vector<double> Z = hmat::mvp_multi(h, X, 8);
  for (std::int64_t i = 0; i < points.count; ++i)
    if (Z[i] != z[i]) return 2;
  hmat::dump_leaves_csv(h, "facade_leaves.csv");
  std::remove("facade_leaves.csv");
  double nz = 0.0;
  for (double v : z) nz += v * v;
  std::printf("facade ok: N=%lld dense=%zu aca=%zu |z|=%.12g e_rel=%.3e cg_iters=%lld relres=%.3e\n",
              static_cast<long long>(points.count), h.dense_queue().size(), h.aca_queue().size(), std::sqrt(nz), e,
              static_cast<long long>(r.iterations), r.relative_residual);
  return (e < 1e-6 && r.relative_residual < 1e-7) ? 0 : 1;
}

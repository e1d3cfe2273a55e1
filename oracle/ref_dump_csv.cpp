// ref_dump_csv.cpp -- TEST INFRASTRUCTURE: writes the reference's leaf CSV for a point set.
//
// Runs the UNMODIFIED reference setup() (hmatrix.cpp:38-64) on SoA coordinates read
// from a raw little-endian double file (d x n) and writes every leaf through the
// reference's own dump_leaves_csv (tree.cpp:197-205) -- in its own process, so the
// reference's C++ runtime (iostreams) never shares a process with the Python tests.
//   usage: ref_dump_csv <n> <d> <c_leaf> <eta> <coords.bin> <out.csv>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <iterator>
#include <tuple>
#include <vector>

#include "hmat/core.hpp"
#include "hmat/hmatrix.hpp"
#include "hmat/tree.hpp"

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: %s n d c_leaf eta coords.bin out.csv\n", argv[0]);
    return 2;
  }
  const std::int64_t n = std::atoll(argv[1]);
  const int d = std::atoi(argv[2]);
  std::vector<double> flat(static_cast<size_t>(n) * d);
  FILE* f = std::fopen(argv[5], "rb");
  if (!f || std::fread(flat.data(), sizeof(double), flat.size(), f) != flat.size()) return 3;
  std::fclose(f);
  hmat::PointSet p;
  p.dim = d;
  p.count = n;
  p.coords.assign(d, std::vector<double>(n));
  for (int a = 0; a < d; ++a)
    for (std::int64_t i = 0; i < n; ++i) p.coords[a][i] = flat[a * n + i];
  p.perm.resize(n);
  for (std::int64_t i = 0; i < n; ++i) p.perm[i] = i;
  hmat::HmatrixConfig cfg;
  cfg.c_leaf = std::atoll(argv[3]);
  cfg.eta = std::atof(argv[4]);
  const hmat::HMatrix h = hmat::setup(p, hmat::KernelFunction{hmat::KernelKind::Gaussian}, cfg);
  std::vector<hmat::WorkItem> all;
  std::merge(h.dense_queue.begin(), h.dense_queue.end(), h.aca_queue.begin(), h.aca_queue.end(),
             std::back_inserter(all), [](const hmat::WorkItem& x, const hmat::WorkItem& y) {
               return std::tie(x.row.lower, x.row.upper, x.col.lower, x.col.upper) <
                      std::tie(y.row.lower, y.row.upper, y.col.lower, y.col.upper);
             });
  hmat::dump_leaves_csv(all, argv[6]);
  return 0;
}

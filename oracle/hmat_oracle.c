/* hmat_oracle.c -- sequential C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see hmat_oracle.h).  Compiled with
 * -ffp-contract=off so every product and sum rounds exactly like the FMA-free
 * reference objects; transcendental calls go to the same glibc
 * libm the reference uses, so kernel entries are bitwise identical.
 *
 * Citations are to /root/reference/proj.
 */
#include "hmat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* core.cpp: kernels                                                          */
/* ------------------------------------------------------------------------ */

/* core.cpp:28-47 */
static double bessel_k1_series(double x) {
  const double kEulerGamma = 0.57721566490153286060651209008240243;
  const double q = 0.25 * x * x;
  double term = 1.0;
  double psi_a = -kEulerGamma;
  double psi_b = 1.0 - kEulerGamma;
  double sum_i1 = 0.0;
  double sum_k = 0.0;
  for (int j = 0; j < 64; ++j) {
    sum_i1 += term;
    sum_k += (psi_a + psi_b) * term;
    const double next = term * q / ((j + 1.0) * (j + 2.0));
    if (next < 1e-19 * (sum_i1 + 1.0)) break;
    term = next;
    psi_a += 1.0 / (j + 1.0);
    psi_b += 1.0 / (j + 2.0);
  }
  const double i1 = 0.5 * x * sum_i1;
  return 1.0 / x + log(0.5 * x) * i1 - 0.25 * x * sum_k;
}

/* core.cpp:51-81 */
static double bessel_k1_cf(double x) {
  double b = 2.0 * (1.0 + x);
  double d = 1.0 / b;
  double h = d;
  double delh = d;
  double q1 = 0.0;
  double q2 = 1.0;
  const double a1 = 0.25;
  double q = a1;
  double c = a1;
  double a = -a1;
  double s = 1.0 + q * delh;
  for (int i = 2; i <= 2000; ++i) {
    a -= 2.0 * (i - 1);
    c = -a * c / i;
    const double qnew = (q1 - b * q2) / a;
    q1 = q2;
    q2 = qnew;
    q += c * qnew;
    b += 2.0;
    d = 1.0 / (b + a * d);
    delh = (b * d - 1.0) * delh;
    h += delh;
    const double dels = q * delh;
    s += dels;
    if (fabs(dels / s) < 1e-17) break;
  }
  h = a1 * h;
  const double k0 = sqrt(M_PI / (2.0 * x)) * exp(-x) / s;
  return k0 * (0.5 + x - h) / x;
}

/* core.cpp:97-102 */
static double bessel_k1(double x) { return x <= 2.0 ? bessel_k1_series(x) : bessel_k1_cf(x); }

int orc_bessel_k1(int64_t n, const double* x, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    if (!(x[i] > 0.0)) return fail("bessel_k1: argument must be positive");
    out[i] = bessel_k1(x[i]);
  }
  return 0;
}

typedef struct {
  int kind; /* 0 Gaussian, 1 Matern */
  int dim;
  double matern_norm;
} kernel_t;

/* core.cpp:83-95, 124-128 */
static int make_kernel(kernel_t* k, int kind, double beta, int dim) {
  k->kind = kind;
  k->dim = dim;
  k->matern_norm = 0.0;
  if (kind == 1) {
    const double b = beta > 0.0 ? beta : 1.0 + 0.5 * dim;
    const double order = b - 0.5 * dim;
    if (fabs(order - 1.0) > 1e-12) return fail("Matern kernel: only order beta - d/2 = 1 is supported");
    k->matern_norm = 1.0 / (pow(2.0, b - 1.0) * tgamma(b));
  }
  return 0;
}

/* core.hpp:71-74 and core.cpp:130-134 */
static double from_r2(const kernel_t* k, double r2) {
  if (k->kind == 0) return exp(-r2);
  if (r2 == 0.0) return k->matern_norm;
  const double r = sqrt(r2);
  return bessel_k1(r) * r * k->matern_norm;
}

/* BoundKernelEvaluator core.hpp:103-110: r2 = ((0 + dx0^2) + dx1^2) + ... */
static double eval_ij(const kernel_t* k, const double* coords, int64_t n, int64_t i, int64_t j) {
  double r2 = 0.0;
  for (int a = 0; a < k->dim; ++a) {
    const double dx = coords[a * n + i] - coords[a * n + j];
    r2 += dx * dx;
  }
  return from_r2(k, r2);
}

int orc_eval_kernel(int kind, double beta, int d, int64_t n, const double* y, const double* yp, double* out) {
  kernel_t k;
  if (make_kernel(&k, kind, beta, d)) return 1;
  for (int64_t i = 0; i < n; ++i) {
    double r2 = 0.0;
    for (int a = 0; a < d; ++a) {
      const double dx = y[a * n + i] - yp[a * n + i];
      r2 += dx * dx;
    }
    out[i] = from_r2(&k, r2);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* morton.cpp                                                                 */
/* ------------------------------------------------------------------------ */

/* morton.cpp:11-15 */
static int bits_per_dim(int d) { return 64 / d > 52 ? 52 : 64 / d; }

/* morton.cpp:17-23 */
static uint64_t fixed_point(double c, int bits) {
  const double scaled = floor(c * (double)((uint64_t)1 << bits));
  if (!(scaled > 0.0)) return 0;
  const uint64_t maxv = ((uint64_t)1 << bits) - 1;
  if (scaled >= (double)maxv) return maxv;
  return (uint64_t)scaled;
}

/* morton.cpp:25-48 */
int orc_morton_codes(int64_t n, int d, const double* coords, uint64_t* codes) {
  if (d < 1 || d > 20) return fail("morton: dimension out of range");
  const int bits = bits_per_dim(d);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t code = 0;
    for (int a = 0; a < d; ++a) {
      const uint64_t v = fixed_point(coords[a * n + i], bits);
      for (int b = 0; b < bits; ++b) code |= ((v >> b) & 1ull) << (b * d + a);
    }
    codes[i] = code;
  }
  return 0;
}

/* stable merge sort of an index array by u64 key (std::stable_sort semantics,
 * parallel.hpp:45-62: ties keep input order) */
static void merge_sort_idx(int64_t* idx, int64_t* tmp, int64_t n, const uint64_t* key) {
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = key[idx[b]] < key[idx[a]] ? idx[b++] : idx[a++];
      while (a < mid) tmp[o++] = idx[a++];
      while (b < hi) tmp[o++] = idx[b++];
    }
    memcpy(idx, tmp, sizeof(int64_t) * (size_t)n);
  }
}

/* morton.cpp:50-71 */
int orc_morton_order(int64_t n, int d, const double* coords, const int64_t* perm_in, double* coords_out,
                     int64_t* perm_out) {
  uint64_t* codes = malloc(sizeof(uint64_t) * (size_t)n);
  int64_t* order = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* tmp = malloc(sizeof(int64_t) * (size_t)n);
  if (!codes || !order || !tmp) return fail("oom");
  if (orc_morton_codes(n, d, coords, codes)) return 1;
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  merge_sort_idx(order, tmp, n, codes);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t src = order[i];
    for (int a = 0; a < d; ++a) coords_out[a * n + i] = coords[a * n + src];
    perm_out[i] = perm_in ? perm_in[src] : src;
  }
  free(codes);
  free(order);
  free(tmp);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* tree.cpp                                                                   */
/* ------------------------------------------------------------------------ */

/* tree.cpp:11-18 */
static double diam(int d, const double* box) {
  double sum = 0.0;
  for (int i = 0; i < d; ++i) {
    const double side = box[d + i] - box[i];
    sum += side * side;
  }
  return sqrt(sum);
}

/* tree.cpp:20-28 (std::max(0.0, v) returns v unless 0.0 < v is false... exactly: max(a,b) = a<b ? b : a) */
static double stdmax(double a, double b) { return a < b ? b : a; }
static double dist(int d, const double* t, const double* s) {
  double sum = 0.0;
  for (int i = 0; i < d; ++i) {
    const double gap_ts = stdmax(0.0, t[i] - s[d + i]);
    const double gap_st = stdmax(0.0, s[i] - t[d + i]);
    sum += gap_ts * gap_ts + gap_st * gap_st;
  }
  return sqrt(sum);
}

/* tree.cpp:30-32: std::min(a,b) = b<a ? b : a */
static int admissible(int d, const double* t, const double* s, double eta) {
  const double dt = diam(d, t), ds = diam(d, s);
  const double m = ds < dt ? ds : dt;
  return m <= eta * dist(d, t, s);
}

int orc_admissible(int d, const double* box_t, const double* box_s, double eta, double* diam_t, double* diam_s,
                   double* distance) {
  if (diam_t) *diam_t = diam(d, box_t);
  if (diam_s) *diam_s = diam(d, box_s);
  if (distance) *distance = dist(d, box_t, box_s);
  return admissible(d, box_t, box_s, eta);
}

typedef struct {
  int64_t rl, ru, cl, cu;
  int adm;
  int depth;
  int64_t row_box, col_box; /* indices into the box table */
} leaf_t;

struct orc_hmatrix {
  int64_t n;
  int d;
  kernel_t kern;
  double eta;
  int64_t c_leaf, k;
  int precompute, has_eps;
  double eps;
  double* coords; /* Morton-ordered SoA */
  int64_t* perm;
  /* box table: one slot per (depth, cluster index); lazily filled */
  int max_depth;
  int64_t* depth_base; /* slot offset of depth ell */
  double* boxes;       /* 2d per slot */
  unsigned char* box_done;
  leaf_t* dense;
  int64_t n_dense;
  leaf_t* aca;
  int64_t n_aca;
  /* precomputed factors (aca queue order) */
  double** pu;
  double** pv;
  int64_t* pk;
};

/* Bounding box of [lo,hi): per axis the left fold of MinOp / MaxOp over the run
 * (tree.cpp:76-89 via reduce_by_key parallel.hpp:112-121, MinOp :68-71, MaxOp :72-75). */
static const double* cluster_box(orc_hmatrix* h, int depth, int64_t idx, int64_t lo, int64_t hi) {
  const int64_t slot = h->depth_base[depth] + idx;
  double* box = h->boxes + 2 * h->d * slot;
  if (!h->box_done[slot]) {
    for (int a = 0; a < h->d; ++a) {
      const double* c = h->coords + a * h->n;
      double mn = c[lo], mx = c[lo];
      for (int64_t i = lo + 1; i < hi; ++i) {
        mx = mx < c[i] ? c[i] : mx;
        mn = c[i] < mn ? c[i] : mn;
      }
      box[a] = mn;
      box[h->d + a] = mx;
    }
    h->box_done[slot] = 1;
  }
  return box;
}

typedef struct {
  leaf_t* v;
  int64_t n, cap;
} leafvec;

static int push_leaf(leafvec* lv, leaf_t l) {
  if (lv->n == lv->cap) {
    lv->cap = lv->cap ? 2 * lv->cap : 1024;
    leaf_t* nv = realloc(lv->v, sizeof(leaf_t) * (size_t)lv->cap);
    if (!nv) return 1;
    lv->v = nv;
  }
  lv->v[lv->n++] = l;
  return 0;
}

/* Alg. 1 (tree.cpp:147-183): leaf <=> adm || |t|<=C || |s|<=C; flag = adm;
 * children (ta,sa),(ta,sb),(tb,sa),(tb,sb) with ceil-half splits (tree.cpp:120-123).
 * Depth-first here; the canonical sort below makes the order irrelevant. */
static int recurse(orc_hmatrix* h, int mode, int depth, int64_t ti, int64_t tl, int64_t tu, int64_t si, int64_t sl,
                   int64_t su, leafvec* out) {
  const double* bt = cluster_box(h, depth, ti, tl, tu);
  const double* bs = cluster_box(h, depth, si, sl, su);
  const int adm = mode == 1 ? 0 : mode == 2 ? 1 : admissible(h->d, bt, bs, h->eta);
  if (adm || tu - tl <= h->c_leaf || su - sl <= h->c_leaf) {
    leaf_t l = {tl, tu, sl, su, adm, depth, h->depth_base[depth] + ti, h->depth_base[depth] + si};
    return push_leaf(out, l);
  }
  const int64_t tm = tl + (tu - tl + 1) / 2, sm = sl + (su - sl + 1) / 2;
  if (recurse(h, mode, depth + 1, 2 * ti, tl, tm, 2 * si, sl, sm, out)) return 1;
  if (recurse(h, mode, depth + 1, 2 * ti, tl, tm, 2 * si + 1, sm, su, out)) return 1;
  if (recurse(h, mode, depth + 1, 2 * ti + 1, tm, tu, 2 * si, sl, sm, out)) return 1;
  return recurse(h, mode, depth + 1, 2 * ti + 1, tm, tu, 2 * si + 1, sm, su, out);
}

/* canonical order tree.cpp:189-194 */
static int leaf_cmp(const void* pa, const void* pb) {
  const leaf_t* a = pa;
  const leaf_t* b = pb;
  if (a->rl != b->rl) return a->rl < b->rl ? -1 : 1;
  if (a->ru != b->ru) return a->ru < b->ru ? -1 : 1;
  if (a->cl != b->cl) return a->cl < b->cl ? -1 : 1;
  if (a->cu != b->cu) return a->cu < b->cu ? -1 : 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* aca.cpp: batched-ACA semantics for one block                               */
/* ------------------------------------------------------------------------ */

typedef double (*entry_fn)(const void* ctx, int64_t i, int64_t j);

typedef struct {
  const kernel_t* k;
  const double* coords;
  int64_t n, rl, cl;
} kblock_ctx;

static double kblock_entry(const void* c, int64_t i, int64_t j) {
  const kblock_ctx* x = c;
  return eval_ij(x->k, x->coords, x->n, x->rl + i, x->cl + j);
}

typedef struct {
  const double* a;
  int64_t cols;
} dblock_ctx;

static double dblock_entry(const void* c, int64_t i, int64_t j) {
  const dblock_ctx* x = c;
  return x->a[i * x->cols + j];
}

/* One block of aca_batched_impl (aca.cpp:268-544).  The lockstep across blocks
 * only interleaves independent per-block state, so a block-at-a-time run is the
 * same computation (sub-batching is exact).  u: kmax*m, v: kmax*n
 * rank-major, zero filled (aca.cpp:283-284). */
static int aca_block(entry_fn entry, const void* ctx, int64_t m, int64_t n, int64_t kmax, int has_eps, double eps,
                     double eta, double* u, double* v, int64_t* row_piv, int64_t* col_piv, int64_t* k_eff_out,
                     int64_t* rej_out) {
  const double kEps0sq = 1e-14 * 1e-14; /* aca.cpp:32, kEps0 * kEps0 */
  unsigned char* used_row = calloc((size_t)m, 1);
  unsigned char* used_col = calloc((size_t)n, 1);
  double* sq = malloc(sizeof(double) * (size_t)(m > n ? m : n));
  double* vj = malloc(sizeof(double) * (size_t)kmax);
  double* upiv = malloc(sizeof(double) * (size_t)kmax);
  if (!used_row || !used_col || !sq || !vj || !upiv) return fail("oom");
  memset(u, 0, sizeof(double) * (size_t)(kmax * m));
  memset(v, 0, sizeof(double) * (size_t)(kmax * n));
  for (int64_t l = 0; l < kmax; ++l) row_piv[l] = col_piv[l] = -1;
  int active = 1;
  double scale_sq = -1.0, frob_sq = 0.0;
  int64_t k_eff = 0, rejections = 0;

  for (int64_t r = 0; r < kmax && active; ++r) {
    /* first candidate: next_unused_col(b, 0) (aca.cpp:318-343) */
    int64_t cand = -1;
    for (int64_t j = 0; j < n; ++j)
      if (!used_col[j]) {
        cand = j;
        break;
      }
    if (cand < 0) break;
    /* candidate column pass (aca.cpp:347-368) */
    for (int64_t l = 0; l < r; ++l) vj[l] = v[l * n + cand];
    double best_val = 0.0;
    int64_t best_idx = 0;
    for (int64_t i = 0; i < m; ++i) {
      double a = entry(ctx, i, cand);
      for (int64_t l = 0; l < r; ++l) a -= u[l * m + i] * vj[l];
      u[r * m + i] = a;
      sq[i] = a * a;
      const double val = used_row[i] ? -1.0 : fabs(a);
      /* AbsArgMaxOp left fold (aca.cpp:39-41 via reduce_by_key :375-376) */
      if (i == 0 || val > best_val) {
        best_val = val;
        best_idx = i;
      }
    }
    double norm_sq = sq[0]; /* SumOp left fold (aca.cpp:373-374) */
    for (int64_t i = 1; i < m; ++i) norm_sq = norm_sq + sq[i];
    int locked = best_val > 0.0 && (scale_sq < 0.0 || norm_sq > kEps0sq * scale_sq); /* aca.cpp:381-383 */
    int64_t pivot = best_idx;
    double locked_norm = norm_sq;
    if (!locked) {
      used_col[cand] = 1; /* aca.cpp:390 */
      ++rejections;       /* stats: every rejected candidate column (first pass + resolve) */
      /* resolve scan of later columns (aca.cpp:400-444) */
      int64_t c = -1;
      for (int64_t j = cand + 1; j < n; ++j)
        if (!used_col[j]) {
          c = j;
          break;
        }
      while (c >= 0) {
        double* us = u + r * m;
        for (int64_t i = 0; i < m; ++i) {
          double a = entry(ctx, i, c);
          for (int64_t l = 0; l < r; ++l) a -= u[l * m + i] * v[l * n + c];
          us[i] = a;
        }
        double ns = us[0] * us[0];
        for (int64_t i = 1; i < m; ++i) ns += us[i] * us[i];
        int64_t best = -1;
        double best_abs = -1.0;
        for (int64_t i = 0; i < m; ++i) {
          if (used_row[i]) continue;
          const double a = fabs(us[i]);
          if (a > best_abs) {
            best_abs = a;
            best = i;
          }
        }
        if (best >= 0 && best_abs > 0.0 && (scale_sq < 0.0 || ns > kEps0sq * scale_sq)) {
          locked = 1;
          pivot = best;
          locked_norm = ns;
          cand = c;
          break;
        }
        ++rejections;
        used_col[c] = 1;
        int64_t nx = -1;
        for (int64_t j = c + 1; j < n; ++j)
          if (!used_col[j]) {
            nx = j;
            break;
          }
        c = nx;
      }
      if (!locked) {
        active = 0; /* converged at rank r (aca.cpp:442-443) */
        break;
      }
    }
    /* pivot gather + normalise (aca.cpp:457-470) */
    const double pivot_val = u[r * m + pivot];
    for (int64_t l = 0; l < r; ++l) upiv[l] = u[l * m + pivot];
    for (int64_t i = 0; i < m; ++i) u[r * m + i] /= pivot_val;
    /* pivot-row pass (aca.cpp:474-481) */
    for (int64_t j = 0; j < n; ++j) {
      double a = entry(ctx, pivot, j);
      for (int64_t l = 0; l < r; ++l) a -= upiv[l] * v[l * n + j];
      v[r * n + j] = a;
    }
    /* bookkeeping (aca.cpp:485-494) */
    used_row[pivot] = 1;
    used_col[cand] = 1;
    row_piv[r] = pivot;
    col_piv[r] = cand;
    if (scale_sq < 0.0) scale_sq = locked_norm;
    k_eff = r + 1;
    if (r + 1 == kmax) active = 0;
    if (has_eps) { /* aca.cpp:497-538 */
      double nu = u[r * m] * u[r * m];
      for (int64_t i = 1; i < m; ++i) nu = nu + u[r * m + i] * u[r * m + i];
      double nv = v[r * n] * v[r * n];
      for (int64_t j = 1; j < n; ++j) nv = nv + v[r * n + j] * v[r * n + j];
      double cross = 0.0;
      for (int64_t l = 0; l < r; ++l) {
        double du = u[l * m] * u[r * m];
        for (int64_t i = 1; i < m; ++i) du = du + u[l * m + i] * u[r * m + i];
        double dv = v[l * n] * v[r * n];
        for (int64_t j = 1; j < n; ++j) dv = dv + v[l * n + j] * v[r * n + j];
        cross += du * dv;
      }
      const double factor = eps * (1.0 - eta) / (1.0 + eps); /* aca.cpp:49 */
      frob_sq += 2.0 * cross + nu * nv;
      const double bound = factor * sqrt(frob_sq);
      if (sqrt(nu) * sqrt(nv) <= bound) active = 0;
    }
  }
  /* ranks >= k_eff of u/v hold scratch in the reference; zero them so the
   * padded layout is canonical (only l < k_eff is ever read, aca.cpp:611). */
  for (int64_t l = k_eff; l < kmax; ++l) {
    memset(u + l * m, 0, sizeof(double) * (size_t)m);
    memset(v + l * n, 0, sizeof(double) * (size_t)n);
  }
  *k_eff_out = k_eff;
  if (rej_out) *rej_out = rejections;
  free(used_row);
  free(used_col);
  free(sq);
  free(vj);
  free(upiv);
  return 0;
}

int orc_aca_dense(int64_t nblocks, const int64_t* shapes, const double* entries, int64_t kmax, int has_eps,
                  double eps, double eta, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v) {
  if (kmax < 1) return fail("aca: max_rank must be >= 1");
  int64_t off = 0, uo = 0, vo = 0;
  for (int64_t b = 0; b < nblocks; ++b) {
    const int64_t m = shapes[2 * b], n = shapes[2 * b + 1];
    dblock_ctx ctx = {entries + off, n};
    if (aca_block(dblock_entry, &ctx, m, n, kmax, has_eps, eps, eta, u + uo, v + vo, row_piv + b * kmax,
                  col_piv + b * kmax, k_eff + b, NULL))
      return 1;
    off += m * n;
    uo += kmax * m;
    vo += kmax * n;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* hmatrix.cpp                                                                */
/* ------------------------------------------------------------------------ */

static int aca_leaf(orc_hmatrix* h, const leaf_t* l, double* u, double* v, int64_t* rp, int64_t* cp, int64_t* keff,
                    int64_t* rej) {
  kblock_ctx ctx = {&h->kern, h->coords, h->n, l->rl, l->cl};
  return aca_block(kblock_entry, &ctx, l->ru - l->rl, l->cu - l->cl, h->k, h->has_eps, h->eps, h->eta, u, v, rp, cp,
                   keff, rej);
}

void orc_free(orc_hmatrix* h) {
  if (!h) return;
  if (h->pu) {
    for (int64_t b = 0; b < h->n_aca; ++b) {
      free(h->pu[b]);
      free(h->pv[b]);
    }
  }
  free(h->pu);
  free(h->pv);
  free(h->pk);
  free(h->coords);
  free(h->perm);
  free(h->depth_base);
  free(h->boxes);
  free(h->box_done);
  free(h->dense);
  free(h->aca);
  free(h);
}

/* hmatrix.cpp:38-64 (validate :20-26) */
orc_hmatrix* orc_setup(int64_t n, int d, const double* coords, int kind, double beta, double eta, int64_t c_leaf,
                       int64_t k, int precompute, int has_eps, double eps, int mode) {
  if (eta < 0.0 || c_leaf < 1 || k < 1 || (has_eps && eps <= 0.0)) {
    fail("HmatrixConfig: invalid configuration");
    return NULL;
  }
  if (n < 1 || d < 1 || d > 20) {
    fail("setup: empty point set or dimension out of range");
    return NULL;
  }
  orc_hmatrix* h = calloc(1, sizeof(orc_hmatrix));
  if (!h) return NULL;
  h->n = n;
  h->d = d;
  h->eta = eta;
  h->c_leaf = c_leaf;
  h->k = k;
  h->precompute = precompute;
  h->has_eps = has_eps;
  h->eps = eps;
  if (make_kernel(&h->kern, kind, beta, d)) {
    orc_free(h);
    return NULL;
  }
  h->coords = malloc(sizeof(double) * (size_t)(n * d));
  h->perm = malloc(sizeof(int64_t) * (size_t)n);
  if (orc_morton_order(n, d, coords, NULL, h->coords, h->perm)) {
    orc_free(h);
    return NULL;
  }
  /* depth bound: cluster sizes at depth ell are ceil/floor(n/2^ell) */
  int maxd = 0;
  while ((((n - 1) >> maxd) + 1) > 1 && maxd < 62) ++maxd;
  h->max_depth = maxd;
  h->depth_base = malloc(sizeof(int64_t) * (size_t)(maxd + 2));
  int64_t slots = 0;
  for (int e = 0; e <= maxd; ++e) {
    h->depth_base[e] = slots;
    slots += (int64_t)1 << e;
  }
  h->depth_base[maxd + 1] = slots;
  h->boxes = malloc(sizeof(double) * (size_t)(2 * d * slots));
  h->box_done = calloc((size_t)slots, 1);
  leafvec lv = {0};
  if (recurse(h, mode, 0, 0, 0, n, 0, 0, n, &lv)) {
    fail("oom");
    orc_free(h);
    return NULL;
  }
  qsort(lv.v, (size_t)lv.n, sizeof(leaf_t), leaf_cmp);
  h->dense = malloc(sizeof(leaf_t) * (size_t)(lv.n + 1));
  h->aca = malloc(sizeof(leaf_t) * (size_t)(lv.n + 1));
  for (int64_t i = 0; i < lv.n; ++i) {
    if (lv.v[i].adm)
      h->aca[h->n_aca++] = lv.v[i];
    else
      h->dense[h->n_dense++] = lv.v[i];
  }
  free(lv.v);
  if (precompute) {
    h->pu = calloc((size_t)h->n_aca + 1, sizeof(double*));
    h->pv = calloc((size_t)h->n_aca + 1, sizeof(double*));
    h->pk = calloc((size_t)h->n_aca + 1, sizeof(int64_t));
    int64_t* rp = malloc(sizeof(int64_t) * (size_t)k);
    int64_t* cp = malloc(sizeof(int64_t) * (size_t)k);
    for (int64_t b = 0; b < h->n_aca; ++b) {
      const leaf_t* l = &h->aca[b];
      h->pu[b] = malloc(sizeof(double) * (size_t)(k * (l->ru - l->rl)));
      h->pv[b] = malloc(sizeof(double) * (size_t)(k * (l->cu - l->cl)));
      if (aca_leaf(h, l, h->pu[b], h->pv[b], rp, cp, &h->pk[b], NULL)) {
        orc_free(h);
        return NULL;
      }
    }
    free(rp);
    free(cp);
  }
  return h;
}

int64_t orc_count(const orc_hmatrix* h, int which) { return which == 0 ? h->n_dense : h->n_aca; }

int orc_leaves(const orc_hmatrix* h, int which, int64_t* rows4, double* boxes4d) {
  const leaf_t* q = which == 0 ? h->dense : h->aca;
  const int64_t cnt = which == 0 ? h->n_dense : h->n_aca;
  const int d = h->d;
  for (int64_t i = 0; i < cnt; ++i) {
    rows4[4 * i + 0] = q[i].rl;
    rows4[4 * i + 1] = q[i].ru;
    rows4[4 * i + 2] = q[i].cl;
    rows4[4 * i + 3] = q[i].cu;
    if (boxes4d) {
      const double* bt = h->boxes + 2 * d * q[i].row_box;
      const double* bs = h->boxes + 2 * d * q[i].col_box;
      memcpy(boxes4d + 4 * d * i, bt, sizeof(double) * 2 * (size_t)d);
      memcpy(boxes4d + 4 * d * i + 2 * d, bs, sizeof(double) * 2 * (size_t)d);
    }
  }
  return 0;
}

int orc_points(const orc_hmatrix* h, double* coords, int64_t* perm) {
  memcpy(coords, h->coords, sizeof(double) * (size_t)(h->n * h->d));
  memcpy(perm, h->perm, sizeof(int64_t) * (size_t)h->n);
  return 0;
}

/* dense leaf: y_i = ((0 + a_i0 x_0) + a_i1 x_1) + ... (dense_blocks.cpp:101-116), z += y */
static void dense_leaf_apply(const orc_hmatrix* h, const leaf_t* l, const double* xm, double* z) {
  for (int64_t i = l->rl; i < l->ru; ++i) {
    double acc = 0.0;
    for (int64_t j = l->cl; j < l->cu; ++j) acc += eval_ij(&h->kern, h->coords, h->n, i, j) * xm[j];
    z[i] += acc;
  }
}

/* low-rank apply (aca.cpp:597-619): t_l = fold(v_l . x), y_i = ((0 + u_0i t_0) + u_1i t_1) ..., z += y */
static void lowrank_apply(const leaf_t* l, int64_t kmax, int64_t keff, const double* u, const double* v,
                          const double* xm, double* z, double* y) {
  const int64_t m = l->ru - l->rl, n = l->cu - l->cl;
  (void)kmax;
  for (int64_t i = 0; i < m; ++i) y[i] = 0.0;
  const double* x = xm + l->cl;
  for (int64_t q = 0; q < keff; ++q) {
    const double* vl = v + q * n;
    double t = vl[0] * x[0];
    for (int64_t j = 1; j < n; ++j) t += vl[j] * x[j];
    const double* ul = u + q * m;
    for (int64_t i = 0; i < m; ++i) y[i] += ul[i] * t;
  }
  for (int64_t i = 0; i < m; ++i) z[l->rl + i] += y[i];
}

static int mvp_leaves(orc_hmatrix* h, const double* xm, double* z, const int64_t* ranges, int64_t nranges) {
  int64_t maxm = 1;
  for (int64_t b = 0; b < h->n_aca; ++b) {
    const int64_t m = h->aca[b].ru - h->aca[b].rl, n = h->aca[b].cu - h->aca[b].cl;
    if (m > maxm) maxm = m;
    if (n > maxm) maxm = n;
  }
  double* u = malloc(sizeof(double) * (size_t)(h->k * maxm));
  double* v = malloc(sizeof(double) * (size_t)(h->k * maxm));
  double* y = malloc(sizeof(double) * (size_t)maxm);
  int64_t* rp = malloc(sizeof(int64_t) * (size_t)h->k);
  int64_t* cp = malloc(sizeof(int64_t) * (size_t)h->k);
  if (!u || !v || !y || !rp || !cp) return fail("oom");
#define HIT(l)                                                                   \
  ({                                                                             \
    int hit_ = nranges < 0;                                                      \
    for (int64_t q_ = 0; q_ < nranges && !hit_; ++q_)                            \
      hit_ = (l)->rl < ranges[2 * q_ + 1] && ranges[2 * q_] < (l)->ru;           \
    hit_;                                                                        \
  })
  /* dense groups first, then ACA batches, each in leaf order (hmatrix.cpp:80-113) */
  for (int64_t b = 0; b < h->n_dense; ++b)
    if (HIT(&h->dense[b])) dense_leaf_apply(h, &h->dense[b], xm, z);
  for (int64_t b = 0; b < h->n_aca; ++b) {
    const leaf_t* l = &h->aca[b];
    if (!HIT(l)) continue;
    if (h->precompute) {
      lowrank_apply(l, h->k, h->pk[b], h->pu[b], h->pv[b], xm, z, y);
    } else {
      int64_t keff;
      if (aca_leaf(h, l, u, v, rp, cp, &keff, NULL)) return 1;
      lowrank_apply(l, h->k, keff, u, v, xm, z, y);
    }
  }
#undef HIT
  free(u);
  free(v);
  free(y);
  free(rp);
  free(cp);
  return 0;
}

/* hmatrix.cpp:66-123 */
int orc_mvp(orc_hmatrix* h, const double* x, double* out) {
  const int64_t n = h->n;
  double* xm = malloc(sizeof(double) * (size_t)n);
  double* z = calloc((size_t)n, sizeof(double));
  if (!xm || !z) return fail("oom");
  for (int64_t i = 0; i < n; ++i) xm[i] = x[h->perm[i]]; /* core.cpp:167-177 forward */
  if (mvp_leaves(h, xm, z, NULL, -1)) return 1;
  for (int64_t i = 0; i < n; ++i) out[h->perm[i]] = z[i]; /* inverse */
  free(xm);
  free(z);
  return 0;
}

int orc_mvp_rows(orc_hmatrix* h, const double* x, int64_t nranges, const int64_t* ranges, double* z_morton) {
  const int64_t n = h->n;
  double* xm = malloc(sizeof(double) * (size_t)n);
  if (!xm) return fail("oom");
  for (int64_t i = 0; i < n; ++i) xm[i] = x[h->perm[i]];
  memset(z_morton, 0, sizeof(double) * (size_t)n);
  const int rc = mvp_leaves(h, xm, z_morton, ranges, nranges);
  free(xm);
  return rc;
}

int orc_aca_all(orc_hmatrix* h, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v,
                int64_t* rejections) {
  int64_t uo = 0, vo = 0;
  int64_t maxm = 1;
  for (int64_t b = 0; b < h->n_aca; ++b) {
    const int64_t m = h->aca[b].ru - h->aca[b].rl, n = h->aca[b].cu - h->aca[b].cl;
    if (m > maxm) maxm = m;
    if (n > maxm) maxm = n;
  }
  double* su = u ? NULL : malloc(sizeof(double) * (size_t)(h->k * maxm));
  double* sv = v ? NULL : malloc(sizeof(double) * (size_t)(h->k * maxm));
  for (int64_t b = 0; b < h->n_aca; ++b) {
    const leaf_t* l = &h->aca[b];
    if (aca_leaf(h, l, u ? u + uo : su, v ? v + vo : sv, row_piv + b * h->k, col_piv + b * h->k, k_eff + b,
                 rejections ? rejections + b : NULL))
      return 1;
    uo += h->k * (l->ru - l->rl);
    vo += h->k * (l->cu - l->cl);
  }
  free(su);
  free(sv);
  return 0;
}

/* oracle.cpp:24-55 (single rhs): acc += a * x_gathered[j], written to original slot */
int orc_dense_mvp(orc_hmatrix* h, const double* x, double* out) {
  const int64_t n = h->n;
  double* xm = malloc(sizeof(double) * (size_t)n);
  if (!xm) return fail("oom");
  for (int64_t i = 0; i < n; ++i) xm[i] = x[h->perm[i]];
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += eval_ij(&h->kern, h->coords, n, i, j) * xm[j];
    out[h->perm[i]] = acc;
  }
  free(xm);
  return 0;
}

/* hmatrix.cpp:125-153 */
int orc_relative_error(orc_hmatrix* h, const double* x, double* out) {
  const int64_t n = h->n;
  if (n > 32768) return fail("relative_error: point count exceeds the dense product limit");
  double* zh = malloc(sizeof(double) * (size_t)n);
  double* ze = malloc(sizeof(double) * (size_t)n);
  if (!zh || !ze) return fail("oom");
  if (orc_mvp(h, x, zh) || orc_dense_mvp(h, x, ze)) return 1;
  double diff_sq = 0.0, ref_sq = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = zh[i] - ze[i];
    diff_sq += d * d;
    ref_sq += ze[i] * ze[i];
  }
  *out = sqrt(diff_sq) / sqrt(ref_sq);
  free(zh);
  free(ze);
  return 0;
}

/* solver.cpp:11-17 */
static double dot(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* solver.cpp:19-73 */
int orc_cg(orc_hmatrix* h, const double* b, double sigma2, double tol, int64_t max_iter, double* x,
           int64_t* iterations, double* rel_res) {
  const int64_t n = h->n;
  if (tol <= 0.0 || max_iter < 1 || sigma2 < 0.0) return fail("cg_solve: invalid configuration");
  double* r = malloc(sizeof(double) * (size_t)n);
  double* p = malloc(sizeof(double) * (size_t)n);
  double* ap = malloc(sizeof(double) * (size_t)n);
  if (!r || !p || !ap) return fail("oom");
  memset(x, 0, sizeof(double) * (size_t)n);
  *iterations = 0;
  *rel_res = 0.0;
  const double b_norm = sqrt(dot(b, b, n));
  if (b_norm == 0.0) return 0;
  memcpy(r, b, sizeof(double) * (size_t)n);
  memcpy(p, r, sizeof(double) * (size_t)n);
  double rs = dot(r, r, n);
  for (int64_t iter = 1; iter <= max_iter; ++iter) {
    if (orc_mvp(h, p, ap)) return 1;
    for (int64_t i = 0; i < n; ++i) ap[i] += sigma2 * p[i];
    const double alpha = rs / dot(p, ap, n);
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    const double rs_next = dot(r, r, n);
    if (!isfinite(rs_next) || !isfinite(alpha)) return fail("cg_solve: non-finite value");
    *iterations = iter;
    if (sqrt(rs_next) <= tol * b_norm) break;
    const double beta = rs_next / rs;
    for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    rs = rs_next;
  }
  if (orc_mvp(h, x, ap)) return 1;
  double diff_sq = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    ap[i] += sigma2 * x[i];
    const double d = b[i] - ap[i];
    diff_sq += d * d;
  }
  *rel_res = sqrt(diff_sq) / b_norm;
  free(r);
  free(p);
  free(ap);
  return 0;
}

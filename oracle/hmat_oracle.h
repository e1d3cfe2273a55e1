/* hmat_oracle.h -- C restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * A sequential, plain-C re-statement of the reference library's
 * setup() + mvp() path (reference: /root/reference/proj, C++20).  It exists only
 * to CHECK the B200 product (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline leg).  It is pinned against the unmodified reference built by
 * oracle/Makefile into oracle/_ref/ and against the golden fixtures in
 * tests/golden/ (see tests/test_oracle_pinning.py).
 *
 * Every function cites the reference file:line it restates.  Conventions match
 * the reference: coordinates are structure-of-arrays (coords[a*n + i]), leaf
 * lists are canonical-ordered (tree.cpp:189-194), factors are rank-major per
 * block (aca.hpp:14-21), vectors passed to orc_mvp are in ORIGINAL order.
 */
#ifndef HMAT_ORACLE_H
#define HMAT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_hmatrix orc_hmatrix;

const char* orc_last_error(void);

/* core.cpp:97-102 / :28-81 */
int orc_bessel_k1(int64_t n, const double* x, double* out);
/* core.hpp:67-92 via eval_kernel core.cpp:141-151; y, yp are SoA d x n pairs */
int orc_eval_kernel(int kind, double beta, int d, int64_t n, const double* y, const double* yp, double* out);
/* morton.cpp:37-48 */
int orc_morton_codes(int64_t n, int d, const double* coords, uint64_t* codes);
/* morton.cpp:50-71 (stable sort + gather + perm composition) */
int orc_morton_order(int64_t n, int d, const double* coords, const int64_t* perm_in, double* coords_out,
                     int64_t* perm_out);
/* tree.cpp:11-32 on explicit boxes (box = a[d] then b[d]) */
int orc_admissible(int d, const double* box_t, const double* box_s, double eta, double* diam_t, double* diam_s,
                   double* dist);

/* hmatrix.cpp:38-64.  mode: 0 geometric, 1 force dense, 2 force admissible. */
orc_hmatrix* orc_setup(int64_t n, int d, const double* coords, int kind, double beta, double eta, int64_t c_leaf,
                       int64_t k, int precompute, int has_eps, double eps, int mode);
void orc_free(orc_hmatrix* h);
/* which: 0 dense queue, 1 aca queue (hmatrix.cpp:51-53) */
int64_t orc_count(const orc_hmatrix* h, int which);
int orc_leaves(const orc_hmatrix* h, int which, int64_t* rows4, double* boxes4d);
int orc_points(const orc_hmatrix* h, double* coords, int64_t* perm);
/* hmatrix.cpp:66-123 (x, z original ordering) */
int orc_mvp(orc_hmatrix* h, const double* x, double* z);
/* Row-sampled product: only leaves whose row range meets one of the [lo,hi)
 * ranges; z_morton valid on those rows. */
int orc_mvp_rows(orc_hmatrix* h, const double* x, int64_t nranges, const int64_t* ranges, double* z_morton);
/* batched-ACA factors of every admissible block (aca.cpp:268-544 semantics).
 * u/v: kmax*m / kmax*n per block, rank-major, zero padded past k_eff.
 * rejections (optional): per-block rejected candidate columns. */
int orc_aca_all(orc_hmatrix* h, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v,
                int64_t* rejections);
/* explicit-matrix seam (aca.cpp:567-578): blocks row-major, shapes (m,n) pairs */
int orc_aca_dense(int64_t nblocks, const int64_t* shapes, const double* entries, int64_t kmax, int has_eps,
                  double eps, double eta, int64_t* k_eff, int64_t* row_piv, int64_t* col_piv, double* u, double* v);
/* hmatrix.cpp:125-153 */
int orc_relative_error(orc_hmatrix* h, const double* x, double* out);
/* solver.cpp:19-73 */
int orc_cg(orc_hmatrix* h, const double* b, double sigma2, double tol, int64_t max_iter, double* x,
           int64_t* iterations, double* rel_res);
/* exact dense product (oracle.cpp:24-55), original ordering */
int orc_dense_mvp(orc_hmatrix* h, const double* x, double* z);

#ifdef __cplusplus
}
#endif
#endif

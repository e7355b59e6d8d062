/* kmf_build.h -- C ABI of the native stencil builder (libkmf_build.so).
 *
 * Host-side setup, not the per-iteration hot path: the bit-exact heavy
 * loops of the reference builder build_stencils (reference
 * pkg/src/kmf/geometry.py:453-518) so the 10M / 40M-point configurations
 * can be generated.  Bound through ctypes by paper_2108_07031_b200/builder.py.
 * All arrays are caller-owned; status 0 ok, 2 invalid argument.
 */
#ifndef KMF_BUILD_H
#define KMF_BUILD_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* OpenMP threads the builder uses. */
int kmfb_threads(void);
/* set them (n <= 0: every processor); returns the new count */
int kmfb_set_threads(int n);

/* Replaces geometry.py:315-346 _knn_neighbors: tie-inclusive k nearest
 * neighbours of points query[0..nq) (all points when query == NULL), self
 * excluded, ascending index.  Call once with rows == NULL to get counts,
 * then with ptr = exclusive prefix sum of counts to fill rows. */
int kmfb_knn(int64_t n, const double *x, const double *y, int k, int64_t nq, const int64_t *query,
             int64_t *counts, const int64_t *ptr, int64_t *rows);

/* Replaces geometry.py:349-374 _radius_neighbors: every j != i with
 * (x_j - x_i)^2 + (y_j - y_i)^2 < eps^2, ascending index.  Call once with
 * rows == NULL to get counts[n], then with ptr = prefix sum to fill rows. */
int kmfb_radius(int64_t n, const double *x, const double *y, double eps, int64_t *counts, const int64_t *ptr,
                int64_t *rows);

/* Replaces the edge loop of geometry.py:396-450 _visibility_filter given
 * the wall statistics (spacing, tol) computed as the reference does.
 * keep[e] = 1 for surviving edges of rows owned by owners[r] (r when NULL);
 * *ambiguous counts nearest-wall ties with disagreeing outcomes. */
int kmfb_visibility(int64_t n, const double *x, const double *y, int64_t nw, const int64_t *wall,
                    const double *wnx, const double *wny, const double *spacing, const double *tol, int64_t nrows,
                    const int64_t *owners, const int64_t *ptr, const int64_t *idx, uint8_t *keep,
                    int64_t *ambiguous);

/* Replaces geometry.py:375-393 / 532-560 (_csr_from_lists offsets,
 * StencilSet sums geometry.py:244-252, d_min / d_mean, sign-split family
 * sums).  sums[4][n] = full sxx, sxy, syy, det; ssum[4][4][n] per family
 * x+, x-, y+, y-; scnt[4][n] family counts. */
int kmfb_assemble(int64_t n, const double *x, const double *y, const int64_t *ptr, const int64_t *idx, double *dx,
                  double *dy, double *sums, double *d_min, double *d_mean, double *ssum, int64_t *scnt);

#ifdef __cplusplus
}
#endif
#endif

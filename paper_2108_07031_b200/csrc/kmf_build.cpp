// kmf_build.cpp -- native stencil builder, host C++/OpenMP.
//
// Bit-exact restatement of the heavy parts of the reference builder
// (geometry.py:315-346 _knn_neighbors, :396-450 _visibility_filter,
// :532-570 _assemble) so the 10M / 40M-point configurations can be built
// at all (the scipy builder needs ~30 min / 32 GB at 10M and ~128 GB at
// 40M).  The orchestration (wall statistics that depend on cKDTree's
// tie order, boundary frames, deficiency scan, widening) stays in Python
// (paper_2108_07031_b200/builder.py) and is shared with the scipy path.
//
// Exactness argument (tests/test_builder.py checks it bit for bit):
//  * cKDTree's distance is sqrt(dx*dx + dy*dy) with both products rounded
//    (verified against scipy here).  The reference keeps every point whose
//    distance is <= the k_eff-th smallest distance (self counted), with the
//    plateau widening, which is exactly the set {j != i : d_ij <= D_k}.
//    kNN here finds D_k^2 exactly in squared space, then collects all j
//    with sqrt(d2_ij) <= sqrt(D_k^2) (sqrt is correctly rounded in both).
//  * visibility: per sample point the nearest wall point is taken at the
//    minimal squared distance, like cKDTree's k=1 query; ties in d^2 are
//    all evaluated; when they disagree the edge is marked undecided (2) and
//    the caller settles it with cKDTree itself, whose first-found tie order
//    is the reference's (a handful of edges per cloud).
//    Edges whose owner is farther from the wall than edge length + twice
//    the largest wall spacing provably pass (triangle inequality) and skip
//    the query.
//  * sums are sequential in CSR order with products rounded first
//    (np.bincount, geometry.py:249-251), built with -ffp-contract=off;
//    d_min / d_mean use libm hypot like np.hypot.
#include "../../include/kmf_build.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// --------------------------------------------------------------- 2-d tree
// Implicit balanced tree over a permutation: node v covers perm[lo, hi),
// split at mid = (lo + hi) / 2 on the wider axis; leaves hold <= kLeaf.
constexpr int kLeaf = 8;

struct Tree {
    const double *x = nullptr, *y = nullptr;
    std::vector<int32_t> perm;
    std::vector<double> split;   // per node
    std::vector<uint8_t> dim;    // per node, 2 = leaf
    int64_t n = 0;

    static int64_t node_count(int64_t n)
    {
        int64_t c = 1;
        while (c * kLeaf < n) c <<= 1;
        return 4 * c + 4;
    }

    void build_rec(int64_t v, int64_t lo, int64_t hi, int depth)
    {
        if (hi - lo <= kLeaf) {
            dim[v] = 2;
            return;
        }
        double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
        for (int64_t k = lo; k < hi; k++) {
            const int32_t p = perm[k];
            xmin = std::min(xmin, x[p]);
            xmax = std::max(xmax, x[p]);
            ymin = std::min(ymin, y[p]);
            ymax = std::max(ymax, y[p]);
        }
        const int d = (xmax - xmin) >= (ymax - ymin) ? 0 : 1;
        const double *c = d == 0 ? x : y;
        const int64_t mid = (lo + hi) / 2;
        std::nth_element(perm.begin() + lo, perm.begin() + mid, perm.begin() + hi,
                         [c](int32_t a, int32_t b) { return c[a] < c[b]; });
        dim[v] = (uint8_t)d;
        split[v] = c[perm[mid]];
        if (depth < 12 && hi - lo > 200000) {
#pragma omp task
            build_rec(2 * v, lo, mid, depth + 1);
#pragma omp task
            build_rec(2 * v + 1, mid, hi, depth + 1);
#pragma omp taskwait
        } else {
            build_rec(2 * v, lo, mid, depth + 1);
            build_rec(2 * v + 1, mid, hi, depth + 1);
        }
    }

    void build(const double *xs, const double *ys, const int32_t *ids, int64_t count)
    {
        x = xs;
        y = ys;
        n = count;
        perm.assign(ids, ids + count);
        const int64_t nn = node_count(count);
        split.assign(nn, 0.0);
        dim.assign(nn, 2);
        if (count == 0) return;
#pragma omp parallel
#pragma omp single
        build_rec(1, 0, count, 0);
    }

    static inline double d2(double qx, double qy, double px, double py)
    {
        const double dx = px - qx, dy = py - qy;
        return dx * dx + dy * dy;
    }

    struct Frame {
        int64_t v, lo, hi;
    };

    // the k smallest (d2, index) pairs, unordered, in h (max-heap on d2)
    int knn_pairs(double qx, double qy, int k, std::pair<double, int32_t> *h) const
    {
        int hn = 0;
        Frame st[128];
        int sp = 0;
        st[sp++] = {1, 0, n};
        while (sp) {
            const Frame f = st[--sp];
            if (dim[f.v] == 2) {
                for (int64_t t = f.lo; t < f.hi; t++) {
                    const int32_t p = perm[t];
                    const double v = d2(qx, qy, x[p], y[p]);
                    if (hn < k) {
                        h[hn++] = {v, p};
                        std::push_heap(h, h + hn);
                    } else if (v < h[0].first) {
                        std::pop_heap(h, h + hn);
                        h[hn - 1] = {v, p};
                        std::push_heap(h, h + hn);
                    }
                }
                continue;
            }
            const int64_t mid = (f.lo + f.hi) / 2;
            const double q = dim[f.v] == 0 ? qx : qy;
            const double diff = q - split[f.v];
            const Frame nearf = diff <= 0.0 ? Frame{2 * f.v, f.lo, mid} : Frame{2 * f.v + 1, mid, f.hi};
            const Frame farf = diff <= 0.0 ? Frame{2 * f.v + 1, mid, f.hi} : Frame{2 * f.v, f.lo, mid};
            if (hn < k || diff * diff <= h[0].first) st[sp++] = farf;
            st[sp++] = nearf;
        }
        return hn;
    }

    // all points with squared distance <= r2, appended to out
    template <class F>
    void range(double qx, double qy, double r2, F &&visit) const
    {
        Frame st[128];
        int sp = 0;
        st[sp++] = {1, 0, n};
        while (sp) {
            const Frame f = st[--sp];
            if (dim[f.v] == 2) {
                for (int64_t t = f.lo; t < f.hi; t++) {
                    const int32_t p = perm[t];
                    const double v = d2(qx, qy, x[p], y[p]);
                    if (v <= r2) visit(p, v);
                }
                continue;
            }
            const int64_t mid = (f.lo + f.hi) / 2;
            const double q = dim[f.v] == 0 ? qx : qy;
            const double diff = q - split[f.v];
            const bool left_near = diff <= 0.0;
            if (diff * diff <= r2) st[sp++] = left_near ? Frame{2 * f.v + 1, mid, f.hi} : Frame{2 * f.v, f.lo, mid};
            st[sp++] = left_near ? Frame{2 * f.v, f.lo, mid} : Frame{2 * f.v + 1, mid, f.hi};
        }
    }

    // minimal squared distance and every point attaining it
    double nearest(double qx, double qy, std::vector<int32_t> &ties) const
    {
        double best = INFINITY;
        ties.clear();
        Frame st[128];
        int sp = 0;
        st[sp++] = {1, 0, n};
        while (sp) {
            const Frame f = st[--sp];
            if (dim[f.v] == 2) {
                for (int64_t t = f.lo; t < f.hi; t++) {
                    const int32_t p = perm[t];
                    const double v = d2(qx, qy, x[p], y[p]);
                    if (v < best) {
                        best = v;
                        ties.clear();
                        ties.push_back(p);
                    } else if (v == best) {
                        ties.push_back(p);
                    }
                }
                continue;
            }
            const int64_t mid = (f.lo + f.hi) / 2;
            const double q = dim[f.v] == 0 ? qx : qy;
            const double diff = q - split[f.v];
            const bool left_near = diff <= 0.0;
            if (diff * diff <= best) st[sp++] = left_near ? Frame{2 * f.v + 1, mid, f.hi} : Frame{2 * f.v, f.lo, mid};
            st[sp++] = left_near ? Frame{2 * f.v, f.lo, mid} : Frame{2 * f.v + 1, mid, f.hi};
        }
        return best;
    }
};

// tree over all points or a subset, built on demand per call
struct Built {
    Tree t;
    Built(const double *x, const double *y, const int32_t *ids, int64_t n) { t.build(x, y, ids, n); }
};

std::vector<int32_t> iota32(int64_t n)
{
    std::vector<int32_t> v(n);
    for (int64_t i = 0; i < n; i++) v[i] = (int32_t)i;
    return v;
}

}  // namespace

extern "C" {

int kmfb_threads(void) { return omp_get_max_threads(); }

// set the OpenMP threads of the builder (n <= 0: every processor); returns
// the new count.  torchrun sets OMP_NUM_THREADS=1 per rank, which would
// leave the one rank that builds a shared connectivity on a single core.
int kmfb_set_threads(int n)
{
    omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
    return omp_get_max_threads();
}

// geometry.py:315-346 tie-inclusive kNN rows (self excluded, ascending).
// Pass 1 (rows == NULL): counts[r] for each query row.  Pass 2: rows
// filled at offsets ptr[r] (caller's prefix sum of counts).
// Rows of the last counting pass, kept for the filling pass of the same
// query (the two-call protocol would otherwise search everything twice).
struct KnnCache {
    const double *x = nullptr, *y = nullptr;
    const int64_t *query = nullptr;
    int64_t n = 0, nq = 0;
    int k = 0;
    std::vector<int64_t> off;
    std::vector<int32_t> rows;
};
static KnnCache g_knn;

int kmfb_knn(int64_t n, const double *x, const double *y, int k, int64_t nq, const int64_t *query,
             int64_t *counts, const int64_t *ptr, int64_t *rows)
{
    if (n <= 0 || k < 1 || nq < 0) return 2;
    if (rows && g_knn.x == x && g_knn.y == y && g_knn.query == query && g_knn.n == n && g_knn.nq == nq &&
        g_knn.k == k) {
#pragma omp parallel for schedule(static, 4096)
        for (int64_t r = 0; r < nq; r++) {
            int64_t o = ptr[r];
            for (int64_t e = g_knn.off[r]; e < g_knn.off[r + 1]; e++) rows[o++] = g_knn.rows[e];
        }
        g_knn = KnnCache();
        return 0;
    }
    g_knn = KnnCache();
    std::vector<int32_t> all = iota32(n);
    Tree t;
    t.build(x, y, all.data(), n);
    const int k_eff = (int)std::min<int64_t>(k + 1, n);
    int bad = 0;
    // one traversal with a padded heap (k_eff + 8 nearest, like the
    // reference's pad, geometry.py:329): D_k is the k_eff-th smallest; if
    // the pad's farthest entry is provably beyond D_k the heap holds every
    // point with d <= D_k, else (a distance plateau) a range query collects
    // them.  sqrt(v) <= D can hold for v slightly above D^2, hence the
    // (1 + 1e-15) widening before the exact filter.
    const int kpad = (int)std::min<int64_t>(k_eff + 8, n);
    const int nt = omp_get_max_threads();
    std::vector<std::vector<int32_t>> tbuf(nt);                   // per-thread row storage
    std::vector<std::vector<std::pair<int64_t, int64_t>>> tloc(nt);  // (query row, start in tbuf)
    std::vector<int64_t> cnt(nq, 0);
#pragma omp parallel
    {
        const int tid = omp_get_thread_num();
        std::vector<std::pair<double, int32_t>> heap(kpad + 1);
        std::vector<int32_t> got;
        got.reserve(64);
#pragma omp for schedule(dynamic, 1024)
        for (int64_t r = 0; r < nq; r++) {
            const int64_t i = query ? query[r] : r;
            if (i < 0 || i >= n) {
#pragma omp atomic write
                bad = 1;
                continue;
            }
            const double qx = x[i], qy = y[i];
            const int hn = t.knn_pairs(qx, qy, kpad, heap.data());
            std::sort(heap.begin(), heap.begin() + hn);
            const double D2 = heap[k_eff - 1].first;
            const double D = std::sqrt(D2);
            got.clear();
            if (hn < n && heap[hn - 1].first > D2 * (1.0 + 1e-15)) {
                for (int h = 0; h < hn; h++)
                    if (heap[h].second != i && std::sqrt(heap[h].first) <= D) got.push_back(heap[h].second);
            } else {
                t.range(qx, qy, D2 * (1.0 + 1e-15), [&](int32_t p, double v) {
                    if (p != i && std::sqrt(v) <= D) got.push_back(p);
                });
            }
            std::sort(got.begin(), got.end());
            cnt[r] = (int64_t)got.size();
            tloc[tid].push_back({r, (int64_t)tbuf[tid].size()});
            tbuf[tid].insert(tbuf[tid].end(), got.begin(), got.end());
        }
    }
    if (bad) return 2;
    std::vector<int64_t> off(nq + 1, 0);
    for (int64_t r = 0; r < nq; r++) off[r + 1] = off[r] + cnt[r];
    if (!rows) {
        // counting pass: report the counts, keep the rows for the fill pass
        std::memcpy(counts, cnt.data(), sizeof(int64_t) * nq);
        g_knn.rows.resize(off[nq]);
        for (int th = 0; th < nt; th++)
            for (const auto &pl : tloc[th])
                std::memcpy(g_knn.rows.data() + off[pl.first], tbuf[th].data() + pl.second,
                            sizeof(int32_t) * cnt[pl.first]);
        g_knn.off = std::move(off);
        g_knn.x = x;
        g_knn.y = y;
        g_knn.query = query;
        g_knn.n = n;
        g_knn.nq = nq;
        g_knn.k = k;
        return 0;
    }
    for (int th = 0; th < nt; th++)
        for (const auto &pl : tloc[th]) {
            int64_t o = ptr[pl.first];
            for (int64_t e = 0; e < cnt[pl.first]; e++) rows[o++] = tbuf[th][pl.second + e];
        }
    return 0;
}

// geometry.py:349-374 radius rows: every j != i with squared distance
// (x_j - x_i)^2 + (y_j - y_i)^2 < eps^2 (both squares and the sum rounded,
// like the reference's numpy filter; the ball query it filters is a
// superset), ascending.  Pass 1 (rows == NULL): counts; pass 2: rows at
// offsets ptr[r].
int kmfb_radius(int64_t n, const double *x, const double *y, double eps, int64_t *counts, const int64_t *ptr,
                int64_t *rows)
{
    if (n <= 0 || !(eps > 0.0)) return 2;
    std::vector<int32_t> all = iota32(n);
    Tree t;
    t.build(x, y, all.data(), n);
    const double eps2 = eps * eps;
#pragma omp parallel
    {
        std::vector<int32_t> got;
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; i++) {
            got.clear();
            t.range(x[i], y[i], eps2 * (1.0 + 1e-12), [&](int32_t p, double v) {
                if (p != i && v < eps2) got.push_back(p);
            });
            if (!rows) {
                counts[i] = (int64_t)got.size();
                continue;
            }
            std::sort(got.begin(), got.end());
            int64_t o = ptr[i];
            for (int32_t p : got) rows[o++] = p;
        }
    }
    return 0;
}

// geometry.py:396-450 visibility filter.  Wall statistics (spacing, tol)
// come from the caller (their cKDTree tie order is part of the contract).
// keep[e] = 1 when edge e (owner owners[r] for r's rows) survives.
// keep[e] = 2 marks an edge with a nearest-wall tie of disagreeing
// outcomes (counted in *ambiguous) for the caller to settle.
int kmfb_visibility(int64_t n, const double *x, const double *y, int64_t nw, const int64_t *wall,
                    const double *wnx, const double *wny, const double *spacing, const double *tol, int64_t nrows,
                    const int64_t *owners, const int64_t *ptr, const int64_t *idx, uint8_t *keep,
                    int64_t *ambiguous)
{
    if (nw < 2) {
        std::memset(keep, 1, (size_t)ptr[nrows]);
        if (ambiguous) *ambiguous = 0;
        return 0;
    }
    std::vector<double> wx(nw), wy(nw);
    double maxsp = 0.0, bx0 = INFINITY, bx1 = -INFINITY, by0 = INFINITY, by1 = -INFINITY;
    for (int64_t a = 0; a < nw; a++) {
        wx[a] = x[wall[a]];
        wy[a] = y[wall[a]];
        maxsp = std::max(maxsp, spacing[a]);
        bx0 = std::min(bx0, wx[a]);
        bx1 = std::max(bx1, wx[a]);
        by0 = std::min(by0, wy[a]);
        by1 = std::max(by1, wy[a]);
    }
    const double margin = 2.0 * maxsp * (1.0 + 1e-12);
    std::vector<int32_t> ids = iota32(nw);
    Tree t;
    t.build(wx.data(), wy.data(), ids.data(), nw);
    int64_t amb = 0;
    const double fr[3] = {0.25, 0.5, 0.75};
#pragma omp parallel reduction(+ : amb)
    {
        std::vector<int32_t> ties;
#pragma omp for schedule(dynamic, 256)
        for (int64_t r = 0; r < nrows; r++) {
            const int64_t o = owners ? owners[r] : r;
            const double x0 = x[o], y0 = y[o];
            // cheap lower bound first: distance to the wall points' bounding
            // box; owners far from the body keep every edge without a query
            double lmax = 0.0;
            for (int64_t e = ptr[r]; e < ptr[r + 1]; e++) {
                const double ex = x[idx[e]] - x0, ey = y[idx[e]] - y0;
                lmax = std::max(lmax, std::sqrt(ex * ex + ey * ey));
            }
            const double gx = std::max(0.0, std::max(bx0 - x0, x0 - bx1));
            const double gy = std::max(0.0, std::max(by0 - y0, y0 - by1));
            const double dbox = std::sqrt(gx * gx + gy * gy);
            if (dbox * (1.0 - 1e-12) - lmax * (1.0 + 1e-12) > margin) {
                for (int64_t e = ptr[r]; e < ptr[r + 1]; e++) keep[e] = 1;
                continue;
            }
            const double D0 = std::sqrt(t.nearest(x0, y0, ties));
            for (int64_t e = ptr[r]; e < ptr[r + 1]; e++) {
                const int64_t j = idx[e];
                const double ddx = x[j] - x0, ddy = y[j] - y0;
                const double len = std::sqrt(ddx * ddx + ddy * ddy);
                // every sample lies within len of the owner: its distance to
                // any wall point exceeds 2*spacing[near] for sure
                if (D0 * (1.0 - 1e-12) - len * (1.0 + 1e-12) > margin) {
                    keep[e] = 1;
                    continue;
                }
                uint8_t out = 1;
                for (int s = 0; s < 3 && out == 1; s++) {
                    const double sx = x0 + fr[s] * ddx;
                    const double sy = y0 + fr[s] * ddy;
                    const double dist = std::sqrt(t.nearest(sx, sy, ties));
                    int verdict = -1;
                    for (int32_t a : ties) {
                        const double depth = (sx - wx[a]) * wnx[a] + (sy - wy[a]) * wny[a];
                        const int v = (dist > 2.0 * spacing[a]) || (depth > -tol[a]);
                        if (verdict < 0) verdict = v;
                        else if (verdict != v) verdict = 2;
                    }
                    if (verdict == 2) {
                        out = 2;  // decided by the caller with the reference's tie order
                        amb++;
                    } else if (verdict == 0) {
                        out = 0;
                    }
                }
                keep[e] = out;
            }
        }
    }
    if (ambiguous) *ambiguous = amb;
    return 0;
}

// geometry.py:532-560 assembly of one CSR: offsets, full sums, d_min /
// d_mean, and the four sign-split families' counts and sums
// (x+: dx <= 0, x-: dx >= 0, y+: dy <= 0, y-: dy >= 0, geometry.py:544-549).
// sums: [4][n] sxx, sxy, syy, det of the full stencil; ssum: [4 fam][4][n];
// scnt: [4][n].
int kmfb_assemble(int64_t n, const double *x, const double *y, const int64_t *ptr, const int64_t *idx, double *dx,
                  double *dy, double *sums, double *d_min, double *d_mean, double *ssum, int64_t *scnt)
{
#pragma omp parallel for schedule(static, 4096)
    for (int64_t i = 0; i < n; i++) {
        double sxx = 0.0, sxy = 0.0, syy = 0.0, dm = INFINITY, ds = 0.0;
        double fxx[4] = {0, 0, 0, 0}, fxy[4] = {0, 0, 0, 0}, fyy[4] = {0, 0, 0, 0};
        int64_t fc[4] = {0, 0, 0, 0};
        for (int64_t e = ptr[i]; e < ptr[i + 1]; e++) {
            const int64_t j = idx[e];
            const double ex = x[j] - x[i], ey = y[j] - y[i];
            dx[e] = ex;
            dy[e] = ey;
            const double pxx = ex * ex, pxy = ex * ey, pyy = ey * ey;
            sxx += pxx;
            sxy += pxy;
            syy += pyy;
            const double len = std::hypot(ex, ey);
            dm = std::min(dm, len);  // np.minimum.at keeps the first of equal values; equal anyway
            ds += len;
            const bool in[4] = {ex <= 0.0, ex >= 0.0, ey <= 0.0, ey >= 0.0};
            for (int f = 0; f < 4; f++) {
                if (in[f]) {
                    fxx[f] += pxx;
                    fxy[f] += pxy;
                    fyy[f] += pyy;
                    fc[f]++;
                }
            }
        }
        sums[i] = sxx;
        sums[n + i] = sxy;
        sums[2 * n + i] = syy;
        sums[3 * n + i] = sxx * syy - sxy * sxy;
        d_min[i] = dm;
        const int64_t cnt = ptr[i + 1] - ptr[i];
        d_mean[i] = ds / (double)(cnt > 1 ? cnt : 1);
        for (int f = 0; f < 4; f++) {
            double *o = ssum + (int64_t)f * 4 * n;
            o[i] = fxx[f];
            o[n + i] = fxy[f];
            o[2 * n + i] = fyy[f];
            o[3 * n + i] = fxx[f] * fyy[f] - fxy[f] * fxy[f];
            scnt[(int64_t)f * n + i] = fc[f];
        }
    }
    return 0;
}

}  // extern "C"

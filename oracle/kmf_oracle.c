/*
 * kmf_oracle.c -- CPU restatement of the reference q-LSKUM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see kmf_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off -fopenmp).  Each function cites the reference
 * file:line it restates; the parenthesisation in every expression mirrors
 * numpy's left-to-right evaluation of the reference source.
 */
#include "kmf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BLOCK 4096 /* solver.py:64 */
#define PI 3.141592653589793

void orc_set_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

int orc_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static void set_err(orc_error *err, int ctx, int64_t count, int64_t first)
{
    if (!err) return;
    err->code = 1;
    err->context = ctx;
    err->count = count;
    err->first = first;
}

/* ---------------------------------------------------------------- state */

/* state.py:132-138 primitives_to_q (validate :80-88) */
int orc_primitives_to_q(int64_t n, const double *pr, double gamma, double *q, orc_error *err)
{
    int64_t bad = 0, first = -1;
    for (int64_t i = 0; i < n; i++) {
        if (!((pr[i] > 0.0) && (pr[3 * n + i] > 0.0))) {
            if (first < 0) first = i;
            bad++;
        }
    }
    if (bad) {
        set_err(err, ORC_CTX_P2Q, bad, first);
        return 1;
    }
    const double gm1 = gamma - 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
        double beta = rho / (2.0 * p);
        double uu = (u1 * u1) + (u2 * u2);
        q[i] = (log(rho) + (log(beta) / gm1)) - (beta * uu);
        q[n + i] = (2.0 * beta) * u1;
        q[2 * n + i] = (2.0 * beta) * u2;
        q[3 * n + i] = -2.0 * beta;
    }
    return 0;
}

/* state.py:141-163 q_to_primitives, one state */
static inline void q2p(double q1, double q2, double q3, double q4, double gamma, double *rho,
                       double *u1, double *u2, double *p)
{
    double beta = -0.5 * q4;
    double a = q2 / (2.0 * beta);
    double b = q3 / (2.0 * beta);
    double r = exp((q1 - (log(beta) / (gamma - 1.0))) + (beta * ((a * a) + (b * b))));
    *rho = r;
    *u1 = a;
    *u2 = b;
    *p = r / (2.0 * beta);
}

int orc_q_to_primitives(int64_t n, const double *q, double gamma, double *pr, orc_error *err)
{
    int64_t bad = 0, first = -1;
    for (int64_t i = 0; i < n; i++)
        if (!(q[3 * n + i] < 0.0)) {
            if (first < 0) first = i;
            bad++;
        }
    if (bad) {
        set_err(err, ORC_CTX_Q2P, bad, first);
        return 1;
    }
    for (int64_t i = 0; i < n; i++)
        q2p(q[i], q[n + i], q[2 * n + i], q[3 * n + i], gamma, &pr[i], &pr[n + i], &pr[2 * n + i],
            &pr[3 * n + i]);
    return 0;
}

/* state.py:91-96 primitives_to_conserved */
int orc_primitives_to_conserved(int64_t n, const double *pr, double gamma, double *U, orc_error *err)
{
    int64_t bad = 0, first = -1;
    for (int64_t i = 0; i < n; i++)
        if (!((pr[i] > 0.0) && (pr[3 * n + i] > 0.0))) {
            if (first < 0) first = i;
            bad++;
        }
    if (bad) {
        set_err(err, ORC_CTX_INITIAL, bad, first);
        return 1;
    }
    for (int64_t i = 0; i < n; i++) {
        double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
        double e = (p / (rho * (gamma - 1.0))) + (0.5 * ((u1 * u1) + (u2 * u2)));
        U[i] = rho;
        U[n + i] = rho * u1;
        U[2 * n + i] = rho * u2;
        U[3 * n + i] = rho * e;
    }
    return 0;
}

/* state.py:99-129 conserved_to_primitives */
int orc_conserved_to_primitives(int64_t n, const double *U, double gamma, double *pr, orc_error *err)
{
    int64_t bad = 0, first = -1;
    for (int64_t i = 0; i < n; i++)
        if (!(U[i] > 0.0)) {
            if (first < 0) first = i;
            bad++;
        }
    if (bad) {
        set_err(err, ORC_CTX_C2P_DENSITY, bad, first);
        return 1;
    }
    for (int64_t i = 0; i < n; i++) {
        double rho = U[i];
        double u1 = U[n + i] / rho, u2 = U[2 * n + i] / rho;
        double p = (gamma - 1.0) * (U[3 * n + i] - ((0.5 * rho) * ((u1 * u1) + (u2 * u2))));
        if (!(p > 0.0)) {
            if (first < 0) first = i;
            bad++;
        }
        pr[i] = rho;
        pr[n + i] = u1;
        pr[2 * n + i] = u2;
        pr[3 * n + i] = p;
    }
    if (bad) {
        set_err(err, ORC_CTX_C2P_PRESSURE, bad, first);
        return 1;
    }
    return 0;
}

/* -------------------------------------------------------------- kinetics */

/* kinetics.py:71-106 split_flux for one state; axis 0 = x, 1 = y; sg = +-1 */
static inline void sflux(double rho, double u1, double u2, double p, int axis, double sg,
                         double gamma, double G[4])
{
    double beta = rho / (2.0 * p);
    double un = axis == 0 ? u1 : u2;
    double ut = axis == 0 ? u2 : u1;
    double s = un * sqrt(beta);
    double A = 0.5 * (1.0 + (sg * erf(s)));
    double B = exp((-s) * s) / (2.0 * sqrt(PI * beta));
    double inv2b = 1.0 / (2.0 * beta);
    double m1 = (un * A) + (sg * B);
    double m2 = (((un * un) + inv2b) * A) + ((sg * un) * B);
    double m3 = ((((un * un) * un) + ((3.0 * un) * inv2b)) * A) +
                ((sg * ((un * un) + (2.0 * inv2b))) * B);
    double i0 = (2.0 - gamma) / ((2.0 * beta) * (gamma - 1.0)); /* kinetics.py:53-56 */
    double energy = rho * ((((i0 + ((0.5 * ut) * ut)) + (0.5 * inv2b)) * m1) + (0.5 * m3));
    G[0] = rho * m1;
    if (axis == 0) {
        G[1] = rho * m2;
        G[2] = (rho * m1) * ut;
    } else {
        G[1] = (rho * ut) * m1;
        G[2] = rho * m2;
    }
    G[3] = energy;
}

void orc_split_flux(int64_t n, const double *pr, int axis, int sign, double gamma, double *G)
{
    double sg = sign >= 0 ? 1.0 : -1.0;
    for (int64_t i = 0; i < n; i++) {
        double g[4];
        sflux(pr[i], pr[n + i], pr[2 * n + i], pr[3 * n + i], axis, sg, gamma, g);
        for (int c = 0; c < 4; c++) G[c * n + i] = g[c];
    }
}

/* kinetics.py:59-68 full_flux */
void orc_full_flux(int64_t n, const double *pr, int axis, double gamma, double *F)
{
    for (int64_t i = 0; i < n; i++) {
        double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
        double e = (p / (rho * (gamma - 1.0))) + (0.5 * ((u1 * u1) + (u2 * u2)));
        double h = p + (rho * e);
        if (axis == 0) {
            F[i] = rho * u1;
            F[n + i] = p + ((rho * u1) * u1);
            F[2 * n + i] = (rho * u1) * u2;
            F[3 * n + i] = h * u1;
        } else {
            F[i] = rho * u2;
            F[n + i] = (rho * u1) * u2;
            F[2 * n + i] = p + ((rho * u2) * u2);
            F[3 * n + i] = h * u2;
        }
    }
}

/* ---------------------------------------------------------------- solver */

/* solver.py:154-159 local_timestep (+ state.py:66-68 speed, :166 sound_speed) */
void orc_local_timestep(const orc_conn *c, const double *pr, double cfl, double gamma, double *dt)
{
    int64_t n = c->n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
        double speed = sqrt((u1 * u1) + (u2 * u2)) + sqrt((gamma * p) / rho);
        dt[i] = (cfl * c->d_min[i]) / speed;
    }
}

/* lsq.py:164-175 first_order_q_gradients: sequential CSR-order bincount */
void orc_first_order_q_gradients(const orc_conn *c, const double *q, double *qx, double *qy)
{
    const orc_stencil *s = &c->full;
    int64_t n = s->n_owners;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double sx[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
        for (int64_t e = s->ptr[i]; e < s->ptr[i + 1]; e++) {
            int64_t j = s->idx[e];
            double dx = s->dx[e], dy = s->dy[e];
            for (int k = 0; k < 4; k++) {
                double dq = q[k * n + j] - q[k * n + i];
                sx[k] = sx[k] + (dx * dq);
                sy[k] = sy[k] + (dy * dq);
            }
        }
        for (int k = 0; k < 4; k++) {
            qx[k * n + i] = ((s->syy[i] * sx[k]) - (s->sxy[i] * sy[k])) / s->det[i];
            qy[k * n + i] = ((s->sxx[i] * sy[k]) - (s->sxy[i] * sx[k])) / s->det[i];
        }
    }
}

/* lsq.py:214-227 one Jacobi sweep (double-buffered) */
static void qsweep(const orc_conn *c, const double *q, const double *qxo, const double *qyo,
                   double *qxn, double *qyn)
{
    const orc_stencil *s = &c->full;
    int64_t n = s->n_owners;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double sx[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
        for (int64_t e = s->ptr[i]; e < s->ptr[i + 1]; e++) {
            int64_t j = s->idx[e];
            double dx = s->dx[e], dy = s->dy[e];
            for (int k = 0; k < 4; k++) {
                double ti = q[k * n + j] - (0.5 * ((dx * qxo[k * n + j]) + (dy * qyo[k * n + j])));
                double t0 = q[k * n + i] - (0.5 * ((dx * qxo[k * n + i]) + (dy * qyo[k * n + i])));
                double dq = ti - t0;
                sx[k] = sx[k] + (dx * dq);
                sy[k] = sy[k] + (dy * dq);
            }
        }
        for (int k = 0; k < 4; k++) {
            qxn[k * n + i] = ((s->syy[i] * sx[k]) - (s->sxy[i] * sy[k])) / s->det[i];
            qyn[k * n + i] = ((s->sxx[i] * sy[k]) - (s->sxy[i] * sx[k])) / s->det[i];
        }
    }
}

/* lsq.py:184-245 compute_q_derivatives (cold start, n_inner sweeps) */
void orc_compute_q_derivatives(const orc_conn *c, const double *q, int n_inner, double *qx,
                               double *qy, double *inner_residuals)
{
    int64_t n = c->n, m = 4 * n;
    double *ax = malloc(sizeof(double) * m), *ay = malloc(sizeof(double) * m);
    orc_first_order_q_gradients(c, q, ax, ay);
    double *cx = ax, *cy = ay, *nx_ = qx, *ny_ = qy;
    /* ping-pong so that the last sweep lands in (qx, qy) */
    if (n_inner % 2 == 0) {
        memcpy(qx, ax, sizeof(double) * m);
        memcpy(qy, ay, sizeof(double) * m);
        cx = qx;
        cy = qy;
        nx_ = ax;
        ny_ = ay;
    }
    for (int it = 0; it < n_inner; it++) {
        qsweep(c, q, cx, cy, nx_, ny_);
        double r = 0.0;
        for (int64_t k = 0; k < m; k++) {
            double a = fabs(nx_[k] - cx[k]), b = fabs(ny_[k] - cy[k]);
            if (a > r) r = a;
            if (b > r) r = b;
        }
        if (inner_residuals) inner_residuals[it] = r;
        double *tx = cx, *ty = cy;
        cx = nx_;
        cy = ny_;
        nx_ = tx;
        ny_ = ty;
    }
    if (cx != qx) {
        memcpy(qx, cx, sizeof(double) * m);
        memcpy(qy, cy, sizeof(double) * m);
    }
    free(ax);
    free(ay);
}

static const int KIND_AXIS[4] = {0, 0, 1, 1};
static const double KIND_SIGN[4] = {1.0, -1.0, 1.0, -1.0};

/* perturbed edge state (solver.py:184-185), component k */
static inline double qtilde(const double *q, const double *qx, const double *qy, int64_t n, int k,
                            int64_t p, double dx, double dy)
{
    return q[k * n + p] - (0.5 * ((dx * qx[k * n + p]) + (dy * qy[k * n + p])));
}

/* positivity pre-scan reproducing the reference's raise order
 * (solver.py:164-170 via _interior_kind_term over _Blocks, :218-229) */
static int64_t n_active(const orc_conn *c) { return c->n_act > 0 && c->n_act < c->n ? c->n_act : c->n; }

static int flux_scan(const orc_conn *c, const double *q, const double *qx, const double *qy, int mode,
                     orc_error *err)
{
    int64_t n = c->n, na = n_active(c);
    int64_t nb = (na + BLOCK - 1) / BLOCK;
    for (int outer = 0; outer < (mode == 0 ? nb : 4); outer++) {
        for (int inner = 0; inner < (mode == 0 ? 4 : nb); inner++) {
            int kind = mode == 0 ? inner : outer;
            int64_t blk = mode == 0 ? outer : inner;
            const orc_stencil *s = &c->split[kind];
            int64_t lo = blk * BLOCK, hi = lo + BLOCK < na ? lo + BLOCK : na;
            int64_t e0 = s->ptr[lo], e1 = s->ptr[hi];
            int64_t bad = 0, first = -1, nan_i = -1, nan_0 = -1, cnt_i = 0, cnt_0 = 0;
            for (int64_t i = lo; i < hi; i++)
                for (int64_t e = s->ptr[i]; e < s->ptr[i + 1]; e++) {
                    double ti = qtilde(q, qx, qy, n, 3, s->idx[e], s->dx[e], s->dy[e]);
                    double t0 = qtilde(q, qx, qy, n, 3, i, s->dx[e], s->dy[e]);
                    if (ti >= 0.0 || t0 >= 0.0) {
                        if (first < 0) first = e - e0;
                        bad++;
                    }
                    if (isnan(ti)) {
                        if (nan_i < 0) nan_i = e - e0;
                        cnt_i++;
                    }
                    if (isnan(t0)) {
                        if (nan_0 < 0) nan_0 = e - e0;
                        cnt_0++;
                    }
                }
            if (bad) {
                set_err(err, ORC_CTX_FLUX_XP + kind, bad, first);
                return 1;
            }
            (void)e1;
            if (nan_i >= 0 || nan_0 >= 0) {
                /* q_to_primitives(q_tilde_i) runs first (solver.py:171) */
                if (nan_i >= 0)
                    set_err(err, ORC_CTX_Q2P, cnt_i, nan_i);
                else
                    set_err(err, ORC_CTX_Q2P, cnt_0, nan_0);
                return 1;
            }
        }
    }
    return 0;
}

/* solver.py:176-195 _interior_kind_term for one point, added into R
 * in kind order x+, x-, y+, y- (solver.py:219-229), then boundary rows
 * zeroed (:233-234). */
int orc_flux_residual(const orc_conn *c, const double *q, const double *qx, const double *qy,
                      int mode, double gamma, double *R, orc_error *err)
{
    int64_t n = c->n, na = n_active(c);
    if (flux_scan(c, q, qx, qy, mode, err)) return 1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        double acc[4] = {0, 0, 0, 0};
        if (c->flag[i] != 0 || i >= na) { /* rows zeroed anyway (solver.py:233-234) */
            for (int k = 0; k < 4; k++) R[k * n + i] = 0.0;
            continue;
        }
        for (int kind = 0; kind < 4; kind++) {
            const orc_stencil *s = &c->split[kind];
            int axis = KIND_AXIS[kind];
            double sg = KIND_SIGN[kind];
            double sxg[4] = {0, 0, 0, 0}, syg[4] = {0, 0, 0, 0};
            for (int64_t e = s->ptr[i]; e < s->ptr[i + 1]; e++) {
                int64_t j = s->idx[e];
                double dx = s->dx[e], dy = s->dy[e];
                double ti[4], t0[4];
                for (int k = 0; k < 4; k++) {
                    ti[k] = qtilde(q, qx, qy, n, k, j, dx, dy);
                    t0[k] = qtilde(q, qx, qy, n, k, i, dx, dy);
                }
                double pi[4], p0[4], gi[4], g0[4];
                q2p(ti[0], ti[1], ti[2], ti[3], gamma, &pi[0], &pi[1], &pi[2], &pi[3]);
                q2p(t0[0], t0[1], t0[2], t0[3], gamma, &p0[0], &p0[1], &p0[2], &p0[3]);
                sflux(pi[0], pi[1], pi[2], pi[3], axis, sg, gamma, gi);
                sflux(p0[0], p0[1], p0[2], p0[3], axis, sg, gamma, g0);
                for (int k = 0; k < 4; k++) {
                    double dg = gi[k] - g0[k];
                    sxg[k] = sxg[k] + (dx * dg);
                    syg[k] = syg[k] + (dy * dg);
                }
            }
            double det = c->det_safe[kind][i];
            for (int k = 0; k < 4; k++) {
                double t;
                if (axis == 0)
                    t = ((s->syy[i] * sxg[k]) - (s->sxy[i] * syg[k])) / det;
                else
                    t = ((s->sxx[i] * syg[k]) - (s->sxy[i] * sxg[k])) / det;
                acc[k] = acc[k] + t;
            }
        }
        for (int k = 0; k < 4; k++) R[k * n + i] = acc[k];
    }
    return 0;
}

/* solver.py:245-274 _frame_edge_states + :277-283 _ls_rows for one frame
 * family; which = 0 (tangent +, G_x+), 1 (tangent -, G_x-), 2 (normal).
 * For the normal family the caller selects the closure (wall / outer). */
typedef struct {
    const orc_conn *c;
    const double *q, *qx, *qy;
    double gamma;
} frame_ctx;

static int frame_scan(const frame_ctx *f, const orc_frame *fr, const orc_stencil *s, int ctx,
                      orc_error *err)
{
    int64_t n = f->c->n;
    int64_t bad = 0, first = -1;
    for (int64_t l = 0; l < fr->b; l++) {
        int64_t own = fr->points[l];
        for (int64_t e = s->ptr[l]; e < s->ptr[l + 1]; e++) {
            double dt = s->dx[e], dn = s->dy[e];
            double dxg = (dt * fr->tx[l]) + (dn * fr->nx[l]);
            double dyg = (dt * fr->ty[l]) + (dn * fr->ny[l]);
            double ti = qtilde(f->q, f->qx, f->qy, n, 3, s->idx[e], dxg, dyg);
            double t0 = qtilde(f->q, f->qx, f->qy, n, 3, own, dxg, dyg);
            if (ti >= 0.0 || t0 >= 0.0) {
                if (first < 0) first = own;
                bad++;
            }
        }
    }
    if (bad) {
        set_err(err, ctx, bad, first);
        return 1;
    }
    return 0;
}

/* edge end states of one frame edge, rotated into the frame and decoded */
static inline void frame_edge(const frame_ctx *f, const orc_frame *fr, const orc_stencil *s,
                              int64_t l, int64_t e, double pi[4], double p0[4])
{
    int64_t n = f->c->n;
    int64_t own = fr->points[l], j = s->idx[e];
    double tx = fr->tx[l], ty = fr->ty[l], nx = fr->nx[l], ny = fr->ny[l];
    double dt = s->dx[e], dn = s->dy[e];
    double dxg = (dt * tx) + (dn * nx);
    double dyg = (dt * ty) + (dn * ny);
    double ti[4], t0[4];
    for (int k = 0; k < 4; k++) {
        ti[k] = qtilde(f->q, f->qx, f->qy, n, k, j, dxg, dyg);
        t0[k] = qtilde(f->q, f->qx, f->qy, n, k, own, dxg, dyg);
    }
    /* _frame_q solver.py:238-242 */
    double fi1 = (tx * ti[1]) + (ty * ti[2]), fi2 = (nx * ti[1]) + (ny * ti[2]);
    double f01 = (tx * t0[1]) + (ty * t0[2]), f02 = (nx * t0[1]) + (ny * t0[2]);
    q2p(ti[0], fi1, fi2, ti[3], f->gamma, &pi[0], &pi[1], &pi[2], &pi[3]);
    q2p(t0[0], f01, f02, t0[3], f->gamma, &p0[0], &p0[1], &p0[2], &p0[3]);
}

/* tangent term ddt of one frame family (solver.py:291-295 / :316-320) */
static void tangent_term(const frame_ctx *f, const orc_frame *fr, const orc_stencil *s, double sg,
                         int64_t l, double out[4])
{
    double st[4] = {0, 0, 0, 0}, sn[4] = {0, 0, 0, 0};
    for (int64_t e = s->ptr[l]; e < s->ptr[l + 1]; e++) {
        double pi[4], p0[4], gi[4], g0[4];
        frame_edge(f, fr, s, l, e, pi, p0);
        sflux(pi[0], pi[1], pi[2], pi[3], 0, sg, f->gamma, gi);
        sflux(p0[0], p0[1], p0[2], p0[3], 0, sg, f->gamma, g0);
        for (int k = 0; k < 4; k++) {
            double dg = gi[k] - g0[k];
            st[k] = st[k] + (s->dx[e] * dg);
            sn[k] = sn[k] + (s->dy[e] * dg);
        }
    }
    for (int k = 0; k < 4; k++) out[k] = ((s->syy[l] * st[k]) - (s->sxy[l] * sn[k])) / s->det[l];
}

/* solver.py:336-373 apply_boundary (+ _wall_rows :286-309, _outer_rows
 * :312-333, _rotate_back :376-382) */
int orc_apply_boundary(const orc_conn *c, const double *q, const double *qx, const double *qy,
                       const double fs[4], double gamma, double *R, orc_error *err)
{
    int64_t n = c->n;
    frame_ctx f = {c, q, qx, qy, gamma};
    for (int which = 0; which < 2; which++) {
        if (which == 0 && !c->has_wall) continue;
        if (which == 1 && !c->has_outer) continue;
        const orc_frame *fr = which == 0 ? &c->wall : &c->outer;
        int ctx_t = which == 0 ? ORC_CTX_WALL_TANGENT : ORC_CTX_OUTER_TANGENT;
        int ctx_n = which == 0 ? ORC_CTX_WALL_NORMAL : ORC_CTX_OUTER_NORMAL;
        if (frame_scan(&f, fr, &fr->tplus, ctx_t, err)) return 1;
        if (frame_scan(&f, fr, &fr->tminus, ctx_t, err)) return 1;
        if (frame_scan(&f, fr, &fr->normal, ctx_n, err)) return 1;
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t l = 0; l < fr->b; l++) {
            double tp[4], tm[4], rows[4];
            tangent_term(&f, fr, &fr->tplus, 1.0, l, tp);
            tangent_term(&f, fr, &fr->tminus, -1.0, l, tm);
            const orc_stencil *s = &fr->normal;
            double st[4] = {0, 0, 0, 0}, sn[4] = {0, 0, 0, 0};
            double gfs[4];
            if (which == 1) {
                double ut = (fs[1] * fr->tx[l]) + (fs[2] * fr->ty[l]);
                double un = (fs[1] * fr->nx[l]) + (fs[2] * fr->ny[l]);
                sflux(fs[0], ut, un, fs[3], 1, -1.0, gamma, gfs);
            }
            for (int64_t e = s->ptr[l]; e < s->ptr[l + 1]; e++) {
                double pi[4], p0[4], dg[4];
                frame_edge(&f, fr, s, l, e, pi, p0);
                if (which == 0) {
                    double gi[4], g0[4];
                    sflux(pi[0], pi[1], pi[2], pi[3], 1, -1.0, gamma, gi);
                    sflux(p0[0], p0[1], p0[2], p0[3], 1, -1.0, gamma, g0);
                    for (int k = 0; k < 4; k++) dg[k] = gi[k] - g0[k];
                } else {
                    double gpi[4], gp0[4], gmi[4];
                    sflux(pi[0], pi[1], pi[2], pi[3], 1, 1.0, gamma, gpi);
                    sflux(p0[0], p0[1], p0[2], p0[3], 1, 1.0, gamma, gp0);
                    sflux(pi[0], pi[1], pi[2], pi[3], 1, -1.0, gamma, gmi);
                    for (int k = 0; k < 4; k++) dg[k] = (gpi[k] - gp0[k]) + (gmi[k] - gfs[k]);
                }
                for (int k = 0; k < 4; k++) {
                    st[k] = st[k] + (s->dx[e] * dg[k]);
                    sn[k] = sn[k] + (s->dy[e] * dg[k]);
                }
            }
            for (int k = 0; k < 4; k++) {
                double ddn = ((s->sxx[l] * sn[k]) - (s->sxy[l] * st[k])) / s->det[l];
                if (which == 0) {
                    double rt = (0.0 + tp[k]) + tm[k];
                    double rn = k == 2 ? 0.0 : (0.0 + (2.0 * ddn));
                    rows[k] = rt + rn;
                } else {
                    rows[k] = ((0.0 + tp[k]) + tm[k]) + ddn;
                }
            }
            int64_t g = fr->points[l];
            R[g] = rows[0];
            R[3 * n + g] = rows[3];
            R[n + g] = (fr->tx[l] * rows[1]) + (fr->nx[l] * rows[2]);
            R[2 * n + g] = (fr->ty[l] * rows[1]) + (fr->ny[l] * rows[2]);
        }
    }
    return 0;
}

/* solver.py:385-409 state_update_rk (no positivity check) */
void orc_state_update_rk(int64_t n, const double *Uo, const double *Us, int stage, const double *dt,
                         const double *R, double *Un)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        for (int k = 0; k < 4; k++) {
            int64_t x = k * n + i;
            if (stage == 3)
                Un[x] = (((2.0 / 3.0) * Uo[x]) + ((1.0 / 3.0) * Us[x])) - ((dt[i] / 6.0) * R[x]);
            else
                Un[x] = Us[x] - ((0.5 * dt[i]) * R[x]);
        }
    }
}

/* CPython math.fsum (Shewchuk partials, correctly rounded); finite inputs */
double orc_fsum(int64_t n, const double *v)
{
    int cap = 64, m = 0;
    double *p = malloc(sizeof(double) * cap);
    for (int64_t t = 0; t < n; t++) {
        double x = v[t];
        int i = 0;
        for (int j = 0; j < m; j++) {
            double y = p[j];
            if (fabs(x) < fabs(y)) {
                double tmp = x;
                x = y;
                y = tmp;
            }
            double hi = x + y;
            double lo = y - (hi - x);
            if (lo != 0.0) p[i++] = lo;
            x = hi;
        }
        m = i;
        if (m + 1 > cap) {
            cap *= 2;
            p = realloc(p, sizeof(double) * cap);
        }
        p[m++] = x;
    }
    double hi = 0.0;
    if (m > 0) {
        int k = m;
        hi = p[--k];
        double lo = 0.0;
        while (k > 0) {
            double x = hi;
            double y = p[--k];
            hi = x + y;
            double yr = hi - x;
            lo = y - yr;
            if (lo != 0.0) break;
        }
        if (k > 0 && ((lo < 0.0 && p[k - 1] < 0.0) || (lo > 0.0 && p[k - 1] > 0.0))) {
            double y = lo * 2.0;
            double x = hi + y;
            double yr = x - hi;
            if (y == yr) hi = x;
        }
    }
    free(p);
    return hi;
}

/* solver.py:412-421 residue_norm */
double orc_residue_norm(int64_t n, const double *Un, const double *Uo)
{
    double *sq = malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++) {
        double d = Un[i] - Uo[i];
        sq[i] = d * d;
    }
    double total = orc_fsum(n, sq);
    free(sq);
    return sqrt(total / (double)n);
}

/* solver.py:477-573 solve, given the initial state */
int orc_solve(const orc_conn *c, const orc_params *p, double *prims, double *U, double *history,
              int *iterations, int *converged, orc_error *err)
{
    int64_t n = c->n, m = 4 * n;
    double gamma = p->gamma;
    orc_error e0 = {0};
    if (!err) err = &e0;
    memset(err, 0, sizeof(*err));
    *iterations = 0;
    *converged = 0;
    if (orc_primitives_to_conserved(n, prims, gamma, U, err)) {
        err->context = ORC_CTX_INITIAL;
        return 1;
    }
    const double *fs = p->fs;
    double *dt = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * m);
    double *qx = malloc(sizeof(double) * m), *qy = malloc(sizeof(double) * m);
    double *R = malloc(sizeof(double) * m), *Uo = malloc(sizeof(double) * m);
    double *Un = malloc(sizeof(double) * m);
    int rc = 0;
    for (int it = 1; it <= p->n_outer; it++) {
        orc_local_timestep(c, prims, p->cfl, gamma, dt);
        memcpy(Uo, U, sizeof(double) * m);
        for (int stage = 1; stage <= 4; stage++) {
            err->iteration = it;
            err->stage = stage;
            if ((rc = orc_primitives_to_q(n, prims, gamma, q, err))) goto done;
            if (p->n_inner > 0) {
                orc_compute_q_derivatives(c, q, p->n_inner, qx, qy, NULL);
            } else {  /* first-order scheme: qx = qy = 0 */
                memset(qx, 0, sizeof(double) * m);
                memset(qy, 0, sizeof(double) * m);
            }
            if ((rc = orc_flux_residual(c, q, qx, qy, p->mode, gamma, R, err))) goto done;
            if ((rc = orc_apply_boundary(c, q, qx, qy, fs, gamma, R, err))) goto done;
            orc_state_update_rk(n, Uo, U, stage, dt, R, Un);
            memcpy(U, Un, sizeof(double) * m);
            if ((rc = orc_conserved_to_primitives(n, U, gamma, prims, err))) goto done;
        }
        err->stage = 0;
        double res = orc_residue_norm(n_active(c), U, Uo);
        history[it - 1] = res;
        *iterations = it;
        if (p->convergence_tol > 0.0 && res <= p->convergence_tol) {
            *converged = 1;
            break;
        }
    }
    err->iteration = 0;
done:
    free(dt);
    free(q);
    free(qx);
    free(qy);
    free(R);
    free(Uo);
    free(Un);
    return rc;
}

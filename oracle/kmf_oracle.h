/*
 * kmf_oracle.h -- CPU restatement of the reference q-LSKUM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * CUDA path (paper_2108_07031_b200/csrc) and the CPU baseline timed by
 * `bench.py --impl reference`.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference legs may load it.  The product never
 * links it and never falls back to it.
 *
 * Every function restates the arithmetic of the reference package
 * (/root/reference/pkg/src/kmf, pure numpy/scipy) operation-for-operation:
 * same evaluation order, products rounded before sums (compiled with
 * -ffp-contract=off), least-squares sums accumulated sequentially in CSR
 * order exactly like np.bincount.  Transcendentals come from glibc libm
 * (log/exp/erf/sqrt), which differ from numpy's SIMD log/exp and
 * scipy.special.erf by <= 1-3 ulp, so transcendental paths are compared
 * by tolerance and all others bitwise.
 *
 * Layout: scalars (n,), four-vectors (4, n) row-major (component c of
 * point i at [c*n + i]) -- reference state.py:14-16.
 */
#ifndef KMF_ORACLE_H
#define KMF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* geometry.py:222-266 StencilSet */
typedef struct {
    int64_t n_owners;
    int64_t n_edges;
    const int64_t *ptr;
    const int64_t *idx;
    const double *dx, *dy;
    const double *sxx, *sxy, *syy, *det;
} orc_stencil;

/* geometry.py:269-291 FrameStencils */
typedef struct {
    int64_t b;
    const int64_t *points;
    const double *tx, *ty, *nx, *ny;
    orc_stencil tplus, tminus, normal;
} orc_frame;

/* geometry.py:294-312 Connectivity */
typedef struct {
    int64_t n;
    const int64_t *flag;
    const double *d_min;
    orc_stencil full;
    orc_stencil split[4]; /* x+, x-, y+, y- */
    const double *det_safe[4];
    int has_wall, has_outer;
    orc_frame wall, outer;
    /* rows whose flux residual (and residue) are computed: a partition's
     * owned points (0 = all n).  Test/bench infrastructure for partitioned
     * checks and bounded CPU samples; the reference has no such field. */
    int64_t n_act;
} orc_conn;

/* error contexts (which reference raise site fired) */
enum {
    ORC_CTX_NONE = 0,
    ORC_CTX_INITIAL = 1,        /* state.py:80-88 validate("initial state") */
    ORC_CTX_FLUX_XP = 2,        /* solver.py:164-170 flux_residual[x+] */
    ORC_CTX_FLUX_XM = 3,
    ORC_CTX_FLUX_YP = 4,
    ORC_CTX_FLUX_YM = 5,
    ORC_CTX_WALL_TANGENT = 6,   /* solver.py:260-265 */
    ORC_CTX_WALL_NORMAL = 7,
    ORC_CTX_OUTER_TANGENT = 8,
    ORC_CTX_OUTER_NORMAL = 9,
    ORC_CTX_C2P_DENSITY = 10,   /* state.py:110-117 */
    ORC_CTX_C2P_PRESSURE = 11,  /* state.py:121-128 */
    ORC_CTX_Q2P = 12,           /* state.py:151-157 */
    ORC_CTX_P2Q = 13            /* state.py:80-88 validate("primitives_to_q") */
};

typedef struct {
    int code;        /* 0 ok, 1 positivity */
    int iteration;   /* 1-based outer iteration, 0 outside solve */
    int stage;       /* 1..4 RK stage, 0 outside */
    int context;     /* ORC_CTX_* */
    int64_t count;   /* number of offending entries */
    int64_t first;   /* first offending index (reference's own numbering) */
} orc_error;

typedef struct {
    double fs[4];             /* free-stream primitives (state.py:170-185), host-computed */
    double gamma, cfl;
    int n_outer, n_inner;
    int mode;                 /* 0 fused, 1 split4 */
    double convergence_tol;   /* <= 0 : none */
} orc_params;

void orc_set_threads(int n);
int orc_get_threads(void);

int orc_primitives_to_q(int64_t n, const double *prims, double gamma, double *q, orc_error *err);
int orc_q_to_primitives(int64_t n, const double *q, double gamma, double *prims, orc_error *err);
int orc_primitives_to_conserved(int64_t n, const double *prims, double gamma, double *U, orc_error *err);
int orc_conserved_to_primitives(int64_t n, const double *U, double gamma, double *prims, orc_error *err);
void orc_split_flux(int64_t n, const double *prims, int axis, int sign, double gamma, double *G);
void orc_full_flux(int64_t n, const double *prims, int axis, double gamma, double *F);

void orc_local_timestep(const orc_conn *c, const double *prims, double cfl, double gamma, double *dt);
void orc_first_order_q_gradients(const orc_conn *c, const double *q, double *qx, double *qy);
void orc_compute_q_derivatives(const orc_conn *c, const double *q, int n_inner,
                               double *qx, double *qy, double *inner_residuals);
int orc_flux_residual(const orc_conn *c, const double *q, const double *qx, const double *qy,
                      int mode, double gamma, double *R, orc_error *err);
int orc_apply_boundary(const orc_conn *c, const double *q, const double *qx, const double *qy,
                       const double fs[4], double gamma, double *R, orc_error *err);
void orc_state_update_rk(int64_t n, const double *U_outer, const double *U_stage, int stage,
                         const double *dt, const double *R, double *U_new);
double orc_residue_norm(int64_t n, const double *U_new, const double *U_old);
double orc_fsum(int64_t n, const double *v);

/* solver.py:477-573 with a given initial state (prims, (4,n)); on return
 * prims/U hold the final state, history[0..iters-1] the residue norms. */
int orc_solve(const orc_conn *c, const orc_params *p, double *prims, double *U,
              double *history, int *iterations, int *converged, orc_error *err);

#ifdef __cplusplus
}
#endif
#endif

/*
 * kmf_b200.h -- C ABI of the B200-native q-LSKUM hot path (libkmf_b200.so).
 *
 * The reference (arXiv 2108.07031 desk re-implementation, package `kmf`,
 * /root/reference/pkg/src/kmf) is pure Python/numpy and has no FFI; its
 * "operator API" is the Python surface of solver.py / lsq.py / state.py /
 * kinetics.py.  Each entry point below replaces one reference function and
 * cites it.  The Python mirror (paper_2108_07031_b200/) binds these through
 * ctypes with exactly the reference's names and argument meaning.
 *
 * Conventions
 *   - plain pointers and sizes, no torch types; host buffers are caller
 *     owned and every call is synchronous on return;
 *   - four-vector fields use the reference layout (4, n) row-major
 *     (component c of point i at [c*n + i]), scalars (n,);
 *   - status codes: KMF_OK, KMF_EPOSITIVITY (reference PositivityError),
 *     KMF_EINVAL (reference ValueError), KMF_ECUDA, KMF_ENCCL, KMF_EPEER
 *     (peer transport deadline);
 *   - a context is bound to one CUDA device and is not thread-safe; use one
 *     context per process/GPU.
 */
#ifndef KMF_B200_H
#define KMF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMF_ABI_VERSION 1

enum {
    KMF_OK = 0,
    KMF_EPOSITIVITY = 1,
    KMF_EINVAL = 2,
    KMF_ECUDA = 3,
    KMF_ENCCL = 4,
    KMF_EPEER = 5   /* peer transport: a peer rank did not arrive within the deadline */
};

/* Which reference raise site a positivity failure corresponds to. */
enum {
    KMF_CTX_NONE = 0,
    KMF_CTX_INITIAL = 1,       /* state.py:80-88 validate("initial state")   */
    KMF_CTX_FLUX_XP = 2,       /* solver.py:164-170 flux_residual[x+]        */
    KMF_CTX_FLUX_XM = 3,       /*                   flux_residual[x-]        */
    KMF_CTX_FLUX_YP = 4,       /*                   flux_residual[y+]        */
    KMF_CTX_FLUX_YM = 5,       /*                   flux_residual[y-]        */
    KMF_CTX_WALL_TANGENT = 6,  /* solver.py:260-265 "wall tangent"           */
    KMF_CTX_WALL_NORMAL = 7,   /*                   "wall normal"            */
    KMF_CTX_OUTER_TANGENT = 8, /*                   "outer tangent"          */
    KMF_CTX_OUTER_NORMAL = 9,  /*                   "outer normal"           */
    KMF_CTX_C2P_DENSITY = 10,  /* state.py:110-117 conserved_to_primitives   */
    KMF_CTX_C2P_PRESSURE = 11, /* state.py:121-128                           */
    KMF_CTX_Q2P = 12,          /* state.py:151-157 q_to_primitives (NaN q4)  */
    KMF_CTX_P2Q = 13           /* state.py:80-88 validate("primitives_to_q") */
};

/* One CSR stencil family with its cached LS sums -- geometry.py:222-266
 * StencilSet.  ptr has n_owners+1 entries; idx/dx/dy n_edges. */
typedef struct {
    int64_t n_owners;
    int64_t n_edges;
    const int64_t *ptr;
    const int64_t *idx;
    const double *dx, *dy;
    const double *sxx, *sxy, *syy, *det;
} kmf_stencil;

/* Rotated-frame stencils of one boundary class -- geometry.py:269-291
 * FrameStencils (dx = dt, dy = dn in the local frame, owners numbered
 * locally 0..b-1, points[] their global indices). */
typedef struct {
    int64_t b;
    const int64_t *points;
    const double *tx, *ty, *nx, *ny;
    kmf_stencil tplus, tminus, normal;
} kmf_frame;

/* Connectivity -- geometry.py:294-312 (+ the cloud, geometry.py:56-112).
 * The four split families (geometry.py:544-549) are order-preserving
 * subsets of `full` selected by dx<=0, dx>=0, dy<=0, dy>=0; only their LS
 * sums and det_safe (geometry.py:505-508) cross the ABI, membership is
 * re-derived on the device from the sign of the full-stencil offsets.
 * When full.dx/dy equal x[idx]-x[owner] bitwise (what build_stencils
 * produces, geometry.py:377-384) the device recomputes them from x, y and
 * never stores per-edge offsets. */
typedef struct {
    int64_t n;
    const double *x, *y;
    const int64_t *flag;        /* 0 interior, 1 wall, 2 outer */
    const double *d_min;        /* geometry.py:537-539 */
    kmf_stencil full;
    const double *split_sxx[4]; /* x+, x-, y+, y- */
    const double *split_sxy[4];
    const double *split_syy[4];
    const double *det_safe[4];
    int has_wall, has_outer;
    kmf_frame wall, outer;
    /* optional point permutation (space-filling-curve order), NULL for
     * identity: device slot k holds caller point perm[k].  Neighbour lists
     * keep their reference order, so results are bitwise identical. */
    const int64_t *perm;
} kmf_geometry;

/* solver.py:69-99 SolverConfig, as consumed by the hot loop */
typedef struct {
    double gamma;
    double cfl;
    double fs[4];            /* free_stream(mach, aoa, gamma) primitives, state.py:170-185 */
    int n_inner;             /* Jacobi sweeps per stage (lsq.py:229); 0 = first-order scheme (qx = qy = 0) */
    int mode;                /* 0 fused, 1 split4 (solver.py:51, :218-229) */
    double convergence_tol;  /* <= 0: none (solver.py:557-559) */
    int instrument;          /* per-stage device timing (solver.py:461-474) */
    int timing_skip;         /* iterations excluded from timing (solver.py:516) */
} kmf_params;

/* Positivity / error report (PositivityError, state.py:28-38). */
typedef struct {
    int code;            /* KMF_* of the failing call */
    int iteration;       /* 1-based outer iteration (solver.py:552) or 0 */
    int stage;           /* RK stage 1..4, or 0 */
    int context;         /* KMF_CTX_* */
    int64_t count;       /* offending entries */
    int64_t n_indices;   /* entries written to kmf_last_indices */
    char message[256];
} kmf_error_info;

typedef struct kmf_ctx kmf_ctx;

int kmf_abi_version(void);
/* number of CUDA devices visible (0 without a GPU; no CUDA call fails) */
int kmf_device_count(void);

/* ---- context: Connectivity upload + the on-device outer loop ------------ */

/* deep-copies the geometry to `device`; replaces the per-call packing the
 * reference does implicitly inside solve (solver.py:500-506) */
int kmf_create(kmf_ctx **out, const kmf_geometry *g, int device);
void kmf_destroy(kmf_ctx *ctx);
/* initial primitives (4,n); the next kmf_run seeds U, q and dt from them
 * with its own gamma/cfl (solver.py:502-506, :520) */
int kmf_set_state(kmf_ctx *ctx, const double *prims);
/* solver.py:515-559: n_iter outer iterations of timestep + 4 SSP-RK stages
 * + residue; history[0..*iters_done-1] = residue_norm per iteration. */
int kmf_run(kmf_ctx *ctx, const kmf_params *p, int n_iter, double *history, int *iters_done,
            int *converged);
/* capture (once) the iteration graphs a kmf_run with these parameters
 * replays -- optional: kmf_run captures on first use; solve() calls it
 * before its timed chunk so graph capture is not timed */
int kmf_prepare(kmf_ctx *ctx, const kmf_params *p);
/* Streaming cases: n_cases independent solves on this context's cloud,
 * case k = kmf_set_state(prims_in[k]) + kmf_run(&params[k], n_iter,
 * instrument off) + kmf_get_state(prims_out[k]) with the same results bit
 * for bit, pipelined: case k+1's upload and case k-1's download run on the
 * copy engines while case k iterates (host buffers should be pinned,
 * kmf_host_alloc; they are read / written asynchronously until the call
 * returns; conserved_out, or any of its entries, may be NULL: the final
 * conserved state is then not downloaded).  The reference's harness runs such
 * batches one solve at a time
 * (bench.py:174-215 sweep).  Outputs per case k: history[k*n_iter + i]
 * (0 past iters_done[k]), iters_done[k], converged[k], status[k]
 * (KMF_OK / KMF_EPOSITIVITY); any may be NULL.  Returns KMF_EPOSITIVITY if
 * a case failed (kmf_last_error: the first failing case), after running
 * every case.  The context keeps the last case's final state. */
int kmf_run_cases(kmf_ctx *ctx, const kmf_params *params, int n_iter, int n_cases,
                  const double *const *prims_in, double *const *prims_out,
                  double *const *conserved_out, double *history, int *iters_done, int *converged,
                  int *status);
/* final primitives and conserved (each (4,n)), either may be NULL */
int kmf_get_state(kmf_ctx *ctx, double *prims, double *U);
/* device seconds per STAGE_NAMES key (solver.py:53-60) accumulated by the
 * last instrumented kmf_run over its timed iterations */
int kmf_stage_seconds(kmf_ctx *ctx, double out[6]);
/* error details of the last failing call on this context (or global) */
int kmf_last_error(kmf_ctx *ctx, kmf_error_info *info);
int kmf_last_indices(kmf_ctx *ctx, int64_t *idx, int64_t cap);

/* ---- positivity diagnostics (PositivityError details) ------------------- *
 * After a KMF_EPOSITIVITY from kmf_run / kmf_op_flux_residual /
 * kmf_op_boundary the device still holds the failing stage's q and
 * gradients (every later kernel was skipped).  These calls recompute the
 * reference's positivity predicates on that data so the host can rebuild
 * the exact PositivityError (context, count, indices) of solver.py:164-170,
 * :260-265 and state.py:110-128.  `which` selects the gradient buffer that
 * holds the final sweep: 0 for the op API and even n_inner, 1 for odd. */
/* per caller-CSR edge of the full stencil: bit0 q~4 >= 0 at either end,
 * bit1 NaN at the neighbour end, bit2 NaN at the owner end */
int kmf_diag_flux(kmf_ctx *ctx, int which, uint8_t *flags);
/* per frame edge of family fam (0 tplus, 1 tminus, 2 normal) over the
 * wall-then-outer boundary table: 1 where q~4 >= 0 at either end */
int kmf_diag_frame(kmf_ctx *ctx, int which, int fam, uint8_t *flags);
/* conserved state written by the failing stage's update, (4,n) */
int kmf_diag_stage_state(kmf_ctx *ctx, int stage, double *U);

/* ---- stage operators on a context (host in/out, synchronous) ------------ */

/* solver.py:154-159 local_timestep */
int kmf_op_timestep(kmf_ctx *ctx, const double *prims, double cfl, double gamma, double *dt);
/* lsq.py:164-175 first_order_q_gradients */
int kmf_op_first_order(kmf_ctx *ctx, const double *q, double *qx, double *qy);
/* lsq.py:184-245 compute_q_derivatives; prev_qx/prev_qy may be NULL (cold
 * start); inner_residuals has n_inner entries (may be NULL) */
int kmf_op_q_derivatives(kmf_ctx *ctx, const double *q, int n_inner, const double *prev_qx,
                         const double *prev_qy, double *qx, double *qy, double *inner_residuals);
/* solver.py:198-235 flux_residual (boundary rows zero) */
int kmf_op_flux_residual(kmf_ctx *ctx, const double *q, const double *qx, const double *qy,
                         int mode, double gamma, double *R);
/* solver.py:336-373 apply_boundary; R is updated in place */
int kmf_op_boundary(kmf_ctx *ctx, const double *q, const double *qx, const double *qy,
                    const double fs[4], double gamma, double *R);

/* ---- context-free point operators --------------------------------------- */

/* state.py:132-138 primitives_to_q; flags[i] != 0 marks validate failures */
int kmf_op_primitives_to_q(int64_t n, const double *prims, double gamma, double *q, uint8_t *flags);
/* state.py:141-163 q_to_primitives; flags[i] != 0 where !(q4 < 0) */
int kmf_op_q_to_primitives(int64_t n, const double *q, double gamma, double *prims, uint8_t *flags);
/* state.py:91-96 primitives_to_conserved */
int kmf_op_primitives_to_conserved(int64_t n, const double *prims, double gamma, double *U,
                                   uint8_t *flags);
/* state.py:99-129 conserved_to_primitives; flags bit0 density, bit1 pressure */
int kmf_op_conserved_to_primitives(int64_t n, const double *U, double gamma, double *prims,
                                   uint8_t *flags);
/* kinetics.py:71-106 split_flux; axis 0/1 = x/y, sign +1/-1 */
int kmf_op_split_flux(int64_t n, const double *prims, int axis, int sign, double gamma, double *G);
/* kinetics.py:59-68 full_flux */
int kmf_op_full_flux(int64_t n, const double *prims, int axis, double gamma, double *F);
/* solver.py:385-409 state_update_rk (positivity is checked by the caller
 * through kmf_op_conserved_to_primitives, as the reference does) */
int kmf_op_state_update(int64_t n, const double *U_outer, const double *U_stage, int stage,
                        const double *dt, const double *R, double *U_new);
/* solver.py:412-421 residue_norm, exactly summed (math.fsum semantics) */
int kmf_op_residue(int64_t n, const double *U_new, const double *U_old, double *out);

/* last global (context-free) error string */
const char *kmf_strerror(void);

/* ---- multi-GPU partition (paper_2108_07031_b200/partition.py) ------------ *
 * A partitioned context holds its rank's owned points (local slots
 * 0..n_owned-1, ordered by DEPTH = hop distance to the nearest halo slot,
 * deepest first) followed by `depth` halo layers L1..Ldepth (depth >=
 * n_inner + 2).  layer_end[k] = n_owned + |L1..Lk| (k = 0..depth);
 * interior_end[k] = owned slots at depth >= k (k = 0..depth+1).  Per stage
 * each kernel runs an INTERIOR pass over the owned slots deep enough not to
 * read this stage's halo data -- overlapping the halo exchange -- and a BAND
 * pass over the rest after it; flux, boundary and update cover the owned
 * points; the residue limbs are summed across ranks before the iteration
 * close, so every rank's arithmetic -- and the history -- is bitwise the
 * single-GPU one.  send_slots/recv_slots are concatenated per peer
 * (peer_ranks order): owned local slots to send, halo local slots to fill. */
int kmf_set_partition(kmf_ctx *ctx, int64_t n_owned, int64_t n_global, int rank, int nranks, int depth,
                      const int64_t *layer_end, const int64_t *interior_end, int npeers, const int *peer_ranks,
                      const int64_t *send_counts, const int64_t *send_slots, const int64_t *recv_counts,
                      const int64_t *recv_slots);
/* NCCL transport (one process per GPU): inside the iteration graph the halo
 * exchange (pack, grouped send/recv per peer, unpack) of every stage runs on
 * a forked stream concurrently with the next stage's interior pass, and the
 * limb all-reduce precedes the iteration close; kmf_run then works as for a
 * single domain.  libnccl.so.2 is loaded at run time. */
int kmf_nccl_get_unique_id(void *out128);
int kmf_nccl_init(kmf_ctx *ctx, const void *id128, int rank, int nranks);
/* one process driving all ranks' contexts (same or peer GPUs): halo moves
 * by device/peer copies, limbs summed on the host */
int kmf_run_group(kmf_ctx **ctxs, int nctx, const kmf_params *p, int n_iter, double *history, int *iters_done,
                  int *converged);

/* Peer transport (csrc/kmf_peer.cuh): no NCCL on the data path.  Every
 * rank maps its peers' q arrays and flag blocks (NVLink / NVSwitch peer
 * memory); each stage update stores the new q of its send points straight
 * into the peers' halo slots (compute and transfer in one kernel), device
 * counters with system-scope release/acquire order the pushes against the
 * peers' band passes, and the residue limbs are all-gathered over peer
 * memory before the iteration close.  Histories stay bitwise the
 * single-GPU ones.  A wait that exceeds 30 s sets KMF_EPEER on the run.
 *
 * Processes (one per GPU): kmf_peer_handle writes this context's
 * KMF_PEER_HANDLE_BYTES of CUDA IPC handles; after an all-gather of them,
 * kmf_peer_open(handles[nranks], dst_counts, dst_slots) maps the peers:
 * per peer in the partition's peer order, the peer's local halo slots that
 * receive this rank's send list (its recv list for this rank).  kmf_run,
 * kmf_run_cases and kmf_bench_steps then run as for one domain.
 * One process: kmf_peer_link(ctxs) links the ranks' contexts directly and
 * kmf_run_linked enqueues every rank's run before awaiting any (kmf_run,
 * kmf_run_cases and kmf_bench_steps refuse such a context alone: its peers
 * would never start).  Ranks sharing a device need
 * CUDA_DEVICE_MAX_CONNECTIONS >= 2 per rank (kmf_peer_link checks). */
#define KMF_PEER_HANDLE_BYTES 128
int kmf_peer_handle(kmf_ctx *ctx, void *out);
int kmf_peer_open(kmf_ctx *ctx, const void *handles, const int64_t *dst_counts, const int64_t *dst_slots);
int kmf_peer_link(kmf_ctx **ctxs, int nctx);
int kmf_run_linked(kmf_ctx **ctxs, int nctx, const kmf_params *p, int n_iter, double *history, int *iters_done,
                   int *converged);
/* diagnostics: out[0..2] = this rank's pushes, band passes, iterations;
 * out[3 + r], out[3 + nranks + r], out[3 + 2 nranks + r] = the data, read
 * and limb counters peer r last published here */
int kmf_peer_counters(kmf_ctx *ctx, uint64_t *out);

/* ---- measurement support (bench.py) -------------------------------------- */

/* 2 x n_steps outer iterations.  First n_steps plain CUDA-graph launches of
 * one iteration, each bracketed by CUDA events on the context stream
 * (step_ms[i]); a flush_bytes memset between steps evicts L2 outside the
 * timed region.  Then n_steps launches of the same iteration with event
 * nodes around its launch groups: kernel_ms[KMF_BENCH_KERNELS*i+k] sums
 * step i's launches of kernel class k (0 interior flux_residual, 1
 * first-order q-gradients, 2 Jacobi sweeps), timed on their own stream;
 * *launches_per_step counts this library's kernel launches per iteration. */
#define KMF_BENCH_KERNELS 3
int kmf_bench_steps(kmf_ctx *ctx, const kmf_params *p, int n_steps, int64_t flush_bytes, double *step_ms,
                    double *kernel_ms, int *launches_per_step);
/* measured FP64 (DFMA) pipe peak of the current device, TFLOP/s */
int kmf_fp64_peak(double *tflops);
/* device transcendentals of the flux path on host inputs (accuracy tests):
 * which 0 and 4 table exp, 1 erf (the kernel's branch-free |s| < 1
 * polynomial and tail), 2 reciprocal, 3 reciprocal square root, 5 table exp
 * without clamps (arguments <= 0) */
int kmf_fastmath_probe(int64_t n, const double *x, int which, double *out);
/* the flux kernel's edge-state path on q vectors (4, n) (test probe of the
 * tolerance arithmetic, state.py:141-163 + kinetics.py:71-106): its decode
 * -> prims (4, n) (p = rho / (2 beta)) and its four split fluxes x+, x-, y+,
 * y- -> flux (16, n), family f in rows 4f..4f+3 */
int kmf_probe_edge_state(int64_t n, const double *q, double gamma, double *prims, double *flux);
/* pinned host memory for host-buffer (end-to-end) transfers */
void *kmf_host_alloc(int64_t bytes);
void kmf_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* KMF_B200_H */

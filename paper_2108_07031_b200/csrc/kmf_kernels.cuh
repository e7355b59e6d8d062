// kmf_kernels.cuh -- sm_100a kernels of the q-LSKUM outer iteration.
//
// Device data layout:
//   * per-point fields are SoA with a padded leading dimension `ld`
//     (component c of device slot i at [c*ld + i]): U_outer[4], U_stage[4],
//     R[4], dt, flags; the fields the stencil gathers are packed per point
//     instead: q as one 32-byte record q[4*i + c] (one 256-bit load per
//     neighbour, qload), the q gradients G with the two derivatives of a
//     component interleaved (two layouts, see gload_cm / gload), and
//     (x, y) as one double2 (pxy);
//   * the full stencil is stored as sliced ELLPACK with slice height 32
//     (one warp): neighbour slot s of point i lives at
//     eoff[i/32] + s*32 + i%32, so the per-slot gathers of a warp are one
//     coalesced 128 B index load; slots keep the reference CSR order
//     (np.sort order, geometry.py:345) because that order IS the summation
//     order of every least-squares sum;
//   * the four split families are not stored: membership is the sign of
//     dx/dy (geometry.py:544-549), recomputed bitwise from x, y.
//
// One thread per point everywhere except the boundary closure (one warp
// per boundary point, lanes over frame edges).
#pragma once
#include "kmf_fastmath.cuh"
#include "kmf_math.cuh"

namespace kmf {

constexpr int kTB = 128;   // threads per block, point kernels
constexpr int kSlotFlux = 0xE00;
constexpr int kSlotUpdate = 0xE01;
constexpr int kStageFinal = 7;

// Control block in device memory.  `state` packs a status and the sequence
// number of the launch that set it: 0 running, (seq<<2)|1 positivity error,
// (seq<<2)|2 converged.  Kernels skip their work once state != 0 unless they
// carry the very same seq (so every block of the failing launch, and the
// boundary kernel that shares its seq, still completes).  The seq is built
// from `epoch`, which the end-of-iteration kernel advances on EVERY replayed
// iteration (also skipped ones), so no later launch can share a seq with the
// failing one; `iter` advances only on completed iterations.
struct Ctrl {
    unsigned long long state;
    int iter;
    int epoch;
    int err_iter;
    int err_stage;
    unsigned int ctx_mask;
    unsigned int blocks_done;   // last-block detection of the stage-4 update
    unsigned long long resmax;  // inner-residual max (bits of a nonnegative double)
    double *history;            // residue_norm of iteration k at history[k - 1], k <= hist_cap
    int hist_cap;
    unsigned long long limbs[kLimbs];
    unsigned long long peer_fail;  // peer transport: a wait for another rank timed out (kmf_peer.cuh)
};

KMF_HD long long seq_of(int epoch, int stage, int slot)
{
    return ((long long)epoch << 16) | ((long long)stage << 12) | (long long)slot;
}

KMF_HD bool should_skip(const Ctrl *c, int stage, int slot)
{
    unsigned long long st = *(volatile const unsigned long long *)&c->state;
    if (st == 0ull) return false;
    long long me = seq_of(*(volatile const int *)&c->epoch, stage, slot);
    return (long long)(st >> 2) != me;
}

__device__ __forceinline__ void raise_err(Ctrl *c, int stage, int slot, int ctx)
{
    atomicOr(&c->ctx_mask, 1u << ctx);
    unsigned long long want = ((unsigned long long)seq_of(c->epoch, stage, slot) << 2) | 1ull;
    if (atomicCAS(&c->state, 0ull, want) == 0ull) {
        c->err_iter = c->iter;
        c->err_stage = stage;
    }
}

// Geometry as seen by the point kernels.
struct DG {
    int n, ld;
    int n_norm;  // residue normalisation (global point count under a partition)
    const double *__restrict__ x;
    const double *__restrict__ y;
    const double2 *__restrict__ pxy;  // (x, y) interleaved: one 16-byte neighbour gather
    const unsigned char *__restrict__ flag;
    const double *__restrict__ dmin;
    const int *__restrict__ eoff;   // per 32-point slice
    const int *__restrict__ deg;    // per point
    const int *__restrict__ eidx;   // ELL neighbour slots
    const double *__restrict__ edx;  // ELL offsets (only when not derived from x, y)
    const double *__restrict__ edy;
    const double *__restrict__ fsum;   // [4][ld] full-stencil sxx, sxy, syy, det
    const double *__restrict__ fcoef;  // [8][ld] (cx, cy) of x+, x-, y+, y-
    const long long *__restrict__ cptr;  // caller CSR ptr of the point in this slot (diag)
};

// Boundary frames (wall entries first, then outer), geometry.py:573-646.
struct DB {
    int nb;
    const int *__restrict__ point;          // device slot of the owner
    const unsigned char *__restrict__ type;  // 1 wall, 2 outer
    const double *__restrict__ frame;       // [4][nb] tx, ty, nx, ny
    const double *__restrict__ coef;        // [6][nb] (ct, cn) of tplus, tminus, normal
    const int *__restrict__ ptr[3];
    const int *__restrict__ idx[3];
    const double *__restrict__ dt[3];
    const double *__restrict__ dn[3];
};

template <bool XY>
KMF_HD void edge_offsets(const DG &g, int ent, int j, double xi, double yi, double &dx, double &dy)
{
    if (XY) {
        const double2 pj = g.pxy[j];
        dx = SUB(pj.x, xi);  // geometry.py:382-383, bitwise
        dy = SUB(pj.y, yi);
    } else {
        dx = g.edx[ent];
        dy = g.edy[ent];
    }
}

KMF_HD int ell_base(const DG &g, int i) { return g.eoff[i >> 5] + (i & 31); }

// the q record of slot i: one 256-bit load (LDG.E.ENL2.256)
struct __align__(32) Q4 {
    double v[4];
};
KMF_HD Q4 qload(const double *__restrict__ q, int i) { return reinterpret_cast<const Q4 *>(q)[i]; }
// components k0 .. k0+NC-1 of slot i's record (NC 4: 256-bit, 2: 128-bit)
template <int NC>
KMF_HD void qload_nc(const double *__restrict__ q, int i, int k0, double (&out)[NC])
{
    if (NC == 4) {
        const Q4 r = qload(q, i);
#pragma unroll
        for (int k = 0; k < NC; k++) out[k] = r.v[k];
    } else if (NC == 2) {
        const double2 r = reinterpret_cast<const double2 *>(q + 4 * i + k0)[0];
        out[0] = r.x;
        out[NC - 1] = r.y;
    } else {
#pragma unroll
        for (int k = 0; k < NC; k++) out[k] = q[4 * i + k0 + k];
    }
}
KMF_HD void qstore(double *__restrict__ q, int i, const double (&v)[4])
{
    Q4 r;
#pragma unroll
    for (int k = 0; k < 4; k++) r.v[k] = v[k];
    reinterpret_cast<Q4 *>(q)[i] = r;
}

// Two gradient layouts.  The q-gradient kernels iterate in the
// component-major one, (qx_k, qy_k) of slot i as one double2 at
// G2[k*ld + i] (gload_cm / gstore_cm: four 128-bit loads per neighbour);
// the LAST sweep of a stage writes the plane layout the flux and boundary
// kernels read, two planes of 32-byte records (qx_2h, qy_2h, qx_2h+1,
// qy_2h+1) at Q4 index h*ld + i (gload / gload_nc: two 256-bit loads per
// neighbour).  Measured: the plane layout is 3 % faster for the flux and
// 2-3 % slower for the sweeps (profiles/r1_summary.md).
KMF_HD double2 gload_cm(const double *__restrict__ G, int ld, int k, int i)
{
    return reinterpret_cast<const double2 *>(G)[k * ld + i];
}
KMF_HD void gstore_cm(double *__restrict__ G, int ld, int k, int i, double gx, double gy)
{
    reinterpret_cast<double2 *>(G)[k * ld + i] = make_double2(gx, gy);
}
KMF_HD double2 gload(const double *__restrict__ G, int ld, int k, int i)
{
    return reinterpret_cast<const double2 *>(G)[2 * ((k >> 1) * ld + i) + (k & 1)];
}
// components k0 .. k0+NC-1 (k0 even for NC >= 2) of slot i, plane layout
template <int NC>
KMF_HD void gload_nc(const double *__restrict__ G, int ld, int i, int k0, double (&gx)[NC], double (&gy)[NC])
{
    if (NC >= 2) {
#pragma unroll
        for (int h = 0; h < NC / 2; h++) {
            const Q4 v = reinterpret_cast<const Q4 *>(G)[((k0 >> 1) + h) * ld + i];
            gx[2 * h] = v.v[0];
            gy[2 * h] = v.v[1];
            gx[(2 * h + 1) % NC] = v.v[2];
            gy[(2 * h + 1) % NC] = v.v[3];
        }
    } else {
        const double2 v = gload(G, ld, k0, i);
        gx[0] = v.x;
        gy[0] = v.y;
    }
}
// store components k0 .. k0+NC-1 of slot i in the plane (P) or the
// component-major layout
template <int NC, bool P>
KMF_HD void gstore_nc(double *__restrict__ G, int ld, int i, int k0, const double (&gx)[NC], const double (&gy)[NC])
{
    if (P && NC >= 2) {
#pragma unroll
        for (int h = 0; h < NC / 2; h++) {
            Q4 v;
            v.v[0] = gx[2 * h];
            v.v[1] = gy[2 * h];
            v.v[2] = gx[(2 * h + 1) % NC];
            v.v[3] = gy[(2 * h + 1) % NC];
            reinterpret_cast<Q4 *>(G)[((k0 >> 1) + h) * ld + i] = v;
        }
    } else if (P) {
        reinterpret_cast<double2 *>(G)[2 * ((k0 >> 1) * ld + i) + (k0 & 1)] = make_double2(gx[0], gy[0]);
    } else {
#pragma unroll
        for (int k = 0; k < NC; k++) gstore_cm(G, ld, k0 + k, i, gx[k], gy[k]);
    }
}

// ---------------------------------------------------------------------------
// Launch ranges.  Every point kernel covers the device slots [lo, hi) of
// its launch: the whole cloud on one GPU, the interior or the halo band of a
// partition (local slots are ordered by depth, so
// each pass is a contiguous range).  Blocks start at the 32-slot SELL slice
// holding lo, so the slices (and their staged index runs) stay aligned.
__host__ __device__ __forceinline__ int range_base(int lo) { return lo & ~31; }

// ---------------------------------------------------------------------------
// q-gradient kernels: NC components of one point per thread (NC = 4 above
// 100K points, 2 below).  The four components of q are independent in every
// LS sum, so splitting them over 4/NC threads keeps each sum sequential in
// CSR order (bitwise) while multiplying the threads in flight.  A 128-thread
// block covers 128*NC/4 points; warp w handles component group w % (4/NC) of
// the 32-point SELL slice w / (4/NC), so slice-local ELL offsets stay
// coalesced.
template <int NC>
KMF_HD void qg_thread(int lo, int &i, int &k0)
{
    constexpr int CG = 4 / NC;   // component groups per point
    constexpr int P = kTB / CG;  // points per block
    const int w = threadIdx.x >> 5;
    i = range_base(lo) + blockIdx.x * P + (w / CG) * 32 + (threadIdx.x & 31);
    k0 = (w % CG) * NC;
}

template <int NC>
__host__ __device__ constexpr int qg_points_per_block() { return kTB * NC / 4; }

// The block's ELL index slices are contiguous in the ELL table (slice
// offsets are multiples of 32 entries, so the source is 128 B aligned and
// the size a multiple of 128 B): ONE TMA bulk copy stages them in shared
// memory.  One thread arms an mbarrier with the byte count and issues
// cp.async.bulk global -> shared; every thread waits on the barrier's phase.
// Replaces one dependent index round trip per slot by a shared-memory read.
// SPB = slices per block.
KMF_HD uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Issue half: one thread arms the mbarrier and starts the copy; every
// thread passes the block barrier (the mbarrier is initialised before anyone
// polls it).  The kernels load their owner data between issue and wait, so
// the copy's latency overlaps those loads; every thread waits before it may
// leave (the copy must land before the CTA's shared memory is released).
template <int SPB>
KMF_HD bool qg_stage_issue(const DG &g, int lo, int *sidx, int cap, int &e0, unsigned long long *mbar)
{
    const int ns = (g.n + 31) >> 5;
    const int s0 = (range_base(lo) >> 5) + blockIdx.x * SPB;
    if (s0 >= ns) return false;
    e0 = g.eoff[s0];
    const int esz = g.eoff[min(s0 + SPB, ns)] - e0;
    const bool staged = esz <= cap && esz > 0;
    const uint32_t bar = smem_u32(mbar);
    if (staged && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t bytes = (uint32_t)esz * 4u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sidx)),
            "l"(g.eidx + e0), "r"(bytes), "r"(bar)
            : "memory");
    }
    __syncthreads();
    return staged;
}

KMF_HD void qg_stage_wait(bool staged, unsigned long long *mbar)
{
    if (!staged) return;
    const uint32_t bar = smem_u32(mbar);
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar)
            : "memory");
}

// One neighbour slot as the q-gradient kernels consume it: the neighbour's
// coordinates (XY) or the stored offsets (!XY), its q components k0.. and
// (WG, the sweeps) its gradients.
template <int NC, bool WG>
struct QgSlot {
    double x, y, q[NC], gx[WG ? NC : 1], gy[WG ? NC : 1];
};

template <bool XY, int NC, bool WG>
KMF_HD void qg_gather(QgSlot<NC, WG> &o, const DG &g, const double *__restrict__ q, const double *__restrict__ G,
                      int ld, int k0, int j, int ent)
{
    if (XY) {
        const double2 pj = g.pxy[j];
        o.x = pj.x;
        o.y = pj.y;
    } else {
        o.x = g.edx[ent];
        o.y = g.edy[ent];
    }
    qload_nc<NC>(q, j, k0, o.q);
#pragma unroll
    for (int k = 0; k < NC; k++) {
        if (WG) {
            const double2 v = gload_cm(G, ld, k0 + k, j);
            o.gx[k] = v.x;
            o.gy[k] = v.y;
        }
    }
}

// Software-pipelined slot loop: slot s+1 is gathered before slot s is
// evaluated, so the HBM/L2 round trip of the next neighbour overlaps the
// arithmetic of this one; slots are evaluated strictly in order 0..d-1 (the
// sums keep their order).  Measured variants (round 1): two slots ahead
// (138 registers) +28 %, unrolled by two with the loads interleaved into
// the arithmetic +4 %.
template <class Slot, class Gather, class Eval>
KMF_HD void qg_pipeline(int d, Gather gather, Eval eval)
{
    if (d <= 0) return;
    Slot cur;
    gather(0, cur);
    for (int s = 0; s < d; s++) {
        Slot nxt;
        gather(min(s + 1, d - 1), nxt);  // past the last slot: a redundant reload
        eval(cur);
        cur = nxt;
    }
}

// Two slot buffers, unrolled by two: while slot s is evaluated from one
// buffer, the gathers of slot s+1 are already in flight into the other
// (issued before slot s's arithmetic in program order).
template <class Slot, class Gather, class Eval>
KMF_HD void qg_pipeline2(int d, Gather gather, Eval eval)
{
    if (d <= 0) return;
    Slot a, b;
    gather(0, a);
    gather(min(1, d - 1), b);
    int s = 0;
    for (; s + 1 < d; s += 2) {
        eval(a);
        gather(min(s + 2, d - 1), a);
        eval(b);
        gather(min(s + 3, d - 1), b);
    }
    if (s < d) eval(a);
}

// The sweeps keep the one-buffer loop (94 registers, 5 blocks/SM): the
// two-buffer loop needs 125 registers (4 blocks/SM) and measured 8-11 %
// slower at 2.5M / 10M; the first-order kernel (bounded to 64 registers
// either way) takes the two-buffer loop (-3 %).
template <class Slot, bool TWO, class Gather, class Eval>
KMF_HD void qg_slots(int d, Gather gather, Eval eval)
{
    if constexpr (TWO)
        qg_pipeline2<Slot>(d, gather, eval);
    else
        qg_pipeline<Slot>(d, gather, eval);
}

// lsq.py:164-175 first_order_q_gradients -- bitwise (CSR-order sums, no FMA)
template <bool XY, int NC>
__global__ void __launch_bounds__(kTB, NC == 4 ? 8 : 0) k_first_order(DG g, int lo, int hi,
                                                                     const double *__restrict__ q,
                                                                     double *__restrict__ G, Ctrl *c, int stage)
{
    constexpr int SPB = qg_points_per_block<NC>() / 32, CAP = SPB * 32 * 24;
    __shared__ __align__(128) int sidx[CAP];
    __shared__ unsigned long long mbar;
    int e0 = 0;
    const bool staged = qg_stage_issue<SPB>(g, lo, sidx, CAP, e0, &mbar);
    int i, k0;
    qg_thread<NC>(lo, i, k0);
    const bool valid = i >= lo && i < hi;
    if (!valid) i = lo;  // a safe slot for the owner loads below
    const int ld = g.ld;
    double qi[NC], sx[NC], sy[NC];
    qload_nc<NC>(q, i, k0, qi);
#pragma unroll
    for (int k = 0; k < NC; k++) {
        sx[k] = 0.0;
        sy[k] = 0.0;
    }
    const double xi = g.x[i], yi = g.y[i];
    const int base = ell_base(g, i), d = g.deg[i];
    qg_stage_wait(staged, &mbar);
    if (!valid || (c && should_skip(c, stage, 0))) return;
    using Slot = QgSlot<NC, false>;
    qg_slots<Slot, true>(
        d,
        [&](int s, Slot &o) {
            const int ent = base + s * 32;
            qg_gather<XY, NC, false>(o, g, q, q, ld, k0, staged ? sidx[ent - e0] : g.eidx[ent], ent);
        },
        [&](const Slot &o) {
            const double dx = XY ? SUB(o.x, xi) : o.x, dy = XY ? SUB(o.y, yi) : o.y;  // geometry.py:382-383
#pragma unroll
            for (int k = 0; k < NC; k++) {
                const double dq = SUB(o.q[k], qi[k]);
                sx[k] = ADD(sx[k], MUL(dx, dq));
                sy[k] = ADD(sy[k], MUL(dy, dq));
            }
        });
    const double sxx = g.fsum[i], sxy = g.fsum[ld + i], syy = g.fsum[2 * ld + i], det = g.fsum[3 * ld + i];
#pragma unroll
    for (int k = 0; k < NC; k++) {
        gstore_cm(G, ld, k0 + k, i, DIV(SUB(MUL(syy, sx[k]), MUL(sxy, sy[k])), det),
                  DIV(SUB(MUL(sxx, sy[k]), MUL(sxy, sx[k])), det));
    }
}

// lsq.py:214-227 one Jacobi sweep of the defect-corrected gradients --
// bitwise.  With want_res the max |new - old| (lsq.py:238-243) is reduced.
// OUTP: the stage's last sweep writes the plane layout the flux and
// boundary kernels read.
template <bool XY, int NC, bool OUTP>
__global__ void __launch_bounds__(kTB) k_sweep(DG g, int lo, int hi, const double *__restrict__ q,
                                               const double *__restrict__ Gin, double *__restrict__ Gout,
                                               Ctrl *c, int stage, int slot, int want_res)
{
    constexpr int SPB = qg_points_per_block<NC>() / 32, CAP = SPB * 32 * 24;
    __shared__ __align__(128) int sidx[CAP];
    __shared__ unsigned long long mbar;
    int e0 = 0;
    const bool staged = qg_stage_issue<SPB>(g, lo, sidx, CAP, e0, &mbar);
    int i, k0;
    qg_thread<NC>(lo, i, k0);
    const bool valid = i >= lo && i < hi;
    if (!valid) i = lo;  // a safe slot for the owner loads below
    const int ld = g.ld;
    double qi[NC], gxi[NC], gyi[NC], sx[NC], sy[NC];
    qload_nc<NC>(q, i, k0, qi);
#pragma unroll
    for (int k = 0; k < NC; k++) {
        const double2 v = gload_cm(Gin, ld, k0 + k, i);
        gxi[k] = v.x;
        gyi[k] = v.y;
        sx[k] = 0.0;
        sy[k] = 0.0;
    }
    const double xi = g.x[i], yi = g.y[i];
    const int base = ell_base(g, i), d = g.deg[i];
    qg_stage_wait(staged, &mbar);
    if (c && should_skip(c, stage, slot)) return;
    double rmax = 0.0;
    if (valid) {
        using Slot = QgSlot<NC, true>;
        qg_slots<Slot, false>(
            d,
            [&](int s, Slot &o) {
                const int ent = base + s * 32;
                qg_gather<XY, NC, true>(o, g, q, Gin, ld, k0, staged ? sidx[ent - e0] : g.eidx[ent], ent);
            },
            [&](const Slot &o) {
                const double dx = XY ? SUB(o.x, xi) : o.x, dy = XY ? SUB(o.y, yi) : o.y;
                const double hdx = MUL(0.5, dx), hdy = MUL(0.5, dy);  // exact: see qtilde_h
#pragma unroll
                for (int k = 0; k < NC; k++) {
                    const double dq = SUB(qtilde_h(o.q[k], o.gx[k], o.gy[k], hdx, hdy),
                                          qtilde_h(qi[k], gxi[k], gyi[k], hdx, hdy));
                    sx[k] = ADD(sx[k], MUL(dx, dq));
                    sy[k] = ADD(sy[k], MUL(dy, dq));
                }
            });
        const double sxx = g.fsum[i], sxy = g.fsum[ld + i], syy = g.fsum[2 * ld + i],
                     det = g.fsum[3 * ld + i];
        double gxn[NC], gyn[NC];
#pragma unroll
        for (int k = 0; k < NC; k++) {
            gxn[k] = DIV(SUB(MUL(syy, sx[k]), MUL(sxy, sy[k])), det);
            gyn[k] = DIV(SUB(MUL(sxx, sy[k]), MUL(sxy, sx[k])), det);
        }
        gstore_nc<NC, OUTP>(Gout, ld, i, k0, gxn, gyn);
        if (want_res) {
            bool nan = false;
#pragma unroll
            for (int k = 0; k < NC; k++) {
                const double ex = gxn[k] - gxi[k], ey = gyn[k] - gyi[k];
                rmax = fmax(rmax, fmax(fabs(ex), fabs(ey)));
                nan |= isnan(ex) || isnan(ey);
            }
            if (nan) rmax = __longlong_as_double(0x7ff8000000000000ll);  // np.max propagates NaN
        }
    }
    if (want_res) {
        unsigned long long b = (unsigned long long)__double_as_longlong(rmax);
        for (int o = 16; o; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
            b = t > b ? t : b;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&c->resmax, b);
    }
}

// ---------------------------------------------------------------------------
// solver.py:385-409 state_update_rk + state.py:99-129 decode (bitwise),
// fused with primitives_to_q for the next stage (state.py:132-138) and, at
// stage 4, local_timestep for the next iteration (solver.py:154-159) and the
// exact residue partial sum (solver.py:412-421).
// Exact warp-aggregated residue accumulation: lanes whose 85-bit shifted
// mantissas start in the same 32-bit limb are summed with __reduce_add_sync
// on 16-bit pieces (exact: 32 * 2^16 < 2^21), and one lane per group adds
// the three limb sums to shared memory.  Every lane of the warp must call.
__device__ __forceinline__ void accum_add_warp(unsigned long long *limbs, double v)
{
    int L = -1;
    unsigned long long lo = 0, hi = 0;
    if (v > 0.0) {
        unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        int be = (int)(bits >> 52);
        unsigned long long m = bits & ((1ull << 52) - 1);
        int e2 = 0;
        if (be) {
            m |= 1ull << 52;
            e2 = be - 1;
        }
        L = e2 >> 5;
        const int sh = e2 & 31;
        lo = m << sh;
        hi = sh ? (m >> (64 - sh)) : 0ull;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, L);
    unsigned piece[6] = {(unsigned)(lo & 0xffff), (unsigned)((lo >> 16) & 0xffff), (unsigned)((lo >> 32) & 0xffff),
                         (unsigned)(lo >> 48), (unsigned)(hi & 0xffff), (unsigned)(hi >> 16)};
    unsigned s[6];
#pragma unroll
    for (int t = 0; t < 6; t++) s[t] = __reduce_add_sync(grp, piece[t]);
    const int lane = threadIdx.x & 31;
    if (L >= 0 && lane == __ffs(grp) - 1) {
        atomicAdd(&limbs[L], (unsigned long long)s[0] + ((unsigned long long)s[1] << 16));
        atomicAdd(&limbs[L + 1], (unsigned long long)s[2] + ((unsigned long long)s[3] << 16));
        const unsigned long long top = (unsigned long long)s[4] + ((unsigned long long)s[5] << 16);
        if (top) atomicAdd(&limbs[L + 2], top);
    }
}

KMF_HD double accum_round(const unsigned long long *limbs);

// Per-launch iteration-close parameters (the history buffer and its size
// live in Ctrl, set per run, so captured graphs do not depend on them).
struct IterOut {
    double tol;
    int close_in_kernel;  // 0 under a partition: limbs are all-reduced first, then k_close
};

// End of an outer iteration, run by one thread of the last stage-4 block:
// residue_norm = sqrt(fsum(drho^2)/n) (solver.py:418-421), history,
// convergence test (solver.py:557-559), counters.  Out of line so the
// per-point update keeps its small register footprint.
__device__ __noinline__ void close_iteration(Ctrl *c, const unsigned long long *limbs, int n, IterOut io)
{
    const int ep = c->epoch;
    const unsigned long long st = *(volatile unsigned long long *)&c->state;
    if (st == 0ull) {
        const double res = sqrt(accum_round(limbs) / (double)n);
        const int it = c->iter;
        const int h = it - 1;
        if (h >= 0 && h < c->hist_cap) c->history[h] = res;
        if (io.tol > 0.0 && res <= io.tol) c->state = ((unsigned long long)seq_of(ep, kStageFinal, 0) << 2) | 2ull;
        c->iter = it + 1;
    }
    c->blocks_done = 0u;
    c->epoch = ep + 1;
    __threadfence();
}

// Peer transport (kmf_peer.cuh): the stage update stores the new q of
// every owned point some peer holds in its halo straight into that peer's
// q array (NVLink / IPC peer memory) -- compute and halo transfer in one
// kernel.  CSR over owned slots; dst = (peer rank << kPeerSlotBits) | slot.
constexpr int kMaxRanks = 16;
constexpr unsigned kPeerSlotBits = 27;
struct PeerPush {
    const int *ptr;        // [n_owned + 1]; null: no push
    const unsigned *dst;
    double *q[kMaxRanks];  // peers' q arrays
};

__device__ __forceinline__ void peer_push(const PeerPush &pp, int i, const double (&v)[4])
{
    const int b = pp.ptr[i], e = pp.ptr[i + 1];
    for (int t = b; t < e; t++) {
        const unsigned d = pp.dst[t];
        qstore(pp.q[d >> kPeerSlotBits], (int)(d & ((1u << kPeerSlotBits) - 1)), v);
    }
    if (e > b) __threadfence_system();  // performed at system scope before this thread retires
}

template <int STAGE>
__global__ void __launch_bounds__(kTB) k_update(DG g, int lo, int hi, double *__restrict__ Uo, double *__restrict__ Us,
                                                const double *__restrict__ R, double *__restrict__ dt,
                                                double *__restrict__ q, double gamma, double cfl, Ctrl *c,
                                                IterOut io, PeerPush pp)
{
    __shared__ unsigned long long sl[kLimbs];
    __shared__ bool last;
    const bool skip = should_skip(c, STAGE, kSlotUpdate);
    if (STAGE != 4 && skip) return;
    if (STAGE == 4) {
        for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) sl[t] = 0ull;
        __syncthreads();
    }
    const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
    const int ld = g.ld;
    double dr2 = 0.0;
    if (!skip && i < hi) {
        double uo[4], us[4], un[4];
        const double d = dt[i];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            uo[k] = Uo[k * ld + i];
            us[k] = STAGE == 1 ? uo[k] : Us[k * ld + i];
            const double r = R[k * ld + i];
            if (STAGE == 3)
                un[k] = SUB(ADD(MUL(2.0 / 3.0, uo[k]), MUL(1.0 / 3.0, us[k])), MUL(DIV(d, 6.0), r));
            else
                un[k] = SUB(us[k], MUL(MUL(0.5, d), r));
        }
        double rho, u1, u2, p;
        const int fl = u2p(un, gamma, rho, u1, u2, p);
        if (fl) raise_err(c, STAGE, kSlotUpdate, (fl & 1) ? 10 : 11);
        double *out = STAGE == 4 ? Uo : Us;
#pragma unroll
        for (int k = 0; k < 4; k++) out[k * ld + i] = un[k];
        double qq[4];
        p2q(rho, u1, u2, p, gamma, qq);
        qstore(q, i, qq);
        if (pp.ptr) peer_push(pp, i, qq);
        if (STAGE == 4) {
            dt[i] = timestep(rho, u1, u2, p, gamma, cfl, g.dmin[i]);
            const double dr = SUB(un[0], uo[0]);
            dr2 = MUL(dr, dr);
        }
    }
    if (STAGE == 4) {
        // exact residue sum (solver.py:418-420), then the last block to
        // finish closes the iteration (residue_norm, history, convergence,
        // counters) -- no separate finalize launch
        accum_add_warp(sl, dr2);
        __syncthreads();
        for (int t = threadIdx.x; t < kLimbs; t += blockDim.x)
            if (sl[t]) atomicAdd(&c->limbs[t], sl[t]);
        if (!io.close_in_kernel) return;  // partition: all-reduce, then k_close
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(&c->blocks_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) sl[t] = atomicExch(&c->limbs[t], 0ull);
            __syncthreads();
            if (threadIdx.x == 0) close_iteration(c, sl, g.n_norm, io);
        }
    }
}

// Iteration close under a partition, after the limbs were summed across
// ranks (ncclAllReduce or the group runner): one block.
__global__ void k_close(Ctrl *c, int n_norm, IterOut io)
{
    __shared__ unsigned long long sl[kLimbs];
    for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) sl[t] = atomicExch(&c->limbs[t], 0ull);
    __syncthreads();
    if (threadIdx.x == 0) close_iteration(c, sl, n_norm, io);
}

// Halo exchange of q (multi-GPU): entry t moves component k of local slot
// slot[t] to/from buf[base[t] + k * stride[t]] (per-peer component-major
// blocks, one contiguous message per peer).
__global__ void k_halo_pack(int total, const int *__restrict__ slot, const int *__restrict__ base,
                            const int *__restrict__ stride, const double *__restrict__ q, int ld,
                            double *__restrict__ buf)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int s = slot[t], b = base[t], st = stride[t];
#pragma unroll
    for (int k = 0; k < 4; k++) buf[b + k * st] = q[4 * s + k];
}

__global__ void k_halo_unpack(int total, const int *__restrict__ slot, const int *__restrict__ base,
                              const int *__restrict__ stride, const double *__restrict__ buf, double *__restrict__ q,
                              int ld)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int s = slot[t], b = base[t], st = stride[t];
#pragma unroll
    for (int k = 0; k < 4; k++) q[4 * s + k] = buf[b + k * st];
}

// 96-bit window of the normalised digit array starting at bit p
KMF_HD unsigned long long bits64_at(const unsigned int *dg, int nd, int p)
{
    int w = p >> 5, sh = p & 31;
    unsigned long long a = (w < nd && w >= 0) ? dg[w] : 0u;
    unsigned long long b = (w + 1 < nd && w + 1 >= 0) ? dg[w + 1] : 0u;
    unsigned long long cc = (w + 2 < nd && w + 2 >= 0) ? dg[w + 2] : 0u;
    unsigned long long lo = (a >> sh) | (b << (32 - sh));
    if (sh == 0) lo = a | (b << 32);
    unsigned long long hi = sh ? (cc << (64 - sh)) : 0ull;
    return lo | hi;
}

// Correctly rounded double of the exact limb sum (math.fsum semantics).
KMF_HD double accum_round(const unsigned long long *limbs)
{
    constexpr int nd = kLimbs + 2;
    unsigned int dg[nd];
    unsigned long long carry = 0;
    for (int l = 0; l < kLimbs; l++) {
        unsigned long long t = limbs[l] + carry;
        dg[l] = (unsigned int)(t & 0xffffffffull);
        carry = t >> 32;
    }
    dg[kLimbs] = (unsigned int)(carry & 0xffffffffull);
    dg[kLimbs + 1] = (unsigned int)(carry >> 32);
    int top = -1;
    for (int l = nd - 1; l >= 0; l--)
        if (dg[l]) {
            top = l;
            break;
        }
    if (top < 0) return 0.0;
    const int T = top * 32 + (31 - __clz(dg[top]));  // MSB position, unit 2^-1074
    if (T < 53) {
        unsigned long long v = (unsigned long long)dg[0] | ((unsigned long long)dg[1] << 32);
        return scalbn((double)v, -1074);
    }
    const int lsb = T - 52;
    unsigned long long mant = bits64_at(dg, nd, lsb) & ((1ull << 53) - 1);
    const int rpos = lsb - 1;
    const unsigned long long rbit = (bits64_at(dg, nd, rpos) & 1ull);
    bool sticky = false;
    if (rpos > 0) {
        const int wfull = rpos >> 5;
        for (int l = 0; l < wfull && !sticky; l++) sticky = dg[l] != 0;
        if (!sticky) sticky = (dg[wfull] & ((1u << (rpos & 31)) - 1u)) != 0;
    }
    int e = lsb;
    if (rbit && (sticky || (mant & 1ull))) {
        mant++;
        if (mant == (1ull << 53)) {
            mant >>= 1;
            e++;
        }
    }
    return scalbn((double)mant, e - 1074);
}


// ---------------------------------------------------------------- set/get

// caller-order SoA (4, n) -> device slots; perm == nullptr: identity
__global__ void k_init(DG g, const double *__restrict__ prims, const long long *__restrict__ perm,
                       double *__restrict__ Uo, double *__restrict__ q, double *__restrict__ dt,
                       double gamma, double cfl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const long long src = perm ? perm[i] : i;
    const int n = g.n, ld = g.ld;
    const double rho = prims[src], u1 = prims[n + src], u2 = prims[2 * n + src], p = prims[3 * n + src];
    double U[4], qq[4];
    p2u(rho, u1, u2, p, gamma, U);
    p2q(rho, u1, u2, p, gamma, qq);
#pragma unroll
    for (int k = 0; k < 4; k++) Uo[k * ld + i] = U[k];
    qstore(q, i, qq);
    dt[i] = timestep(rho, u1, u2, p, gamma, cfl, g.dmin[i]);
}

// continuation of a previous run: q and dt of slots [0, hi) from the current
// U exactly as the stage-4 update produced them (decode -> p2q / timestep,
// bitwise); under a partition the halo q then comes from its owners
__global__ void k_refresh(DG g, int hi, const double *__restrict__ Uo, double *__restrict__ q,
                          double *__restrict__ dt, double gamma, double cfl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int ld = g.ld;
    double u[4], qq[4], rho, u1, u2, p;
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = Uo[k * ld + i];
    u2p(u, gamma, rho, u1, u2, p);
    p2q(rho, u1, u2, p, gamma, qq);
    qstore(q, i, qq);
    dt[i] = timestep(rho, u1, u2, p, gamma, cfl, g.dmin[i]);
}

__global__ void k_get_state(DG g, const double *__restrict__ Uo, const long long *__restrict__ perm,
                            double gamma, double *__restrict__ prims, double *__restrict__ U)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const long long dst = perm ? perm[i] : i;
    const int n = g.n, ld = g.ld;
    double u[4];
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = Uo[k * ld + i];
    double rho, u1, u2, p;
    u2p(u, gamma, rho, u1, u2, p);
    if (prims) {
        prims[dst] = rho;
        prims[n + dst] = u1;
        prims[2 * n + dst] = u2;
        prims[3 * n + dst] = p;
    }
    if (U)
#pragma unroll
        for (int k = 0; k < 4; k++) U[k * n + dst] = u[k];
}

// device slots <-> caller order for (nc, n) SoA fields
// host (nc, n) caller order <-> device slots; field k of slot i at
// dst[k * fs + i * ps] (ps = 1, fs = ld: SoA; ps = 2, fs = 2 ld: one half of
// the interleaved gradient layout)
__global__ void k_to_dev(int n, long long fs, int ps, int nc, const double *__restrict__ src,
                         const long long *__restrict__ perm, double *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long s = perm ? perm[i] : i;
    for (int k = 0; k < nc; k++) dst[k * fs + (long long)i * ps] = src[(long long)k * n + s];
}

__global__ void k_from_dev(int n, long long fs, int ps, int nc, const double *__restrict__ src,
                           const long long *__restrict__ perm, double *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long s = perm ? perm[i] : i;
    for (int k = 0; k < nc; k++) dst[(long long)k * n + s] = src[k * fs + (long long)i * ps];
}

// --------------------------------------------------------------- diagnostics

// per caller-CSR edge: bit0 q~4 >= 0 at either end, bit1 NaN q~4 at the
// neighbour end, bit2 NaN q~4 at the owner end (solver.py:164-171)
template <bool XY>
__global__ void k_diag_flux(DG g, const double *__restrict__ q, const double *__restrict__ G,
                            unsigned char *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const int ld = g.ld;
    const double xi = g.x[i], yi = g.y[i];
    const int base = ell_base(g, i), d = g.deg[i];
    const long long e0 = g.cptr[i];
    for (int s = 0; s < d; s++) {
        const int ent = base + s * 32;
        const int j = g.eidx[ent];
        double dx, dy;
        edge_offsets<XY>(g, ent, j, xi, yi, dx, dy);
        double ti = qtilde(q[4 * j + 3], gload(G, ld, 3, j).x, gload(G, ld, 3, j).y, dx, dy);
        double t0 = qtilde(q[4 * i + 3], gload(G, ld, 3, i).x, gload(G, ld, 3, i).y, dx, dy);
        unsigned char f = 0;
        if (ti >= 0.0 || t0 >= 0.0) f |= 1;
        if (isnan(ti)) f |= 2;
        if (isnan(t0)) f |= 4;
        out[e0 + s] = f;
    }
}

// per frame edge (all three families, concatenated): bit0 q~4 >= 0
__global__ void k_diag_frame(DG g, DB b, int fam, const double *__restrict__ q, const double *__restrict__ G,
                             unsigned char *__restrict__ out)
{
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= b.nb) return;
    const int ld = g.ld, pt = b.point[w];
    const double tx = b.frame[w], ty = b.frame[b.nb + w], nx = b.frame[2 * b.nb + w],
                 ny = b.frame[3 * b.nb + w];
    for (int e = b.ptr[fam][w]; e < b.ptr[fam][w + 1]; e++) {
        const int j = b.idx[fam][e];
        const double dt = b.dt[fam][e], dn = b.dn[fam][e];
        const double dxg = ADD(MUL(dt, tx), MUL(dn, nx));
        const double dyg = ADD(MUL(dt, ty), MUL(dn, ny));
        double ti = qtilde(q[4 * j + 3], gload(G, ld, 3, j).x, gload(G, ld, 3, j).y, dxg, dyg);
        double t0 = qtilde(q[4 * pt + 3], gload(G, ld, 3, pt).x, gload(G, ld, 3, pt).y, dxg, dyg);
        out[e] = (ti >= 0.0 || t0 >= 0.0) ? 1 : 0;
    }
}

// ------------------------------------------------------- point operators
// Context-free (n,) / (4,n) kernels for the stage-operator API.

__global__ void k_op_p2q(int n, const double *pr, double gamma, double *q, unsigned char *fl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
    fl[i] = !((rho > 0.0) && (p > 0.0));
    double qq[4];
    p2q(rho, u1, u2, p, gamma, qq);
    for (int k = 0; k < 4; k++) q[(long long)k * n + i] = qq[k];
}

__global__ void k_op_q2p(int n, const double *q, double gamma, double *pr, unsigned char *fl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double qq[4] = {q[i], q[n + i], q[2 * n + i], q[3 * n + i]};
    fl[i] = !(qq[3] < 0.0);
    double rho, u1, u2, p;
    q2p_ref(qq, gamma, rho, u1, u2, p);
    pr[i] = rho;
    pr[n + i] = u1;
    pr[2 * n + i] = u2;
    pr[3 * n + i] = p;
}

__global__ void k_op_p2u(int n, const double *pr, double gamma, double *U, unsigned char *fl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
    fl[i] = !((rho > 0.0) && (p > 0.0));
    double u[4];
    p2u(rho, u1, u2, p, gamma, u);
    for (int k = 0; k < 4; k++) U[(long long)k * n + i] = u[k];
}

__global__ void k_op_u2p(int n, const double *U, double gamma, double *pr, unsigned char *fl)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double u[4] = {U[i], U[n + i], U[2 * n + i], U[3 * n + i]};
    double rho, u1, u2, p;
    fl[i] = (unsigned char)u2p(u, gamma, rho, u1, u2, p);
    pr[i] = rho;
    pr[n + i] = u1;
    pr[2 * n + i] = u2;
    pr[3 * n + i] = p;
}

// kinetics.py:59-68
__global__ void k_op_full_flux(int n, const double *pr, int yaxis, double gamma, double *F)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rho = pr[i], u1 = pr[n + i], u2 = pr[2 * n + i], p = pr[3 * n + i];
    const double e = ADD(DIV(p, MUL(rho, SUB(gamma, 1.0))), MUL(0.5, ADD(MUL(u1, u1), MUL(u2, u2))));
    const double h = ADD(p, MUL(rho, e));
    double f[4];
    if (!yaxis) {
        f[0] = MUL(rho, u1);
        f[1] = ADD(p, MUL(MUL(rho, u1), u1));
        f[2] = MUL(MUL(rho, u1), u2);
        f[3] = MUL(h, u1);
    } else {
        f[0] = MUL(rho, u2);
        f[1] = MUL(MUL(rho, u1), u2);
        f[2] = ADD(p, MUL(MUL(rho, u2), u2));
        f[3] = MUL(h, u2);
    }
    for (int k = 0; k < 4; k++) F[(long long)k * n + i] = f[k];
}

__global__ void k_op_update(int n, const double *Uo, const double *Us, int stage, const double *dt,
                            const double *R, double *Un)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double d = dt[i];
    for (int k = 0; k < 4; k++) {
        const long long x = (long long)k * n + i;
        if (stage == 3)
            Un[x] = SUB(ADD(MUL(2.0 / 3.0, Uo[x]), MUL(1.0 / 3.0, Us[x])), MUL(DIV(d, 6.0), R[x]));
        else
            Un[x] = SUB(Us[x], MUL(MUL(0.5, d), R[x]));
    }
}

__global__ void k_op_residue(int n, const double *Un, const double *Uold, unsigned long long *limbs)
{
    __shared__ unsigned long long sl[kLimbs];
    for (int t = threadIdx.x; t < kLimbs; t += blockDim.x) sl[t] = 0ull;
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double d2 = 0.0;
    if (i < n) {
        const double d = SUB(Un[i], Uold[i]);
        d2 = MUL(d, d);
    }
    accum_add_warp(sl, d2);
    __syncthreads();
    for (int t = threadIdx.x; t < kLimbs; t += blockDim.x)
        if (sl[t]) atomicAdd(&limbs[t], sl[t]);
}

__global__ void k_op_residue_fin(int n, const unsigned long long *limbs, double *out)
{
    *out = sqrt(accum_round(limbs) / (double)n);
}

__global__ void k_op_timestep(DG g, const double *__restrict__ pr_dev, double cfl, double gamma,
                              double *__restrict__ dt_dev)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    const int ld = g.ld;
    dt_dev[i] = timestep(pr_dev[i], pr_dev[ld + i], pr_dev[2 * ld + i], pr_dev[3 * ld + i], gamma, cfl,
                         g.dmin[i]);
}

}  // namespace kmf

namespace kmf {
// FP64 pipe peak probe: 8 independent DFMA chains per thread.
__global__ void k_fp64_peak(int iters, double seed, double *out)
{
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = seed + k * 1e-3 + threadIdx.x * 1e-9;
    const double b = 0.999999, cc = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, cc);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace kmf


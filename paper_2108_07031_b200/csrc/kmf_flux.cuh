// kmf_flux.cuh -- flux_residual interior kernel, wall/outer closures and the
// device functions they share (perturbed-state decode, split fluxes).
//
// Per edge the two perturbed states q~_i, q~_0 (solver.py:184-185) are
// decoded ONCE and shared by the x- and the y-family split flux (the
// reference decodes them once per family); each family derivative is
// accumulated as sum_e w_f(e) * dG_f(e) in CSR order with the static weight
// w_f(e) = cx_f*dx + cy_f*dy (cx, cy = rows of the family's inverse 2x2
// matrix, solver.py:192-195).
//
// The edge body is ONE basic block, so the FP64 pipe always has independent
// work:
//   * both decodes and all four split fluxes are independent chains of an
//     unrolled M-wide loop (fsflux_m), which ptxas interleaves;
//   * the exp underflow path is a select (results below 2^-1020 flush to 0);
//   * the erf polynomial is evaluated branch-free for |s| < 1 and patched
//     afterwards by one rare, warp-voted branch for the tail (|s| >= 1);
//   * positivity is folded into a flag (a failing launch raises, its R is
//     never used); boundary owners run a separate positivity-only loop;
//   * split-axis ties (dx == 0 / dy == 0, geometry.py:544-549) are a rare
//     branch after the main body.
// Every value is produced by the same explicit operations whatever the
// family selection, so fused (FAM < 0) and split4 (FAM = 0..3, R
// accumulated x+, x-, y+, y-) stay bitwise equal (tests/test_gpu_parity.py).
#pragma once
#include "kmf_kernels.cuh"

namespace kmf {

// state.py:141-163 q_to_primitives restated for the FP64 pipe, plus the
// per-state constants of the split-flux moment algebra (kinetics.py:53-56,
// :85-106): beta = -q4/2, r = 1/(2 beta) = -1/q4, u = q r, rho = exp(...).
// GK selects the beta^(-1/(gamma-1)) evaluation: 1 -> gamma = 7/5
// (beta^-2.5 = (2r)^2 rsqrt(beta)), 2 -> gamma = 5/3 (beta^-1.5 = 2r
// rsqrt(beta)), 0 -> any gamma via log/exp.  T = the staged exp table.
template <int GK>
KMF_HD void fdecode(double q1, double q2, double q3, double q4, double inv_gm1, double c_i0, FState &s,
                    const double2 *T)
{
    const double beta = -0.5 * q4;
    s.r = frcp(-q4);
    s.u1 = q2 * s.r;
    s.u2 = q3 * s.r;
    const double rsb = frsqrt(beta);
    s.sb = beta * rsb;
    s.bc = rsb * kInv2SqrtPi;
    s.i0 = c_i0 * s.r;
    const double uu = fma(s.u1, s.u1, s.u2 * s.u2);
    if (GK == 1) {
        const double r2 = 2.0 * s.r;
        s.rho = fexp_tab(fma(beta, uu, q1), T) * (r2 * r2 * rsb);
    } else if (GK == 2) {
        s.rho = fexp_tab(fma(beta, uu, q1), T) * (2.0 * s.r * rsb);
    } else {
        s.rho = fexp_tab(fma(beta, uu, fma(-log(beta), inv_gm1, q1)), T);
    }
    s.rho_h = 0.5 * s.rho;
    s.c2 = fma(2.0, s.i0, s.r);
    s.r3 = 3.0 * s.r;
}

// The same constants from primitives (kinetics.py:85: split_flux recomputes
// beta = rho / (2 p) from the decoded primitives) -- the split_flux operator
// and the free-stream Maxwellian of the outer closure.
KMF_HD void fstate_prims(double rho, double u1, double u2, double p, double c_i0, FState &s)
{
    const double beta = rho / (2.0 * p);
    const double rsb = frsqrt(beta);
    s.rho = rho;
    s.u1 = u1;
    s.u2 = u2;
    s.r = 1.0 / (2.0 * beta);
    s.sb = beta * rsb;
    s.bc = rsb * kInv2SqrtPi;
    s.i0 = c_i0 * s.r;
    s.rho_h = 0.5 * s.rho;
    s.c2 = fma(2.0, s.i0, s.r);
    s.r3 = 3.0 * s.r;
}

// kinetics.py:71-106: M split fluxes of decoded states st[m] along axis Y[m]
// (compile-time per m through the caller's unrolled loops) with half range
// sg[m] = +-1, in lock step.  Output rows in the caller's axis order:
// x -> [rho m1, rho m2, rho m1 ut, E], y -> [rho m1, rho m1 ut, rho m2, E].
template <int M>
KMF_HD void fsflux_m(const FState *const (&st)[M], const bool (&Y)[M], const double (&sg)[M], double (&G)[M][4],
                     const double2 *T)
{
    double un[M], sarg[M], e2[M], E[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        un[m] = Y[m] ? st[m]->u2 : st[m]->u1;
        sarg[m] = un[m] * st[m]->sb;
    }
#pragma unroll
    for (int m = 0; m < M; m++) e2[m] = fexp_tab<false>(-(sarg[m] * sarg[m]), T);
    bool tail = false;
#pragma unroll
    for (int m = 0; m < M; m++) {
        E[m] = sarg[m] * horner(kErfP, sarg[m] * sarg[m]);
        tail |= !(fabs(sarg[m]) < 1.0);
    }
    if (tail) {  // |s| >= 1: supersonic normal speed ratio, rare
#pragma unroll
        for (int m = 0; m < M; m++)
            if (!(fabs(sarg[m]) < 1.0)) E[m] = ferf_tail(sarg[m], e2[m]);
    }
#pragma unroll
    for (int m = 0; m < M; m++) {
        const FState &s = *st[m];
        const double ut = Y[m] ? s.u1 : s.u2;
        // A = (1 + sg erf s) / 2 as ONE fma: scaling by 1/2 is exact, so
        // fma(+-1/2, E, 1/2) rounds to exactly 0.5 * fma(sg, E, 1)
        const double A = fma(copysign(0.5, sg[m]), E[m], 0.5);
        const double B = e2[m] * s.bc;
        const double sgB = copysign(B, sg[m]);  // sg = +-1 as a sign flip (ALU, not the FP64 pipe)
        const double unsq = un[m] * un[m];
        const double m1 = fma(un[m], A, sgB);
        const double m2 = fma(unsq + s.r, A, un[m] * sgB);
        const double m3 = fma(fma(unsq, un[m], un[m] * s.r3), A, fma(2.0, s.r, unsq) * sgB);
        // E = rho ((ut^2/2 + r/2 + I0) m1 + m3/2) with the 0.5 factors folded
        // into the per-state constants: (rho/2) ((ut^2 + r + 2 I0) m1 + m3)
        const double energy = s.rho_h * fma(fma(ut, ut, s.c2), m1, m3);
        const double rm1 = s.rho * m1;
        const double rm2 = s.rho * m2;
        G[m][0] = rm1;
        G[m][1] = Y[m] ? rm1 * ut : rm2;
        G[m][2] = Y[m] ? rm2 : rm1 * ut;
        G[m][3] = energy;
    }
}

// solver.py:162-235 interior rows of the points [lo, hi); FAM < 0 fused,
// 0..3 one split family.  XY (offsets recomputed from coordinates): the
// next edge's gathers (x, y, q, qx, qy of the neighbour) are issued into
// registers while the current edge is evaluated, its index one edge earlier
// still -- the HBM/L2 round trip overlaps ~700 issue cycles of edge
// arithmetic.  The owner's q and gradients are re-read from L1 per edge
// through a laundered index the compiler cannot hoist (pinning them would
// cost 40 registers of an occupancy-bound kernel).  Perturbed states: FMA-
// contracted for q1..q3 (tolerance path, <= 1 ulp each); q4 stays bitwise
// (solver.py:184-185) because its sign IS the reference's positivity test.
template <bool XY, int FAM, int GK>
__global__ void __launch_bounds__(kTB, 3) k_flux(DG g, int lo, int hi, const double *__restrict__ q,
                                                 const double *__restrict__ G, double *__restrict__ R,
                                                 double inv_gm1, double c_i0, int zero_boundary, Ctrl *c, int stage)
{
    __shared__ double2 sT[64];
    stage_exp_table(sT);
    const double2 *T = sT;
    const int i = range_base(lo) + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < lo || i >= hi) return;
    if (c && should_skip(c, stage, kSlotFlux)) return;
    const int ld = g.ld;
    const bool interior = g.flag[i] == 0;
    const double xi = g.x[i], yi = g.y[i];
    const int base = ell_base(g, i), d = g.deg[i];
    bool bad = false;

    if (!interior) {
        // boundary owners: rows are zeroed (solver.py:233-234) but their
        // family edges are still decoded by the reference -> positivity only
        for (int s = 0; s < d; s++) {
            const int ent = base + s * 32;
            const int j = g.eidx[ent];
            double dx, dy;
            edge_offsets<XY>(g, ent, j, xi, yi, dx, dy);
            if (FAM == 0 && !(dx <= 0.0)) continue;
            if (FAM == 1 && !(dx >= 0.0)) continue;
            if (FAM == 2 && !(dy <= 0.0)) continue;
            if (FAM == 3 && !(dy >= 0.0)) continue;
            const double ti = qtilde(q[4 * j + 3], gload(G, ld, 3, j).x, gload(G, ld, 3, j).y, dx, dy);
            const double t0 = qtilde(q[4 * i + 3], gload(G, ld, 3, i).x, gload(G, ld, 3, i).y, dx, dy);
            bad |= !(ti < 0.0) || !(t0 < 0.0);
        }
        if (bad && c) raise_err(c, stage, kSlotFlux, 2);
        if (zero_boundary && FAM <= 0) {
#pragma unroll
            for (int k = 0; k < 4; k++) R[k * ld + i] = 0.0;
        }
        return;
    }

    double acc[4][4];
#pragma unroll
    for (int f = 0; f < 4; f++)
#pragma unroll
        for (int k = 0; k < 4; k++) acc[f][k] = 0.0;

    double nX = 0.0, nY = 0.0, nQ[4] = {}, nGX[4] = {}, nGY[4] = {};
    auto gat = [&](int j) {
        const double2 pj = g.pxy[j];
        nX = pj.x;
        nY = pj.y;
        const Q4 r = qload(q, j);
#pragma unroll
        for (int k = 0; k < 4; k++) nQ[k] = r.v[k];
        gload_nc<4>(G, ld, j, 0, nGX, nGY);
    };
    if (XY && d > 0) gat(g.eidx[base]);
    int j_nx = (XY && d > 1) ? g.eidx[base + 32] : 0;
    for (int s = 0; s < d; s++) {
        const int ent = base + s * 32;
        const int j = XY ? 0 : g.eidx[ent];
        double cQ[4], cGX[4], cGY[4];
        double dx, dy;
        if (XY) {
            dx = SUB(nX, xi);  // geometry.py:382-383, bitwise
            dy = SUB(nY, yi);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                cQ[k] = nQ[k];
                cGX[k] = nGX[k];
                cGY[k] = nGY[k];
            }
            gat(j_nx);  // past the last edge: a redundant gather of a loaded point
            if (s + 2 < d) j_nx = g.eidx[base + (s + 2) * 32];
        } else {
            edge_offsets<XY>(g, ent, j, xi, yi, dx, dy);
            const Q4 r = qload(q, j);
            gload_nc<4>(G, ld, j, 0, cGX, cGY);
#pragma unroll
            for (int k = 0; k < 4; k++) cQ[k] = r.v[k];
        }
        if (FAM == 0 && !(dx <= 0.0)) continue;
        if (FAM == 1 && !(dx >= 0.0)) continue;
        if (FAM == 2 && !(dy <= 0.0)) continue;
        if (FAM == 3 && !(dy >= 0.0)) continue;
        int io;
        asm volatile("mov.b32 %0, %1;" : "=r"(io) : "r"(i));
        double ti[4], t0[4];
        const double hdx = 0.5 * dx, hdy = 0.5 * dy;
        const Q4 qo = qload(q, io);
        double ogx[4], ogy[4];
        gload_nc<4>(G, ld, io, 0, ogx, ogy);
#pragma unroll
        for (int k = 0; k < 3; k++) {
            ti[k] = fma(-hdx, cGX[k], fma(-hdy, cGY[k], cQ[k]));
            t0[k] = fma(-hdx, ogx[k], fma(-hdy, ogy[k], qo.v[k]));
        }
        ti[3] = qtilde(cQ[3], cGX[3], cGY[3], dx, dy);
        t0[3] = qtilde(qo.v[3], ogx[3], ogy[3], dx, dy);
        bad |= !(ti[3] < 0.0) || !(t0[3] < 0.0);  // solver.py:164 (NaN caught too)
        FState si, s0;
        fdecode<GK>(ti[0], ti[1], ti[2], ti[3], inv_gm1, c_i0, si, T);
        fdecode<GK>(t0[0], t0[1], t0[2], t0[3], inv_gm1, c_i0, s0, T);
        const double *cf = g.fcoef + io;  // cf[k * ld]: (cx, cy) of x+, x-, y+, y-
        const bool px = dx <= 0.0, py = dy <= 0.0;
        if (FAM < 0) {
            const FState *st[4] = {&si, &s0, &si, &s0};
            const bool Y[4] = {false, false, true, true};
            const double sgx = px ? 1.0 : -1.0, sgy = py ? 1.0 : -1.0;
            const double sg[4] = {sgx, sgx, sgy, sgy};
            double F[4][4];
            fsflux_m<4>(st, Y, sg, F, T);
            const double wx = fma(cf[(px ? 0 : 2) * ld], dx, cf[(px ? 1 : 3) * ld] * dy);
            const double wy = fma(cf[(py ? 4 : 6) * ld], dx, cf[(py ? 5 : 7) * ld] * dy);
            // both families of an axis take an FMA, the one the edge is not
            // in with weight 0 (adds +-0: value-identical sums): 2 DFMA
            // instead of 1 DFMA + 6 FSEL per component and axis
            const double wxp = px ? wx : 0.0, wxm = px ? 0.0 : wx;
            const double wyp = py ? wy : 0.0, wym = py ? 0.0 : wy;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const double gx = F[0][k] - F[1][k], gy = F[2][k] - F[3][k];
                acc[0][k] = fma(wxp, gx, acc[0][k]);
                acc[1][k] = fma(wxm, gx, acc[1][k]);
                acc[2][k] = fma(wyp, gy, acc[2][k]);
                acc[3][k] = fma(wym, gy, acc[3][k]);
            }
            if (dx == 0.0 || dy == 0.0) {  // ties: the edge is in both families of the axis
                const bool tx = dx == 0.0;
                const FState *st2[2] = {&si, &s0};
                const bool Y2[2] = {!tx, !tx};
                const double sg2[2] = {-1.0, -1.0};
                double F2[2][4];
                fsflux_m<2>(st2, Y2, sg2, F2, T);
                const double w2 = tx ? fma(cf[2 * ld], dx, cf[3 * ld] * dy) : fma(cf[6 * ld], dx, cf[7 * ld] * dy);
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const double a = fma(w2, F2[0][k] - F2[1][k], tx ? acc[1][k] : acc[3][k]);
                    if (tx)
                        acc[1][k] = a;
                    else
                        acc[3][k] = a;
                }
                if (tx && dy == 0.0) {  // both ties (coincident points cannot occur; kept exact)
                    const bool Y3[2] = {true, true};
                    fsflux_m<2>(st2, Y3, sg2, F2, T);
                    const double w3 = fma(cf[6 * ld], dx, cf[7 * ld] * dy);
#pragma unroll
                    for (int k = 0; k < 4; k++) acc[3][k] = fma(w3, F2[0][k] - F2[1][k], acc[3][k]);
                }
            }
        } else {
            const FState *st[2] = {&si, &s0};
            const bool Y[2] = {FAM >= 2, FAM >= 2};
            const double sgv = (FAM == 0 || FAM == 2) ? 1.0 : -1.0;
            const double sg[2] = {sgv, sgv};
            double F[2][4];
            fsflux_m<2>(st, Y, sg, F, T);
            const double w = fma(cf[(2 * FAM) * ld], dx, cf[(2 * FAM + 1) * ld] * dy);
#pragma unroll
            for (int k = 0; k < 4; k++) acc[FAM][k] = fma(w, F[0][k] - F[1][k], acc[FAM][k]);
        }
    }
    if (bad && c) raise_err(c, stage, kSlotFlux, 2 /*KMF_CTX_FLUX_XP: refined on host*/);
#pragma unroll
    for (int k = 0; k < 4; k++) {
        double r;
        if (FAM < 0)
            r = ADD(ADD(ADD(acc[0][k], acc[1][k]), acc[2][k]), acc[3][k]);
        else if (FAM == 0)
            r = acc[0][k];
        else
            r = ADD(R[k * ld + i], acc[FAM][k]);
        R[k * ld + i] = r;
    }
}

// ---------------------------------------------------------------------------
// solver.py:336-382 apply_boundary: wall / outer frame closures.  One warp
// per boundary point; lanes stride over the frame edges of tplus, tminus
// and the one-sided normal family; warp-tree sums (tolerance path).  The
// perturbed states, decode and split fluxes are the interior kernel's
// device functions.
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int GK>
__global__ void __launch_bounds__(kTB) k_boundary(DG g, DB b, const double *__restrict__ q,
                                                  const double *__restrict__ G, double *__restrict__ R,
                                                  double inv_gm1, double c_i0, double fsr, double fsu,
                                                  double fsv, double fsp, Ctrl *c, int stage)
{
    __shared__ double2 sT[64];
    stage_exp_table(sT);
    const double2 *T = sT;
    if (c && should_skip(c, stage, kSlotFlux)) return;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= b.nb) return;  // whole warp leaves together
    const int ld = g.ld;
    const int pt = b.point[w];
    const bool wall = b.type[w] == 1;
    const double tx = b.frame[w], ty = b.frame[b.nb + w], nx = b.frame[2 * b.nb + w],
                 ny = b.frame[3 * b.nb + w];
    double qi[4], gxi[4], gyi[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        qi[k] = q[4 * pt + k];
        gxi[k] = gload(G, ld, k, pt).x;
        gyi[k] = gload(G, ld, k, pt).y;
    }
    // free-stream Maxwellian in this point's frame (solver.py:365-369)
    double gfs[4] = {0, 0, 0, 0};
    if (!wall) {
        FState fs;
        fstate_prims(fsr, ADD(MUL(fsu, tx), MUL(fsv, ty)), ADD(MUL(fsu, nx), MUL(fsv, ny)), fsp, c_i0, fs);
        const FState *st[1] = {&fs};
        const bool Y[1] = {true};
        const double sg[1] = {-1.0};
        double F[1][4];
        fsflux_m<1>(st, Y, sg, F, T);
#pragma unroll
        for (int k = 0; k < 4; k++) gfs[k] = F[0][k];
    }
    double acc[3][4];
#pragma unroll
    for (int f = 0; f < 3; f++)
#pragma unroll
        for (int k = 0; k < 4; k++) acc[f][k] = 0.0;
    unsigned badmask = 0;
#pragma unroll 1
    for (int f = 0; f < 3; f++) {
        const int e0 = b.ptr[f][w], e1 = b.ptr[f][w + 1];
        const double ct = b.coef[(2 * f) * b.nb + w], cn = b.coef[(2 * f + 1) * b.nb + w];
        for (int e = e0 + lane; e < e1; e += 32) {
            const int j = b.idx[f][e];
            const double dt = b.dt[f][e], dn = b.dn[f][e];
            // solver.py:255-256 global offsets rebuilt from the rotated ones
            const double dxg = ADD(MUL(dt, tx), MUL(dn, nx));
            const double dyg = ADD(MUL(dt, ty), MUL(dn, ny));
            double ti[4], t0[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                ti[k] = qtilde(q[4 * j + k], gload(G, ld, k, j).x, gload(G, ld, k, j).y, dxg, dyg);
                t0[k] = qtilde(qi[k], gxi[k], gyi[k], dxg, dyg);
            }
            if (!(ti[3] < 0.0) || !(t0[3] < 0.0)) {
                badmask |= 1u << f;
                continue;
            }
            // _frame_q (solver.py:238-242): rotate the velocity pair
            FState si, s0;
            fdecode<GK>(ti[0], ADD(MUL(tx, ti[1]), MUL(ty, ti[2])), ADD(MUL(nx, ti[1]), MUL(ny, ti[2])), ti[3],
                        inv_gm1, c_i0, si, T);
            fdecode<GK>(t0[0], ADD(MUL(tx, t0[1]), MUL(ty, t0[2])), ADD(MUL(nx, t0[1]), MUL(ny, t0[2])), t0[3],
                        inv_gm1, c_i0, s0, T);
            double dg[4];
            if (f < 2) {  // tangent: G_x(+/-) in the frame
                const FState *st[2] = {&si, &s0};
                const bool Y[2] = {false, false};
                const double sgv = f == 0 ? 1.0 : -1.0;
                const double sg[2] = {sgv, sgv};
                double F[2][4];
                fsflux_m<2>(st, Y, sg, F, T);
#pragma unroll
                for (int k = 0; k < 4; k++) dg[k] = F[0][k] - F[1][k];
            } else if (wall) {  // wall normal: G_y-
                const FState *st[2] = {&si, &s0};
                const bool Y[2] = {true, true};
                const double sg[2] = {-1.0, -1.0};
                double F[2][4];
                fsflux_m<2>(st, Y, sg, F, T);
#pragma unroll
                for (int k = 0; k < 4; k++) dg[k] = F[0][k] - F[1][k];
            } else {  // outer normal: (G_y+(q~_i) - G_y+(q~_0)) + (G_y-(q~_i) - G_y-(free stream))
                const FState *st[3] = {&si, &s0, &si};
                const bool Y[3] = {true, true, true};
                const double sg[3] = {1.0, 1.0, -1.0};
                double F[3][4];
                fsflux_m<3>(st, Y, sg, F, T);
#pragma unroll
                for (int k = 0; k < 4; k++) dg[k] = (F[0][k] - F[1][k]) + (F[2][k] - gfs[k]);
            }
            const double wgt = fma(ct, dt, cn * dn);
#pragma unroll
            for (int k = 0; k < 4; k++) acc[f][k] = fma(wgt, dg[k], acc[f][k]);
        }
    }
#pragma unroll
    for (int f = 0; f < 3; f++)
#pragma unroll
        for (int k = 0; k < 4; k++) acc[f][k] = warp_sum(acc[f][k]);
    unsigned anybad = __reduce_or_sync(0xffffffffu, badmask);
    if (lane == 0) {
        if (anybad && c) {
            if (anybad & 3u) raise_err(c, stage, kSlotFlux, wall ? 6 : 8);
            if (anybad & 4u) raise_err(c, stage, kSlotFlux, wall ? 7 : 9);
        }
        double rows[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            double rt = acc[0][k] + acc[1][k];
            if (wall)
                rows[k] = rt + (k == 2 ? 0.0 : 2.0 * acc[2][k]);  // solver.py:303-309
            else
                rows[k] = rt + acc[2][k];  // solver.py:322-333
        }
        // _rotate_back solver.py:376-382
        R[pt] = rows[0];
        R[3 * ld + pt] = rows[3];
        R[ld + pt] = ADD(MUL(tx, rows[1]), MUL(nx, rows[2]));
        R[2 * ld + pt] = ADD(MUL(ty, rows[1]), MUL(ny, rows[2]));
    }
}

// ------------------------------------------------------------ operator API

// kinetics.py:71-106 split_flux through the flux kernel's own device
// function (fsflux_m) on the state constants the reference recomputes
// from the primitives (beta = rho / (2 p), kinetics.py:85)
__global__ void k_op_split_flux(int n, const double *pr, int yaxis, double sg, double c_i0, double *Gout)
{
    __shared__ double2 sT[64];
    stage_exp_table(sT);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    FState s;
    fstate_prims(pr[i], pr[n + i], pr[2 * n + i], pr[3 * n + i], c_i0, s);
    const FState *st[1] = {&s};
    const bool Y[1] = {yaxis != 0};
    const double sgv[1] = {sg};
    double F[1][4];
    fsflux_m<1>(st, Y, sgv, F, sT);
    for (int k = 0; k < 4; k++) Gout[(long long)k * n + i] = F[0][k];
}

// The flux kernel's edge-state path on given q vectors (test probe): the
// decode (fdecode<GK>) and the four split fluxes x+, x-, y+, y- (fsflux_m<4>)
// exactly as the interior kernel evaluates them.  prims (4, n): rho, u1, u2,
// p = rho r; flux (16, n): family f rows 4 f .. 4 f + 3.
template <int GK>
__global__ void k_probe_edge_state(int n, const double *qv, double inv_gm1, double c_i0, double *prims, double *flux)
{
    __shared__ double2 sT[64];
    stage_exp_table(sT);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    FState s;
    fdecode<GK>(qv[i], qv[n + i], qv[2 * n + i], qv[3 * n + i], inv_gm1, c_i0, s, sT);
    prims[i] = s.rho;
    prims[n + i] = s.u1;
    prims[2 * n + i] = s.u2;
    prims[3 * n + i] = s.rho * s.r;
    const FState *st[4] = {&s, &s, &s, &s};
    const bool Y[4] = {false, false, true, true};
    const double sg[4] = {1.0, -1.0, 1.0, -1.0};
    double F[4][4];
    fsflux_m<4>(st, Y, sg, F, sT);
    for (int f = 0; f < 4; f++)
        for (int k = 0; k < 4; k++) flux[(long long)(4 * f + k) * n + i] = F[f][k];
}

// accuracy probe of the flux-path transcendentals (tests/test_gpu_fastmath.py)
__global__ void k_fastmath_probe(int n, const double *x, int which, double *out)
{
    __shared__ double2 sT[64];
    stage_exp_table(sT);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    double r;
    switch (which) {
    case 0:
    case 4: r = fexp_tab(v, sT); break;
    case 1: r = ferf(v, fexp_tab<false>(-(v * v), sT)); break;
    case 2: r = frcp(v); break;
    case 5: r = fexp_tab<false>(v, sT); break;
    default: r = frsqrt(v); break;
    }
    out[i] = r;
}

}  // namespace kmf

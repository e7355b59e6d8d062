// kmf_qgrad2.cuh -- q-gradient kernels with a straight-line slot body.
//
// Same bitwise contract as k_first_order / k_sweep (lsq.py:164-175,
// 214-227): each least-squares sum is a sequential fp64 sum in CSR slot
// order with products rounded before the add.
//
// k_first_order / k_sweep walk the slots in a runtime loop, so every slot
// costs two dependent round trips (index, then gathers) that the warp must
// wait out before the next slot starts: the kernels are gather-latency
// bound (ncu: long-scoreboard stalls, FP64 pipe ~43 % busy).  Here the
// first MAXD slots are one basic block: slot indices are clamped to the
// point's last slot (so every load is unconditional and safe), the loads
// of all slots are free to be issued ahead of the arithmetic, and slots
// past the point's degree are masked out of the sums by a select (the
// accumulator is left untouched, so the sum is bit-identical).  Slots
// beyond MAXD (widened stencils, geometry.py:491-501) run a plain loop.
#pragma once
#include "kmf_kernels.cuh"

namespace kmf {

template <bool XY, bool SWEEP, int NC>
KMF_HD void qg_slot(const DG &g, const double *__restrict__ q, const double *__restrict__ Gin, int ent, int j,
                    double xi, double yi, int k0, const double (&qi)[NC], const double (&gxi)[NC],
                    const double (&gyi)[NC], bool live, double (&sx)[NC], double (&sy)[NC])
{
    const int ld = g.ld;
    double dx, dy;
    edge_offsets<XY>(g, ent, j, xi, yi, dx, dy);
#pragma unroll
    for (int k = 0; k < NC; k++) {
        double dq;
        if (SWEEP) {
            const double ti = qtilde(q[(k0 + k) * ld + j], Gin[(k0 + k) * ld + j], Gin[(4 + k0 + k) * ld + j], dx, dy);
            const double t0 = qtilde(qi[k], gxi[k], gyi[k], dx, dy);
            dq = SUB(ti, t0);
        } else {
            dq = SUB(q[(k0 + k) * ld + j], qi[k]);
        }
        const double ax = ADD(sx[k], MUL(dx, dq));
        const double ay = ADD(sy[k], MUL(dy, dq));
        sx[k] = live ? ax : sx[k];
        sy[k] = live ? ay : sy[k];
    }
}

// SWEEP = false: lsq.py:164-175 first order; true: one Jacobi sweep
// (lsq.py:214-227) with the max-update diagnostic when want_res.
template <bool XY, bool SWEEP, int NC, int MAXD, int MINB>
__global__ void __launch_bounds__(kTB, MINB) k_qgrad2(DG g, const double *__restrict__ q,
                                                      const double *__restrict__ Gin, double *__restrict__ Gout,
                                                      Ctrl *c, int stage, int slot, int want_res)
{
    if (c && should_skip(c, stage, slot)) return;
    int i, k0;
    qg_thread<NC>(i, k0);
    double rmax = 0.0;
    if (i < g.n) {
        const int ld = g.ld;
        double qi[NC], gxi[NC], gyi[NC], sx[NC], sy[NC];
#pragma unroll
        for (int k = 0; k < NC; k++) {
            qi[k] = q[(k0 + k) * ld + i];
            gxi[k] = SWEEP ? Gin[(k0 + k) * ld + i] : 0.0;
            gyi[k] = SWEEP ? Gin[(4 + k0 + k) * ld + i] : 0.0;
            sx[k] = 0.0;
            sy[k] = 0.0;
        }
        const double xi = g.x[i], yi = g.y[i];
        const int base = ell_base(g, i), d = g.deg[i];
        if (d > 0) {  // halo points past a partition's depth have no slots at all
#pragma unroll
            for (int s = 0; s < MAXD; s++) {
                const int ent = base + min(s, d - 1) * 32;
                qg_slot<XY, SWEEP, NC>(g, q, Gin, ent, g.eidx[ent], xi, yi, k0, qi, gxi, gyi, s < d, sx, sy);
            }
        }
        for (int s = MAXD; s < d; s++) {
            const int ent = base + s * 32;
            qg_slot<XY, SWEEP, NC>(g, q, Gin, ent, g.eidx[ent], xi, yi, k0, qi, gxi, gyi, true, sx, sy);
        }
        const double sxx = g.fsum[i], sxy = g.fsum[ld + i], syy = g.fsum[2 * ld + i], det = g.fsum[3 * ld + i];
#pragma unroll
        for (int k = 0; k < NC; k++) {
            const double nx_ = DIV(SUB(MUL(syy, sx[k]), MUL(sxy, sy[k])), det);
            const double ny_ = DIV(SUB(MUL(sxx, sy[k]), MUL(sxy, sx[k])), det);
            Gout[(k0 + k) * ld + i] = nx_;
            Gout[(4 + k0 + k) * ld + i] = ny_;
            if (SWEEP && want_res) {
                rmax = fmax(rmax, fabs(nx_ - gxi[k]));
                rmax = fmax(rmax, fabs(ny_ - gyi[k]));
                if (isnan(nx_ - gxi[k]) || isnan(ny_ - gyi[k])) rmax = __longlong_as_double(0x7ff8000000000000ll);
            }
        }
    }
    if (SWEEP && want_res) {
        unsigned long long b = (unsigned long long)__double_as_longlong(rmax);
        for (int o = 16; o; o >>= 1) {
            unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
            b = t > b ? t : b;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&c->resmax, b);
    }
}

}  // namespace kmf

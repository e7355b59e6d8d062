// kmf_math.cuh -- device arithmetic of the q-LSKUM hot path (sm_100a, fp64).
//
// Two kinds of arithmetic live here:
//
//  * BITWISE paths (state transforms, q-gradients, state update, time step,
//    residue): every +,-,*,/ is an explicit round-to-nearest intrinsic so no
//    FMA contraction can happen, and the operation order mirrors numpy's
//    left-to-right evaluation of the reference source.  With identical
//    inputs these reproduce the reference bit for bit.
//
//  * TOLERANCE paths (perturbed-state decode and kinetic split fluxes inside
//    flux_residual / apply_boundary): algebraically identical to the
//    reference but re-associated for the FP64 pipe (reciprocal instead of
//    three divisions, shared sqrt/rsqrt, explicit fma).  Deviation is a few
//    ulp per flux value; the contract is
//    |dR| <= 1e-11 * max(max|R_row|, 1) per call.
//
// The library is compiled with -fmad=false, so any fma() below is one the
// source asked for explicitly; fused and split4 flux modes therefore share
// bit-identical per-edge arithmetic.
#pragma once
#include <cstdint>

#define KMF_HD __device__ __forceinline__

// exact ops (never contracted)
#define MUL(a, b) __dmul_rn((a), (b))
#define ADD(a, b) __dadd_rn((a), (b))
#define SUB(a, b) __dsub_rn((a), (b))
#define DIV(a, b) __ddiv_rn((a), (b))

namespace kmf {

constexpr double kPi = 3.141592653589793;
constexpr double kInv2SqrtPi = 0.28209479177387814;  // 1/(2 sqrt(pi))

// ---------------------------------------------------------------- bitwise

// state.py:91-96 primitives_to_conserved
KMF_HD void p2u(double rho, double u1, double u2, double p, double gamma, double U[4])
{
    double e = ADD(DIV(p, MUL(rho, SUB(gamma, 1.0))), MUL(0.5, ADD(MUL(u1, u1), MUL(u2, u2))));
    U[0] = rho;
    U[1] = MUL(rho, u1);
    U[2] = MUL(rho, u2);
    U[3] = MUL(rho, e);
}

// state.py:99-129 conserved_to_primitives; returns bit0 density, bit1 pressure
KMF_HD int u2p(const double U[4], double gamma, double &rho, double &u1, double &u2, double &p)
{
    rho = U[0];
    u1 = DIV(U[1], rho);
    u2 = DIV(U[2], rho);
    p = MUL(SUB(gamma, 1.0), SUB(U[3], MUL(MUL(0.5, rho), ADD(MUL(u1, u1), MUL(u2, u2)))));
    int f = 0;
    if (!(rho > 0.0)) f |= 1;
    if (!(p > 0.0)) f |= 2;
    return f;
}

// state.py:132-138 primitives_to_q (log from libdevice: <= 1 ulp vs numpy)
KMF_HD void p2q(double rho, double u1, double u2, double p, double gamma, double q[4])
{
    double beta = DIV(rho, MUL(2.0, p));
    double uu = ADD(MUL(u1, u1), MUL(u2, u2));
    q[0] = SUB(ADD(log(rho), DIV(log(beta), SUB(gamma, 1.0))), MUL(beta, uu));
    double b2 = MUL(2.0, beta);
    q[1] = MUL(b2, u1);
    q[2] = MUL(b2, u2);
    q[3] = MUL(-2.0, beta);
}

// state.py:141-163 q_to_primitives, reference-shaped (used by the op API)
KMF_HD void q2p_ref(const double q[4], double gamma, double &rho, double &u1, double &u2, double &p)
{
    double beta = MUL(-0.5, q[3]);
    double b2 = MUL(2.0, beta);
    u1 = DIV(q[1], b2);
    u2 = DIV(q[2], b2);
    rho = exp(ADD(SUB(q[0], DIV(log(beta), SUB(gamma, 1.0))), MUL(beta, ADD(MUL(u1, u1), MUL(u2, u2)))));
    p = DIV(rho, b2);
}

// solver.py:154-159 local_timestep: (cfl*d_min) / (|u| + a)
KMF_HD double timestep(double rho, double u1, double u2, double p, double gamma, double cfl, double dmin)
{
    double speed = ADD(sqrt(ADD(MUL(u1, u1), MUL(u2, u2))), sqrt(DIV(MUL(gamma, p), rho)));
    return DIV(MUL(cfl, dmin), speed);
}

// solver.py:184-185 / lsq.py:219-220 perturbed value q - 0.5*(dx*gx + dy*gy)
KMF_HD double qtilde(double q, double gx, double gy, double dx, double dy)
{
    return SUB(q, MUL(0.5, ADD(MUL(dx, gx), MUL(dy, gy))));
}

// The same value from pre-halved offsets hdx = 0.5*dx, hdy = 0.5*dy (shared
// by all components of an edge): scaling by 0.5 commutes with round-to-
// nearest as long as no intermediate drops below 2^-1021 (|dx*gx| far from
// subnormal here), so RN(hdx*gx) + RN(hdy*gy) rounds to exactly
// 0.5*RN(RN(dx*gx) + RN(dy*gy)): bit-identical with one multiply fewer on
// the dependency chain.
KMF_HD double qtilde_h(double q, double gx, double gy, double hdx, double hdy)
{
    return SUB(q, ADD(MUL(hdx, gx), MUL(hdy, gy)));
}

// ------------------------------------------------------------- tolerance

// Decoded perturbed edge state (state.py:141-163 restated for the FP64
// pipe): beta = -q4/2, r = 1/(2 beta) = -1/q4, u = q*r, rho = exp(...).
struct EState {
    double rho, u1, u2, beta, r;
};

KMF_HD void decode(double q1, double q2, double q3, double q4, double inv_gm1, EState &s)
{
    s.beta = -0.5 * q4;
    s.r = __drcp_rn(-q4);
    s.u1 = q2 * s.r;
    s.u2 = q3 * s.r;
    double uu = fma(s.u1, s.u1, s.u2 * s.u2);
    s.rho = exp(fma(s.beta, uu, fma(-log(s.beta), inv_gm1, q1)));
}

// Per-state quantities shared by every split flux of that state.
struct EShared {
    double sb;  // sqrt(beta)
    double bc;  // 1/(2 sqrt(pi beta))
    double i0;  // (2-gamma)/(2 beta (gamma-1))  kinetics.py:53-56
};

KMF_HD void shared_of(const EState &s, double c_i0, EShared &h)
{
    h.sb = sqrt(s.beta);
    h.bc = rsqrt(s.beta) * kInv2SqrtPi;
    h.i0 = c_i0 * s.r;
}

// kinetics.py:71-106 split_flux for one state.  yaxis selects G_y (normal
// velocity u2), sg = +1 / -1 the half range.  Rows: x -> [rho m1, rho m2,
// rho m1 ut, E], y -> [rho m1, rho m1 ut, rho m2, E].
KMF_HD void sflux(const EState &s, const EShared &h, bool yaxis, double sg, double G[4])
{
    const double un = yaxis ? s.u2 : s.u1;
    const double ut = yaxis ? s.u1 : s.u2;
    const double r = s.r;  // 1/(2 beta)
    double sarg = un * h.sb;
    double E = erf(sarg);
    double A = 0.5 * fma(sg, E, 1.0);
    double B = exp(-(sarg * sarg)) * h.bc;
    double sgB = sg * B;
    double unsq = un * un;
    double m1 = fma(un, A, sgB);
    double m2 = fma(unsq + r, A, un * sgB);
    double m3 = fma(fma(unsq, un, 3.0 * un * r), A, fma(2.0, r, unsq) * sgB);
    double energy = s.rho * fma(fma(0.5 * ut, ut, fma(0.5, r, h.i0)), m1, 0.5 * m3);
    double rm1 = s.rho * m1;
    double rm2 = s.rho * m2;
    G[0] = rm1;
    G[1] = yaxis ? rm1 * ut : rm2;
    G[2] = yaxis ? rm2 : rm1 * ut;
    G[3] = energy;
}

// ------------------------------------------------- exact residue (fsum)
//
// Superaccumulator: a nonnegative double v = m * 2^(e2-1074), m < 2^53,
// is added exactly as three 32-bit digits into 64-bit limbs at positions
// e2/32 .. e2/32+2.  Limb l weighs 2^(32 l - 1074).  Each limb absorbs
// 2^32 additions before it could overflow (n <= 4e9 points).
constexpr int kLimbs = 68;

KMF_HD void accum_add(unsigned long long *limbs, double v)
{
    if (!(v > 0.0)) return;  // zeros (and the impossible negatives) add nothing
    unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    int be = (int)(bits >> 52);
    unsigned long long m = bits & ((1ull << 52) - 1);
    int e2;
    if (be == 0) {
        e2 = 0;
    } else {
        m |= 1ull << 52;
        e2 = be - 1;
    }
    int L = e2 >> 5, sh = e2 & 31;
    unsigned long long lo = m << sh;                          // bits 0..63 of m<<sh
    unsigned long long hi = sh ? (m >> (64 - sh)) : 0ull;      // bits 64..84
    atomicAdd(&limbs[L], lo & 0xffffffffull);
    atomicAdd(&limbs[L + 1], lo >> 32);
    if (hi) atomicAdd(&limbs[L + 2], hi);
}

}  // namespace kmf

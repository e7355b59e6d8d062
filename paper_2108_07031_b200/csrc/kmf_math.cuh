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
//    flux_residual / apply_boundary, kmf_flux.cuh): algebraically identical
//    to the reference but re-associated for the FP64 pipe (reciprocal
//    instead of three divisions, shared sqrt/rsqrt, explicit fma, lean
//    transcendentals of kmf_fastmath.cuh).  Deviation is a few ulp per flux
//    value; the contract is |dR| <= 1e-11 * max(max|R_row|, 1)
//    per call.
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

// ------------------------------------------------- exact residue (fsum)
//
// Superaccumulator: a nonnegative double v = m * 2^(e2-1074), m < 2^53,
// is added exactly as three 32-bit digits into 64-bit limbs at positions
// e2/32 .. e2/32+2.  Limb l weighs 2^(32 l - 1074).  Each limb absorbs
// 2^32 additions before it could overflow (n <= 4e9 points).
constexpr int kLimbs = 68;

}  // namespace kmf

// ABIA per-link steps in base coordinates, shared by the TMA-pipelined kernel
// (abia_tma.cu) and the plain lane kernel (abia.cu) so both execute the same
// arithmetic. See abia.cu for the derivation and the reference mapping.
#pragma once

#include "pd_batch.cuh"

namespace pd {

// Spatial inertia of link i expressed in base coordinates, J0 = Ad(X)^T J Ad(X)
// for X = (R, p) mapping base to link coordinates: same mass, com at
// X^{-1}(c) = R^T (c - p), rotational inertia R^T Ic R about the com.
__device__ __forceinline__ Inertia inertia_to_base(const Inertia& J, const SE3d& X) {
  Inertia o;
  o.m = J.m;
  o.c = mulT(X.R, J.c - X.p);
  double T[9];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const Vec3d col = sym3_mul(J.I, mk(X.R.m[c], X.R.m[3 + c], X.R.m[6 + c]));
    T[c] = col.x;
    T[3 + c] = col.y;
    T[6 + c] = col.z;
  }
  const int idx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int r = idx[k][0], c = idx[k][1];
    o.I[k] = fma(X.R.m[r], T[c], fma(X.R.m[3 + r], T[3 + c], X.R.m[6 + r] * T[6 + c]));
  }
  return o;
}

// trace of Ad(Y)^T P Ad(Y) for Y = X^{-1} = (R^T, -R^T p): the link-frame
// trace the reference's degeneracy test uses (forward_dynamics.cpp:140).
// Rotations keep traces; the shift by q = -R^T p adds 2 tr(B q^) - q^T D q + |q|^2 tr(D).
__device__ __forceinline__ double link_frame_trace_q(const Sym6& P, const Vec3d q) {
  const double trD = P.D[0] + P.D[3] + P.D[5];
  const double trBq = q.x * (P.B[5] - P.B[7]) + q.y * (P.B[6] - P.B[2]) + q.z * (P.B[1] - P.B[3]);
  const Vec3d Dq = sym3_mul(P.D, q);
  return P.A[0] + P.A[3] + P.A[5] + 2.0 * trBq - dot(q, Dq) + dot(q, q) * trD + trD;
}
__device__ __forceinline__ double link_frame_trace(const Sym6& P, const SE3d& X) {
  return link_frame_trace_q(P, -1.0 * mulT(X.R, X.p));
}

// X_{i-1} = rel_i^{-1} * X_i
__device__ __forceinline__ SE3d step_back(const SE3d& rel, const SE3d& X) {
  SE3d o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o.R.m[3 * r + c] = fma(rel.R.m[r], X.R.m[c], fma(rel.R.m[3 + r], X.R.m[3 + c], rel.R.m[6 + r] * X.R.m[6 + c]));
  o.p = mulT(rel.R, X.p - rel.p);
  return o;
}

// The link-step algebra below is written as FMA chains where a generic
// helper would spend a separate multiply or add (one FP64 pipe slot each):
// the ABIA kernels are FP64-issue bound.

// Compose (a*b) with the translation accumulated in the same FMA chain.
__device__ __forceinline__ SE3d compose_f(const SE3d& a, const SE3d& b) {
  return {matmul(a.R, b.R), mul_acc(a.R, b.p, a.p)};
}
// J x for J = (m, c, Ic): lin = m (v + w x c), ang = Ic w + c x lin
__device__ __forceinline__ Sv inertia_apply_f(const Inertia& J, const Sv& x) {
  const Vec3d lin = J.m * cross_acc(x.a, J.c, x.l);
  return {cross_acc(J.c, lin, sym3_mul(J.I, x.a)), lin};
}
// inertia_sym6(J) + P: J's zero entries add nothing, m c is formed once
__device__ __forceinline__ Sym6 inertia_plus_sym6(const Inertia& J, const Sym6& P) {
  Sym6 o;
  const double m = J.m, cx = J.c.x, cy = J.c.y, cz = J.c.z;
  const double c2 = fma(cx, cx, fma(cy, cy, cz * cz));
  const double mx = m * cx, my = m * cy, mz = m * cz;
  o.A[0] = fma(m, c2 - cx * cx, J.I[0] + P.A[0]);
  o.A[1] = fma(-mx, cy, J.I[1] + P.A[1]);
  o.A[2] = fma(-mx, cz, J.I[2] + P.A[2]);
  o.A[3] = fma(m, c2 - cy * cy, J.I[3] + P.A[3]);
  o.A[4] = fma(-my, cz, J.I[4] + P.A[4]);
  o.A[5] = fma(m, c2 - cz * cz, J.I[5] + P.A[5]);
  o.B[0] = P.B[0];      o.B[1] = P.B[1] - mz; o.B[2] = P.B[2] + my;
  o.B[3] = P.B[3] + mz; o.B[4] = P.B[4];      o.B[5] = P.B[5] - mx;
  o.B[6] = P.B[6] - my; o.B[7] = P.B[7] + mx; o.B[8] = P.B[8];
  o.D[0] = P.D[0] + m; o.D[1] = P.D[1]; o.D[2] = P.D[2];
  o.D[3] = P.D[3] + m; o.D[4] = P.D[4]; o.D[5] = P.D[5] + m;
  return o;
}
// P x with each component one FMA chain: (A a + B l, B^T a + D l)
__device__ __forceinline__ Sv sym6_apply_f(const Sym6& P, const Sv& x) {
  const double* A = P.A;
  const double* B = P.B;
  const double* D = P.D;
  const Vec3d a = x.a, l = x.l;
  return {mk(fma(A[0], a.x, fma(A[1], a.y, fma(A[2], a.z, fma(B[0], l.x, fma(B[1], l.y, B[2] * l.z))))),
             fma(A[1], a.x, fma(A[3], a.y, fma(A[4], a.z, fma(B[3], l.x, fma(B[4], l.y, B[5] * l.z))))),
             fma(A[2], a.x, fma(A[4], a.y, fma(A[5], a.z, fma(B[6], l.x, fma(B[7], l.y, B[8] * l.z)))))),
          mk(fma(B[0], a.x, fma(B[3], a.y, fma(B[6], a.z, fma(D[0], l.x, fma(D[1], l.y, D[2] * l.z))))),
             fma(B[1], a.x, fma(B[4], a.y, fma(B[7], a.z, fma(D[1], l.x, fma(D[3], l.y, D[4] * l.z))))),
             fma(B[2], a.x, fma(B[5], a.y, fma(B[8], a.z, fma(D[2], l.x, fma(D[4], l.y, D[5] * l.z))))))};
}
// acc - x . y as one FMA chain
__device__ __forceinline__ double sub_dot(double acc, const Sv& x, const Sv& y) {
  return fma(-x.a.x, y.a.x, fma(-x.a.y, y.a.y, fma(-x.a.z, y.a.z, fma(-x.l.x, y.l.x, fma(-x.l.y, y.l.y,
                                                                                          fma(-x.l.z, y.l.z, acc))))));
}

// Per-link record between pass B and pass C: base-frame gain g0 = U0/lambda
// (6), base-frame screw S0 (6), free joint rate u (1).
constexpr int kRec = 13;

struct AbiaState {
  SE3d X;       // base -> current link
  Sv V0, A0;    // base-frame twist / bias acceleration of the current link
  Sv F0, Z0;    // sums of base-frame wrenches / z-sweep terms (tip side)
  Sym6 P0;      // projected articulated inertia of the child link
  Sv a0;        // pass C acceleration
  int code, eidx;
  double qpoison;  // sum of 0 * q_k over the links beyond the current one: NaN iff one is not finite
};

__device__ __forceinline__ void abia_init(AbiaState& st, Vec3d g) {
#pragma unroll
  for (int k = 0; k < 9; ++k) st.X.R.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
  st.X.p = mk(0, 0, 0);
  st.V0 = svzero();
  st.A0 = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};  // gravity as base acceleration (inverse_dynamics.cpp:135-140)
  st.F0 = svzero();
  st.Z0 = svzero();
  st.a0 = svzero();
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    st.P0.A[k] = 0.0;
    st.P0.D[k] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) st.P0.B[k] = 0.0;
  st.code = PD_SLOT_OK;
  st.eidx = 0;
  st.qpoison = 0.0;
}

// The reference's degeneracy verdict for link i (forward_dynamics.cpp:140-144),
// !(lambda > 1e-14 tr(I^A_i)), evaluated on its link-frame quantities. Those
// depend on the joint angles of the links beyond i only, while the base-frame
// lambda here also sees the links before i; so with a non-finite joint angle
// the reference's lambda_i is NaN iff one lies beyond i (nan_tip), and a NaN
// reaching lambda only from the base side leaves the reference's test passing.
__device__ __forceinline__ bool abia_degenerate(bool nan_tip, double lambda, double threshold) {
  return nan_tip | ((lambda == lambda) & !(lambda > threshold));  // branch-free
}

// pass A, link i (base -> tip): X_i = rel_i X_{i-1}, V0 and A0 (qddot = 0)
//   inverse_dynamics.cpp:43-48 (velocity source), :72-80 (acceleration source)
// rel = joint_transform(S, HR, hp, q) is history independent; callers may
// compute it ahead (software pipelining across links).
__device__ __forceinline__ void abia_pass_a(AbiaState& st, const SE3d& rel, const Sv& S, double qd) {
  st.X = compose_f(rel, st.X);
  const Sv S0 = adinv_screw(st.X, S);
  st.V0 = svfma(qd, S0, st.V0);
  st.A0 = adv_acc(st.V0, qd * S0, st.A0);
}

// pass B, link i (tip -> base): link wrench and tau_delta, articulated
// inertia, z sweep and u; writes the 13-double record; steps back to link i-1.
__device__ __forceinline__ void abia_pass_b(AbiaState& st, int i, int n, const SE3d& rel, const Sv& S, double qd,
                                            const Inertia& Jl, double tau, double rec[kRec], double q) {
  const Sv S0 = adinv_screw(st.X, S);
  const Inertia J0 = inertia_to_base(Jl, st.X);
  // link wrench, bias torque                      inverse_dynamics.cpp:103-112,146-150
  const Sv h = inertia_apply_f(J0, st.V0);
  st.F0 = neg_advT_acc(st.V0, h, inertia_apply_acc(J0, st.A0, st.F0));
  const double tau_delta = sub_dot(tau, S0, st.F0);
  // articulated inertia                            forward_dynamics.cpp:136-156
  // P0 is zero at the tip (abia_init), so the carry is added unconditionally:
  // no branch splits the link step's scheduling region
  const Sym6 Ia = inertia_plus_sym6(J0, st.P0);
  const Sv U = sym6_apply_f(Ia, S0);
  const double lambda = dot(S0, U);
  // degeneracy test on the link-frame trace (forward_dynamics.cpp:140-144).
  // ||Ad(X^-1)|| <= 1 + |p|, so tr_link <= (1 + |p|)^2 tr_base <= 2 (1 + |p|^2)
  // tr_base: the exact trace is only needed when lambda fails that cheap bound
  // (never, for sane chains).
  const double pn2 = dot(st.X.p, st.X.p);
  const bool nan_tip = st.qpoison != st.qpoison;
  if (nan_tip || !(lambda > 2e-14 * (1.0 + pn2) * sym6_trace(Ia))) {
    if (abia_degenerate(nan_tip, lambda, 1e-14 * link_frame_trace(Ia, st.X)) && st.code == PD_SLOT_OK) {
      st.code = PD_SLOT_DEGENERATE_ARTICULATION;
      st.eidx = i;
    }
  }
  const double inv_l = rcp_nr(lambda);
  const double u = sub_dot(tau_delta, S0, st.Z0) * inv_l;  // forward_dynamics.cpp:202-212
  const Sv g0 = inv_l * U;                                 // gain (base frame)
  rec[0] = g0.a.x;
  rec[1] = g0.a.y;
  rec[2] = g0.a.z;
  rec[3] = g0.l.x;
  rec[4] = g0.l.y;
  rec[5] = g0.l.z;
  rec[6] = S0.a.x;
  rec[7] = S0.a.y;
  rec[8] = S0.a.z;
  rec[9] = S0.l.x;
  rec[10] = S0.l.y;
  rec[11] = S0.l.z;
  rec[12] = u;
  {  // (at i = 0 the carried state is dead: updating it anyway keeps the step branch-free)
    st.Z0 = svfma(u, U, st.Z0);  // forward_dynamics.cpp:186-197
    // projected = I^A - U U^T / lambda = I^A - U g0^T   (:150-156)
    st.P0 = Ia;
    const double ua[3] = {U.a.x, U.a.y, U.a.z}, ul[3] = {U.l.x, U.l.y, U.l.z};
    const double ga[3] = {g0.a.x, g0.a.y, g0.a.z}, gl[3] = {g0.l.x, g0.l.y, g0.l.z};
    const int sidx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      st.P0.A[k] = fma(-ua[sidx[k][0]], ga[sidx[k][1]], st.P0.A[k]);
      st.P0.D[k] = fma(-ul[sidx[k][0]], gl[sidx[k][1]], st.P0.D[k]);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) st.P0.B[3 * r + c] = fma(-ua[r], gl[c], st.P0.B[3 * r + c]);
    // parent's link states and frame
    const Sv rate0 = qd * S0;
    st.A0 = adv_acc(st.V0, -1.0 * rate0, st.A0);
    st.V0 = svfma(-qd, S0, st.V0);
    st.X = step_back(rel, st.X);
  }
  st.qpoison = fma(q, 0.0, st.qpoison);  // NaN / inf angle poisons the links below it
}

// pass B reduced to the bias (the torque-surplus mode of the ring kernels,
// CFA's tau_delta pre-pass): link wrench, tau_delta = tau - S0 . F0
// (forward_dynamics.cpp:35-42, inverse_dynamics.cpp:103-112,146-150), then
// the step back to link i-1 -- the articulated-inertia part left out.
__device__ __forceinline__ double abia_pass_b_bias(AbiaState& st, const SE3d& rel, const Sv& S, double qd,
                                                   const Inertia& Jl, double tau) {
  const Sv S0 = adinv_screw(st.X, S);
  const Inertia J0 = inertia_to_base(Jl, st.X);
  const Sv h = inertia_apply_f(J0, st.V0);
  st.F0 = neg_advT_acc(st.V0, h, inertia_apply_acc(J0, st.A0, st.F0));
  const double tau_delta = sub_dot(tau, S0, st.F0);
  const Sv rate0 = qd * S0;
  st.A0 = adv_acc(st.V0, -1.0 * rate0, st.A0);
  st.V0 = svfma(-qd, S0, st.V0);
  st.X = step_back(rel, st.X);
  return tau_delta;
}

// pass C, link i (base -> tip): qdd_i = u_i - g0_i . a0_{i-1}; a0_i = a0_{i-1} + S0_i qdd_i
//   forward_dynamics.cpp:199-235
__device__ __forceinline__ double abia_pass_c(AbiaState& st, const double rec[kRec]) {
  const Sv g0 = {mk(rec[0], rec[1], rec[2]), mk(rec[3], rec[4], rec[5])};
  const Sv S0 = {mk(rec[6], rec[7], rec[8]), mk(rec[9], rec[10], rec[11])};
  const double qdd = rec[12] - dot(g0, st.a0);
  st.a0 = svfma(qdd, S0, st.a0);
  return qdd;
}

}  // namespace pd

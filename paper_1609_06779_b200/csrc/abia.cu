// ABIA forward dynamics, batched, one lane per chain.
//
// Reference: abia_forward_dynamics (proj/core/src/forward_dynamics.cpp:165-243)
// = kinematics (model.cpp:117-146) + torque surplus through inverse dynamics
// with qddot = 0 (forward_dynamics.cpp:35-42, inverse_dynamics.cpp:122-164)
// + articulated-body inertias (forward_dynamics.cpp:120-163) + the z
// (upper) and a (lower) bi-diagonal sweeps + per-joint extraction.
//
// B200 mapping. For batches of independent chains every bi-diagonal system
// is solved by its work-optimal sequential recurrence inside one lane (the
// scan is what the reference uses to expose intra-chain parallelism; with
// 65k+ chains the batch already fills the machine 4x over, and a Hillis-Steele
// scan would multiply the FP64 work by ~log2(n) x 7). The whole solve is three
// fused passes over the links with no intermediate HBM traffic except a
// 7-double per-link record (g_i, u_i) between the tip-to-base and the
// base-to-tip pass:
//   pass A (base->tip): joint transforms, V_i, A_i (A with qddot = 0, gravity
//     as base acceleration -g); only the tip values are kept.
//   pass B (tip->base): transforms recomputed; V_i, A_i recovered backwards
//     through Ad^{-1}; link wrench F_i and bias torque -> tau_delta_i; the
//     articulated inertia recursion (I^A, lambda, gain); the z sweep; the
//     free joint rate u_i = (tau_delta_i - S_i.z_i)/lambda_i.
//   pass C (base->tip): a_i = Ad a_{i-1} + S_i qdd_i with
//     qdd_i = u_i - g_i . (Ad a_{i-1})  (forward_dynamics.cpp:199-235).
#include "pd_batch.cuh"

namespace pd {

struct LinkKinParams {
  Sv S;
  Mat3d HR;
  Vec3d hp;
};

__device__ __forceinline__ LinkKinParams load_kin(const ModelView& mv, int i, int64_t mc) {
  return {mv.screw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc)};
}

__global__ void __launch_bounds__(128) abia_lane_kernel(ModelView mv, BatchIO io, double* __restrict__ scratch) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= io.B) return;
  const int n = mv.n;
  const int64_t B = io.B;
  const int64_t mc = mv.model_of(p);
  if (model_rejected(mv, io, p, mc)) return;

  // ---- pass A: base -> tip ----------------------------------------------
  const Vec3d g = mv.gravity(mc);
  Sv V = svzero();
  Sv A = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};  // inverse_dynamics.cpp:135-140
  for (int i = 0; i < n; ++i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const SE3d T = joint_transform(L.S, L.HR, L.hp, io.ld(io.q, i, p));
    const Sv rate = io.ld(io.qd, i, p) * L.S;
    V = ad_apply(T, V) + rate;                  // inverse_dynamics.cpp:43-48
    A = ad_apply(T, A) + adv_apply(V, rate);    // inverse_dynamics.cpp:72-80 (qddot = 0)
  }

  // ---- pass B: tip -> base ----------------------------------------------
  Sv carryF = svzero();  // Ad_i^T F_{i+1}
  Sv carryZ = svzero();  // Ad_i^T (z_{i+1} + U_{i+1} u_{i+1})
  Sym6 carryI;           // Ad_i^T P_{i+1} Ad_i
  int code = PD_SLOT_OK, eidx = 0;
  for (int i = n - 1; i >= 0; --i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const double qdi = io.ld(io.qd, i, p);
    const SE3d T = joint_transform(L.S, L.HR, L.hp, io.ld(io.q, i, p));
    const Inertia J = mv.inertia(i, mc);

    // link wrench and bias torque                 inverse_dynamics.cpp:103-112,146-150
    const Sv h = inertia_apply(J, V);
    const Sv F = inertia_apply(J, A) + neg_advT_apply(V, h) + carryF;
    const double tau_delta = io.ld(io.tau, i, p) - dot(L.S, F);

    // articulated inertia                          forward_dynamics.cpp:136-156
    Sym6 Ia = inertia_sym6(J);
    if (i < n - 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        Ia.A[k] += carryI.A[k];
        Ia.D[k] += carryI.D[k];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) Ia.B[k] += carryI.B[k];
    }
    const Sv U = sym6_apply(Ia, L.S);
    const double lambda = dot(L.S, U);
    if (!(lambda > 1e-14 * sym6_trace(Ia)) && code == PD_SLOT_OK) {
      code = PD_SLOT_DEGENERATE_ARTICULATION;
      eidx = i;
    }
    const double inv_l = 1.0 / lambda;
    // z_i is carryZ; free joint rate                forward_dynamics.cpp:186-212
    const double u = (tau_delta - dot(L.S, carryZ)) * inv_l;
    double* rec = scratch + (int64_t)i * 7 * B + p;
    rec[0] = U.a.x * inv_l;
    rec[B] = U.a.y * inv_l;
    rec[2 * B] = U.a.z * inv_l;
    rec[3 * B] = U.l.x * inv_l;
    rec[4 * B] = U.l.y * inv_l;
    rec[5 * B] = U.l.z * inv_l;
    rec[6 * B] = u;

    if (i > 0) {
      carryF = adT_apply(T, F);
      carryZ = adT_apply(T, carryZ + u * U);
      // projected = I^A - U U^T / lambda, carried across joint i   (:150-156)
      Sym6 P = Ia;
      const double ua[3] = {U.a.x, U.a.y, U.a.z}, ul[3] = {U.l.x, U.l.y, U.l.z};
      const int sidx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        P.A[k] -= ua[sidx[k][0]] * ua[sidx[k][1]] * inv_l;
        P.D[k] -= ul[sidx[k][0]] * ul[sidx[k][1]] * inv_l;
      }
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) P.B[3 * r + c] -= ua[r] * ul[c] * inv_l;
      carryI = sym6_congruence(P, T);
      // recover the parent's link states through Ad(rel_i)^{-1}
      const Sv rate = qdi * L.S;
      A = adinv_apply(T, A - adv_apply(V, rate));
      V = adinv_apply(T, V - rate);
    }
  }

  // ---- pass C: base -> tip ----------------------------------------------
  Sv a = svzero();
  for (int i = 0; i < n; ++i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const SE3d T = joint_transform(L.S, L.HR, L.hp, io.ld(io.q, i, p));
    const double* rec = scratch + (int64_t)i * 7 * B + p;
    const Sv gi = {mk(rec[0], rec[B], rec[2 * B]), mk(rec[3 * B], rec[4 * B], rec[5 * B])};
    const double u = rec[6 * B];
    const Sv ap = ad_apply(T, a);
    const double qddi = u - dot(gi, ap);
    a = ap + qddi * L.S;
    io.qdd[(int64_t)i * B + p] = qddi;
  }
  io.status[p] = code;
  io.eround[p] = 0;
  io.eindex[p] = eidx;
}

void launch_abia(const ModelView& mv, const BatchIO& io, double* scratch, cudaStream_t s) {
  const int threads = 128;
  const int64_t blocks = (io.B + threads - 1) / threads;
  abia_lane_kernel<<<(unsigned)blocks, threads, 0, s>>>(mv, io, scratch);
}

// Batched inverse dynamics with default IdOptions (inverse_dynamics.cpp:122-173):
// io.tau carries qddot in, io.qdd carries the joint torques out. Same fused
// pass structure as ABIA's first two passes.
__global__ void __launch_bounds__(128) invdyn_lane_kernel(ModelView mv, BatchIO io) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= io.B) return;
  const int n = mv.n;
  const int64_t mc = mv.model_of(p);
  if (model_rejected(mv, io, p, mc)) return;
  const Vec3d g = mv.gravity(mc);
  Sv V = svzero();
  Sv A = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};
  for (int i = 0; i < n; ++i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const SE3d T = joint_transform(L.S, L.HR, L.hp, io.ld(io.q, i, p));
    const Sv rate = io.ld(io.qd, i, p) * L.S;
    V = ad_apply(T, V) + rate;
    A = ad_apply(T, A) + io.ld(io.tau, i, p) * L.S + adv_apply(V, rate);
  }
  Sv carryF = svzero();
  for (int i = n - 1; i >= 0; --i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const SE3d T = joint_transform(L.S, L.HR, L.hp, io.ld(io.q, i, p));
    const Inertia J = mv.inertia(i, mc);
    const Sv h = inertia_apply(J, V);
    const Sv F = inertia_apply(J, A) + neg_advT_apply(V, h) + carryF;
    io.qdd[(int64_t)i * io.B + p] = dot(L.S, F);
    if (i > 0) {
      carryF = adT_apply(T, F);
      const Sv rate = io.ld(io.qd, i, p) * L.S;
      A = adinv_apply(T, A - io.ld(io.tau, i, p) * L.S - adv_apply(V, rate));
      V = adinv_apply(T, V - rate);
    }
  }
  io.status[p] = PD_SLOT_OK;
  io.eround[p] = 0;
  io.eindex[p] = 0;
}

void launch_invdyn(const ModelView& mv, const BatchIO& io, cudaStream_t s) {
  const int threads = 128;
  invdyn_lane_kernel<<<(unsigned)((io.B + threads - 1) / threads), threads, 0, s>>>(mv, io);
}

}  // namespace pd

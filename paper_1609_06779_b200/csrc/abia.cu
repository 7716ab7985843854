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
// 13-double per-link record (g0_i, S0_i, u_i) between the tip-to-base and the
// base-to-tip pass:
//   pass A (base->tip): joint transforms, V_i, A_i (A with qddot = 0, gravity
//     as base acceleration -g); only the tip values are kept.
//   pass B (tip->base): transforms recomputed; V_i, A_i recovered backwards
//     through Ad^{-1}; link wrench F_i and bias torque -> tau_delta_i; the
//     articulated inertia recursion (I^A, lambda, gain); the z sweep; the
//     free joint rate u_i = (tau_delta_i - S_i.z_i)/lambda_i.
//   pass C (base->tip): a_i = Ad a_{i-1} + S_i qdd_i with
//     qdd_i = u_i - g_i . (Ad a_{i-1})  (forward_dynamics.cpp:199-235).
#include "abia_common.cuh"

namespace pd {

struct LinkKinParams {
  Sv S;
  double iw;
  Mat3d HR;
  Vec3d hp;
};

__device__ __forceinline__ LinkKinParams load_kin(const ModelView& mv, int i, int64_t mc) {
  return {mv.screw(i, mc), mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc)};
}

// The whole solve runs in base coordinates. With X_i = rel_i * ... * rel_0
// (base -> link i), every link-frame quantity q_i of the reference has a
// base-frame twin: twists Ad(X_i)^{-1} x, wrenches Ad(X_i)^T f, inertias
// Ad(X_i)^T J Ad(X_i). Transport between neighbours then disappears:
//   V0_i = V0_{i-1} + S0_i qd_i,  A0_i = A0_{i-1} + ad_{V0_i}(S0_i qd_i)
//   F0_i = F0_{i+1} + f0_i,       IA0_i = J0_i + P0_{i+1}
//   z0_i = z0_{i+1} + U0_{i+1} u_{i+1},  a0_i = a0_{i-1} + S0_i qdd_i
// and the scalars (tau, lambda, u, qdd) are frame invariant, so qdd is the
// reference's ABIA result. X_i is rebuilt tip-to-base as rel_i^{-1} X_i.
// This plain variant reads the model with __ldg (shared models, odd strides);
// abia_tma.cu is the TMA-pipelined variant used for batches.
__global__ void __launch_bounds__(128) abia_lane_kernel(ModelView mv, BatchIO io, double* __restrict__ scratch) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= io.B) return;
  const int n = mv.n;
  const int64_t B = io.B;
  const int64_t mc = mv.model_of(p);
  if (model_rejected(mv, io, p, mc)) return;
  AbiaState st;
  abia_init(st, mv.gravity(mc));
  for (int i = 0; i < n; ++i) {
    const Sv S = mv.screw(i, mc);
    abia_pass_a(st, joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p)), S,
                io.ld(io.qd, i, p));
  }
  for (int i = n - 1; i >= 0; --i) {
    double rec[kRec];
    const Sv S = mv.screw(i, mc);
    abia_pass_b(st, i, n, joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p)), S,
                io.ld(io.qd, i, p), mv.inertia(i, mc), io.ld(io.tau, i, p), rec, io.ld(io.q, i, p));
#pragma unroll
    for (int k = 0; k < kRec; ++k) scratch[((int64_t)i * kRec + k) * B + p] = rec[k];
  }
  for (int i = 0; i < n; ++i) {
    double rec[kRec];
#pragma unroll
    for (int k = 0; k < kRec; ++k) rec[k] = scratch[((int64_t)i * kRec + k) * B + p];
    io.put_qdd(i, p, abia_pass_c(st, rec));
  }
  io.status[p] = st.code;
  io.eround[p] = 0;
  io.eindex[p] = st.eidx;
}

int abia_scratch_doubles_per_link() { return kRec + 2; }  // records + (sin, cos)

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
    const SE3d T = joint_transform(L.S, L.iw, L.HR, L.hp, io.ld(io.q, i, p));
    const Sv rate = io.ld(io.qd, i, p) * L.S;
    V = ad_apply(T, V) + rate;
    A = ad_apply(T, A) + io.ld(io.tau, i, p) * L.S + adv_apply(V, rate);
  }
  Sv carryF = svzero();
  for (int i = n - 1; i >= 0; --i) {
    const LinkKinParams L = load_kin(mv, i, mc);
    const SE3d T = joint_transform(L.S, L.iw, L.HR, L.hp, io.ld(io.q, i, p));
    const Inertia J = mv.inertia(i, mc);
    const Sv h = inertia_apply(J, V);
    const Sv F = inertia_apply(J, A) + neg_advT_apply(V, h) + carryF;
    io.put_qdd(i, p, dot(L.S, F));
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

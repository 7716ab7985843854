// Batched inverse dynamics with the reference's full IdOptions, and the link
// states of one evaluation.
//
// Reference (proj/core/src/inverse_dynamics.cpp):
//   propagate_velocities     :27-51   V_0 = Ad(rel_0) V_base + S_0 qd_0,
//                                     V_i = Ad(rel_i) V_{i-1} + S_i qd_i
//   propagate_accelerations  :53-84   A_i = Ad(rel_i) A_{i-1} + S_i qdd_i + ad_{V_i}(S_i qd_i),
//                                     A_base = base_acceleration (- gravity if apply_gravity, :135-140)
//   propagate_forces         :86-120  F_i = Ad(rel_{i+1})^T F_{i+1} + J_i A_i - ad_{V_i}^T (J_i V_i),
//                                     F_{n-1} += tip_wrench (last link's frame)
//   tau_i = S_i . F_i                 :146-150
//   bias_torque              :175-179 (qdd = 0, default options)
//   link_states              :181-196 (V, A, F of every link)
//
// Lane per chain, sequential recurrences (work-optimal for batches of
// independent chains): the forward pass carries V, A; the backward pass
// recovers them through Ad^{-1} and carries F. The packed model lives in
// joint-aligned frames F'_i = Q_i F_i (frames.cuh); link states and the tip
// wrench are rotated between the two frames with Q_i rebuilt from the raw
// screw, so every reported quantity is in the reference's link frames.
#include "frames.cuh"

namespace pd {

struct IdOpts {
  double bv[6], ba[6], tip[6];  // base twist, base acceleration (angular, linear); tip wrench (moment, force)
  int gravity;
};

namespace {

__device__ __forceinline__ Sv sv_of(const double* v) { return {mk(v[0], v[1], v[2]), mk(v[3], v[4], v[5])}; }
__device__ __forceinline__ Sv rot(const Mat3d& Q, const Sv& x) { return {mul(Q, x.a), mul(Q, x.l)}; }
__device__ __forceinline__ Sv rotT(const Mat3d& Q, const Sv& x) { return {mulT(Q, x.a), mulT(Q, x.l)}; }

// [n][6][lds] link-state array (link, component, problem)
__device__ __forceinline__ void put_sv(double* a, int64_t lds, int i, int64_t p, const Sv& x) {
  const double v[6] = {x.a.x, x.a.y, x.a.z, x.l.x, x.l.y, x.l.z};
#pragma unroll
  for (int k = 0; k < 6; ++k) a[((int64_t)i * 6 + k) * lds + p] = v[k];
}

__device__ __forceinline__ Mat3d frame_of(const double* raw, int n, int64_t mc, int i) {
  Mat3d Q;
  raw_joint_frame(raw, n, mc, i, Q.m);
  return Q;
}

}  // namespace

// io.tau carries qddot in, io.qdd carries the joint torques out.
template <bool STATES, bool TIP>
__global__ void __launch_bounds__(128) idyn_lane_kernel(ModelView mv, BatchIO io, IdOpts o,
                                                        const double* __restrict__ raw, double* __restrict__ vel,
                                                        double* __restrict__ acc, double* __restrict__ frc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= io.B) return;
  const int n = mv.n;
  const int64_t mc = mv.model_of(p);
  if (model_rejected(mv, io, p, mc)) return;
  Sv V = sv_of(o.bv);
  Sv A = sv_of(o.ba);
  if (o.gravity) A.l = A.l - mv.gravity(mc);  // inverse_dynamics.cpp:135-140
  for (int i = 0; i < n; ++i) {
    const Sv S = mv.screw(i, mc);
    const SE3d T = joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p));
    const Sv rate = io.ld(io.qd, i, p) * S;
    V = ad_apply(T, V) + rate;
    A = ad_apply(T, A) + io.ld(io.tau, i, p) * S + adv_apply(V, rate);
    if (STATES) {
      const Mat3d Q = frame_of(raw, n, mc, i);
      put_sv(vel, io.lds, i, p, rotT(Q, V));
      put_sv(acc, io.lds, i, p, rotT(Q, A));
    }
  }
  Sv carryF = svzero();
  if (TIP) carryF = rot(frame_of(raw, n, mc, n - 1), sv_of(o.tip));  // F_{n-1} += tip (:117)
  for (int i = n - 1; i >= 0; --i) {
    const Sv S = mv.screw(i, mc);
    const SE3d T = joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p));
    const Inertia J = mv.inertia(i, mc);
    const Sv h = inertia_apply(J, V);
    const Sv F = inertia_apply(J, A) + neg_advT_apply(V, h) + carryF;
    io.put_qdd(i, p, dot(S, F));
    if (STATES) put_sv(frc, io.lds, i, p, rotT(frame_of(raw, n, mc, i), F));
    if (i > 0) {
      carryF = adT_apply(T, F);
      const Sv rate = io.ld(io.qd, i, p) * S;
      A = adinv_apply(T, A - io.ld(io.tau, i, p) * S - adv_apply(V, rate));
      V = adinv_apply(T, V - rate);
    }
  }
  io.status[p] = PD_SLOT_OK;
  io.eround[p] = 0;
  io.eindex[p] = 0;
}

// Torque surplus tau_delta = tau - ID(q, qd, 0) (forward_dynamics.cpp:35-42),
// lane per chain, into td[link][problem] (stride io.lds): the bias stage of
// the CTA-per-chain CFA kernel for large batches, where sequential per-lane
// recurrences beat CTA-wide scans (no barriers, work-optimal).
__global__ void __launch_bounds__(128, 4) tau_surplus_lane_kernel(ModelView mv, BatchIO io, double* __restrict__ td) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= io.B) return;
  const int n = mv.n;
  const int64_t mc = mv.model_of(p);
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) return;  // the CFA kernel reports the model's rule
  Sv V = svzero();
  const Vec3d g = mv.gravity(mc);
  Sv A = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};  // inverse_dynamics.cpp:135-140
  for (int i = 0; i < n; ++i) {
    const Sv S = mv.screw(i, mc);
    const SE3d T = joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p));
    const Sv rate = io.ld(io.qd, i, p) * S;
    V = ad_apply(T, V) + rate;
    A = ad_apply(T, A) + adv_apply(V, rate);
  }
  Sv carryF = svzero();
  for (int i = n - 1; i >= 0; --i) {
    const Sv S = mv.screw(i, mc);
    const SE3d T = joint_transform(S, mv.screw_iw(i, mc), mv.home_R(i, mc), mv.home_p(i, mc), io.ld(io.q, i, p));
    const Inertia J = mv.inertia(i, mc);
    const Sv h = inertia_apply(J, V);
    const Sv F = inertia_apply(J, A) + neg_advT_apply(V, h) + carryF;
    td[(int64_t)i * io.lds + p] = io.ld(io.tau, i, p) - dot(S, F);
    if (i > 0) {
      carryF = adT_apply(T, F);
      const Sv rate = io.ld(io.qd, i, p) * S;
      A = adinv_apply(T, A - adv_apply(V, rate));
      V = adinv_apply(T, V - rate);
    }
  }
}

void launch_tau_surplus(const ModelView& mv, const BatchIO& io, double* td, cudaStream_t s) {
  tau_surplus_lane_kernel<<<(unsigned)((io.B + 127) / 128), 128, 0, s>>>(mv, io, td);
}

void launch_idyn(const ModelView& mv, const BatchIO& io, const IdOpts& o, const double* raw, double* vel, double* acc,
                 double* frc, cudaStream_t s) {
  const int threads = 128;
  const unsigned blocks = (unsigned)((io.B + threads - 1) / threads);
  bool tip = false;
  for (int k = 0; k < 6; ++k) tip = tip || o.tip[k] != 0.0;
  const bool states = vel != nullptr;
  if (states)
    idyn_lane_kernel<true, true><<<blocks, threads, 0, s>>>(mv, io, o, raw, vel, acc, frc);
  else if (tip)
    idyn_lane_kernel<false, true><<<blocks, threads, 0, s>>>(mv, io, o, raw, vel, acc, frc);
  else
    idyn_lane_kernel<false, false><<<blocks, threads, 0, s>>>(mv, io, o, raw, vel, acc, frc);
}

}  // namespace pd

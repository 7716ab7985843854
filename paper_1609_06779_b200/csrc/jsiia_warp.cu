// JSIIA, one warp per chain (n <= 32), lane i = link i = row i of M.
//
// Same algorithm as the reference's jsiia_forward_dynamics
// (forward_dynamics.cpp:82-118): torque surplus, joint-space inertia M,
// LLT(M), qdd = M^{-1} td, one refinement step under the 1e-9 residual
// contract. Everything lives in registers; the warp is the unit.
//
//  * bias torque + composite inertias in base coordinates (see
//    cta_common.cuh): X_i = rel_i X_{i-1} is a warp-shuffle prefix product,
//    V0 / A0 prefix sums, F0 and Ic0 = sum_{k>=i} J0_k suffix sums.
//  * M_ij = S0_min(i,j) . (Ic0_max S0_max): lane i builds row i (j <= i) from
//    the S0_j broadcast through shared memory: M[i][j] = S0_j . FB_i.
//  * Cholesky, left-looking by rows: at step m lane m publishes row m of L in
//    shared memory; lanes i > m form L[i][m]; every lane i < m captures
//    L[m][i] from the same broadcast, so it also holds column i of L and the
//    back substitution needs one broadcast per step, like the forward one.
//  * residual td - M x in O(n): (M x)_i = S0_i . (Ic0_i P_i + Q_i) with
//    P_i = sum_{j<=i} S0_j x_j and Q_i = sum_{j>i} FB_j x_j (two 6-wide scans) --
//    the same matrix as the explicit M, evaluated through its CRBA form.
#include "abia_common.cuh"

namespace pd {

namespace {

constexpr int kWarps = 4;  // chains per CTA

template <int K>
struct A {
  double v[K];
};
template <int K>
__device__ __forceinline__ A<K> shup(const A<K>& x, int d) {
  A<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) o.v[k] = __shfl_up_sync(0xffffffffu, x.v[k], d);
  return o;
}
template <int K>
__device__ __forceinline__ A<K> shdn(const A<K>& x, int d) {
  A<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) o.v[k] = __shfl_down_sync(0xffffffffu, x.v[k], d);
  return o;
}

// inclusive warp prefix sum (REVERSE: suffix sum) of K doubles
template <int K, bool REVERSE>
__device__ __forceinline__ A<K> warp_sum_scan(A<K> x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const A<K> y = REVERSE ? shdn(x, d) : shup(x, d);
    const bool take = REVERSE ? (lane + d < 32) : (lane >= d);
    if (take) {
#pragma unroll
      for (int k = 0; k < K; ++k) x.v[k] += y.v[k];
    }
  }
  return x;
}

__device__ __forceinline__ A<12> pack_se3(const SE3d& T) {
  A<12> a;
#pragma unroll
  for (int k = 0; k < 9; ++k) a.v[k] = T.R.m[k];
  a.v[9] = T.p.x;
  a.v[10] = T.p.y;
  a.v[11] = T.p.z;
  return a;
}
__device__ __forceinline__ SE3d unpack_se3(const A<12>& a) {
  SE3d T;
#pragma unroll
  for (int k = 0; k < 9; ++k) T.R.m[k] = a.v[k];
  T.p = mk(a.v[9], a.v[10], a.v[11]);
  return T;
}
// X_i = rel_i * rel_{i-1} * ... * rel_0 (later factor on the left)
__device__ __forceinline__ SE3d warp_se3_prefix(SE3d T, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const SE3d E = unpack_se3(shup(pack_se3(T), d));
    if (lane >= d) T = compose(T, E);
  }
  return T;
}
__device__ __forceinline__ A<6> sv_pack(const Sv& x) { return {{x.a.x, x.a.y, x.a.z, x.l.x, x.l.y, x.l.z}}; }
__device__ __forceinline__ Sv sv_unpack(const A<6>& a) { return {mk(a.v[0], a.v[1], a.v[2]), mk(a.v[3], a.v[4], a.v[5])}; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

struct WarpSmem {
  double s0[6][32];   // base-frame screws S0_j
  double L[32][33];   // Cholesky factor, row-major, padded (conflict-free rows and columns)
};

}  // namespace

// Model read from the link-fastest copy mcl[(chain * F_COUNT + field) * n + link].
__global__ void __launch_bounds__(32 * kWarps) jsiia_warp_kernel(ModelView mv, const double* __restrict__ mcl,
                                                                  BatchIO io) {
  __shared__ WarpSmem wsm[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // No early returns: every warp runs the collectives convergently (an
  // early exit would make the compiler wrap each shuffle in a divergence
  // fallback); out-of-range warps compute on chain 0 and store nothing.
  const int64_t p_raw = (int64_t)blockIdx.x * kWarps + w;
  const bool in_range = p_raw < io.B;
  const int64_t p = in_range ? p_raw : 0;
  const int n = mv.n;
  const int64_t mc = mv.model_of(p);
  const bool rejected = __ldg(mv.mstatus + mc) != PD_SLOT_OK;
  if (in_range && rejected && lane == 0) model_rejected(mv, io, p, mc);
  const bool store = in_range && !rejected;
  WarpSmem& sm = wsm[w];
  const bool on = lane < n;
  const int li = on ? lane : 0;
  const double* m = mcl + (size_t)mc * F_COUNT * n;
  auto F = [&](int f) { return on ? __ldg(m + f * n + li) : 0.0; };

  // ---- kinematics, X prefix --------------------------------------------------
  const Sv S = joint_screw(F(F_SW), F(F_SVX), F(F_SVZ));
  const Mat3d HR = quat_to_R(F(F_HQ), F(F_HQ + 1), F(F_HQ + 2), F(F_HQ + 3));
  const double q = on ? io.ld(io.q, li, p) : 0.0;
  const double qd = on ? io.ld(io.qd, li, p) : 0.0;
  const double tau = on ? io.ld(io.tau, li, p) : 0.0;
  SE3d rel = joint_transform(S, F(F_SIW), HR, mk(F(F_HP), F(F_HP + 1), F(F_HP + 2)), q);
  if (!on) {
#pragma unroll
    for (int k = 0; k < 9; ++k) rel.R.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
    rel.p = mk(0, 0, 0);
  }
  const SE3d X = warp_se3_prefix(rel, lane);

  // ---- bias torque (base frame) ------------------------------------------------
  const Sv S0 = adinv_screw(X, S);
  const Sv rate0 = qd * S0;
  const Sv V0 = sv_unpack(warp_sum_scan<6, false>(sv_pack(rate0), lane));
  const Vec3d g = mv.gravity(mc);
  const Sv Abase = {mk(0, 0, 0), mk(-g.x, -g.y, -g.z)};
  const Sv A0 = Abase + sv_unpack(warp_sum_scan<6, false>(sv_pack(on ? adv_apply(V0, rate0) : svzero()), lane));
  Inertia Jl;
  Jl.m = F(F_MASS);
  Jl.c = mk(F(F_COM), F(F_COM + 1), F(F_COM + 2));
#pragma unroll
  for (int j = 0; j < 6; ++j) Jl.I[j] = F(F_IC + j);
  const Inertia J0 = inertia_to_base(Jl, X);
  const Sv h = inertia_apply(J0, V0);
  const Sv f0 = on ? neg_advT_acc(V0, h, inertia_apply(J0, A0)) : svzero();
  const Sv F0 = sv_unpack(warp_sum_scan<6, true>(sv_pack(f0), lane));
  const double td = tau - dot(S0, F0);  // forward_dynamics.cpp:35-42

  // ---- composite inertias, FB = Ic0 S0 -------------------------------------------
  A<21> ic;
  {
    const Sym6 Js = inertia_sym6(J0);
#pragma unroll
    for (int k = 0; k < 6; ++k) ic.v[k] = on ? Js.A[k] : 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) ic.v[6 + k] = on ? Js.B[k] : 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) ic.v[15 + k] = on ? Js.D[k] : 0.0;
  }
  ic = warp_sum_scan<21, true>(ic, lane);
  Sym6 Ic;
#pragma unroll
  for (int k = 0; k < 6; ++k) Ic.A[k] = ic.v[k];
#pragma unroll
  for (int k = 0; k < 9; ++k) Ic.B[k] = ic.v[6 + k];
#pragma unroll
  for (int k = 0; k < 6; ++k) Ic.D[k] = ic.v[15 + k];
  const Sv FB = sym6_apply(Ic, S0);
  {
    const A<6> s0p = sv_pack(S0);
#pragma unroll
    for (int k = 0; k < 6; ++k) sm.s0[k][lane] = s0p.v[k];
  }
  __syncwarp();

  // ---- M row i (lower part) ------------------------------------------------------
  double L[32];  // row i of M, overwritten by row i of L
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j < n && j <= lane) {  // divergent but shuffle-free
      const Sv Sj = {mk(sm.s0[0][j], sm.s0[1][j], sm.s0[2][j]), mk(sm.s0[3][j], sm.s0[4][j], sm.s0[5][j])};
      L[j] = dot(Sj, FB);
    } else {
      L[j] = 0.0;
    }
  }

  // ---- Cholesky, left-looking by rows -------------------------------------------
  // Lane i owns row i (registers); every new entry L[i][m] is also stored to
  // the warp's shared L, so at step m row m is read there as a broadcast and
  // the back substitution can read columns. Steps run for all 32 lanes
  // unconditionally (collectives stay convergent); rows >= n are padding.
  double inv_diag = 0.0;
  bool spd = true;
#pragma unroll
  for (int mm = 0; mm < 32; ++mm) {
    // four independent partial sums: the inner product is the critical path
    double a4[4] = {L[mm], 0.0, 0.0, 0.0};
#pragma unroll
    for (int pp = 0; pp < mm; ++pp) a4[pp & 3] = fma(-L[pp], sm.L[mm][pp], a4[pp & 3]);
    const double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    const bool real = mm < n;
    const double dmm = __shfl_sync(0xffffffffu, acc, mm);  // M[mm][mm] - sum_p L[mm][p]^2
    spd = spd && (!real || dmm > 0.0);                      // Eigen LLT: fails iff a pivot <= 0
    const double lmm = sqrt(real ? dmm : 1.0);
    const double inv = 1.0 / lmm;
    inv_diag = (lane == mm) ? inv : inv_diag;
    L[mm] = (lane == mm) ? lmm : ((lane > mm) ? acc * inv : L[mm]);
    sm.L[lane][mm] = L[mm];
    __syncwarp();
  }

  // ---- solve + residual contract (forward_dynamics.cpp:99-116) --------------------
  // pass 0: x = (L L^T)^{-1} td; pass 1 (only if the residual check fails):
  // x += (L L^T)^{-1} r. Written as one loop so the solver and the O(n) M x
  // appear once in the instruction stream. All lanes run every collective.
  const double scale = fmax(sqrt(warp_sum(on ? td * td : 0.0)), 2.2250738585072014e-308);
  double x = 0.0, rhs = on ? td : 0.0;
  int code = PD_SLOT_OK;
  for (int pass = 0; pass < 2; ++pass) {
    // forward: y_m = (b_m - sum_{p<m} L[m][p] y_p) / L[m][m]
    double y = 0.0, acc = rhs;
#pragma unroll
    for (int mm = 0; mm < 32; ++mm) {
      const double ym = __shfl_sync(0xffffffffu, acc * inv_diag, mm);
      y = (lane == mm) ? ym : y;
      acc = (lane > mm && mm < n) ? fma(-L[mm], ym, acc) : acc;
    }
    // backward: x_m = (y_m - sum_{j>m} L[j][m] x_j) / L[m][m]
    double dx = 0.0;
    acc = y;
#pragma unroll
    for (int mm = 31; mm >= 0; --mm) {
      const double xm = __shfl_sync(0xffffffffu, acc * inv_diag, mm);
      dx = (lane == mm) ? xm : dx;
      acc = (lane < mm && mm < n) ? fma(-sm.L[mm][lane], xm, acc) : acc;
    }
    x = on ? x + dx : 0.0;
    // (M x)_i = S0_i . (Ic0_i P_i + Q_i), P inclusive prefix of S0 x, Q exclusive suffix of FB x
    const Sv sx = on ? x * S0 : svzero();
    const Sv fx = on ? x * FB : svzero();
    const Sv P = sv_unpack(warp_sum_scan<6, false>(sv_pack(sx), lane));
    const Sv Q = sv_unpack(warp_sum_scan<6, true>(sv_pack(fx), lane)) - fx;
    const double mx = dot(S0, sym6_apply(Ic, P) + Q);
    rhs = on ? td - mx : 0.0;
    const double rn = sqrt(warp_sum(rhs * rhs));
    if (!(rn > 1e-9 * scale) || !spd) break;  // warp-uniform
    if (pass == 1) code = PD_SLOT_JSI_REFINE_FAILED;
  }
  if (!spd) code = PD_SLOT_JSI_NOT_SPD;  // forward_dynamics.cpp:93-98
  if (store && on) io.put_qdd(lane, p, x);
  if (store && lane == 0) {
    io.status[p] = code;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

bool launch_jsiia_warp(const ModelView& mv, const double* mcl, const BatchIO& io, cudaStream_t s) {
  if (mv.n > 32) return false;
  const unsigned blocks = (unsigned)((io.B + kWarps - 1) / kWarps);
  jsiia_warp_kernel<<<blocks, 32 * kWarps, 0, s>>>(mv, mcl, io);
  return true;
}

}  // namespace pd

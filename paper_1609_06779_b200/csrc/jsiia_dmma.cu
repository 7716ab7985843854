// JSIIA for chains of up to 64 links, one warp per chain, with the joint-space
// inertia matrix M built and factored on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64) in 8x8 blocks held in registers.
//
// Reference: jsiia_forward_dynamics (proj/core/src/forward_dynamics.cpp:82-118)
//   torque surplus td = tau - ID(q, qd, 0)            (:35-42)
//   M = joint_space_inertia_assembled, symmetrised    (:44-66)
//   LLT(M), DynamicsError if not SPD                  (:93-98)
//   qdd = M^{-1} td, one refinement step when ||td - M qdd|| > 1e-9 ||td||,
//   DynamicsError if still above                       (:99-116)
//
// B200 mapping (NB = ceil(n/8) blocks, LPL = links per lane):
//  * Prologue in base coordinates, lane l owns links [l*LPL, (l+1)*LPL):
//    X_i = rel_i ... rel_0 (local compose + warp SE(3) scan), S0 = Ad(X)^-1 S,
//    V0 / A0 prefix sums, F0 = suffix sum of link wrenches, td = tau - S0.F0,
//    composite inertias Ic0_i = sum_{k>=i} J0_k (21-wide suffix sum) and
//    FB_i = Ic0_i S0_i. The reference's n column probes evaluate the closed
//    form M_ij = S0_min(i,j) . FB_max(i,j) (exactly symmetric).
//  * M block (I,J), I >= J: FB_I (8x6) * S0_J^T (6x8) = 2 DMMA (k = 6 padded
//    to 8). Padding links carry zero S0/FB and a unit diagonal.
//  * Blocked Cholesky over k: the 8x8 diagonal block is factored and inverted
//    in registers with quad shuffles; panel blocks L_ik = A_ik L_kk^-T and the
//    updates A_ij -= L_ik L_jk^T are DMMAs. NB <= 4: right-looking over the
//    whole block triangle in registers; NB > 4 (c5): left-looking, so only the
//    L blocks and one block column are live (no spills).
//  * Solves L y = b, L^T x = y by block substitution with the diagonal
//    inverses (vectors ride in column 0 of a DMMA tile).
//  * Residual (M x)_i = FB_i . P_i + S0_i . Q_i with P = prefix sum of S0_j x_j
//    and Q = exclusive suffix sum of FB_j x_j (the same M, O(n)).
//
// Fragment layouts (lane = 4 g + t): C-layout of an 8x8 block X holds
// X[g][2t], X[g][2t+1]; the N-frag holds X[g][t], X[g][4+t] (A operand of X
// in two k-halves, and B operand of X^T); the T-frag holds X[t][g], X[4+t][g]
// (A operand of X^T, B operand of X).
#include "abia_common.cuh"

namespace pd {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kDWarps = 4;  // chains per CTA

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(kFull, v, src); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// C-layout -> N-frag
__device__ __forceinline__ void c_to_n(const double (&c)[2], double (&f)[2], int g, int t) {
  const int s0 = 4 * g + (t >> 1), s1 = s0 + 2;
  const double a0 = shfl(c[0], s0), a1 = shfl(c[1], s0), b0 = shfl(c[0], s1), b1 = shfl(c[1], s1);
  f[0] = (t & 1) ? a1 : a0;
  f[1] = (t & 1) ? b1 : b0;
}
// N-frag -> T-frag
__device__ __forceinline__ void n_to_t(const double (&n)[2], double (&f)[2], int g, int t) {
  const int s0 = 4 * t + (g & 3), s1 = s0 + 16;
  const double a0 = shfl(n[0], s0), a1 = shfl(n[1], s0), b0 = shfl(n[0], s1), b1 = shfl(n[1], s1);
  f[0] = (g >> 2) ? a1 : a0;
  f[1] = (g >> 2) ? b1 : b0;
}
// column-0 vector (v[g] at lanes t == 0) -> T-frag of the 8x8 matrix [v 0 ... 0]
__device__ __forceinline__ void vec_to_t(double v, double (&f)[2], int g, int t) {
  const double a = shfl(v, 4 * t), b = shfl(v, 16 + 4 * t);
  f[0] = g == 0 ? a : 0.0;
  f[1] = g == 0 ? b : 0.0;
}

// In-register Cholesky of the lower triangle of an 8x8 C-layout block and the
// inverse of its factor. On return c holds L (lower; the strict upper part is
// not meaningful), x holds L^{-1}. spd is cleared if a pivot is <= 0 (Eigen
// LLT's failure rule).
__device__ __forceinline__ void potrf_inv8(double (&c)[2], double (&x)[2], bool& spd, int g, int t) {
  x[0] = (g == 2 * t) ? 1.0 : 0.0;
  x[1] = (g == 2 * t + 1) ? 1.0 : 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int tm = m >> 1, e = m & 1;
    // every operand of step m is fetched unscaled at once and scaled locally,
    // so one shuffle latency and one rsqrt sit on the pivot-to-pivot path
    const double d = shfl(c[e], 4 * m + tm);                                  // A[m][m]
    const double ag = shfl(c[e], 4 * g + tm);                                 // A[g][m]
    const double ac0 = shfl(c[e], 8 * t + tm), ac1 = shfl(c[e], 8 * t + 4 + tm);  // A[2t][m], A[2t+1][m]
    const double xu0 = shfl(x[0], 4 * m + t), xu1 = shfl(x[1], 4 * m + t);   // X[m][2t], X[m][2t+1]
    spd = spd && !(d <= 0.0);  // Eigen LLT: fails iff a pivot <= 0 (NaN propagates)
    const double il = rsqrt_nr(d);  // 1 / L[m][m]; L[m][m] itself is never needed again
    const double lg = ag * il, lc0 = ac0 * il, lc1 = ac1 * il;
    if (t == tm) c[e] = (g == m) ? d * il : ((g > m) ? lg : c[e]);
    if (g > m) {
      if (2 * t > m) c[0] = fma(-lg, lc0, c[0]);
      if (2 * t + 1 > m) c[1] = fma(-lg, lc1, c[1]);
    }
    const double xm0 = xu0 * il, xm1 = xu1 * il;  // row m of L^{-1}
    if (g == m) {
      x[0] = xm0;
      x[1] = xm1;
    }
    if (g > m) {
      x[0] = fma(-lg, xm0, x[0]);
      x[1] = fma(-lg, xm1, x[1]);
    }
  }
}

template <int K>
struct Vk {
  double v[K];
};

// Warp scan over lanes of per-lane totals: exclusive prefix (REV: suffix over
// higher lanes) of K doubles; Hillis-Steele inclusive + one shift. ROLL keeps
// the 5 rounds as a loop: for the NB > 4 kernels the smaller instruction
// footprint wins (c5j 25.6 -> 24.3 ms), for NB <= 4 it loses (c2j 559 -> 569 us).
template <int K, bool REV, bool ROLL>
__device__ __forceinline__ Vk<K> warp_excl(Vk<K> x, int lane) {
#pragma unroll(ROLL ? 1 : 5)
  for (int d = 1; d < 32; d <<= 1) {
    Vk<K> y;
#pragma unroll
    for (int k = 0; k < K; ++k) y.v[k] = REV ? __shfl_down_sync(kFull, x.v[k], d) : __shfl_up_sync(kFull, x.v[k], d);
    const bool take = REV ? (lane + d < 32) : (lane >= d);
    if (take) {
#pragma unroll
      for (int k = 0; k < K; ++k) x.v[k] += y.v[k];
    }
  }
  Vk<K> o;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double s = REV ? __shfl_down_sync(kFull, x.v[k], 1) : __shfl_up_sync(kFull, x.v[k], 1);
    o.v[k] = (REV ? (lane == 31) : (lane == 0)) ? 0.0 : s;
  }
  return o;
}

// Inclusive (or exclusive) scan of K-vectors over the chain's links, lane l
// holding links l*LPL + e; REV = suffix sums.
template <int K, bool REV>
__device__ __forceinline__ Vk<K> warp_incl(Vk<K> x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Vk<K> y;
#pragma unroll
    for (int k = 0; k < K; ++k) y.v[k] = REV ? __shfl_down_sync(kFull, x.v[k], d) : __shfl_up_sync(kFull, x.v[k], d);
    const bool take = REV ? (lane + d < 32) : (lane >= d);
    if (take) {
#pragma unroll
      for (int k = 0; k < K; ++k) x.v[k] += y.v[k];
    }
  }
  return x;
}

template <int K, int LPL, bool REV, bool INCL>
__device__ __forceinline__ void link_scan(Vk<K> (&a)[LPL], int lane) {
  if (LPL == 1 && INCL) {
    a[0] = warp_incl<K, REV>(a[0], lane);
    return;
  }
  Vk<K> tot;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < LPL; ++e) s += a[REV ? LPL - 1 - e : e].v[k];
    tot.v[k] = s;
  }
  const Vk<K> base = warp_excl<K, REV, (LPL > 1)>(tot, lane);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double run = base.v[k];
#pragma unroll
    for (int ee = 0; ee < LPL; ++ee) {
      const int e = REV ? LPL - 1 - ee : ee;
      const double own = a[e].v[k];
      if (INCL) {
        run += own;
        a[e].v[k] = run;
      } else {
        a[e].v[k] = run;
        run += own;
      }
    }
  }
}

__device__ __forceinline__ Vk<6> sv6(const Sv& x) { return {{x.a.x, x.a.y, x.a.z, x.l.x, x.l.y, x.l.z}}; }
__device__ __forceinline__ Sv un6(const Vk<6>& a) { return {mk(a.v[0], a.v[1], a.v[2]), mk(a.v[3], a.v[4], a.v[5])}; }

template <int NB>
struct DSmem {
  double s0[6][NB * 8];
  double fb[6][NB * 8];
  double vec[NB * 8];
};

constexpr __host__ __device__ int bidx(int i, int j) { return i * (i + 1) / 2 + j; }

}  // namespace

// Model read from the link-fastest copy mcl[(chain * F_COUNT + field) * n + link].
template <int NB>
__global__ void __launch_bounds__(32 * kDWarps, NB <= 4 ? 5 : 3) jsiia_dmma_kernel(ModelView mv, const double* __restrict__ mcl,
                                                                 BatchIO io) {
  constexpr int NP = NB * 8;               // padded links
  constexpr int LPL = (NP + 31) / 32;      // links per lane
  constexpr int NBLK = NB * (NB + 1) / 2;  // lower blocks
  __shared__ DSmem<NB> wsm[kDWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t p_raw = (int64_t)blockIdx.x * kDWarps + w;
  const bool in_range = p_raw < io.B;
  const int64_t p = in_range ? p_raw : 0;
  const int n = mv.n;
  const int64_t mc = mv.model_of(p);
  const bool rejected = __ldg(mv.mstatus + mc) != PD_SLOT_OK;
  if (in_range && rejected && lane == 0) model_rejected(mv, io, p, mc);
  const bool store = in_range && !rejected;
  DSmem<NB>& sm = wsm[w];
  const double* m = mcl + (size_t)mc * F_COUNT * n;

  // ---- prologue: kinematics, bias torque, composite inertias (lane-link layout)
  SE3d X[LPL];
  Sv S0[LPL], FB[LPL];
  double td[LPL];
  {
    SE3d rel[LPL];
    Sv S[LPL];
    double qd[LPL], tau[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      const int i = lane * LPL + e;
      const bool on = i < n;
      const int li = on ? i : 0;
      auto F = [&](int f) { return on ? __ldg(m + f * n + li) : 0.0; };
      S[e] = joint_screw(F(F_SW), F(F_SVX), F(F_SVZ));
      const Mat3d HR = quat_to_R(F(F_HQ), F(F_HQ + 1), F(F_HQ + 2), F(F_HQ + 3));
      const double q = on ? io.ld(io.q, li, p) : 0.0;
      qd[e] = on ? io.ld(io.qd, li, p) : 0.0;
      tau[e] = on ? io.ld(io.tau, li, p) : 0.0;
      rel[e] = joint_transform(S[e], F(F_SIW), HR, mk(F(F_HP), F(F_HP + 1), F(F_HP + 2)), q);
      if (!on) {
#pragma unroll
        for (int k = 0; k < 9; ++k) rel[e].R.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
        rel[e].p = mk(0, 0, 0);
      }
    }
    // X prefix: lane aggregate, warp scan (later factor on the left), local replay
    SE3d agg = rel[0];
#pragma unroll
    for (int e = 1; e < LPL; ++e) agg = compose(rel[e], agg);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      SE3d o;
#pragma unroll
      for (int k = 0; k < 9; ++k) o.R.m[k] = __shfl_up_sync(kFull, agg.R.m[k], d);
      o.p = mk(__shfl_up_sync(kFull, agg.p.x, d), __shfl_up_sync(kFull, agg.p.y, d), __shfl_up_sync(kFull, agg.p.z, d));
      if (lane >= d) agg = compose(agg, o);
    }
    if (LPL == 1) {
      X[0] = agg;
    } else {
      SE3d ex;
#pragma unroll
      for (int k = 0; k < 9; ++k) ex.R.m[k] = __shfl_up_sync(kFull, agg.R.m[k], 1);
      ex.p = mk(__shfl_up_sync(kFull, agg.p.x, 1), __shfl_up_sync(kFull, agg.p.y, 1), __shfl_up_sync(kFull, agg.p.z, 1));
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 9; ++k) ex.R.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
        ex.p = mk(0, 0, 0);
      }
      X[0] = compose(rel[0], ex);
#pragma unroll
      for (int e = 1; e < LPL; ++e) X[e] = compose(rel[e], X[e - 1]);
    }
    // velocities, bias accelerations (base frame)        inverse_dynamics.cpp:27-84
    Vk<6> V[LPL], A[LPL];
    Sv rate[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      S0[e] = adinv_screw(X[e], S[e]);
      rate[e] = qd[e] * S0[e];
      V[e] = sv6(rate[e]);
    }
    link_scan<6, LPL, false, true>(V, lane);
#pragma unroll
    for (int e = 0; e < LPL; ++e) A[e] = sv6(adv_apply(un6(V[e]), rate[e]));
    link_scan<6, LPL, false, true>(A, lane);
    const Vec3d grav = mv.gravity(mc);
    // link wrenches, suffix sums, bias torque               :86-120, :146-150
    Vk<6> Fw[LPL];
    Vk<10> Ic[LPL];  // composite rigid-body inertia: m, h = m c, rotational inertia about the base origin
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      const int i = lane * LPL + e;
      const bool on = i < n;
      const int li = on ? i : 0;
      auto F = [&](int f) { return on ? __ldg(m + f * n + li) : 0.0; };
      Inertia Jl;
      Jl.m = F(F_MASS);
      Jl.c = mk(F(F_COM), F(F_COM + 1), F(F_COM + 2));
#pragma unroll
      for (int j = 0; j < 6; ++j) Jl.I[j] = F(F_IC + j);
      const Inertia J0 = inertia_to_base(Jl, X[e]);
      const Sv V0 = un6(V[e]);
      Sv A0 = un6(A[e]);
      A0.l = A0.l - grav;  // gravity as base acceleration (inverse_dynamics.cpp:135-140)
      const Sv h = inertia_apply(J0, V0);
      Fw[e] = sv6(on ? neg_advT_acc(V0, h, inertia_apply(J0, A0)) : svzero());
      // a sum of rigid-body inertias is one: 10 numbers instead of the 21 of a
      // general symmetric 6x6 ([[A, h^], [h^T, m 1]], spatial.cpp:89-98)
      const Sym6 Js = inertia_sym6(J0);
      Ic[e].v[0] = J0.m;
      Ic[e].v[1] = J0.m * J0.c.x;
      Ic[e].v[2] = J0.m * J0.c.y;
      Ic[e].v[3] = J0.m * J0.c.z;
#pragma unroll
      for (int k = 0; k < 6; ++k) Ic[e].v[4 + k] = Js.A[k];
    }
    // the wrench and composite-inertia suffix sums: one 16-wide scan for a link
    // per lane (more shuffles in flight per round: c2j -0.7 %); two scans for
    // NB > 4, where the wider live set spills (c5j +0.5 %)
    if constexpr (LPL > 1) {
      link_scan<6, LPL, true, true>(Fw, lane);
      link_scan<10, LPL, true, true>(Ic, lane);
    } else {
      Vk<16> FI[LPL];
#pragma unroll
      for (int e = 0; e < LPL; ++e) {
#pragma unroll
        for (int k = 0; k < 6; ++k) FI[e].v[k] = Fw[e].v[k];
#pragma unroll
        for (int k = 0; k < 10; ++k) FI[e].v[6 + k] = Ic[e].v[k];
      }
      link_scan<16, LPL, true, true>(FI, lane);
#pragma unroll
      for (int e = 0; e < LPL; ++e) {
#pragma unroll
        for (int k = 0; k < 6; ++k) Fw[e].v[k] = FI[e].v[k];
#pragma unroll
        for (int k = 0; k < 10; ++k) Ic[e].v[k] = FI[e].v[6 + k];
      }
    }
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      td[e] = tau[e] - dot(S0[e], un6(Fw[e]));
      // FB = Ic S0 = (A w + h x v, m v + w x h)
      const double mt = Ic[e].v[0];
      const Vec3d h = mk(Ic[e].v[1], Ic[e].v[2], Ic[e].v[3]);
      FB[e] = {cross_acc(h, S0[e].l, sym3_mul(Ic[e].v + 4, S0[e].a)), cross_acc(S0[e].a, h, mt * S0[e].l)};
    }
  }
#pragma unroll
  for (int e = 0; e < LPL; ++e) {
    const int i = lane * LPL + e;
    const Vk<6> s = sv6(S0[e]), f = sv6(FB[e]);
    if (i < NP) {  // lanes past the padded length (NB < 4) hold nothing
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        sm.s0[k][i] = s.v[k];
        sm.fb[k][i] = f.v[k];
      }
    }
  }
  __syncwarp();

  // ---- M blocks and their blocked Cholesky ---------------------------------------
  // LN[bidx(i,k)]: N-frag of L_ik (i > k) or of L_kk^{-1} (i == k)
  double LN[NBLK][2];
  bool spd = true;
  auto m_block = [&](int I, int J, double (&c)[2]) {  // M_IJ = FB_I S0_J^T: 2 DMMA (k = 6 padded to 8)
    const double alo = sm.fb[t][8 * I + g], ahi = t < 2 ? sm.fb[4 + t][8 * I + g] : 0.0;
    c[0] = 0.0;
    c[1] = 0.0;
    dmma(c, alo, sm.s0[t][8 * J + g]);
    dmma(c, ahi, t < 2 ? sm.s0[4 + t][8 * J + g] : 0.0);
    if (I == J && 8 * I + g >= n) {  // padding: unit diagonal
      if (g == 2 * t) c[0] = 1.0;
      if (g == 2 * t + 1) c[1] = 1.0;
    }
  };
  auto panel = [&](int k, const double (&a_ik)[2], double (&l_ik)[2]) {  // L_ik = A_ik L_kk^{-T}
    double a[2], d[2] = {0.0, 0.0};
    c_to_n(a_ik, a, g, t);
    dmma(d, a[0], LN[bidx(k, k)][0]);
    dmma(d, a[1], LN[bidx(k, k)][1]);
    c_to_n(d, l_ik, g, t);
  };
  if constexpr (NB > 4) {
    // Left-looking: block column k is built when it is factored (M_ik minus
    // sum_{j<k} L_ij L_kj^T), so only the L blocks and one column are live --
    // never the whole trailing matrix (the c5 kernel would spill it).
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      double col[NB][2];  // rows i >= k of block column k
#pragma unroll
      for (int i = k; i < NB; ++i) {
        m_block(i, k, col[i]);
#pragma unroll
        for (int j = 0; j < k; ++j) {
          dmma(col[i], -LN[bidx(i, j)][0], LN[bidx(k, j)][0]);
          dmma(col[i], -LN[bidx(i, j)][1], LN[bidx(k, j)][1]);
        }
      }
      double xinv[2];
      potrf_inv8(col[k], xinv, spd, g, t);
      c_to_n(xinv, LN[bidx(k, k)], g, t);
#pragma unroll
      for (int i = k + 1; i < NB; ++i) panel(k, col[i], LN[bidx(i, k)]);
    }
  } else {
    // Right-looking over the whole lower block triangle (small NB: it fits).
    double C[NBLK][2];
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J) m_block(I, J, C[bidx(I, J)]);
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      double xinv[2];
      potrf_inv8(C[bidx(k, k)], xinv, spd, g, t);
      c_to_n(xinv, LN[bidx(k, k)], g, t);
#pragma unroll
      for (int i = k + 1; i < NB; ++i) panel(k, C[bidx(i, k)], LN[bidx(i, k)]);
#pragma unroll
      for (int i = k + 1; i < NB; ++i) {
        const double na0 = -LN[bidx(i, k)][0], na1 = -LN[bidx(i, k)][1];
#pragma unroll
        for (int j = k + 1; j <= i; ++j) {
          dmma(C[bidx(i, j)], na0, LN[bidx(j, k)][0]);
          dmma(C[bidx(i, j)], na1, LN[bidx(j, k)][1]);
        }
      }
    }
  }

  // ---- solve + residual contract (forward_dynamics.cpp:99-116) ------------------
  double ssq = 0.0;
#pragma unroll
  for (int e = 0; e < LPL; ++e) ssq = fma(td[e], td[e], ssq);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) ssq += __shfl_xor_sync(kFull, ssq, d);
  const double scale = fmax(sqrt(ssq), 2.2250738585072014e-308);
  double x[LPL], rhs[LPL];
#pragma unroll
  for (int e = 0; e < LPL; ++e) {
    x[e] = 0.0;
    rhs[e] = td[e];
  }
  int code = PD_SLOT_OK;
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int e = 0; e < LPL; ++e)
      if (lane * LPL + e < NP) sm.vec[lane * LPL + e] = rhs[e];
    __syncwarp();
    double y[NB];
#pragma unroll
    for (int K = 0; K < NB; ++K) {  // L y = b
      double c[2] = {t == 0 ? sm.vec[8 * K + g] : 0.0, 0.0};
#pragma unroll
      for (int J = 0; J < K; ++J) {
        double f[2];
        vec_to_t(-y[J], f, g, t);
        dmma(c, LN[bidx(K, J)][0], f[0]);
        dmma(c, LN[bidx(K, J)][1], f[1]);
      }
      double f[2], r[2] = {0.0, 0.0};
      vec_to_t(c[0], f, g, t);
      dmma(r, LN[bidx(K, K)][0], f[0]);
      dmma(r, LN[bidx(K, K)][1], f[1]);
      y[K] = r[0];
    }
#pragma unroll
    for (int K = NB - 1; K >= 0; --K) {  // L^T x = y
      double c[2] = {y[K], 0.0};
#pragma unroll
      for (int J = K + 1; J < NB; ++J) {
        double lt[2], f[2];
        n_to_t(LN[bidx(J, K)], lt, g, t);
        vec_to_t(-y[J], f, g, t);
        dmma(c, lt[0], f[0]);
        dmma(c, lt[1], f[1]);
      }
      double lt[2], f[2], r[2] = {0.0, 0.0};
      n_to_t(LN[bidx(K, K)], lt, g, t);
      vec_to_t(c[0], f, g, t);
      dmma(r, lt[0], f[0]);
      dmma(r, lt[1], f[1]);
      y[K] = r[0];  // x_K (y_K is dead)
    }
    __syncwarp();
#pragma unroll
    for (int K = 0; K < NB; ++K)
      if (t == 0) sm.vec[8 * K + g] = y[K];
    __syncwarp();
    // x (+)= dx; residual r = td - M x
    Vk<6> P[LPL], Q[LPL];
    Sv s0l[LPL], fbl[LPL];
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      const int i = lane * LPL + e;
      const int ii = i < NP ? i : 0;
      x[e] = i < n ? x[e] + sm.vec[ii] : 0.0;
      s0l[e] = {mk(sm.s0[0][ii], sm.s0[1][ii], sm.s0[2][ii]), mk(sm.s0[3][ii], sm.s0[4][ii], sm.s0[5][ii])};
      fbl[e] = {mk(sm.fb[0][ii], sm.fb[1][ii], sm.fb[2][ii]), mk(sm.fb[3][ii], sm.fb[4][ii], sm.fb[5][ii])};
      if (i >= n) {
        s0l[e] = svzero();
        fbl[e] = svzero();
      }
      P[e] = sv6(x[e] * s0l[e]);
      Q[e] = sv6(x[e] * fbl[e]);
    }
    // (one fused round loop for P and Q spills at NB = 4: c2j +1.4 %)
    link_scan<6, LPL, false, true>(P, lane);
    link_scan<6, LPL, true, false>(Q, lane);
    double rs = 0.0;
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      const int i = lane * LPL + e;
      const double mx = dot(fbl[e], un6(P[e])) + dot(s0l[e], un6(Q[e]));
      rhs[e] = i < n ? td[e] - mx : 0.0;
      rs = fma(rhs[e], rhs[e], rs);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) rs += __shfl_xor_sync(kFull, rs, d);
    if (!(sqrt(rs) > 1e-9 * scale) || !spd) break;  // warp-uniform
    if (pass == 1) code = PD_SLOT_JSI_REFINE_FAILED;
  }
  if (!spd) code = PD_SLOT_JSI_NOT_SPD;  // forward_dynamics.cpp:93-98
  if (store) {
#pragma unroll
    for (int e = 0; e < LPL; ++e) {
      const int i = lane * LPL + e;
      if (i < n) io.put_qdd(i, p, x[e]);
    }
    if (lane == 0) {
      io.status[p] = code;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
  }
}

bool launch_jsiia_dmma(const ModelView& mv, const double* mcl, const BatchIO& io, cudaStream_t s) {
  const unsigned blocks = (unsigned)((io.B + kDWarps - 1) / kDWarps);
  const int nb = (mv.n + 7) / 8;
  switch (nb) {
    case 1: jsiia_dmma_kernel<1><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 2: jsiia_dmma_kernel<2><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 3: jsiia_dmma_kernel<3><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 4: jsiia_dmma_kernel<4><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 5: jsiia_dmma_kernel<5><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 6: jsiia_dmma_kernel<6><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 7: jsiia_dmma_kernel<7><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    case 8: jsiia_dmma_kernel<8><<<blocks, 32 * kDWarps, 0, s>>>(mv, mcl, io); return true;
    default: return false;
  }
}

}  // namespace pd

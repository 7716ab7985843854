// CFA forward dynamics (the paper's Algorithm 1), one CTA per chain, one
// thread per link (LPT consecutive links per thread for long chains).
//
// Reference: cfa_forward_dynamics (proj/core/src/forward_dynamics.cpp:418-450)
//   = kinematics + torque surplus (3 scans)           -> cta_kinematics / cta_bias_torque
//   + build_constraint_basis (:245-259)               -> householder_basis
//   + build_cfa_operators (:261-357)                   -> stage "operators"
//   + rhs = -apply_cross(tau_delta) (:359-376, :433-436)
//   + oee_solve<5,1> (include/pardyn/oee.hpp:149-189)  -> stage "OEE"
//   + qdd = apply_joint(td) + apply_cross_transpose(F_c) (:378-416, :441-442)
//
// OEE (the paper's building block 2, Eq. 17, row-centric form of
// oee.hpp:73-145). Each round every row factors its own pivot D_k once
// (Cholesky, 5x5) and publishes (L_k, 1/L_k,jj, Y_k = L_k^{-1} U_k,
// Rt_k = L_k^{-1} R_k); after one barrier every row applies both eliminations
// from published data only:
//   up   (pivot i+h): W = L^{-1} U_i^T, D_i -= W^T W, R_i -= W^T Rt,
//                     U_i <- -W^T Y_{i+h}                  (only if i+2h < n)
//   down (pivot i-h): D_i -= Y^T Y, R_i -= Y^T Rt.
// Pivots are Schur complements of the SPD constraint operator (SURVEY.md
// §7.4.6), so a symmetric factorization is valid; the rank test mirrors
// FullPivLU::isInvertible (|pivot| > 5 eps max|diag|). The reported error
// is the reference's: smallest failing row, its first failing pivot.
#include <cooperative_groups.h>
#include <cstdlib>

#include "cta_common.cuh"

namespace pd {

namespace cfa {
// Workspace field offsets (units of n doubles, ws[field * n + link]).
constexpr int TD = 0, XS = 1, XB = 6, XD = 11, JD = 16, JO = 17;  // persistent
constexpr int REL = 18;                                           // 12, until operators done
constexpr int X = 30, V = 42, TMP = 48;                           // bias-torque phase only
constexpr int AD = 30, UP = 45;                                   // 15 + 25: operators -> OEE D_i, U_i
constexpr int HT = 70;                                            // 36: H columns (operators phase)
constexpr int HH = 70;                                            // 21: H^T H for row i+1
constexpr int PL = 18, SG = 28;                                   // OEE published: L (10), singular flag
constexpr int PY = 70, PR = 95, PI = 100, OR = 105;               // Y (25), Rt (5), 1/d (5), R_i (5)
constexpr int FIELDS = 110;
}  // namespace cfa

__device__ __forceinline__ int pk(int r, int c) { return r * (r + 1) / 2 + c; }   // packed lower incl diag
__device__ __forceinline__ int pks(int r, int c) { return r * (r - 1) / 2 + c; }  // packed strict lower
// index of (r, c) in Sym6's 3x3 packing (xx xy xz yy yz zz)
__device__ __forceinline__ int s3(int r, int c) {
  const int lo = r < c ? r : c, hi = r < c ? c : r;
  return lo == 0 ? hi : (lo == 1 ? 2 + hi : 5);
}

// Orthonormal complement of the screw: last five columns of the Householder
// reflector Eigen's HouseholderQR builds for the 6x1 screw
// (forward_dynamics.cpp:245-259: makeHouseholder + applyHouseholderOnTheLeft).
// z[c][r]: column c of Z = [W | S].
__device__ __forceinline__ void householder_basis(const Sv& S, double z[6][6]) {
  const double s[6] = {S.a.x, S.a.y, S.a.z, S.l.x, S.l.y, S.l.z};
  double tail = 0.0;
#pragma unroll
  for (int k = 1; k < 6; ++k) tail = fma(s[k], s[k], tail);
  const double c0 = s[0];
  double v[6] = {1.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double tau = 0.0;
  if (tail > 2.2250738585072014e-308) {
    double beta = sqrt(fma(c0, c0, tail));
    if (c0 >= 0.0) beta = -beta;
    const double iden = rcp_nr(c0 - beta);  // branch-free reciprocals instead of 6 divisions
#pragma unroll
    for (int k = 1; k < 6; ++k) v[k] = s[k] * iden;
    tau = (beta - c0) * rcp_nr(beta);
  }
#pragma unroll
  for (int c = 0; c < 5; ++c)
#pragma unroll
    for (int r = 0; r < 6; ++r) z[c][r] = (r == c + 1 ? 1.0 : 0.0) - (tau * v[r]) * v[c + 1];
#pragma unroll
  for (int r = 0; r < 6; ++r) z[5][r] = s[r];
}

// The link's spatial inertia J factored in (linear, angular) block order.
// The reference takes LLT(J) (forward_dynamics.cpp:302-305) only to apply
// J^{-1} inside the operator products (G^T G, G^T H, H^T H with G = L^{-1} Z),
// which any L with L L^T = P J P^T gives the same way. With P swapping the
// blocks, J = [[Ic + m c^ c^T, m c^], [m c^T, m 1]] (spatial.cpp:88-99)
// factors in closed form:
//   L = [[sqrt(m) 1, 0], [sqrt(m) c^, chol(Ic)]]
// (the Schur complement of m 1 is exactly Ic), so a 3x3 Cholesky replaces the
// 6x6 one and each solve is a cross product, three scalings and a 3x3
// triangular solve. J is positive definite iff m > 0 and Ic is, so the
// failure test is Eigen LLT's (a pivot <= 0) on m and on Ic's pivots.
struct JFactor {
  double ism;    // 1 / sqrt(m)
  Vec3d c;       // centre of mass
  double Lc[6];  // chol(Ic), packed lower rows: 00 | 10 11 | 20 21 22
  double il[3];  // 1 / Lc_jj
};
__device__ __forceinline__ bool jfactor(const Inertia& J, JFactor& f) {
  const double* I = J.I;  // xx xy xz yy yz zz (about the com)
  bool ok = !(J.m <= 0.0);
  f.ism = rsqrt_nr(J.m);
  f.c = J.c;
  double x = I[0];
  ok = ok && !(x <= 0.0);
  f.il[0] = rsqrt_nr(x);
  f.Lc[0] = x * f.il[0];
  f.Lc[1] = I[1] * f.il[0];
  f.Lc[3] = I[2] * f.il[0];
  x = fma(-f.Lc[1], f.Lc[1], I[3]);
  ok = ok && !(x <= 0.0);
  f.il[1] = rsqrt_nr(x);
  f.Lc[2] = x * f.il[1];
  f.Lc[4] = fma(-f.Lc[3], f.Lc[1], I[4]) * f.il[1];
  x = fma(-f.Lc[4], f.Lc[4], fma(-f.Lc[3], f.Lc[3], I[5]));
  ok = ok && !(x <= 0.0);
  f.il[2] = rsqrt_nr(x);
  f.Lc[5] = x * f.il[2];
  return ok;
}
// x <- L^{-1} P x for x = (angular, linear): (x_lin / sqrt(m), chol(Ic)^{-1} (x_ang - c x x_lin))
__device__ __forceinline__ void jsolve(const JFactor& f, double x[6]) {
  const Vec3d xl = mk(x[3], x[4], x[5]);
  const Vec3d r = mk(x[0], x[1], x[2]) - cross(f.c, xl);
  const double y0 = r.x * f.il[0];
  const double y1 = fma(-f.Lc[1], y0, r.y) * f.il[1];
  const double y2 = fma(-f.Lc[4], y1, fma(-f.Lc[3], y0, r.z)) * f.il[2];
  x[0] = xl.x * f.ism;
  x[1] = xl.y * f.ism;
  x[2] = xl.z * f.ism;
  x[3] = y0;
  x[4] = y1;
  x[5] = y2;
}

// ---- OEE row algebra on packed 5x5 blocks (Cholesky form) -------------------
// Pivots are Schur complements of the SPD constraint operator, so each is
// factored D_k = L L^T (L lower with its diagonal kept as 1/L_jj); with
// Y_k = L^{-1} U_k, rt_k = L^{-1} R_k and W = L_k^{-1} U_i^T the eliminations
// are plain Gram products: D_i -= W^T W, R_i -= W^T rt_k, U_i <- -W^T Y_k (up),
// D_i -= Y_k^T Y_k, R_i -= Y_k^T rt_k (down) -- no pivot scaling pass.
// The rank test is FullPivLU::isInvertible's: the LDL^T pivot (the square of
// L_jj, before the root) must exceed 5 eps max|diag| (oee.hpp:43,209,225).
__device__ __forceinline__ bool chol5(const double D[15], double L[10], double il[5]) {
  double maxd = 0.0;
#pragma unroll
  for (int k = 0; k < 5; ++k) maxd = fmax(maxd, fabs(D[pk(k, k)]));
  const double thr = 5.0 * 2.220446049250313e-16 * maxd;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    double x = D[pk(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) x = fma(-L[pks(j, k)], L[pks(j, k)], x);
    ok = ok && (x > thr);
    il[j] = rsqrt_nr(fabs(x));
#pragma unroll
    for (int i = j + 1; i < 5; ++i) {
      double s = D[pk(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) s = fma(-L[pks(i, k)], L[pks(j, k)], s);
      L[pks(i, j)] = s * il[j];
    }
  }
  return ok;
}
__device__ __forceinline__ void lsolve5(const double L[10], const double il[5], double x[5]) {  // x <- L^{-1} x
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    double s = x[r];
#pragma unroll
    for (int c = 0; c < r; ++c) s = fma(-L[pks(r, c)], x[c], s);
    x[r] = s * il[r];
  }
}
__device__ __forceinline__ void ltsolve5(const double L[10], const double il[5], double x[5]) {  // x <- L^{-T} x
#pragma unroll
  for (int r = 4; r >= 0; --r) {
    double s = x[r];
#pragma unroll
    for (int c = r + 1; c < 5; ++c) s = fma(-L[pks(c, r)], x[c], s);
    x[r] = s * il[r];
  }
}
// Up elimination of row i by pivot k = i + h. yk(r, c) = Y_k[r][c]; U is
// replaced by the distance-2h coupling when next (i < n - 2h).
template <class YF>
__device__ __forceinline__ void oee_up(double D[15], double R[5], double U[25], const double L[10], const double il[5],
                                       const double rt[5], bool next, YF yk) {
  double W[5][5];
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int r = 0; r < 5; ++r) W[a][r] = U[a * 5 + r];
    lsolve5(L, il, W[a]);
  }
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      double s = D[pk(a, b)];
#pragma unroll
      for (int r = 0; r < 5; ++r) s = fma(-W[a][r], W[b][r], s);
      D[pk(a, b)] = s;
    }
    double s = R[a];
#pragma unroll
    for (int r = 0; r < 5; ++r) s = fma(-W[a][r], rt[r], s);
    R[a] = s;
  }
  if (next) {
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      double yc[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) yc[r] = yk(r, c);
#pragma unroll
      for (int a = 0; a < 5; ++a) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < 5; ++r) s = fma(W[a][r], yc[r], s);
        U[a * 5 + c] = -s;
      }
    }
  }
}
// Down elimination of row i by pivot k = i - h.
template <class YF>
__device__ __forceinline__ void oee_down(double D[15], double R[5], const double rt[5], YF yk) {
  double Y[5][5];
#pragma unroll
  for (int r = 0; r < 5; ++r)
#pragma unroll
    for (int c = 0; c < 5; ++c) Y[r][c] = yk(r, c);
#pragma unroll
  for (int a = 0; a < 5; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) {
      double s = D[pk(a, b)];
#pragma unroll
      for (int r = 0; r < 5; ++r) s = fma(-Y[r][a], Y[r][b], s);
      D[pk(a, b)] = s;
    }
    double s = R[a];
#pragma unroll
    for (int r = 0; r < 5; ++r) s = fma(-Y[r][a], rt[r], s);
    R[a] = s;
  }
}
// Final block solve x = D^{-1} R in place; false if the block is singular.
__device__ __forceinline__ bool oee_final(const double D[15], double R[5]) {
  double L[10], il[5];
  const bool ok = chol5(D, L, il);
  lsolve5(L, il, R);
  ltsolve5(L, il, R);
  return ok;
}

template <int K>
__device__ __forceinline__ void ws_load(const double* ws, int n, int f0, int i, double* out) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = ws[(f0 + k) * n + i];
}
template <int K>
__device__ __forceinline__ void ws_store(double* ws, int n, int f0, int i, const double* in) {
#pragma unroll
  for (int k = 0; k < K; ++k) ws[(f0 + k) * n + i] = in[k];
}

// PREP 1: stop after the OEE initial state is in the (global) workspace;
// PREP 2: stop after the joint transforms and tau_delta -- the grid-wide
// cfa_oee_coop then builds the operators, the initial state and runs the OEE
// (long chains, c4).
// Operators of link i (forward_dynamics.cpp:261-357): Z_i = [W_i | S_i],
// C_i = Ad(rel_{i+1})^T Z_{i+1}, J_i = L L^T, G = L^{-1} Z_i, H = L^{-1} C_i:
// own blocks G^T G (AD, XD, JD), couplings G^T H (UP, XS, XB, JO), the next
// row's carried blocks H^T H (HH). Reads rel_{i+1} from the workspace (HT is
// this link's scratch). Returns false if J_i is not positive definite.
__device__ __forceinline__ bool cfa_link_ops(const ModelView& mv, int64_t mc, double* ws, int n, int i) {
    JFactor jf;
  const bool ok = jfactor(mv.inertia(i, mc), jf);
  double G[6][6];
  householder_basis(mv.screw(i, mc), G);
#pragma unroll
  for (int c = 0; c < 6; ++c) jsolve(jf, G[c]);
  {
    double ad[15], xd[5];
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s = fma(G[r][k], G[c][k], s);
      if (r < 5) ad[pk(r, c)] = s;
      else if (c < 5) xd[c] = s;
      else ws[cfa::JD * n + i] = s;
    }
    ws_store<15>(ws, n, cfa::AD, i, ad);
    ws_store<5>(ws, n, cfa::XD, i, xd);
  }
  if (i + 1 < n) {
    const SE3d T1 = ws_get_se3(ws, n, cfa::REL, i + 1);
    double Z1[6][6];
    householder_basis(mv.screw(i + 1, mc), Z1);
    double up[25], xs[5], xb[5];
#pragma unroll
    for (int c = 0; c < 6; ++c) {
    const Sv col = adT_apply(T1, Sv{mk(Z1[c][0], Z1[c][1], Z1[c][2]), mk(Z1[c][3], Z1[c][4], Z1[c][5])});
    double h[6] = {col.a.x, col.a.y, col.a.z, col.l.x, col.l.y, col.l.z};
    jsolve(jf, h);
    ws_store<6>(ws, n, cfa::HT + 6 * c, i, h);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s = fma(G[r][k], h[k], s);
      if (r < 5 && c < 5) up[r * 5 + c] = -s;       // upper_i       (:347)
      else if (r < 5) xs[r] = -s;                    // cross_super_i (:348)
      else if (c < 5) xb[c] = -s;                    // cross_sub_i   (:349)
      else ws[cfa::JO * n + i] = -s;                 // joint_off_i   (:350)
    }
    }
    ws_store<25>(ws, n, cfa::UP, i, up);
    ws_store<5>(ws, n, cfa::XS, i, xs);
    ws_store<5>(ws, n, cfa::XB, i, xb);
    double hh[21];
#pragma unroll
    for (int r = 0; r < 6; ++r) {
    double hr[6];
    ws_load<6>(ws, n, cfa::HT + 6 * r, i, hr);
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) s = fma(hr[k], ws[(cfa::HT + 6 * c + k) * n + i], s);
      hh[pk(r, c)] = s;
    }
    }
    ws_store<21>(ws, n, cfa::HH, i, hh);
  }
  return ok;
}

// OEE initial state of row i: D_i = A_diag (+ row i-1's H^T H), U_i = upper_i,
// R_i = -apply_cross(td)_i; ld(f, j) reads neighbour fields (the grid-wide
// path reads them through L2). Writes the updated AD / XD / JD and OR.
template <class LD>
__device__ __forceinline__ void cfa_oee_init(double* ws, int n, int i, LD ld) {
  double d[15], xd[5];
  ws_load<15>(ws, n, cfa::AD, i, d);
  ws_load<5>(ws, n, cfa::XD, i, xd);
  double jd = ws[cfa::JD * n + i];
  if (i > 0) {
    double hh[21];
#pragma unroll
    for (int k = 0; k < 21; ++k) hh[k] = ld(cfa::HH + k, i - 1);
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) d[pk(r, c)] += hh[pk(r, c)];
#pragma unroll
    for (int r = 0; r < 5; ++r) xd[r] += hh[pk(5, r)];
    jd += hh[pk(5, 5)];
  }
  const double td = ld(cfa::TD, i);
  double r5[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) r5[r] = xd[r] * td;
  if (i > 0) {
    const double tdm = ld(cfa::TD, i - 1);
#pragma unroll
    for (int r = 0; r < 5; ++r) r5[r] = fma(ld(cfa::XB + r, i - 1), tdm, r5[r]);
  }
  if (i + 1 < n) {
    const double tdp = ld(cfa::TD, i + 1);
#pragma unroll
    for (int r = 0; r < 5; ++r) r5[r] = fma(ws[(cfa::XS + r) * n + i], tdp, r5[r]);
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) r5[r] = -r5[r];
  ws_store<15>(ws, n, cfa::AD, i, d);
  ws_store<5>(ws, n, cfa::XD, i, xd);
  ws[cfa::JD * n + i] = jd;
  ws_store<5>(ws, n, cfa::OR, i, r5);
}

// td_pre: tau_delta precomputed by tau_surplus_lane_kernel ([link][problem],
// stride io.lds) -- the CTA then skips its scan-based bias stage.
template <bool SMEM, int PREP = 0, int NT = 256>
__global__ void __launch_bounds__(NT) cfa_cta_kernel(ModelView mv, BatchIO io, double* __restrict__ gws, int lpt,
                                                       int64_t p_off, const double* __restrict__ td_pre = nullptr) {
  extern __shared__ double dyn_smem[];
  __shared__ ScanSmem scan_sm;
  __shared__ int s_bad, s_link_fail;
  const int n = mv.n;
  const int64_t p = p_off + blockIdx.x;
  const int64_t mc = mv.model_of(p);
  double* ws = SMEM ? dyn_smem : gws + (int64_t)blockIdx.x * cfa::FIELDS * n;
  const int t = threadIdx.x;
  const int i0 = t * lpt, i1 = min(n, i0 + lpt);
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
    if (t == 0) model_rejected(mv, io, p, mc);
    return;
  }
  if (t == 0) {
    s_bad = n;
    s_link_fail = 0;
  }

  // ---- kinematics + torque surplus ----------------------------------------
  const IdFields idf{cfa::REL, cfa::X, cfa::V, cfa::TMP, cfa::TD};
  cta_kinematics(mv, io, p, mc, ws, idf, lpt);
  if (td_pre) {
    for (int i = i0; i < i1; ++i) ws[cfa::TD * n + i] = __ldg(td_pre + (int64_t)i * io.lds + p);
    __syncthreads();
  } else {
    cta_bias_torque(mv, io, p, mc, ws, idf, lpt, scan_sm);  // ends with a barrier
  }

  if (PREP == 2) return;  // kinematics + tau_delta only: the grid-wide path does the rest
  // ---- operators (forward_dynamics.cpp:261-357) ----------------------------
  for (int i = i0; i < i1; ++i)
    if (!cfa_link_ops(mv, mc, ws, n, i)) atomicOr(&s_link_fail, 1);
  __syncthreads();
  if (s_link_fail) {  // forward_dynamics.cpp:317-320
    if (t == 0) {
      io.status[p] = PD_SLOT_LINK_INERTIA_NOT_PD;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }

  // ---- OEE initial state ----------------------------------------------------
  for (int i = i0; i < i1; ++i) cfa_oee_init(ws, n, i, [&](int f, int j) { return ws[f * n + j]; });
  __syncthreads();
  if (PREP) return;

  const int rounds = ceil_log2_dev(n);
  if (lpt == 1) {
    // ---- OEE with the row's own state (D, U, R) in registers ---------------------
    const int i = t;
    const bool own = i < n;
    double D[15], U[25], R[5];
    if (own) {
      ws_load<15>(ws, n, cfa::AD, i, D);
      ws_load<5>(ws, n, cfa::OR, i, R);
      if (i + 1 < n) ws_load<25>(ws, n, cfa::UP, i, U);
    }
    __syncthreads();  // AD/UP/OR are overwritten by the published fields below
    int h = 1;
    for (int round = 1; round <= rounds; ++round, h <<= 1) {
      if (own) {  // publish own pivot factorization: L, 1/L_jj, L^{-1} R, L^{-1} U
        double Lk[10], il[5], rt[5];
        const bool ok = chol5(D, Lk, il);
        ws_store<10>(ws, n, cfa::PL, i, Lk);
        ws_store<5>(ws, n, cfa::PI, i, il);
        ws[cfa::SG * n + i] = ok ? 0.0 : 1.0;
#pragma unroll
        for (int r = 0; r < 5; ++r) rt[r] = R[r];
        lsolve5(Lk, il, rt);
        ws_store<5>(ws, n, cfa::PR, i, rt);
        if (i < n - h) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            double col[5];
#pragma unroll
            for (int r = 0; r < 5; ++r) col[r] = U[r * 5 + c];
            lsolve5(Lk, il, col);
#pragma unroll
            for (int r = 0; r < 5; ++r) ws[(cfa::PY + r * 5 + c) * n + i] = col[r];
          }
        }
      }
      __syncthreads();
      if (own) {
        // singular pivots: smallest failing row, its first failing pivot (oee.hpp:88-138)
        const bool up_bad = (i < n - h) && ws[cfa::SG * n + i + h] != 0.0;
        const bool dn_bad = (i >= h) && ws[cfa::SG * n + i - h] != 0.0;
        if (up_bad || dn_bad) atomicMin(&s_bad, i);
        if (i < n - h) {
          const int k = i + h;
          double Lk[10], il[5], rt[5];
          ws_load<10>(ws, n, cfa::PL, k, Lk);
          ws_load<5>(ws, n, cfa::PI, k, il);
          ws_load<5>(ws, n, cfa::PR, k, rt);
          oee_up(D, R, U, Lk, il, rt, i < n - 2 * h, [&](int r, int c) { return ws[(cfa::PY + r * 5 + c) * n + k]; });
        }
        if (i >= h) {
          const int k = i - h;
          double rt[5];
          ws_load<5>(ws, n, cfa::PR, k, rt);
          oee_down(D, R, rt, [&](int r, int c) { return ws[(cfa::PY + r * 5 + c) * n + k]; });
        }
      }
      __syncthreads();
      if (s_bad < n) {
        if (t == 0) {
          const int ib = s_bad;
          const bool up_bad = (ib < n - h) && ws[cfa::SG * n + ib + h] != 0.0;
          io.status[p] = PD_SLOT_OEE_SINGULAR_PIVOT;
          io.eround[p] = round;
          io.eindex[p] = up_bad ? ib + h : ib - h;
        }
        return;
      }
    }
    // final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187)
    if (own) {
      if (!oee_final(D, R)) atomicMin(&s_bad, i);
      ws_store<5>(ws, n, cfa::OR, i, R);  // constraint force F_c,i
    }
    __syncthreads();
  } else {
  // ---- OEE rounds -----------------------------------------------------------
  int h = 1;
  for (int round = 1; round <= rounds; ++round, h <<= 1) {
    // publish own pivot factorization
    for (int k = i0; k < i1; ++k) {
      double D[15], Lk[10], il[5];
      ws_load<15>(ws, n, cfa::AD, k, D);
      const bool ok = chol5(D, Lk, il);
      ws_store<10>(ws, n, cfa::PL, k, Lk);
      ws_store<5>(ws, n, cfa::PI, k, il);
      ws[cfa::SG * n + k] = ok ? 0.0 : 1.0;
      double rt[5];
      ws_load<5>(ws, n, cfa::OR, k, rt);
      lsolve5(Lk, il, rt);
      ws_store<5>(ws, n, cfa::PR, k, rt);
      if (k < n - h) {  // U_k exists at distance h
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double col[5];
#pragma unroll
          for (int r = 0; r < 5; ++r) col[r] = ws[(cfa::UP + r * 5 + c) * n + k];
          lsolve5(Lk, il, col);
#pragma unroll
          for (int r = 0; r < 5; ++r) ws[(cfa::PY + r * 5 + c) * n + k] = col[r];
        }
      }
    }
    __syncthreads();
    // singular pivots: smallest failing row reports its first failing pivot (oee.hpp:88-138)
    for (int i = i0; i < i1; ++i) {
      const bool up_bad = (i < n - h) && ws[cfa::SG * n + i + h] != 0.0;
      const bool dn_bad = (i >= h) && ws[cfa::SG * n + i - h] != 0.0;
      if (up_bad || dn_bad) atomicMin(&s_bad, i);
    }
    __syncthreads();
    if (s_bad < n) {
      if (t == 0) {
        const int i = s_bad;
        const bool up_bad = (i < n - h) && ws[cfa::SG * n + i + h] != 0.0;
        io.status[p] = PD_SLOT_OEE_SINGULAR_PIVOT;
        io.eround[p] = round;
        io.eindex[p] = up_bad ? i + h : i - h;
      }
      return;
    }
    // eliminate
    for (int i = i0; i < i1; ++i) {
      double D[15], R[5], U[25];
      ws_load<15>(ws, n, cfa::AD, i, D);
      ws_load<5>(ws, n, cfa::OR, i, R);
      if (i < n - h) {
        const int k = i + h;
        double Lk[10], il[5], rt[5];
        ws_load<10>(ws, n, cfa::PL, k, Lk);
        ws_load<5>(ws, n, cfa::PI, k, il);
        ws_load<5>(ws, n, cfa::PR, k, rt);
        ws_load<25>(ws, n, cfa::UP, i, U);
        const bool next = i < n - 2 * h;
        oee_up(D, R, U, Lk, il, rt, next, [&](int r, int c) { return ws[(cfa::PY + r * 5 + c) * n + k]; });
        if (next) ws_store<25>(ws, n, cfa::UP, i, U);
      }
      if (i >= h) {
        const int k = i - h;
        double rt[5];
        ws_load<5>(ws, n, cfa::PR, k, rt);
        oee_down(D, R, rt, [&](int r, int c) { return ws[(cfa::PY + r * 5 + c) * n + k]; });
      }
      ws_store<15>(ws, n, cfa::AD, i, D);
      ws_store<5>(ws, n, cfa::OR, i, R);
    }
    __syncthreads();
  }

  // ---- final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187) -------------
  for (int i = i0; i < i1; ++i) {
    double D[15], x[5];
    ws_load<15>(ws, n, cfa::AD, i, D);
    ws_load<5>(ws, n, cfa::OR, i, x);
    if (!oee_final(D, x)) atomicMin(&s_bad, i);
    ws_store<5>(ws, n, cfa::OR, i, x);  // constraint force F_c,i
  }
  __syncthreads();
  }  // smem-row OEE path
  if (s_bad < n) {
    if (t == 0) {
      io.status[p] = PD_SLOT_OEE_SINGULAR_FINAL;
      io.eround[p] = rounds;
      io.eindex[p] = s_bad;
    }
    return;
  }

  // ---- qdd = apply_joint(td) + apply_cross_transpose(F_c) ------------------
  for (int i = i0; i < i1; ++i) {
    const double td = ws[cfa::TD * n + i];
    double v = ws[cfa::JD * n + i] * td;
    double f[5];
    ws_load<5>(ws, n, cfa::OR, i, f);
#pragma unroll
    for (int r = 0; r < 5; ++r) v = fma(ws[(cfa::XD + r) * n + i], f[r], v);
    if (i > 0) {
      v = fma(ws[cfa::JO * n + i - 1], ws[cfa::TD * n + i - 1], v);
#pragma unroll
      for (int r = 0; r < 5; ++r) v = fma(ws[(cfa::XS + r) * n + i - 1], ws[(cfa::OR + r) * n + i - 1], v);
    }
    if (i + 1 < n) {
      v = fma(ws[cfa::JO * n + i], ws[cfa::TD * n + i + 1], v);
#pragma unroll
      for (int r = 0; r < 5; ++r) v = fma(ws[(cfa::XB + r) * n + i], ws[(cfa::OR + r) * n + i + 1], v);
    }
    io.put_qdd(i, p, v);
  }
  if (t == 0) {
    io.status[p] = PD_SLOT_OK;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

// OEE rounds, final block solves and the q-dot extraction of long chains in
// small batches (c4) on a cooperative grid: a thread per row spread over
// many SMs (the row's D, U, R in registers, as in the CTA kernel), the
// published pivot data in the global workspace read through L2
// (ld.global.cg), a grid barrier where the CTA kernel has __syncthreads.
// Chains one after the other; cfa_cta_kernel<false, 2> left each chain's
// joint transforms and tau_delta in workspace slot c.
__global__ void __launch_bounds__(128) cfa_oee_coop(ModelView mv, BatchIO io, double* __restrict__ gws, int n,
                                                    int count, int* __restrict__ bad) {
  namespace cgr = cooperative_groups;
  cgr::grid_group grid = cgr::this_grid();
  const int i = (int)(blockIdx.x * blockDim.x + threadIdx.x);
  const bool own = i < n;
  const int rounds = ceil_log2_dev(n);
  for (int c = 0; c < count; ++c) {
    double* ws = gws + (size_t)c * cfa::FIELDS * n;
    const int64_t p = c;
    if (__ldg(mv.mstatus + mv.model_of(p)) != PD_SLOT_OK) continue;  // the CTA kernel reported the model's rule
    if (i == 0) *bad = n;
    grid.sync();
    // operators and the OEE initial state, a thread per link (the CTA kernel
    // left rel_i and tau_delta in the workspace)
    if (own && !cfa_link_ops(mv, mv.model_of(p), ws, n, i)) atomicMin(bad, -1);
    grid.sync();
    if (__ldcg(bad) < 0) {  // forward_dynamics.cpp:317-320
      if (i == 0) {
        io.status[p] = PD_SLOT_LINK_INERTIA_NOT_PD;
        io.eround[p] = 0;
        io.eindex[p] = 0;
      }
      grid.sync();
      continue;
    }
    if (own) cfa_oee_init(ws, n, i, [&](int f, int j) { return __ldcg(ws + (size_t)f * n + j); });
    grid.sync();
    double D[15], U[25], R[5];
    if (own) {
#pragma unroll
      for (int k = 0; k < 15; ++k) D[k] = __ldcg(ws + (size_t)(cfa::AD + k) * n + i);
#pragma unroll
      for (int k = 0; k < 5; ++k) R[k] = __ldcg(ws + (size_t)(cfa::OR + k) * n + i);
#pragma unroll
      for (int k = 0; k < 25; ++k) U[k] = (i + 1 < n) ? __ldcg(ws + (size_t)(cfa::UP + k) * n + i) : 0.0;
    }
    grid.sync();
    int h = 1;
    bool failed = false;
    for (int round = 1; round <= rounds; ++round, h <<= 1) {
      if (own) {  // publish own pivot factorization
        double Lk[10], il[5], rt[5];
        const bool ok = chol5(D, Lk, il);
        ws_store<10>(ws, n, cfa::PL, i, Lk);
        ws_store<5>(ws, n, cfa::PI, i, il);
        ws[(size_t)cfa::SG * n + i] = ok ? 0.0 : 1.0;
#pragma unroll
        for (int r = 0; r < 5; ++r) rt[r] = R[r];
        lsolve5(Lk, il, rt);
        ws_store<5>(ws, n, cfa::PR, i, rt);
        if (i < n - h) {
#pragma unroll
          for (int cc = 0; cc < 5; ++cc) {
            double col[5];
#pragma unroll
            for (int r = 0; r < 5; ++r) col[r] = U[r * 5 + cc];
            lsolve5(Lk, il, col);
#pragma unroll
            for (int r = 0; r < 5; ++r) ws[(size_t)(cfa::PY + r * 5 + cc) * n + i] = col[r];
          }
        }
      }
      grid.sync();
      if (own) {
        // singular pivots: smallest failing row, its first failing pivot (oee.hpp:88-138)
        const bool up_bad = (i < n - h) && __ldcg(ws + (size_t)cfa::SG * n + i + h) != 0.0;
        const bool dn_bad = (i >= h) && __ldcg(ws + (size_t)cfa::SG * n + i - h) != 0.0;
        if (up_bad || dn_bad) atomicMin(bad, i);
        // each neighbour's published data is requested in one batch (one L2
        // round trip) before the elimination uses any of it
        if (i < n - h) {
          const int k = i + h;
          double Lk[10], il[5], rt[5], Y[25];
#pragma unroll
          for (int q = 0; q < 10; ++q) Lk[q] = __ldcg(ws + (size_t)(cfa::PL + q) * n + k);
#pragma unroll
          for (int q = 0; q < 5; ++q) il[q] = __ldcg(ws + (size_t)(cfa::PI + q) * n + k);
#pragma unroll
          for (int q = 0; q < 5; ++q) rt[q] = __ldcg(ws + (size_t)(cfa::PR + q) * n + k);
#pragma unroll
          for (int q = 0; q < 25; ++q) Y[q] = __ldcg(ws + (size_t)(cfa::PY + q) * n + k);
          oee_up(D, R, U, Lk, il, rt, i < n - 2 * h, [&](int r, int c) { return Y[r * 5 + c]; });
        }
        if (i >= h) {
          const int k = i - h;
          double rt[5], Y[25];
#pragma unroll
          for (int q = 0; q < 5; ++q) rt[q] = __ldcg(ws + (size_t)(cfa::PR + q) * n + k);
#pragma unroll
          for (int q = 0; q < 25; ++q) Y[q] = __ldcg(ws + (size_t)(cfa::PY + q) * n + k);
          oee_down(D, R, rt, [&](int r, int c) { return Y[r * 5 + c]; });
        }
      }
      grid.sync();
      const int sb = __ldcg(bad);
      if (sb < n) {
        if (i == 0) {
          const bool up_bad = (sb < n - h) && __ldcg(ws + (size_t)cfa::SG * n + sb + h) != 0.0;
          io.status[p] = PD_SLOT_OEE_SINGULAR_PIVOT;
          io.eround[p] = round;
          io.eindex[p] = up_bad ? sb + h : sb - h;
        }
        failed = true;
        break;  // grid-uniform
      }
    }
    if (!failed) {
      // final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187)
      if (own) {
        if (!oee_final(D, R)) atomicMin(bad, i);
        ws_store<5>(ws, n, cfa::OR, i, R);  // constraint force F_c,i
      }
      grid.sync();
      const int sb = __ldcg(bad);
      if (sb < n) {
        if (i == 0) {
          io.status[p] = PD_SLOT_OEE_SINGULAR_FINAL;
          io.eround[p] = rounds;
          io.eindex[p] = sb;
        }
      } else {
        // qdd = apply_joint(td) + apply_cross_transpose(F_c)
        if (own) {
          auto g = [&](int f, int j) { return __ldcg(ws + (size_t)f * n + j); };
          const double td = g(cfa::TD, i);
          double v = g(cfa::JD, i) * td;
#pragma unroll
          for (int r = 0; r < 5; ++r) v = fma(g(cfa::XD + r, i), R[r], v);
          if (i > 0) {
            v = fma(g(cfa::JO, i - 1), g(cfa::TD, i - 1), v);
#pragma unroll
            for (int r = 0; r < 5; ++r) v = fma(g(cfa::XS + r, i - 1), g(cfa::OR + r, i - 1), v);
          }
          if (i + 1 < n) {
            v = fma(g(cfa::JO, i), g(cfa::TD, i + 1), v);
#pragma unroll
            for (int r = 0; r < 5; ++r) v = fma(g(cfa::XB + r, i), g(cfa::OR + r, i + 1), v);
          }
          io.put_qdd(i, p, v);
        }
        if (i == 0) {
          io.status[p] = PD_SLOT_OK;
          io.eround[p] = 0;
          io.eindex[p] = 0;
        }
      }
    }
    grid.sync();  // workspace / flag reuse by the next chain
  }
}

bool cfa_coop_path(int n, int64_t batch) { return (size_t)cfa::FIELDS * n * sizeof(double) > 224 * 1024 && batch <= 4; }

// Long chains in small batches: CTA prologue (kinematics, bias torque,
// operators, OEE initial state) for every chain, then the grid-wide OEE.
void launch_cfa_coop(const ModelView& mv, const BatchIO& io, double* gws, int* bad, int sm_count, cudaStream_t s) {
  const int n = mv.n;
  // 512 threads, 2 links each (1024-link chain): 256 x 4 0.159 ms, 512 x 2
  // 0.132, 1024 x 1 0.146 (spills at 64 registers) for c4
  constexpr int kPrepThreads = 512;
  const int lpt = (n + kPrepThreads - 1) / kPrepThreads;
  cfa_cta_kernel<false, 2, kPrepThreads><<<(unsigned)io.B, kPrepThreads, 0, s>>>(mv, io, gws, lpt, 0);
  int count = (int)io.B;
  int nn = n;
  BatchIO iol = io;
  ModelView mvl = mv;
  void* args[] = {&mvl, &iol, &gws, &nn, &count, &bad};
  const unsigned grid = (unsigned)((n + 127) / 128);
  (void)sm_count;
  cudaLaunchCooperativeKernel((const void*)cfa_oee_coop, dim3(grid), dim3(128), args, 0, s);
}


// ---------------------------------------------------------------------------
// cfa_row_kernel: the n <= 256 case (a thread per link / row, everything in
// shared memory). The operator blocks a row owns (its diagonal block D and
// coupling U, the H columns) stay in registers from the operator stage through
// the OEE rounds, so only what neighbours read lives in shared memory and the
// workspace shrinks from 110 to 70 doubles per link (fields reused across
// stages) and each round's shared-memory traffic is only the published pivot
// data. (c5: 46.8 -> 35.7 ms against the workspace-resident kernel.)
namespace cfr {
constexpr int TD = 0, XS = 1, XB = 6, XD = 11, JD = 16, JO = 17;  // persistent
constexpr int REL = 18, X = 30, V = 42, TMP = 48;                 // kinematics / bias stage
constexpr int HH = 30;                                            // 21: operators -> initial state
constexpr int PL = 18, SG = 28, PY = 30, PR = 55, PI = 60, OR = 65;  // OEE
constexpr int FIELDS = 70;
}  // namespace cfr

// The row stages of the CFA kernels after kinematics and tau_delta: operators
// (rows' own blocks into registers), OEE initial state, the OEE rounds, the
// final block solves and the extraction, on the thread group `grp` (thread =
// row). rel_{i+1} is read from relws (field relf), tau_delta from ws (TD).
// after_ops() runs on every group thread right after the operator stage (the
// last read of relws). s_bad / s_link_fail are the group's shared flags, set
// to (n, 0) by the caller before a group barrier.
template <class G, class AfterOps>
__device__ __forceinline__ void cfa_rows(const ModelView& mv, const BatchIO& io, int64_t p, int64_t mc, double* ws,
                                         const double* relws, int relf, int* s_bad, int* s_link_fail, int pf_stride,
                                         int grp_threads, const G& grp, AfterOps after_ops) {
  const int n = mv.n;
  const int t = grp.tid(), i = t;
  const bool own = i < n;
  // ---- operators (forward_dynamics.cpp:261-357): own blocks into registers
  double D[15], U[25], R[5];
  if (own) {
    JFactor jf;
    if (!jfactor(mv.inertia(i, mc), jf)) atomicOr(s_link_fail, 1);
    double G[6][6];
    householder_basis(mv.screw(i, mc), G);
#pragma unroll
    for (int c = 0; c < 6; ++c) jsolve(jf, G[c]);
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) {
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k) sacc = fma(G[r][k], G[c][k], sacc);
        if (r < 5) D[pk(r, c)] = sacc;
        else if (c < 5) ws[(cfr::XD + c) * n + i] = sacc;
        else ws[cfr::JD * n + i] = sacc;
      }
    if (i + 1 < n) {
      const SE3d T1 = ws_get_se3(relws, n, relf, i + 1);
      double Z1[6][6], H[6][6];
      householder_basis(mv.screw(i + 1, mc), Z1);
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const Sv col = adT_apply(T1, Sv{mk(Z1[c][0], Z1[c][1], Z1[c][2]), mk(Z1[c][3], Z1[c][4], Z1[c][5])});
        double* h = H[c];
        h[0] = col.a.x; h[1] = col.a.y; h[2] = col.a.z; h[3] = col.l.x; h[4] = col.l.y; h[5] = col.l.z;
        jsolve(jf, h);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          double sacc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) sacc = fma(G[r][k], h[k], sacc);
          if (r < 5 && c < 5) U[r * 5 + c] = -sacc;            // upper_i       (:347)
          else if (r < 5) ws[(cfr::XS + r) * n + i] = -sacc;   // cross_super_i (:348)
          else if (c < 5) ws[(cfr::XB + c) * n + i] = -sacc;   // cross_sub_i   (:349)
          else ws[cfr::JO * n + i] = -sacc;                    // joint_off_i   (:350)
        }
      }
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) {
          double sacc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) sacc = fma(H[r][k], H[c][k], sacc);
          ws[(cfr::HH + pk(r, c)) * n + i] = sacc;
        }
    }
  }
  grp.sync();
  after_ops();  // REL (and the caller's td copy) are no longer read
  if (*s_link_fail) {  // forward_dynamics.cpp:317-320
    if (t == 0) {
      io.status[p] = PD_SLOT_LINK_INERTIA_NOT_PD;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }
  // ---- OEE initial state: D_i gains row i-1's H^T H; R_i = -apply_cross(td)_i
  if (own) {
    double xd[5];
    ws_load<5>(ws, n, cfr::XD, i, xd);
    double jd = ws[cfr::JD * n + i];
    if (i > 0) {
#pragma unroll
      for (int r = 0; r < 5; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) D[pk(r, c)] += ws[(cfr::HH + pk(r, c)) * n + i - 1];
#pragma unroll
      for (int r = 0; r < 5; ++r) xd[r] += ws[(cfr::HH + pk(5, r)) * n + i - 1];
      jd += ws[(cfr::HH + pk(5, 5)) * n + i - 1];
    }
    const double td = ws[cfr::TD * n + i];
#pragma unroll
    for (int r = 0; r < 5; ++r) R[r] = xd[r] * td;
    if (i > 0) {
      const double tdm = ws[cfr::TD * n + i - 1];
#pragma unroll
      for (int r = 0; r < 5; ++r) R[r] = fma(ws[(cfr::XB + r) * n + i - 1], tdm, R[r]);
    }
    if (i + 1 < n) {
      const double tdp = ws[cfr::TD * n + i + 1];
#pragma unroll
      for (int r = 0; r < 5; ++r) R[r] = fma(ws[(cfr::XS + r) * n + i], tdp, R[r]);
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) R[r] = -R[r];
    ws_store<5>(ws, n, cfr::XD, i, xd);
    ws[cfr::JD * n + i] = jd;
  }
  grp.sync();  // HH is reused by the published pivots below
  // ---- warm L2 for the chain the SM will most likely run next: CTAs are
  // dispatched in order, so the successor of this one is p + pf_stride (the
  // resident CTAs). Its model (contiguous in the link-fastest copy) and
  // q / qd / tau rows are prefetched into L2 while this chain runs its OEE
  // rounds, so that chain's kinematics loads hit L2 instead of DRAM.
  {
    const int64_t pn = p + pf_stride;
    if (pf_stride > 0 && pn < io.B) {
      const char* base = reinterpret_cast<const char*>(mv.fcl + (int64_t)mv.model_of(pn) * F_COUNT * n);
      const int bytes = F_COUNT * n * (int)sizeof(double);
      for (int off = t * 128; off < bytes; off += grp_threads * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
      if (own) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(io.q + (int64_t)i * io.lds + pn));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(io.qd + (int64_t)i * io.lds + pn));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(io.tau + (int64_t)i * io.lds + pn));
      }
    }
  }
  // ---- OEE rounds (oee.hpp:73-145), row state in registers
  const int rounds = ceil_log2_dev(n);
  int h = 1;
  for (int round = 1; round <= rounds; ++round, h <<= 1) {
    if (own) {
      double Lk[10], il[5], rt[5];
      const bool ok = chol5(D, Lk, il);
      ws_store<10>(ws, n, cfr::PL, i, Lk);
      ws_store<5>(ws, n, cfr::PI, i, il);
      ws[cfr::SG * n + i] = ok ? 0.0 : 1.0;
#pragma unroll
      for (int r = 0; r < 5; ++r) rt[r] = R[r];
      lsolve5(Lk, il, rt);
      ws_store<5>(ws, n, cfr::PR, i, rt);
      if (i < n - h) {
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double col[5];
#pragma unroll
          for (int r = 0; r < 5; ++r) col[r] = U[r * 5 + c];
          lsolve5(Lk, il, col);
#pragma unroll
          for (int r = 0; r < 5; ++r) ws[(cfr::PY + r * 5 + c) * n + i] = col[r];
        }
      }
    }
    grp.sync();
    if (own) {
      const bool up_bad = (i < n - h) && ws[cfr::SG * n + i + h] != 0.0;
      const bool dn_bad = (i >= h) && ws[cfr::SG * n + i - h] != 0.0;
      if (up_bad || dn_bad) atomicMin(s_bad, i);
      if (i < n - h) {
        const int k = i + h;
        double Lk[10], il[5], rt[5];
        ws_load<10>(ws, n, cfr::PL, k, Lk);
        ws_load<5>(ws, n, cfr::PI, k, il);
        ws_load<5>(ws, n, cfr::PR, k, rt);
        oee_up(D, R, U, Lk, il, rt, i < n - 2 * h, [&](int r, int c) { return ws[(cfr::PY + r * 5 + c) * n + k]; });
      }
      if (i >= h) {
        const int k = i - h;
        double rt[5];
        ws_load<5>(ws, n, cfr::PR, k, rt);
        oee_down(D, R, rt, [&](int r, int c) { return ws[(cfr::PY + r * 5 + c) * n + k]; });
      }
    }
    grp.sync();
    if (*s_bad < n) {
      if (t == 0) {
        const int ib = *s_bad;
        const bool up_bad = (ib < n - h) && ws[cfr::SG * n + ib + h] != 0.0;
        io.status[p] = PD_SLOT_OEE_SINGULAR_PIVOT;
        io.eround[p] = round;
        io.eindex[p] = up_bad ? ib + h : ib - h;
      }
      return;
    }
  }
  // final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187)
  if (own) {
    if (!oee_final(D, R)) atomicMin(s_bad, i);
    ws_store<5>(ws, n, cfr::OR, i, R);  // constraint force F_c,i
  }
  grp.sync();
  if (*s_bad < n) {
    if (t == 0) {
      io.status[p] = PD_SLOT_OEE_SINGULAR_FINAL;
      io.eround[p] = rounds;
      io.eindex[p] = *s_bad;
    }
    return;
  }
  // ---- qdd = apply_joint(td) + apply_cross_transpose(F_c) (:378-416, :441-442)
  if (own) {
    const double td = ws[cfr::TD * n + i];
    double v = ws[cfr::JD * n + i] * td;
#pragma unroll
    for (int r = 0; r < 5; ++r) v = fma(ws[(cfr::XD + r) * n + i], R[r], v);
    if (i > 0) {
      v = fma(ws[cfr::JO * n + i - 1], ws[cfr::TD * n + i - 1], v);
#pragma unroll
      for (int r = 0; r < 5; ++r) v = fma(ws[(cfr::XS + r) * n + i - 1], ws[(cfr::OR + r) * n + i - 1], v);
    }
    if (i + 1 < n) {
      v = fma(ws[cfr::JO * n + i], ws[cfr::TD * n + i + 1], v);
#pragma unroll
      for (int r = 0; r < 5; ++r) v = fma(ws[(cfr::XB + r) * n + i], ws[(cfr::OR + r) * n + i + 1], v);
    }
    io.put_qdd(i, p, v);
  }
  if (t == 0) {
    io.status[p] = PD_SLOT_OK;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) cfa_row_kernel(ModelView mv, BatchIO io, const double* __restrict__ td_pre,
                                                           int pf_stride) {
  extern __shared__ double dyn_smem[];
  __shared__ ScanSmem scan_sm;
  __shared__ int s_bad, s_link_fail;
  const int n = mv.n;
  const int64_t p = blockIdx.x;
  const int64_t mc = mv.model_of(p);
  double* ws = dyn_smem;
  const int t = threadIdx.x, i = t;
  const bool own = i < n;
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
    if (t == 0) model_rejected(mv, io, p, mc);
    return;
  }
  if (t == 0) {
    s_bad = n;
    s_link_fail = 0;
  }
  // ---- kinematics + torque surplus
  const IdFields idf{cfr::REL, cfr::X, cfr::V, cfr::TMP, cfr::TD};
  cta_kinematics(mv, io, p, mc, ws, idf, 1);
  if (td_pre) {
    if (own) ws[cfr::TD * n + i] = __ldg(td_pre + (int64_t)i * io.lds + p);
    __syncthreads();
  } else {
    cta_bias_torque(mv, io, p, mc, ws, idf, 1, scan_sm);  // ends with a barrier
  }
  cfa_rows(mv, io, p, mc, ws, ws, cfr::REL, &s_bad, &s_link_fail, pf_stride, NT, CtaGroup{}, [] {});
}

// Warp-specialised CFA for batches of long chains (128 < n <= 256, c3):
// persistent CTAs of 384 threads run two chains at once on two thread groups.
//   rows      threads 0..255 (2 warpgroups, setmaxnreg 208): operators, OEE,
//             extraction of chain k (cfa_rows, thread = row);
//   prologue  threads 256..383 (1 warpgroup, setmaxnreg 88): joint
//             transforms and tau_delta of chain k+1 (cta_kinematics /
//             cta_bias_torque, 2 links per thread).
// The one-chain-per-SM row kernel ran the latency-bound CTA scans of the
// prologue alone (~35 % of c3); here they fill the issue slots the OEE rounds
// leave idle. Handoff through shared memory (rel: 12 fields, tau_delta: 1) with
// named barriers: 1 rows, 2 prologue, 3 "chain ready" (prologue arrives, rows
// wait), 4 "handoff free" (rows arrive once the operators have read rel,
// prologue waits before writing the next chain). setmaxnreg only moves
// registers inside the CTA's launch allocation (384 x 168): 256 x 208 +
// 128 x 88 = 384 x 168 (split sweep on c3: 200/104 0.828, 208/88 0.822,
// 216/72 0.888, 224/56 0.990 ms -- the prologue's scans spill below 88).
namespace cws {
constexpr int REL = 0, TD = 12, X = 13, V = 25, TMP = 31, FIELDS = 37;  // handoff + prologue scratch
constexpr int kRows = 256, kPro = 128, kAll = kRows + kPro;
}  // namespace cws

__global__ void __launch_bounds__(cws::kAll, 1) cfa_ws_kernel(ModelView mv, BatchIO io) {
  extern __shared__ double dyn_smem[];
  __shared__ ScanSmem scan_pro;
  __shared__ int s_bad, s_link_fail;
  const int n = mv.n;
  double* ws = dyn_smem;                // cfr::FIELDS x n: the rows' workspace
  double* hand = ws + cfr::FIELDS * n;  // cws::FIELDS x n: handoff + prologue scratch
  if (threadIdx.x < cws::kRows) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
    const NamedGroup grp{0, cws::kRows, 1};
    const int t = grp.tid();
    for (int64_t p = blockIdx.x; p < io.B; p += gridDim.x) {
      asm volatile("bar.sync 3, %0;" ::"n"(cws::kAll) : "memory");  // chain p's rel / tau_delta are in `hand`
      const int64_t mc = mv.model_of(p);
      if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
        if (t == 0) model_rejected(mv, io, p, mc);
        asm volatile("bar.arrive 4, %0;" ::"n"(cws::kAll) : "memory");
        continue;
      }
      if (t == 0) {
        s_bad = n;
        s_link_fail = 0;
      }
      if (t < n) ws[cfr::TD * n + t] = hand[cws::TD * n + t];
      grp.sync();
      cfa_rows(mv, io, p, mc, ws, hand, cws::REL, &s_bad, &s_link_fail, 0, cws::kRows, grp,
               [] { asm volatile("bar.arrive 4, %0;" ::"n"(cws::kAll) : "memory"); });
      grp.sync();  // the flags and the workspace are reused by the next chain
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
    const NamedGroup grp{cws::kRows, cws::kPro, 2};
    bool first = true;
    for (int64_t p = blockIdx.x; p < io.B; p += gridDim.x) {
      {  // warm L2 with the chain after this one (its model rows and states)
        const int64_t pn = p + gridDim.x;
        const int t = grp.tid();
        if (mv.fcl && pn < io.B) {
          const char* base = reinterpret_cast<const char*>(mv.fcl + (int64_t)mv.model_of(pn) * F_COUNT * n);
          for (int off = t * 128; off < F_COUNT * n * (int)sizeof(double); off += cws::kPro * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
          for (int i = t; i < n; i += cws::kPro) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(io.q + (int64_t)i * io.lds + pn));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(io.qd + (int64_t)i * io.lds + pn));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(io.tau + (int64_t)i * io.lds + pn));
          }
        }
      }
      if (!first) asm volatile("bar.sync 4, %0;" ::"n"(cws::kAll) : "memory");  // rows done with the previous chain's rel
      first = false;
      const int64_t mc = mv.model_of(p);
      if (__ldg(mv.mstatus + mc) == PD_SLOT_OK) {
        const IdFields idf{cws::REL, cws::X, cws::V, cws::TMP, cws::TD};
        cta_kinematics(mv, io, p, mc, hand, idf, 2, grp);
        cta_bias_torque(mv, io, p, mc, hand, idf, 2, scan_pro, grp);  // ends with a group barrier
      }
      __threadfence_block();
      asm volatile("bar.arrive 3, %0;" ::"n"(cws::kAll) : "memory");
    }
    if (!first) asm volatile("bar.sync 4, %0;" ::"n"(cws::kAll) : "memory");  // the last chain's release
  }
}

bool cfa_ws_fits(int n) { return n > 128 && n <= 256; }

size_t cfa_ws_smem_bytes(int n) { return (size_t)(cfr::FIELDS + cws::FIELDS) * n * sizeof(double); }

void launch_cfa_ws(const ModelView& mv, const BatchIO& io, int sm_count, cudaStream_t s) {
  const size_t smem = cfa_ws_smem_bytes(mv.n);
  cudaFuncSetAttribute(cfa_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)(io.B < sm_count ? io.B : sm_count);
  cfa_ws_kernel<<<grid, cws::kAll, smem, s>>>(mv, io);
}

size_t cfa_workspace_bytes(int n) { return (size_t)cfa::FIELDS * n * sizeof(double); }

// Shared-memory workspace when the caller passes no global slots (n <= 256
// rows with the compact row kernel, the full workspace up to 220 KB), otherwise
// one global slot per CTA in flight, launched in waves of gws_slots CTAs.
void launch_cfa(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, cudaStream_t s,
                const double* td_pre) {
  const int n = mv.n;
  int nt = ((n + 31) / 32) * 32;
  if (nt > 256) nt = 256;
  const int lpt = (n + nt - 1) / nt;
  const size_t ws_bytes = cfa_workspace_bytes(n);
  if (n <= 256) {  // thread per row, compact workspace, register cap per size class
    const size_t rb = (size_t)cfr::FIELDS * n * sizeof(double);
    auto go = [&](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rb);
      int per_sm = 0, dev = 0;
      cudaGetDevice(&dev);
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, rb);
      kernel<<<(unsigned)io.B, nt, rb, s>>>(mv, io, td_pre, mv.fcl ? sms * (per_sm > 0 ? per_sm : 1) : 0);
    };
    // (a c5 sweep of 4 / 5 / 6 chains per SM: register caps that spill lose more
    // than the extra warps gain; 4 x 64 threads at <= 255 registers is best)
    if (nt <= 64)
      go(cfa_row_kernel<64, 4>);
    else if (nt <= 128)
      go(cfa_row_kernel<128, 2>);
    else
      go(cfa_row_kernel<256, 1>);
  } else if (gws_slots == 0) {
    cudaFuncSetAttribute(cfa_cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
    cfa_cta_kernel<true><<<(unsigned)io.B, nt, ws_bytes, s>>>(mv, io, nullptr, lpt, 0, td_pre);
  } else {
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      cfa_cta_kernel<false><<<(unsigned)nb, nt, 0, s>>>(mv, io, gws, lpt, b0, td_pre);
    }
  }
}

}  // namespace pd

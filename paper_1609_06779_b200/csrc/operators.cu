// The reference's per-chain operator builders as standalone batched device
// kernels, in the reference's dense representation (the public types of
// model.hpp / forward_dynamics.hpp: 6x6 adjoint matrices, 6x6 spatial
// inertias, 6x5 constraint bases, 5x5 / 5x1 operator blocks). The fused
// solve kernels never materialise these; they exist so the drop-in API's
// assemble_kinematics, link_inertias, articulated_body_inertias,
// build_constraint_basis, build_cfa_operators and CfaOperators::apply_* run on
// the device like the solves do.
//
// Layouts (all row-major blocks, problem-major arrays):
//   rel        [b][n][12]  R (9) then p (3)
//   transport  [b][n-1][36], base_transport [b][36]
//   screw      [b][n][6], inertia [b][n][36] (or [1][n][36] shared)
//   abi        [b][n][36], joint_inertia [b][n], gain [b][n][6]
//   basis      [k][30] (6x5)
//   cfa ops    diag [b][n][25], upper [b][n-1][25], cross_sub / cross_super
//              [b][n-1][5], cross_diag [b][n][5], joint_diag [b][n],
//              joint_off [b][n-1]
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "../../include/pardyn_c.h"

namespace pd {
namespace {

__device__ __forceinline__ void skew3(const double* a, double* m) {
  m[0] = 0.0;   m[1] = -a[2]; m[2] = a[1];
  m[3] = a[2];  m[4] = 0.0;   m[5] = -a[0];
  m[6] = -a[1]; m[7] = a[0];  m[8] = 0.0;
}

// C = A B for row-major R x K times K x C blocks.
template <int R, int K, int C>
__device__ __forceinline__ void mm(const double* A, const double* B, double* out) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(A[i * K + k], B[k * C + j], s);
      out[i * C + j] = s;
    }
}
// out = A^T B for A: K x R, B: K x C.
template <int R, int K, int C>
__device__ __forceinline__ void mtm(const double* A, const double* B, double* out) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(A[k * R + i], B[k * C + j], s);
      out[i * C + j] = s;
    }
}

// In-place lower Cholesky of a row-major 6x6 (Eigen LLT's test: a pivot
// x <= 0 fails, NaN passes through, forward_dynamics.cpp:302).
__device__ __forceinline__ bool chol6(double* L) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double x = L[k * 6 + k];
#pragma unroll
    for (int j = 0; j < k; ++j) x -= L[k * 6 + j] * L[k * 6 + j];
    if (x <= 0.0) ok = false;
    const double d = sqrt(x);
    L[k * 6 + k] = d;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      double v = L[i * 6 + k];
#pragma unroll
      for (int j = 0; j < k; ++j) v -= L[i * 6 + j] * L[k * 6 + j];
      L[i * 6 + k] = v / d;
    }
  }
  return ok;
}
// Solve L L^T x = b for the C columns of a row-major 6 x C block, in place.
template <int C>
__device__ __forceinline__ void chol6_solve(const double* L, double* b) {
#pragma unroll
  for (int c = 0; c < C; ++c) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double v = b[i * C + c];
#pragma unroll
      for (int j = 0; j < i; ++j) v -= L[i * 6 + j] * b[j * C + c];
      b[i * C + c] = v / L[i * 6 + i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
      double v = b[i * C + c];
#pragma unroll
      for (int j = i + 1; j < 6; ++j) v -= L[j * 6 + i] * b[j * C + c];
      b[i * C + c] = v / L[i * 6 + i];
    }
  }
}

// Adjoint of (R, p): [[R, 0], [skew(p) R, R]] (spatial.cpp:27-34).
__device__ __forceinline__ void adjoint6(const double* R, const double* p, double* A) {
  double px[9], pR[9];
  skew3(p, px);
  mm<3, 3, 3>(px, R, pR);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[r * 6 + c] = R[r * 3 + c];
      A[r * 6 + 3 + c] = 0.0;
      A[(3 + r) * 6 + c] = pR[r * 3 + c];
      A[(3 + r) * 6 + 3 + c] = R[r * 3 + c];
    }
}

// rel_i = screw_exp(S_i, -q_i) * home_i (model.cpp:117-146, spatial.cpp:43-68),
// in the reference's own Rodrigues form (no joint-aligned frames here).
__global__ void kinematics_kernel(const double* __restrict__ raw, int n, int64_t n_models, int64_t batch,
                                  const double* __restrict__ q, double* __restrict__ rel,
                                  double* __restrict__ base_transport, double* __restrict__ transport,
                                  double* __restrict__ screw) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * n) return;
  const int64_t p = t / n;
  const int i = (int)(t - p * n);
  const double* L = raw + ((n_models == 1 ? 0 : p) * n + i) * PD_LINK_FIELDS;
  const double* s = L + 13;
  const double* HR = L + 19;
  const double* hp = L + 28;
  const double qq = -q[t];
  const double wn = sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
  double ER[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, ep[3];
  if (wn < 1e-12) {
    for (int k = 0; k < 3; ++k) ep[k] = qq * s[3 + k];
  } else {
    double wx[9], wx2[9];
    skew3(s, wx);
    mm<3, 3, 3>(wx, wx, wx2);
    double st, ct;
    sincos(wn * qq, &st, &ct);
    const double a = st / wn, b = (1.0 - ct) / (wn * wn), c = (qq - st / wn) / (wn * wn);
    double V[9];
    for (int k = 0; k < 9; ++k) {
      ER[k] += a * wx[k] + b * wx2[k];
      V[k] = b * wx[k] + c * wx2[k];
    }
    V[0] += qq;
    V[4] += qq;
    V[8] += qq;
    mm<3, 3, 1>(V, s + 3, ep);
  }
  double R[9], pv[3];
  mm<3, 3, 3>(ER, HR, R);
  mm<3, 3, 1>(ER, hp, pv);
  for (int k = 0; k < 3; ++k) pv[k] += ep[k];
  double* o = rel + t * 12;
  for (int k = 0; k < 9; ++k) o[k] = R[k];
  for (int k = 0; k < 3; ++k) o[9 + k] = pv[k];
  for (int k = 0; k < 6; ++k) screw[t * 6 + k] = s[k];
  double A[36];
  adjoint6(R, pv, A);
  double* dst = i == 0 ? base_transport + p * 36 : transport + (p * (n - 1) + (i - 1)) * 36;
  for (int k = 0; k < 36; ++k) dst[k] = A[k];
}

// J = [[Ic + m cx cx^T, m cx], [m cx^T, m I]] (spatial.cpp:88-99).
__global__ void link_inertia_kernel(const double* __restrict__ raw, int64_t count, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const double* L = raw + t * PD_LINK_FIELDS;
  const double m = L[0];
  double cx[9], cc[9];
  skew3(L + 1, cx);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double v = 0.0;
      for (int k = 0; k < 3; ++k) v = fma(cx[r * 3 + k], cx[c * 3 + k], v);
      cc[r * 3 + c] = v;
    }
  double* J = out + t * 36;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      J[r * 6 + c] = L[4 + r * 3 + c] + m * cc[r * 3 + c];
      J[r * 6 + 3 + c] = m * cx[r * 3 + c];
      J[(3 + r) * 6 + c] = m * cx[c * 3 + r];
      J[(3 + r) * 6 + 3 + c] = r == c ? m : 0.0;
    }
}

// Articulated-body inertias, tip to base (forward_dynamics.cpp:120-163): one
// thread per chain carries I_i through the n-link recursion (the reference's
// longest_sequential_link_chain = n). Degenerate articulation -> slot code
// with the joint index.
__global__ void abi_kernel(int64_t batch, int n, const double* __restrict__ transport,
                           const double* __restrict__ inertia, int64_t inertia_stride,
                           const double* __restrict__ screw, double* __restrict__ abi,
                           double* __restrict__ joint_inertia, double* __restrict__ gain, int32_t* status,
                           int32_t* index) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= batch) return;
  double I[36], T[36], P[36], W[36];
  const double* J = inertia + p * inertia_stride;
  for (int k = 0; k < 36; ++k) I[k] = J[(int64_t)(n - 1) * 36 + k];
  int32_t st = PD_SLOT_OK, bad = 0;
  for (int i = n - 1; i >= 0; --i) {
    const double* s = screw + (p * n + i) * 6;
    double Is[6];
    mm<6, 6, 1>(I, s, Is);
    double lam = 0.0, tr = 0.0;
    for (int k = 0; k < 6; ++k) {
      lam = fma(s[k], Is[k], lam);
      tr += I[k * 7];
    }
    double* Io = abi + (p * n + i) * 36;
    for (int k = 0; k < 36; ++k) Io[k] = I[k];
    if (!(lam > 1e-14 * tr)) {
      st = PD_SLOT_DEGENERATE_ARTICULATION;
      bad = i;
      break;
    }
    joint_inertia[p * n + i] = lam;
    for (int k = 0; k < 6; ++k) gain[(p * n + i) * 6 + k] = Is[k] / lam;
    if (i == 0) break;
    // projected = I - (I s)(I s)^T / lambda, carried across joint i-1
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) P[r * 6 + c] = I[r * 6 + c] - Is[r] * Is[c] / lam;
    const double* Tg = transport + (p * (n - 1) + (i - 1)) * 36;
    for (int k = 0; k < 36; ++k) T[k] = Tg[k];
    mm<6, 6, 6>(P, T, W);       // P T
    mtm<6, 6, 6>(T, W, P);      // T^T P T
    const double* Jp = J + (int64_t)(i - 1) * 36;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) W[r * 6 + c] = Jp[r * 6 + c] + P[r * 6 + c];
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) I[r * 6 + c] = 0.5 * (W[r * 6 + c] + W[c * 6 + r]);
  }
  status[p] = st;
  index[p] = bad;
}

// Last five columns of the Householder Q of each screw, with Eigen's
// makeHouseholder / applyHouseholderOnTheLeft arithmetic
// (forward_dynamics.cpp:245-259): deterministic, orthonormal complement.
__global__ void basis_kernel(int64_t count, const double* __restrict__ screw, double* __restrict__ basis) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const double* s = screw + t * 6;
  double tail_sq = 0.0;
  for (int i = 1; i < 6; ++i) tail_sq += s[i] * s[i];
  const double c0 = s[0];
  double tau = 0.0, ess[5] = {0, 0, 0, 0, 0};
  if (tail_sq > DBL_MIN) {
    double beta = sqrt(c0 * c0 + tail_sq);
    if (c0 >= 0.0) beta = -beta;
    for (int i = 0; i < 5; ++i) ess[i] = s[i + 1] / (c0 - beta);
    tau = (beta - c0) / beta;
  }
  double* W = basis + t * 30;
  // Q = I - tau v v^T with v = (1, ess); column c of Q, c = 1..5
  for (int c = 1; c < 6; ++c) {
    double col[6] = {0, 0, 0, 0, 0, 0};
    col[c] = 1.0;
    if (tau != 0.0) {
      double tmp = col[0];
      for (int r = 1; r < 6; ++r) tmp += ess[r - 1] * col[r];
      col[0] -= tau * tmp;
      for (int r = 1; r < 6; ++r) col[r] -= tau * ess[r - 1] * tmp;
    }
    for (int r = 0; r < 6; ++r) W[r * 5 + (c - 1)] = col[r];
  }
}

// Link i's factor-solves: sb = J^-1 W (6x5), ss = J^-1 s, and for i < n-1
// the carried columns cb = T_i^T W_{i+1}, cs = T_i^T s_{i+1} with their solves.
struct LinkSolves {
  double sb[30], ss[6], cb[30], cs[6], scb[30], scs[6];
};

__device__ bool link_solves(int64_t p, int i, int n, const double* inertia, int64_t istride,
                            const double* transport, const double* screw, const double* basis, LinkSolves& o,
                            bool carried) {
  double L[36];
  const double* J = inertia + p * istride + (int64_t)i * 36;
  for (int k = 0; k < 36; ++k) L[k] = J[k];
  const bool ok = chol6(L);
  const double* W = basis + (p * n + i) * 30;
  const double* s = screw + (p * n + i) * 6;
  for (int k = 0; k < 30; ++k) o.sb[k] = W[k];
  for (int k = 0; k < 6; ++k) o.ss[k] = s[k];
  chol6_solve<5>(L, o.sb);
  chol6_solve<1>(L, o.ss);
  if (carried) {
    const double* T = transport + (p * (n - 1) + i) * 36;
    mtm<6, 6, 5>(T, basis + (p * n + i + 1) * 30, o.cb);
    mtm<6, 6, 1>(T, screw + (p * n + i + 1) * 6, o.cs);
    for (int k = 0; k < 30; ++k) o.scb[k] = o.cb[k];
    for (int k = 0; k < 6; ++k) o.scs[k] = o.cs[k];
    chol6_solve<5>(L, o.scb);
    chol6_solve<1>(L, o.scs);
  }
  return ok;
}

// CFA operators (forward_dynamics.cpp:261-357): thread per (chain, row). Row
// i's diagonal blocks need link i-1's carried solves, which the thread
// recomputes (no cross-thread dependency, no barrier).
__global__ void cfa_ops_kernel(int64_t batch, int n, const double* __restrict__ inertia, int64_t istride,
                               const double* __restrict__ transport, const double* __restrict__ screw,
                               const double* __restrict__ basis, double* __restrict__ diag,
                               double* __restrict__ upper, double* __restrict__ cross_sub,
                               double* __restrict__ cross_diag, double* __restrict__ cross_super,
                               double* __restrict__ joint_diag, double* __restrict__ joint_off, int32_t* bad_link) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * n) return;
  const int64_t p = t / n;
  const int i = (int)(t - p * n);
  LinkSolves own;
  bool ok = link_solves(p, i, n, inertia, istride, transport, screw, basis, own, i + 1 < n);
  const double* W = basis + t * 30;
  const double* s = screw + t * 6;
  double A[25], Bd[5], c = 0.0;
  mtm<5, 6, 5>(W, own.sb, A);
  mtm<5, 6, 1>(W, own.ss, Bd);
  for (int k = 0; k < 6; ++k) c = fma(s[k], own.ss[k], c);
  if (i > 0) {
    LinkSolves prev;
    ok = link_solves(p, i - 1, n, inertia, istride, transport, screw, basis, prev, true) && ok;
    double A2[25], B2[5];
    mtm<5, 6, 5>(prev.cb, prev.scb, A2);
    mtm<5, 6, 1>(prev.cb, prev.scs, B2);
    for (int k = 0; k < 25; ++k) A[k] += A2[k];
    for (int k = 0; k < 5; ++k) Bd[k] += B2[k];
    double c2 = 0.0;
    for (int k = 0; k < 6; ++k) c2 = fma(prev.cs[k], prev.scs[k], c2);
    c += c2;
  }
  if (!ok) atomicMin(bad_link + p, i);
  double* D = diag + t * 25;
  for (int r = 0; r < 5; ++r)
    for (int q = 0; q < 5; ++q) D[r * 5 + q] = 0.5 * (A[r * 5 + q] + A[q * 5 + r]);
  for (int k = 0; k < 5; ++k) cross_diag[t * 5 + k] = Bd[k];
  joint_diag[t] = c;
  if (i + 1 < n) {
    const int64_t e = p * (n - 1) + i;
    double U[25], Bs[5], Bb[5];
    mtm<5, 6, 5>(W, own.scb, U);
    mtm<5, 6, 1>(W, own.scs, Bs);
    mtm<5, 6, 1>(own.cb, own.ss, Bb);
    for (int k = 0; k < 25; ++k) upper[e * 25 + k] = -U[k];
    for (int k = 0; k < 5; ++k) {
      cross_super[e * 5 + k] = -Bs[k];
      cross_sub[e * 5 + k] = -Bb[k];
    }
    double jo = 0.0;
    for (int k = 0; k < 6; ++k) jo = fma(s[k], own.scs[k], jo);
    joint_off[e] = -jo;
  }
}

// CfaOperators::apply_cross / apply_cross_transpose / apply_joint
// (forward_dynamics.cpp:359-416): tri-diagonal stencils, thread per (chain, row).
__global__ void cfa_apply_kernel(int op, int64_t batch, int n, const double* __restrict__ cross_sub,
                                 const double* __restrict__ cross_diag, const double* __restrict__ cross_super,
                                 const double* __restrict__ joint_diag, const double* __restrict__ joint_off,
                                 const double* __restrict__ in, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * n) return;
  const int64_t p = t / n;
  const int i = (int)(t - p * n);
  const int64_t e = p * (n - 1);
  if (op == 0) {  // v (n) -> B v (n x 5)
    double v[5];
    for (int k = 0; k < 5; ++k) v[k] = in[t] * cross_diag[t * 5 + k];
    if (i > 0)
      for (int k = 0; k < 5; ++k) v[k] += in[t - 1] * cross_sub[(e + i - 1) * 5 + k];
    if (i + 1 < n)
      for (int k = 0; k < 5; ++k) v[k] += in[t + 1] * cross_super[(e + i) * 5 + k];
    for (int k = 0; k < 5; ++k) out[t * 5 + k] = v[k];
  } else if (op == 1) {  // f (n x 5) -> B^T f (n)
    double v = 0.0;
    for (int k = 0; k < 5; ++k) v += cross_diag[t * 5 + k] * in[t * 5 + k];
    if (i + 1 < n) {
      double w = 0.0;
      for (int k = 0; k < 5; ++k) w += cross_sub[(e + i) * 5 + k] * in[(t + 1) * 5 + k];
      v += w;
    }
    if (i > 0) {
      double w = 0.0;
      for (int k = 0; k < 5; ++k) w += cross_super[(e + i - 1) * 5 + k] * in[(t - 1) * 5 + k];
      v += w;
    }
    out[t] = v;
  } else {  // v (n) -> C v (n)
    double v = joint_diag[t] * in[t];
    if (i > 0) v += joint_off[e + i - 1] * in[t - 1];
    if (i + 1 < n) v += joint_off[e + i] * in[t + 1];
    out[t] = v;
  }
}

// small_adjoint(V) x = (w x xa, v x xa + w x xl) and its transpose applied to f:
// ad(V)^T f = (-(w x fa) - (v x fl), -(w x fl))   (spatial.cpp:18-25)
__device__ __forceinline__ void adv_mul(const double* V, const double* x, double* o) {
  const double* w = V;
  const double* v = V + 3;
  double c1[3], c2[3], c3[3];
  auto cross = [](const double* a, const double* b, double* r) {
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
  };
  cross(w, x, c1);
  cross(v, x, c2);
  cross(w, x + 3, c3);
  for (int k = 0; k < 3; ++k) {
    o[k] = c1[k];
    o[3 + k] = c2[k] + c3[k];
  }
}
__device__ __forceinline__ void advT_mul(const double* V, const double* f, double* o) {
  const double* w = V;
  const double* v = V + 3;
  auto cross = [](const double* a, const double* b, double* r) {
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
  };
  double c1[3], c2[3], c3[3];
  cross(w, f, c1);
  cross(v, f + 3, c2);
  cross(w, f + 3, c3);
  for (int k = 0; k < 3; ++k) {
    o[k] = -c1[k] - c2[k];
    o[3 + k] = -c3[k];
  }
}

// The three propagations of inverse_dynamics.cpp:27-120 as block bi-diagonal
// systems (the reference solves them with its scan): this kernel builds the
// couplings and right-hand sides, thread per (problem, link), and the system
// goes to bidiag6_kernel (the building-block scan).
//   kind 0 velocities    lower, coupling transport[i-1], rhs qd_i S_i (+ Ad_base V_base at i = 0)
//   kind 1 accelerations lower, rhs qdd_i S_i + ad_{V_i}(qd_i S_i) (+ Ad_base A_base)
//   kind 2 forces        upper, coupling transport[i]^T, rhs J_i A_i - ad_{V_i}^T (J_i V_i) (+ tip at n-1)
__global__ void propagate_setup_kernel(int kind, int64_t batch, int n, const double* __restrict__ base_transport,
                                       const double* __restrict__ transport, const double* __restrict__ screw,
                                       const double* __restrict__ inertia, int64_t istride,
                                       const double* __restrict__ qdot, const double* __restrict__ qddot,
                                       const double* __restrict__ vel, const double* __restrict__ acc,
                                       const double* __restrict__ boundary, double* __restrict__ coupling,
                                       double* __restrict__ rhs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * n) return;
  const int64_t p = t / n;
  const int i = (int)(t - p * n);
  const double* S = screw + t * 6;
  double r[6];
  if (kind == 0 || kind == 1) {
    const double qd = qdot[t];
    for (int k = 0; k < 6; ++k) r[k] = (kind == 0 ? qd : qddot[t]) * S[k];
    if (kind == 1) {
      double rate[6], a[6];
      for (int k = 0; k < 6; ++k) rate[k] = qd * S[k];
      adv_mul(vel + t * 6, rate, a);
      for (int k = 0; k < 6; ++k) r[k] += a[k];
    }
    if (i == 0) {
      double b[6];
      mm<6, 6, 1>(base_transport + p * 36, boundary, b);
      for (int k = 0; k < 6; ++k) r[k] += b[k];
    }
    if (i >= 1) {
      const double* T = transport + (p * (n - 1) + (i - 1)) * 36;
      double* C = coupling + (p * (n - 1) + (i - 1)) * 36;
      for (int k = 0; k < 36; ++k) C[k] = T[k];
    }
  } else {
    const double* J = inertia + p * istride + (int64_t)i * 36;
    double JA[6], JV[6], adf[6];
    mm<6, 6, 1>(J, acc + t * 6, JA);
    mm<6, 6, 1>(J, vel + t * 6, JV);
    advT_mul(vel + t * 6, JV, adf);
    for (int k = 0; k < 6; ++k) r[k] = JA[k] - adf[k];  // J A - ad_V^T (J V)   (inverse_dynamics.cpp:105-111)
    if (i == n - 1)
      for (int k = 0; k < 6; ++k) r[k] += boundary[k];
    if (i + 1 < n) {
      const double* T = transport + (p * (n - 1) + i) * 36;
      double* C = coupling + (p * (n - 1) + i) * 36;
      for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b) C[a * 6 + b] = T[b * 6 + a];
    }
  }
  for (int k = 0; k < 6; ++k) rhs[t * 6 + k] = r[k];
}

__global__ void fill_i32_kernel(int32_t* a, int64_t count, int32_t v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) a[t] = v;
}

unsigned blocks_for(int64_t work, int threads) { return (unsigned)((work + threads - 1) / threads); }

}  // namespace

void launch_kinematics(const double* raw, int n, int64_t n_models, int64_t batch, const double* q, double* rel,
                       double* base_transport, double* transport, double* screw, cudaStream_t s) {
  kinematics_kernel<<<blocks_for(batch * n, 128), 128, 0, s>>>(raw, n, n_models, batch, q, rel, base_transport,
                                                                transport, screw);
}
void launch_link_inertias(const double* raw, int64_t count, double* out, cudaStream_t s) {
  link_inertia_kernel<<<blocks_for(count, 128), 128, 0, s>>>(raw, count, out);
}
void launch_abi(int64_t batch, int n, const double* transport, const double* inertia, int64_t inertia_stride,
                const double* screw, double* abi, double* joint_inertia, double* gain, int32_t* status,
                int32_t* index, cudaStream_t s) {
  abi_kernel<<<blocks_for(batch, 64), 64, 0, s>>>(batch, n, transport, inertia, inertia_stride, screw, abi,
                                                  joint_inertia, gain, status, index);
}
void launch_basis(int64_t count, const double* screw, double* basis, cudaStream_t s) {
  basis_kernel<<<blocks_for(count, 128), 128, 0, s>>>(count, screw, basis);
}
void launch_cfa_ops(int64_t batch, int n, const double* inertia, int64_t istride, const double* transport,
                    const double* screw, const double* basis, double* diag, double* upper, double* cross_sub,
                    double* cross_diag, double* cross_super, double* joint_diag, double* joint_off, int32_t* bad_link,
                    cudaStream_t s) {
  fill_i32_kernel<<<blocks_for(batch, 256), 256, 0, s>>>(bad_link, batch, n);
  cfa_ops_kernel<<<blocks_for(batch * n, 64), 64, 0, s>>>(batch, n, inertia, istride, transport, screw, basis, diag,
                                                          upper, cross_sub, cross_diag, cross_super, joint_diag,
                                                          joint_off, bad_link);
}
void launch_propagate_setup(int kind, int64_t batch, int n, const double* base_transport, const double* transport,
                            const double* screw, const double* inertia, int64_t istride, const double* qdot,
                            const double* qddot, const double* vel, const double* acc, const double* boundary,
                            double* coupling, double* rhs, cudaStream_t s) {
  propagate_setup_kernel<<<blocks_for(batch * n, 128), 128, 0, s>>>(kind, batch, n, base_transport, transport, screw,
                                                                     inertia, istride, qdot, qddot, vel, acc, boundary,
                                                                     coupling, rhs);
}
void launch_cfa_apply(int op, int64_t batch, int n, const double* cross_sub, const double* cross_diag,
                      const double* cross_super, const double* joint_diag, const double* joint_off, const double* in,
                      double* out, cudaStream_t s) {
  cfa_apply_kernel<<<blocks_for(batch * n, 128), 128, 0, s>>>(op, batch, n, cross_sub, cross_diag, cross_super,
                                                               joint_diag, joint_off, in, out);
}

}  // namespace pd

// Device-side spatial algebra for the batched forward-dynamics kernels.
//
// Everything is FP64 and structure-aware: transforms stay as (R, p) and are
// applied through cross products instead of dense 6x6 adjoints, spatial
// inertias are applied from (m, c, Ic), symmetric 6x6 articulated inertias
// are kept as three 3x3 blocks (21 doubles). Conventions follow the
// reference (proj/core/include/pardyn/spatial.hpp:7-10, src/spatial.cpp):
// twists stack (angular, linear), wrenches (moment, force),
// Ad(R,p) = [[R,0],[p^R,R]], ad_V = [[w^,0],[v^,w^]].
#pragma once

#include <cstdint>

#include "../../include/pardyn_c.h"

namespace pd {

// Packed device model record, 21 doubles per link, stored SoA as
// model[(field * n_links + link) * n_models + chain] (chain fastest), in the
// joint-aligned link frames of capi.cu pack_models_kernel: the screw is
// (0, 0, w, vx, 0, vz) and only its three free components are stored, with
// 1/w beside them; the home rotation is a unit quaternion (4 doubles instead
// of 9: the model is streamed from HBM once per pass, so every field is
// bandwidth). The kinematic fields F_SW..F_HP are contiguous.
enum ModelField : int {
  F_MASS = 0,
  F_COM = 1,    // 3
  F_IC = 4,     // 6: xx xy xz yy yz zz (rotational inertia about the COM)
  F_SW = 10,    // |w| of the joint screw
  F_SVX = 11,   // v'x
  F_SVZ = 12,   // v'z
  F_SIW = 13,   // 1/|w| (0 for a pure translation, |w| < 1e-12)
  F_HQ = 14,    // 4: home rotation as a unit quaternion (w, x, y, z)
  F_HP = 18,    // 3: home translation
  F_COUNT = 21,
  F_KIN = F_SW,     // first kinematic field
  F_NKIN = 11       // kinematic fields (screw, 1/w, home)
};

struct Vec3d {
  double x, y, z;
};

__device__ __forceinline__ Vec3d mk(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ Vec3d operator+(Vec3d a, Vec3d b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ Vec3d operator-(Vec3d a, Vec3d b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ Vec3d operator*(double s, Vec3d a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(Vec3d a, Vec3d b) { return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ Vec3d cross(Vec3d a, Vec3d b) {
  return {fma(a.y, b.z, -a.z * b.y), fma(a.z, b.x, -a.x * b.z), fma(a.x, b.y, -a.y * b.x)};
}
__device__ __forceinline__ Vec3d fmav(double s, Vec3d a, Vec3d b) {  // s*a + b
  return {fma(s, a.x, b.x), fma(s, a.y, b.y), fma(s, a.z, b.z)};
}

// acc + a x b, fused (2 FMA per component, no separate multiply / add)
__device__ __forceinline__ Vec3d cross_acc(Vec3d a, Vec3d b, Vec3d acc) {
  return {fma(a.y, b.z, fma(-a.z, b.y, acc.x)), fma(a.z, b.x, fma(-a.x, b.z, acc.y)),
          fma(a.x, b.y, fma(-a.y, b.x, acc.z))};
}

// 3x3 row-major rotation.
struct Mat3d {
  double m[9];
};
__device__ __forceinline__ Vec3d mul(const Mat3d& R, Vec3d v) {
  return {fma(R.m[0], v.x, fma(R.m[1], v.y, R.m[2] * v.z)), fma(R.m[3], v.x, fma(R.m[4], v.y, R.m[5] * v.z)),
          fma(R.m[6], v.x, fma(R.m[7], v.y, R.m[8] * v.z))};
}
__device__ __forceinline__ Vec3d mulT(const Mat3d& R, Vec3d v) {
  return {fma(R.m[0], v.x, fma(R.m[3], v.y, R.m[6] * v.z)), fma(R.m[1], v.x, fma(R.m[4], v.y, R.m[7] * v.z)),
          fma(R.m[2], v.x, fma(R.m[5], v.y, R.m[8] * v.z))};
}
__device__ __forceinline__ Vec3d mul_acc(const Mat3d& R, Vec3d v, Vec3d acc) {
  return {fma(R.m[0], v.x, fma(R.m[1], v.y, fma(R.m[2], v.z, acc.x))),
          fma(R.m[3], v.x, fma(R.m[4], v.y, fma(R.m[5], v.z, acc.y))),
          fma(R.m[6], v.x, fma(R.m[7], v.y, fma(R.m[8], v.z, acc.z)))};
}
__device__ __forceinline__ Mat3d matmul(const Mat3d& A, const Mat3d& B) {
  Mat3d C;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C.m[3 * r + c] = fma(A.m[3 * r], B.m[c], fma(A.m[3 * r + 1], B.m[3 + c], A.m[3 * r + 2] * B.m[6 + c]));
  return C;
}

// Rotation matrix of a unit quaternion (w, x, y, z).
__device__ __forceinline__ Mat3d quat_to_R(double w, double x, double y, double z) {
  const double x2 = x + x, y2 = y + y, z2 = z + z;
  const double xx = x * x2, yy = y * y2, zz = z * z2, xy = x * y2, xz = x * z2, yz = y * z2, wx = w * x2,
               wy = w * y2, wz = w * z2;
  Mat3d R;
  R.m[0] = 1.0 - (yy + zz);
  R.m[1] = xy - wz;
  R.m[2] = xz + wy;
  R.m[3] = xy + wz;
  R.m[4] = 1.0 - (xx + zz);
  R.m[5] = yz - wx;
  R.m[6] = xz - wy;
  R.m[7] = yz + wx;
  R.m[8] = 1.0 - (xx + yy);
  return R;
}

struct SE3d {
  Mat3d R;
  Vec3d p;
};

// Spatial 6-vectors as (angular/moment, linear/force) 3-vector pairs.
struct Sv {
  Vec3d a, l;
};
__device__ __forceinline__ Sv operator+(const Sv& x, const Sv& y) { return {x.a + y.a, x.l + y.l}; }
__device__ __forceinline__ Sv operator-(const Sv& x, const Sv& y) { return {x.a - y.a, x.l - y.l}; }
__device__ __forceinline__ Sv operator*(double s, const Sv& x) { return {s * x.a, s * x.l}; }
__device__ __forceinline__ double dot(const Sv& x, const Sv& y) { return dot(x.a, y.a) + dot(x.l, y.l); }
__device__ __forceinline__ Sv svzero() { return {mk(0, 0, 0), mk(0, 0, 0)}; }

// Ad(R,p) x = (R w, R v + p x (R w))                         spatial.cpp:27-34
__device__ __forceinline__ Sv ad_apply(const SE3d& T, const Sv& x) {
  const Vec3d rw = mul(T.R, x.a);
  return {rw, mul(T.R, x.l) + cross(T.p, rw)};
}
// Ad(R,p)^T f = (R^T (m - p x f), R^T f)
__device__ __forceinline__ Sv adT_apply(const SE3d& T, const Sv& f) {
  return {mulT(T.R, f.a - cross(T.p, f.l)), mulT(T.R, f.l)};
}
// Ad(R,p)^{-1} x = (R^T w, R^T (v - p x w))
__device__ __forceinline__ Sv adinv_apply(const SE3d& T, const Sv& x) {
  return {mulT(T.R, x.a), mulT(T.R, x.l - cross(T.p, x.a))};
}
// Ad(R,p)^{-T} f = (R m + p x (R f), R f)   (wrench carried from link to base coords)
__device__ __forceinline__ Sv adinvT_apply(const SE3d& T, const Sv& f) {
  const Vec3d rf = mul(T.R, f.l);
  return {mul(T.R, f.a) + cross(T.p, rf), rf};
}
// ad_V x = (w x xw, v x xw + w x xv)                           spatial.cpp:18-25
__device__ __forceinline__ Sv adv_apply(const Sv& V, const Sv& x) {
  return {cross(V.a, x.a), cross(V.l, x.a) + cross(V.a, x.l)};
}
// acc + ad_V x
__device__ __forceinline__ Sv adv_acc(const Sv& V, const Sv& x, const Sv& acc) {
  return {cross_acc(V.a, x.a, acc.a), cross_acc(V.a, x.l, cross_acc(V.l, x.a, acc.l))};
}
// acc + s x
__device__ __forceinline__ Sv svfma(double s, const Sv& x, const Sv& acc) {
  return {fmav(s, x.a, acc.a), fmav(s, x.l, acc.l)};
}
// -ad_V^T h = (w x ha + v x hl, w x hl)
__device__ __forceinline__ Sv neg_advT_apply(const Sv& V, const Sv& h) {
  return {cross(V.a, h.a) + cross(V.l, h.l), cross(V.a, h.l)};
}
// Compose (a*b)(x) = a(b(x))                                     spatial.hpp:80-82
__device__ __forceinline__ SE3d compose(const SE3d& a, const SE3d& b) {
  return {matmul(a.R, b.R), mul(a.R, b.p) + a.p};
}

// Link inertia parameters; J = [[Ic + m c^ c^T, m c^], [m c^T, m I]].
struct Inertia {
  double m;
  Vec3d c;
  double I[6];  // xx xy xz yy yz zz
};
__device__ __forceinline__ Vec3d sym3_mul(const double* I, Vec3d w) {
  return {fma(I[0], w.x, fma(I[1], w.y, I[2] * w.z)), fma(I[1], w.x, fma(I[3], w.y, I[4] * w.z)),
          fma(I[2], w.x, fma(I[4], w.y, I[5] * w.z))};
}
__device__ __forceinline__ Vec3d sym3_mul_acc(const double* I, Vec3d w, Vec3d acc) {
  return {fma(I[0], w.x, fma(I[1], w.y, fma(I[2], w.z, acc.x))), fma(I[1], w.x, fma(I[3], w.y, fma(I[4], w.z, acc.y))),
          fma(I[2], w.x, fma(I[4], w.y, fma(I[5], w.z, acc.z)))};
}
// J (w, v): lin = m (v - c x w); ang = Ic w + c x lin
__device__ __forceinline__ Sv inertia_apply(const Inertia& J, const Sv& x) {
  const Vec3d lin = J.m * (x.l - cross(J.c, x.a));
  return {sym3_mul(J.I, x.a) + cross(J.c, lin), lin};
}
// acc + J x, fused
__device__ __forceinline__ Sv inertia_apply_acc(const Inertia& J, const Sv& x, const Sv& acc) {
  const Vec3d lin = J.m * cross_acc(x.a, J.c, x.l);  // m (v - c x w) = m (v + w x c)
  return {cross_acc(J.c, lin, sym3_mul_acc(J.I, x.a, acc.a)), acc.l + lin};
}
// acc - ad_V^T h = acc + (w x ha + v x hl, w x hl), fused
__device__ __forceinline__ Sv neg_advT_acc(const Sv& V, const Sv& h, const Sv& acc) {
  return {cross_acc(V.a, h.a, cross_acc(V.l, h.l, acc.a)), cross_acc(V.a, h.l, acc.l)};
}

// Symmetric 6x6 as blocks [[A, B], [B^T, D]]; A, D packed sym (xx xy xz yy yz zz),
// B row-major 3x3.
struct Sym6 {
  double A[6];
  double B[9];
  double D[6];
};
__device__ __forceinline__ Sv sym6_apply(const Sym6& P, const Sv& x) {
  const Vec3d bl = mul(*reinterpret_cast<const Mat3d*>(P.B), x.l);
  const Vec3d btw = mulT(*reinterpret_cast<const Mat3d*>(P.B), x.a);
  return {sym3_mul(P.A, x.a) + bl, btw + sym3_mul(P.D, x.l)};
}
__device__ __forceinline__ double sym6_trace(const Sym6& P) { return P.A[0] + P.A[3] + P.A[5] + P.D[0] + P.D[3] + P.D[5]; }

// Explicit J as Sym6 (spatial.cpp:89-98: Ic + m * (cx cx^T), m cx, m I).
__device__ __forceinline__ Sym6 inertia_sym6(const Inertia& J) {
  Sym6 P;
  const double cx = J.c.x, cy = J.c.y, cz = J.c.z;
  // cx^ cx^T = |c|^2 I - c c^T
  const double c2 = fma(cx, cx, fma(cy, cy, cz * cz));
  P.A[0] = fma(J.m, c2 - cx * cx, J.I[0]);
  P.A[1] = fma(J.m, -cx * cy, J.I[1]);
  P.A[2] = fma(J.m, -cx * cz, J.I[2]);
  P.A[3] = fma(J.m, c2 - cy * cy, J.I[3]);
  P.A[4] = fma(J.m, -cy * cz, J.I[4]);
  P.A[5] = fma(J.m, c2 - cz * cz, J.I[5]);
  // m c^ = m [[0,-cz,cy],[cz,0,-cx],[-cy,cx,0]]
  P.B[0] = 0.0;        P.B[1] = -J.m * cz; P.B[2] = J.m * cy;
  P.B[3] = J.m * cz;   P.B[4] = 0.0;       P.B[5] = -J.m * cx;
  P.B[6] = -J.m * cy;  P.B[7] = J.m * cx;  P.B[8] = 0.0;
  P.D[0] = J.m; P.D[1] = 0.0; P.D[2] = 0.0; P.D[3] = J.m; P.D[4] = 0.0; P.D[5] = J.m;
  return P;
}

// R^T S R for symmetric packed S -> symmetric packed.
__device__ __forceinline__ void sym3_congruence(const double* S, const Mat3d& R, double* out) {
  // T = S R (3x3)
  double T[9];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const Vec3d col = sym3_mul(S, mk(R.m[c], R.m[3 + c], R.m[6 + c]));
    T[c] = col.x;
    T[3 + c] = col.y;
    T[6 + c] = col.z;
  }
  // out = R^T T
  const int idx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int r = idx[k][0], c = idx[k][1];
    out[k] = fma(R.m[r], T[c], fma(R.m[3 + r], T[3 + c], R.m[6 + r] * T[6 + c]));
  }
}

// Ad(T)^T P Ad(T) for symmetric P (articulated-inertia carry across a joint,
// forward_dynamics.cpp:150-156). Shift of reference point by p, then rotation:
//   Y = B - p^ D ; X11 = A - p^ B^T + Y p^ ; out = (R^T X11 R, R^T Y R, R^T D R).
__device__ __forceinline__ Sym6 sym6_congruence(const Sym6& P, const SE3d& T) {
  const Vec3d p = T.p;
  double Y[9];
  // columns of p^ D: p x D[:,j]
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int j0 = j == 0 ? 0 : (j == 1 ? 1 : 2);
    const int j1 = j == 0 ? 1 : (j == 1 ? 3 : 4);
    const int j2 = j == 0 ? 2 : (j == 1 ? 4 : 5);
    const Vec3d dcol = mk(P.D[j0], P.D[j1], P.D[j2]);
    const Vec3d pd = cross(p, dcol);
    Y[j] = P.B[j] - pd.x;
    Y[3 + j] = P.B[3 + j] - pd.y;
    Y[6 + j] = P.B[6 + j] - pd.z;
  }
  // K = p^ B^T : column j of B^T is row j of B
  double K[9];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const Vec3d pb = cross(p, mk(P.B[3 * j], P.B[3 * j + 1], P.B[3 * j + 2]));
    K[j] = pb.x;
    K[3 + j] = pb.y;
    K[6 + j] = pb.z;
  }
  // W = Y p^ : row r of W = -(p x Y[r,:])
  double W[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const Vec3d py = cross(p, mk(Y[3 * r], Y[3 * r + 1], Y[3 * r + 2]));
    W[3 * r] = -py.x;
    W[3 * r + 1] = -py.y;
    W[3 * r + 2] = -py.z;
  }
  double X11[6];
  X11[0] = P.A[0] - K[0] + W[0];
  X11[1] = P.A[1] - 0.5 * (K[1] + K[3]) + 0.5 * (W[1] + W[3]);
  X11[2] = P.A[2] - 0.5 * (K[2] + K[6]) + 0.5 * (W[2] + W[6]);
  X11[3] = P.A[3] - K[4] + W[4];
  X11[4] = P.A[4] - 0.5 * (K[5] + K[7]) + 0.5 * (W[5] + W[7]);
  X11[5] = P.A[5] - K[8] + W[8];
  Sym6 out;
  sym3_congruence(X11, T.R, out.A);
  sym3_congruence(P.D, T.R, out.D);
  // R^T Y R
  double T1[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      T1[3 * r + c] = fma(Y[3 * r], T.R.m[c], fma(Y[3 * r + 1], T.R.m[3 + c], Y[3 * r + 2] * T.R.m[6 + c]));
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      out.B[3 * r + c] = fma(T.R.m[r], T1[c], fma(T.R.m[3 + r], T1[3 + c], T.R.m[6 + r] * T1[6 + c]));
  return out;
}

// Joint transform rel = screw_exp(S, -q) * home                 model.cpp:117-146
// screw_exp: Rodrigues for a not-necessarily-unit angular part, pure
// translation if |w| < 1e-12                                     spatial.cpp:43-68
// Packed models live in joint-aligned frames (capi.cu pack_models_kernel):
// S = (0, 0, w, vx, 0, vz) with w = |w| >= 0, so exp(-q S) is a rotation by
// theta = -w q about z plus t = (vx sin(theta)/w, vx (1 - cos(theta))/w, -q vz)
// (the reference's R = I + a w^ + b w^2, t = (q I + b w^ + c w^2) v with the
// zeros of S substituted), and rel = (E H, E h + t) mixes only two rows.
// joint_angle_sincos gives (sin, cos) of theta (the expensive,
// history-independent part); joint_transform_sc assembles rel from it.
// sin / cos of x: Cody-Waite reduction by pi/2 (three-part constant, exact
// products through FMA) and the fdlibm minimax kernels on [-pi/4, pi/4]
// evaluated in Estrin form, so the dependent chain is ~10 FP64 ops instead of
// a Horner chain (the joint angle sits on every pass's critical path). Error
// <= ~1 ulp, like the reference's libm sin/cos. |x| > 2^20 (never a joint
// angle in practice) falls back to the CUDA routine.
__device__ __forceinline__ void fast_sincos(double x, double* s, double* c) {
  if (!(fabs(x) < 1048576.0)) {
    sincos(x, s, c);
    return;
  }
  const double j = rint(x * 0.63661977236758134308);  // 2/pi
  // pi/2 = pio2_1 (33 bits) + pio2_2 (33 bits) + pio2_2t (fdlibm's split):
  // j * pio2_1 and j * pio2_2 are exact for |j| < 2^20, the FMAs round once
  double r = fma(-j, 1.57079632673412561417e+00, x);
  r = fma(-j, 6.07710050630396597660e-11, r);
  r = fma(-j, 2.02226624879595063154e-21, r);
  const double z = r * r, z2 = z * z, z4 = z2 * z2;
  const double ps = fma(z4, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                        fma(z2, fma(z, 2.75573137070700676789e-06, -1.98412698298579493134e-04),
                            fma(z, 8.33333333332248946124e-03, -1.66666666666666324348e-01)));
  // cos kernel: 1 - z/2 + z^2 (C1 + z C2 + z^2 C3 + z^3 C4 + z^4 C5 + z^5 C6)
  const double qc = fma(z4, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                        fma(z2, fma(z, -2.75573143513906633035e-07, 2.48015872894767294178e-05),
                            fma(z, -1.38888888888741095749e-03, 4.16666666666666019037e-02)));
  const double sr = fma(r * z, ps, r);
  const double cr = fma(z2, qc, fma(-0.5, z, 1.0));
  const int qd = (int)(((long long)j) & 3);
  const double sa = (qd & 1) ? cr : sr, ca = (qd & 1) ? sr : cr;
  *s = (qd & 2) ? -sa : sa;
  *c = ((qd + 1) & 2) ? -ca : ca;
}

__device__ __forceinline__ void joint_angle_sincos(const Sv& S, double q, double* st, double* ct) {
  const double w = S.a.z;
  if (w * w < 1e-24) {
    *st = 0.0;
    *ct = 1.0;
    return;
  }
  fast_sincos(w * (-q), st, ct);
}

// iw = 1/w from the packed model (F_SIW)
__device__ __forceinline__ SE3d joint_transform_sc(const Sv& S, double iw, const Mat3d& HR, Vec3d hp, double q,
                                                   double st, double ct) {
  const double w = S.a.z, vx = S.l.x, vz = S.l.z;
  Vec3d t;
  double c = ct, s = st;
  if (w * w < 1e-24) {  // |w| < 1e-12: pure translation
    c = 1.0;
    s = 0.0;
    t = mk(-q * vx, 0.0, -q * vz);
  } else {
    t = mk(vx * (st * iw), vx * ((1.0 - ct) * iw), -q * vz);
  }
  SE3d T;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T.R.m[k] = fma(c, HR.m[k], -s * HR.m[3 + k]);
    T.R.m[3 + k] = fma(s, HR.m[k], c * HR.m[3 + k]);
    T.R.m[6 + k] = HR.m[6 + k];
  }
  T.p = mk(fma(c, hp.x, fma(-s, hp.y, t.x)), fma(s, hp.x, fma(c, hp.y, t.y)), hp.z + t.z);
  return T;
}

__device__ __forceinline__ SE3d joint_transform(const Sv& S, double iw, const Mat3d& HR, Vec3d hp, double q) {
  double st, ct;
  joint_angle_sincos(S, q, &st, &ct);
  return joint_transform_sc(S, iw, HR, hp, q, st, ct);
}

// 1/x without the division routine's branches: the hardware approximation
// (rel. error ~1e-6) and two Newton steps (exact to the last bit in a 3.2M-
// sample probe against 1.0 / x, tools/micro/rcp_probe.cu).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}


// 1/sqrt(x) without the library routine's range-check branch: the hardware
// approximation (rel. error ~1e-6) refined to ~1 ulp (below). Used on pivot
// chains of the factorizations, where a CALL to the slow path would split the
// unrolled code into blocks. (A/B: c2j -1.9 %, c5c -1.1 %, c3 -0.5 % against
// two Newton steps.)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // one third-order step y (1 + e/2 + 3e^2/8), e = 1 - x y^2: the hardware's
  // ~1e-6 becomes ~1e-18 before rounding (max rel. error 2.2e-16 measured,
  // tools/micro/rsqrt_probe.cu; two Newton steps: 2.6e-16), 5 operations
  // instead of 8
  const double e = fma(-x, y * y, 1.0);
  return fma(y, fma(0.375, e, 0.5) * e, y);
}

// joint screw from its stored components
__device__ __forceinline__ Sv joint_screw(double w, double vx, double vz) { return {mk(0.0, 0.0, w), mk(vx, 0.0, vz)}; }

// Ad(R,p)^{-1} S for a joint-aligned screw S = (0, 0, w, vx, 0, vz):
// (w R^T e_z, R^T (v - p x w e_z)), p x (w e_z) = w (py, -px, 0)
__device__ __forceinline__ Sv adinv_screw(const SE3d& T, const Sv& S) {
  const double w = S.a.z;
  const Vec3d u = mk(fma(-w, T.p.y, S.l.x), w * T.p.x, S.l.z);
  return {mk(w * T.R.m[6], w * T.R.m[7], w * T.R.m[8]), mulT(T.R, u)};
}

// Kernel-side error record: first failure wins per slot.
__device__ __forceinline__ void set_slot_error(int32_t* status, int32_t* eround, int32_t* eindex, int64_t slot,
                                               int code, int round, int index) {
  if (status[slot] == PD_SLOT_OK) {
    status[slot] = code;
    eround[slot] = round;
    eindex[slot] = index;
  }
}

__device__ __forceinline__ int ceil_log2_dev(int n) { return n <= 1 ? 0 : 32 - __clz(n - 1); }

}  // namespace pd

// Joint-aligned link frames shared by the model packer (capi.cu) and the
// kernels that report link-frame quantities in the reference's frames
// (idyn.cu: link states, tip wrench).
#pragma once

#include "pd_batch.cuh"

namespace pd {

// Joint-aligned link frames. Link i's coordinates are re-expressed in a
// rotated frame F'_i = Q_i F_i (same origin) chosen so that its screw reads
// S' = Ad(Q_i) S = (0, 0, |w|, v'x, 0, v'z): z' along the rotation axis (or
// along v for a pure prismatic screw) and x' along the part of v normal to
// it. The chain is physically unchanged: rel'_i = Q_i rel_i Q_{i-1}^T with
// home' = (Q_i R_h Q_{i-1}^T, Q_i p_h), com' = Q_i c, Ic' = Q_i Ic Q_i^T, and
// the base frame (Q_{-1} = I, gravity) untouched. Joint-space results (qdd,
// tau, M, lambda, traces about the link origin) are frame invariant; the
// kernels exploit the zeros: exp(-q S') is a rotation about z plus a
// translation in the x-z plane (pd_common.cuh joint_transform_sc).
__device__ inline void joint_frame(const double* s, double Q[9], double sz[3]) {
  const double w2 = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
  const double v2 = s[3] * s[3] + s[4] * s[4] + s[5] * s[5];
  double z[3] = {0.0, 0.0, 1.0};
  if (w2 > 0.0) {
    const double iw = 1.0 / sqrt(w2);
    z[0] = s[0] * iw; z[1] = s[1] * iw; z[2] = s[2] * iw;
  } else if (v2 > 0.0) {
    const double iv = 1.0 / sqrt(v2);
    z[0] = s[3] * iv; z[1] = s[4] * iv; z[2] = s[5] * iv;
  }
  // x': component u of v normal to z' (Gram-Schmidt twice, so x' is normal to
  // z' to rounding even when u is small), else the world axis least aligned
  // with z'. Either way |v'y| = |y'.u| is at rounding level and is stored as 0.
  const double vz = z[0] * s[3] + z[1] * s[4] + z[2] * s[5];
  double x[3] = {s[3] - vz * z[0], s[4] - vz * z[1], s[5] - vz * z[2]};
  double x2 = x[0] * x[0] + x[1] * x[1] + x[2] * x[2];
  if (!(x2 > 1e-280)) {
    const int a = (fabs(z[0]) <= fabs(z[1]) && fabs(z[0]) <= fabs(z[2])) ? 0 : (fabs(z[1]) <= fabs(z[2]) ? 1 : 2);
    x[0] = (a == 0) - z[a] * z[0]; x[1] = (a == 1) - z[a] * z[1]; x[2] = (a == 2) - z[a] * z[2];
    x2 = x[0] * x[0] + x[1] * x[1] + x[2] * x[2];
  }
  for (int pass = 0; pass < 2; ++pass) {
    const double ix = 1.0 / sqrt(x2);
    x[0] *= ix; x[1] *= ix; x[2] *= ix;
    const double xz = x[0] * z[0] + x[1] * z[1] + x[2] * z[2];
    x[0] -= xz * z[0]; x[1] -= xz * z[1]; x[2] -= xz * z[2];
    x2 = x[0] * x[0] + x[1] * x[1] + x[2] * x[2];
  }
  {
    const double ix = 1.0 / sqrt(x2);
    x[0] *= ix; x[1] *= ix; x[2] *= ix;
  }
  const double y[3] = {z[1] * x[2] - z[2] * x[1], z[2] * x[0] - z[0] * x[2], z[0] * x[1] - z[1] * x[0]};
  for (int k = 0; k < 3; ++k) {
    Q[k] = x[k];
    Q[3 + k] = y[k];
    Q[6 + k] = z[k];
  }
  sz[0] = sqrt(w2);                                  // |w| (the reference's w_n)
  sz[1] = x[0] * s[3] + x[1] * s[4] + x[2] * s[5];   // v'x
  sz[2] = vz;                                        // v'z
}

// Q_i of link i of model mc from the raw upload ([M][n][31], screw at +13).
__device__ __forceinline__ void raw_joint_frame(const double* raw, int n, int64_t mc, int i, double Q[9]) {
  const double* r = raw + ((int64_t)mc * n + i) * PD_LINK_FIELDS + 13;
  double s[6], sz[3];
#pragma unroll
  for (int k = 0; k < 6; ++k) s[k] = __ldg(r + k);
  joint_frame(s, Q, sz);
}

}  // namespace pd

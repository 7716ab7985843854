// Batch views shared by the kernels: packed SoA models and [link][problem]
// state arrays (problem fastest, so a warp of lane-per-chain threads reads
// 32 consecutive doubles per field and link).
#pragma once

#include "pd_common.cuh"

namespace pd {

struct ModelView {
  const double* __restrict__ f;  // [F_COUNT][n][M]
  const double* __restrict__ g;  // gravity [3][M]
  const int32_t* __restrict__ mstatus;  // [M] PD_SLOT_OK or PD_SLOT_BAD_MODEL
  const int32_t* __restrict__ mrule;    // [M]
  // Optional link-fastest copy [chain][field][link] (nullptr if absent). Lane-per-
  // chain kernels read the chain-fastest SoA above (coalesced across chains);
  // CTA/warp-per-chain kernels read this copy (coalesced across links).
  const double* __restrict__ fcl;
  int n;
  int64_t M;    // models in this view (1 = one model shared by every problem)
  int64_t ld;   // stride between links of one field (>= M, even: TMA needs 16-byte strides)
  int64_t gld;  // stride between gravity components
  __device__ __forceinline__ double at(int field, int link, int64_t mc) const {
    return fcl ? __ldg(fcl + ((int64_t)mc * F_COUNT + field) * n + link)
               : __ldg(f + ((int64_t)field * n + link) * ld + mc);
  }
  __device__ __forceinline__ int64_t model_of(int64_t p) const { return M == 1 ? 0 : p; }
  __device__ __forceinline__ Vec3d gravity(int64_t mc) const {
    return mk(__ldg(g + mc), __ldg(g + gld + mc), __ldg(g + 2 * gld + mc));
  }
  __device__ __forceinline__ Sv screw(int i, int64_t mc) const {
    return joint_screw(at(F_SW, i, mc), at(F_SVX, i, mc), at(F_SVZ, i, mc));
  }
  __device__ __forceinline__ double screw_iw(int i, int64_t mc) const { return at(F_SIW, i, mc); }
  __device__ __forceinline__ Mat3d home_R(int i, int64_t mc) const {
    return quat_to_R(at(F_HQ, i, mc), at(F_HQ + 1, i, mc), at(F_HQ + 2, i, mc), at(F_HQ + 3, i, mc));
  }
  __device__ __forceinline__ Vec3d home_p(int i, int64_t mc) const {
    return mk(at(F_HP, i, mc), at(F_HP + 1, i, mc), at(F_HP + 2, i, mc));
  }
  __device__ __forceinline__ Inertia inertia(int i, int64_t mc) const {
    Inertia J;
    J.m = at(F_MASS, i, mc);
    J.c = mk(at(F_COM, i, mc), at(F_COM + 1, i, mc), at(F_COM + 2, i, mc));
#pragma unroll
    for (int k = 0; k < 6; ++k) J.I[k] = at(F_IC + k, i, mc);
    return J;
  }
};

struct BatchIO {
  const double* __restrict__ q;    // [n][B]
  const double* __restrict__ qd;   // [n][B]
  const double* __restrict__ tau;  // [n][B]
  double* __restrict__ qdd;        // [n][B]
  int32_t* __restrict__ status;    // [B]
  int32_t* __restrict__ eround;    // [B]
  int32_t* __restrict__ eindex;    // [B]
  int64_t B;
  int64_t lds;  // stride between links of the state arrays (>= B)
  __device__ __forceinline__ double ld(const double* a, int i, int64_t p) const { return __ldg(a + (int64_t)i * lds + p); }
  __device__ __forceinline__ void put_qdd(int i, int64_t p, double v) const { qdd[(int64_t)i * lds + p] = v; }
};

// Host-validated model problems short-circuit with the model's rule.
__device__ __forceinline__ bool model_rejected(const ModelView& mv, const BatchIO& io, int64_t p, int64_t mc) {
  const int32_t ms = __ldg(mv.mstatus + mc);
  if (ms != PD_SLOT_OK) {
    io.status[p] = ms;
    io.eround[p] = 0;
    io.eindex[p] = __ldg(mv.mrule + mc);
    return true;
  }
  return false;
}

}  // namespace pd

// ABIA for long chains / small batches: one CTA per chain.
//
// Everything that is parallel over links runs CTA-wide (cta_common.cuh):
// joint transforms, the SE(3) prefix X_i, the bias torque (V0/A0 prefix sums,
// F0 suffix sum -> tau_delta), and the base-frame S0_i, J0_i of every link.
// What remains is the inherently sequential part of ABIA -- the articulated
// inertia recursion (forward_dynamics.cpp:120-163) with the z sweep and u,
// and the 12-FMA acceleration sweep -- which one thread runs over
// precomputed per-link data, prefetching link i-1 while it works on link i.
// In base coordinates that recursion has no 6x6 congruence (abia_common.cuh),
// so its per-link dependency chain is short.
#include "abia_common.cuh"
#include "cta_common.cuh"

namespace pd {

namespace abc {
// workspace fields (units of n doubles)
constexpr int REL = 0, X = 12, V = 24, TMP = 30, TD = 36;  // bias stage (cta_common)
constexpr int S0 = 37, J0 = 43;                             // 6 + 21 (Sym6 order A, B, D)
constexpr int G = 64, U = 70;                               // gain g0 (6), u (1)
constexpr int FIELDS = 71;
}  // namespace abc

size_t abia_cta_workspace_bytes(int n) { return (size_t)abc::FIELDS * n * sizeof(double); }

template <bool SMEM>
__global__ void __launch_bounds__(256) abia_cta_kernel(ModelView mv, BatchIO io, double* __restrict__ gws, int lpt,
                                                        int64_t p_off) {
  extern __shared__ double dyn_smem[];
  __shared__ ScanSmem scan_sm;
  const int n = mv.n;
  const int64_t p = p_off + blockIdx.x;
  const int64_t mc = mv.model_of(p);
  double* ws = SMEM ? dyn_smem : gws + (int64_t)blockIdx.x * abc::FIELDS * n;
  const int t = threadIdx.x;
  const int i0 = t * lpt, i1 = min(n, i0 + lpt);
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
    if (t == 0) model_rejected(mv, io, p, mc);
    return;
  }
  const IdFields idf{abc::REL, abc::X, abc::V, abc::TMP, abc::TD};
  cta_kinematics(mv, io, p, mc, ws, idf, lpt);
  cta_bias_torque(mv, io, p, mc, ws, idf, lpt, scan_sm);  // ends with a barrier; X holds X_i

  for (int i = i0; i < i1; ++i) {
    const SE3d Xi = ws_get_se3(ws, n, abc::X, i);
    ws_put_sv(ws, n, abc::S0, i, adinv_screw(Xi, mv.screw(i, mc)));
    const Sym6 J = inertia_sym6(inertia_to_base(mv.inertia(i, mc), Xi));
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(abc::J0 + k) * n + i] = J.A[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) ws[(abc::J0 + 6 + k) * n + i] = J.B[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(abc::J0 + 15 + k) * n + i] = J.D[k];
  }
  __syncthreads();
  if (t != 0) return;

  // ---- sequential articulated-inertia recursion + z sweep (tip -> base) ------
  Sym6 P;
  Sv Z = svzero();
  int code = PD_SLOT_OK, eidx = 0;
  double nx[28];  // prefetched S0 (6), J0 (21), td (1) of the next link
  auto fetch = [&](int i) {
#pragma unroll
    for (int k = 0; k < 6; ++k) nx[k] = ws[(abc::S0 + k) * n + i];
#pragma unroll
    for (int k = 0; k < 21; ++k) nx[6 + k] = ws[(abc::J0 + k) * n + i];
    nx[27] = ws[abc::TD * n + i];
  };
  fetch(n - 1);
  for (int i = n - 1; i >= 0; --i) {
    const Sv S0 = {mk(nx[0], nx[1], nx[2]), mk(nx[3], nx[4], nx[5])};
    Sym6 Ia;
#pragma unroll
    for (int k = 0; k < 6; ++k) Ia.A[k] = nx[6 + k];
#pragma unroll
    for (int k = 0; k < 9; ++k) Ia.B[k] = nx[12 + k];
#pragma unroll
    for (int k = 0; k < 6; ++k) Ia.D[k] = nx[21 + k];
    const double td = nx[27];
    if (i > 0) fetch(i - 1);
    if (i < n - 1) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        Ia.A[k] += P.A[k];
        Ia.D[k] += P.D[k];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) Ia.B[k] += P.B[k];
    }
    const Sv U = sym6_apply(Ia, S0);
    const double lambda = dot(S0, U);
    if (!(lambda > 1e-14 * link_frame_trace(Ia, ws_get_se3(ws, n, abc::X, i))) && code == PD_SLOT_OK) {
      code = PD_SLOT_DEGENERATE_ARTICULATION;  // forward_dynamics.cpp:140-144
      eidx = i;
    }
    const double inv_l = 1.0 / lambda;
    const double u = (td - dot(S0, Z)) * inv_l;
    const Sv g0 = inv_l * U;
    ws_put_sv(ws, n, abc::G, i, g0);
    ws[abc::U * n + i] = u;
    Z = svfma(u, U, Z);
    const double ua[3] = {U.a.x, U.a.y, U.a.z}, ul[3] = {U.l.x, U.l.y, U.l.z};
    const double ga[3] = {g0.a.x, g0.a.y, g0.a.z}, gl[3] = {g0.l.x, g0.l.y, g0.l.z};
    const int sidx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      P.A[k] = fma(-ua[sidx[k][0]], ga[sidx[k][1]], Ia.A[k]);
      P.D[k] = fma(-ul[sidx[k][0]], gl[sidx[k][1]], Ia.D[k]);
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) P.B[3 * r + c] = fma(-ua[r], gl[c], Ia.B[3 * r + c]);
  }
  // ---- acceleration sweep (base -> tip) --------------------------------------
  Sv a0 = svzero();
  for (int i = 0; i < n; ++i) {
    const double qdd = ws[abc::U * n + i] - dot(ws_get_sv(ws, n, abc::G, i), a0);
    a0 = svfma(qdd, ws_get_sv(ws, n, abc::S0, i), a0);
    io.put_qdd(i, p, qdd);
  }
  io.status[p] = code;
  io.eround[p] = 0;
  io.eindex[p] = eidx;
}

void launch_abia_cta(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, cudaStream_t s) {
  const int n = mv.n;
  int nt = ((n + 31) / 32) * 32;
  if (nt > 256) nt = 256;
  const int lpt = (n + nt - 1) / nt;
  const size_t ws_bytes = abia_cta_workspace_bytes(n);
  if (ws_bytes <= 200 * 1024) {
    cudaFuncSetAttribute(abia_cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
    abia_cta_kernel<true><<<(unsigned)io.B, nt, ws_bytes, s>>>(mv, io, nullptr, lpt, 0);
  } else {
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      abia_cta_kernel<false><<<(unsigned)nb, nt, 0, s>>>(mv, io, gws, lpt, b0);
    }
  }
}

}  // namespace pd

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

// Sequential part for the global-workspace case (long chains, c4). The
// per-link inputs live in L2, so instead of an L2 round trip per link, warps
// 1.. stage the next chunk of links into shared memory (double buffer) while
// thread 0 runs the recursion over the current one. The helpers also take
// everything that does not depend on the carried inertia P off thread 0's
// dependency chain: with I^A = J0 + P, U = J0 S0 + P S0 and
// lambda = S0.J0 S0 + S0.(P S0), and the degeneracy trace is linear in I^A.
// Thread 0 prefetches link i-1 into registers while it works on link i.
constexpr int kCh = 64;  // links per staged chunk

// staged per link (backward): S0 6 | J0 21 | td | JS = J0 S0 6 | lamJ | trJ | q 3 | 0 * joint angle
constexpr int kS0 = 0, kJ0 = 6, kTd = 27, kJS = 28, kLJ = 34, kTJ = 35, kQv = 36, kQf = 39, kStB = 40;
constexpr int kStC = 13;  // forward: g0 6 | S0 6 | u
// g0 / u of every link stay in shared memory when they fit, else in the
// workspace's G / U fields (same [7][n] layout)
bool abia_cta_gu_smem(int n) { return (size_t)(2 * kStB * kCh + 7 * n) * sizeof(double) <= 200 * 1024; }
size_t abia_cta_stage_bytes(int n) { return (size_t)(2 * kStB * kCh + (abia_cta_gu_smem(n) ? 7 * n : 0)) * sizeof(double); }

__device__ __forceinline__ void sequential_staged(const ModelView& mv, const BatchIO& io, int64_t p, double* ws,
                                                  double* sm, bool gu_smem) {
  const int n = mv.n, t = threadIdx.x, nt = blockDim.x;
  const int nch = (n + kCh - 1) / kCh;
  // [7][n]: g0 (6), u -- written by thread 0, read by the forward staging
  double* gu = gu_smem ? sm + 2 * kStB * kCh : ws + abc::G * n;
  // backward chunk c covers links [max(0, n - (c+1) kCh), n - c kCh); one link per helper thread
  auto stage_b = [&](int c, int tid, int nthr) {
    double* b = sm + (c & 1) * kStB * kCh;
    const int hi = n - c * kCh, lo = max(0, hi - kCh);
    for (int i = lo + tid; i < hi; i += nthr) {
      const int j = i - lo;
      const Sv S0 = ws_get_sv(ws, n, abc::S0, i);
      Sym6 J;
#pragma unroll
      for (int k = 0; k < 6; ++k) J.A[k] = ws[(abc::J0 + k) * n + i];
#pragma unroll
      for (int k = 0; k < 9; ++k) J.B[k] = ws[(abc::J0 + 6 + k) * n + i];
#pragma unroll
      for (int k = 0; k < 6; ++k) J.D[k] = ws[(abc::J0 + 15 + k) * n + i];
      const SE3d X = ws_get_se3(ws, n, abc::X, i);
      const Vec3d qv = -1.0 * mulT(X.R, X.p);
      const Sv JS = sym6_apply(J, S0);
      const double v[kStB] = {S0.a.x, S0.a.y, S0.a.z, S0.l.x, S0.l.y, S0.l.z,
                              J.A[0], J.A[1], J.A[2], J.A[3], J.A[4], J.A[5],
                              J.B[0], J.B[1], J.B[2], J.B[3], J.B[4], J.B[5], J.B[6], J.B[7], J.B[8],
                              J.D[0], J.D[1], J.D[2], J.D[3], J.D[4], J.D[5],
                              ws[abc::TD * n + i],
                              JS.a.x, JS.a.y, JS.a.z, JS.l.x, JS.l.y, JS.l.z,
                              dot(S0, JS), link_frame_trace_q(J, qv), qv.x, qv.y, qv.z,
                              io.ld(io.q, i, p) * 0.0};
#pragma unroll
      for (int f = 0; f < kStB; ++f) b[f * kCh + j] = v[f];
    }
  };
  auto stage_c = [&](int c, int tid, int nthr) {  // forward chunk c covers [c kCh, min(n, (c+1) kCh))
    double* b = sm + (c & 1) * kStB * kCh;
    const int lo = c * kCh, hi = min(n, lo + kCh);
    for (int e = tid; e < (hi - lo) * kStC; e += nthr) {
      const int j = e % (hi - lo), f = e / (hi - lo), i = lo + j;
      b[f * kCh + j] = f < 6 ? gu[f * n + i] : (f < 12 ? ws[(abc::S0 + f - 6) * n + i] : gu[6 * n + i]);
    }
  };
  stage_b(0, t, nt);
  __syncthreads();
  Sym6 P = {};
  Sv Z = svzero();
  int code = PD_SLOT_OK, eidx = 0;
  double qpoison = 0.0;  // NaN once a non-finite joint angle beyond the current link was seen
  for (int c = 0; c < nch; ++c) {
    if (t >= 32) {
      if (c + 1 < nch) stage_b(c + 1, t - 32, nt - 32);
    } else if (t == 0) {
      const double* b = sm + (c & 1) * kStB * kCh;
      const int hi = n - c * kCh, lo = max(0, hi - kCh);
      auto load = [&](double (&v)[kStB], int i) {
#pragma unroll
        for (int f = 0; f < kStB; ++f) v[f] = b[f * kCh + (i - lo)];
      };
      auto step = [&](const double (&cur)[kStB], int i) {
        const Sv S0 = {mk(cur[0], cur[1], cur[2]), mk(cur[3], cur[4], cur[5])};
        const Sv PS = sym6_apply(P, S0);
        const Sv U = {mk(cur[kJS] + PS.a.x, cur[kJS + 1] + PS.a.y, cur[kJS + 2] + PS.a.z),
                      mk(cur[kJS + 3] + PS.l.x, cur[kJS + 4] + PS.l.y, cur[kJS + 5] + PS.l.z)};
        const double lambda = cur[kLJ] + dot(S0, PS);
        // degeneracy test on the link-frame trace of I^A (forward_dynamics.cpp:140-144)
        const double tr = cur[kTJ] + link_frame_trace_q(P, mk(cur[kQv], cur[kQv + 1], cur[kQv + 2]));
        const bool bad = abia_degenerate(qpoison != qpoison, lambda, 1e-14 * tr) & (code == PD_SLOT_OK);
        qpoison += cur[kQf];  // 0, or NaN for a non-finite joint angle
        code = bad ? PD_SLOT_DEGENERATE_ARTICULATION : code;
        eidx = bad ? i : eidx;
        const double inv_l = rcp_nr(lambda);
        const double u = (cur[kTd] - dot(S0, Z)) * inv_l;
        const Sv g0 = inv_l * U;
        gu[0 * n + i] = g0.a.x;
        gu[1 * n + i] = g0.a.y;
        gu[2 * n + i] = g0.a.z;
        gu[3 * n + i] = g0.l.x;
        gu[4 * n + i] = g0.l.y;
        gu[5 * n + i] = g0.l.z;
        gu[6 * n + i] = u;
        Z = svfma(u, U, Z);
        // P <- J0 + P - U g0^T (projected articulated inertia, :150-156)
        const double ua[3] = {U.a.x, U.a.y, U.a.z}, ul[3] = {U.l.x, U.l.y, U.l.z};
        const double ga[3] = {g0.a.x, g0.a.y, g0.a.z}, gl[3] = {g0.l.x, g0.l.y, g0.l.z};
        const int sidx[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          P.A[k] = fma(-ua[sidx[k][0]], ga[sidx[k][1]], cur[kJ0 + k] + P.A[k]);
          P.D[k] = fma(-ul[sidx[k][0]], gl[sidx[k][1]], cur[kJ0 + 15 + k] + P.D[k]);
        }
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            P.B[3 * r + cc] = fma(-ua[r], gl[cc], cur[kJ0 + 6 + 3 * r + cc] + P.B[3 * r + cc]);
      };
      // two register sets, ping-pong: the loads of link i-1 are in flight during link i
      double va[kStB], vb[kStB];
      load(va, hi - 1);
      int i = hi - 1;
      for (; i - 1 >= lo; i -= 2) {
        load(vb, i - 1);
        step(va, i);
        if (i - 2 >= lo) load(va, i - 2);
        step(vb, i - 1);
      }
      if (i >= lo) step(va, i);
    }
    __syncthreads();
  }
  // acceleration sweep (base -> tip), same staging
  stage_c(0, t, nt);
  __syncthreads();
  Sv a0 = svzero();
  for (int c = 0; c < nch; ++c) {
    if (t >= 32) {
      if (c + 1 < nch) stage_c(c + 1, t - 32, nt - 32);
    } else if (t == 0) {
      const double* b = sm + (c & 1) * kStB * kCh;
      const int lo = c * kCh, hi = min(n, lo + kCh);
      auto load = [&](double (&v)[kStC], int i) {
#pragma unroll
        for (int f = 0; f < kStC; ++f) v[f] = b[f * kCh + (i - lo)];
      };
      auto step = [&](const double (&cur)[kStC], int i) {
        const Sv g0 = {mk(cur[0], cur[1], cur[2]), mk(cur[3], cur[4], cur[5])};
        const Sv S0 = {mk(cur[6], cur[7], cur[8]), mk(cur[9], cur[10], cur[11])};
        const double qdd = cur[12] - dot(g0, a0);
        a0 = svfma(qdd, S0, a0);
        io.put_qdd(i, p, qdd);
      };
      double va[kStC], vb[kStC];
      load(va, lo);
      int i = lo;
      for (; i + 1 < hi; i += 2) {
        load(vb, i + 1);
        step(va, i);
        if (i + 2 < hi) load(va, i + 2);
        step(vb, i + 1);
      }
      if (i < hi) step(va, i);
    }
    __syncthreads();
  }
  if (t == 0) {
    io.status[p] = code;
    io.eround[p] = 0;
    io.eindex[p] = eidx;
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(256) abia_cta_kernel(ModelView mv, BatchIO io, double* __restrict__ gws, int lpt,
                                                        int64_t p_off, bool gu_smem = false) {
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
  if (!SMEM) {
    sequential_staged(mv, io, p, ws, dyn_smem, gu_smem);
    return;
  }
  if (t != 0) return;
  // ---- sequential articulated-inertia recursion + z sweep (tip -> base) ------
  Sym6 P;
  Sv Z = svzero();
  int code = PD_SLOT_OK, eidx = 0;
  bool nan_tip = false;
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
    if (abia_degenerate(nan_tip, lambda, 1e-14 * link_frame_trace(Ia, ws_get_se3(ws, n, abc::X, i))) &&
        code == PD_SLOT_OK) {
      code = PD_SLOT_DEGENERATE_ARTICULATION;  // forward_dynamics.cpp:140-144
      eidx = i;
    }
    nan_tip = nan_tip || !isfinite(io.ld(io.q, i, p));
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
    cudaFuncSetAttribute(abia_cta_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)abia_cta_stage_bytes(n));
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      abia_cta_kernel<false><<<(unsigned)nb, nt, abia_cta_stage_bytes(n), s>>>(mv, io, gws, lpt, b0,
                                                                                 abia_cta_gu_smem(n));
    }
  }
}

}  // namespace pd

// JSIIA forward dynamics, one CTA per chain.
//
// Reference: jsiia_forward_dynamics (proj/core/src/forward_dynamics.cpp:82-118)
//   = kinematics + torque surplus (3 scans)                 -> cta_bias_torque
//   + joint_space_inertia_assembled (:44-66): column j of M is the torque of
//     unit acceleration of joint j from rest, gravity off, then M = (M+M^T)/2
//   + LLT(M) (DynamicsError if not SPD, :93-98), qdd = M^{-1} td (:99),
//     one refinement step if ||td - M qdd|| > 1e-9 ||td||, error if still
//     above (:105-116).
//
// B200 mapping. The n column probes of the reference (n inverse-dynamics
// solves, 3 scans each) are replaced by the closed form they evaluate: in base
// coordinates the probe of column j accumulates Ic_j = sum_{k>=j} J_k^b, so
// M_ij = S_i^b . (Ic_{max(i,j)}^b S_{max(i,j)}^b)... = S^b_min . F^b_max with
// F^b_k = Ic^b_k S^b_k, S^b_k = Ad(X_k)^{-1} S_k, J^b_k = Ad(X_k)^T J_k Ad(X_k).
// That is one SE(3) prefix scan (shared with the bias stage) and one 21-wide
// suffix sum instead of 3n scans; M comes out exactly symmetric (same
// expression for (i,j) and (j,i)). Cholesky, triangular solves and the
// refinement run CTA-parallel with M in shared memory (column-major, odd
// leading dimension).
#include "cta_common.cuh"

namespace pd {

namespace jsi {
constexpr int REL = 0, X = 12, V = 24, TMP = 30, TD = 36, SB = 37, FB = 43, IC = 49;
constexpr int FIELDS = 70;
constexpr int VEC_Y = 0, VEC_X = 1, VEC_R = 2, VEC_DG = 3, VEC_D = 4;  // n-vectors after the fields
constexpr int NVEC = 5;
}  // namespace jsi

__host__ __device__ __forceinline__ int jsi_ld(int n) { return n | 1; }
__host__ __device__ __forceinline__ size_t jsi_workspace_doubles(int n) {
  return (size_t)(jsi::FIELDS + jsi::NVEC) * n + (size_t)jsi_ld(n) * n;
}

struct BlockReduce {
  double part[kMaxWarps];
};
// Deterministic CTA sum (fixed order), result broadcast to all threads.
__device__ double block_sum(double v, BlockReduce& br) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  if (lane == 0) br.part[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += br.part[w];
  __syncthreads();
  return s;
}

// Solve (L L^T) v = v in place (vec field f of the workspace); L in the lower
// triangle of column-major M.
__device__ void cta_llt_solve(double* ws, int n, const double* M, int ld, double* v) {
  const int t = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < n; ++k) {  // forward: L y = v
    const double yk = v[k] / M[k * ld + k];
    __syncthreads();
    for (int i = k + 1 + t; i < n; i += nt) v[i] = fma(-M[k * ld + i], yk, v[i]);
    if (t == 0) v[k] = yk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // backward: L^T x = y
    const double xk = v[k] / M[k * ld + k];
    __syncthreads();
    for (int i = t; i < k; i += nt) v[i] = fma(-M[i * ld + k], xk, v[i]);
    if (t == 0) v[k] = xk;
    __syncthreads();
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(256) jsiia_cta_kernel(ModelView mv, BatchIO io, double* __restrict__ gws, int lpt,
                                                         int64_t p_off) {
  extern __shared__ double dyn_smem[];
  __shared__ ScanSmem scan_sm;
  __shared__ BlockReduce br;
  __shared__ int s_fail;
  const int n = mv.n;
  const int64_t p = p_off + blockIdx.x;
  const int64_t mc = mv.model_of(p);
  double* ws = SMEM ? dyn_smem : gws + (int64_t)blockIdx.x * jsi_workspace_doubles(n);
  const int t = threadIdx.x, nt = blockDim.x;
  const int i0 = t * lpt, i1 = min(n, i0 + lpt);
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
    if (t == 0) model_rejected(mv, io, p, mc);
    return;
  }
  if (t == 0) s_fail = 0;
  const int ld = jsi_ld(n);
  double* vec = ws + jsi::FIELDS * n;
  double* M = ws + (jsi::FIELDS + jsi::NVEC) * n;  // column-major, M[j*ld + i] = M_ij

  // ---- kinematics + torque surplus ----------------------------------------
  const IdFields idf{jsi::REL, jsi::X, jsi::V, jsi::TMP, jsi::TD};
  cta_kinematics(mv, io, p, mc, ws, idf, lpt);
  cta_bias_torque(mv, io, p, mc, ws, idf, lpt, scan_sm);

  // ---- composite inertias in base coordinates -------------------------------
  for (int i = i0; i < i1; ++i) {
    const SE3d X = ws_get_se3(ws, n, jsi::X, i);
    const Sym6 Jb = sym6_congruence(inertia_sym6(mv.inertia(i, mc)), X);
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(jsi::IC + k) * n + i] = Jb.A[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) ws[(jsi::IC + 6 + k) * n + i] = Jb.B[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(jsi::IC + 15 + k) * n + i] = Jb.D[k];
    ws_put_sv(ws, n, jsi::SB, i, adinv_apply(X, mv.screw(i, mc)));
  }
  __syncthreads();
  ws_scan<12, true>(ws, n, jsi::IC, lpt, AddOp{}, scan_sm);
  __syncthreads();
  ws_scan<9, true>(ws, n, jsi::IC + 12, lpt, AddOp{}, scan_sm);
  __syncthreads();
  for (int i = i0; i < i1; ++i) {
    Sym6 Ic;
#pragma unroll
    for (int k = 0; k < 6; ++k) Ic.A[k] = ws[(jsi::IC + k) * n + i];
#pragma unroll
    for (int k = 0; k < 9; ++k) Ic.B[k] = ws[(jsi::IC + 6 + k) * n + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) Ic.D[k] = ws[(jsi::IC + 15 + k) * n + i];
    ws_put_sv(ws, n, jsi::FB, i, sym6_apply(Ic, ws_get_sv(ws, n, jsi::SB, i)));
  }
  __syncthreads();

  // ---- M_ij = S^b_min(i,j) . F^b_max(i,j) ------------------------------------
  for (int j = t; j < n; j += nt) {
    const Sv Sj = ws_get_sv(ws, n, jsi::SB, j);
    const Sv Fj = ws_get_sv(ws, n, jsi::FB, j);
    for (int i = 0; i < n; ++i) {
      const double mij = (i <= j) ? dot(ws_get_sv(ws, n, jsi::SB, i), Fj) : dot(Sj, ws_get_sv(ws, n, jsi::FB, i));
      M[j * ld + i] = mij;
    }
    vec[jsi::VEC_DG * n + j] = M[j * ld + j];
    vec[jsi::VEC_X * n + j] = ws[jsi::TD * n + j];  // rhs
  }
  __syncthreads();

  // ---- Cholesky (right-looking, lower triangle) -----------------------------
  for (int k = 0; k < n; ++k) {
    const double piv = M[k * ld + k];
    if (!(piv > 0.0)) {
      if (t == 0) s_fail = 1;
    }
    const double lkk = sqrt(piv);
    const double inv = 1.0 / lkk;
    for (int i = k + 1 + t; i < n; i += nt) M[k * ld + i] *= inv;
    __syncthreads();
    if (t == 0) M[k * ld + k] = lkk;
    for (int j = k + 1 + t; j < n; j += nt) {
      const double ljk = M[k * ld + j];
      for (int i = j; i < n; ++i) M[j * ld + i] = fma(-M[k * ld + i], ljk, M[j * ld + i]);
    }
    __syncthreads();
  }
  if (s_fail) {  // forward_dynamics.cpp:93-98
    if (t == 0) {
      io.status[p] = PD_SLOT_JSI_NOT_SPD;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }

  // ---- solve + residual contract (forward_dynamics.cpp:99-116) --------------
  double* xv = vec + jsi::VEC_X * n;
  double* rv = vec + jsi::VEC_R * n;
  double* dg = vec + jsi::VEC_DG * n;
  double* dv = vec + jsi::VEC_D * n;
  cta_llt_solve(ws, n, M, ld, xv);
  double sq = 0.0;
  for (int i = t; i < n; i += nt) sq = fma(ws[jsi::TD * n + i], ws[jsi::TD * n + i], sq);
  const double scale = fmax(sqrt(block_sum(sq, br)), 2.2250738585072014e-308);
  int code = PD_SLOT_OK;
  for (int pass = 0; pass < 2; ++pass) {
    double rr = 0.0;
    for (int i = t; i < n; i += nt) {
      double s = ws[jsi::TD * n + i];
      for (int j = 0; j < n; ++j) {
        const double mij = (i < j) ? M[j * ld + i] : ((i > j) ? M[i * ld + j] : dg[i]);
        s = fma(-mij, xv[j], s);
      }
      rv[i] = s;
      dv[i] = s;
      rr = fma(s, s, rr);
    }
    const double rn = sqrt(block_sum(rr, br));
    if (!(rn > 1e-9 * scale)) break;
    if (pass == 1) {
      code = PD_SLOT_JSI_REFINE_FAILED;
      break;
    }
    cta_llt_solve(ws, n, M, ld, dv);
    for (int i = t; i < n; i += nt) xv[i] += dv[i];
    __syncthreads();
  }
  for (int i = t; i < n; i += nt) io.put_qdd(i, p, xv[i]);
  if (t == 0) {
    io.status[p] = code;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

size_t jsiia_workspace_bytes(int n) { return jsi_workspace_doubles(n) * sizeof(double); }

void launch_jsiia(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, cudaStream_t s) {
  const int n = mv.n;
  int nt = ((n + 31) / 32) * 32;
  if (nt > 256) nt = 256;
  const int lpt = (n + nt - 1) / nt;
  const size_t ws_bytes = jsiia_workspace_bytes(n);
  if (ws_bytes <= 220 * 1024) {
    cudaFuncSetAttribute(jsiia_cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
    jsiia_cta_kernel<true><<<(unsigned)io.B, nt, ws_bytes, s>>>(mv, io, nullptr, lpt, 0);
  } else {
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      jsiia_cta_kernel<false><<<(unsigned)nb, nt, 0, s>>>(mv, io, gws, lpt, b0);
    }
  }
}

}  // namespace pd

// JSIIA forward dynamics for chains longer than one warp (n > 32): one CTA per
// chain, M factored by a blocked (32x32-tile) right-looking Cholesky.
//
// Reference: jsiia_forward_dynamics (proj/core/src/forward_dynamics.cpp:82-118)
//   = kinematics + torque surplus (3 scans)                 -> cta_bias_torque
//   + joint_space_inertia_assembled (:44-66): column j of M is the torque of
//     unit acceleration of joint j from rest, gravity off, then M = (M+M^T)/2
//   + LLT(M) (DynamicsError if not SPD, :93-98), qdd = M^{-1} td (:99),
//     one refinement step if ||td - M qdd|| > 1e-9 ||td||, error if still
//     above (:105-116).
//
// B200 mapping.
//  * The n column probes of the reference (n inverse-dynamics solves) are
//    replaced by the closed form they evaluate: in base coordinates
//    M_ij = S0_min(i,j) . (Ic0_max S0_max), Ic0_k = sum_{l>=k} J0_l -- one SE(3)
//    prefix scan (shared with the bias stage) and one 21-wide suffix sum. The
//    expression is the same for (i,j) and (j,i), so M is exactly symmetric.
//  * M is stored row-major, padded to npad = 32*ceil(n/32) with an identity
//    block (so the padding needs no special cases anywhere), leading
//    dimension npad+2 (16-byte rows for double2 loads; 4-way banked columns).
//    It lives in shared memory when the chain's workspace fits (n <= ~150),
//    else in a per-CTA global slot (L2-resident).
//  * Cholesky by 32x32 tiles, one warp per tile task, lane = tile row with the
//    row in registers: POTRF (left-looking by rows, broadcast of row m),
//    TRSM (same recurrence against the factored diagonal tile) and the
//    trailing update C -= A B^T (double2 broadcasts of B rows, 2 FMA per
//    load). Tasks of one panel step are spread over the CTA's warps.
//    L overwrites the lower triangle; the strict upper triangle keeps M and
//    the diagonal of M is saved, so the residual uses M itself, as the
//    reference does.
#include <cooperative_groups.h>

#include "abia_common.cuh"
#include "cta_common.cuh"

namespace pd {

namespace jst {
// workspace fields, units of n doubles. TD, S0, FB stay live while M is built
// (M starts right after them and overwrites the dead kinematics fields).
constexpr int TD = 0, S0 = 1, FB = 7, REL = 13, X = 25, V = 37, TMP = 43, IC = 49;
constexpr int FIELDS = 70;
constexpr int KEEP = 13;
constexpr int NVEC = 4;  // after M: x, work vector, diag(M), 1/diag(L)
}  // namespace jst

struct JstLayout {
  int n, np, npad, ld;
  size_t m_off, v_off, total;  // doubles
};

__host__ __device__ inline JstLayout jst_layout(int n) {
  JstLayout L;
  L.n = n;
  L.np = (n + 31) / 32;
  L.npad = 32 * L.np;
  L.ld = L.npad + 2;
  L.m_off = ((size_t)jst::KEEP * n + 1) & ~(size_t)1;  // 16-byte aligned
  L.v_off = L.m_off + (size_t)L.npad * L.ld;
  size_t end = L.v_off + (size_t)jst::NVEC * L.npad + 1;  // + the cooperative path's fail flag (last double)
  const size_t phase_a = (size_t)jst::FIELDS * n;
  if (end < phase_a) end = phase_a;
  L.total = (end + 1) & ~(size_t)1;
  return L;
}

size_t jsiia_workspace_bytes(int n) { return jst_layout(n).total * sizeof(double); }

namespace {

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

// CG: the tile lives in global memory written by other CTAs of a cooperative
// grid -- read it through L2 (ld.global.cg), never from a stale L1 line.
template <bool CG = false>
__device__ __forceinline__ double2 ld2(const double* p) {
  return CG ? __ldcg(reinterpret_cast<const double2*>(p)) : *reinterpret_cast<const double2*>(p);
}
template <bool CG = false>
__device__ __forceinline__ double ld1(const double* p) {
  return CG ? __ldcg(p) : *p;
}

template <bool CG = false>
__device__ __forceinline__ void load_row(double (&r)[32], const double* row) {
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const double2 v = ld2<CG>(row + j);
    r[j] = v.x;
    r[j + 1] = v.y;
  }
}

// Cholesky of a diagonal tile in place (lower triangle; the strict upper
// triangle is read back unchanged). invd[i] = 1 / L_ii. Returns false iff a
// pivot is <= 0 (Eigen LLT's failure condition). Warp-uniform result.
template <bool CG = false>
__device__ bool tile_potrf(double* A, int ld, double* invd, int lane) {
  double r[32];
  load_row<CG>(r, A + lane * ld);
  bool spd = true;
  double inv_d = 0.0;
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    double a4[4] = {r[m], 0.0, 0.0, 0.0};
#pragma unroll
    for (int p = 0; p < m; ++p) a4[p & 3] = fma(-r[p], ld1<CG>(A + m * ld + p), a4[p & 3]);
    const double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    const double dmm = __shfl_sync(0xffffffffu, acc, m);
    spd = spd && !(dmm <= 0.0);  // Eigen LLT: fails iff a pivot <= 0 (NaN propagates)
    // one reciprocal square root per pivot: 1/L_mm, L_mm = d * (1/L_mm)
    const double inv = rsqrt_nr(dmm > 0.0 ? dmm : 1.0);
    const double lmm = (dmm > 0.0 ? dmm : 1.0) * inv;
    inv_d = (lane == m) ? inv : inv_d;
    r[m] = (lane == m) ? lmm : ((lane > m) ? acc * inv : r[m]);
    A[lane * ld + m] = r[m];
    __syncwarp();
  }
  invd[lane] = inv_d;
  return spd;
}

// B := B L^{-T} for an off-diagonal tile B of the panel of the factored L.
template <bool CG = false>
__device__ void tile_trsm(const double* Lkk, int ld, const double* invd, double* B, int lane) {
  double r[32];
  load_row<CG>(r, B + lane * ld);
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    double a4[4] = {r[m], 0.0, 0.0, 0.0};
#pragma unroll
    for (int p = 0; p < m; ++p) a4[p & 3] = fma(-r[p], ld1<CG>(Lkk + m * ld + p), a4[p & 3]);
    r[m] = ((a4[0] + a4[1]) + (a4[2] + a4[3])) * ld1<CG>(invd + m);
  }
#pragma unroll
  for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(B + lane * ld + j) = make_double2(r[j], r[j + 1]);
}

// C -= A B^T (32x32 tiles). On a diagonal tile only the lower triangle is
// written back (the strict upper triangle holds M).
template <bool CG = false>
__device__ void tile_gemm(double* C, const double* A, const double* Bt, int ld, bool diag, int lane) {
  double r[32];
  load_row<CG>(r, C + lane * ld);
#pragma unroll 1
  for (int p = 0; p < 32; p += 2) {
    const double2 a = ld2<CG>(A + lane * ld + p);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 b = ld2<CG>(Bt + j * ld + p);
      r[j] = fma(-a.x, b.x, r[j]);
      r[j] = fma(-a.y, b.y, r[j]);
    }
  }
  double* row = C + lane * ld;
  if (diag) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j <= lane) row[j] = r[j];
  } else {
#pragma unroll
    for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(row + j) = make_double2(r[j], r[j + 1]);
  }
}

// (L L^T) v = v in place, one warp. L: lower triangle of the padded matrix.
__device__ void warp_llt_solve(const double* Mb, int ld, int np, const double* invd, double* v, int lane) {
  double r[32];
  // forward: L y = v
  for (int I = 0; I < np; ++I) {
    double acc = v[32 * I + lane];
    for (int K = 0; K < I; ++K) {
      const double* a = Mb + (size_t)(32 * I + lane) * ld + 32 * K;
      const double* y = v + 32 * K;
#pragma unroll 8
      for (int p = 0; p < 32; p += 2) {
        const double2 av = *reinterpret_cast<const double2*>(a + p);
        const double2 yv = *reinterpret_cast<const double2*>(y + p);
        acc = fma(-av.x, yv.x, acc);
        acc = fma(-av.y, yv.y, acc);
      }
    }
    load_row(r, Mb + (size_t)(32 * I + lane) * ld + 32 * I);
    const double id = invd[32 * I + lane];
    double yo = 0.0;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      const double ym = __shfl_sync(0xffffffffu, acc * id, m);
      yo = (lane == m) ? ym : yo;
      acc = (lane > m) ? fma(-r[m], ym, acc) : acc;
    }
    v[32 * I + lane] = yo;
    __syncwarp();
  }
  // backward: L^T x = y
  for (int I = np - 1; I >= 0; --I) {
    double acc = v[32 * I + lane];
    for (int J = I + 1; J < np; ++J) {
      const double* col = Mb + (size_t)(32 * J) * ld + 32 * I + lane;
      const double* x = v + 32 * J;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) acc = fma(-col[(size_t)j * ld], x[j], acc);
    }
    const double* dt = Mb + (size_t)(32 * I) * ld + 32 * I + lane;
    const double id = invd[32 * I + lane];
    double xo = 0.0;
#pragma unroll
    for (int m = 31; m >= 0; --m) {
      const double xm = __shfl_sync(0xffffffffu, acc * id, m);
      xo = (lane == m) ? xm : xo;
      acc = (lane < m) ? fma(-dt[(size_t)m * ld], xm, acc) : acc;
    }
    v[32 * I + lane] = xo;
    __syncwarp();
  }
}

}  // namespace

// MODE 0: the whole solve in this CTA.
// MODE 1: joint_space_inertia (forward_dynamics.cpp:70-80) -- write M of every
//         problem to mout[p][i][j] after the build and stop.
// MODE 2: build M and tau_delta in the (global) workspace and stop; the grid-
//         wide Cholesky (jsiia_factor_coop) runs next, then MODE 3.
// MODE 3: solve + residual contract on a workspace MODE 2 / the cooperative
//         factorization left (fail flag in the workspace tail).
template <bool SMEM, int MODE = 0, int NT = 256>
__global__ void __launch_bounds__(NT) jsiia_tiled_kernel(ModelView mv, BatchIO io, double* __restrict__ gws,
                                                           int64_t p_off, double* __restrict__ mout = nullptr) {
  constexpr bool MOUT = MODE == 1;
  extern __shared__ __align__(16) double dyn_smem[];
  __shared__ ScanSmem scan_sm;
  __shared__ BlockReduce br;
  __shared__ int s_fail;
  const int n = mv.n;
  const JstLayout L = jst_layout(n);
  const int64_t p = p_off + blockIdx.x;
  const int64_t mc = mv.model_of(p);
  double* ws = SMEM ? dyn_smem : gws + (int64_t)blockIdx.x * L.total;
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, warp = t >> 5, nw = nt >> 5;
  const int lpt = (n + nt - 1) / nt;
  const int i0 = t * lpt, i1 = min(n, i0 + lpt);
  if (__ldg(mv.mstatus + mc) != PD_SLOT_OK) {
    if (t == 0) model_rejected(mv, io, p, mc);
    return;
  }
  if (t == 0) s_fail = 0;
  const int np = L.np, npad = L.npad, ld = L.ld;
  double* Mb = ws + L.m_off;
  double* vx = ws + L.v_off;
  double* vw = vx + npad;
  double* dg = vw + npad;
  double* invd = dg + npad;
  auto tile = [&](int I, int J) { return Mb + (size_t)(32 * I) * ld + 32 * J; };
  if (MODE == 3) {
    if (t == 0) s_fail = (int)ws[L.total - 1];
    __syncthreads();
  } else {

  // ---- kinematics + torque surplus ------------------------------------------
  const IdFields idf{jst::REL, jst::X, jst::V, jst::TMP, jst::TD};
  cta_kinematics(mv, io, p, mc, ws, idf, lpt);
  if (MOUT) {  // the X_i = rel_i X_{i-1} scan the bias stage would run
    __syncthreads();
    ws_scan<12, false>(ws, n, jst::X, lpt, ComposeOp{}, scan_sm);
    __syncthreads();
  } else
    cta_bias_torque(mv, io, p, mc, ws, idf, lpt, scan_sm);

  // ---- composite inertias in base coordinates ---------------------------------
  for (int i = i0; i < i1; ++i) {
    const SE3d X = ws_get_se3(ws, n, jst::X, i);
    const Sym6 Jb = inertia_sym6(inertia_to_base(mv.inertia(i, mc), X));
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(jst::IC + k) * n + i] = Jb.A[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) ws[(jst::IC + 6 + k) * n + i] = Jb.B[k];
#pragma unroll
    for (int k = 0; k < 6; ++k) ws[(jst::IC + 15 + k) * n + i] = Jb.D[k];
    ws_put_sv(ws, n, jst::S0, i, adinv_screw(X, mv.screw(i, mc)));
  }
  __syncthreads();
  ws_scan<12, true>(ws, n, jst::IC, lpt, AddOp{}, scan_sm);
  __syncthreads();
  ws_scan<9, true>(ws, n, jst::IC + 12, lpt, AddOp{}, scan_sm);
  __syncthreads();
  for (int i = i0; i < i1; ++i) {
    Sym6 Ic;
#pragma unroll
    for (int k = 0; k < 6; ++k) Ic.A[k] = ws[(jst::IC + k) * n + i];
#pragma unroll
    for (int k = 0; k < 9; ++k) Ic.B[k] = ws[(jst::IC + 6 + k) * n + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) Ic.D[k] = ws[(jst::IC + 15 + k) * n + i];
    ws_put_sv(ws, n, jst::FB, i, sym6_apply(Ic, ws_get_sv(ws, n, jst::S0, i)));
  }
  __syncthreads();
  if (MODE == 2) return;  // M is built grid-wide by jsiia_factor_coop

  // ---- M_ij = S0_min(i,j) . FB_max(i,j), identity padding ---------------------
  for (int J = 0; J < np; ++J) {
    const int j = 32 * J + lane;
    const bool jr = j < n;
    const Sv Sj = jr ? ws_get_sv(ws, n, jst::S0, j) : svzero();
    const Sv Fj = jr ? ws_get_sv(ws, n, jst::FB, j) : svzero();
    for (int i = warp; i < npad; i += nw) {
      double mij;
      if (i < n && jr) {
        const bool low = j <= i;  // lower: S0_j . FB_i, upper: S0_i . FB_j
        const Sv c = low ? Sj : Fj;
        const Sv rv = ws_get_sv(ws, n, low ? jst::FB : jst::S0, i);
        mij = dot(c, rv);
      } else {
        mij = (i == j) ? 1.0 : 0.0;
      }
      Mb[(size_t)i * ld + j] = mij;
      if (i == j) dg[i] = mij;
    }
  }
  if (MOUT) {
    __syncthreads();
    double* out = mout + (size_t)p * n * n;
    for (int e = t; e < n * n; e += nt) out[e] = Mb[(size_t)(e / n) * ld + e % n];
    if (t == 0) {
      io.status[p] = PD_SLOT_OK;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }
  for (int i = t; i < npad; i += nt) vx[i] = (i < n) ? ws[jst::TD * n + i] : 0.0;
  __syncthreads();

  // ---- blocked Cholesky, right-looking by 32-column panels -------------------
  for (int K = 0; K < np; ++K) {
    if (warp == 0) {
      const bool ok = tile_potrf(tile(K, K), ld, invd + 32 * K, lane);
      if (!ok && lane == 0) s_fail = 1;
    }
    __syncthreads();
    if (s_fail) break;  // forward_dynamics.cpp:93-98 (CTA-uniform)
    for (int I = K + 1 + warp; I < np; I += nw) tile_trsm(tile(K, K), ld, invd + 32 * K, tile(I, K), lane);
    __syncthreads();
    const int m = np - 1 - K;  // trailing tiles (I, J), K < J <= I
    const int tasks = m * (m + 1) / 2;
    for (int q = warp; q < tasks; q += nw) {
      // row-major enumeration of the lower triangle: q -> (a, b), b <= a
      int a = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= q) ++a;
      while (a * (a + 1) / 2 > q) --a;
      const int b = q - a * (a + 1) / 2;
      const int I = K + 1 + a, J = K + 1 + b;
      tile_gemm(tile(I, J), tile(I, K), tile(J, K), ld, I == J, lane);
    }
    __syncthreads();
  }
  }  // MODE != 3
  if (s_fail) {
    if (t == 0) {
      io.status[p] = PD_SLOT_JSI_NOT_SPD;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }

  // ---- solve + residual contract (forward_dynamics.cpp:99-116) --------------
  if (warp == 0) warp_llt_solve(Mb, ld, np, invd, vx, lane);
  double sq = 0.0;
  for (int i = t; i < n; i += nt) sq = fma(ws[jst::TD * n + i], ws[jst::TD * n + i], sq);
  const double scale = fmax(sqrt(block_sum(sq, br)), 2.2250738585072014e-308);  // block_sum syncs
  int code = PD_SLOT_OK;
  for (int pass = 0; pass < 2; ++pass) {
    double rr = 0.0;
    for (int i = t; i < npad; i += nt) {
      // (M x)_i from the saved diagonal and the untouched strict upper triangle
      double s = (i < n) ? ws[jst::TD * n + i] : 0.0;
      s = fma(-dg[i], vx[i], s);
      for (int j = 0; j < i; ++j) s = fma(-Mb[(size_t)j * ld + i], vx[j], s);
      for (int j = i + 1; j < npad; ++j) s = fma(-Mb[(size_t)i * ld + j], vx[j], s);
      vw[i] = s;
      rr = fma(s, s, rr);
    }
    const double rn = sqrt(block_sum(rr, br));
    if (!(rn > 1e-9 * scale)) break;
    if (pass == 1) {
      code = PD_SLOT_JSI_REFINE_FAILED;
      break;
    }
    if (warp == 0) warp_llt_solve(Mb, ld, np, invd, vw, lane);
    __syncthreads();
    for (int i = t; i < npad; i += nt) vx[i] += vw[i];
    __syncthreads();
  }
  for (int i = t; i < n; i += nt) io.put_qdd(i, p, vx[i]);
  if (t == 0) {
    io.status[p] = code;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

// Warps per CTA: one for two panels or fewer (the tile tasks of a step are
// serial there); otherwise enough to cover a panel step's trailing update,
// fewer when the batch alone fills the GPU.
int jsiia_warps(int n, int64_t batch, int sm_count) {
  const int np = (n + 31) / 32;
  if (np <= 2) return 1;
  const int tiles = np * (np - 1) / 2;
  if (batch >= 4 * (int64_t)sm_count) return np <= 4 ? 2 : 4;
  return tiles < 8 ? tiles : 8;
}

bool jsiia_smem_path(int n) { return jsiia_workspace_bytes(n) <= 200 * 1024; }

void launch_jsiia(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, int sm_count,
                  int64_t sel_B, cudaStream_t s) {
  const int n = mv.n;
  const int nt = 32 * jsiia_warps(n, sel_B, sm_count);
  const size_t ws_bytes = jsiia_workspace_bytes(n);
  if (jsiia_smem_path(n)) {
    cudaFuncSetAttribute(jsiia_tiled_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
    jsiia_tiled_kernel<true><<<(unsigned)io.B, nt, ws_bytes, s>>>(mv, io, nullptr, 0);
  } else {
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      jsiia_tiled_kernel<false><<<(unsigned)nb, nt, 0, s>>>(mv, io, gws, b0);
    }
  }
}

// Grid-wide M build + blocked Cholesky for long chains in small batches (c4).
// A MODE-2 build left S0, FB = Ic0 S0 and tau_delta of each chain in
// workspace slots 0..count-1; here every warp of a cooperative grid works on
// one chain after the other:
//   phase 0: M tiles M_ij = S0_min . FB_max (both triangles, identity padding),
//            diag(M), x = tau_delta -- a tile per warp task, rows staged in smem;
//   panels:  TRSM of the panel, then the trailing update, with the next
//            diagonal tile updated first by warp 0 and factored right away
//            (two grid barriers per panel).
// Tiles are staged through per-warp shared memory and read from global memory
// through L2 (ld.global.cg, never a stale L1 line); the SPD verdict goes to
// the slot's flag for the MODE-3 solve.
constexpr int kTs = 34;  // smem tile leading dimension (16-byte rows)

// NT tiles staged at once: every load is issued before the first shared
// store, so the warp pays one L2 round trip for all of them (the tiles were
// written by other SMs just before the grid barrier; a round trip is ~1 us).
template <int NT>
__device__ __forceinline__ void warp_tiles_in(double* const (&dst)[NT], const double* const (&src)[NT], int ld,
                                              int lane) {
  double2 v[NT][16];
#pragma unroll
  for (int k = 0; k < NT; ++k)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = lane + 32 * q, r = e >> 4, c = (e & 15) * 2;
      v[k][q] = __ldcg(reinterpret_cast<const double2*>(src[k] + (size_t)r * ld + c));
    }
#pragma unroll
  for (int k = 0; k < NT; ++k)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = lane + 32 * q, r = e >> 4, c = (e & 15) * 2;
      *reinterpret_cast<double2*>(dst[k] + r * kTs + c) = v[k][q];
    }
  __syncwarp();
}
__device__ __forceinline__ void warp_tile_in(double* dst, const double* src, int ld, int lane) {
  double* const d[1] = {dst};
  const double* const s[1] = {src};
  warp_tiles_in<1>(d, s, ld, lane);
}
__device__ __forceinline__ void warp_tile_out(double* dst, int ld, const double* src, int lane, bool lower_only) {
  __syncwarp();
#pragma unroll 4
  for (int e = lane; e < 32 * 16; e += 32) {
    const int r = e >> 4, c = (e & 15) * 2;
    const double2 v = *reinterpret_cast<const double2*>(src + r * kTs + c);
    if (!lower_only || c + 1 <= r) {
      *reinterpret_cast<double2*>(dst + (size_t)r * ld + c) = v;
    } else if (c <= r) {
      dst[(size_t)r * ld + c] = v.x;
    }
  }
  __syncwarp();
}
// r (row `lane` of C) -= row `lane` of A times B^T, A and B^T staged in smem.
__device__ __forceinline__ void tile_gemm_rows(double (&r)[32], const double* sA, const double* sB, int lane) {
#pragma unroll 1
  for (int p = 0; p < 32; p += 2) {
    const double2 a = *reinterpret_cast<const double2*>(sA + lane * kTs + p);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 b = *reinterpret_cast<const double2*>(sB + j * kTs + p);
      r[j] = fma(-a.x, b.x, r[j]);
      r[j] = fma(-a.y, b.y, r[j]);
    }
  }
}

__global__ void __launch_bounds__(256) jsiia_factor_coop(double* __restrict__ gws, int n, int count) {
  namespace cgr = cooperative_groups;
  cgr::grid_group grid = cgr::this_grid();
  extern __shared__ __align__(16) double coop_smem[];  // per warp: A, B tiles + 32 reciprocals
  double (*stile)[3][32 * kTs] = reinterpret_cast<double (*)[3][32 * kTs]>(coop_smem);
  double (*sinv)[32] = reinterpret_cast<double (*)[32]>(coop_smem + 8 * 3 * 32 * kTs);
  const JstLayout L = jst_layout(n);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  // task slot of this warp: consecutive slots on different SMs (warp 0 of every
  // CTA first), so the few tasks of the late panels -- the critical path --
  // each get an SM to themselves instead of sharing CTA 0's
  const int gw = wl * (int)gridDim.x + (int)blockIdx.x;
  const int np = L.np, npad = L.npad, ld = L.ld;
  double* sA = stile[wl][0];
  double* sB = stile[wl][1];
  double* sC = stile[wl][2];
  for (int c = 0; c < count; ++c) {
    double* ws = gws + (size_t)c * L.total;
    double* Mb = ws + L.m_off;
    double* vx = ws + L.v_off;
    double* dg = vx + 2 * (size_t)npad;
    double* invd = vx + 3 * (size_t)npad;
    double* flag = ws + L.total - 1;
    auto tile = [&](int I, int J) { return Mb + (size_t)(32 * I) * ld + 32 * J; };
    // ---- phase 0: M = [S0_min . FB_max], identity padding, diag, x = td
    for (int q = gw; q < np * np; q += nwarps) {
      const int I = q / np, J = q % np;
      // rows i = 32 I + r: S0_i (sA) and FB_i (sB), 6 doubles each, field-major in ws
      for (int e = lane; e < 6 * 32; e += 32) {
        const int f = e >> 5, r = e & 31, i = 32 * I + r;
        sA[f * 32 + r] = i < n ? __ldcg(ws + (size_t)(jst::S0 + f) * n + i) : 0.0;
        sB[f * 32 + r] = i < n ? __ldcg(ws + (size_t)(jst::FB + f) * n + i) : 0.0;
      }
      __syncwarp();
      const int j = 32 * J + lane;
      const bool jr = j < n;
      double sj[6], fj[6];
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        sj[f] = jr ? __ldcg(ws + (size_t)(jst::S0 + f) * n + j) : 0.0;
        fj[f] = jr ? __ldcg(ws + (size_t)(jst::FB + f) * n + j) : 0.0;
      }
      for (int r = 0; r < 32; ++r) {
        const int i = 32 * I + r;
        double mij;
        if (i < n && jr) {
          const bool low = j <= i;  // lower: S0_j . FB_i, upper: S0_i . FB_j
          double acc = 0.0;
#pragma unroll
          for (int f = 0; f < 6; ++f) acc = fma(low ? sj[f] : sA[f * 32 + r], low ? sB[f * 32 + r] : fj[f], acc);
          mij = acc;
        } else {
          mij = (i == j) ? 1.0 : 0.0;
        }
        Mb[(size_t)i * ld + j] = mij;
        if (i == j) dg[i] = mij;
      }
      __syncwarp();
    }
    for (int i = (int)(blockIdx.x * blockDim.x + threadIdx.x); i < npad; i += (int)(gridDim.x * blockDim.x))
      vx[i] = i < n ? __ldcg(ws + (size_t)jst::TD * n + i) : 0.0;
    grid.sync();
    // ---- blocked Cholesky
    if (gw == 0) {
      warp_tile_in(sA, tile(0, 0), ld, lane);
      const bool ok = tile_potrf(sA, kTs, invd, lane);
      warp_tile_out(tile(0, 0), ld, sA, lane, true);
      if (lane == 0) *flag = ok ? 0.0 : 1.0;
    }
    grid.sync();
    for (int K = 0; K < np; ++K) {
      if (__ldcg(flag) != 0.0) break;  // grid-uniform: forward_dynamics.cpp:93-98
      if (K + 1 + gw < np) {
        sinv[wl][lane] = __ldcg(invd + 32 * K + lane);
        bool first = true;
        for (int I = K + 1 + gw; I < np; I += nwarps) {
          if (first) {  // L_KK and the first panel tile in one round trip
            double* const d[2] = {sA, sB};
            const double* const src[2] = {tile(K, K), tile(I, K)};
            warp_tiles_in<2>(d, src, ld, lane);
            first = false;
          } else {
            warp_tile_in(sB, tile(I, K), ld, lane);
          }
          tile_trsm(sA, kTs, sinv[wl], sB, lane);
          warp_tile_out(tile(I, K), ld, sB, lane, false);
        }
      }
      grid.sync();
      const int m = np - 1 - K;  // trailing tiles (I, J), K < J <= I; task 0 = the next diagonal tile
      const int tasks = m * (m + 1) / 2;
      for (int q = gw; q < tasks; q += nwarps) {
        int a = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
        while ((a + 1) * (a + 2) / 2 <= q) ++a;
        while (a * (a + 1) / 2 > q) --a;
        const int b = q - a * (a + 1) / 2;
        const int I = K + 1 + a, J = K + 1 + b;
        {  // L_IK, L_JK and C_IJ in one round trip, all coalesced
          double* const d[3] = {sA, sB, sC};
          const double* const src[3] = {tile(I, K), tile(J, K), tile(I, J)};
          warp_tiles_in<3>(d, src, ld, lane);
        }
        double r[32];
        load_row<false>(r, sC + lane * kTs);
        tile_gemm_rows(r, sA, sB, lane);
        if (q == 0) {  // the next diagonal tile: keep it in smem and factor it right away
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(sA + lane * kTs + j) = make_double2(r[j], r[j + 1]);
          __syncwarp();
          const bool ok = tile_potrf(sA, kTs, invd + 32 * (K + 1), lane);
          warp_tile_out(tile(K + 1, K + 1), ld, sA, lane, true);
          if (!ok && lane == 0) *flag = 1.0;
        } else {
          double* row = tile(I, J) + (size_t)lane * ld;
          if (I == J) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j <= lane) row[j] = r[j];
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 2) *reinterpret_cast<double2*>(row + j) = make_double2(r[j], r[j + 1]);
          }
        }
      }
      grid.sync();
    }
  }
}

// Solve + residual contract (forward_dynamics.cpp:99-116) for the
// cooperative path: one CTA of kWideWarps warps per chain. Tile rows of the
// right-hand side are owned round-robin by the warps. An owner folds each
// earlier block into its own as soon as that block is published (a shared
// flag per tile row, no CTA barrier per step): the rows of the tile it folds
// next are loaded before it waits, so a step's critical path is one 32-wide
// dot product plus the diagonal recurrence against the owner's staged
// diagonal tile. The residual uses the closed form of M (residual_closed).
constexpr int kWideWarps = 16;

// Flags are read and written with shared-memory atomics, bracketed by block
// fences: release (data, fence, flag) on the publishing side, acquire (flag,
// fence, data) on the waiting side.
// (one lane polls, so the warp's spin is one atomic at a time)
__device__ __forceinline__ void wait_flag(int* f, int want, int lane) {
  if (lane == 0)
    while (atomicAdd(f, 0) != want) {
    }
  __syncwarp();
  __threadfence_block();
}
__device__ __forceinline__ void publish(double* v, int J, int lane, double val, int* ready, int epoch) {
  v[32 * J + lane] = val;
  __threadfence_block();
  __syncwarp();
  if (lane == 0) atomicExch(ready + J, epoch);
}
__device__ __forceinline__ void stage_diag(const double* Mb, int ld, int J, double* T, int lane) {
#pragma unroll 8
  for (int e = lane; e < 32 * 32; e += 32)
    T[(e >> 5) * 33 + (e & 31)] = Mb[(size_t)(32 * J + (e >> 5)) * ld + 32 * J + (e & 31)];
  __syncwarp();
}
__device__ __forceinline__ double dot32(const double (&a)[32], const double* y) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    s0 = fma(a[c], y[c], s0);
    s1 = fma(a[c + 1], y[c + 1], s1);
    s2 = fma(a[c + 2], y[c + 2], s2);
    s3 = fma(a[c + 3], y[c + 3], s3);
  }
  return (s0 + s1) + (s2 + s3);
}

// (L L^T) v = v in place; flags `ready` take the values epoch (forward) and
// epoch + 1 (backward), so they never need resetting between solves.
__device__ void wide_llt_solve(const double* Mb, int ld, int np, const double* invd, double* v, double* sT,
                               int* ready, int epoch, int warp, int lane) {
  double* T = sT + warp * 32 * 33;
  // forward: L y = v, tile rows ascending
  for (int J = warp; J < np; J += kWideWarps) {
    stage_diag(Mb, ld, J, T, lane);
    double acc = v[32 * J + lane];
    const double* rowJ = Mb + (size_t)(32 * J + lane) * ld;
    for (int I = 0; I < J; ++I) {
      double a[32];  // row `lane` of L_JI, loaded before the wait
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const double2 t = *reinterpret_cast<const double2*>(rowJ + 32 * I + c);
        a[c] = t.x;
        a[c + 1] = t.y;
      }
      wait_flag(ready + I, epoch, lane);
      acc -= dot32(a, v + 32 * I);
    }
    const double id = invd[32 * J + lane];
    double yo = 0.0;
#pragma unroll 8
    for (int m = 0; m < 32; ++m) {
      const double ym = __shfl_sync(0xffffffffu, acc * id, m);
      yo = (lane == m) ? ym : yo;
      acc = (lane > m) ? fma(-T[lane * 33 + m], ym, acc) : acc;
    }
    publish(v, J, lane, yo, ready, epoch);
  }
  __syncthreads();
  // backward: L^T x = y, tile rows descending
  const int last = warp + ((np - 1 - warp) / kWideWarps) * kWideWarps;
  for (int J = last; J >= 0 && warp < np; J -= kWideWarps) {
    stage_diag(Mb, ld, J, T, lane);
    double acc = v[32 * J + lane];
    for (int I = np - 1; I > J; --I) {
      double a[32];  // column `lane` of L_IJ (coalesced), loaded before the wait
#pragma unroll
      for (int c = 0; c < 32; ++c) a[c] = Mb[(size_t)(32 * I + c) * ld + 32 * J + lane];
      wait_flag(ready + I, epoch + 1, lane);
      acc -= dot32(a, v + 32 * I);
    }
    const double id = invd[32 * J + lane];
    double xo = 0.0;
#pragma unroll 8
    for (int m = 31; m >= 0; --m) {
      const double xm = __shfl_sync(0xffffffffu, acc * id, m);
      xo = (lane == m) ? xm : xo;
      acc = (lane < m) ? fma(-T[m * 33 + lane], xm, acc) : acc;
    }
    publish(v, J, lane, xo, ready, epoch + 1);
  }
  __syncthreads();
}

// r = td - M x from the closed form of M (M_ij = S0_min(i,j) . FB_max(i,j), the
// same dot products the factorization's M holds): (M x)_i = FB_i . P_i +
// S0_i . Q_i with P_i = sum_{j<=i} S0_j x_j and Q_i = sum_{j>i} FB_j x_j. Two
// CTA scans of 6-vectors instead of reading all n^2 entries of M through one
// SM. Returns sum r_i^2 (every thread).
__device__ double residual_closed(const double* ws, int n, const double* x, double* r, ScanSmem& sm,
                                  BlockReduce& br) {
  const int t = threadIdx.x, nt = blockDim.x;
  const int lpt = (n + nt - 1) / nt;
  const int i0 = t * lpt, i1 = min(n, i0 + lpt), nact = (n + lpt - 1) / lpt;
  const double* td = ws + (size_t)jst::TD * n;
  auto s0 = [&](int i) { return ws_get_sv(ws, n, jst::S0, i); };
  auto fb = [&](int i) { return ws_get_sv(ws, n, jst::FB, i); };
  auto arr = [](const Sv& v) { return Arr<6>{{v.a.x, v.a.y, v.a.z, v.l.x, v.l.y, v.l.z}}; };
  auto sv = [](const Arr<6>& a) { return Sv{mk(a.v[0], a.v[1], a.v[2]), mk(a.v[3], a.v[4], a.v[5])}; };
  Sv lp = svzero(), lq = svzero();
  for (int i = i0; i < i1; ++i) {
    lp = svfma(x[i], s0(i), lp);
    lq = svfma(x[i], fb(i), lq);
  }
  const Sv P0 = sv(block_exclusive<6, false>(arr(lp), AddOp{}, sm, nact));
  const Sv Q0 = sv(block_exclusive<6, true>(arr(lq), AddOp{}, sm, nact));
  // P inclusive walking up, Q exclusive walking down; r_i = td_i - FB_i.P_i - S0_i.Q_i
  Sv P = P0;
  for (int i = i0; i < i1; ++i) {
    P = svfma(x[i], s0(i), P);
    r[i] = td[i] - dot(fb(i), P);
  }
  Sv Q = Q0;
  double rr = 0.0;
  for (int i = i1 - 1; i >= i0; --i) {
    const double ri = r[i] - dot(s0(i), Q);
    r[i] = ri;
    rr = fma(ri, ri, rr);
    Q = svfma(x[i], fb(i), Q);
  }
  return block_sum(rr, br);
}

size_t wide_solve_smem(int np) { return sizeof(double) * kWideWarps * 32 * 33 + sizeof(int) * np; }

__global__ void __launch_bounds__(32 * kWideWarps) jsiia_solve_wide(BatchIO io, double* __restrict__ gws, int n) {
  extern __shared__ double wide_smem[];
  __shared__ BlockReduce br;
  __shared__ ScanSmem scan_sm;
  double* sT = wide_smem;
  int* ready = reinterpret_cast<int*>(wide_smem + kWideWarps * 32 * 33);
  const JstLayout L = jst_layout(n);
  const int64_t p = blockIdx.x;
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, warp = t >> 5;
  double* ws = gws + (size_t)blockIdx.x * L.total;
  const int np = L.np, npad = L.npad, ld = L.ld;
  const double* Mb = ws + L.m_off;
  double* vx = ws + L.v_off;
  double* vw = vx + npad;
  const double* invd = vx + 3 * (size_t)npad;
  for (int k = t; k < np; k += nt) ready[k] = 0;
  __syncthreads();
  if (ws[L.total - 1] != 0.0) {  // forward_dynamics.cpp:93-98
    if (t == 0) {
      io.status[p] = PD_SLOT_JSI_NOT_SPD;
      io.eround[p] = 0;
      io.eindex[p] = 0;
    }
    return;
  }
  const double* td = ws + (size_t)jst::TD * n;
  wide_llt_solve(Mb, ld, np, invd, vx, sT, ready, 1, warp, lane);
  double sq = 0.0;
  for (int i = t; i < n; i += nt) sq = fma(td[i], td[i], sq);
  const double scale = fmax(sqrt(block_sum(sq, br)), 2.2250738585072014e-308);
  int code = PD_SLOT_OK;
  for (int pass = 0; pass < 2; ++pass) {
    __syncthreads();  // x complete
    for (int i = n + t; i < npad; i += nt) vw[i] = 0.0;
    const double rn = sqrt(residual_closed(ws, n, vx, vw, scan_sm, br));  // syncs
    if (!(rn > 1e-9 * scale)) break;
    if (pass == 1) {
      code = PD_SLOT_JSI_REFINE_FAILED;
      break;
    }
    wide_llt_solve(Mb, ld, np, invd, vw, sT, ready, 3, warp, lane);
    for (int i = t; i < npad; i += nt) vx[i] += vw[i];
    __syncthreads();
  }
  for (int i = t; i < n; i += nt) io.put_qdd(i, p, vx[i]);
  if (t == 0) {
    io.status[p] = code;
    io.eround[p] = 0;
    io.eindex[p] = 0;
  }
}

// Long chains in small batches: build (MODE 2, a CTA per chain), grid-wide
// factorization, solve (MODE 3). Workspace slots 0..B-1 of gws.
bool jsiia_coop_path(int n, int64_t batch) { return !jsiia_smem_path(n) && batch <= 4; }

void launch_jsiia_coop(const ModelView& mv, const BatchIO& io, double* gws, int sm_count, int64_t sel_B,
                       cudaStream_t s) {
  const int n = mv.n;
  (void)sel_B;
  // 512 threads, 2 links each (1024-link chain): 256 x 4 0.861 ms, 512 x 2
  // 0.811, 1024 x 1 0.836 (spills at 64 registers) for c4 JSIIA end to end
  constexpr int kPrepThreads = 512;
  jsiia_tiled_kernel<false, 2, kPrepThreads><<<(unsigned)io.B, kPrepThreads, 0, s>>>(mv, io, gws, 0);
  int count = (int)io.B;
  void* args[] = {&gws, (void*)&n, &count};
  const size_t smem = sizeof(double) * 8 * (3 * 32 * kTs + 32);
  cudaFuncSetAttribute(jsiia_factor_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchCooperativeKernel((const void*)jsiia_factor_coop, dim3((unsigned)sm_count), dim3(256), args, smem, s);
  const size_t wsm = wide_solve_smem(jst_layout(n).np);
  cudaFuncSetAttribute(jsiia_solve_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
  jsiia_solve_wide<<<(unsigned)io.B, 32 * kWideWarps, wsm, s>>>(io, gws, n);
}

// Joint-space inertia of every problem into d_M[p][i][j] (same build as the
// solve path: CRBA closed form, exactly symmetric).
void launch_jsi(const ModelView& mv, const BatchIO& io, double* gws, int64_t gws_slots, int sm_count, double* d_M,
                cudaStream_t s) {
  const int n = mv.n;
  const int nt = 32 * jsiia_warps(n, io.B, sm_count);
  const size_t ws_bytes = jsiia_workspace_bytes(n);
  if (jsiia_smem_path(n)) {
    cudaFuncSetAttribute(jsiia_tiled_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
    jsiia_tiled_kernel<true, 1><<<(unsigned)io.B, nt, ws_bytes, s>>>(mv, io, nullptr, 0, d_M);
  } else {
    for (int64_t b0 = 0; b0 < io.B; b0 += gws_slots) {
      const int64_t nb = (io.B - b0 < gws_slots) ? io.B - b0 : gws_slots;
      jsiia_tiled_kernel<false, 1><<<(unsigned)nb, nt, 0, s>>>(mv, io, gws, b0, d_M);
    }
  }
}

}  // namespace pd

// The paper's building block 2 on its own: batched symmetric block
// tri-diagonal solves by odd-even elimination, oee_solve<B, M>
// (include/pardyn/oee.hpp:149-189) for block sizes B = 1..6 and M = 1..4
// right-hand-side columns (the system CFA reduces to is B = 5, M = 1), for
// user systems whose pivots need not be positive definite.
//
// A CTA per system, a thread per block row (n <= 256), the row's D, U, R in
// registers. Every round each row publishes what its two partners read -- a
// full-pivot LU of its pivot D_k (FullPivLU semantics: largest |a| of the
// trailing corner, first in column-major order on ties; invertible iff every
// |u_jj| > B eps |max pivot|), its coupling U_k and right-hand side R_k --
// then, after one barrier, solves its own coefficients from the published
// factors exactly as oee_eliminate_round (oee.hpp:73-145) does:
//   up   (pivot k = i+h): E = D_k^{-1} U_i^T, D_i -= E^T U_i^T, R_i -= E^T R_k,
//                         U_i <- -E^T U_k                 (only if i + 2h < n)
//   down (pivot k = i-h): K = D_k^{-1} U_k,   D_i -= K^T U_k,   R_i -= K^T R_k.
// Errors follow the reference: the smallest failing row reports its first
// failing pivot (up before down) and the round; the final block solves report
// the smallest singular row.
//
// The CFA kernels (cfa.cu) keep their Cholesky form: their pivots are Schur
// complements of the SPD constraint operator.
#include "pd_batch.cuh"

namespace pd {

namespace {

constexpr double kEps = 2.220446049250313e-16;

// In-place full-pivot LU of a row-major BxB; rowt / colt are the successive
// transpositions (Eigen's m_rowsTranspositions / m_colsTranspositions).
template <int B>
struct Lu {
  double a[B * B];
  int rowt[B], colt[B];
  bool invertible;
};

template <int B>
__device__ __forceinline__ void lu_factor(Lu<B>& f) {
  int nonzero = B;
  double maxpivot = 0.0;
  for (int k = 0; k < B; ++k) {
    double big = -1.0;
    int br = k, bc = k;
    for (int c = k; c < B; ++c)
      for (int r = k; r < B; ++r) {
        const double v = fabs(f.a[r * B + c]);
        if (v > big) {
          big = v;
          br = r;
          bc = c;
        }
      }
    if (big == 0.0) {
      nonzero = k;
      for (int i = k; i < B; ++i) f.rowt[i] = f.colt[i] = i;
      break;
    }
    maxpivot = fmax(maxpivot, big);
    f.rowt[k] = br;
    f.colt[k] = bc;
    if (br != k)
      for (int c = 0; c < B; ++c) {
        const double t = f.a[k * B + c];
        f.a[k * B + c] = f.a[br * B + c];
        f.a[br * B + c] = t;
      }
    if (bc != k)
      for (int r = 0; r < B; ++r) {
        const double t = f.a[r * B + k];
        f.a[r * B + k] = f.a[r * B + bc];
        f.a[r * B + bc] = t;
      }
    for (int r = k + 1; r < B; ++r) f.a[r * B + k] /= f.a[k * B + k];
    for (int r = k + 1; r < B; ++r)
      for (int c = k + 1; c < B; ++c) f.a[r * B + c] -= f.a[r * B + k] * f.a[k * B + c];
  }
  int rank = 0;
  const double thr = (double)B * kEps * fabs(maxpivot);  // FullPivLU threshold: diagonal size x eps
  for (int i = 0; i < nonzero; ++i)
    if (fabs(f.a[i * B + i]) > thr) ++rank;
  f.invertible = rank == B;
}

// x <- D^{-1} x for one column, from factors read through `lu` (field-major
// ws[f * n + k] or registers).
template <int B, class G>
__device__ __forceinline__ void lu_solve(G lu, const int* rowt, const int* colt, double c[B]) {
  for (int k = 0; k < B; ++k)
    if (rowt[k] != k) {
      const double t = c[k];
      c[k] = c[rowt[k]];
      c[rowt[k]] = t;
    }
  for (int r = 0; r < B; ++r)
    for (int k = 0; k < r; ++k) c[r] -= lu(r * B + k) * c[k];
  for (int r = B - 1; r >= 0; --r) {
    for (int k = r + 1; k < B; ++k) c[r] -= lu(r * B + k) * c[k];
    c[r] /= lu(r * B + r);
  }
  for (int k = B - 1; k >= 0; --k)
    if (colt[k] != k) {
      const double t = c[k];
      c[k] = c[colt[k]];
      c[colt[k]] = t;
    }
}

// published fields per row (ws[f * n + k]): LU (B*B), U (B*B), R (B*M)
template <int B, int M>
struct Pub {
  static constexpr int LU = 0, U = B * B, R = 2 * B * B, FIELDS = 2 * B * B + B * M;
};

}  // namespace

// rhs / x blocks are row-major B x M: element (r, c) at r * M + c.
// Rounds: the state enters at coupling distance h0 after round0 rounds
// (OeeState, oee.hpp:57-67; `upper` holds coupling[i] for i < n - h0) and
// nrounds rounds run. With st == nullptr the final block solves follow (the
// full oee_solve); otherwise the advanced state (diag, coupling at the new
// distance, rhs) is written to st_* -- oee_eliminate_round repeated.
struct OeeRounds {
  int h0, round0, nrounds;
  double *st_diag, *st_coupling, *st_rhs;
};

template <int B, int M>
__global__ void __launch_bounds__(256) oee_block_kernel(const double* __restrict__ diag,
                                                        const double* __restrict__ upper,
                                                        const double* __restrict__ rhs, double* __restrict__ x, int n,
                                                        int32_t* __restrict__ status, int32_t* __restrict__ eround,
                                                        int32_t* __restrict__ eindex, OeeRounds rr) {
  using P = Pub<B, M>;
  extern __shared__ double ws[];                                 // [P::FIELDS][n]
  int* perm = reinterpret_cast<int*>(ws + P::FIELDS * n);         // [2B][n]: rowt, colt
  unsigned char* okf = reinterpret_cast<unsigned char*>(perm + 2 * B * n);  // [n]
  __shared__ int s_bad;
  const int64_t p = blockIdx.x;
  const int i = threadIdx.x;
  const bool own = i < n;
  const int h0 = rr.h0, nu0 = n > h0 ? n - h0 : 0;
  const double* Dg = diag + (size_t)p * n * B * B;
  const double* Ug = upper + (size_t)p * nu0 * B * B;
  const double* Rg = rhs + (size_t)p * n * B * M;
  double D[B * B], U[B * B], R[B * M];
  if (own) {
    for (int k = 0; k < B * B; ++k) D[k] = __ldg(Dg + (size_t)i * B * B + k);
    for (int k = 0; k < B * B; ++k) U[k] = (i + h0 < n) ? __ldg(Ug + (size_t)i * B * B + k) : 0.0;
    for (int k = 0; k < B * M; ++k) R[k] = __ldg(Rg + (size_t)i * B * M + k);
  }
  const int rounds = rr.round0 + rr.nrounds;
  int h = h0;
  for (int round = rr.round0 + 1; round <= rounds; ++round, h <<= 1) {
    if (i == 0) s_bad = n;
    if (own) {  // publish: LU of the pivot, the coupling to i + h, the rhs
      Lu<B> f;
      for (int k = 0; k < B * B; ++k) f.a[k] = D[k];
      lu_factor<B>(f);
      for (int k = 0; k < B * B; ++k) ws[(P::LU + k) * n + i] = f.a[k];
      for (int k = 0; k < B; ++k) {
        perm[k * n + i] = f.rowt[k];
        perm[(B + k) * n + i] = f.colt[k];
      }
      okf[i] = f.invertible ? 1 : 0;
      for (int k = 0; k < B * B; ++k) ws[(P::U + k) * n + i] = U[k];
      for (int k = 0; k < B * M; ++k) ws[(P::R + k) * n + i] = R[k];
    }
    __syncthreads();
    if (own) {
      int bad_pivot = -1;
      if (i < n - h && !okf[i + h]) bad_pivot = i + h;
      else if (i >= h && !okf[i - h]) bad_pivot = i - h;
      if (bad_pivot >= 0) {
        atomicMin(&s_bad, i);
      } else {
        double nD[B * B], nR[B * M];
        for (int k = 0; k < B * B; ++k) nD[k] = D[k];
        for (int k = 0; k < B * M; ++k) nR[k] = R[k];
        if (i < n - h) {  // E = D_k^{-1} U_i^T
          const int k = i + h;
          int rt[B], ct[B];
          for (int j = 0; j < B; ++j) {
            rt[j] = perm[j * n + k];
            ct[j] = perm[(B + j) * n + k];
          }
          auto lu = [&](int f) { return ws[(P::LU + f) * n + k]; };
          double E[B][B];  // E[col][row]
          for (int c = 0; c < B; ++c) {
            for (int r = 0; r < B; ++r) E[c][r] = U[c * B + r];  // column c of U^T = row c of U
            lu_solve<B>(lu, rt, ct, E[c]);
          }
          // D -= E^T U^T: (E^T U^T)[a][b] = sum_r E[a][r] U[b][r]
          for (int a = 0; a < B; ++a)
            for (int b = 0; b < B; ++b) {
              double s = 0.0;
              for (int r = 0; r < B; ++r) s += E[a][r] * U[b * B + r];
              nD[a * B + b] -= s;
            }
          for (int a = 0; a < B; ++a)
            for (int c = 0; c < M; ++c) {
              double s = 0.0;
              for (int r = 0; r < B; ++r) s += E[a][r] * ws[(P::R + r * M + c) * n + k];
              nR[a * M + c] -= s;
            }
          if (i < n - 2 * h) {  // U_i <- -E^T U_k
            double nU[B * B];
            for (int a = 0; a < B; ++a)
              for (int b = 0; b < B; ++b) {
                double s = 0.0;
                for (int r = 0; r < B; ++r) s += E[a][r] * ws[(P::U + r * B + b) * n + k];
                nU[a * B + b] = -s;
              }
            for (int q = 0; q < B * B; ++q) U[q] = nU[q];
          }
        }
        if (i >= h) {  // K = D_k^{-1} U_k
          const int k = i - h;
          int rt[B], ct[B];
          for (int j = 0; j < B; ++j) {
            rt[j] = perm[j * n + k];
            ct[j] = perm[(B + j) * n + k];
          }
          auto lu = [&](int f) { return ws[(P::LU + f) * n + k]; };
          double K[B][B];  // K[col][row]
          for (int c = 0; c < B; ++c) {
            for (int r = 0; r < B; ++r) K[c][r] = ws[(P::U + r * B + c) * n + k];
            lu_solve<B>(lu, rt, ct, K[c]);
          }
          for (int a = 0; a < B; ++a)
            for (int b = 0; b < B; ++b) {
              double s = 0.0;
              for (int r = 0; r < B; ++r) s += K[a][r] * ws[(P::U + r * B + b) * n + k];
              nD[a * B + b] -= s;
            }
          for (int a = 0; a < B; ++a)
            for (int c = 0; c < M; ++c) {
              double s = 0.0;
              for (int r = 0; r < B; ++r) s += K[a][r] * ws[(P::R + r * M + c) * n + k];
              nR[a * M + c] -= s;
            }
        }
        for (int k = 0; k < B * B; ++k) D[k] = nD[k];
        for (int k = 0; k < B * M; ++k) R[k] = nR[k];
      }
    }
    __syncthreads();
    if (s_bad < n) {
      if (i == s_bad) {  // the smallest failing row names its first failing pivot
        status[p] = PD_SLOT_OEE_SINGULAR_PIVOT;
        eround[p] = round;
        eindex[p] = (i < n - h && !okf[i + h]) ? i + h : i - h;
      }
      return;
    }
    __syncthreads();  // published fields are rewritten next round
  }
  if (rr.st_diag) {  // the advanced state: coupling now at distance h
    if (own) {
      for (int k = 0; k < B * B; ++k) rr.st_diag[((size_t)p * n + i) * B * B + k] = D[k];
      for (int k = 0; k < B * M; ++k) rr.st_rhs[((size_t)p * n + i) * B * M + k] = R[k];
      const int nu = n > h ? n - h : 0;
      if (i < nu)
        for (int k = 0; k < B * B; ++k) rr.st_coupling[((size_t)p * nu + i) * B * B + k] = U[k];
    }
    if (i == 0) {
      status[p] = PD_SLOT_OK;
      eround[p] = 0;
      eindex[p] = 0;
    }
    return;
  }
  // final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187)
  if (i == 0) s_bad = n;
  __syncthreads();
  if (own) {
    Lu<B> f;
    for (int k = 0; k < B * B; ++k) f.a[k] = D[k];
    lu_factor<B>(f);
    if (!f.invertible) atomicMin(&s_bad, i);
    for (int c = 0; c < M; ++c) {
      double col[B];
      for (int r = 0; r < B; ++r) col[r] = R[r * M + c];
      lu_solve<B>([&](int q) { return f.a[q]; }, f.rowt, f.colt, col);
      for (int r = 0; r < B; ++r) x[((size_t)p * n + i) * B * M + r * M + c] = col[r];
    }
  }
  __syncthreads();
  if (i == 0) {
    status[p] = s_bad < n ? PD_SLOT_OEE_SINGULAR_FINAL : PD_SLOT_OK;
    eround[p] = s_bad < n ? rounds : 0;
    eindex[p] = s_bad < n ? s_bad : 0;
  }
}

namespace {
struct OeeArgs {
  const double *diag, *upper, *rhs;
  double* x;
  int64_t batch;
  int n;
  int32_t *status, *eround, *eindex;
  OeeRounds rr;
};

template <int B, int M>
void go_oee(const OeeArgs& a, cudaStream_t s) {
  const size_t bytes = (size_t)Pub<B, M>::FIELDS * a.n * sizeof(double) + (size_t)2 * B * a.n * sizeof(int) + a.n;
  cudaFuncSetAttribute(oee_block_kernel<B, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  oee_block_kernel<B, M><<<(unsigned)a.batch, ((a.n + 31) / 32) * 32, bytes, s>>>(
      a.diag, a.upper, a.rhs, a.x, a.n, a.status, a.eround, a.eindex, a.rr);
}
template <int B>
bool go_oee_m(int m, const OeeArgs& a, cudaStream_t s) {
  switch (m) {
    case 1: go_oee<B, 1>(a, s); return true;
    case 2: go_oee<B, 2>(a, s); return true;
    case 3: go_oee<B, 3>(a, s); return true;
    case 4: go_oee<B, 4>(a, s); return true;
    default: return false;
  }
}
bool go_oee_b(int b, int m, const OeeArgs& a, cudaStream_t s) {
  if (a.n < 1 || a.n > 256) return false;
  switch (b) {
    case 1: return go_oee_m<1>(m, a, s);
    case 2: return go_oee_m<2>(m, a, s);
    case 3: return go_oee_m<3>(m, a, s);
    case 4: return go_oee_m<4>(m, a, s);
    case 5: return go_oee_m<5>(m, a, s);
    case 6: return go_oee_m<6>(m, a, s);
    default: return false;
  }
}
}  // namespace

bool launch_oee_block(int b, int m, const double* diag, const double* upper, const double* rhs, double* x,
                      int64_t batch, int n, int32_t* status, int32_t* eround, int32_t* eindex, cudaStream_t s) {
  int rounds = 0;
  while ((1 << rounds) < n) ++rounds;
  return go_oee_b(b, m, OeeArgs{diag, upper, rhs, x, batch, n, status, eround, eindex, OeeRounds{1, 0, rounds, nullptr, nullptr, nullptr}}, s);
}

bool launch_oee_rounds(int b, int m, const double* diag, const double* coupling, const double* rhs, int64_t batch,
                       int n, int distance, int round0, int nrounds, double* diag_out, double* coupling_out,
                       double* rhs_out, int32_t* status, int32_t* eround, int32_t* eindex, cudaStream_t s) {
  return go_oee_b(b, m, OeeArgs{diag, coupling, rhs, nullptr, batch, n, status, eround, eindex,
                                OeeRounds{distance, round0, nrounds, diag_out, coupling_out, rhs_out}}, s);
}

}  // namespace pd

// The paper's building block 2 on its own: batched symmetric block
// tri-diagonal solves by odd-even elimination with 5x5 blocks
// (oee_solve<5,1>, include/pardyn/oee.hpp:149-189 -- the system CFA reduces
// to), for user systems whose pivots need not be positive definite.
//
// A CTA per system, a thread per block row (n <= 256), the row's D, U, R in
// registers. Every round each row publishes what its two partners read -- a
// full-pivot LU of its pivot D_k (FullPivLU semantics: largest |a| of the
// trailing corner, first in column-major order on ties; invertible iff every
// |u_jj| > 5 eps |max pivot|), its coupling U_k and right-hand side R_k --
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

// In-place full-pivot LU of a row-major 5x5; rowt / colt are the successive
// transpositions (Eigen's m_rowsTranspositions / m_colsTranspositions).
struct Lu5 {
  double a[25];
  int rowt[5], colt[5];
  bool invertible;
};

__device__ __forceinline__ void lu5_factor(Lu5& f) {
  int nonzero = 5;
  double maxpivot = 0.0;
  for (int k = 0; k < 5; ++k) {
    double big = -1.0;
    int br = k, bc = k;
    for (int c = k; c < 5; ++c)
      for (int r = k; r < 5; ++r) {
        const double v = fabs(f.a[r * 5 + c]);
        if (v > big) {
          big = v;
          br = r;
          bc = c;
        }
      }
    if (big == 0.0) {
      nonzero = k;
      for (int i = k; i < 5; ++i) f.rowt[i] = f.colt[i] = i;
      break;
    }
    maxpivot = fmax(maxpivot, big);
    f.rowt[k] = br;
    f.colt[k] = bc;
    if (br != k)
      for (int c = 0; c < 5; ++c) {
        const double t = f.a[k * 5 + c];
        f.a[k * 5 + c] = f.a[br * 5 + c];
        f.a[br * 5 + c] = t;
      }
    if (bc != k)
      for (int r = 0; r < 5; ++r) {
        const double t = f.a[r * 5 + k];
        f.a[r * 5 + k] = f.a[r * 5 + bc];
        f.a[r * 5 + bc] = t;
      }
    for (int r = k + 1; r < 5; ++r) f.a[r * 5 + k] /= f.a[k * 5 + k];
    for (int r = k + 1; r < 5; ++r)
      for (int c = k + 1; c < 5; ++c) f.a[r * 5 + c] -= f.a[r * 5 + k] * f.a[k * 5 + c];
  }
  int rank = 0;
  const double thr = 5.0 * kEps * fabs(maxpivot);
  for (int i = 0; i < nonzero; ++i)
    if (fabs(f.a[i * 5 + i]) > thr) ++rank;
  f.invertible = rank == 5;
}

// x <- D^{-1} x for one column, from factors in shared memory (field-major
// ws[f * n + k]: 25 LU entries, then the 10 transpositions as doubles).
template <class G>
__device__ __forceinline__ void lu5_solve(G lu, const int* rowt, const int* colt, double c[5]) {
  for (int k = 0; k < 5; ++k)
    if (rowt[k] != k) {
      const double t = c[k];
      c[k] = c[rowt[k]];
      c[rowt[k]] = t;
    }
  for (int r = 0; r < 5; ++r)
    for (int k = 0; k < r; ++k) c[r] -= lu(r * 5 + k) * c[k];
  for (int r = 4; r >= 0; --r) {
    for (int k = r + 1; k < 5; ++k) c[r] -= lu(r * 5 + k) * c[k];
    c[r] /= lu(r * 5 + r);
  }
  for (int k = 4; k >= 0; --k)
    if (colt[k] != k) {
      const double t = c[k];
      c[k] = c[colt[k]];
      c[colt[k]] = t;
    }
}

// published fields per row (ws[f * n + k])
constexpr int P_LU = 0, P_U = 25, P_R = 50, P_FIELDS = 55;

}  // namespace

__global__ void __launch_bounds__(256) oee5_kernel(const double* __restrict__ diag, const double* __restrict__ upper,
                                                   const double* __restrict__ rhs, double* __restrict__ x, int n,
                                                   int32_t* __restrict__ status, int32_t* __restrict__ eround,
                                                   int32_t* __restrict__ eindex) {
  extern __shared__ double ws[];                       // [P_FIELDS][n]
  int* perm = reinterpret_cast<int*>(ws + P_FIELDS * n);  // [10][n]: rowt, colt
  unsigned char* okf = reinterpret_cast<unsigned char*>(perm + 10 * n);  // [n]
  __shared__ int s_bad, s_pivot;
  const int64_t p = blockIdx.x;
  const int i = threadIdx.x;
  const bool own = i < n;
  const double* Dg = diag + (size_t)p * n * 25;
  const double* Ug = upper + (size_t)p * (n > 0 ? n - 1 : 0) * 25;
  const double* Rg = rhs + (size_t)p * n * 5;
  double D[25], U[25], R[5];
  if (own) {
    for (int k = 0; k < 25; ++k) D[k] = __ldg(Dg + (size_t)i * 25 + k);
    for (int k = 0; k < 25; ++k) U[k] = (i + 1 < n) ? __ldg(Ug + (size_t)i * 25 + k) : 0.0;
    for (int r = 0; r < 5; ++r) R[r] = __ldg(Rg + (size_t)i * 5 + r);
  }
  const int rounds = ceil_log2_dev(n);
  int h = 1;
  for (int round = 1; round <= rounds; ++round, h <<= 1) {
    if (i == 0) {
      s_bad = n;
      s_pivot = 0;
    }
    if (own) {  // publish: LU of the pivot, the coupling to i + h, the rhs
      Lu5 f;
      for (int k = 0; k < 25; ++k) f.a[k] = D[k];
      lu5_factor(f);
      for (int k = 0; k < 25; ++k) ws[(P_LU + k) * n + i] = f.a[k];
      for (int k = 0; k < 5; ++k) {
        perm[k * n + i] = f.rowt[k];
        perm[(5 + k) * n + i] = f.colt[k];
      }
      okf[i] = f.invertible ? 1 : 0;
      for (int k = 0; k < 25; ++k) ws[(P_U + k) * n + i] = U[k];
      for (int r = 0; r < 5; ++r) ws[(P_R + r) * n + i] = R[r];
    }
    __syncthreads();
    if (own) {
      int bad_pivot = -1;
      if (i < n - h && !okf[i + h]) bad_pivot = i + h;
      else if (i >= h && !okf[i - h]) bad_pivot = i - h;
      if (bad_pivot >= 0) {
        atomicMin(&s_bad, i);
      } else {
        double nD[25], nR[5];
        for (int k = 0; k < 25; ++k) nD[k] = D[k];
        for (int r = 0; r < 5; ++r) nR[r] = R[r];
        if (i < n - h) {  // E = D_k^{-1} U_i^T
          const int k = i + h;
          int rt[5], ct[5];
          for (int j = 0; j < 5; ++j) {
            rt[j] = perm[j * n + k];
            ct[j] = perm[(5 + j) * n + k];
          }
          auto lu = [&](int f) { return ws[(P_LU + f) * n + k]; };
          double E[5][5];  // E[col][row]
          for (int c = 0; c < 5; ++c) {
            for (int r = 0; r < 5; ++r) E[c][r] = U[c * 5 + r];  // column c of U^T = row c of U
            lu5_solve(lu, rt, ct, E[c]);
          }
          // D -= E^T U^T: (E^T U^T)[a][b] = sum_r E[a][r] U[b][r]
          for (int a = 0; a < 5; ++a)
            for (int b = 0; b < 5; ++b) {
              double s = 0.0;
              for (int r = 0; r < 5; ++r) s += E[a][r] * U[b * 5 + r];
              nD[a * 5 + b] -= s;
            }
          for (int a = 0; a < 5; ++a) {
            double s = 0.0;
            for (int r = 0; r < 5; ++r) s += E[a][r] * ws[(P_R + r) * n + k];
            nR[a] -= s;
          }
          if (i < n - 2 * h) {  // U_i <- -E^T U_k
            double nU[25];
            for (int a = 0; a < 5; ++a)
              for (int b = 0; b < 5; ++b) {
                double s = 0.0;
                for (int r = 0; r < 5; ++r) s += E[a][r] * ws[(P_U + r * 5 + b) * n + k];
                nU[a * 5 + b] = -s;
              }
            for (int q = 0; q < 25; ++q) U[q] = nU[q];
          }
        }
        if (i >= h) {  // K = D_k^{-1} U_k
          const int k = i - h;
          int rt[5], ct[5];
          for (int j = 0; j < 5; ++j) {
            rt[j] = perm[j * n + k];
            ct[j] = perm[(5 + j) * n + k];
          }
          auto lu = [&](int f) { return ws[(P_LU + f) * n + k]; };
          double K[5][5];  // K[col][row]
          for (int c = 0; c < 5; ++c) {
            for (int r = 0; r < 5; ++r) K[c][r] = ws[(P_U + r * 5 + c) * n + k];
            lu5_solve(lu, rt, ct, K[c]);
          }
          for (int a = 0; a < 5; ++a)
            for (int b = 0; b < 5; ++b) {
              double s = 0.0;
              for (int r = 0; r < 5; ++r) s += K[a][r] * ws[(P_U + r * 5 + b) * n + k];
              nD[a * 5 + b] -= s;
            }
          for (int a = 0; a < 5; ++a) {
            double s = 0.0;
            for (int r = 0; r < 5; ++r) s += K[a][r] * ws[(P_R + r) * n + k];
            nR[a] -= s;
          }
        }
        for (int k = 0; k < 25; ++k) D[k] = nD[k];
        for (int r = 0; r < 5; ++r) R[r] = nR[r];
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
  // final block solves x_i = D_i^{-1} R_i (oee.hpp:168-187)
  if (i == 0) s_bad = n;
  __syncthreads();
  if (own) {
    Lu5 f;
    for (int k = 0; k < 25; ++k) f.a[k] = D[k];
    lu5_factor(f);
    if (!f.invertible) atomicMin(&s_bad, i);
    lu5_solve([&](int q) { return f.a[q]; }, f.rowt, f.colt, R);
    for (int r = 0; r < 5; ++r) x[((size_t)p * n + i) * 5 + r] = R[r];
  }
  __syncthreads();
  if (i == 0) {
    status[p] = s_bad < n ? PD_SLOT_OEE_SINGULAR_FINAL : PD_SLOT_OK;
    eround[p] = s_bad < n ? rounds : 0;
    eindex[p] = s_bad < n ? s_bad : 0;
  }
}

bool launch_oee5(const double* diag, const double* upper, const double* rhs, double* x, int64_t batch, int n,
                 int32_t* status, int32_t* eround, int32_t* eindex, cudaStream_t s) {
  if (n < 1 || n > 256) return false;
  const size_t bytes = (size_t)P_FIELDS * n * sizeof(double) + (size_t)10 * n * sizeof(int) + n;
  cudaFuncSetAttribute(oee5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  oee5_kernel<<<(unsigned)batch, ((n + 31) / 32) * 32, bytes, s>>>(diag, upper, rhs, x, n, status, eround, eindex);
  return true;
}

}  // namespace pd

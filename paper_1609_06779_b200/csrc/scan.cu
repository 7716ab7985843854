// The paper's building block 1 on its own: batched block bi-diagonal solves
// by an all-prefix scan of affine elements (scan.hpp:100-168,
// BlockBiDiagSystem<D> with solve_lower_bidiag / solve_upper_bidiag, D = 1..6;
// the dynamics use D = 6):
//   lower: x[0] = rhs[0],   x[k] = coupling[k-1] x[k-1] + rhs[k]
//   upper: x[n-1] = rhs[n-1], x[k] = coupling[k] x[k+1] + rhs[k]
// A warp per system, lane l owning a contiguous chunk of rows (in the
// recursion's order): each lane composes its chunk's affine map (transfer
// matrix, zero-input response), a warp-shuffle Hillis-Steele scan combines the
// 32 chunk maps with compose(first, second) = (C2 C1, C2 o1 + o2)
// (scan.hpp:82-97), and each lane replays its rows from the incoming state.
// Work per row ~ DxD product + two DxD mat-vecs instead of the reference's
// log2(n) dense composes per row.
#include <cstdint>

#include "../../include/pardyn_c.h"

namespace pd {
namespace {

constexpr unsigned kFull = 0xffffffffu;

template <int D>
struct Aff {
  double C[D * D];  // row-major
  double o[D];
};

template <int D>
__device__ __forceinline__ void aff_identity(Aff<D>& a) {
#pragma unroll
  for (int k = 0; k < D * D; ++k) a.C[k] = (k % (D + 1) == 0) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) a.o[k] = 0.0;
}
// r = compose(first, second) = (C2 C1, C2 o1 + o2): `second` applied after `first`
template <int D>
__device__ __forceinline__ void aff_compose(const Aff<D>& first, const Aff<D>& second, Aff<D>& r) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s = fma(second.C[i * D + k], first.C[k * D + j], s);
      r.C[i * D + j] = s;
    }
    double s = second.o[i];
#pragma unroll
    for (int k = 0; k < D; ++k) s = fma(second.C[i * D + k], first.o[k], s);
    r.o[i] = s;
  }
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(128) bidiag_kernel(const double* __restrict__ coupling,
                                                      const double* __restrict__ rhs, double* __restrict__ x,
                                                      int64_t batch, int n, int upper) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= batch) return;  // warp-uniform
  const double* Cg = coupling + (size_t)p * (n > 0 ? n - 1 : 0) * D * D;
  const double* Rg = rhs + (size_t)p * n * D;
  double* Xg = x + (size_t)p * n * D;
  const int chunk = (n + 31) / 32;
  const int k0 = lane * chunk, k1 = min(n, k0 + chunk);
  // step k in recursion order: row(k), coefficient (identity-free first step)
  auto row_of = [&](int k) { return upper ? n - 1 - k : k; };
  auto coeff_of = [&](int k) -> const double* { return Cg + (size_t)(upper ? n - 1 - k : k - 1) * D * D; };
  // 1. chunk map
  Aff<D> agg;
  aff_identity(agg);
  for (int k = k0; k < k1; ++k) {
    const double* r = Rg + (size_t)row_of(k) * D;
    Aff<D> step, t;
    if (k == 0) {
#pragma unroll
      for (int e = 0; e < D * D; ++e) step.C[e] = 0.0;  // x[first] = rhs: nothing flows in
    } else {
      const double* c = coeff_of(k);
#pragma unroll
      for (int e = 0; e < D * D; ++e) step.C[e] = __ldg(c + e);
    }
#pragma unroll
    for (int e = 0; e < D; ++e) step.o[e] = __ldg(r + e);
    aff_compose(agg, step, t);
    agg = t;
  }
  // 2. inclusive warp scan of the chunk maps (lane order = recursion order)
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {
    Aff<D> other, t;
#pragma unroll
    for (int e = 0; e < D * D; ++e) other.C[e] = __shfl_up_sync(kFull, agg.C[e], d);
#pragma unroll
    for (int e = 0; e < D; ++e) other.o[e] = __shfl_up_sync(kFull, agg.o[e], d);
    if (lane >= d) {
      aff_compose(other, agg, t);
      agg = t;
    }
  }
  // 3. state entering the chunk: the previous lane's prefix applied to nothing
  double xin[D];
#pragma unroll
  for (int e = 0; e < D; ++e) {
    const double v = __shfl_up_sync(kFull, agg.o[e], 1);
    xin[e] = lane == 0 ? 0.0 : v;
  }
  // 4. replay the chunk's rows
  for (int k = k0; k < k1; ++k) {
    const double* r = Rg + (size_t)row_of(k) * D;
    double xn[D];
    if (k == 0) {
#pragma unroll
      for (int e = 0; e < D; ++e) xn[e] = __ldg(r + e);
    } else {
      const double* c = coeff_of(k);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = __ldg(r + i);
#pragma unroll
        for (int j = 0; j < D; ++j) s = fma(__ldg(c + i * D + j), xin[j], s);
        xn[i] = s;
      }
    }
    double* xo = Xg + (size_t)row_of(k) * D;
#pragma unroll
    for (int e = 0; e < D; ++e) {
      xo[e] = xn[e];
      xin[e] = xn[e];
    }
  }
}

bool launch_bidiag(int dim, const double* coupling, const double* rhs, double* x, int64_t batch, int n, int upper,
                   cudaStream_t s) {
  const unsigned grid = (unsigned)((batch + 3) / 4);
  switch (dim) {
    case 1: bidiag_kernel<1><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    case 2: bidiag_kernel<2><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    case 3: bidiag_kernel<3><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    case 4: bidiag_kernel<4><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    case 5: bidiag_kernel<5><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    case 6: bidiag_kernel<6><<<grid, 128, 0, s>>>(coupling, rhs, x, batch, n, upper); return true;
    default: return false;
  }
}

void launch_bidiag6(const double* coupling, const double* rhs, double* x, int64_t batch, int n, int upper,
                    cudaStream_t s) {
  launch_bidiag(6, coupling, rhs, x, batch, n, upper, s);
}

}  // namespace pd

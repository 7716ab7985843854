// Device-side synthetic workloads: the reference
// benchmark's chains generated on the GPU, one thread per chain, so a 1M-chain
// model set never exists on the host.
//
//   workload_chains  bench.cpp:357-366 -> random_chain(n, mix(cell ^ (0xC0FFEE + g)))
//   random_chain     model.cpp:157-185 (draw order as GCC 13 evaluates the
//                    reference source, see workload.cpp)
//   std::mt19937_64  the standard's 64-bit Mersenne twister, state per thread
//
// Agreement with the host generator (workload.cpp, pinned to the reference's
// outputs by tests/golden): this file is compiled with --fmad=false so every
// product and sum rounds exactly as the host's SSE2 code does, and sqrt is IEEE
// correctly rounded on both sides, so every draw is bit exact. sin/cos -- the
// only transcendental functions -- are evaluated in double-double arithmetic
// and rounded once (correctly rounded); glibc's sin/cos are not correctly
// rounded in ~0.3% of evaluations (2M-sample check against libquadmath), so
// fields derived through them can differ from the host in the last bit.
#include <cstdint>

#include "../../include/pardyn_c.h"

namespace pd {
namespace wdev {

struct Mt64 {
  uint64_t mt[312];
  int idx;
  __device__ void seed(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    idx = 312;
  }
  __device__ void twist() {
    for (int k = 0; k < 312; ++k) {
      const uint64_t x = (mt[k] & 0xFFFFFFFF80000000ULL) | (mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      mt[k] = mt[(k + 156) % 312] ^ xa;
    }
    idx = 0;
  }
  __device__ uint64_t next() {
    if (idx >= 312) twist();
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
  }
};

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// ---- double-double arithmetic (error-free transforms via FMA) --------------
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}

// sin / cos of x in [0, 2 pi) (the generator's angles), correctly rounded:
// x - k pi/2 with pi/2 in three exact 53-bit parts, Taylor series of the
// reduced argument (|r| <= pi/4) in double-double to ~1e-31, one rounding.
__device__ void cr_sincos(double x, double* s_out, double* c_out) {
  const double p1 = 1.5707963267948966192e+00, p2 = 6.1232339957367658e-17, p3 = -1.4973849048591698e-33;
  const double k = rint(x * 0.63661977236758134308);
  // r = x - k p1 - k p2 - k p3, exactly for k * p1 (k small, p1 53 bits) in dd
  dd r = two_prod(-k, p1);
  r = dd_add({x, 0.0}, r);
  r = dd_add(r, two_prod(-k, p2));
  r = dd_add(r, {-k * p3, 0.0});
  const dd r2 = dd_mul(r, r);
  // sin(r) = r (1 - r^2/3! + r^4/5! - ...), cos(r) = 1 - r^2/2! + ...
  dd s = {1.0, 0.0}, c = {1.0, 0.0};
  dd ts = {1.0, 0.0}, tc = {1.0, 0.0};
  for (int j = 1; j <= 14; ++j) {
    // ts *= -r2 / ((2j)(2j+1)), tc *= -r2 / ((2j-1)(2j))
    ts = dd_mul(ts, r2);
    tc = dd_mul(tc, r2);
    const double ds = (double)(2 * j) * (double)(2 * j + 1), dc = (double)(2 * j - 1) * (double)(2 * j);
    // divide by an exactly representable integer in dd
    auto dd_div_d = [](dd a, double b) {
      const double q1 = a.hi / b;
      dd p = two_prod(q1, b);
      const double q2 = ((a.hi - p.hi) - p.lo + a.lo) / b;
      return quick_two_sum(q1, q2);
    };
    ts = dd_div_d(ts, ds);
    tc = dd_div_d(tc, dc);
    ts = {-ts.hi, -ts.lo};
    tc = {-tc.hi, -tc.lo};
    s = dd_add(s, ts);
    c = dd_add(c, tc);
  }
  s = dd_mul(s, r);
  const int q = (int)(((long long)k) & 3);
  dd sv = (q & 1) ? c : s, cv = (q & 1) ? s : c;
  if (q & 2) sv = {-sv.hi, -sv.lo};
  if ((q + 1) & 2) cv = {-cv.hi, -cv.lo};
  *s_out = sv.hi + sv.lo;
  *c_out = cv.hi + cv.lo;
}

struct Draw {
  Mt64 e;
  __device__ double u() { return (double)(e.next() >> 11) * 0x1.0p-53; }
  __device__ double u(double lo, double hi) { return lo + (hi - lo) * u(); }
  __device__ void unit(double out[3]) {
    const double z = u(-1.0, 1.0);
    const double phi = u(0.0, 2.0 * 3.14159265358979323846);
    const double r = sqrt(fmax(0.0, 1.0 - z * z));
    double sp, cp;
    cr_sincos(phi, &sp, &cp);
    out[0] = r * cp;
    out[1] = r * sp;
    out[2] = z;
  }
  __device__ void rot(double R[9]) {
    const double u1 = u();
    const double a2 = u(0.0, 2.0 * 3.14159265358979323846);
    const double a3 = u(0.0, 2.0 * 3.14159265358979323846);
    const double s1 = sqrt(1.0 - u1), s2 = sqrt(u1);
    double s_a2, c_a2, s_a3, c_a3;
    cr_sincos(a2, &s_a2, &c_a2);
    cr_sincos(a3, &s_a3, &c_a3);
    const double w = s2 * c_a3, x = s1 * s_a2, y = s1 * c_a2, z = s2 * s_a3;
    const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
    const double twx = tx * w, twy = ty * w, twz = tz * w;
    const double txx = tx * x, txy = ty * x, txz = tz * x;
    const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    R[0] = 1 - (tyy + tzz); R[1] = txy - twz;       R[2] = txz + twy;
    R[3] = txy + twz;       R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
    R[6] = txz - twy;       R[7] = tyz + twx;       R[8] = 1 - (txx + tyy);
  }
};

// one thread per chain g of [g0, g0 + count): links[g][i][31]
__global__ void __launch_bounds__(128) workload_chains_kernel(uint64_t cell, int n, int64_t g0, int64_t count,
                                                              double* __restrict__ links) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= count) return;
  Draw d;
  d.e.seed(mix(cell ^ (0xC0FFEEULL + (uint64_t)(g0 + g))));
  double* out = links + (size_t)g * n * PD_LINK_FIELDS;
  for (int i = 0; i < n; ++i) {
    double* f = out + (size_t)i * PD_LINK_FIELDS;
    f[0] = d.u(0.1, 10.0);
    const double cz = d.u(-0.3, 0.3), cy = d.u(-0.3, 0.3), cx = d.u(-0.3, 0.3);
    f[1] = cx;
    f[2] = cy;
    f[3] = cz;
    double A[9];
    d.rot(A);
    const double mz = d.u(0.1, 1.0), my = d.u(0.1, 1.0), mx = d.u(0.1, 1.0);
    const double m[3] = {mx, my, mz};
    double I[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += (A[3 * r + k] * m[k]) * A[3 * c + k];
        I[3 * r + c] = s;
      }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) f[4 + 3 * r + c] = 0.5 * (I[3 * r + c] + I[3 * c + r]);
    double s[3];
    d.unit(s);
    f[13] = s[0];
    f[14] = s[1];
    f[15] = s[2];
    f[16] = f[17] = f[18] = 0.0;
    d.rot(f + 19);
    double dir[3];
    d.unit(dir);
    const double mag = d.u(0.1, 1.0);
    for (int k = 0; k < 3; ++k) f[28 + k] = mag * dir[k];
  }
}

// spatial_inertia_from's rules per model (spatial.cpp:72-87) on the device,
// the same arithmetic as capi.cu's host link_rule (no FMA contraction here or
// there, IEEE sqrt / division): mstatus = PD_SLOT_BAD_MODEL + the first failing
// link's rule, else PD_SLOT_OK.
__device__ double sym3_min_eig(double m[3][3]) {
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = m[0][1] * m[0][1] + m[0][2] * m[0][2] + m[1][2] * m[1][2];
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (m[p][q] == 0.0) continue;
        const double th = (m[q][q] - m[p][p]) / (2.0 * m[p][q]);
        const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        for (int k = 0; k < 3; ++k) {
          const double a = m[k][p], b = m[k][q];
          m[k][p] = c * a - s * b;
          m[k][q] = s * a + c * b;
        }
        for (int k = 0; k < 3; ++k) {
          const double a = m[p][k], b = m[q][k];
          m[p][k] = c * a - s * b;
          m[q][k] = s * a + c * b;
        }
      }
  }
  return fmin(m[0][0], fmin(m[1][1], m[2][2]));
}

__device__ int link_rule(const double* r) {
  const double mass = r[0];
  if (!(mass > 0.0) || !isfinite(mass)) return PD_RULE_MASS;
  for (int k = 1; k < 13; ++k)
    if (!isfinite(r[k])) return PD_RULE_FINITE;
  double scale = 0.0, asym = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      scale = fmax(scale, fabs(r[4 + 3 * a + b]));
      asym = fmax(asym, fabs(r[4 + 3 * a + b] - r[4 + 3 * b + a]));
    }
  if (asym > 1e-9 * fmax(scale, 1.0)) return PD_RULE_SYMMETRIC;
  double m[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) m[a][b] = r[4 + 3 * a + b];
  if (!(sym3_min_eig(m) > 0.0)) return PD_RULE_PD;
  return 0;
}

// One thread per (model, link): every link runs spatial_inertia_from's rules
// at once; the first failing link of a model wins through an atomicMin on
// key = link * 8 + rule (the reference validates links in order and throws at
// the first bad one, model.cpp:148-155).
__global__ void validate_links_kernel(const double* __restrict__ raw, int n, int64_t M, int32_t* __restrict__ key) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * n) return;
  const int r = link_rule(raw + (size_t)t * PD_LINK_FIELDS);
  if (r) {
    const int64_t m = t / n;
    atomicMin(key + m, (int32_t)((t - m * n) * 8 + r));
  }
}

__global__ void finish_validation_kernel(int64_t M, int32_t* __restrict__ status, int32_t* __restrict__ rule) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int32_t k = rule[m];  // 0x7f7f7f7f: no failing link
  const bool bad = k != 0x7f7f7f7f;
  status[m] = bad ? PD_SLOT_BAD_MODEL : PD_SLOT_OK;
  rule[m] = bad ? (k & 7) : 0;
}

}  // namespace wdev

void launch_validate_models(const double* raw, int n, int64_t M, int32_t* status, int32_t* rule, cudaStream_t s) {
  cudaMemsetAsync(rule, 0x7f, sizeof(int32_t) * M, s);
  wdev::validate_links_kernel<<<(unsigned)((M * n + 127) / 128), 128, 0, s>>>(raw, n, M, rule);
  wdev::finish_validation_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(M, status, rule);
}

void launch_workload_chains(uint64_t cell, int n, int64_t g0, int64_t count, double* d_links, cudaStream_t s) {
  wdev::workload_chains_kernel<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(cell, n, g0, count, d_links);
}

}  // namespace pd

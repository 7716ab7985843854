// Accuracy of rsqrt.approx.ftz.f64 with 1 / 2 Newton steps, and with one
// third-order step y (1 + e/2 + 3e^2/8), vs CUDA rsqrt (and 1/sqrt); and of
// rcp.approx.ftz.f64 with two Newton steps vs one second-order step r (1 + e + e^2).
#include <cstdio>
#include <cmath>
__device__ double rsa(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(double* out) {
  double m0 = 0, m1 = 0, m2 = 0, mc = 0, m3 = 0, r2 = 0, r3 = 0;
  for (int t = 0; t < 100000; ++t) {
    double x = exp((t * 0.000731 + threadIdx.x * 0.37) - 30.0) * (1.0 + 0.123 * sin(t * 1.0));
    double q = 1.0 / sqrt(x), y = rsa(x);
    {
      const double e3 = fma(-x, y * y, 1.0);
      const double y3 = fma(y, fma(0.375, e3, 0.5) * e3, y);
      m3 = fmax(m3, fabs(y3 - q) / q);
      const double rq = 1.0 / x;
      double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
      double er = fma(-x, r, 1.0), ra = fma(r, er, r); er = fma(-x, ra, 1.0); ra = fma(ra, er, ra);
      r2 = fmax(r2, fabs(ra - rq) / rq);
      er = fma(-x, r, 1.0);
      const double rb = fma(r, fma(er, er, er), r);
      r3 = fmax(r3, fabs(rb - rq) / rq);
    }
    m0 = fmax(m0, fabs(y - q) / q);
    double e = fma(-x, y * y, 1.0); y = fma(0.5 * y, e, y);
    m1 = fmax(m1, fabs(y - q) / q);
    e = fma(-x, y * y, 1.0); y = fma(0.5 * y, e, y);
    m2 = fmax(m2, fabs(y - q) / q);
    mc = fmax(mc, fabs(rsqrt(x) - q) / q);
  }
  out[threadIdx.x * 8] = m0; out[threadIdx.x * 8 + 1] = m1; out[threadIdx.x * 8 + 2] = m2; out[threadIdx.x * 8 + 3] = mc;
  out[threadIdx.x * 8 + 4] = m3; out[threadIdx.x * 8 + 5] = r2; out[threadIdx.x * 8 + 6] = r3;
}
int main() {
  double* d; cudaMalloc(&d, 32 * 8 * 8); k<<<1, 32>>>(d); double h[256]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double a = 0, b = 0, c = 0, e = 0, f = 0, g = 0, hh = 0;
  for (int i = 0; i < 32; ++i) {
    a = fmax(a, h[8*i]); b = fmax(b, h[8*i+1]); c = fmax(c, h[8*i+2]); e = fmax(e, h[8*i+3]);
    f = fmax(f, h[8*i+4]); g = fmax(g, h[8*i+5]); hh = fmax(hh, h[8*i+6]);
  }
  printf("rsqrt.approx rel err %.3e, +1 NR %.3e, +2 NR %.3e, one 3rd-order step %.3e (CUDA rsqrt %.3e) vs 1/sqrt\n", a, b, c, f, e);
  printf("rcp.approx + 2 NR %.3e, one 2nd-order step %.3e vs 1/x\n", g, hh);
  return 0;
}

// Accuracy of rsqrt.approx.ftz.f64 with 1 / 2 Newton steps vs CUDA rsqrt (and 1/sqrt).
#include <cstdio>
#include <cmath>
__device__ double rsa(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(double* out) {
  double m0 = 0, m1 = 0, m2 = 0, mc = 0;
  for (int t = 0; t < 100000; ++t) {
    double x = exp((t * 0.000731 + threadIdx.x * 0.37) - 30.0) * (1.0 + 0.123 * sin(t * 1.0));
    double q = 1.0 / sqrt(x), y = rsa(x);
    m0 = fmax(m0, fabs(y - q) / q);
    double e = fma(-x, y * y, 1.0); y = fma(0.5 * y, e, y);
    m1 = fmax(m1, fabs(y - q) / q);
    e = fma(-x, y * y, 1.0); y = fma(0.5 * y, e, y);
    m2 = fmax(m2, fabs(y - q) / q);
    mc = fmax(mc, fabs(rsqrt(x) - q) / q);
  }
  out[threadIdx.x * 4] = m0; out[threadIdx.x * 4 + 1] = m1; out[threadIdx.x * 4 + 2] = m2; out[threadIdx.x * 4 + 3] = mc;
}
int main() {
  double* d; cudaMalloc(&d, 32 * 4 * 8); k<<<1, 32>>>(d); double h[128]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double a = 0, b = 0, c = 0, e = 0;
  for (int i = 0; i < 32; ++i) { a = fmax(a, h[4*i]); b = fmax(b, h[4*i+1]); c = fmax(c, h[4*i+2]); e = fmax(e, h[4*i+3]); }
  printf("rsqrt.approx rel err %.3e, +1 NR %.3e, +2 NR %.3e (CUDA rsqrt %.3e) vs 1/sqrt\n", a, b, c, e); return 0;
}

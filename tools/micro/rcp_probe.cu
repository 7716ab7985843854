// Accuracy of rcp.approx.ftz.f64 alone and with 1 / 2 Newton steps vs 1.0 / x.
#include <cstdio>
#include <cmath>
__device__ double rcpa(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(double* out) {
  double m0 = 0, m1 = 0, m2 = 0;
  for (int t = 0; t < 100000; ++t) {
    double x = exp((t * 0.000731 + threadIdx.x * 0.37) - 30.0) * (1.0 + 0.123 * sin(t * 1.0));
    double r = rcpa(x), q = 1.0 / x;
    m0 = fmax(m0, fabs(r - q) / q);
    double e = fma(-x, r, 1.0); r = fma(r, e, r);
    m1 = fmax(m1, fabs(r - q) / q);
    e = fma(-x, r, 1.0); r = fma(r, e, r);
    m2 = fmax(m2, fabs(r - q) / q);
  }
  out[threadIdx.x * 3] = m0; out[threadIdx.x * 3 + 1] = m1; out[threadIdx.x * 3 + 2] = m2;
}
int main() {
  double* d; cudaMalloc(&d, 32 * 3 * 8); k<<<1, 32>>>(d); double h[96]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double a = 0, b = 0, c = 0; for (int i = 0; i < 32; ++i) { a = fmax(a, h[3*i]); b = fmax(b, h[3*i+1]); c = fmax(c, h[3*i+2]); }
  printf("rcp.approx rel err %.3e, +1 NR %.3e, +2 NR %.3e\n", a, b, c); return 0;
}

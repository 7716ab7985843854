// Single-thread dependent-chain latencies on the device (clock64 cycles per op):
// DFMA, DADD, DMUL, double division, rcp-based 1/x, sqrt, shared-memory load.
#include <cstdio>
__global__ void probe(double* out, double x0, int iters) {
  __shared__ double sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = 0.0;
  __syncthreads();
  if (threadIdx.x) return;
  double a = x0, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = a + c;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) a = a * b;
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) a = 1.0 / a;
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) a = sqrt(a);
  long long t5 = clock64();
  int idx = (int)a & 0;
  double s = 0;
  for (int i = 0; i < iters; ++i) { s = sm[idx]; idx = (int)s; }
  long long t6 = clock64();
  out[0] = a + s;
  printf("cycles/op: dfma %.1f dadd %.1f dmul %.1f div %.1f sqrt %.1f lds %.1f\n", (t1 - t0) / (double)iters,
         (t2 - t1) / (double)iters, (t3 - t2) / (double)iters, (t4 - t3) / (double)iters, (t5 - t4) / (double)iters,
         (t6 - t5) / (double)iters);
}
int main() {
  double* d;
  cudaMalloc(&d, 8);
  probe<<<1, 32>>>(d, 1.5, 4096);
  cudaDeviceSynchronize();
  probe<<<1, 32>>>(d, 1.5, 4096);
  cudaDeviceSynchronize();
  return 0;
}

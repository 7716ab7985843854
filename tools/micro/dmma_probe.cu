// Microbenchmark: FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) vs DFMA
// throughput and latency on this GPU. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters) {
  double d[CH][2];
  const double a = 1e-3 * threadIdx.x, b = 0.999;
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = c + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = fma(a[c], 0.999999, 1e-9);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  // throughput: many warps
  for (int wps : {4, 8, 16, 32}) {
    float ms = run(k_dmma<4>, sms, 32 * wps, iters, out);
    double fl = 2.0 * 256 * 4 * iters * (double)sms * wps;
    float ms2 = run(k_dfma<8>, sms, 32 * wps, iters, out);
    double fl2 = 2.0 * 8 * iters * (double)sms * 32 * wps;
    printf("warps/SM %2d  DMMA %.2f TF/s   DFMA %.2f TF/s\n", wps, fl / ms / 1e9, fl2 / ms2 / 1e9);
  }
  // latency: one warp per SM, dependent chain
  {
    float ms = run(k_dmma<1>, 1, 32, iters, out);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("DMMA dependent latency ~ %.1f cycles\n", ms * 1e-3 * clk * 1e3 / iters);
    float ms2 = run(k_dfma<1>, 1, 32, iters, out);
    printf("DFMA dependent latency ~ %.1f cycles\n", ms2 * 1e-3 * clk * 1e3 / iters);
    float ms3 = run(k_dfma<2>, 1, 32, iters, out);
    printf("DFMA 2 chains, 1 warp: %.1f cycles/iter\n", ms3 * 1e-3 * clk * 1e3 / iters);
    float ms4 = run(k_dfma<4>, 1, 32, iters, out);
    printf("DFMA 4 chains, 1 warp: %.1f cycles/iter\n", ms4 * 1e-3 * clk * 1e3 / iters);
    float ms5 = run(k_dfma<8>, 1, 128, iters, out);
    printf("DFMA 8 chains, 4 warps: %.1f cycles/iter\n", ms5 * 1e-3 * clk * 1e3 / iters);
  }
  return 0;
}

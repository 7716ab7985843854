// Zero-copy PCIe probe: SM-driven reads of pinned host memory (and writes to
// it) vs cudaMemcpyAsync, at the c2 host-path sizes (48 MiB in, 16 MiB out).
#include <cuda_runtime.h>
#include <cstdio>

__global__ void zc_read(const double2* __restrict__ h, double2* __restrict__ d, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void zc_read4(const double2* __restrict__ h, double2* __restrict__ d, size_t n2) {
  // 4 independent 16-byte loads in flight per thread
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n2) v[k] = h[i + k * stride];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n2) d[i + k * stride] = v[k];
  }
}
__global__ void zc_write(const double2* __restrict__ d, double2* __restrict__ h, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) h[i] = d[i];
}

int main() {
  const size_t in_b = 48ull << 20, out_b = 16ull << 20;
  double2 *hi, *ho, *di, *dout;
  cudaHostAlloc(&hi, in_b, cudaHostAllocDefault);
  cudaHostAlloc(&ho, out_b, cudaHostAllocDefault);
  cudaMalloc(&di, in_b);
  cudaMalloc(&dout, out_b);
  cudaMemset(dout, 0, out_b);
  for (size_t i = 0; i < in_b / 16; ++i) hi[i] = make_double2(i, i);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, size_t bytes, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, s1);
    for (int r = 0; r < 10; ++r) fn();
    cudaEventRecord(b, s1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    printf("%-44s %.3f ms  %.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  timeit("memcpy H2D 48MiB (one copy)", in_b, [&] { cudaMemcpyAsync(di, hi, in_b, cudaMemcpyHostToDevice, s1); });
  timeit("memcpy H2D 24 x 2MiB", in_b, [&] {
    for (int c = 0; c < 24; ++c)
      cudaMemcpyAsync((char*)di + c * (2 << 20), (char*)hi + c * (2 << 20), 2 << 20, cudaMemcpyHostToDevice, s1);
  });
  timeit("memcpy D2H 16MiB", out_b, [&] { cudaMemcpyAsync(ho, dout, out_b, cudaMemcpyDeviceToHost, s1); });
  const int grids[] = {16, 32, 64, 148, 296};
  for (int g : grids) {
    char nm[64];
    snprintf(nm, sizeof nm, "zc read  48MiB grid %d x 256", g);
    timeit(nm, in_b, [&] { zc_read<<<g, 256, 0, s1>>>(hi, di, in_b / 16); });
    snprintf(nm, sizeof nm, "zc read4 48MiB grid %d x 256", g);
    timeit(nm, in_b, [&] { zc_read4<<<g, 256, 0, s1>>>(hi, di, in_b / 16); });
    snprintf(nm, sizeof nm, "zc write 16MiB grid %d x 256", g);
    timeit(nm, out_b, [&] { zc_write<<<g, 256, 0, s1>>>(dout, ho, out_b / 16); });
  }
  cudaEvent_t fork;
  cudaEventCreate(&fork);
  timeit("zc read4(64) + zc write(32) concurrently", in_b + out_b, [&] {
    cudaEventRecord(fork, s1);
    cudaStreamWaitEvent(s2, fork, 0);
    zc_write<<<32, 256, 0, s2>>>(dout, ho, out_b / 16);
    zc_read4<<<64, 256, 0, s1>>>(hi, di, in_b / 16);
    cudaEventRecord(fork, s2);
    cudaStreamWaitEvent(s1, fork, 0);
  });
  timeit("memcpy H2D + memcpy D2H concurrently", in_b + out_b, [&] {
    cudaEventRecord(fork, s1);
    cudaStreamWaitEvent(s2, fork, 0);
    cudaMemcpyAsync(ho, dout, out_b, cudaMemcpyDeviceToHost, s2);
    cudaMemcpyAsync(di, hi, in_b, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(fork, s2);
    cudaStreamWaitEvent(s1, fork, 0);
  });
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

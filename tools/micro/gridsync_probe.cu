// Cost of a cooperative-groups grid barrier on this GPU: one CTA per SM
// (256 threads) running K grid.sync()s, timed with events.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void syncs(int k, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < k; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = k;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d;
  cudaMalloc(&d, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {128, 256, 1024}) {
    for (int k : {1, 1000}) {
      void* args[] = {&k, &d};
      cudaLaunchCooperativeKernel((const void*)syncs, sms, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((const void*)syncs, sms, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d x %d threads, %4d grid.sync: %.3f ms (%.2f us per sync)\n", sms, threads, k, ms, 1000 * ms / k);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

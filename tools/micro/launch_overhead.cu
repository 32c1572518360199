// Launch-overhead probe: event-timed back-to-back launches of a null kernel
// at several dynamic-smem sizes and grid shapes (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void nullk(int* p) { if (p && threadIdx.x == 1234567) p[0] = 1; }
__global__ void spin(int* p, long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0; while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (p && threadIdx.x == 1234567) p[0] = 1;
}
int main() {
  cudaFuncSetAttribute(nullk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {148, 296};
  int smems[] = {0, 96 * 1024, 200 * 1024};
  for (int g : grids) for (int sm : smems) for (int th : {192, 352}) {
    if (sm > 100 * 1024 && g > 148) continue;
    for (int i = 0; i < 10; ++i) nullk<<<g, th, sm>>>(nullptr);
    cudaDeviceSynchronize();
    float tot = 0;
    for (int r = 0; r < 50; ++r) {
      cudaEventRecord(a); nullk<<<g, th, sm>>>(nullptr); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
    }
    cudaEventRecord(a);
    for (int r = 0; r < 200; ++r) nullk<<<g, th, sm>>>(nullptr);
    cudaEventRecord(b); cudaEventSynchronize(b); float ms2; cudaEventElapsedTime(&ms2, a, b);
    cudaEventRecord(a);
    for (int r = 0; r < 200; ++r) spin<<<g, th, sm>>>(nullptr, 20000);
    cudaEventRecord(b); cudaEventSynchronize(b); float ms3; cudaEventElapsedTime(&ms3, a, b);
    printf("grid %d thr %d smem %6d: single %.2f us, b2b null %.2f us/launch, b2b 20us-spin %.2f us/launch\n",
           g, th, sm, tot / 50 * 1e3, ms2 / 200 * 1e3, ms3 / 200 * 1e3);
  }
  return 0;
}

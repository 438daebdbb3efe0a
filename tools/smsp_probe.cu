// Which SM sub-partition (warp scheduler) do the 9 warps of a 288-thread CTA land on, 4 CTAs per SM?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smsp_probe_bin tools/smsp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(288, 4) k(unsigned* out) {
  extern __shared__ unsigned char pad[];
  unsigned smid, warpid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(warpid));
  if ((threadIdx.x & 31) == 0) {
    const unsigned w = threadIdx.x >> 5;
    // out[blockIdx][w] = smid << 8 | warpid
    out[blockIdx.x * 9 + w] = (smid << 8) | warpid;
  }
  // keep the CTAs resident together for a while
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
  if (pad[threadIdx.x] == 77) out[0] = 0;
}
int main() {
  const int grid = 592;
  unsigned* d;
  cudaMalloc(&d, grid * 9 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 33000);
  k<<<grid, 288, 33000>>>(d);
  cudaDeviceSynchronize();
  static unsigned h[592 * 9];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int hist[4] = {0, 0, 0, 0}, all[4] = {0, 0, 0, 0};
  for (int b = 0; b < grid; b++)
    for (int w = 0; w < 9; w++) {
      all[h[b * 9 + w] & 3]++;
      if (w == 8) hist[h[b * 9 + w] & 3]++;
    }
  printf("service warp (warp 8) scheduler (warpid & 3) histogram: %d %d %d %d\n", hist[0], hist[1], hist[2], hist[3]);
  printf("all warps: %d %d %d %d\n", all[0], all[1], all[2], all[3]);
  for (int b = 0; b < 8; b++) {
    printf("block %d sm %u warpids:", b, h[b * 9] >> 8);
    for (int w = 0; w < 9; w++) printf(" %u", h[b * 9 + w] & 0xFF);
    printf("\n");
  }
  // per SM: how many service warps per scheduler
  int worst = 0;
  for (unsigned sm = 0; sm < 148; sm++) {
    int c[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; b++)
      if ((h[b * 9 + 8] >> 8) == sm) c[h[b * 9 + 8] & 3]++;
    int m = c[0];
    for (int i = 1; i < 4; i++) m = m > c[i] ? m : c[i];
    worst = worst > m ? worst : m;
    if (sm < 4) printf("sm %u service warps per scheduler: %d %d %d %d\n", sm, c[0], c[1], c[2], c[3]);
  }
  printf("max service warps on one scheduler of an SM: %d\n", worst);
  return 0;
}

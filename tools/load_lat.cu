// load_lat.cu -- loaded latency of a warp's 2 KiB row load (4 x LDG.128 per
// lane) with the transcode kernels' lane layout (64-byte lane stride) versus a
// coalesced layout (512-byte contiguous per instruction), while 4 CTAs per SM
// stream 1 GiB with some ALU work per row (perf helper; not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/load_lat_bin tools/load_lat.cu
#include <cstdio>
#include <cstdint>

template <int MODE, bool SYNC>
__global__ void __launch_bounds__(256, 4) kern(const uint8_t* buf, size_t rows, int work,
                                               unsigned long long* acc) {
  const unsigned lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  unsigned long long lat = 0, cnt = 0;
  uint32_t sink = 0;
  const size_t iters = (rows + nw - 1) / nw;
  for (size_t it = 0; it < iters; it++) {
    const size_t r = gw + it * nw;
    if (SYNC) __syncthreads();  // all warps of the CTA load together (as after a barrier)
    if (r >= rows) continue;
    const uint8_t* row = buf + r * 2048;
    const long long t0 = clock64();
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const size_t off = MODE == 0 ? 64 * lane + 16 * k : 512 * k + 16 * lane;
      v[k] = __ldg(reinterpret_cast<const uint4*>(row + off));
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) x ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    if (x == 0x12345678u) sink++;
    const long long t1 = clock64();
    lat += t1 - t0;
    cnt++;
    // stand-in for the per-row ALU work
    for (int i = 0; i < work; i++) x = __funnelshift_l(x, x ^ i, 7) + 0x9E3779B9u;
    sink ^= x;
  }
  if (lane == 0) {
    atomicAdd(&acc[0], lat);
    atomicAdd(&acc[1], cnt);
  }
  if (sink == 0xFFFFFFFFu) acc[2] = sink;
}

int main() {
  const size_t bytes = 1ull << 30, rows = bytes / 2048;
  uint8_t* buf;
  unsigned long long* acc;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaMalloc(&acc, 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int work : {0, 200, 400}) {
    for (int mode = 0; mode < 3; mode++) {
      for (int rep = 0; rep < 3; rep++) {
        cudaMemset(acc, 0, 24);
        cudaEventRecord(e0);
        if (mode == 0) kern<0, false><<<148 * 4, 256>>>(buf, rows, work, acc);
        else if (mode == 1) kern<1, false><<<148 * 4, 256>>>(buf, rows, work, acc);
        else kern<0, true><<<148 * 4, 256>>>(buf, rows, work, acc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[2];
        cudaMemcpy(h, acc, 16, cudaMemcpyDeviceToHost);
        if (rep == 2)
          printf("work %3d %-10s: %.3f ms (%.0f GB/s), load latency %.0f cycles\n", work,
                 mode == 0 ? "lane64" : mode == 1 ? "coalesced" : "lane64+sync", ms, bytes / ms / 1e6, (double)h[0] / h[1]);
      }
    }
  }
  return 0;
}

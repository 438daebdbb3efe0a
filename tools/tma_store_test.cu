// tma_store_test.cu -- does a 1D TMA tensor store accept element coordinates
// that are not 16-byte aligned (UINT16 and UINT8 elements)?  (probe; not part
// of the library)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_store_test_bin tools/tma_store_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void store_box(const __grid_constant__ CUtensorMap tm, int coord, int elem_bytes) {
  __shared__ __align__(128) uint8_t buf[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) buf[i] = (uint8_t)(i * 7 + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
                 "r"(coord), "r"(0), "r"(s)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  (void)elem_bytes;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  int fails = 0;
  for (int eb : {2, 1}) {
    for (int coord : {0, 1, 3, 5, 8, 13}) {
      const size_t n = 4096;
      uint8_t* d;
      cudaMalloc(&d, n);
      cudaMemset(d, 0xEE, n);
      CUtensorMap tm;
      cuuint64_t dim[2] = {n / eb, 1}, str[1] = {n};
      cuuint32_t box[2] = {256, 1}, es[2] = {1, 1};
      CUresult r = enc(&tm, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d,
                       dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d (eb %d)\n", (int)r, eb); return 1; }
      store_box<<<1, 128>>>(tm, coord, eb);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint8_t> h(n);
      cudaMemcpy(h.data(), d, n, cudaMemcpyDeviceToHost);
      int bad = 0;
      const int start = coord * eb, len = 256 * eb;
      for (int i = 0; i < (int)n; i++) {
        const uint8_t want = (i >= start && i < start + len) ? (uint8_t)((i - start) * 7 + 1) : 0xEE;
        if (h[i] != want) bad++;
      }
      printf("elem %d B, coord %2d: %s (%d bad bytes, err %s)\n", eb, coord, bad ? "FAIL" : "ok", bad,
             cudaGetErrorString(e));
      fails += bad != 0;
      cudaFree(d);
    }
  }
  return fails ? 1 : 0;
}

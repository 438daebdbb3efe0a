// k_datagen.cu -- device-side generation of the BASELINE.json workloads
// (vt_gen.cuh): one thread per chunk, two passes (sizes, then placement at
// the exclusive scan of the sizes).  Generating in HBM avoids pushing 1-32 GiB
// over PCIe for every benchmark run.
#include "vt_gen.cuh"
#include "vt_kernels.h"

namespace vt {

__global__ void gen_sizes_kernel(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                                 uint64_t* sizes) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nchunks) return;
  CountSink s;
  gen_chunk(cfg, seed, chunk0 + i, s);
  sizes[i] = s.n;
}

template <class T>
__global__ void gen_write_kernel(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                                 const uint64_t* offsets, uint64_t limit, T* out,
                                 unsigned long long* end) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nchunks) return;
  const uint64_t start = offsets[i];
  if (start > limit) return;
  WriteSink<T> w{out, start, limit};
  gen_chunk(cfg, seed, chunk0 + i, w);
  atomicMax(&end[0], (unsigned long long)w.off);
  if (w.first_bad != ~0ull) atomicMin(&end[1], (unsigned long long)w.first_bad);
}

int launch_gen_sizes(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks, uint64_t* sizes,
                     cudaStream_t s) {
  if (nchunks == 0) return 0;
  gen_sizes_kernel<<<(unsigned)((nchunks + 127) / 128), 128, 0, s>>>(cfg, seed, chunk0, nchunks,
                                                                     sizes);
  return (int)cudaGetLastError();
}

int launch_gen_write(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                     const uint64_t* offsets, uint64_t limit, void* out, uint64_t* end_pos,
                     cudaStream_t s) {
  unsigned long long init[2] = {0ull, ~0ull};
  int rc = (int)cudaMemcpyAsync(end_pos, init, sizeof init, cudaMemcpyHostToDevice, s);
  if (rc) return rc;
  // the host copy source must stay valid until the copy ran
  rc = (int)cudaStreamSynchronize(s);
  if (rc) return rc;
  if (nchunks == 0) return 0;
  const unsigned blocks = (unsigned)((nchunks + 127) / 128);
  auto* e = reinterpret_cast<unsigned long long*>(end_pos);
  if (cfg == 3)
    gen_write_kernel<uint16_t><<<blocks, 128, 0, s>>>(cfg, seed, chunk0, nchunks, offsets, limit,
                                                      static_cast<uint16_t*>(out), e);
  else
    gen_write_kernel<uint8_t><<<blocks, 128, 0, s>>>(cfg, seed, chunk0, nchunks, offsets, limit,
                                                     static_cast<uint8_t*>(out), e);
  return (int)cudaGetLastError();
}

}  // namespace vt

extern "C" uint64_t vt_gen_chunk_draws(int) { return vt::kDraws; }

// Host-side generation of one chunk (tests of the generator's determinism and
// class mix run on the CPU).  Returns the chunk size; writes at most `cap`
// elements (bytes, or units for cfg 3) to `out`.
extern "C" uint64_t vt_gen_host_chunk(int cfg, uint64_t seed, uint64_t chunk, void* out,
                                      uint64_t cap, uint64_t* first_bad) {
  if (cfg == 3) {
    vt::WriteSink<uint16_t> w{static_cast<uint16_t*>(out), 0, cap};
    vt::gen_chunk(cfg, seed, chunk, w);
    if (first_bad) *first_bad = w.first_bad;
    return w.off;
  }
  vt::WriteSink<uint8_t> w{static_cast<uint8_t*>(out), 0, cap};
  vt::gen_chunk(cfg, seed, chunk, w);
  if (first_bad) *first_bad = w.first_bad;
  return w.off;
}

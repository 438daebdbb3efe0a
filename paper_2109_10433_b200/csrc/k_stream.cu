// k_stream.cu -- streaming UTF-8 validation and character-class counts
// (SURVEY.md 8(f) row 4).
//
// The reference's Utf8BlockValidator (proj/include/vtrans/validation.hpp:15-24)
// carries the SIMD checker state across 64-byte blocks; on the GPU a fed chunk
// is validated by the whole-buffer kernel, and only the seams need state: the
// incomplete sequence the previous chunks ended with (<= 3 bytes).  One thread
// completes that carried sequence from the head of the new chunk (seam), the
// validate kernel scans the rest (skipping the bytes the seam consumed), and one
// thread turns a first error that is only "cut by the chunk end" into the new
// carry (tail).  The first error index therefore equals rule A on the
// concatenated stream, which is what whole-buffer
// validation reports.
#include "vt_device.cuh"
#include "vt_kernels.h"

#include <algorithm>

namespace vt {

__device__ __forceinline__ unsigned seq_len(unsigned b) {
  return b < 0x80u ? 1u : b < 0xC2u ? 0u : b < 0xE0u ? 2u : b < 0xF0u ? 3u : b < 0xF5u ? 4u : 0u;
}

// Second byte ranges of proj/src/codec_core.cpp:5-38 (overlong E0/F0,
// surrogates ED, > U+10FFFF F4); later bytes only need to be continuations.
__device__ __forceinline__ bool second_ok(unsigned lead, unsigned b) {
  if ((b & 0xC0u) != 0x80u) return false;
  if (lead == 0xE0u) return b >= 0xA0u;
  if (lead == 0xEDu) return b < 0xA0u;
  if (lead == 0xF0u) return b >= 0x90u;
  if (lead == 0xF4u) return b < 0x90u;
  return true;
}

__global__ void stream_seam_kernel(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n) {
  if (st->error_at >= 0) {  // already failed: nothing more to check
    st->skip = kSkipAll;
    return;
  }
  const unsigned L = st->carry_len;
  if (L == 0) {
    st->skip = 0;
    return;
  }
  const unsigned lead = st->carry[0], len = seq_len(lead);
  const unsigned need = len - L;
  const unsigned m = n < need ? (unsigned)n : need;
  for (unsigned i = 0; i < m; i++) {
    const unsigned b = chunk[i];
    const bool ok = L + i == 1 ? second_ok(lead, b) : (b & 0xC0u) == 0x80u;
    if (!ok) {
      st->error_at = (long long)(st->fed - L);  // rule A: the lead fails
      st->skip = kSkipAll;
      return;
    }
  }
  if (m < need) {  // still incomplete: the whole chunk extends the carry
    for (unsigned i = 0; i < m; i++) st->carry[L + i] = chunk[i];
    st->carry_len = L + m;
    st->skip = m;
    return;
  }
  uint32_t v = 0;
  for (unsigned i = 0; i < 4; i++) {
    const unsigned b = i < L ? st->carry[i] : i < len ? chunk[i - L] : 0u;
    v |= b << (8 * i);
  }
  if (!decode_ok(v)) st->error_at = (long long)(st->fed - L);
  st->carry_len = 0;
  st->skip = need;
}

// res: the validate kernel's result over chunk[skip, n).
__global__ void stream_tail_kernel(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n,
                                   const vt_result* res) {
  const uint64_t fed = st->fed;
  st->fed = fed + n;
  if (st->error_at >= 0 || res->error_at < 0) return;
  const uint64_t p = (uint64_t)st->skip + (uint64_t)res->error_at;
  const unsigned b0 = chunk[p], len = seq_len(b0);
  // only cut by the end of the chunk: a lead with a valid beginning
  bool cut = len >= 2 && p + len > n;
  for (uint64_t i = p + 1; cut && i < n; i++)
    cut = i == p + 1 ? second_ok(b0, chunk[i]) : (chunk[i] & 0xC0u) == 0x80u;
  if (cut) {
    const unsigned k = (unsigned)(n - p);
    for (unsigned i = 0; i < k; i++) st->carry[i] = chunk[p + i];
    st->carry_len = k;
  } else {
    st->error_at = (long long)(fed + p);
  }
}

int launch_stream_seam(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n, cudaStream_t s) {
  stream_seam_kernel<<<1, 1, 0, s>>>(st, chunk, n);
  return (int)cudaGetLastError();
}

int launch_stream_tail(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n, const vt_result* res,
                       cudaStream_t s) {
  stream_tail_kernel<<<1, 1, 0, s>>>(st, chunk, n, res);
  return (int)cudaGetLastError();
}

// ---- character classes ---------------------------------------------------------
// Non-continuation bytes by lead class: < 0x80, C0..DF, E0..EF, F0..F7 (valid
// input only, so each lead starts exactly one character).  16 bytes per
// thread per step with SWAR plane counts; one atomic per warp per class.
__global__ void utf8_class_count_kernel(const uint8_t* d, uint64_t n, unsigned long long* counts) {
  const uint64_t nvec = n / 16;
  const uint4* v = reinterpret_cast<const uint4*>(d);
  unsigned long long c1 = 0, c2 = 0, c3 = 0, c4 = 0;
  auto word = [&](uint32_t x) {
    const uint32_t H = 0x80808080u;
    const uint32_t x2 = x << 1;
    const uint32_t ascii = ~x & H, l2 = x & x2 & H;
    const uint32_t l3 = l2 & (x << 2), l4 = l3 & (x << 3);
    c1 += __popc(ascii);
    c2 += __popc(l2 & ~l3);
    c3 += __popc(l3 & ~l4);
    c4 += __popc(l4);
  };
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q = __ldg(v + i);
    word(q.x); word(q.y); word(q.z); word(q.w);
  }
  // tail bytes (n % 16), first thread only
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t i = nvec * 16; i < n; i++) {
      const unsigned b = d[i];
      if (b < 0x80u) c1++;
      else if (b >= 0xF0u) c4++;
      else if (b >= 0xE0u) c3++;
      else if (b >= 0xC0u) c2++;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    c3 += __shfl_xor_sync(0xffffffffu, c3, o);
    c4 += __shfl_xor_sync(0xffffffffu, c4, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (c1) atomicAdd(&counts[0], c1);
    if (c2) atomicAdd(&counts[1], c2);
    if (c3) atomicAdd(&counts[2], c3);
    if (c4) atomicAdd(&counts[3], c4);
  }
}

int launch_utf8_class_counts(const uint8_t* d, uint64_t n, unsigned long long* counts,
                             cudaStream_t s) {
  if (n == 0) return 0;
  if ((uintptr_t)d & 15) return (int)cudaErrorInvalidValue;  // callers pass cudaMalloc buffers
  const uint64_t nvec = n / 16;
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nvec + 255) / 256, 148 * 8));
  utf8_class_count_kernel<<<blocks, 256, 0, s>>>(d, n, counts);
  return (int)cudaGetLastError();
}

}  // namespace vt

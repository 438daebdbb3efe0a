// k_batch.cu -- many-short-strings validation on sm_100a.
//
// The reference is called millions of times on tiny inputs by its fuzzer and
// exhaustive suites (proj/src/harness.cpp:388-436, proj/tests/acceptance.cpp:
// 138-204).  A per-call kernel launch would be latency-bound, so these
// entry points validate a whole batch of strings in one launch: one thread per
// string walks it with the decode rules of proj/src/codec_core.cpp:5-38 and
// reports the first failing index.
#include "vt_device.cuh"
#include "vt_kernels.h"

#include <algorithm>

namespace vt {

// First error index of bytes [p, p+n), or -1.
__device__ __forceinline__ long long first_error_seq(const uint8_t* p, unsigned long long n) {
  unsigned long long i = 0;
  while (i < n) {
    const unsigned b0 = p[i];
    if (b0 < 0x80u) {
      i++;
      continue;
    }
    unsigned len, cp, lo;
    if ((b0 & 0xE0u) == 0xC0u) {
      len = 2; cp = b0 & 0x1Fu; lo = 0x80u;
    } else if ((b0 & 0xF0u) == 0xE0u) {
      len = 3; cp = b0 & 0x0Fu; lo = 0x800u;
    } else if ((b0 & 0xF8u) == 0xF0u) {
      len = 4; cp = b0 & 0x07u; lo = 0x10000u;
    } else {
      return (long long)i;
    }
    if (i + len > n) return (long long)i;
    for (unsigned k = 1; k < len; k++) {
      const unsigned c = p[i + k];
      if ((c & 0xC0u) != 0x80u) return (long long)i;
      cp = (cp << 6) | (c & 0x3Fu);
    }
    if (cp < lo || cp > 0x10FFFFu || (cp >= 0xD800u && cp <= 0xDFFFu)) return (long long)i;
    i += len;
  }
  return -1;
}

__global__ void batch_validate_kernel(const uint8_t* data, const uint64_t* offsets,
                                      uint64_t count, int64_t* first_err) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t s = offsets[i], e = offsets[i + 1];
  first_err[i] = first_error_seq(data + s, e - s);
}

// ---- batched transcoding (one thread per string) ------------------------------
// The reference's fuzz and exhaustive drivers transcode millions of short
// strings one call at a time (proj/src/harness.cpp:357-375, 388-436); here a
// whole batch is one launch.  String i = data[off[i], off[i+1]); its output
// goes to the same offsets in units (UTF-8 -> UTF-16: capacity = its byte
// length) or to 3*off[i] in bytes (UTF-16 -> UTF-8: capacity 3 per unit), so
// no scan is needed; res[i] = its TranscodeResult.  The decode follows
// proj/src/codec_core.cpp:5-125 character by character, stopping at the first
// invalid one (validate), or without checks (validate = 0: the reference's
// validate=false, same result on valid input, bounded output otherwise).
__global__ void batch_u8to16_kernel(const uint8_t* data, const uint64_t* off, uint64_t count,
                                    uint16_t* out, vt_result* res, int validate) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const uint64_t b = off[s], n = off[s + 1] - b;
  const uint8_t* p = data + b;
  uint16_t* o = out + b;
  uint64_t i = 0, q = 0;
  long long err = -1;
  while (i < n) {
    const unsigned b0 = p[i];
    if (b0 < 0x80u) {
      o[q++] = (uint16_t)b0;
      i++;
      continue;
    }
    unsigned len = (b0 & 0xE0u) == 0xC0u ? 2u : (b0 & 0xF0u) == 0xE0u ? 3u : (b0 & 0xF8u) == 0xF0u ? 4u : 0u;
    if (validate) {
      if (len == 0 || first_error_seq(p + i, min((uint64_t)len, n - i)) == 0 || i + len > n) {
        err = (long long)i;
        break;
      }
    } else {
      // no checks: a malformed lead or a cut sequence decodes as far as the
      // input goes (each unit still consumes at least one byte)
      if (len == 0) len = 1;
      if (i + len > n) len = (unsigned)(n - i);
    }
    uint32_t cp = len == 1 ? b0 : b0 & (0x7Fu >> len);
    for (unsigned k = 1; k < len; k++) cp = (cp << 6) | (p[i + k] & 0x3Fu);
    if (cp >= 0x10000u && len == 4) {
      cp -= 0x10000u;
      o[q++] = (uint16_t)(0xD800u + (cp >> 10));
      o[q++] = (uint16_t)(0xDC00u + (cp & 0x3FFu));
    } else {
      o[q++] = (uint16_t)cp;
    }
    i += len;
  }
  vt_result r;
  r.written = q;
  r.consumed = err < 0 ? n : (uint64_t)err;
  r.error_at = err;
  res[s] = r;
}

__global__ void batch_u16to8_kernel(const uint16_t* data, const uint64_t* off, uint64_t count,
                                    uint8_t* out, vt_result* res) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const uint64_t b = off[s], n = off[s + 1] - b;
  const uint16_t* p = data + b;
  uint8_t* o = out + 3 * b;
  uint64_t i = 0, q = 0;
  long long err = -1;
  while (i < n) {
    uint32_t cp = p[i];
    unsigned len = 1;
    if ((cp & 0xF800u) == 0xD800u) {  // surrogate: a high one followed by a low one
      if (cp >= 0xDC00u || i + 1 >= n || (p[i + 1] & 0xFC00u) != 0xDC00u) {
        err = (long long)i;
        break;
      }
      cp = 0x10000u + ((cp - 0xD800u) << 10) + (p[i + 1] - 0xDC00u);
      len = 2;
    }
    if (cp < 0x80u) {
      o[q++] = (uint8_t)cp;
    } else if (cp < 0x800u) {
      o[q++] = (uint8_t)(0xC0u | (cp >> 6));
      o[q++] = (uint8_t)(0x80u | (cp & 0x3Fu));
    } else if (cp < 0x10000u) {
      o[q++] = (uint8_t)(0xE0u | (cp >> 12));
      o[q++] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
      o[q++] = (uint8_t)(0x80u | (cp & 0x3Fu));
    } else {
      o[q++] = (uint8_t)(0xF0u | (cp >> 18));
      o[q++] = (uint8_t)(0x80u | ((cp >> 12) & 0x3Fu));
      o[q++] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
      o[q++] = (uint8_t)(0x80u | (cp & 0x3Fu));
    }
    i += len;
  }
  vt_result r;
  r.written = q;
  r.consumed = err < 0 ? n : (uint64_t)err;
  r.error_at = err;
  res[s] = r;
}

int launch_utf8_to_utf16_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                               uint16_t* out, vt_result* res, int validate, cudaStream_t s) {
  if (count == 0) return 0;
  const unsigned threads = 128;
  batch_u8to16_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, s>>>(
      data, offsets, count, out, res, validate);
  return (int)cudaGetLastError();
}

int launch_utf16_to_utf8_batch(const uint16_t* data, const uint64_t* offsets, uint64_t count,
                               uint8_t* out, vt_result* res, cudaStream_t s) {
  if (count == 0) return 0;
  const unsigned threads = 128;
  batch_u16to8_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, s>>>(
      data, offsets, count, out, res);
  return (int)cudaGetLastError();
}

// Input number k of the 1/2/3-byte enumeration (acceptance.cpp:147-167).
__global__ void exhaustive_short_kernel(uint8_t* verdicts) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 256u + 65536u + 16777216u) return;
  uint8_t b[3];
  unsigned len;
  uint32_t v;
  if (k < 256u) {
    len = 1; v = k;
  } else if (k < 256u + 65536u) {
    len = 2; v = k - 256u;
  } else {
    len = 3; v = k - 256u - 65536u;
  }
  for (unsigned i = 0; i < len; i++) b[i] = (uint8_t)(v >> (8 * (len - 1 - i)));
  verdicts[k] = first_error_seq(b, len) < 0 ? 1 : 0;
}

// UTF-16LE <-> UTF-16BE: swap the two bytes of every unit (n units).
__global__ void bswap16_kernel(const uint32_t* in, uint32_t* out, uint64_t nwords) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = prmt(in[i], 0, 0x2301);
}

int launch_bswap16(const uint16_t* in, uint16_t* out, uint64_t n, cudaStream_t s) {
  if (n == 0) return 0;
  // device buffers from cudaMalloc: 4-byte aligned; an odd tail unit is padded
  const uint64_t nwords = (n + 1) / 2;
  bswap16_kernel<<<(unsigned)std::min<uint64_t>((nwords + 255) / 256, 148 * 8), 256, 0, s>>>(
      reinterpret_cast<const uint32_t*>(in), reinterpret_cast<uint32_t*>(out), nwords);
  return (int)cudaGetLastError();
}

int launch_validate_utf8_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                               int64_t* first_err, cudaStream_t s) {
  if (count == 0) return 0;
  const unsigned threads = 128;
  const uint64_t blocks = (count + threads - 1) / threads;
  batch_validate_kernel<<<(unsigned)blocks, threads, 0, s>>>(data, offsets, count, first_err);
  return (int)cudaGetLastError();
}

int launch_exhaustive_short(uint8_t* verdicts, cudaStream_t s) {
  const unsigned total = 256u + 65536u + 16777216u;
  exhaustive_short_kernel<<<(total + 255) / 256, 256, 0, s>>>(verdicts);
  return (int)cudaGetLastError();
}

}  // namespace vt

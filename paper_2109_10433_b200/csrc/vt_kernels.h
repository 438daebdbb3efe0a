// vt_kernels.h -- host-visible launch interface of the sm_100a kernels
// (internal to libvtrans_gpu.so; the public boundary is include/vtrans_gpu.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vtrans_gpu.h"

namespace vt {

struct Ctl;

// UTF-8 side: `base` is the input rounded down to 16 bytes, `head` the offset
// of the first input byte from it.  Tiles cover virtual bytes [0, head + n).

struct U8Args {
  const uint8_t* base;
  unsigned long long head;
  unsigned long long n;
  unsigned ntiles;
  unsigned epoch;
  uint16_t* out;
  unsigned long long* status;
  Ctl* ctl;
  vt_result* res;
  unsigned dbg;  // debug switches (VT_DEBUG env), 0 in production
  const unsigned* skip;  // validate only: device count of leading bytes to skip, or null
  unsigned* rows;        // validate only: per-row running totals of each warp (rows_utf8 entries)
  unsigned long long out_cap;  // output capacity in bytes (VT_CHECKS builds check it)
};

// UTF-16 side: same conventions in units (`head` in units, 0..7).
struct U16Args {
  const uint16_t* base;
  unsigned long long head;
  unsigned long long n;
  unsigned ntiles;
  unsigned epoch;
  uint8_t* out;
  unsigned long long* status;
  Ctl* ctl;
  vt_result* res;
  unsigned* rows;  // validate only: per-row running totals of each warp (rows_utf16 entries)
  unsigned long long out_cap;  // output capacity in bytes (VT_CHECKS builds check it)
};

// launch modes: validate/count, transcode to UTF-16LE / UTF-8, transcode to
// UTF-16BE (UTF-8 side) / from UTF-16BE (UTF-16 side)
constexpr int kModeValidate = 0, kModeTranscode = 1, kModeTranscodeBE = 2, kModeValidateBE = 3;
// length only: the validate kernel counting output elements (UTF-16 units of a
// UTF-8 input, UTF-8 bytes of a UTF-16 input) instead of code points
constexpr int kModeLength = 4;
// UTF-8 -> UTF-16LE without validation (the reference's validate=false)
constexpr int kModeTranscodeNV = 5;

int launch_utf8(const U8Args& a, int mode, int grid, cudaStream_t s);
int occupancy_utf8(bool transcode);
unsigned tiles_utf8(unsigned long long head, unsigned long long n);
unsigned rows_utf8(unsigned long long head, unsigned long long n);


int launch_utf16(const U16Args& a, int mode, int grid, cudaStream_t s);
int occupancy_utf16(bool transcode);
unsigned tiles_utf16(unsigned long long head, unsigned long long n);
unsigned rows_utf16(unsigned long long head, unsigned long long n);

// Batched validation of many short strings (one warp per string).
int launch_validate_utf8_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                               int64_t* first_err, cudaStream_t s);
// Batched transcoding of many short strings (one thread per string, k_batch.cu)
int launch_utf8_to_utf16_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                               uint16_t* out, vt_result* res, int validate, cudaStream_t s);
int launch_utf16_to_utf8_batch(const uint16_t* data, const uint64_t* offsets, uint64_t count,
                               uint8_t* out, vt_result* res, cudaStream_t s);
// skip value meaning "nothing of this chunk is scanned" (the stream failed)
constexpr unsigned kSkipAll = 0xFFFFFFFFu;
// Streaming UTF-8 validation (k_stream.cu): seam check before, carry/error
// update after a validate launch over the chunk (with a.skip = &st->skip).
int launch_stream_seam(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n, cudaStream_t s);
int launch_stream_tail(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n, const vt_result* res,
                       cudaStream_t s);
// Character-length histogram of valid UTF-8 (k_stream.cu): counts[0..3] +=
// number of 1/2/3/4-byte characters.
int launch_utf8_class_counts(const uint8_t* d, uint64_t n, unsigned long long* counts,
                             cudaStream_t s);
// Byte swap of n UTF-16 units (device buffers, 4-byte aligned).
int launch_bswap16(const uint16_t* in, uint16_t* out, uint64_t n, cudaStream_t s);
// Every 1/2/3-byte input (acceptance C3 order), verdict per input.
int launch_exhaustive_short(uint8_t* verdicts, cudaStream_t s);

// Synthetic workload generators (bench.py / tests): see k_datagen.cu.
int launch_gen_sizes(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks, uint64_t* sizes,
                     cudaStream_t s);
int launch_gen_write(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                     const uint64_t* offsets, uint64_t limit, void* out, uint64_t* end_pos,
                     cudaStream_t s);

}  // namespace vt

/* vtrans_gpu.h -- C ABI of the B200 (sm_100a) transcoding library
 * libvtrans_gpu.so.
 *
 * Plain pointers and sizes; no C++ or torch types.  Every entry point returns
 * an int status: 0 on success, a CUDA runtime error code (> 0) on a device or
 * runtime failure, or a negative VT_E* code.  Data errors (invalid UTF-8 /
 * UTF-16) are never statuses: they are reported in-band through vt_result,
 * exactly like vtrans::TranscodeResult (proj/include/vtrans/codec_core.hpp:11-21).
 *
 * Reference interfaces replaced (paths relative to the reference root):
 *   vt_host_utf8_to_utf16    vtrans::utf8_to_utf16(span, u16*, bool, PathCounters*)
 *                            proj/include/vtrans/utf8_to_utf16.hpp:29-30
 *   vt_host_utf16_to_utf8    vtrans::utf16_to_utf8(span, u8*)
 *                            proj/include/vtrans/utf16_to_utf8.hpp:15
 *   vt_host_validate_utf8    vtrans::validate_utf8(span)  proj/include/vtrans/validation.hpp:27
 *   vt_host_validate_utf16   vtrans::validate_utf16(span) proj/include/vtrans/validation.hpp:31
 *   vt_host_count_utf8/16    vtrans::scalar::count_codepoints_utf8/16
 *                            proj/include/vtrans/codec_core.hpp:66-67
 * The vt_* device-pointer forms are the same operations on device-resident
 * buffers, enqueued on a caller stream; the bench and the sharder use them.
 * The vtrans:: C++ drop-in (include/vtrans/*.hpp) is a thin layer over the
 * vt_host_* entry points.
 */
#ifndef VTRANS_GPU_H
#define VTRANS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same meaning and layout as the reference's TranscodeResult:
 * error_at == -1 is the empty optional; when error_at >= 0, consumed ==
 * error_at and out[0..written) is the exact transcoding of the valid prefix.
 * For the validate/count entry points `written` is the number of code points
 * in the valid prefix (== the full count when error_at == -1). */
typedef struct vt_result {
  uint64_t consumed;
  uint64_t written;
  int64_t error_at;
} vt_result;

typedef struct CUstream_st* vt_stream; /* == cudaStream_t; NULL = legacy default stream */

#define VT_E_NODEVICE (-1)  /* no CUDA device visible: there is no CPU fallback */
#define VT_E_ARG (-2)       /* invalid argument */
#define VT_E_ARCH (-3)      /* device is not sm_100 (the kernels are sm_100a-only) */

/* ---- device-pointer API ------------------------------------------------
 * Inputs and outputs are device (or host-mapped) pointers.  The *_async forms
 * enqueue on `stream` and write the result to device memory `d_res`; the plain
 * forms additionally wait and return the result in host memory `h_res`.
 * Capacities (the reference's contracts): UTF-8 -> UTF-16 needs >= n units,
 * UTF-16 -> UTF-8 needs >= 3n + 16 bytes.  Only out[0..written) is defined. */
int vt_utf8_to_utf16_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* d_res,
                           vt_stream stream);
int vt_utf16_to_utf8_async(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* d_res,
                           vt_stream stream);
int vt_validate_utf8_async(const uint8_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream);
int vt_validate_utf16_async(const uint16_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream);

int vt_utf8_to_utf16(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* h_res,
                     vt_stream stream);
int vt_utf16_to_utf8(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* h_res,
                     vt_stream stream);
int vt_validate_utf8(const uint8_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream);
int vt_validate_utf16(const uint16_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream);

/* ---- host-pointer API (the drop-in boundary) ------------------------------
 * Host buffers in, host buffers out; staging, transfers and the kernels are
 * handled internally on a per-thread stream.  Thread-safe. */
int vt_host_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, vt_result* res);
int vt_host_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, vt_result* res);
/* first_err: index of the first invalid byte / unit, or -1 when valid. */
int vt_host_validate_utf8(const uint8_t* in, uint64_t n, int64_t* first_err);
int vt_host_validate_utf16(const uint16_t* in, uint64_t n, int64_t* first_err);
/* count: code points, or -1 when the input is invalid (std::nullopt). */
int vt_host_count_utf8(const uint8_t* in, uint64_t n, int64_t* count);
int vt_host_count_utf16(const uint16_t* in, uint64_t n, int64_t* count);

/* ---- non-validating UTF-8 -> UTF-16LE --------------
 * The reference's validate=false path (proj/src/utf8_to_utf16.cpp:230-239,
 * vtrans::utf8_to_utf16(..., validate=false)): no structure or range checks.
 * Identical results on valid input; on invalid input the output is
 * unspecified (as in the reference) but never exceeds n units, and the result
 * reports no error (consumed = n). */
int vt_utf8_to_utf16_nonvalidating_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out,
                                         vt_result* d_res, vt_stream stream);
int vt_host_utf8_to_utf16_nonvalidating(const uint8_t* in, uint64_t n, uint16_t* out,
                                        vt_result* res);

/* ---- UTF-16 big-endian and byte-order marks --------
 * The reference converts big-endian UTF-16 with a separate byte-swap pass
 * around its little-endian kernels (proj/src/harness.cpp:178-199); here the
 * swap is fused into the kernels' loads (UTF-16BE input) and stores (UTF-16BE
 * output).  Same results and contracts as the little-endian entry points. */
int vt_utf8_to_utf16be_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* d_res,
                             vt_stream stream);
int vt_utf16be_to_utf8_async(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* d_res,
                             vt_stream stream);
int vt_validate_utf16be_async(const uint16_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream);
int vt_host_utf8_to_utf16be(const uint8_t* in, uint64_t n, uint16_t* out, vt_result* res);
int vt_host_utf16be_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, vt_result* res);
int vt_host_validate_utf16be(const uint16_t* in, uint64_t n, int64_t* first_err);

/* Whole-buffer transcode with BOM detection and endianness handling, the
 * semantics of vtrans::harness::transcode_bytes (proj/include/vtrans/harness.hpp:
 * 60-69, proj/src/harness.cpp:202-294).  Formats: 0 UTF-8, 1 UTF-16LE,
 * 2 UTF-16BE; BOM policy: 0 keep, 1 strip, 2 add.  `out` needs
 * 2n + 4 bytes (UTF-8 -> UTF-16), 3n/2 + 20 (UTF-16 -> UTF-8) or n + 4.
 * *exit_code: 0 ok, 1 error (the reference's exit codes); *status:
 * 0 ok, 1 BOM conflicts with the declared endianness, 2 odd byte count,
 * 3 invalid UTF-8 at *error_at (bytes, after a stripped BOM), 4 invalid UTF-16
 * at *error_at (units); bit 8 set: a UTF-8 BOM was stripped from the input. */
int vt_host_transcode_bytes(const uint8_t* in, uint64_t n, int from, int to, int bom,
                            uint8_t* out, uint64_t out_cap, uint64_t* out_len, int* exit_code,
                            int* status, int64_t* error_at);

/* ---- output lengths ---------------------------------------------------------
 * How many elements the transcoding would write: UTF-16 units of a UTF-8 input
 * (characters + supplementary characters), UTF-8 bytes of a UTF-16 input.
 * As for validation, res.written holds the length of the valid prefix and
 * res.error_at the first invalid index (-1 if none); the host forms return -1
 * for invalid input.  One read of the input, no output written. */
int vt_utf16_len_from_utf8_async(const uint8_t* d_in, uint64_t n, vt_result* d_res,
                                 vt_stream stream);
int vt_utf8_len_from_utf16_async(const uint16_t* d_in, uint64_t n, vt_result* d_res,
                                 vt_stream stream);
int vt_utf16_len_from_utf8(const uint8_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream);
int vt_utf8_len_from_utf16(const uint16_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream);
int vt_host_utf16_len_from_utf8(const uint8_t* in, uint64_t n, int64_t* len);
int vt_host_utf8_len_from_utf16(const uint16_t* in, uint64_t n, int64_t* len);

/* ---- streaming UTF-8 validation -------------------------------------------
 * The GPU form of vtrans::Utf8BlockValidator (proj/include/vtrans/
 * validation.hpp:15-24, proj/src/validation.cpp:13-22,82-93): chunks of any
 * length are fed in order; a character may straddle chunk seams.  The state
 * is 32 bytes, zero-initialised (vt_utf8_stream_init), and lives in device
 * memory for the _async call or host memory for the vt_host_ call.
 *   ok so far  <=> error_at < 0
 *   finish     <=> error_at < 0 && carry_len == 0   (no dangling sequence)
 * error_at is the first invalid byte in stream coordinates, the same index
 * whole-buffer validation of the concatenated chunks reports (rule A of
 * SURVEY.md 8(a)); a sequence cut by the end of the stream so far is not an
 * error until finish. */
typedef struct vt_utf8_stream {
  uint64_t fed;       /* bytes fed so far */
  int64_t error_at;   /* -1 = valid so far */
  uint8_t carry[4];   /* the incomplete trailing sequence (carry_len bytes) */
  uint32_t carry_len;
  uint32_t skip;      /* scratch for the current feed */
  uint32_t reserved;
} vt_utf8_stream;

void vt_utf8_stream_init(vt_utf8_stream* st);
int vt_utf8_stream_feed_async(vt_utf8_stream* d_st, const uint8_t* d_chunk, uint64_t n,
                              vt_stream stream);
int vt_host_utf8_stream_feed(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n);
int vt_utf8_stream_ok(const vt_utf8_stream* st);      /* host state: 1 = valid so far */
int vt_utf8_stream_finish(const vt_utf8_stream* st);  /* host state: 1 = valid and complete */

/* ---- corpus statistics -----------------------------------------------------
 * vtrans::harness::compute_stats (proj/include/vtrans/harness.hpp:47-55,
 * proj/src/harness.cpp): counts[0..3] = number of 1/2/3/4-byte characters of
 * a valid buffer; *valid = 0 (and counts zero) when it is not valid UTF-8. */
int vt_host_utf8_class_counts(const uint8_t* in, uint64_t n, uint64_t counts[4], int* valid);

/* ---- batched short strings ------------------------------------------------
 * `count` strings back to back in `d_data`; string i is
 * [d_offsets[i], d_offsets[i+1]).  Writes the first error index or -1. */
int vt_validate_utf8_batch(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           int64_t* d_first_err, vt_stream stream);
/* Batched transcoding, one launch for the whole batch (the reference's fuzz
 * driver makes one call per case, proj/src/harness.cpp:357-375).  String i is
 * [d_offsets[i], d_offsets[i+1]) of d_data; its output is written at the same
 * offset in d_out (UTF-8 -> UTF-16: in units, capacity = the string's byte
 * length) or at 3 * d_offsets[i] bytes (UTF-16 -> UTF-8: capacity 3 bytes per
 * unit); d_res[i] is its result, exactly as one vt_host_* call on that string
 * would return it.  validate = 0 selects the non-validating decode (same
 * result on valid strings). */
int vt_utf8_to_utf16_batch(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           uint16_t* d_out, vt_result* d_res, int validate, vt_stream stream);
int vt_utf16_to_utf8_batch(const uint16_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           uint8_t* d_out, vt_result* d_res, vt_stream stream);
/* Verdict (1 = valid) of every 1-, 2- and 3-byte input in the enumeration
 * order of acceptance C3 (proj/tests/acceptance.cpp:147-167);
 * d_verdicts holds 16843008 bytes. */
int vt_exhaustive_short_verdicts(uint8_t* d_verdicts, vt_stream stream);

/* ---- multi-GPU sharder ------------------------------------------------------
 * Splits a host buffer at character boundaries into `ndev` shards (0 = one
 * per visible GPU; shard k runs on GPU k % count),
 * runs the single-GPU path per shard concurrently (one persistent host worker
 * thread per GPU, no collective), and combines: output offsets by exclusive scan of the
 * per-shard `written`, error from the first failing shard. */
int vt_sharded_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, int ndev,
                             vt_result* res);
int vt_sharded_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, int ndev,
                             vt_result* res);
/* Device-resident shards (weak scaling without PCIe): shard k is
 * d_in[k][0..n[k]) on device dev[k], and the shards are consecutive
 * character-boundary pieces of one stream (cut with vt_split_point_*).  Every
 * device transcodes its own shard into d_out[k] (capacity as for the single
 * calls) concurrently on a library-owned stream; no host threads, no copies,
 * no collective.  shard_res[k] (may be NULL) = shard k's own result,
 * out_offsets[k] (may be NULL) = where shard k's output goes in the combined
 * stream, *res = the combined result (first failing shard decides).  Several
 * shards may name the same device (they run in order on it). */
int vt_sharded_device_utf8_to_utf16(int nshards, const int* dev, const uint8_t* const* d_in,
                                    const uint64_t* n, uint16_t* const* d_out,
                                    vt_result* shard_res, uint64_t* out_offsets, vt_result* res);
int vt_sharded_device_utf16_to_utf8(int nshards, const int* dev, const uint16_t* const* d_in,
                                    const uint64_t* n, uint8_t* const* d_out,
                                    vt_result* shard_res, uint64_t* out_offsets, vt_result* res);
/* Host-side split-point rules the sharder uses (exposed for tests). */
uint64_t vt_split_point_utf8(const uint8_t* in, uint64_t n, uint64_t cut);
uint64_t vt_split_point_utf16(const uint16_t* in, uint64_t n, uint64_t cut);

/* ---- synthetic workloads (BASELINE.json configs 1-5) ----------------------
 * Deterministic, chunked: chunk c of configuration `cfg` is a function of
 * (seed, c) only.  vt_gen_sizes writes each chunk's size in bytes (UTF-8) or
 * units (UTF-16, cfg 3); vt_gen_write writes the chunks at `d_offsets`
 * (exclusive scan of the sizes), dropping every character that would end past
 * `limit`, and stores the end of the last whole character below `limit` to
 * *d_end (device). */
int vt_gen_sizes(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks, uint64_t* d_sizes,
                 vt_stream stream);
int vt_gen_write(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                 const uint64_t* d_offsets, uint64_t limit, void* d_out, uint64_t* d_end,
                 vt_stream stream);
uint64_t vt_gen_chunk_draws(int cfg);
/* One chunk generated on the host (same definition); returns its size and
 * writes at most `cap` elements.  *first_bad: offset of the first injected
 * malformed sequence (cfg 4) or UINT64_MAX. */
uint64_t vt_gen_host_chunk(int cfg, uint64_t seed, uint64_t chunk, void* out, uint64_t cap,
                           uint64_t* first_bad);

/* ---- misc ------------------------------------------------------------------- */
const char* vt_status_string(int status);
int vt_device_count(void);
/* Number of kernels this library launched so far in the calling process. */
uint64_t vt_launch_count(void);
/* Cumulative host<->device bytes moved by the calling thread's vt_host_*
 * transcoding calls (pipelined copies, or mapped-memory traffic of the
 * zero-copy path), for end-to-end accounting. */
void vt_host_transfer_counts(uint64_t* h2d, uint64_t* d2h);
const char* vt_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* VTRANS_GPU_H */

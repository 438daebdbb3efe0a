// vtrans_dropin.hpp -- the C++ drop-in surface of libvtrans_gpu.so.
//
// A program written against the reference library (arXiv 2109.10433's
// `vtrans`, headers in proj/include/vtrans/) recompiles and links against
// libvtrans_gpu.so unchanged: the forwarding headers include/vtrans/*.hpp
// keep the reference's include paths, and this file declares the same
// entry points with the same types and layouts.  The work runs on an sm_100a
// GPU through the C ABI in vtrans_gpu.h; there is no CPU fallback: a missing
// or failing device raises std::runtime_error.
//
//   reference declaration                                 drop-in behaviour
//   codec_core.hpp:14-21   TranscodeResult                identical layout/semantics
//   utf8_to_utf16.hpp:12-22 PathCounters                  only total_bytes is
//                                                         accumulated (the other
//                                                         fields count CPU branches)
//   utf8_to_utf16.hpp:29-33 utf8_to_utf16 (2 overloads)   GPU, always validating
//   utf16_to_utf8.hpp:15-17 utf16_to_utf8 (2 overloads)   GPU
//   validation.hpp:15-24   Utf8BlockValidator            GPU (one launch group per
//                                                         feed; the chunked form is
//                                                         vt_utf8_stream_* in vtrans_gpu.h)
//   validation.hpp:27,31   validate_utf8 / validate_utf16 GPU
//   vec128.hpp:17-21       Backend, active_backend, ...   report the GPU backend
//
// The reference's scalar codec (vtrans::scalar::*) is NOT redefined here: it
// stays the reference's (the oracle).  GPU code-point counts are in
// vtrans::gpu.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <vector>

namespace vtrans {

struct TranscodeResult {
  std::size_t consumed = 0;             // input elements accepted
  std::size_t written = 0;              // output elements produced
  std::optional<std::size_t> error_at{};  // first invalid input index (then consumed == error_at)

  bool ok() const { return !error_at.has_value(); }
  friend bool operator==(const TranscodeResult&, const TranscodeResult&) = default;
};

struct PathCounters {
  uint64_t total_bytes = 0;
  uint64_t ascii64_blocks = 0;
  uint64_t ascii64_bytes = 0;
  uint64_t fast_ascii16 = 0;
  uint64_t fast_twobyte16 = 0;
  uint64_t fast_threebyte12 = 0;
  uint64_t block12 = 0;
  uint64_t scalar_fallback_chars = 0;
  uint64_t inner_iterations = 0;
};

enum class Backend { emulated, native };

// Backend reporting for link compatibility.  `native` is the GPU; there is no
// second implementation to switch to, so force_emulated_backend only records
// the request (active_backend() then reports `emulated` while the same GPU path
// keeps running).
Backend active_backend();
void force_emulated_backend(bool force);
bool native_backend_available();

// UTF-8 -> UTF-16LE.  `out` must hold input.size() units.  `validate` is
// accepted for signature compatibility; the GPU always validates (allowed: the
// reference leaves non-validating results on invalid input unspecified).
TranscodeResult utf8_to_utf16(std::span<const uint8_t> input, uint16_t* out, bool validate,
                              PathCounters* counters = nullptr);
std::vector<uint16_t> utf8_to_utf16(std::span<const uint8_t> input, bool validate,
                                    TranscodeResult& res, PathCounters* counters = nullptr);

// UTF-16LE -> UTF-8.  `out` must hold 3 * input.size() + 16 bytes.
TranscodeResult utf16_to_utf8(std::span<const uint16_t> input, uint8_t* out);
std::vector<uint8_t> utf16_to_utf8(std::span<const uint16_t> input, TranscodeResult& res);

// Streaming UTF-8 validator over 64-byte blocks, same layout and member
// meaning as the reference's: `error` is all zero while the stream is valid,
// `prev_incomplete` all zero when no sequence is left dangling at the end
// (here: its bytes, then their count at [4]), `prev_input` the last 16 bytes.
struct Utf8BlockValidator {
  std::array<uint8_t, 16> error{};
  std::array<uint8_t, 16> prev_input{};
  std::array<uint8_t, 16> prev_incomplete{};

  void feed(const uint8_t* block64);
  bool ok_so_far() const;
  bool finish() const;
};

bool validate_utf8(std::span<const uint8_t> bytes);
std::optional<std::size_t> validate_utf16(std::span<const uint16_t> units);

namespace gpu {
// Code points, or nullopt when invalid (same meaning as the reference's
// scalar::count_codepoints_utf8/16, proj/include/vtrans/codec_core.hpp:66-67).
std::optional<std::size_t> count_codepoints_utf8(std::span<const uint8_t> bytes);
std::optional<std::size_t> count_codepoints_utf16(std::span<const uint16_t> units);
}  // namespace gpu

}  // namespace vtrans

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
// The reference's scalar codec (vtrans::scalar::*) is declared (in
// vtrans/codec_core.hpp) but NOT defined here: it stays the reference's (the
// oracle).  GPU code-point counts are in vtrans::gpu.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>

#include "vtrans/codec_core.hpp"
#include "vtrans/utf16_to_utf8.hpp"
#include "vtrans/utf8_to_utf16.hpp"
#include "vtrans/validation.hpp"
#include "vtrans/vec128.hpp"

namespace vtrans {
namespace gpu {
// Code points, or nullopt when invalid (same meaning as the reference's
// scalar::count_codepoints_utf8/16, proj/include/vtrans/codec_core.hpp:66-67).
std::optional<std::size_t> count_codepoints_utf8(std::span<const uint8_t> bytes);
std::optional<std::size_t> count_codepoints_utf16(std::span<const uint16_t> units);
}  // namespace gpu
}  // namespace vtrans

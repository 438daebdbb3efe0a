// vtrans/utf16_to_utf8.hpp (drop-in) -- mirrors
// proj/include/vtrans/utf16_to_utf8.hpp:15-17 of the reference; defined by
// libvtrans_gpu.so (csrc/shim.cpp), computed on the GPU (always validating).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "vtrans/codec_core.hpp"

namespace vtrans {

// UTF-16LE -> UTF-8 into `out` (capacity: 3 * input.size() bytes).
TranscodeResult utf16_to_utf8(std::span<const uint16_t> input, uint8_t* out);
std::vector<uint8_t> utf16_to_utf8(std::span<const uint16_t> input, TranscodeResult& res);

}  // namespace vtrans

// vtrans/vec128.hpp (drop-in) -- the backend-reporting part of
// proj/include/vtrans/vec128.hpp:17-21.  The reference's 128-bit CPU vector
// types (EmuVec / SseVec) are the machinery of its SIMD loops, which the GPU
// kernels replace; they are not part of the drop-in surface.  `native` is the
// GPU; force_emulated_backend only records the request (there is no second
// implementation to switch to).
#pragma once

namespace vtrans {

enum class Backend { emulated, native };

Backend active_backend();
void force_emulated_backend(bool force);
bool native_backend_available();

}  // namespace vtrans

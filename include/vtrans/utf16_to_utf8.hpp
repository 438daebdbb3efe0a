// Forwarding header: keeps the reference's include path
// (proj/include/vtrans/utf16_to_utf8.hpp) working against libvtrans_gpu.so.
#pragma once
#include "../vtrans_dropin.hpp"

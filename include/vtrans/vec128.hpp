// Forwarding header: keeps the reference's include path
// (proj/include/vtrans/vec128.hpp) working against libvtrans_gpu.so.
#pragma once
#include "../vtrans_dropin.hpp"

// shim.cpp -- the vtrans:: C++ drop-in (include/vtrans_dropin.hpp) over the C
// ABI.  Same signatures, return values and error semantics as the reference
// entry points (proj/include/vtrans/utf8_to_utf16.hpp:29-33,
// utf16_to_utf8.hpp:15-17, validation.hpp:27-31, vec128.hpp:19-21); the work is
// done by the sm_100a kernels behind vt_host_*.  Device/runtime failures, which
// the reference API cannot express, throw std::runtime_error.
#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/vtrans_dropin.hpp"
#include "../../include/vtrans_gpu.h"

namespace vtrans {

namespace {

std::atomic<bool> g_force_emulated{false};

void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string("vtrans (GPU): ") + what + ": " + vt_status_string(rc));
}

TranscodeResult to_result(const vt_result& r) {
  TranscodeResult t;
  t.consumed = r.consumed;
  t.written = r.written;
  if (r.error_at >= 0) t.error_at = static_cast<std::size_t>(r.error_at);
  return t;
}

}  // namespace

Backend active_backend() {
  return g_force_emulated.load() ? Backend::emulated : Backend::native;
}

void force_emulated_backend(bool force) { g_force_emulated.store(force); }

bool native_backend_available() { return vt_device_count() > 0; }

TranscodeResult utf8_to_utf16(std::span<const uint8_t> input, uint16_t* out, bool validate,
                              PathCounters* counters) {
  if (counters) counters->total_bytes += input.size();
  vt_result r;
  // validate=false: the non-validating kernel (same result on valid input,
  // unspecified output on invalid input, proj/src/utf8_to_utf16.cpp:230-239)
  check(validate ? vt_host_utf8_to_utf16(input.data(), input.size(), out, &r)
                 : vt_host_utf8_to_utf16_nonvalidating(input.data(), input.size(), out, &r),
        "utf8_to_utf16");
  return to_result(r);
}

std::vector<uint16_t> utf8_to_utf16(std::span<const uint8_t> input, bool validate,
                                    TranscodeResult& res, PathCounters* counters) {
  std::vector<uint16_t> out(input.size() + 8);
  res = utf8_to_utf16(input, out.data(), validate, counters);
  out.resize(res.written);
  return out;
}

TranscodeResult utf16_to_utf8(std::span<const uint16_t> input, uint8_t* out) {
  vt_result r;
  check(vt_host_utf16_to_utf8(input.data(), input.size(), out, &r), "utf16_to_utf8");
  return to_result(r);
}

std::vector<uint8_t> utf16_to_utf8(std::span<const uint16_t> input, TranscodeResult& res) {
  std::vector<uint8_t> out(3 * input.size() + 16);
  res = utf16_to_utf8(input, out.data());
  out.resize(res.written);
  return out;
}

void Utf8BlockValidator::feed(const uint8_t* block64) {
  vt_utf8_stream st;
  vt_utf8_stream_init(&st);
  if (error[0]) st.error_at = 0;  // (no index at this layer)
  st.carry_len = prev_incomplete[4];
  std::memcpy(st.carry, prev_incomplete.data(), 4);
  check(vt_host_utf8_stream_feed(&st, block64, 64), "Utf8BlockValidator::feed");
  error.fill(0);
  error[0] = st.error_at >= 0 ? 1 : 0;
  prev_incomplete.fill(0);
  std::memcpy(prev_incomplete.data(), st.carry, st.carry_len);
  prev_incomplete[4] = (uint8_t)st.carry_len;
  std::memcpy(prev_input.data(), block64 + 48, 16);
}

bool Utf8BlockValidator::ok_so_far() const {
  for (uint8_t b : error)
    if (b) return false;
  return true;
}

bool Utf8BlockValidator::finish() const {
  if (!ok_so_far()) return false;
  for (uint8_t b : prev_incomplete)
    if (b) return false;
  return true;
}

bool validate_utf8(std::span<const uint8_t> bytes) {
  int64_t e = -1;
  check(vt_host_validate_utf8(bytes.data(), bytes.size(), &e), "validate_utf8");
  return e < 0;
}

std::optional<std::size_t> validate_utf16(std::span<const uint16_t> units) {
  int64_t e = -1;
  check(vt_host_validate_utf16(units.data(), units.size(), &e), "validate_utf16");
  if (e < 0) return std::nullopt;
  return static_cast<std::size_t>(e);
}

namespace gpu {

std::optional<std::size_t> count_codepoints_utf8(std::span<const uint8_t> bytes) {
  int64_t c = -1;
  check(vt_host_count_utf8(bytes.data(), bytes.size(), &c), "count_codepoints_utf8");
  if (c < 0) return std::nullopt;
  return static_cast<std::size_t>(c);
}

std::optional<std::size_t> count_codepoints_utf16(std::span<const uint16_t> units) {
  int64_t c = -1;
  check(vt_host_count_utf16(units.data(), units.size(), &c), "count_codepoints_utf16");
  if (c < 0) return std::nullopt;
  return static_cast<std::size_t>(c);
}

}  // namespace gpu

}  // namespace vtrans

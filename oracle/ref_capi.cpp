// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library, which
// oracle/Makefile compiles out of tree from /root/reference/proj/src into
// oracle/_ref/libvtrans_ref.so.  Used (a) to pin the C restatement in
// vt_oracle.c, (b) to generate tests/golden/ fixtures, and (c) as bench.py's
// CPU baseline ("reference" kind): the reference's own SIMD path, run on
// character-boundary shards over all host threads.
//
// This file contains no reference code; it only calls the reference API
// declared in proj/include/vtrans/*.hpp.
#include <algorithm>
#include <cstdint>
#include <span>
#include <thread>
#include <vector>

#include "vtrans/codec_core.hpp"
#include "vtrans/harness.hpp"
#include "vtrans/utf16_to_utf8.hpp"
#include "vtrans/utf8_to_utf16.hpp"
#include "vtrans/validation.hpp"
#include "vtrans/vec128.hpp"

namespace {

struct CRes {
  uint64_t consumed, written;
  int64_t error_at;
};

void put(const vtrans::TranscodeResult& r, CRes* out) {
  out->consumed = r.consumed;
  out->written = r.written;
  out->error_at = r.error_at ? static_cast<int64_t>(*r.error_at) : -1;
}

// Character-boundary shard starts.
std::vector<uint64_t> shard_starts_utf8(const uint8_t* s, uint64_t n, int k) {
  std::vector<uint64_t> st(k + 1, 0);
  for (int i = 1; i < k; i++) {
    uint64_t cut = n / k * i;
    uint64_t c = cut;
    for (uint64_t d = 0; d <= 3 && d <= cut && cut < n; d++)
      if ((s[cut - d] & 0xC0) != 0x80) {
        c = cut - d;
        break;
      }
    st[i] = std::max(c, st[i - 1]);
  }
  st[k] = n;
  return st;
}

std::vector<uint64_t> shard_starts_utf16(const uint16_t* s, uint64_t n, int k) {
  std::vector<uint64_t> st(k + 1, 0);
  for (int i = 1; i < k; i++) {
    uint64_t c = n / k * i;
    if (c > 0 && c < n && s[c] >= 0xDC00 && s[c] <= 0xDFFF && s[c - 1] >= 0xD800 &&
        s[c - 1] <= 0xDBFF)
      c--;
    st[i] = std::max(c, st[i - 1]);
  }
  st[k] = n;
  return st;
}

// Runs fn(shard_in, shard_n, shard_out) per shard on its own thread.  Every
// shard writes into `out` at an offset computed from an upper bound
// (mult * shard start), then the shards are compacted left in order.
template <typename In, typename Out, typename Fn>
void sharded(const In* in, uint64_t n, Out* out, int threads, uint64_t mult,
             const std::vector<uint64_t>& st, Fn fn, CRes* res) {
  std::vector<vtrans::TranscodeResult> rs(threads);
  std::vector<std::vector<Out>> bufs(threads);
  std::vector<std::thread> ts;
  for (int k = 0; k < threads; k++) {
    ts.emplace_back([&, k] {
      const uint64_t len = st[k + 1] - st[k];
      bufs[k].resize(len * mult + 16);
      rs[k] = fn(std::span<const In>(in + st[k], len), bufs[k].data());
    });
  }
  for (auto& t : ts) t.join();
  uint64_t written = 0;
  res->error_at = -1;
  res->consumed = n;
  for (int k = 0; k < threads; k++) {
    if (out) std::copy(bufs[k].begin(), bufs[k].begin() + rs[k].written, out + written);
    written += rs[k].written;
    if (rs[k].error_at) {
      res->error_at = static_cast<int64_t>(st[k] + *rs[k].error_at);
      res->consumed = static_cast<uint64_t>(res->error_at);
      break;
    }
  }
  res->written = written;
}

}  // namespace

extern "C" {

// vtrans::utf8_to_utf16 (proj/include/vtrans/utf8_to_utf16.hpp:29-30), SIMD driver.
void vtr_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, int validate, CRes* res) {
  put(vtrans::utf8_to_utf16(std::span<const uint8_t>(in, n), out, validate != 0), res);
}

// vtrans::utf16_to_utf8 (proj/include/vtrans/utf16_to_utf8.hpp:15).
void vtr_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, CRes* res) {
  put(vtrans::utf16_to_utf8(std::span<const uint16_t>(in, n), out), res);
}

int vtr_validate_utf8(const uint8_t* in, uint64_t n) {
  return vtrans::validate_utf8(std::span<const uint8_t>(in, n)) ? 1 : 0;
}

int64_t vtr_validate_utf16(const uint16_t* in, uint64_t n) {
  auto r = vtrans::validate_utf16(std::span<const uint16_t>(in, n));
  return r ? static_cast<int64_t>(*r) : -1;
}

void vtr_scalar_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, CRes* res) {
  put(vtrans::scalar::utf8_to_utf16(std::span<const uint8_t>(in, n), out), res);
}

void vtr_scalar_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, CRes* res) {
  put(vtrans::scalar::utf16_to_utf8(std::span<const uint16_t>(in, n), out), res);
}

int64_t vtr_count_utf8(const uint8_t* in, uint64_t n) {
  auto r = vtrans::scalar::count_codepoints_utf8(std::span<const uint8_t>(in, n));
  return r ? static_cast<int64_t>(*r) : -1;
}

int64_t vtr_count_utf16(const uint16_t* in, uint64_t n) {
  auto r = vtrans::scalar::count_codepoints_utf16(std::span<const uint16_t>(in, n));
  return r ? static_cast<int64_t>(*r) : -1;
}

int vtr_native_backend(void) {
  return vtrans::native_backend_available() && vtrans::active_backend() == vtrans::Backend::native;
}

// The reference SIMD path on `threads` character-boundary shards (bench CPU
// baseline on all host cores; the reference itself is single-threaded).
void vtr_utf8_to_utf16_mt(const uint8_t* in, uint64_t n, uint16_t* out, int threads, CRes* res) {
  if (threads < 1) threads = 1;
  auto st = shard_starts_utf8(in, n, threads);
  sharded(in, n, out, threads, 1, st,
          [](std::span<const uint8_t> s, uint16_t* o) { return vtrans::utf8_to_utf16(s, o, true); },
          res);
}

void vtr_utf16_to_utf8_mt(const uint16_t* in, uint64_t n, uint8_t* out, int threads, CRes* res) {
  if (threads < 1) threads = 1;
  auto st = shard_starts_utf16(in, n, threads);
  sharded(in, n, out, threads, 3, st,
          [](std::span<const uint16_t> s, uint8_t* o) { return vtrans::utf16_to_utf8(s, o); },
          res);
}

int vtr_validate_utf8_mt(const uint8_t* in, uint64_t n, int threads) {
  if (threads < 1) threads = 1;
  auto st = shard_starts_utf8(in, n, threads);
  std::vector<int> ok(threads, 1);
  std::vector<std::thread> ts;
  for (int k = 0; k < threads; k++)
    ts.emplace_back([&, k] {
      ok[k] = vtrans::validate_utf8(std::span<const uint8_t>(in + st[k], st[k + 1] - st[k]));
    });
  for (auto& t : ts) t.join();
  return std::all_of(ok.begin(), ok.end(), [](int v) { return v != 0; }) ? 1 : 0;
}

// Verdicts of vtrans::validate_utf8 over every 1-, 2- and 3-byte input, in the
// enumeration order of proj/tests/acceptance.cpp:147-167 (1 = valid).
uint64_t vtr_exhaustive_short_verdicts(uint8_t* verdict) {
  uint64_t k = 0;
  uint8_t b[3];
  for (int len = 1; len <= 3; len++) {
    const uint32_t total = 1u << (8 * len);
    for (uint32_t v = 0; v < total; v++) {
      for (int i = 0; i < len; i++) b[i] = static_cast<uint8_t>(v >> (8 * (len - 1 - i)));
      verdict[k++] = vtrans::validate_utf8(std::span<const uint8_t>(b, len)) ? 1 : 0;
    }
  }
  return k;
}

// vtrans::harness::transcode_bytes (proj/include/vtrans/harness.hpp:60-69).
// Writes up to cap output bytes and the message (NUL-terminated, up to mcap).
int vtr_transcode_bytes(const uint8_t* in, uint64_t n, int from, int to, int bom, uint8_t* out,
                        uint64_t cap, uint64_t* out_len, char* msg, uint64_t mcap) {
  using namespace vtrans::harness;
  const Format f[3] = {Format::utf8, Format::utf16le, Format::utf16be};
  const BomPolicy b[3] = {BomPolicy::keep, BomPolicy::strip, BomPolicy::add};
  auto r = transcode_bytes(std::span<const uint8_t>(in, n), f[from], f[to], b[bom]);
  const uint64_t k = std::min<uint64_t>(cap, r.output.size());
  std::copy(r.output.begin(), r.output.begin() + k, out);
  *out_len = r.output.size();
  const uint64_t m = std::min<uint64_t>(mcap - 1, r.message.size());
  std::copy(r.message.begin(), r.message.begin() + m, msg);
  msg[m] = 0;
  return r.exit_code;
}

}  // extern "C"

// vt_gen.cuh -- deterministic synthetic workloads for BASELINE.json configs 1-5
// (host and device).  Stand-ins for the paper's lipsum / Wikipedia-Mars corpora
// (PAPER.md:467-516), which are not available here; shapes follow BASELINE.json.
//
// The stream is cut into chunks of kDraws draws.  Chunk c is generated from a
// splitmix64 sequence seeded by (cfg, seed, c) alone, so chunks can be sized
// and written independently (in parallel) and concatenated: every chunk holds
// whole characters only.
//
//  cfg 1: 90% U+0020-007E, 10% U+0080-07FF                         (UTF-8)
//  cfg 2: 75% U+4E00-9FFF; 20% ASCII event: p=0.1 a run of U[8,64] chars of
//         U+0020-007E, else one such char; 5% U+0080-07FF            (UTF-8)
//  cfg 3: 60% U+0020-007E, 15% U+0080-07FF, 15% U+0800-FFFF minus
//         surrogates, 10% U+10000-10FFFF (surrogate pairs)         (UTF-16LE)
//  cfg 4: 25/25/25/25% 1/2/3/4-byte characters uniform over their ranges;
//         with probability 2.5/2^26 per draw (about one per 64 MiB) the draw
//         is replaced by one of 8 malformed sequences, class uniform   (UTF-8)
//  cfg 5: the cfg-3 mixture encoded as UTF-8                          (UTF-8)
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define VT_HD __host__ __device__ __forceinline__
#else
#define VT_HD inline
#endif

namespace vt {

constexpr uint64_t kDraws = 4096;

struct Rng {
  uint64_t s;
  VT_HD uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  // uniform in [0, m)
  VT_HD uint32_t below(uint32_t m) { return (uint32_t)(((next() >> 32) * (uint64_t)m) >> 32); }
  // true with probability num / 2^32
  VT_HD bool chance(uint32_t num) { return (uint32_t)(next() >> 32) < num; }
};

VT_HD Rng chunk_rng(int cfg, uint64_t seed, uint64_t chunk) {
  Rng r{seed * 0xD1B54A32D192ED03ull ^ (chunk + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)cfg << 56};
  r.next();
  r.next();
  return r;
}

VT_HD unsigned enc8(uint32_t cp, uint8_t* b) {
  if (cp < 0x80u) { b[0] = (uint8_t)cp; return 1; }
  if (cp < 0x800u) { b[0] = (uint8_t)(0xC0u | (cp >> 6)); b[1] = (uint8_t)(0x80u | (cp & 0x3Fu)); return 2; }
  if (cp < 0x10000u) {
    b[0] = (uint8_t)(0xE0u | (cp >> 12)); b[1] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
    b[2] = (uint8_t)(0x80u | (cp & 0x3Fu)); return 3;
  }
  b[0] = (uint8_t)(0xF0u | (cp >> 18)); b[1] = (uint8_t)(0x80u | ((cp >> 12) & 0x3Fu));
  b[2] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu)); b[3] = (uint8_t)(0x80u | (cp & 0x3Fu));
  return 4;
}

VT_HD uint32_t bmp_nonsurrogate(Rng& r) {  // uniform over U+0800-FFFF minus D800-DFFF
  uint32_t cp = 0x800u + r.below(0xF000u);
  if (cp >= 0xD800u) cp += 0x800u;
  return cp;
}

VT_HD uint32_t cfg3_cp(Rng& r) {
  const uint32_t p = r.below(100);
  if (p < 60) return 0x20u + r.below(0x5Fu);
  if (p < 75) return 0x80u + r.below(0x780u);
  if (p < 90) return bmp_nonsurrogate(r);
  return 0x10000u + r.below(0x100000u);
}

// One malformed sequence of class k (0..7) into b; returns its length.
VT_HD unsigned malformed(Rng& r, unsigned k, uint8_t* b) {
  const auto cont = [&](uint32_t lo, uint32_t hi) { return (uint8_t)(lo + r.below(hi - lo + 1)); };
  switch (k) {
    case 0: b[0] = (uint8_t)(0xC0u + r.below(2)); b[1] = cont(0x80, 0xBF); return 2;  // overlong 2
    case 1: b[0] = 0xE0; b[1] = cont(0x80, 0x9F); b[2] = cont(0x80, 0xBF); return 3;  // overlong 3
    case 2:                                                                           // overlong 4
      b[0] = 0xF0; b[1] = cont(0x80, 0x8F); b[2] = cont(0x80, 0xBF); b[3] = cont(0x80, 0xBF);
      return 4;
    case 3: b[0] = 0xED; b[1] = cont(0xA0, 0xBF); b[2] = cont(0x80, 0xBF); return 3;  // surrogate
    case 4:                                                                           // > U+10FFFF
      if (r.below(2)) {
        b[0] = 0xF4; b[1] = cont(0x90, 0xBF);
      } else {
        b[0] = (uint8_t)(0xF5u + r.below(3)); b[1] = cont(0x80, 0xBF);
      }
      b[2] = cont(0x80, 0xBF); b[3] = cont(0x80, 0xBF);
      return 4;
    case 5: {  // truncated: a lead with too few continuations (next draw starts a character)
      const unsigned len = 2 + r.below(3);
      unsigned have;
      if (len == 2) { b[0] = (uint8_t)(0xC2u + r.below(0x1E)); have = 0; }
      else if (len == 3) { b[0] = (uint8_t)(0xE1u + r.below(0xC)); have = r.below(2); }
      else { b[0] = (uint8_t)(0xF1u + r.below(3)); have = r.below(3); }
      for (unsigned i = 0; i < have; i++) b[1 + i] = cont(0x80, 0xBF);
      return 1 + have;
    }
    case 6: b[0] = cont(0x80, 0xBF); return 1;  // stray continuation
    default: b[0] = (uint8_t)(0xF8u + r.below(8)); return 1;  // F8..FF
  }
}

// Walks chunk `chunk` of configuration `cfg`, calling sink.chr(bytes_or_units,
// len, injected) once per character (or malformed sequence).  UTF-16 (cfg 3)
// passes units as uint16_t, all others bytes.  Stops early when sink.chr
// returns false.
template <class Sink>
VT_HD void gen_chunk(int cfg, uint64_t seed, uint64_t chunk, Sink& sink) {
  Rng r = chunk_rng(cfg, seed, chunk);
  uint8_t b[4];
  for (uint64_t d = 0; d < kDraws; d++) {
    if (cfg == 1) {
      const uint32_t cp = r.below(10) < 9 ? 0x20u + r.below(0x5Fu) : 0x80u + r.below(0x780u);
      if (!sink.chr(b, enc8(cp, b), false)) return;
    } else if (cfg == 2) {
      const uint32_t p = r.below(100);
      if (p < 75) {
        if (!sink.chr(b, enc8(0x4E00u + r.below(0x5200u), b), false)) return;
      } else if (p < 95) {
        const uint32_t run = r.below(10) == 0 ? 8u + r.below(57u) : 1u;
        for (uint32_t i = 0; i < run; i++) {
          b[0] = (uint8_t)(0x20u + r.below(0x5Fu));
          if (!sink.chr(b, 1, false)) return;
        }
      } else {
        if (!sink.chr(b, enc8(0x80u + r.below(0x780u), b), false)) return;
      }
    } else if (cfg == 3) {
      const uint32_t cp = cfg3_cp(r);
      uint16_t u[2];
      unsigned len = 1;
      if (cp < 0x10000u) {
        u[0] = (uint16_t)cp;
      } else {
        const uint32_t v = cp - 0x10000u;
        u[0] = (uint16_t)(0xD800u + (v >> 10));
        u[1] = (uint16_t)(0xDC00u + (v & 0x3FFu));
        len = 2;
      }
      if (!sink.chr(u, len, false)) return;
    } else if (cfg == 4) {
      // one malformed sequence per ~64 MiB: 2.5 bytes per draw on average
      if (r.next() < 0x0000002800000000ull * 4ull) {  // 2^64 * 2.5 / 2^26
        const unsigned k = r.below(8);
        if (!sink.chr(b, malformed(r, k, b), true)) return;
        continue;
      }
      const uint32_t cls = r.below(4);
      uint32_t cp;
      if (cls == 0) cp = r.below(0x80u);
      else if (cls == 1) cp = 0x80u + r.below(0x780u);
      else if (cls == 2) cp = bmp_nonsurrogate(r);
      else cp = 0x10000u + r.below(0x100000u);
      if (!sink.chr(b, enc8(cp, b), false)) return;
    } else {  // cfg 5
      if (!sink.chr(b, enc8(cfg3_cp(r), b), false)) return;
    }
  }
}

struct CountSink {
  uint64_t n = 0;
  template <class T>
  VT_HD bool chr(const T*, unsigned len, bool) {
    n += len;
    return true;
  }
};

template <class T>
struct WriteSink {
  T* out;           // output base
  uint64_t off;     // current element offset
  uint64_t limit;   // elements: drop characters ending past this
  uint64_t first_bad = ~0ull;
  bool stopped = false;
  VT_HD bool chr(const void* src, unsigned len, bool injected) {
    if (off + len > limit) {
      stopped = true;
      return false;
    }
    const T* s = static_cast<const T*>(src);
    for (unsigned i = 0; i < len; i++) out[off + i] = s[i];
    if (injected && first_bad == ~0ull) first_bad = off;
    off += len;
    return true;
  }
};

}  // namespace vt

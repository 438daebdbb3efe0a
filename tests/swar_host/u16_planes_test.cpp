// Host check of the byte-plane SWAR arithmetic in csrc/vt_swar.cuh (LOP3 / PRMT
// emulated bit-exactly): the UTF-16 -> UTF-8 planes against a plain scalar
// encoder, and the pairing / count planes against the scalar pairing rule.
// Built and run by tests/test_swar_host.py; prints "OK <cases>" or the first
// mismatch.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2109_10433_b200/csrc/vt_swar.cuh"

using namespace vt::swar;

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t rnd() {
  uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static bool is_hi(unsigned u) { return (u & 0xFC00u) == 0xD800u; }
static bool is_lo(unsigned u) { return (u & 0xFC00u) == 0xDC00u; }

// plain UTF-8 of a code point
static void put_cp(std::vector<uint8_t>& o, unsigned cp) {
  if (cp < 0x80) {
    o.push_back(cp);
  } else if (cp < 0x800) {
    o.push_back(0xC0 | (cp >> 6));
    o.push_back(0x80 | (cp & 0x3F));
  } else if (cp < 0x10000) {
    o.push_back(0xE0 | (cp >> 12));
    o.push_back(0x80 | ((cp >> 6) & 0x3F));
    o.push_back(0x80 | (cp & 0x3F));
  } else {
    o.push_back(0xF0 | (cp >> 18));
    o.push_back(0x80 | ((cp >> 12) & 0x3F));
    o.push_back(0x80 | ((cp >> 6) & 0x3F));
    o.push_back(0x80 | (cp & 0x3F));
  }
}

// a valid unit stream of n units (n even is not required; pairs never cut)
static std::vector<uint16_t> valid_stream(size_t n, int mode) {
  std::vector<uint16_t> u;
  while (u.size() < n) {
    const unsigned r = rnd() % 100;
    unsigned cls = mode == 0 ? (r < 60 ? 0 : r < 75 ? 1 : r < 90 ? 2 : 3) : (unsigned)(rnd() % 4);
    if (mode == 2) cls = 3;
    if (mode == 3) cls = rnd() % 2 ? 3 : 2;
    if (cls == 3 && u.size() + 2 > n) cls = 2;
    if (cls == 0) u.push_back(rnd() % 0x80);
    else if (cls == 1) u.push_back(0x80 + rnd() % 0x780);
    else if (cls == 2) {
      unsigned c;
      do c = 0x800 + rnd() % 0xF800; while (c >= 0xD800 && c <= 0xDFFF);
      // edge values more often
      if (rnd() % 8 == 0) { const unsigned e[] = {0x800, 0xFFF, 0x1000, 0xD7FF, 0xE000, 0xFFFF, 0x7FF + 1, 0xFFFE}; c = e[rnd() % 8]; }
      u.push_back(c);
    } else {
      unsigned cp = 0x10000 + rnd() % 0x100000;
      if (rnd() % 8 == 0) { const unsigned e[] = {0x10000, 0x10FFFF, 0x1FFFF, 0x20000, 0xFFFFF, 0x100000, 0x103FF, 0x10400}; cp = e[rnd() % 8]; }
      cp -= 0x10000;
      u.push_back(0xD800 + (cp >> 10));
      u.push_back(0xDC00 + (cp & 0x3FF));
    }
  }
  return u;
}

// encodes units [0, n) of s (n a multiple of 4) group by group the way the
// kernel does; `prev` is the unit before s[0]
static void planes_encode(const uint16_t* s, size_t n, unsigned prev, std::vector<uint8_t>& out) {
  const K16 k = make_k16();
  uint32_t w_prev = (uint32_t)prev << 16;
  for (size_t g = 0; g < n; g += 4) {
    const uint32_t x0 = s[g] | ((uint32_t)s[g + 1] << 16), x1 = s[g + 2] | ((uint32_t)s[g + 3] << 16);
    const uint32_t lo = lo_plane(x0, x1), hi = hi_plane(x0, x1);
    const Enc16 e = encode_group16(lo, hi, w_prev, k);
    for (int i = 0; i < 4; i++) {
      out.push_back((e.F >> (8 * i)) & 0xFF);
      if ((e.z80 >> (8 * i)) & 0x80) out.push_back((e.S >> (8 * i)) & 0xFF);
      if ((e.is3 >> (8 * i)) & 0x80) out.push_back((e.T >> (8 * i)) & 0xFF);
    }
    w_prev = x1;
  }
}

static int fail(const char* what, size_t i) {
  printf("MISMATCH %s at %zu\n", what, i);
  return 1;
}

int main() {
  size_t cases = 0;
  // 1. every BMP unit in every lane, among random valid neighbours
  for (unsigned v = 0; v < 0x10000; v++) {
    if (v >= 0xD800 && v <= 0xDFFF) continue;
    for (int lane = 0; lane < 4; lane++) {
      uint16_t s[4];
      for (int i = 0; i < 4; i++) {
        unsigned c;
        do c = rnd() % 0x10000; while (c >= 0xD800 && c <= 0xDFFF);
        s[i] = c;
      }
      s[lane] = v;
      std::vector<uint8_t> got, want;
      planes_encode(s, 4, rnd() & 0xFFFF, got);
      for (int i = 0; i < 4; i++) put_cp(want, s[i]);
      if (got != want) return fail("bmp", v);
      cases++;
    }
  }
  // 2. every surrogate pair position within / across groups: all high halves
  //    with sampled low halves and all low halves with sampled high halves
  for (unsigned h = 0xD800; h < 0xDC00; h++) {
    for (int rep = 0; rep < 8; rep++) {
      for (int pos = 0; pos < 7; pos++) {
        uint16_t s[8];
        for (int i = 0; i < 8; i++) s[i] = rnd() % 0xD800;
        const unsigned l = rep < 4 ? 0xDC00 + (rnd() % 0x400) : 0xDC00 + ((h * 37 + rep * 251) & 0x3FF);
        s[pos] = h;
        s[pos + 1] = l;
        std::vector<uint8_t> got, want;
        planes_encode(s, 8, 0x41, got);
        for (int i = 0; i < 8; i++) {
          if (i == pos) { put_cp(want, 0x10000 + ((h - 0xD800u) << 10) + (l - 0xDC00u)); i++; }
          else put_cp(want, s[i]);
        }
        if (got != want) return fail("pair-h", h);
        cases++;
      }
    }
  }
  for (unsigned l = 0xDC00; l < 0xE000; l++) {
    for (int pos = 0; pos < 7; pos++) {
      uint16_t s[8];
      for (int i = 0; i < 8; i++) s[i] = 0xE000 + rnd() % 0x2000;
      const unsigned h = 0xD800 + (rnd() % 0x400);
      s[pos] = h;
      s[pos + 1] = l;
      std::vector<uint8_t> got, want;
      planes_encode(s, 8, 0x41, got);
      for (int i = 0; i < 8; i++) {
        if (i == pos) { put_cp(want, 0x10000 + ((h - 0xD800u) << 10) + (l - 0xDC00u)); i++; }
        else put_cp(want, s[i]);
      }
      if (got != want) return fail("pair-l", l);
      cases++;
    }
  }
  // 3. a pair cut by the start of the range: the low half alone writes the
  //    last two bytes of the 4-byte sequence
  for (int it = 0; it < 200000; it++) {
    const unsigned cp = 0x10000 + rnd() % 0x100000;
    const unsigned h = 0xD800 + ((cp - 0x10000) >> 10), l = 0xDC00 + ((cp - 0x10000) & 0x3FF);
    uint16_t s[4] = {(uint16_t)l, (uint16_t)(rnd() % 0x80), (uint16_t)(0x80 + rnd() % 0x700), (uint16_t)(0xE000 + rnd() % 0x1000)};
    std::vector<uint8_t> got, want, all;
    planes_encode(s, 4, h, got);
    put_cp(all, cp);
    want.assign(all.begin() + 2, all.end());
    for (int i = 1; i < 4; i++) put_cp(want, s[i]);
    if (got != want) return fail("cut-pair", it);
    cases++;
  }
  // 4. long valid streams of several mixes against the plain encoder
  for (int it = 0; it < 3000; it++) {
    const size_t n = 4 * (1 + rnd() % 64);
    std::vector<uint16_t> s = valid_stream(n, it % 4);
    std::vector<uint8_t> got, want;
    planes_encode(s.data(), n, 0, got);
    for (size_t i = 0; i < n; i++) {
      if (is_hi(s[i])) { put_cp(want, 0x10000 + ((s[i] - 0xD800u) << 10) + (s[i + 1] - 0xDC00u)); i++; }
      else put_cp(want, s[i]);
    }
    if (got != want) return fail("stream", it);
    cases++;
  }
  // 5. count phase on arbitrary (also invalid) windows of 32 units with the
  //    unit before and after: flags, bytes, code points
  const K16 k = make_k16();
  for (int it = 0; it < 400000; it++) {
    uint16_t w[34];
    const int mode = it % 5;
    for (int i = 0; i < 34; i++) {
      const unsigned r = rnd() % 100;
      if (mode == 0) w[i] = rnd();
      else if (mode == 1) w[i] = r < 50 ? 0xD800 + rnd() % 0x800 : rnd();
      else w[i] = r < 10 ? 0xD800 + rnd() % 0x400 : r < 20 ? 0xDC00 + rnd() % 0x400 : r < 60 ? rnd() % 0x80 : rnd();
    }
    if (mode >= 3) {  // valid windows (pairs may be cut by the ends, which is flagged)
      std::vector<uint16_t> s = valid_stream(34, it % 4);
      memcpy(w, s.data(), sizeof(w));
    }
    Count16 c{};
    c.hp = hs_plane(hi_plane(0, w[0] | ((uint32_t)w[0] << 16)), k.k58);
    for (int g = 0; g < 8; g++) {
      const uint32_t x0 = w[1 + 4 * g] | ((uint32_t)w[2 + 4 * g] << 16), x1 = w[3 + 4 * g] | ((uint32_t)w[4 + 4 * g] << 16);
      count_group16<true>(lo_plane(x0, x1), hi_plane(x0, x1), k.k58, c);
    }
    count_group16<false>(lo_plane(w[33], 0), hi_plane(w[33], 0), k.k58, c);
    bool bad = false;
    for (int i = 1; i <= 33; i++) bad |= is_hi(w[i - 1]) != is_lo(w[i]);
    if (bad != (c.err != 0)) return fail("pairing flag", it);
    unsigned bytes = 0, chars = 0;
    for (int i = 1; i <= 32; i++) {
      const unsigned u = w[i];
      bytes += u < 0x80 ? 1 : u < 0x800 ? 2 : (u >= 0xD800 && u <= 0xDFFF) ? 2 : 3;
      chars += is_lo(u) ? 0 : 1;
    }
    const unsigned gb = 32 + lane_sum(c.acc) - lane_sum(c.nsur), gc = 32 - lane_sum(c.nlo);
    if (gb != bytes) return fail("bytes", it);
    if (gc != chars) return fail("chars", it);
    cases++;
  }
  printf("OK %zu\n", cases);
  return 0;
}

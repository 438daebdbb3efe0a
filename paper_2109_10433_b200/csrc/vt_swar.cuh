// vt_swar.cuh -- the byte-plane SWAR arithmetic of the UTF-16 -> UTF-8 direction,
// written so that the same source runs on the device (LOP3 / PRMT through
// inline PTX) and on the host (bit-exact emulation of those two instructions),
// where tests/test_swar_host.py checks it exhaustively without a GPU.
//
// Four UTF-16 units per 32-bit operation: two input words (u0 u1 | u2 u3) are
// split into the plane of their low bytes and the plane of their high bytes
// (one PRMT each), and every classification and encoding step works on the
// four byte lanes at once.  (The first version of this kernel worked on 16-bit
// lanes, two units per operation; the kernel is bound by the ALU pipe, so the
// per-unit instruction count is what matters.)
//
// Replaces the reference's 8-unit register dispatch with pack tables,
// proj/src/utf16_to_utf8.cpp:12-107; the byte layout of every unit is
// proj/src/codec_core.cpp:60-72 (encode_utf8) with a surrogate pair's 4 bytes
// split 2 + 2 between its halves.
#pragma once

#include <cstdint>

#if defined(__CUDA_ARCH__)
#define VT_SWAR_FN __device__ __forceinline__
#else
#define VT_SWAR_FN inline
#endif

namespace vt {
namespace swar {

// LOP3: bit i of LUT is the result for (a, b, c) = (i>>2 & 1, i>>1 & 1, i & 1)
template <int LUT>
VT_SWAR_FN uint32_t l3(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
#else
  uint32_t r = 0;
  for (int i = 0; i < 8; i++)
    if ((LUT >> i) & 1) r |= ((i & 4) ? a : ~a) & ((i & 2) ? b : ~b) & ((i & 1) ? c : ~c);
  return r;
#endif
}

// PRMT, default mode: result byte k = byte (sel nibble k & 7) of {a: 0..3, b: 4..7};
// nibble bit 3 replicates that byte's sign bit instead
VT_SWAR_FN uint32_t pr(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
#else
  const uint64_t v = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int k = 0; k < 4; k++) {
    const unsigned s = (sel >> (4 * k)) & 0xF;
    uint32_t byte = (uint32_t)(v >> (8 * (s & 7))) & 0xFFu;
    if (s & 8) byte = (byte & 0x80u) ? 0xFFu : 0x00u;
    r |= byte << (8 * k);
  }
  return r;
#endif
}

// (hi:lo) << s, upper word: the funnel shift SHF.L.W
VT_SWAR_FN uint32_t fsl(uint32_t lo, uint32_t hi, unsigned s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_l(lo, hi, s);
#else
  s &= 31;
  return s ? (hi << s) | (lo >> (32 - s)) : hi;
#endif
}

constexpr uint32_t H8 = 0x80808080u;

// Constants that follow a masked value into a LOP3 ("(v & imm) | K" is one
// instruction only when K sits in a register: LOP3 takes one immediate).
struct K16 {
  uint32_t k80, kE0, k58;
};
VT_SWAR_FN K16 make_k16() {
  K16 k{0x80808080u, 0xE0E0E0E0u, 0x58585858u};
#if defined(__CUDA_ARCH__)
  // opaque to ptxas, or it folds them back into two instructions per use
  asm volatile("" : "+r"(k.k80), "+r"(k.kE0), "+r"(k.k58));
#endif
  return k;
}

// Low-byte / high-byte planes of the four units of two words.
VT_SWAR_FN uint32_t lo_plane(uint32_t x0, uint32_t x1) { return pr(x0, x1, 0x6420); }
VT_SWAR_FN uint32_t hi_plane(uint32_t x0, uint32_t x1) { return pr(x0, x1, 0x7531); }

// D800..DFFF lanes as a clean bit-7 plane: the high byte is 1101 1xxx.
// t = (hi & 0x78) ^ 0x58 is 0 exactly for x101 1xxx, and t + 0x78 carries into
// bit 7 exactly when t != 0 (t is a multiple of 8, at most 0x78: no carry
// leaves the lane).
VT_SWAR_FN uint32_t sur_plane(uint32_t hi, uint32_t k58) {
  const uint32_t t = l3<0x6A>(hi, 0x78787878u, k58);  // (a & b) ^ c
  return l3<0x20>(hi, t + 0x78787878u, H8);           // a & ~b & c
}

// ---- count phase ------------------------------------------------------------
// Running state of a thread's classification (byte-lane counters; a thread has
// 8 groups, so no lane overflows).
struct Count16 {
  uint32_t hp;    // high-surrogate plane of the previous group (pairing check)
  uint32_t err;   // some pair of neighbouring units fails the pairing rule
  uint32_t acc;   // + [u >= 0x80] + [u >= 0x800] per lane
  uint32_t nsur;  // + [surrogate] per lane
  uint32_t nlo;   // + [low surrogate] per lane
};

// (v >> 7) + acc for a clean bit-7 plane v: one LEA.HI
VT_SWAR_FN uint32_t add_plane(uint32_t v, uint32_t acc) { return (v >> 7) + acc; }

// The high-surrogate plane of a group, for the pairing check of the group
// after it (the thread's previous word).
VT_SWAR_FN uint32_t hs_plane(uint32_t hi, uint32_t k58) {
  return sur_plane(hi, k58) & ~(hi << 5);  // bit 10 of the unit clear: high
}

// One group of the count phase.  `own`: the group lies in the thread's range
// (counts); otherwise it is the group after the range, whose first unit only
// closes the last pair (mask 0x80).
// Pairing (rule C of SURVEY.md 8(a)): the unit before each unit is a high
// surrogate exactly when the unit is a low one; one XOR flags both failures.
// A pair whose other unit lies outside the thread's range may flag a
// neighbour's error: the thread then runs the exact check and finds none of
// its own.
template <bool kOwn>
VT_SWAR_FN void count_group16(uint32_t lo, uint32_t hi, uint32_t k58, Count16& c) {
  const uint32_t sur = sur_plane(hi, k58);
  const uint32_t x5 = hi << 5;  // bit 10 of the unit (low surrogate) -> bit 7
  const uint32_t hm = sur & ~x5, lm = sur & x5;
  const uint32_t prev_hi = fsl(c.hp, hm, 8);  // lane i: unit i-1 is a high surrogate
  if (kOwn) {
    c.err |= prev_hi ^ lm;
    c.hp = hm;
    const uint32_t h7 = hi & 0x7F7F7F7Fu;
    // u >= 0x80: the high byte is not zero, or bit 7 of the low byte
    const uint32_t nz = l3<0xA8>(h7 + 0x7F7F7F7Fu, hi, H8);  // (a | b) & c
    const uint32_t g80 = l3<0xF8>(nz, lo, H8);               // a | (b & c)
    const uint32_t g800 = l3<0xA8>(h7 + 0x78787878u, hi, H8);  // high byte >= 8
    c.acc = add_plane(g80, c.acc);
    c.acc = add_plane(g800, c.acc);
    c.nsur = add_plane(sur, c.nsur);
    c.nlo = add_plane(lm, c.nlo);
  } else {
    c.err |= (prev_hi ^ lm) & 0x00000080u;
  }
}

VT_SWAR_FN unsigned lane_sum(uint32_t v) { return (v * 0x01010101u) >> 24; }

// ---- encode phase -----------------------------------------------------------
// UTF-8 bytes of the four units of a group as three planes: F (first byte,
// every unit), S (second byte, units >= 0x80: bit 7 of z80), T (third byte,
// 3-byte BMP units: bit 7 of is3).  A surrogate pair's 4 bytes are split 2 + 2:
// with w = (hi & 0x3FF) + 0x40 (code point bits 10..20) the high half writes
// F0 | w>>8, 80 | (w>>2 & 3F) and the low half 80 | (w&3)<<4 | (lo>>6 & F),
// 80 | lo & 3F, where w & 3 == hi & 3 -- so a low surrogate needs only two
// bits of the unit before it (`w_prev`: the word before the group, whose upper
// unit that is for lane 0).
struct Enc16 {
  uint32_t F, S, T, z80, is3;
};

VT_SWAR_FN Enc16 encode_group16(uint32_t lo, uint32_t hi, uint32_t w_prev, const K16& k) {
  Enc16 e;
  const uint32_t h7 = hi & 0x7F7F7F7Fu;
  e.z80 = l3<0xFE>(h7 + 0x7F7F7F7Fu, hi, lo);  // bit 7: u >= 0x80
  const uint32_t sur = sur_plane(hi, k.k58);
  const uint32_t hm = sur & ~(hi << 5);
  e.is3 = l3<0x54>(h7 + 0x78787878u, hi, sur);  // (a | b) & ~c, bit 7: 3-byte BMP unit
  // full-byte lane masks from bit 7
  const uint32_t m80 = pr(e.z80, 0, 0xBA98), m3 = pr(e.is3, 0, 0xBA98);
  const uint32_t ms = pr(sur, 0, 0xBA98), mh = pr(hm, 0, 0xBA98);
  // M = bits 6..13 of the unit: the next lane's bits that the shifts bring in
  // are masked by the merge
  const uint32_t M = l3<0xE2>(hi << 2, 0xFCFCFCFCu, lo >> 6);  // (a & b) | (c & ~b)
  // first byte
  const uint32_t F2 = M | 0xC0C0C0C0u;                        // u < 0x800: M < 0x20
  const uint32_t F3 = l3<0xEA>(hi >> 4, 0x0F0F0F0Fu, k.kE0);  // (a & b) | c
  const uint32_t M0 = l3<0xEA>(M, 0x0F0F0F0Fu, k.k80);        // 80 | bits 6..9
  // w >> 6 = (bits 6..9 of the unit) + 1: adding 0x40 to the low 10 bits adds
  // 1 to bits 6 and up whatever the low 6 bits are.  (Bit 7 of M0 rides along
  // and is masked wherever W6 is used; the 0x40 added on top lands on bit 4
  // after the shift, the 0x10 that turns E0 into the F0 of a 4-byte lead.)
  const uint32_t W6 = M0 + 0x41414141u;
  const uint32_t Fh = l3<0xEA>(W6 >> 2, 0x17171717u, k.kE0);
  const uint32_t PL = pr(w_prev, lo, 0x6542);  // lane i: low byte of unit i-1
  const uint32_t Fl = l3<0xEA>(PL << 4, 0x30303030u, M0);
  // (mux(m, a, b) = m ? a : b is LOP3 0xCA with the mask first)
  const uint32_t Fn = l3<0xCA>(ms, l3<0xCA>(mh, Fh, Fl), l3<0xCA>(m3, F3, F2));
  e.F = l3<0xCA>(m80, Fn, lo);
  // second byte: 2-byte and low surrogate lo & 3F; 3-byte M & 3F; high
  // surrogate (w >> 2) & 3F = (W6 & 3) << 4 | bits 2..5 of the unit
  const uint32_t Sh = l3<0xE2>(W6 << 4, 0x30303030u, lo >> 2);
  e.S = l3<0xEA>(l3<0xCA>(m3, M, l3<0xCA>(mh, Sh, lo)), 0x3F3F3F3Fu, k.k80);
  e.T = l3<0xEA>(lo, 0x3F3F3F3Fu, k.k80);
  return e;
}

}  // namespace swar
}  // namespace vt

// k_utf8.cu -- validated UTF-8 -> UTF-16LE transcoding and UTF-8 validation /
// code-point counting on sm_100a.
//
// Replaces the reference's 64-byte block driver (proj/src/utf8_to_utf16.cpp:
// 88-226) and the nibble-table checker (proj/include/vtrans/utf8_checker.hpp:
// 28-137).  One persistent kernel; per 16 KiB tile, each thread owns 64
// contiguous bytes (16 words):
//   A. SWAR classification, 4 bytes per 32-bit op: continuation / >=C0 /
//      >=E0 / >=F0 bit planes, the lead/continuation structure check (a byte
//      must be a continuation iff a lead 1..3 bytes back requires it), and a
//      cheap filter for the only leads whose value range needs checking
//      (C0 C1, E0 ED EE EF; F0..FF go to the 4-byte path).  Counting is
//      SWAR too: units = characters + 4-byte characters.
//   B. any flag -> the exact first-error rule of SURVEY.md 8(a) fact A over
//      the thread's bytes (the scalar decoder's error_at, proj/src/
//      codec_core.cpp:85-104, without a sequential re-scan);
//   C. block scan + decoupled look-back for the output offset;
//   D. branch-free SWAR decode of BMP characters (lead-attributed byte planes:
//      low and high byte of each character's UTF-16 unit), predicated 16-bit
//      stores into a shared-memory staging buffer; threads with 4-byte or
//      range-checked leads decode per character instead;
//   E. aligned 16-byte stores of the staged tile to the (arbitrarily aligned)
//      output.
// Tiles at the ends of the input (partial, or whose halo leaves the input)
// and tiles containing an error take a simple masked per-character path.
#include <cstdio>

#include "vt_kernels.h"
#include "vt_pipeline.cuh"

namespace vt {

constexpr int K8_THREADS = kComputeThreads;
#ifndef VT_K8_WPT
#define VT_K8_WPT 16
#endif
constexpr int K8_WPT = VT_K8_WPT;               // words per thread
constexpr int K8_BPT = 4 * K8_WPT;              // bytes per thread
constexpr int K8_TILE = K8_THREADS * K8_BPT;    // bytes per tile
constexpr unsigned kNone = 0xFFFFFFFFu;
constexpr uint32_t H = 0x80808080u;

__device__ __forceinline__ unsigned leadlen(unsigned b) {
  return b < 0xC0u ? 1u : b < 0xE0u ? 2u : b < 0xF0u ? 3u : b < 0xF8u ? 4u : 1u;
}

// Input description passed by value to out-of-line helpers (a reference to
// the kernel parameters would force a local-memory copy of them).
struct Src {
  const uint8_t* base;
  unsigned long long head, n;
};

// A thread's 64 bytes plus the word before and the word after.
struct Words {
  uint32_t w[K8_WPT + 2];  // w[0] = previous word, w[1..16] = own, w[17] = next
};

// One word straddling an end of the input, byte by byte (rare; out of line).
__device__ __noinline__ uint32_t straddle_word(Src a, long long p) {
  const long long lo = (long long)a.head, hi = (long long)(a.head + a.n);
  uint32_t x = 0;
  for (int b = 0; b < 4; b++)
    if (p + b >= lo && p + b < hi) x |= (uint32_t)a.base[p + b] << (8 * b);
  return x;
}

// A thread's window at the ends of the input, bytes outside [head, head + n)
// as 0x00: the whole words inside the input are loaded at once (they are
// 4-byte aligned in the virtual range), the at most two straddling words byte
// by byte.  Zeros are ASCII to the classification, so an end tile takes the
// SWAR path like any other (its counts minus the zeros); a character cut by an
// end, or a continuation byte at the start, still shows as a structure error.
// (A byte-serial masked load here cost ~70 dependent memory round trips, some
// 40 us, at the first and the last tile of every call.)
__device__ __forceinline__ void load_edge(Src a, long long v0, uint32_t* w) {
  constexpr int NW = K8_WPT + 2;
  const long long s0 = v0 - 4;  // virtual position of word 0
  const long long lo = (long long)a.head, hi = (long long)(a.head + a.n);
  const int kf = (int)max(0LL, min((long long)NW, (lo - s0 + 3) >> 2));  // words [kf, kl)
  const int kl = (int)max((long long)kf, min((long long)NW, (hi - s0) >> 2));  // are inside
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(a.base + s0);
#pragma unroll
  for (int k = 0; k < NW; k++) w[k] = (k >= kf && k < kl) ? __ldg(wp + k) : 0u;
#pragma unroll
  for (int k = 0; k < NW; k++)
    if ((k == kf - 1 || k == kl) && s0 + 4 * k + 4 > lo && s0 + 4 * k < hi)
      w[k] = straddle_word(a, s0 + 4 * k);
}

// byte j in [-4, 8) of the 12-byte window (pw, cw, nw) around word cw
__device__ __forceinline__ unsigned b12(uint32_t pw, uint32_t cw, uint32_t nw, int j) {
  return j < 0 ? (pw >> (8 * (j + 4))) & 0xFFu : j < 4 ? (cw >> (8 * j)) & 0xFFu
                                                       : (nw >> (8 * (j - 4))) & 0xFFu;
}

// Exact first error among positions [lo, hi) of a thread's window (rule A of
// SURVEY.md 8(a)): the smallest position whose lead fails to decode or whose
// continuation no lead 1..3 bytes back reaches.  Rare path (tiles with an
// error), out of line, on a copy of the caller's window (so the hot path keeps
// its words in registers); one loop step per word with the words before and
// after in registers.
//
// The scan starts 3 bytes before the first lane where the lead/continuation
// planes disagree or a special lead fails its range check (first_violation):
// no rule-A error lies further back -- an orphan continuation is itself such a
// lane, a lead that fails to decode either fails its range check at its own
// lane or leaves one of its next 3 lanes short of a continuation (the argument
// in classify) -- so the per-byte loop runs over a few bytes instead of 64
// (the loop is serial: ~40 dependent steps per byte on one thread, which the
// whole tile waits for).
__device__ __forceinline__ unsigned long long need_plane(uint32_t l2, uint32_t l3, uint32_t l4);
__device__ __noinline__ unsigned first_violation(const Words& W);

__device__ __noinline__ unsigned first_error_w(const Words& W, unsigned lo, unsigned hi) {
  const unsigned v = first_violation(W);
  if (v != kNone && v >= 3 && v - 3 > lo) lo = v - 3;
  const int k0 = (int)(lo >> 2);
  uint32_t pw = W.w[k0], cw = W.w[k0 + 1];
  for (int k = k0; k < K8_WPT; k++) {
    const uint32_t nw = W.w[k + 2];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const unsigned i = 4 * k + j;
      if (i < lo || i >= hi) continue;
      const unsigned b = b12(pw, cw, nw, j);
      if ((b & 0xC0u) == 0x80u) {
        const bool covered = leadlen(b12(pw, cw, nw, j - 1)) > 1u ||
                             leadlen(b12(pw, cw, nw, j - 2)) > 2u ||
                             leadlen(b12(pw, cw, nw, j - 3)) > 3u;
        if (!covered) return i;
      } else if (b >= 0x80u) {
        const uint32_t v = b | (b12(pw, cw, nw, j + 1) << 8) | (b12(pw, cw, nw, j + 2) << 16) |
                           (b12(pw, cw, nw, j + 3) << 24);
        if (!decode_ok(v)) return i;
      }
    }
    pw = cw;
    cw = nw;
  }
  return kNone;
}

struct ClassOut {
  unsigned units;  // UTF-16 units of characters starting here (transcode) / characters
  unsigned chars;
  bool viol;       // lead/continuation structure violated near our bytes
  bool susp;       // a lead whose value range must be checked (C0 C1 E0 ED EE EF)
  bool four;       // a 4-byte lead (or F8..FF) in our bytes
};


// Continuation requirements of the lead planes of one word as a 64-bit sum:
// lane i+1 (l2), i+2 (l3), i+3 (l4); the high half belongs to the next word.
__device__ __forceinline__ unsigned long long need_plane(uint32_t l2, uint32_t l3, uint32_t l4) {
  return (unsigned long long)l2 * 0x100u + (unsigned long long)l3 * 0x10000u +
         (unsigned long long)l4 * 0x1000000u;
}

// Leads whose value range depends on the next byte, as bit 7 of each lane:
// C0 C1, E0, ED..FF (EE EF and F1..F3 are harmless extras, checked exactly like
// the rest).  Per-lane unsigned compares x >= K on the low 7 bits (all leads
// have bit 7 set; no carry crosses a lane): the adds run on the FMA pipe
// (VIADD), the selections are single LOP3s.
__device__ __forceinline__ uint32_t special_lanes(uint32_t x, uint32_t l2, uint32_t l3) {
  const uint32_t x7 = x & 0x7F7F7F7Fu;
  const uint32_t ge_c2 = x7 + 0x3E3E3E3Eu, ge_e1 = x7 + 0x1F1F1F1Fu;
  const uint32_t ge_ed = x7 + 0x13131313u;
  // (excluding F1..F3 as well costs two more ops per word and saves nothing:
  // a warp with any flagged lane runs the exact check anyway)
  const uint32_t h = lop3<0xA2>(ge_ed, ge_e1, l3);     // (a | ~b) & c: E0, ED..FF
  return lop3<0xBA>(l2, ge_c2, h);                     // (a & ~b) | c: + C0 C1
}

// Exact range check of the special leads of every word, for the threads the
// filter flagged; out of line (inlining it costs the hot path registers) and
// branch-free.  With the structure already checked, the only range errors are
// on the lead and the byte after it (C0 C1; E0 + 80..9F; ED + A0..BF;
// F0 + 80..8F; F4 + 90..BF; F5..FF): all lanes of a word at once.
// Also counts the thread's 4-byte leads (F0..FF are special leads, so a
// thread without special leads has none): bit 31 = range error, low byte =
// 4-byte leads.  The count moved here off the hot loop (one ALU op per word).
__device__ __noinline__ unsigned specials_check(const Words W) {
  uint32_t bad = 0, cf = 0;
#pragma unroll
  for (int k = 1; k <= K8_WPT; k++) {
    const uint32_t x = W.w[k], x2 = x << 1;
    const uint32_t l2 = x & x2 & H, l3 = l2 & (x << 2), l4 = l3 & (x << 3);
    const uint32_t x7 = x & 0x7F7F7F7Fu;
    const uint32_t ge_c2 = x7 + 0x3E3E3E3Eu, ge_e1 = x7 + 0x1F1F1F1Fu;
    const uint32_t ge_ed = x7 + 0x13131313u, ge_ee = x7 + 0x12121212u;
    const uint32_t ge_f1 = x7 + 0x0F0F0F0Fu, ge_f4 = x7 + 0x0C0C0C0Cu, ge_f5 = x7 + 0x0B0B0B0Bu;
    const uint32_t n1 = prmt(x, W.w[k + 1], 0x4321);  // byte i = the byte after it
    const uint32_t b5 = n1 << 2, b45 = (n1 | (n1 << 1)) << 2;  // bit 7: n1 >= A0 / >= 90
    bad |= (l2 & ~ge_c2) | (l3 & ~ge_e1 & ~b5) | (l3 & ge_ed & ~ge_ee & b5) |
           (l4 & ~ge_f1 & ~b45) | (l4 & ge_f4 & ~ge_f5 & b45) | (l4 & ge_f5);
    cf += l4 >> 7;
  }
  return ((bad & H) != 0 ? 0x80000000u : 0u) | ((cf * 0x01010101u) >> 24);
}

// Phase A over the 16 own words (SWAR, branch-free): structure check,
// special-lead flag, counts.
//
// Structure: lane i must be a continuation exactly when a lead at i-1 (any
// lead), i-2 (3/4-byte) or i-3 (4-byte) requires it.  The requirement planes
// are summed, not ORed, as one 64-bit multiply-add chain per word (FMA pipe;
// the high half spills into the next word): a lane required twice reads as not
// required, but then the first lead inside the range of the earliest
// overlapping lead is required exactly once while not being a continuation, so
// "some lane differs" is unchanged.
__device__ __forceinline__ ClassOut classify(const Words& W) {
  uint32_t carry;  // requirement bits the previous word spills into this one
  {
    const uint32_t x = W.w[0], x2 = x << 1;
    const uint32_t l2 = x & x2 & H, l3 = l2 & (x << 2), l4 = l3 & (x << 3);
    carry = (uint32_t)(need_plane(l2, l3, l4) >> 32);
  }
  uint32_t viol = 0, spec = 0, ccont = 0;
#pragma unroll
  for (int k = 1; k <= K8_WPT + 1; k++) {
    const uint32_t x = W.w[k], x2 = x << 1;
    const uint32_t c = x & ~x2 & H;
    const uint32_t l2 = x & x2 & H;
    const uint32_t l3 = l2 & (x << 2);
    const uint32_t l4 = l3 & (x << 3);
    const unsigned long long t = need_plane(l2, l3, l4);
    const uint32_t need = (uint32_t)t + carry;
    carry = (uint32_t)(t >> 32);
    if (k <= K8_WPT) {
      viol = lop3<0xF6>(viol, need, c);  // a | (b ^ c)
      spec |= special_lanes(x, l2, l3);
      // counts by shift + add on the ALU pipe: the count phase is FMA-bound
      // (need_plane's IMAD.WIDE are quarter rate, and so is IMAD.HI, which
      // summed these before: 0.900 -> 0.883 ms cfg2, validation 0.335 -> 0.320)
      ccont += c >> 7;   // + continuation lanes
    } else {
      viol |= (need ^ c) & 0x00808080u;  // next word: lanes that can blame our bytes
    }
  }
  ClassOut o;
  const unsigned nc = (ccont * 0x01010101u) >> 24;
  const unsigned sc = (spec & H) != 0 ? specials_check(W) : 0u;
  const unsigned n4 = sc & 0xFFu;
  o.chars = K8_BPT - nc;
  o.units = o.chars + n4;
  o.viol = (viol & H) != 0 || (sc >> 31) != 0;
  o.susp = (spec & H) != 0;
  o.four = n4 != 0;
  return o;
}

// Non-validating count (the reference's validate=false path, proj/src/
// utf8_to_utf16.cpp:230-239): no structure or range checks, only what the
// emit will store -- one unit per non-continuation byte, plus the low
// surrogate of every F0..FF lead whose next byte is a continuation (that
// lane is where emit_word_four<kNV=true> stores it).  Bounded by the input
// length on any input: each extra unit consumes a continuation byte.
__device__ __forceinline__ ClassOut classify_nv(const Words& W) {
  uint32_t ccont = 0, pairs = 0, four = 0;
#pragma unroll
  for (int k = 1; k <= K8_WPT; k++) {
    const uint32_t x = W.w[k], x2 = x << 1;
    const uint32_t c = x & ~x2 & H;                       // continuation lanes
    const uint32_t f4 = x & x2 & (x << 2) & (x << 3) & H;  // F0..FF lanes
    const uint32_t n = W.w[k + 1];
    // continuation plane of the byte after each lane
    const uint32_t cn = prmt(c, n & ~(n << 1) & H, 0x4321);
    ccont += c >> 7;
    pairs += (f4 & cn) >> 7;
    four |= f4;
  }
  ClassOut o;
  o.chars = K8_BPT - ((ccont * 0x01010101u) >> 24);
  o.units = o.chars + ((pairs * 0x01010101u) >> 24);
  o.viol = false;
  o.susp = false;
  o.four = four != 0;
  return o;
}

// First lane (0..63 own bytes, 64..66 the next word's) where the summed
// requirement plane and the continuation plane differ, or a special lead's
// range check fails (the planes of classify / specials_check); kNone if none.
__device__ __noinline__ unsigned first_violation(const Words& W) {
  uint32_t carry;
  {
    const uint32_t x = W.w[0], x2 = x << 1;
    const uint32_t l2 = x & x2 & H, l3 = l2 & (x << 2), l4 = l3 & (x << 3);
    carry = (uint32_t)(need_plane(l2, l3, l4) >> 32);
  }
  for (int k = 1; k <= K8_WPT + 1; k++) {
    const uint32_t x = W.w[k], x2 = x << 1;
    const uint32_t c = x & ~x2 & H;
    const uint32_t l2 = x & x2 & H, l3 = l2 & (x << 2), l4 = l3 & (x << 3);
    const unsigned long long t = need_plane(l2, l3, l4);
    const uint32_t need = (uint32_t)t + carry;
    carry = (uint32_t)(t >> 32);
    uint32_t bad = (need ^ c) & H;
    if (k <= K8_WPT) {
      const uint32_t x7 = x & 0x7F7F7F7Fu;
      const uint32_t ge_c2 = x7 + 0x3E3E3E3Eu, ge_e1 = x7 + 0x1F1F1F1Fu;
      const uint32_t ge_ed = x7 + 0x13131313u, ge_ee = x7 + 0x12121212u;
      const uint32_t ge_f1 = x7 + 0x0F0F0F0Fu, ge_f4 = x7 + 0x0C0C0C0Cu, ge_f5 = x7 + 0x0B0B0B0Bu;
      const uint32_t n1 = prmt(x, W.w[k + 1], 0x4321);
      const uint32_t b5 = n1 << 2, b45 = (n1 | (n1 << 1)) << 2;
      bad |= ((l2 & ~ge_c2) | (l3 & ~ge_e1 & ~b5) | (l3 & ge_ed & ~ge_ee & b5) | (l4 & ~ge_f1 & ~b45) |
              (l4 & ge_f4 & ~ge_f5 & b45) | (l4 & ge_f5)) & H;
    } else {
      bad &= 0x00808080u;  // only the next word's lanes 0..2 can concern our bytes
    }
    if (bad) return 4u * (k - 1) + ((unsigned)__ffs(bad) - 1u) / 8u;
  }
  return kNone;
}

// ---- generic path (ends of the input, tiles with an error): rare, per byte --
// Counts (units or characters) of the characters starting at positions
// [lo, lim) of the thread's bytes; with `dst`, also writes their units.
__device__ __forceinline__ uint16_t bswap16(unsigned u) {
  return (uint16_t)(((u & 0xFFu) << 8) | ((u >> 8) & 0xFFu));
}

__device__ __noinline__ unsigned generic_chars(const Words& W, unsigned lo, unsigned lim,
                                               bool units, uint16_t* dst, bool be = false) {
  unsigned q = 0;
  uint32_t pw = W.w[0], cw = W.w[1];
  for (int k = 0; k < K8_WPT; k++) {
    const uint32_t nw = W.w[k + 2];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const unsigned p = 4 * k + j;
      if (p < lo || p >= lim) continue;
      const unsigned b0 = b12(pw, cw, nw, j);
      if ((b0 & 0xC0u) == 0x80u) continue;  // continuation
      const unsigned b1 = b12(pw, cw, nw, j + 1) & 0x3F, b2 = b12(pw, cw, nw, j + 2) & 0x3F,
                     b3 = b12(pw, cw, nw, j + 3) & 0x3F;
      unsigned cp;
      if (b0 < 0x80u) cp = b0;
      else if (b0 < 0xE0u) cp = ((b0 & 0x1Fu) << 6) | b1;
      else if (b0 < 0xF0u) cp = ((b0 & 0x0Fu) << 12) | (b1 << 6) | b2;
      else cp = ((b0 & 0x07u) << 18) | (b1 << 12) | (b2 << 6) | b3;
      if (!units) {
        q++;
      } else if (cp < 0x10000u) {
        if (dst) {
          VT_CHECK_STS(smem_addr(dst + q), 2);
          dst[q] = be ? bswap16(cp) : (uint16_t)cp;
        }
        q++;
      } else {
        const unsigned s = cp - 0x10000u;
        if (dst) {
          const unsigned h = 0xD800u + (s >> 10), l = 0xDC00u + (s & 0x3FFu);
          VT_CHECK_STS(smem_addr(dst + q), 4);
          dst[q] = be ? bswap16(h) : (uint16_t)h;
          dst[q + 1] = be ? bswap16(l) : (uint16_t)l;
        }
        q += 2;
      }
    }
    pw = cw;
    cw = nw;
  }
  return q;
}

// Characters (or UTF-16 units) starting at positions [lo, lim) of a thread's
// window, for a range of whole valid characters (the valid prefix of a tile
// with an error, an end tile): non-continuation bytes in range, plus one per
// 4-byte lead for units.  SWAR with a lane-range mask per word; it replaced
// the per-byte generic_chars count on the error path (the tile waits for it).
__device__ __noinline__ unsigned swar_count(const Words W, unsigned lo, unsigned lim, bool units) {
  unsigned cnt = 0;
#pragma unroll
  for (int k = 0; k < K8_WPT; k++) {
    const uint32_t x = W.w[k + 1], x2 = x << 1;
    const int s0 = min(max((int)lo - 4 * k, 0), 4), e0 = min(max((int)lim - 4 * k, 0), 4);
    const uint32_t hi_m = e0 >= 4 ? 0xFFFFFFFFu : (1u << (8 * e0)) - 1u;
    const uint32_t m = e0 <= s0 ? 0u : hi_m & ~((1u << (8 * s0)) - 1u);
    cnt += __popc(~(x & ~x2) & H & m);
    if (units) cnt += __popc(x & x2 & (x << 2) & (x << 3) & H & m);
  }
  return cnt;
}

// Predicated 16-bit store at q, q += 2, when (~c | c2) has bit MASK set.
template <uint32_t MASK>
__device__ __forceinline__ void sts16_if_lead(uint32_t& q, uint32_t c, uint32_t c2, uint32_t v) {
  if (VT_CHECKS && ((~c | c2) & MASK)) VT_CHECK_STS(q, 2);
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 d;\n\t"
      "lop3.or.b32 d|p, %1, %2, %3, 0x8A, 0;\n\t"  // (~a | b) & c
#ifdef VT_EXP_PREDOFF
      "{\n\t.reg .pred p2;\n\tsetp.eq.and.u32 p2, %5, 0xFFFFFFFF, p;\n\t"
      "@p2 st.shared.u16 [%5], %4;\n\t}\n\t"
#elif !defined(VT_EXP_NOSTS)
      "@p st.shared.u16 [%5], %4;\n\t"
#endif
      "@p add.u32 %0, %0, 2;\n\t}"
      : "+r"(q)
      : "r"(c), "r"(c2), "n"(MASK), "h"((unsigned short)v), "r"(VT_LANE_ADDR(q)));
}

// The four predicated stores of one word in one asm block (the running
// address stays in one register; the high units move down inside).
#ifndef VT_STS4
#define VT_STS4 0
#endif
#ifndef VT_R2P
#define VT_R2P 1
#endif
__device__ __forceinline__ void sts16x4_if_lead(uint32_t& q, uint32_t c, uint32_t c2, uint32_t u01,
                                                uint32_t u23) {
  if (VT_CHECKS) VT_CHECK_STS(q, 2 * __popc((~c | c2) & 0x80808080u));
  asm volatile(
      "{\n\t.reg .pred p0, p1, p2, p3;\n\t.reg .b32 d0, d1, d2, d3, h1, h3;\n\t"
      "lop3.or.b32 d0|p0, %1, %2, 0x00000080, 0x8A, 0;\n\t"
      "lop3.or.b32 d1|p1, %1, %2, 0x00008000, 0x8A, 0;\n\t"
      "lop3.or.b32 d2|p2, %1, %2, 0x00800000, 0x8A, 0;\n\t"
      "lop3.or.b32 d3|p3, %1, %2, 0x80000000, 0x8A, 0;\n\t"
      "shr.b32 h1, %3, 16;\n\t"
      "shr.b32 h3, %4, 16;\n\t"
      "@p0 st.shared.b16 [%0], %3;\n\t"
      "@p0 add.u32 %0, %0, 2;\n\t"
      "@p1 st.shared.b16 [%0], h1;\n\t"
      "@p1 add.u32 %0, %0, 2;\n\t"
      "@p2 st.shared.b16 [%0], %4;\n\t"
      "@p2 add.u32 %0, %0, 2;\n\t"
      "@p3 st.shared.b16 [%0], h3;\n\t"
      "@p3 add.u32 %0, %0, 2;\n\t}"
      : "+r"(q)
      : "r"(c), "r"(c2), "r"(u01), "r"(u23));
}

// Branch-free decode of one word: lead-attributed byte planes of each
// character's UTF-16 unit (BMP only; words with 4-byte characters take
// emit_word_four).  Predicated 16-bit stores at the running offset q.
template <bool kBE>
__device__ __forceinline__ void emit_word(uint32_t c, uint32_t n, uint32_t& q) {
  const uint32_t n1 = prmt(c, n, 0x4321);  // byte i = b[i+1]
  const uint32_t n2 = prmt(c, n, 0x5432);  // byte i = b[i+2]
  const uint32_t c2 = c << 1;
  const uint32_t ge_e0 = c & c2 & (c << 2);            // bit 7: 3-byte (or 4-byte) lead
  // full-byte lane masks from bit 7 (PRMT sign-replicate selectors 8..B)
  const uint32_t mna = prmt(c, 0, 0xBA98);             // non-ASCII lanes
  const uint32_t m3 = prmt(ge_e0, 0, 0xBA98);
  const uint32_t A = (n1 & m3) | (c & ~m3);            // 3-byte: 2nd byte; 2-byte: lead
  const uint32_t B = (n2 & m3) | (n1 & ~m3);           // last byte of the character
  const uint32_t lom = lop3<0xE2>(B, 0x3F3F3F3Fu, A << 6);       // (a & b) | (c & ~b)
  const uint32_t lo = (c & ~mna) | (lom & mna);
  const uint32_t him = ((A >> 2) & 0x0F0F0F0Fu) | ((c << 4) & 0xF0F0F0F0u & m3);
  const uint32_t hi = him & mna;
  // units of lanes 0,1 and 2,3 (little-endian; UTF-16BE swaps the two bytes)
  const uint32_t u01 = prmt(lo, hi, kBE ? 0x1504 : 0x5140);
  const uint32_t u23 = prmt(lo, hi, kBE ? 0x3726 : 0x7362);
  // lane i starts a character: (~c | c2) bit 8i+7, tested straight into the
  // store predicate (one 3-input LOP3 per lane, no lead plane)
#if VT_R2P
  {
    // the four lead tests as one register-to-predicate move: the clean lead
    // plane (bit 7 of each lane), gathered into bits 1..4 by the high half of
    // one multiply (FMA pipe; the lane bits land on distinct product bits, so
    // no carries), then R2P -- 2 ALU-pipe instructions instead of 4
    const uint32_t lead7 = lop3<0x8A>(c, c2, H);  // (~a | b) & c
    // (bits 1..4: ptxas keeps P0 out of R2P and would test bit 0 separately)
    const uint32_t m = __umulhi(lead7, 0x04081020u);
    if (m & 2u) { sts16(q, u01); q += 2; }
    if (m & 4u) { sts16(q, u01 >> 16); q += 2; }
    if (m & 8u) { sts16(q, u23); q += 2; }
    if (m & 16u) { sts16(q, u23 >> 16); q += 2; }
  }
#elif VT_STS4
  sts16x4_if_lead(q, c, c2, u01, u23);
#else
  sts16_if_lead<0x00000080u>(q, c, c2, u01);
  sts16_if_lead<0x00008000u>(q, c, c2, u01 >> 16);
  sts16_if_lead<0x00800000u>(q, c, c2, u23);
  sts16_if_lead<0x80000000u>(q, c, c2, u23 >> 16);
#endif
}

// Words with 4-byte characters: one unit per lane, like the BMP form.  A
// 4-byte lead's lane writes the high surrogate, and the first continuation
// after it (an "ls lane") writes the low surrogate: 0xDC00 | (cp & 0x3FF) is
// made of the two bytes after that lane exactly like a 3-byte character's
// unit is made of the two bytes after its lead (lo plane), with DC | (b >> 2)
// & 3 as the high byte.  So every lane stores at most one unit (4 predicated
// stores per word, not 8).  `carry4` (bit 7) says the previous word's lane 3
// was a 4-byte lead of this thread; a lead in the thread's last byte has its
// ls lane in the next thread and is finished by emit_tail_ls.
template <bool kBE, bool kNV = false, bool kMasked = false>
__device__ __forceinline__ void emit_word_four(uint32_t c, uint32_t n, uint32_t& q,
                                               uint32_t& carry4, uint32_t KDC, uint32_t range = ~0u) {
  const uint32_t n1 = prmt(c, n, 0x4321);  // byte i = b[i+1]
  const uint32_t n2 = prmt(c, n, 0x5432);  // byte i = b[i+2]
  const uint32_t c2 = c << 1;
  const uint32_t lead7 = ~(c & ~c2) & H;
  const uint32_t ge_e0 = c & c2 & (c << 2);            // bit 7: 3-byte or 4-byte lead
  const uint32_t four7 = ge_e0 & (c << 3) & H;         // 4-byte lead
  const uint32_t ls7 = (four7 << 8) | carry4;          // first continuation after one
  carry4 = four7 >> 24;
  const uint32_t mna = prmt(c, 0, 0xBA98);
  const uint32_t m3 = prmt(ge_e0 | ls7, 0, 0xBA98);    // unit from the two bytes after
  const uint32_t mls = prmt(ls7, 0, 0xBA98);
  const uint32_t A = (n1 & m3) | (c & ~m3);
  const uint32_t B = (n2 & m3) | (n1 & ~m3);
  const uint32_t lom = lop3<0xE2>(B, 0x3F3F3F3Fu, A << 6);       // (a & b) | (c & ~b)
  const uint32_t lo = (c & ~mna) | (lom & mna);
  const uint32_t A2 = A >> 2;
  const uint32_t him = ((A2 & 0x0F0F0F0Fu) | ((c << 4) & 0xF0F0F0F0u & m3)) & mna;
  // (an ls lane is an m3 lane, so A is n1 there: the shift is shared)
  const uint32_t hi_ls = lop3<0xEA>(A2, 0x03030303u, KDC);  // (a & b) | c
  const uint32_t hi = lop3<0xCA>(mls, hi_ls, him);
  uint32_t u01 = prmt(lo, hi, kBE ? 0x1504 : 0x5140), u23 = prmt(lo, hi, kBE ? 0x3726 : 0x7362);
  // 4-byte leads: high surrogate = 0xD7C0 + (cp >> 10)
  const uint32_t m4 = prmt(four7, 0, 0xBA98);
  const uint32_t X = ((n1 << 2) & 0xFCFCFCFCu) | ((n2 >> 4) & 0x03030303u);
  const uint32_t c7 = c & 0x07070707u;
  uint32_t hs01 = prmt(X, c7, 0x5140) + 0xD7C0D7C0u;
  uint32_t hs23 = prmt(X, c7, 0x7362) + 0xD7C0D7C0u;
  if (kBE) {
    hs01 = prmt(hs01, 0, 0x2301);
    hs23 = prmt(hs23, 0, 0x2301);
  }
  u01 = lop3<0xCA>(prmt(m4, 0, 0x1100), hs01, u01);
  u23 = lop3<0xCA>(prmt(m4, 0, 0x3322), hs23, u23);
  // (non-validating: an ls lane stores only if it is a continuation, so the
  // stores match classify_nv's count on any input)
  // (kMasked: only characters starting in the lanes `range` selects -- the
  // valid prefix of a tile with an error, the input part of an end tile)
  const uint32_t st7 = (kNV ? lead7 | (ls7 & c & ~c2) : lead7 | ls7) & (kMasked ? range : ~0u);
#if VT_R2P
  const uint32_t m = __umulhi(st7, 0x04081020u);  // lanes -> bits 1..4, one R2P (see emit_word)
  if (m & 2u) { sts16(q, u01); q += 2; }
  if (m & 4u) { sts16(q, (u01 >> 16)); q += 2; }
  if (m & 8u) { sts16(q, u23); q += 2; }
  if (m & 16u) { sts16(q, (u23 >> 16)); q += 2; }
#else
  if (st7 & 0x00000080u) { sts16(q, u01); q += 2; }
  if (st7 & 0x00008000u) { sts16(q, (u01 >> 16)); q += 2; }
  if (st7 & 0x00800000u) { sts16(q, u23); q += 2; }
  if (st7 & 0x80000000u) { sts16(q, (u23 >> 16)); q += 2; }
#endif
}

// The low surrogate of a 4-byte character whose lead is the thread's last
// byte: its ls lane is byte 0 of the next word n (bytes 1 and 2 of n follow).
template <bool kBE>
__device__ __forceinline__ void emit_tail_ls(uint32_t n, uint32_t q) {
  const uint32_t b2 = (n >> 8) & 0xFFu, b3 = (n >> 16) & 0xFFu;
  const uint32_t u = 0xDC00u | ((b2 & 0x0Fu) << 6) | (b3 & 0x3Fu);
  sts16(q, kBE ? (((u & 0xFFu) << 8) | (u >> 8)) : u);
}

// ---- per-tile front half: load, classify, locate errors, count -------------
struct TileCount {
  Words W;
  long long v0;
  unsigned lo, lim;  // in-input positions [lo, lim) of the thread (clipped at the tile's error)
  bool simple;       // interior tile without error: SWAR emission from W
  bool four;         // the thread has 4-byte characters
  bool ascii;        // interior tile and the thread's 64 bytes are ASCII (emit_ascii_row)
  unsigned cnt;      // units (transcode) or characters of the thread
};

template <bool kTranscode, int NT, class Sync, bool kNV = false>
__device__ __forceinline__ void count_tile(const U8Args& a, unsigned tile, unsigned* red,
                                           unsigned* scan, TileCount& tc, unsigned& off,
                                           unsigned& agg, const uint8_t* pf = nullptr,
                                           unsigned long long* early = nullptr) {
  const unsigned lane = threadIdx.x & 31;
  const long long vt0 = (long long)tile * K8_TILE;  // virtual start of the tile
  // interior: the tile and both halo words lie inside the input.  head < 16, so
  // every tile but the first starts past it; `last_in` is uniform (kernel
  // parameters only), so the test is one compare per tile and the interior
  // path carries no 64-bit range arithmetic (it was ~50 instructions per tile
  // and thread).
  const unsigned long long endv = a.head + a.n;
  const unsigned last_in = endv >= K8_TILE + 4 ? (unsigned)((endv - 4) / K8_TILE) : 0u;  // tiles [1, last_in) are interior
  const bool interior = tile >= 1 && tile < last_in;
  unsigned hi;
  if (pf) {
    // prefetched by the pipeline (an interior tile): pf = 16 bytes before the
    // tile, the tile, 16 bytes behind it, in shared memory
    load_smem_words<K8_WPT>(smem_addr(pf) + 16u + (unsigned)K8_BPT * threadIdx.x, tc.W.w);
    tc.lo = 0;
    hi = K8_BPT;
  } else if (interior) {
    load_lane_words<K8_WPT>(a.base + (size_t)tile * K8_TILE + (size_t)(K8_BPT * threadIdx.x), lane, tc.W.w);
    tc.lo = 0;
    hi = K8_BPT;
  } else {
    tc.v0 = vt0 + (long long)K8_BPT * threadIdx.x;
    const Src src{a.base, a.head, a.n};
    load_edge(src, tc.v0, tc.W.w);
    const long long s = (long long)a.head - tc.v0, e = (long long)(a.head + a.n) - tc.v0;
    tc.lo = (unsigned)max(0LL, min((long long)K8_BPT, s));
    hi = (unsigned)max((long long)tc.lo, min((long long)K8_BPT, e));
  }
#ifdef VT_PHASES
  {  // sub-phase probe: wait for the loads
    uint32_t z = 0;
#pragma unroll
    for (int k = 0; k < K8_WPT + 2; k++) z ^= tc.W.w[k];
    if (z == 0x9E3779B9u) asm volatile("trap;");
    const long long t = clock64();
    if (threadIdx.x == 0) atomicAdd(&g_phase_sub[0], (unsigned long long)t);
  }
#endif
  const ClassOut co = kNV ? classify_nv(tc.W) : classify(tc.W);
#ifdef VT_PHASES
  {
    const long long t = clock64() + (co.units == 0x7FFFFFFF ? 1 : 0);
    if (threadIdx.x == 0) atomicAdd(&g_phase_sub[1], (unsigned long long)t);
  }
#endif
  tc.four = co.four;
  tc.lim = hi;
  // all 64 bytes ASCII: no continuation byte and no 4-byte lead in the thread
  // (then any other lead would need its continuation inside the thread, or
  // the structure check fails) and the last byte is not a lead whose
  // continuation belongs to the next thread
  tc.ascii = !kNV && (interior || pf) && co.chars == K8_BPT && co.units == K8_BPT &&
             (tc.W.w[K8_WPT] & 0x80000000u) == 0;
  unsigned my_err = kNone;
  if (co.viol) {
    const Words tmp = tc.W;  // (a copy: tc.W itself stays in registers)
    const unsigned er = first_error_w(tmp, tc.lo, hi);
    if (er != kNone) my_err = K8_BPT * threadIdx.x + er;
  }
  {
    // fast path: one scan; bits kErrShift..31 count the threads that found an error
    // (NT << kErrShift <= 2^31: no wrap; counts stay below 2^kErrShift)
    constexpr int kErrShift = NT <= 256 ? 23 : 22;  // NT << kErrShift <= 2^31
    static_assert(NT <= 512 && 2 * K8_TILE < (1 << kErrShift), "packed scan fields");
    // (end tiles: the zeros outside the input counted as one ASCII character each)
    tc.cnt = (kTranscode ? co.units : co.chars) - (K8_BPT - (hi - tc.lo));
    unsigned total;
    if (early)
      publish_total_early<NT>(my_err == kNone ? tc.cnt : (1u << kErrShift), early, &a.status[tile],
                              tile == 0 ? kFlagPre : kFlagAgg, a.epoch, kErrShift);
#if VT_SCAN1
    off = block_excl_scan1<NT, Sync>(my_err == kNone ? tc.cnt : (1u << kErrShift), scan, total);
#else
    off = block_excl_scan<NT, Sync, false>(my_err == kNone ? tc.cnt : (1u << kErrShift), scan, total);
#endif
    if ((total >> kErrShift) == 0) {
      tc.simple = true;
      agg = total;
      return;
    }
  }
  // ends of the input, or an error in the tile: exact, clipped counts
  const unsigned tile_err = block_min<NT, Sync>(my_err, red);
  tc.simple = false;
  if (tile_err != kNone) {
    const unsigned start = K8_BPT * threadIdx.x;
    tc.lim = max(tc.lo, min(hi, tile_err <= start ? 0u : tile_err - start));
    if (threadIdx.x == 0) {
      const unsigned long long pos = (unsigned long long)(vt0 + tile_err) - a.head;
      atomicMin(&a.ctl->err, pos);
      VT_TR_MIN(1);
    }
  }
  tc.cnt = swar_count(tc.W, tc.lo, tc.lim, kTranscode);
  off = block_excl_scan<NT, Sync, false>(tc.cnt, scan, agg);
}

// ---- per-tile back half: decode into the staging buffer -----------------------
// A warp whose 2 KiB row is all ASCII.  Every lane then writes exactly 128
// bytes, so the lanes' staging addresses are 128 bytes apart: all 32 in one
// bank, and the per-word stores of the general path conflict 32-way (measured:
// pure ASCII ran at 4.0 ms per GiB against 0.8 for mixed text).  Here lane t
// handles its words in the order t, t+1, ... (mod 16) -- re-read from global
// memory (an L1 hit), since registers cannot be indexed by lane -- which
// spreads the lanes of one store over 16 bank pairs.  Warp-uniform: the row's
// alignment in the staging buffer is the same for every lane.
template <bool kBE>
__device__ __forceinline__ void emit_ascii_row(const U8Args& a, unsigned tile, uint16_t* stage,
                                               unsigned off) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t* p = reinterpret_cast<const uint32_t*>(a.base + (size_t)tile * K8_TILE +
                                                        (size_t)(K8_BPT * threadIdx.x));
  const uint32_t qb = smem_addr(stage) + 2u * off;
  const bool aligned4 = (qb & 2u) == 0;  // (same for every lane: off = row start + 64 * lane)
#pragma unroll 4
  for (unsigned k = 0; k < (unsigned)K8_WPT; k++) {
    const unsigned j = (k + lane) & (K8_WPT - 1);
    const uint32_t x = __ldg(p + j);
    const uint32_t u01 = prmt(x, 0, kBE ? 0x1404 : 0x4140), u23 = prmt(x, 0, kBE ? 0x3424 : 0x4342);
    const uint32_t q = qb + 8u * j;
    if (aligned4) {
      VT_CHECK_STS(q, 8);
      asm volatile("st.shared.u32 [%0], %1;\n\tst.shared.u32 [%0+4], %2;" ::"r"(q), "r"(u01), "r"(u23));
    } else {
      sts16(q, u01);
      sts16(q + 2, u01 >> 16);
      sts16(q + 4, u23);
      sts16(q + 6, u23 >> 16);
    }
  }
}

template <bool kBE, bool kNV, class Mid>
__device__ __forceinline__ void emit_tile(const U8Args& a, const TileCount& tc, uint16_t* stage,
                                          unsigned off, unsigned tile, Mid&& mid) {
  if (tc.simple && __all_sync(0xffffffffu, tc.ascii)) {
    emit_ascii_row<kBE>(a, tile, stage, off);
    mid();
    return;
  }
  if (tc.simple) {
    // (tc.lo > 0 only for the first thread of a call: the zeros before the
    // input are decoded too and land in the pad before the staging buffer)
    uint32_t q = smem_addr(stage) + 2u * off - 2u * tc.lo;
    // warp-uniform choice (the 4-byte-capable form handles every word): a
    // per-thread choice would run both forms in mixed warps
    if (!__any_sync(0xffffffffu, tc.four)) {
#pragma unroll
      for (int k = 1; k <= K8_WPT; k++) {
        if (k == VT_GRAB_AT_U8 + 1) mid();
        emit_word<kBE>(tc.W.w[k], tc.W.w[k + 1], q);
      }
      if (VT_GRAB_AT_U8 >= K8_WPT) mid();
    } else {
      uint32_t carry4 = 0;  // a lead in the previous thread finishes its own pair
      uint32_t KDC = 0xDCDCDCDCu;  // in a register: "(v & imm) | KDC" is one LOP3
      asm volatile("" : "+r"(KDC));
#pragma unroll
      for (int k = 1; k <= K8_WPT; k++) {
        if (k == VT_GRAB_AT_U8 + 1) mid();
        emit_word_four<kBE, kNV>(tc.W.w[k], tc.W.w[k + 1], q, carry4, KDC);
      }
      if (VT_GRAB_AT_U8 >= K8_WPT) mid();
      // (non-validating: only if the byte after the lead is a continuation)
      if (carry4 && (!kNV || (tc.W.w[K8_WPT + 1] & 0xC0u) == 0x80u))
        emit_tail_ls<kBE>(tc.W.w[K8_WPT + 1], q);
    }
  } else {
    // a tile with an error: the same SWAR decode (4-byte-capable form), its
    // stores limited to the characters starting in [lo, lim) -- whole valid
    // characters, the count swar_count gave (the per-byte generic path this
    // replaced kept the whole tile waiting ~20 us)
    mid();
    uint32_t q = smem_addr(stage) + 2u * off;
    uint32_t carry4 = 0, KDC = 0xDCDCDCDCu;
    asm volatile("" : "+r"(KDC));
#pragma unroll
    for (int k = 1; k <= K8_WPT; k++) {
      const int s0 = min(max((int)tc.lo - 4 * (k - 1), 0), 4), e0 = min(max((int)tc.lim - 4 * (k - 1), 0), 4);
      const uint32_t hi_m = e0 >= 4 ? 0xFFFFFFFFu : (1u << (8 * e0)) - 1u;
      const uint32_t m = e0 <= s0 ? 0u : hi_m & ~((1u << (8 * s0)) - 1u);
      emit_word_four<kBE, kNV, true>(tc.W.w[k], tc.W.w[k + 1], q, carry4, KDC, m);
    }
    // (a 4-byte lead in the last byte finishes its pair only if it is in range)
    if (carry4 && tc.lim >= (unsigned)K8_BPT) emit_tail_ls<kBE>(tc.W.w[K8_WPT + 1], q);
  }
}

#ifndef VT_NSTAGE8
#define VT_NSTAGE8 1
#endif

template <bool kBE, bool kNV = false>
struct Utf8Codec {
  using Args = U8Args;
  using TileCount = vt::TileCount;
  static constexpr int kTileElems = K8_TILE;
  static constexpr int kStageBytes = 2 * K8_TILE;
  static constexpr int kNStage = VT_NSTAGE8;
  static constexpr int kOutBytes = 2;
  // input prefetch (vt_pipeline.cuh, VT_PREFETCH): a tile with 16 readable bytes
  // on either side, copied as [tile start - 16, tile end + 16)
  static constexpr int kPrefetchBytes = VT_PREFETCH ? K8_TILE + 32 : 0;
  __device__ __forceinline__ static bool prefetchable(const Args& a, unsigned t) {
    return t >= 1 && (unsigned long long)(t + 1) * K8_TILE + 16 <= a.head + a.n;
  }
  __device__ __forceinline__ static const uint8_t* prefetch_src(const Args& a, unsigned t) {
    return a.base + (size_t)t * K8_TILE - 16;
  }
  template <bool kTranscode, int NT, class Sync>
  __device__ __forceinline__ static void count(const Args& a, unsigned tile, unsigned* red,
                                               unsigned* scan, TileCount& tc, unsigned& off,
                                               unsigned& agg, const uint8_t* pf = nullptr,
                                               unsigned long long* early = nullptr) {
    count_tile<kTranscode, NT, Sync, kNV>(a, tile, red, scan, tc, off, agg, pf, early);
  }
  template <class Mid>
  __device__ __forceinline__ static void emit(const Args& a, const TileCount& tc, uint8_t* stage,
                                              unsigned off, unsigned tile, Mid&& mid) {
    emit_tile<kBE, kNV>(a, tc, reinterpret_cast<uint16_t*>(stage), off, tile, mid);
  }
};


// ---- validation / lengths without barriers ----------------------------------------
// Validation needs no offsets, so no block scan: each warp takes 2 KiB rows
// (64 bytes per lane, the same loads and classify as the transcode) in grid
// stride, keeps its count in registers and records the row's count (one REDUX)
// for the rare error case.  The only atomics are per error and per CTA.  The
// last CTA finalises: without an error the total is the answer; with one, the
// rows before the error row (all valid) are summed from row_counts and the error
// row is recounted up to the error.  kUnits counts UTF-16 units instead of code
// points (the length entry points).
constexpr int K8_ROW = 32 * K8_BPT;  // bytes per warp row

template <bool kUnits>
__global__ void __launch_bounds__(256, 4) utf8_validate_rows_kernel(U8Args a) {
  unsigned* const row_counts = a.rows;
  if (a.skip) {
    // streaming validator: the first *skip bytes completed the previous
    // chunk's trailing character (k_stream.cu) and are not part of this scan
    const unsigned s = *a.skip;
    if (s == kSkipAll) {
      a.n = 0;
    } else {
      a.head += s;
      a.n -= s;
    }
  }
  __shared__ unsigned long long warp_tot[8];
  __shared__ bool last;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  const long long head = (long long)a.head, end = (long long)(a.head + a.n);
  const unsigned long long nrows = (unsigned long long)(end + K8_ROW - 1) / K8_ROW;
  const Src src{a.base, a.head, a.n};
  unsigned long long total = 0;
  unsigned wtot = 0;  // this warp's running total (rows so far)
  if (threadIdx.x == 0) VT_TR_MIN(8);
  // Stop behind a known error (warp-uniform).  The error word is loaded at the
  // top of every row and tested at the top of the next one, so the check adds
  // no latency and a warp runs at most one row past a found error.
  unsigned long long e_prev = kNoError;
  // rows [1, last_in) lie inside the input together with both halo words (head < 16)
  const unsigned long long last_in = end >= K8_ROW + 4 ? (unsigned long long)(end - 4) / K8_ROW : 0ull;
  for (unsigned long long row = gw; row < nrows; row += nwarps) {
    const long long r0 = (long long)row * K8_ROW;
    if (e_prev != kNoError && (long long)e_prev + head < r0) break;
    const unsigned long long e_next = lane == 0 ? load_relaxed(&a.ctl->err) : 0ull;
    const long long v0 = r0 + (long long)K8_BPT * lane;
    // interior rows (all but the first and the last one or two): one uniform
    // compare, no 64-bit range arithmetic (as count_tile)
    const bool interior = row >= 1 && row < last_in;
    Words W;
    if (interior) {
      load_lane_words<K8_WPT>(a.base + v0, lane, W.w);
    } else {
      load_edge(src, v0, W.w);
    }
    const ClassOut co = classify(W);
    unsigned cnt;
    if (!co.viol) {
      if (interior) {
        cnt = kUnits ? co.units : co.chars;
      } else {
        const unsigned lo = (unsigned)max(0LL, min((long long)K8_BPT, head - v0));
        const unsigned hi = (unsigned)max((long long)lo, min((long long)K8_BPT, end - v0));
        cnt = (kUnits ? co.units : co.chars) - (K8_BPT - (hi - lo));  // minus the zeros outside
      }
    } else {
      const unsigned lo = (unsigned)max(0LL, min((long long)K8_BPT, head - v0));
      const unsigned hi = (unsigned)max((long long)lo, min((long long)K8_BPT, end - v0));
      const Words tmp = W;
      const unsigned er = first_error_w(tmp, lo, hi);
      if (er != kNone) {
        atomicMin(&a.ctl->err, (unsigned long long)(v0 + er - head));
        VT_TR_MIN(1);
      }
      // (exact only up to the error, which is all the finalize uses of a row
      // that holds one)
      cnt = swar_count(W, lo, er != kNone ? er : hi, kUnits);
    }
    total += cnt;
    const unsigned rc = __reduce_add_sync(0xffffffffu, cnt);
    wtot += rc;
    if (lane == 0) row_counts[row] = wtot;
    e_prev = __shfl_sync(0xffffffffu, e_next, 0);
  }
  // per-CTA total, one atomic
  if (lane == 0) VT_TR_MAX(9);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  if (lane == 0) warp_tot[wib] = total;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (unsigned w = 0; w < blockDim.x / 32; w++) t += warp_tot[w];
    if (t) atomicAdd(&a.ctl->count, t);
    __threadfence();
    last = atomicAdd(&a.ctl->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) VT_TR_MAX(10);
  __threadfence();
  const unsigned long long e = load_relaxed(&a.ctl->err);
  unsigned long long written = load_relaxed(&a.ctl->count);
  if (e != kNoError) {
    // valid prefix: rows before the error row, then the error row up to e
    const unsigned long long erow = (e + a.head) / K8_ROW;
    unsigned long long t = prefix_rows(row_counts, erow, nwarps);
    if (wib == 0) {
      const long long v0 = (long long)erow * K8_ROW + (long long)K8_BPT * lane;
      const long long stop = (long long)e + head;
      const unsigned lo = (unsigned)max(0LL, min((long long)K8_BPT, head - v0));
      const unsigned lim = (unsigned)max((long long)lo, min((long long)K8_BPT, stop - v0));
      Words tmp;
      load_edge(src, v0, tmp.w);
      t += swar_count(tmp, lo, lim, kUnits);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) warp_tot[wib] = t;
    __syncthreads();
    written = 0;
    for (unsigned w = 0; w < blockDim.x / 32; w++) written += warp_tot[w];
  }
  if (threadIdx.x == 0) {
    vt_result r;
    r.written = written;
    r.consumed = e == kNoError ? a.n : e;
    r.error_at = e == kNoError ? -1 : (long long)e;
    *a.res = r;
    a.ctl->tile_counter = 0;
    a.ctl->count = 0;
    a.ctl->err = kNoError;
    __threadfence();
    a.ctl->done = 0;
    VT_TR_MAX(11);
  }
}

unsigned rows_utf8(unsigned long long head, unsigned long long n) {
  return (unsigned)((head + n + K8_ROW - 1) / K8_ROW);
}

#ifndef VT_K8_MINB
#define VT_K8_MINB 4
#endif
// UTF-8 -> UTF-16LE (kBE = false) or UTF-16BE (kBE = true)
// (kNV: the non-validating variant, LE output only)
template <bool kBE, bool kNV = false>
__global__ void __launch_bounds__(kPipeBlock, VT_K8_MINB) utf8_transcode_kernel(U8Args a) {
  extern __shared__ __align__(16) uint8_t k8_dyn_smem[];
  transcode_body<Utf8Codec<kBE, kNV>>(
      a, *reinterpret_cast<PipeSmem<Utf8Codec<kBE, kNV>>*>(k8_dyn_smem));
}

static int set_smem_attr() {
  // (no carveout preference: forcing the largest shared-memory carveout
  // leaves too little L1 for the input loads -- measured 1.37 vs 1.32 ms on
  // cfg3)
  for (const void* f : {(const void*)utf8_transcode_kernel<false>, (const void*)utf8_transcode_kernel<true>,
                        (const void*)utf8_transcode_kernel<false, true>}) {
    const int rc = (int)cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sizeof(PipeSmem<Utf8Codec<false>>));
    if (rc) return rc;
#ifdef VT_CARVEOUT
    // (A/B: preferred shared-memory carveout in percent; more than 4 CTAs per SM
    // need more shared memory than the driver's default choice provides)
    if (cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, VT_CARVEOUT)) return 1;
#endif
  }
  return 0;
}

int launch_utf8(const U8Args& a, int mode, int grid, cudaStream_t s) {
  static const int attr_rc = set_smem_attr();
  if (attr_rc) return attr_rc;
  if (mode == kModeTranscode)
    utf8_transcode_kernel<false><<<grid, kPipeBlock, sizeof(PipeSmem<Utf8Codec<false>>), s>>>(a);
  else if (mode == kModeTranscodeBE)
    utf8_transcode_kernel<true><<<grid, kPipeBlock, sizeof(PipeSmem<Utf8Codec<true>>), s>>>(a);
  else if (mode == kModeTranscodeNV)
    utf8_transcode_kernel<false, true>
        <<<grid, kPipeBlock, sizeof(PipeSmem<Utf8Codec<false, true>>), s>>>(a);
  else if (mode == kModeLength)
    utf8_validate_rows_kernel<true><<<grid, 256, 0, s>>>(a);
  else
    utf8_validate_rows_kernel<false><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

int occupancy_utf8(bool transcode) {
  int n = 0;
  if (transcode) {
    if (set_smem_attr()) return 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf8_transcode_kernel<false>, kPipeBlock,
                                                  sizeof(PipeSmem<Utf8Codec<false>>));
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf8_validate_rows_kernel<false>, 256, 0);
  }
  return n;
}

#ifdef VT_TRACE
// reads and re-arms this translation unit's trace stamps (mins start at ~0)
int read_trace8(unsigned long long* out16) {
  int rc = (int)cudaMemcpyFromSymbol(out16, g_trace, sizeof(g_trace));
  unsigned long long init[16];
  for (int i = 0; i < 16; i++) init[i] = (i == 0 || i == 1 || i == 8) ? ~0ull : 0ull;
  if (!rc) rc = (int)cudaMemcpyToSymbol(g_trace, init, sizeof(init));
  return rc;
}
#endif

#ifdef VT_PHASES
int read_phases(unsigned long long* out8) {
  int rc = (int)cudaMemcpyFromSymbol(out8, g_phase, sizeof(g_phase));
  if (!rc) rc = (int)cudaMemcpyFromSymbol(out8 + 8, g_phase_sub, sizeof(g_phase_sub));
  if (!rc) rc = (int)cudaMemcpyFromSymbol(out8 + 12, g_phase_lb, sizeof(g_phase_lb));
  return rc;
}
#endif

unsigned tiles_utf8(unsigned long long head, unsigned long long n) {
  const unsigned long long t = (head + n + K8_TILE - 1) / K8_TILE;
  return (unsigned)(t ? t : 1);
}

}  // namespace vt

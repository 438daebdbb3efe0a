// k_utf16.cu -- UTF-16LE -> UTF-8 transcoding (always validating) and UTF-16
// validation / code-point counting on sm_100a.
//
// Replaces the reference's 8-unit register dispatch with its pack tables and
// scalar surrogate fallback (proj/src/utf16_to_utf8.cpp:12-107) and the
// surrogate scan of proj/src/validation.cpp:51-77.  No tables: a unit's UTF-8
// length is a function of the unit and its neighbours (<0x80: 1, <0x800: 2,
// high surrogate followed by a low one: 4, that low one: 0, other BMP: 3), and
// the first error is the first unit failing the local pairing rule (SURVEY.md
// 8(a) fact C) -- exactly where the scalar decoder (proj/src/codec_core.cpp:
// 74-83,106-125) stops.
//
// Same tile pipeline as k_utf8.cu (vt_pipeline.cuh).  Per 8192-unit tile each
// thread owns 32 consecutive units (16 words of two units):
//   A. SWAR over 16-bit lanes: high/low-surrogate planes, the pairing check
//      against the neighbouring units, and the byte count (lengths summed
//      in 16-bit lane counters);
//   B. a thread that sees an error finds its exact first failing unit; tiles
//      with an error, and the tiles at the ends of the input, take a masked
//      per-unit path;
//   C. encode: per unit the UTF-8 bytes are assembled in one register
//      (bit fields spread by shifts, lead marks or'ed in) and stored byte-wise
//      into the shared-memory staging buffer.
#include "vt_kernels.h"
#include "vt_pipeline.cuh"
#include "vt_swar.cuh"

namespace vt {

constexpr int K16_WPT = 16;                              // words (2 units) per thread
constexpr int K16_UPT = 2 * K16_WPT;                     // units per thread
constexpr int K16_TILE = kComputeThreads * K16_UPT;      // units per tile
constexpr unsigned kNone16 = 0xFFFFFFFFu;
constexpr uint32_t H16 = 0x80008000u;

// bit 15 of each 16-bit lane: v != 0, for v with bits only in 10..15 / 26..31
__device__ __forceinline__ uint32_t nz_hi6(uint32_t v) {
  return ((v >> 1) + 0x7E007E00u) & H16;
}

// Per-lane unsigned compares u >= 0x80 / u >= 0x800 (bit 15 of each lane):
// the low 15 bits plus a bias carry into bit 15, or bit 15 is already set.
__device__ __forceinline__ uint32_t ge80_16(uint32_t x, uint32_t x15) {
  return lop3<0xA8>(x15 + 0x7F807F80u, x, H16);  // (a | b) & c
}
__device__ __forceinline__ uint32_t ge800_16(uint32_t x, uint32_t x15) {
  return lop3<0xA8>(x15 + 0x78007800u, x, H16);
}
// D800..DFFF lanes (bit 15)
__device__ __forceinline__ uint32_t sur16(uint32_t x) {
  return ~nz_hi6((x & 0xF800F800u) ^ 0xD800D800u) & H16;
}

struct Src16 {
  const uint16_t* base;
  unsigned long long head, n;
  bool be;  // UTF-16BE input: bytes of each unit swapped on load
};

struct Words16 {
  uint32_t w[K16_WPT + 2];  // w[0] = previous word, w[1..16] own, w[17] next
};

// One word straddling an end of the input, unit by unit (rare; out of line).
__device__ __noinline__ uint32_t straddle_word16(Src16 a, long long p) {
  const long long lo = (long long)a.head, hi = (long long)(a.head + a.n);
  uint32_t x = 0;
  for (int b = 0; b < 2; b++) {
    if (p + b >= lo && p + b < hi) {
      uint32_t u = a.base[p + b];
      if (a.be) u = ((u & 0xFFu) << 8) | (u >> 8);
      x |= u << (16 * b);
    }
  }
  return x;
}

// A thread's window at the ends of the input, units outside [head, head + n)
// as 0x0000 (as load_edge in k_utf8.cu): whole words at once, the at most two
// straddling words unit by unit.  Zeros are ASCII, so an end tile takes the
// SWAR path (counts minus the zeros); a surrogate cut from its partner by an
// end still shows as a pairing error.
template <bool kBE>
__device__ __forceinline__ void load_edge16(Src16 a, long long v0, uint32_t* w) {
  constexpr int NW = K16_WPT + 2;
  const long long s0 = v0 - 2;  // virtual unit position of word 0
  const long long lo = (long long)a.head, hi = (long long)(a.head + a.n);
  const int kf = (int)max(0LL, min((long long)NW, (lo - s0 + 1) >> 1));  // words [kf, kl)
  const int kl = (int)max((long long)kf, min((long long)NW, (hi - s0) >> 1));  // are inside
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(a.base + s0);
#pragma unroll
  for (int k = 0; k < NW; k++) {
    const uint32_t x = (k >= kf && k < kl) ? __ldg(wp + k) : 0u;
    w[k] = kBE ? prmt(x, 0, 0x2301) : x;
  }
#pragma unroll
  for (int k = 0; k < NW; k++)
    if ((k == kf - 1 || k == kl) && s0 + 2 * k + 2 > lo && s0 + 2 * k < hi)
      w[k] = straddle_word16(a, s0 + 2 * k);
}

__device__ __forceinline__ bool is_hi(unsigned u) { return (u & 0xFC00u) == 0xD800u; }
__device__ __forceinline__ bool is_lo(unsigned u) { return (u & 0xFC00u) == 0xDC00u; }

// UTF-8 bytes written for the unit u (little-endian in the result) and their
// number; `pv` is the unit before it.  A surrogate pair's 4 bytes are split
// 2 + 2 between its halves (see emit_word16_v3), so each unit writes 1-3
// bytes and a pair may straddle threads and tiles.
__device__ __forceinline__ uint32_t encode_unit(unsigned u, unsigned pv, unsigned& len) {
  if (u < 0x80u) {
    len = 1;
    return u;
  }
  if (u < 0x800u) {
    len = 2;
    return 0x80C0u | (u >> 6) | ((u & 0x3Fu) << 8);
  }
  if (is_hi(u)) {  // code point bits 10..20: w = (u & 0x3FF) + 0x40
    const unsigned w = (u & 0x3FFu) + 0x40u;
    len = 2;
    return (0xF0u | (w >> 8)) | ((0x80u | ((w >> 2) & 0x3Fu)) << 8);
  }
  if (is_lo(u)) {  // (w & 3) == (pv & 3)
    len = 2;
    return (0x80u | ((pv & 3u) << 4) | ((u >> 6) & 0xFu)) | ((0x80u | (u & 0x3Fu)) << 8);
  }
  len = 3;
  return 0x8080E0u | (u >> 12) | (((u >> 6) & 0x3Fu) << 8) | ((u & 0x3Fu) << 16);
}

// Exact path (tiles with an error) on a copy of the caller's window, one loop
// step per word (both units) with the neighbouring words in registers, so
// the hot path keeps its words in registers and nothing is reloaded.
// first_error16: the smallest unit in [lo, hi) failing the pairing rule C of
// SURVEY.md 8(a) (a low surrogate not after a high one, a high one not before
// a low one); generic_units: bytes (or code points) of units [lo, lim), with
// `dst` also their UTF-8 bytes.
__device__ __noinline__ unsigned first_error16(const Words16& W, unsigned lo, unsigned hi) {
  uint32_t pw = W.w[0], cw = W.w[1];
  for (int k = 0; k < K16_WPT; k++) {
    const uint32_t nw = W.w[k + 2];
    const unsigned u0 = cw & 0xFFFFu, u1 = cw >> 16;
    const unsigned i = 2 * k;
    if (i >= lo && i < hi &&
        ((is_lo(u0) && !is_hi(pw >> 16)) || (is_hi(u0) && !is_lo(u1))))
      return i;
    if (i + 1 >= lo && i + 1 < hi &&
        ((is_lo(u1) && !is_hi(u0)) || (is_hi(u1) && !is_lo(nw & 0xFFFFu))))
      return i + 1;
    pw = cw;
    cw = nw;
  }
  return kNone16;
}

__device__ __noinline__ unsigned generic_units(const Words16& W, unsigned lo, unsigned lim,
                                               bool bytes, uint8_t* dst) {
  unsigned q = 0;
  uint32_t pw = W.w[0];
  for (int k = 0; k < K16_WPT; k++) {
    const uint32_t cw = W.w[k + 1];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const unsigned i = 2 * k + h;
      if (i < lo || i >= lim) continue;
      const unsigned u = h ? cw >> 16 : cw & 0xFFFFu;
      const unsigned pv = h ? cw & 0xFFFFu : pw >> 16;
      if (!bytes) {
        q += is_lo(u) ? 0u : 1u;
        continue;
      }
      unsigned len;
      const uint32_t p = encode_unit(u, pv, len);
      if (dst) {
        VT_CHECK_STS(smem_addr(dst + q), len);
        for (unsigned b = 0; b < len; b++) dst[q + b] = (uint8_t)(p >> (8 * b));
      }
      q += len;
    }
    pw = cw;
  }
  return q;
}

// UTF-8 bytes (or code points) of units [lo, lim) of a thread's window, for a
// range of whole valid characters (bytes per unit as in classify16: 1 +
// [>= 0x80] + [>= 0x800] - [surrogate]; code points: units minus low
// surrogates).  SWAR with a lane-range mask per word, for the error path.
__device__ __noinline__ unsigned swar_count16(const Words16 W, unsigned lo, unsigned lim, bool bytes) {
  unsigned cnt = 0;
#pragma unroll
  for (int k = 0; k < K16_WPT; k++) {
    const uint32_t x = W.w[k + 1];
    const unsigned i = 2 * k;
    const uint32_t m = (i >= lo && i < lim ? 0x00008000u : 0u) | (i + 1 >= lo && i + 1 < lim ? 0x80000000u : 0u);
    const uint32_t x15 = x & 0x7FFF7FFFu;
    const uint32_t sr = sur16(x);
    if (bytes)
      cnt += __popc(m) + __popc(ge80_16(x, x15) & m) + __popc(ge800_16(x, x15) & m) - __popc(sr & m);
    else
      cnt += __popc(m) - __popc(sr & (x << 5) & m);
  }
  return cnt;
}

struct TileCount16 {
  Words16 W;
  long long v0;
  unsigned lo, lim;
  bool simple;
  bool ascii;  // interior tile and the thread's 32 units are ASCII (emit_ascii_row16)
  unsigned cnt;
};

struct Class16 {
  unsigned bytes, chars;
  bool err;
};

// Phase A over the thread's 32 units: pairing check and counts, four units per
// operation on the low-byte / high-byte planes of each pair of words
// (vt_swar.cuh; the kernel is bound by the ALU pipe, and the 16-bit-lane form
// this replaces spent twice the instructions per unit).
__device__ __forceinline__ Class16 classify16(const Words16& W) {
  using namespace swar;
  uint32_t k58 = 0x58585858u;
  asm volatile("" : "+r"(k58));  // (a & imm) ^ k58 is one LOP3 only with k58 in a register
  Count16 c;
  c.err = c.acc = c.nsur = c.nlo = 0;
  c.hp = hs_plane(hi_plane(0u, W.w[0]), k58);  // (lane 3: the unit before the range)
#pragma unroll
  for (int g = 0; g < K16_WPT / 2; g++) {
    const uint32_t x0 = W.w[1 + 2 * g], x1 = W.w[2 + 2 * g];
    count_group16<true>(lo_plane(x0, x1), hi_plane(x0, x1), k58, c);
  }
  // the unit after the range closes the last pair
  count_group16<false>(lo_plane(W.w[K16_WPT + 1], 0u), hi_plane(W.w[K16_WPT + 1], 0u), k58, c);
  Class16 r;
  // bytes per unit: 1 + [u >= 0x80] + [u >= 0x800] - [surrogate] (2 + 2 per pair)
  r.bytes = K16_UPT + lane_sum(c.acc) - lane_sum(c.nsur);
  r.chars = K16_UPT - lane_sum(c.nlo);
  r.err = c.err != 0;
  return r;
}

template <bool kTranscode, int NT, class Sync, bool kBE = false>
__device__ __forceinline__ void count_tile16(const U16Args& a, unsigned tile, unsigned* red,
                                             unsigned* scan, TileCount16& tc, unsigned& off,
                                             unsigned& agg, unsigned long long* early = nullptr) {
  const unsigned lane = threadIdx.x & 31;
  const long long vt0 = (long long)tile * K16_TILE;
  // interior tiles (all but the first and the last one or two): one uniform
  // compare, no 64-bit range arithmetic (as count_tile in k_utf8.cu)
  const unsigned long long endv = a.head + a.n;
  const unsigned last_in = endv >= K16_TILE + 2 ? (unsigned)((endv - 2) / K16_TILE) : 0u;
  const bool interior = tile >= 1 && tile < last_in;
  unsigned hi;
  if (interior) {
    load_lane_words<K16_WPT>(reinterpret_cast<const uint8_t*>(a.base) + (size_t)tile * (2 * K16_TILE) +
                                 (size_t)(2 * K16_UPT * threadIdx.x),
                             lane, tc.W.w);
    if (kBE) {
#pragma unroll
      for (int k = 0; k < K16_WPT + 2; k++) tc.W.w[k] = prmt(tc.W.w[k], 0, 0x2301);
    }
    tc.lo = 0;
    hi = K16_UPT;
  } else {
    tc.v0 = vt0 + (long long)K16_UPT * threadIdx.x;
    const Src16 src{a.base, a.head, a.n, kBE};
    load_edge16<kBE>(src, tc.v0, tc.W.w);
    const long long s = (long long)a.head - tc.v0, e = (long long)(a.head + a.n) - tc.v0;
    tc.lo = (unsigned)max(0LL, min((long long)K16_UPT, s));
    hi = (unsigned)max((long long)tc.lo, min((long long)K16_UPT, e));
  }
  tc.lim = hi;
  const Class16 c = classify16(tc.W);
  // (every unit >= 0x80 adds at least one byte: 32 bytes <=> 32 ASCII units)
  tc.ascii = kTranscode && interior && c.bytes == K16_UPT;
  unsigned my_err = kNone16;
  if (c.err) {
    const Words16 tmp = tc.W;  // (a copy: tc.W itself stays in registers)
    const unsigned er = first_error16(tmp, tc.lo, hi);
    if (er != kNone16) my_err = K16_UPT * threadIdx.x + er;
  }
  {
    constexpr int kErrShift = NT <= 256 ? 23 : 22;  // NT << kErrShift <= 2^31
    static_assert(NT <= 512 && 4 * K16_TILE < (1 << kErrShift), "packed scan fields");
    // (end tiles: the zeros outside the input counted as one ASCII unit each)
    tc.cnt = (kTranscode ? c.bytes : c.chars) - (K16_UPT - (hi - tc.lo));
    unsigned total;
    if (early)
      publish_total_early<NT>(my_err == kNone16 ? tc.cnt : (1u << kErrShift), early, &a.status[tile],
                              tile == 0 ? kFlagPre : kFlagAgg, a.epoch, kErrShift);
#if VT_SCAN1
    off = block_excl_scan1<NT, Sync>(my_err == kNone16 ? tc.cnt : (1u << kErrShift), scan, total);
#else
    off = block_excl_scan<NT, Sync, false>(my_err == kNone16 ? tc.cnt : (1u << kErrShift), scan, total);
#endif
    if ((total >> kErrShift) == 0) {
      tc.simple = true;
      agg = total;
      return;
    }
  }
  const unsigned tile_err = block_min<NT, Sync>(my_err, red);
  tc.simple = false;
  if (tile_err != kNone16) {
    const unsigned start = K16_UPT * threadIdx.x;
    tc.lim = max(tc.lo, min(hi, tile_err <= start ? 0u : tile_err - start));
    if (threadIdx.x == 0) {
      const unsigned long long pos = (unsigned long long)(vt0 + tile_err) - a.head;
      atomicMin(&a.ctl->err, pos);
      VT_TR_MIN(1);
    }
  }
  tc.cnt = swar_count16(tc.W, tc.lo, tc.lim, kTranscode);
  off = block_excl_scan<NT, Sync, false>(tc.cnt, scan, agg);
}

// ---- encode: four units per operation (vt_swar.cuh) -------------------------
// encode_group16 gives the UTF-8 bytes of a group's four units as three byte
// planes (first / second / third byte) and the planes saying which units have
// a second and a third byte.  Every unit writes 1-3 bytes (a surrogate pair's
// 4 bytes are split 2 + 2 between its halves, so a pair may straddle threads
// and tiles): the first byte unconditionally, the second and third predicated
// on the unit having them, the tests going straight into the predicates (one
// LOP3 each) which also advance the running address.  Nothing is written
// beyond a unit's own bytes, so no word needs a special form.
#ifndef VT_GRAB_AT_G16
#define VT_GRAB_AT_G16 5  // groups encoded before the next tile is taken (of 8)
#endif
// (unit I of its group: the unconditional byte per unit sits in the immediate
// offsets, the running address takes only the predicated increments -- two
// adds per unit -- and moves on by 4 once per group)
template <uint32_t MASK, int I>
__device__ __forceinline__ void store_unit16(uint32_t& q, uint32_t F, uint32_t S, uint32_t T,
                                             uint32_t z80, uint32_t is3) {
  if (VT_CHECKS) VT_CHECK_STS(q + I, 1 + ((z80 & MASK) ? 1 : 0) + ((is3 & MASK) ? 1 : 0));
  asm volatile(
      "{\n\t.reg .pred p, r;\n\t.reg .b32 d;\n\t"
      "lop3.or.b32 d|p, %4, 0, %6, 0xA0, 0;\n\t"  // a & c
      "lop3.or.b32 d|r, %5, 0, %6, 0xA0, 0;\n\t"
      "st.shared.u8 [%0+%7], %1;\n\t"
      "@p st.shared.u8 [%0+%8], %2;\n\t"
      "@r st.shared.u8 [%0+%9], %3;\n\t"
      "@p add.u32 %0, %0, 1;\n\t"
      "@r add.u32 %0, %0, 1;\n\t}"
      : "+r"(q)
      : "r"(F), "r"(S), "r"(T), "r"(z80), "r"(is3), "n"(MASK), "n"(I), "n"(I + 1), "n"(I + 2));
}

#ifndef VT_NSTAGE16
#define VT_NSTAGE16 1  // two buffers: 1.375 vs 1.370 ms on cfg3 (with the L1 they take away)
#endif

template <bool kBE>
struct Utf16Codec {
  using Args = U16Args;
  using TileCount = TileCount16;
  static constexpr int kTileElems = K16_TILE;
  static constexpr int kStageBytes = 3 * K16_TILE;
  static constexpr int kNStage = VT_NSTAGE16;
  static constexpr int kOutBytes = 1;
  static constexpr int kPrefetchBytes = 0;  // (no input prefetch for this direction)
  __device__ __forceinline__ static bool prefetchable(const Args&, unsigned) { return false; }
  __device__ __forceinline__ static const uint8_t* prefetch_src(const Args&, unsigned) { return nullptr; }
  template <bool kTranscode, int NT, class Sync>
  __device__ __forceinline__ static void count(const Args& a, unsigned tile, unsigned* red,
                                               unsigned* scan, TileCount& tc, unsigned& off,
                                               unsigned& agg, const uint8_t* = nullptr,
                                               unsigned long long* early = nullptr) {
    count_tile16<kTranscode, NT, Sync, kBE>(a, tile, red, scan, tc, off, agg, early);
  }
  template <class Mid>
  __device__ __forceinline__ static void emit(const Args& a, const TileCount& tc, uint8_t* stage,
                                              unsigned off, unsigned tile, Mid&& mid) {
    if (tc.simple && __all_sync(0xffffffffu, tc.ascii)) {
      // A warp whose 1024 units are all ASCII: every lane writes exactly 32
      // bytes, the lanes' addresses are 32 bytes apart and the byte stores of
      // the general path conflict 8-way (and more so the stores of one lane
      // land in few words).  Each lane packs four units into one word and
      // stores its eight words in a lane-dependent order (re-read from global
      // memory, an L1 hit), so that the 32 words of one store fall into 32
      // different banks.  Warp-uniform alignment: the lanes are 32 bytes apart.
      const unsigned lane = threadIdx.x & 31;
      const uint2* p = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(a.base) +
                                                      (size_t)tile * (2 * K16_TILE) +
                                                      (size_t)(2 * K16_UPT * threadIdx.x));
      const uint32_t qb = smem_addr(stage) + off;
      const bool aligned4 = (qb & 3u) == 0;
#pragma unroll 4
      for (unsigned k = 0; k < (unsigned)K16_WPT / 2; k++) {
        const unsigned j = (k + (lane >> 2)) & (K16_WPT / 2 - 1);
        const uint2 x = __ldg(p + j);
        const uint32_t w = prmt(x.x, x.y, kBE ? 0x7531 : 0x6420);  // the four low bytes
        const uint32_t q = qb + 4u * j;
        if (aligned4) {
          VT_CHECK_STS(q, 4);
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(q), "r"(w));
        } else {
          sts8(q, w);
          sts8(q + 1, w >> 8);
          sts8(q + 2, w >> 16);
          sts8(q + 3, w >> 24);
        }
      }
      mid();
    } else if (tc.simple) {
      // (tc.lo > 0 only for the first thread of a call: the zeros before the
      // input are encoded too and land in the pad before the staging buffer)
      uint32_t q = smem_addr(stage) + off - tc.lo;
      using namespace swar;
      const K16 k = make_k16();
#pragma unroll
      for (int g = 0; g < K16_WPT / 2; g++) {
        if (g == VT_GRAB_AT_G16) {
          mid();
          __syncwarp();  // (keeps ptxas from sinking the atomic behind the stores)
        }
        const uint32_t x0 = tc.W.w[1 + 2 * g], x1 = tc.W.w[2 + 2 * g];
        const uint32_t lo = lo_plane(x0, x1), hi = hi_plane(x0, x1);
        const Enc16 e = encode_group16(lo, hi, tc.W.w[2 * g], k);
        store_unit16<0x00000080u, 0>(q, e.F, e.S, e.T, e.z80, e.is3);
        store_unit16<0x00008000u, 1>(q, e.F >> 8, e.S >> 8, e.T >> 8, e.z80, e.is3);
        store_unit16<0x00800000u, 2>(q, e.F >> 16, e.S >> 16, e.T >> 16, e.z80, e.is3);
        store_unit16<0x80000000u, 3>(q, e.F >> 24, e.S >> 24, e.T >> 24, e.z80, e.is3);
        q += 4;
      }
      if (VT_GRAB_AT_G16 >= K16_WPT / 2) mid();
    } else {
      mid();
      const Words16 tmp = tc.W;
      generic_units(tmp, tc.lo, tc.lim, true, stage + off);
    }
  }
};

// Validation / lengths without barriers: warp rows of 1024 units in grid
// stride, per-row counts for the error case (as utf8_validate_rows_kernel).
constexpr int K16_ROW = 32 * K16_UPT;  // units per warp row

template <bool kBE, bool kUnits = false>
__global__ void __launch_bounds__(256, 4) utf16_validate_rows_kernel(U16Args a) {
  unsigned* const row_counts = a.rows;
  __shared__ unsigned long long warp_tot[8];
  __shared__ bool last;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  const long long head = (long long)a.head, end = (long long)(a.head + a.n);
  const unsigned long long nrows = (unsigned long long)(end + K16_ROW - 1) / K16_ROW;
  const Src16 src{a.base, a.head, a.n, kBE};
  unsigned long long total = 0;
  unsigned wtot = 0;  // this warp's running total (rows so far)
  if (threadIdx.x == 0) VT_TR_MIN(8);
  // Stop behind a known error (warp-uniform).  The error word is loaded at the
  // top of every row and tested at the top of the next one, so the check adds
  // no latency and a warp runs at most one row past a found error.
  unsigned long long e_prev = kNoError;
  // rows [1, last_in) lie inside the input together with both halo words (head < 8 units)
  const unsigned long long last_in = end >= K16_ROW + 2 ? (unsigned long long)(end - 2) / K16_ROW : 0ull;
  for (unsigned long long row = gw; row < nrows; row += nwarps) {
    const long long r0 = (long long)row * K16_ROW;
    if (e_prev != kNoError && (long long)e_prev + head < r0) break;
    const unsigned long long e_next = lane == 0 ? load_relaxed(&a.ctl->err) : 0ull;
    const long long v0 = r0 + (long long)K16_UPT * lane;
    const bool interior = row >= 1 && row < last_in;  // (one uniform compare, as count_tile16)
    Words16 W;
    if (interior) {
      load_lane_words<K16_WPT>(reinterpret_cast<const uint8_t*>(a.base + v0), lane, W.w);
      if (kBE) {
#pragma unroll
        for (int k = 0; k < K16_WPT + 2; k++) W.w[k] = prmt(W.w[k], 0, 0x2301);
      }
    } else {
      load_edge16<kBE>(src, v0, W.w);
    }
    const Class16 c = classify16(W);
    unsigned cnt;
    if (!c.err) {
      if (interior) {
        cnt = kUnits ? c.bytes : c.chars;
      } else {
        const unsigned lo = (unsigned)max(0LL, min((long long)K16_UPT, head - v0));
        const unsigned hi = (unsigned)max((long long)lo, min((long long)K16_UPT, end - v0));
        cnt = (kUnits ? c.bytes : c.chars) - (K16_UPT - (hi - lo));  // minus the zeros outside
      }
    } else {
      const unsigned lo = (unsigned)max(0LL, min((long long)K16_UPT, head - v0));
      const unsigned hi = (unsigned)max((long long)lo, min((long long)K16_UPT, end - v0));
      const Words16 tmp = W;
      const unsigned er = first_error16(tmp, lo, hi);
      if (er != kNone16) {
        atomicMin(&a.ctl->err, (unsigned long long)(v0 + er - head));
        VT_TR_MIN(1);
      }
      cnt = swar_count16(W, lo, er != kNone16 ? er : hi, kUnits);
    }
    total += cnt;
    const unsigned rc = __reduce_add_sync(0xffffffffu, cnt);
    wtot += rc;
    if (lane == 0) row_counts[row] = wtot;
    e_prev = __shfl_sync(0xffffffffu, e_next, 0);
  }
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
    const unsigned long long erow = (e + a.head) / K16_ROW;
    unsigned long long t = prefix_rows(row_counts, erow, nwarps);
    if (wib == 0) {
      const long long v0 = (long long)erow * K16_ROW + (long long)K16_UPT * lane;
      const long long stop = (long long)e + head;
      const unsigned lo = (unsigned)max(0LL, min((long long)K16_UPT, head - v0));
      const unsigned lim = (unsigned)max((long long)lo, min((long long)K16_UPT, stop - v0));
      Words16 tmp;
      load_edge16<kBE>(src, v0, tmp.w);
      t += swar_count16(tmp, lo, lim, kUnits);
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

unsigned rows_utf16(unsigned long long head, unsigned long long n) {
  return (unsigned)((head + n + K16_ROW - 1) / K16_ROW);
}

// UTF-16LE (kBE = false) or UTF-16BE (kBE = true) -> UTF-8
template <bool kBE>
#ifndef VT_K16_MINB
#define VT_K16_MINB 4
#endif
__global__ void __launch_bounds__(kPipeBlock, VT_K16_MINB) utf16_transcode_kernel(U16Args a) {
  extern __shared__ __align__(16) uint8_t k16_dyn_smem[];
  transcode_body<Utf16Codec<kBE>>(a, *reinterpret_cast<PipeSmem<Utf16Codec<kBE>>*>(k16_dyn_smem));
}

static int set_smem_attr16() {
  // (no carveout preference: forcing the largest shared-memory carveout
  // leaves too little L1 for the input loads -- measured 1.37 vs 1.32 ms on
  // cfg3)
  for (const void* f :
       {(const void*)utf16_transcode_kernel<false>, (const void*)utf16_transcode_kernel<true>}) {
    const int rc = (int)cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sizeof(PipeSmem<Utf16Codec<false>>));
    if (rc) return rc;
#ifdef VT_CARVEOUT
    // (A/B: preferred shared-memory carveout in percent; more than 4 CTAs per SM
    // need more shared memory than the driver's default choice provides)
    if (cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, VT_CARVEOUT)) return 1;
#endif
  }
  return 0;
}

int launch_utf16(const U16Args& a, int mode, int grid, cudaStream_t s) {
  static const int attr_rc = set_smem_attr16();
  if (attr_rc) return attr_rc;
  if (mode == kModeTranscode)
    utf16_transcode_kernel<false><<<grid, kPipeBlock, sizeof(PipeSmem<Utf16Codec<false>>), s>>>(a);
  else if (mode == kModeTranscodeBE)
    utf16_transcode_kernel<true><<<grid, kPipeBlock, sizeof(PipeSmem<Utf16Codec<true>>), s>>>(a);
  else if (mode == kModeValidateBE)
    utf16_validate_rows_kernel<true><<<grid, 256, 0, s>>>(a);
  else if (mode == kModeLength)
    utf16_validate_rows_kernel<false, true><<<grid, 256, 0, s>>>(a);
  else
    utf16_validate_rows_kernel<false><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

int occupancy_utf16(bool transcode) {
  int n = 0;
  if (transcode) {
    if (set_smem_attr16()) return 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf16_transcode_kernel<false>, kPipeBlock,
                                                  sizeof(PipeSmem<Utf16Codec<false>>));
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf16_validate_rows_kernel<false>, 256, 0);
  }
  return n;
}

#ifdef VT_TRACE
int read_trace16(unsigned long long* out16) {
  int rc = (int)cudaMemcpyFromSymbol(out16, g_trace, sizeof(g_trace));
  unsigned long long init[16];
  for (int i = 0; i < 16; i++) init[i] = (i == 0 || i == 1 || i == 8) ? ~0ull : 0ull;
  if (!rc) rc = (int)cudaMemcpyToSymbol(g_trace, init, sizeof(init));
  return rc;
}
#endif

#ifdef VT_PHASES
int read_phases16(unsigned long long* out8) {
  int rc = (int)cudaMemcpyFromSymbol(out8, g_phase, sizeof(g_phase));
  if (!rc) rc = (int)cudaMemcpyFromSymbol(out8 + 8, g_phase_sub, sizeof(g_phase_sub));
  if (!rc) rc = (int)cudaMemcpyFromSymbol(out8 + 12, g_phase_lb, sizeof(g_phase_lb));
  return rc;
}
#endif

unsigned tiles_utf16(unsigned long long head, unsigned long long n) {
  const unsigned long long t = (head + n + K16_TILE - 1) / K16_TILE;
  return (unsigned)(t ? t : 1);
}

}  // namespace vt

// k_utf8.cu -- validated UTF-8 -> UTF-16LE transcoding and UTF-8 validation /
// code-point counting on sm_100a.
//
// Replaces the reference's 64-byte block driver (proj/src/utf8_to_utf16.cpp:
// 88-226) and the nibble-table checker (proj/include/vtrans/utf8_checker.hpp:
// 28-137).  One persistent kernel does, per 8 KiB tile:
//   1. coalesced 16-byte loads of the tile plus a 16-byte halo on each side
//      into shared memory (zero-filled outside the input, which makes the
//      start and the end of the input behave like the reference's zero-padded
//      final block, proj/src/validation.cpp:41-47);
//   2. per-thread SWAR classification of 16 bytes: continuation / 2-, 3-,
//      4-byte lead bit planes, the lead/continuation structure check and the
//      value-range check of the special leads (C0 C1 E0 ED F0 F4..FF);
//   3. on any flag, the exact per-byte first-error rule (SURVEY.md 8(a) fact
//      A) over the thread's bytes -- the scalar decoder's error_at
//      (proj/src/codec_core.cpp:85-104) without a sequential re-scan;
//   4. output length per thread (one unit per character, two for 4-byte
//      characters), block scan, decoupled look-back for the tile offset;
//   5. decode into a shared-memory staging buffer and aligned 16-byte stores.
#include "vt_device.cuh"
#include "vt_kernels.h"

namespace vt {

constexpr int U8_THREADS = 256;
constexpr int U8_ROWS = 2;
constexpr int U8_ROW = U8_THREADS * 16;   // bytes per row
constexpr int U8_TILE = U8_ROW * U8_ROWS;  // bytes per tile
constexpr unsigned kNone = 0xFFFFFFFFu;

// ---- byte-plane masks (bit 7 of each byte lane) ----------------------------
__device__ __forceinline__ uint32_t hi_bits(uint32_t x) { return x & 0x80808080u; }
__device__ __forceinline__ uint32_t m_cont(uint32_t x) { return x & ~(x << 1) & 0x80808080u; }
__device__ __forceinline__ uint32_t m_ge_c0(uint32_t x) { return x & (x << 1) & 0x80808080u; }
__device__ __forceinline__ uint32_t m_ge_e0(uint32_t x) { return m_ge_c0(x) & (x << 2); }
__device__ __forceinline__ uint32_t m_ge_f0(uint32_t x) { return m_ge_e0(x) & (x << 3); }

// Gathers bit 7 of each byte lane into a 4-bit nibble (lane k -> bit k).
__device__ __forceinline__ uint32_t gather4(uint32_t m) {
  return ((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u);
}

// Leads whose value range needs the second byte (C0 C1 E0 ED F0 F4..FF).
// The low nibble of every lane is looked up in two 16-entry tables with one
// PRMT each: entries 0..7 are table bytes, entries 8..15 replicate the sign
// bit of entry k-8 (PRMT's sign-extend selector mode).
__device__ __forceinline__ uint32_t m_special_lead(uint32_t x, uint32_t ge_c0, uint32_t ge_e0,
                                                   uint32_t ge_f0) {
  const uint32_t t = x & 0x0F0F0F0Fu;
  const uint32_t u = t | (t >> 4);
  const uint32_t sel = prmt(u, 0, 0x7720) & 0xFFFFu;  // nibbles ln0 ln1 ln2 ln3
  // E row: special at low nibble 0 (E0) and 13 (ED).  bit 0 of the entry.
  const uint32_t e_tab = prmt(0x00000001u, 0x00008000u, sel) & 0x01010101u;
  // F row: special at 0 (F0) and 4..15 (F4..FF).  bit 0 of the entry.
  const uint32_t f_tab = prmt(0x80808081u, 0x81818181u, sel) & 0x01010101u;
  // C/D row: only C0 and C1, i.e. bits 1..4 clear.
  const uint32_t x1e = x & 0x1E1E1E1Eu;
  const uint32_t c_zero = ~((x1e + 0x7F7F7F7Fu) | x1e) & 0x80808080u;  // lane == 0
  const uint32_t row_c = ge_c0 & ~ge_e0, row_e = ge_e0 & ~ge_f0, row_f = ge_f0;
  return (row_c & c_zero) | (row_e & (e_tab << 7)) | (row_f & (f_tab << 7));
}

__device__ __forceinline__ unsigned leadlen(unsigned b) {
  return b < 0x80u ? 1u : b < 0xC0u ? 1u : b < 0xE0u ? 2u : b < 0xF0u ? 3u : b < 0xF8u ? 4u : 1u;
}

// proj/src/codec_core.cpp:5-38 on a 4-byte window (bytes past the input are
// zero, which fails exactly like the truncation test at :28).
__device__ __forceinline__ bool decode_ok(uint32_t v) {
  const unsigned b0 = v & 0xFF, b1 = (v >> 8) & 0xFF, b2 = (v >> 16) & 0xFF, b3 = v >> 24;
  if (b0 < 0x80u) return true;
  unsigned len, cp, lo;
  if ((b0 & 0xE0u) == 0xC0u) {
    len = 2; cp = b0 & 0x1Fu; lo = 0x80u;
  } else if ((b0 & 0xF0u) == 0xE0u) {
    len = 3; cp = b0 & 0x0Fu; lo = 0x800u;
  } else if ((b0 & 0xF8u) == 0xF0u) {
    len = 4; cp = b0 & 0x07u; lo = 0x10000u;
  } else {
    return false;
  }
  if ((b1 & 0xC0u) != 0x80u) return false;
  cp = (cp << 6) | (b1 & 0x3Fu);
  if (len >= 3) {
    if ((b2 & 0xC0u) != 0x80u) return false;
    cp = (cp << 6) | (b2 & 0x3Fu);
  }
  if (len == 4) {
    if ((b3 & 0xC0u) != 0x80u) return false;
    cp = (cp << 6) | (b3 & 0x3Fu);
  }
  return cp >= lo && cp <= 0x10FFFFu && (cp < 0xD800u || cp > 0xDFFFu);
}

// Per-thread view of one row: 16 own bytes (w[0..3]) and 4 bytes either side.
struct Window {
  uint32_t pw, w[5];  // w[4] = next word
};

// Exact first error among the thread's 16 byte positions:
// a non-continuation byte whose decode fails, or a continuation byte no lead
// in the 3 bytes before it reaches.  `lo`/`hi` bound the in-input positions.
__device__ __noinline__ unsigned first_error_rule_a(const Window& win, unsigned lo, unsigned hi) {
  uint32_t buf[6] = {win.pw, win.w[0], win.w[1], win.w[2], win.w[3], win.w[4]};
  auto byte_at = [&](int p) -> unsigned {  // p in [-4, 20)
    const int q = p + 4;
    return (buf[q >> 2] >> ((q & 3) * 8)) & 0xFFu;
  };
  for (unsigned i = lo; i < hi; i++) {
    const unsigned b = byte_at((int)i);
    if ((b & 0xC0u) == 0x80u) {
      bool covered = false;
      for (int j = (int)i - 3; j < (int)i; j++) {
        if (leadlen(byte_at(j)) > (unsigned)((int)i - j)) covered = true;
      }
      if (!covered) return i;
    } else {
      const uint32_t v = byte_at((int)i) | (byte_at((int)i + 1) << 8) |
                         (byte_at((int)i + 2) << 16) | (byte_at((int)i + 3) << 24);
      if (!decode_ok(v)) return i;
    }
  }
  return kNone;
}

struct RowInfo {
  uint32_t lead;  // bit p: a character starts at position p (in input, before any error)
  uint32_t four;  // bit p: that character is 4 bytes long (2 UTF-16 units)
  uint32_t ascii_words;  // bit k: word k is 4 in-input ASCII bytes
};

// Phase 1 for one row of one thread: masks and the thread-local first error.
__device__ __forceinline__ unsigned classify(const Window& win, unsigned lo, unsigned hi,
                                             RowInfo& ri) {
  uint32_t c[5], l2[5], l3[5], l4[5];
  const uint32_t pl2 = m_ge_c0(win.pw), pl3 = m_ge_e0(win.pw), pl4 = m_ge_f0(win.pw);
#pragma unroll
  for (int k = 0; k < 5; k++) {
    c[k] = m_cont(win.w[k]);
    l2[k] = m_ge_c0(win.w[k]);
    l3[k] = m_ge_e0(win.w[k]);
    l4[k] = m_ge_f0(win.w[k]);
  }
  uint32_t viol = 0, special = 0, lead = 0, four = 0, ascii = 0;
#pragma unroll
  for (int k = 0; k < 5; k++) {
    const uint32_t p2 = k ? l2[k - 1] : pl2, p3 = k ? l3[k - 1] : pl3, p4 = k ? l4[k - 1] : pl4;
    const uint32_t need = __funnelshift_l(p2, l2[k], 8) | __funnelshift_l(p3, l3[k], 16) |
                          __funnelshift_l(p4, l4[k], 24);
    uint32_t v = (need ^ c[k]) & 0x80808080u;
    if (k == 4) v &= 0x00808080u;  // next word: only lanes that can blame our bytes
    viol |= v;
    if (k < 4) {
      special |= gather4(m_special_lead(win.w[k], l2[k], l3[k], l4[k])) << (4 * k);
      lead |= gather4(~c[k] & 0x80808080u) << (4 * k);
      four |= gather4(l4[k]) << (4 * k);
      if (hi_bits(win.w[k]) == 0) ascii |= 1u << k;
    }
  }
  const uint32_t inmask = (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
  special &= inmask & lead;
  unsigned err = kNone;
  bool check = viol != 0;
  if (special) {
    // exact range check of the special leads
    uint32_t s = special;
    while (s) {
      const unsigned p = __ffs(s) - 1;
      s &= s - 1;
      const unsigned k = p >> 2, sh = (p & 3) * 8;
      uint32_t a = win.w[0], b = win.w[1];
      if (k == 1) { a = win.w[1]; b = win.w[2]; }
      if (k == 2) { a = win.w[2]; b = win.w[3]; }
      if (k == 3) { a = win.w[3]; b = win.w[4]; }
      if (!decode_ok(__funnelshift_r(a, b, sh))) check = true;
    }
  }
  if (check) err = first_error_rule_a(win, lo, hi);
  ri.lead = lead & inmask;
  ri.four = four & inmask;
  uint32_t aw = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if ((ascii >> k) & 1u) aw |= (((inmask >> (4 * k)) & 0xFu) == 0xFu) ? (1u << k) : 0u;
  ri.ascii_words = aw;
  return err;
}

// Decodes the characters starting in this row's bytes (bits of `lead`) and
// stores their UTF-16 units to shared memory at `dst`.
__device__ __forceinline__ void emit_row(const Window& win, const RowInfo& ri, uint16_t* dst) {
  unsigned q = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t x = win.w[k];
    const uint32_t lw = (ri.lead >> (4 * k)) & 0xFu;
    if ((ri.ascii_words >> k) & 1u) {
      dst[q + 0] = (uint16_t)(x & 0xFF);
      dst[q + 1] = (uint16_t)((x >> 8) & 0xFF);
      dst[q + 2] = (uint16_t)((x >> 16) & 0xFF);
      dst[q + 3] = (uint16_t)(x >> 24);
      q += 4;
      continue;
    }
    uint32_t m = lw;
    while (m) {
      const unsigned lane = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t v = __funnelshift_r(x, win.w[k + 1], lane * 8);
      const unsigned b0 = v & 0xFF, b1 = (v >> 8) & 0x3F, b2 = (v >> 16) & 0x3F, b3 = (v >> 24) & 0x3F;
      unsigned cp;
      if (b0 < 0x80u) {
        cp = b0;
      } else if (b0 < 0xE0u) {
        cp = ((b0 & 0x1Fu) << 6) | b1;
      } else if (b0 < 0xF0u) {
        cp = ((b0 & 0x0Fu) << 12) | (b1 << 6) | b2;
      } else {
        cp = ((b0 & 0x07u) << 18) | (b1 << 12) | (b2 << 6) | b3;
      }
      if (cp < 0x10000u) {
        dst[q++] = (uint16_t)cp;
      } else {
        const unsigned s = cp - 0x10000u;
        dst[q] = (uint16_t)(0xD800u + (s >> 10));
        dst[q + 1] = (uint16_t)(0xDC00u + (s & 0x3FFu));
        q += 2;
      }
    }
  }
}

struct U8Smem {
  alignas(16) uint8_t in[16 + U8_TILE + 16];
  alignas(16) uint8_t out_pad[32];
  alignas(16) uint16_t out[U8_TILE];
  alignas(16) uint8_t out_tail[32];
  unsigned scan[U8_THREADS / 32];
  unsigned red[U8_THREADS / 32];
  unsigned long long excl;
  unsigned tile;
  unsigned flag;
};

// Loads tile `tile` (16-byte chunks, zero outside the input) into smem.
__device__ __forceinline__ void load_tile(const U8Args& a, unsigned tile, uint8_t* in_s) {
  const unsigned long long vbase = (unsigned long long)tile * U8_TILE;  // virtual byte of in_s[16]
  const unsigned long long vend = a.head + a.n;
  for (int j = threadIdx.x; j < U8_TILE / 16 + 2; j += U8_THREADS) {
    const long long vc = (long long)vbase - 16 + 16LL * j;  // virtual start of chunk
    uint4 v = make_uint4(0, 0, 0, 0);
    if (vc >= 0 && (unsigned long long)vc < vend && (unsigned long long)vc + 16 > a.head) {
      v = __ldcs(reinterpret_cast<const uint4*>(a.base + vc));
      if ((unsigned long long)vc < a.head || (unsigned long long)vc + 16 > vend) {
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int b = 0; b < 16; b++) {
          const unsigned long long pos = (unsigned long long)vc + b;
          if (pos < a.head || pos >= vend) w[b >> 2] &= ~(0xFFu << ((b & 3) * 8));
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    *reinterpret_cast<uint4*>(in_s + 16 * j) = v;
  }
}

__device__ __forceinline__ void thread_bounds(const U8Args& a, unsigned tile, int row,
                                              unsigned& lo, unsigned& hi) {
  const long long v0 = (long long)tile * U8_TILE + row * U8_ROW + 16 * threadIdx.x;
  const long long s = (long long)a.head - v0, e = (long long)(a.head + a.n) - v0;
  lo = (unsigned)max(0LL, min(16LL, s));
  hi = (unsigned)max(0LL, min(16LL, e));
  if (hi < lo) hi = lo;
}

__device__ __forceinline__ Window load_window(const uint8_t* in_s, int row) {
  const uint8_t* p = in_s + 16 + row * U8_ROW + 16 * threadIdx.x;
  Window w;
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  w.pw = *reinterpret_cast<const uint32_t*>(p - 4);
  w.w[0] = v.x; w.w[1] = v.y; w.w[2] = v.z; w.w[3] = v.w;
  w.w[4] = *reinterpret_cast<const uint32_t*>(p + 16);
  return w;
}

__device__ __forceinline__ void finalize_if_last(const U8Args& a, bool transcode) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long e = load_relaxed(&a.ctl->err);
      vt_result r;
      if (transcode) {
        unsigned long long written;
        if (e == kNoError) {
          written = load_status(&a.status[a.ntiles - 1]) & kValMask;
        } else {
          const unsigned et = (unsigned)((e + a.head) / U8_TILE);
          written = load_status(&a.status[et]) & kValMask;
        }
        r.written = written;
      } else {
        r.written = load_relaxed(&a.ctl->count);
      }
      r.consumed = e == kNoError ? a.n : e;
      r.error_at = e == kNoError ? -1 : (long long)e;
      *a.res = r;
      a.ctl->tile_counter = 0;
      a.ctl->count = 0;
      a.ctl->err = kNoError;
      __threadfence();
      a.ctl->done = 0;
    }
  }
}

template <bool kTranscode>
__global__ void __launch_bounds__(U8_THREADS) utf8_kernel(U8Args a) {
  __shared__ U8Smem sm;
  while (true) {
    if (threadIdx.x == 0) {
      unsigned t = atomicAdd(&a.ctl->tile_counter, 1u);
      const unsigned long long e = load_relaxed(&a.ctl->err);
      // tiles behind a known error never matter: stop (the reference stops too)
      if (t < a.ntiles && e != kNoError && (e + a.head) / U8_TILE < t) t = a.ntiles;
      sm.tile = t;
    }
    __syncthreads();
    const unsigned tile = sm.tile;
    if (tile >= a.ntiles) break;

    load_tile(a, tile, sm.in);
    __syncthreads();

    Window win[U8_ROWS];
    RowInfo ri[U8_ROWS];
    unsigned lo[U8_ROWS], hi[U8_ROWS];
    unsigned my_err = kNone;
#pragma unroll
    for (int r = 0; r < U8_ROWS; r++) {
      win[r] = load_window(sm.in, r);
      thread_bounds(a, tile, r, lo[r], hi[r]);
      const unsigned e = classify(win[r], lo[r], hi[r], ri[r]);
      if (e != kNone && my_err == kNone) my_err = r * U8_ROW + 16 * threadIdx.x + e;
    }
    const unsigned tile_err = block_min<U8_THREADS>(my_err, sm.red);
    // keep only characters before the tile's first error
    unsigned cnt[U8_ROWS];
#pragma unroll
    for (int r = 0; r < U8_ROWS; r++) {
      const unsigned start = r * U8_ROW + 16 * threadIdx.x;
      if (tile_err != kNone) {
        const unsigned lim = tile_err <= start ? 0u : min(16u, tile_err - start);
        const uint32_t keep = lim >= 32 ? 0xFFFFFFFFu : ((1u << lim) - 1u);
        ri[r].lead &= keep;
        ri[r].four &= keep;
        uint32_t aw = 0;
        for (int k = 0; k < 4; k++)
          if (((ri[r].ascii_words >> k) & 1u) && ((keep >> (4 * k)) & 0xFu) == 0xFu) aw |= 1u << k;
        ri[r].ascii_words = aw;
      }
      cnt[r] = kTranscode ? __popc(ri[r].lead) + __popc(ri[r].four) : __popc(ri[r].lead);
    }
    if (tile_err != kNone && threadIdx.x == 0) {
      const unsigned long long pos = (unsigned long long)tile * U8_TILE + tile_err - a.head;
      atomicMin(&a.ctl->err, pos);
    }

    if (!kTranscode) {
      unsigned total;
      block_excl_scan<U8_THREADS>(cnt[0] + cnt[1], sm.scan, total);
      if (threadIdx.x == 0 && total) atomicAdd(&a.ctl->count, (unsigned long long)total);
      __syncthreads();
      continue;
    }

    unsigned tot0, tot1;
    const unsigned off0 = block_excl_scan<U8_THREADS>(cnt[0], sm.scan, tot0);
    const unsigned off1 = block_excl_scan<U8_THREADS>(cnt[1], sm.scan, tot1) + tot0;
    const unsigned agg = tot0 + tot1;

    // publish the aggregate, then resolve the exclusive prefix
    if (threadIdx.x < 32) {
      unsigned long long excl = 0;
      if (tile == 0) {
        if (threadIdx.x == 0) store_status(&a.status[0], pack_status(kFlagPre, a.epoch, agg));
      } else {
        if (threadIdx.x == 0) store_status(&a.status[tile], pack_status(kFlagAgg, a.epoch, agg));
        excl = lookback(a.status, a.epoch, tile, a.ctl, U8_TILE, a.head);
        if (threadIdx.x == 0 && excl != ~0ull)
          store_status(&a.status[tile], pack_status(kFlagPre, a.epoch, excl + agg));
      }
      if (threadIdx.x == 0) sm.excl = excl;
    }
    emit_row(win[0], ri[0], sm.out + off0);
    emit_row(win[1], ri[1], sm.out + off1);
    __syncthreads();
    const unsigned long long excl = sm.excl;
    if (excl != ~0ull)
      copy_out(reinterpret_cast<uint8_t*>(a.out + excl), reinterpret_cast<const uint8_t*>(sm.out),
               2u * agg);
    __syncthreads();
  }
  finalize_if_last(a, kTranscode);
}

int launch_utf8(const U8Args& a, bool transcode, int grid, cudaStream_t s) {
  if (transcode)
    utf8_kernel<true><<<grid, U8_THREADS, 0, s>>>(a);
  else
    utf8_kernel<false><<<grid, U8_THREADS, 0, s>>>(a);
  return (int)cudaGetLastError();
}

int occupancy_utf8(bool transcode) {
  int n = 0;
  if (transcode)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf8_kernel<true>, U8_THREADS, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf8_kernel<false>, U8_THREADS, 0);
  return n;
}

unsigned tiles_utf8(unsigned long long head, unsigned long long n) {
  const unsigned long long t = (head + n + U8_TILE - 1) / U8_TILE;
  return (unsigned)(t ? t : 1);
}

}  // namespace vt

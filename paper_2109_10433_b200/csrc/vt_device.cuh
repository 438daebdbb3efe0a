// vt_device.cuh -- shared sm_100a device machinery for the transcoding kernels.
//
//  * tile scheduling: persistent CTAs pull tile ids from an atomic counter, so
//    every tile's predecessors are owned by CTAs that are already running
//    (the forward-progress condition of the decoupled look-back);
//  * the single-pass decoupled look-back scan over per-tile output counts
//    (epoch-tagged 64-bit status words: no per-call memset of the status array);
//  * first-error resolution across tiles (atomicMin on the input position;
//    tiles behind a known error stop early, like the reference's early exit at
//    proj/src/utf8_to_utf16.cpp:121,144 and proj/src/validation.cpp:38);
//  * the "last CTA finalises" epilogue that writes the TranscodeResult and
//    re-arms the control block for the next call on the same scratch;
//  * an aligned 16-byte copy-out from the shared-memory staging buffer to an
//    arbitrarily aligned global destination.
#pragma once

#include <cstdint>
#include <cstdio>

#include "../../include/vtrans_gpu.h"

namespace vt {

constexpr unsigned long long kNoError = ~0ull;

// PRMT in its default mode: selector nibble bit 3 replicates the sign bit of the
// selected byte (the 16-entry lookup trick in k_utf8.cu depends on it).
template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Shared-memory accesses through 32-bit shared-window addresses (a generic
// pointer into shared memory costs an address conversion per access).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// VT_TRACE builds (tools/cfg4_trace.py): global-timer stamps of the phases of
// an early-error call, per translation unit (read with vt_debug_trace).
#ifdef VT_TRACE
static __device__ unsigned long long g_trace[16];
__device__ __forceinline__ unsigned long long vt_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define VT_TR_MIN(i) atomicMin(&g_trace[i], vt_gtimer())
#define VT_TR_MAX(i) atomicMax(&g_trace[i], vt_gtimer())
#else
#define VT_TR_MIN(i) \
  do {               \
  } while (0)
#define VT_TR_MAX(i) \
  do {               \
  } while (0)
#endif

// VT_CHECKS builds (tools/gpu_checked.sh): every staging store and every
// copy-out range is bounds-checked and traps with a message when out of range
// (the pool has compute-sanitizer closed; this is the substitute).
#ifndef VT_CHECKS
#define VT_CHECKS 0
#endif
extern __shared__ __align__(16) uint8_t vt_dyn_smem[];
// bytes of PipeSmem after its staging region (scan .. excl, vt_pipeline.cuh
// static_asserts it): a staging store must land before them
#ifndef VT_COMPUTE_THREADS
#define VT_COMPUTE_THREADS 256
#endif
constexpr unsigned kPipeTail = 8 * (VT_COMPUTE_THREADS / 32) + 64;

static __device__ __noinline__ void vt_check_fail(const char* what, unsigned long long a,
                                                  unsigned long long b, unsigned long long lo,
                                                  unsigned long long hi) {
  printf("VT_CHECKS: %s [%llu, +%llu) outside [%llu, %llu) block %d thread %d\n", what, a, b, lo, hi,
         blockIdx.x, threadIdx.x);
  __trap();
}

static __device__ __forceinline__ void vt_check_sts(uint32_t a, unsigned bytes) {
  uint32_t dsz;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
  const uint32_t lo = (uint32_t)__cvta_generic_to_shared(vt_dyn_smem), hi = lo + dsz - kPipeTail;
  if (a < lo || a + bytes > hi) vt_check_fail("staging store", a, bytes, lo, hi);
}
#if VT_CHECKS
#define VT_CHECK_STS(a, b) vt_check_sts((a), (b))
#else
#define VT_CHECK_STS(a, b) \
  do {                     \
  } while (0)
#endif

// A/B probes of the staging-store cost (timing only, output is garbage):
// VT_EXP_LANESTS keeps every store but sends lane i to bank i (no conflicts).
#ifdef VT_EXP_LANESTS
#define VT_LANE_ADDR(a) (((a) & ~0x7Fu) | ((threadIdx.x & 31u) << 2) | ((a) & 3u))
#elif defined(VT_EXP_PREDOFF)
// VT_EXP_PREDOFF: every store's address and value are computed, the store is
// predicated off at run time (measures the emit's ALU work without the stores)
#define VT_LANE_ADDR(a) ((a) | 0xFFFF0000u)
#else
#define VT_LANE_ADDR(a) (a)
#endif
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  VT_CHECK_STS(a, 2);
  a = VT_LANE_ADDR(a);
#ifdef VT_EXP_NOSTS
  asm volatile("" ::"r"(a), "r"(v));
#elif defined(VT_EXP_PREDOFF)
  if (a == 0xFFFFFFFFu) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
#else
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
#endif
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  // stores the low byte of v (no masking instruction needed)
  VT_CHECK_STS(a, 1);
  a = VT_LANE_ADDR(a);
#ifdef VT_EXP_NOSTS
  asm volatile("" ::"r"(a), "r"(v));
#elif defined(VT_EXP_PREDOFF)
  if (a == 0xFFFFFFFFu) asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
#else
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
#endif
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// Per-call control block.  Zeroed once at allocation; the finalising CTA of
// every launch re-arms it, so consecutive calls on one stream need no memset.
// The tile counter takes one atomic per tile from every CTA: it has a 128-byte
// line to itself, so the error word every tile reads is not queued behind it.
struct Ctl {
  alignas(128) unsigned int tile_counter;
  unsigned int line_pad[31];
  unsigned long long err;    // smallest failing input index seen, kNoError if none
  unsigned long long count;  // validate/count kernels: code points in the valid prefix
  unsigned int done;
  unsigned long long pad[5];
};

// ---- status words -----------------------------------------------------------
// [63:62] flag (1 = aggregate, 2 = inclusive prefix), [61:48] epoch, [47:0] value
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 48) - 1;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, unsigned epoch,
                                                          unsigned long long v) {
  return flag | ((unsigned long long)(epoch & 0x3FFF) << 48) | (v & kValMask);
}

// Relaxed device-scope accesses to global words as plain PTX (the libcu++
// atomic_ref forms compiled to generic-address loads behind a dispatch: ncu
// counted ~3 % of the kernel's instructions in them, all on the look-back warp
// and thread 0).
__device__ __forceinline__ void store_status(unsigned long long* p, unsigned long long s) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(s) : "memory");
}

__device__ __forceinline__ unsigned long long load_status(unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Relaxed fetch-and-increment whose position among the (volatile) shared
// stores of the emit is kept: the next-tile grab is issued part-way through
// the decode and its round trip overlaps the rest of it.
// (predicated inside the asm: a branch around it lets ptxas sink the block
// behind the stores that follow)
__device__ __forceinline__ void atom_inc_pinned(unsigned* p, bool pred, unsigned& r) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q atom.relaxed.gpu.global.add.u32 %0, [%1], 1;\n\t}"
      : "+r"(r)
      : "l"(p), "r"((unsigned)pred));
}

__device__ __forceinline__ unsigned long long load_relaxed(unsigned long long* p) {
  return load_status(p);
}

// Warp-cooperative decoupled look-back for tile `tile` (> 0), executed by one
// full warp.  Returns the exclusive prefix, or ~0ull when the tile became
// irrelevant (a tile before it reported an error, so its output is never read).
//
// Each step loads VT_LB_WIN windows of 32 status words at once (window k, lane
// i: tile base - 32k - i; independent loads, one L2 round trip), then walks
// them newest first: a fully-ready window without an inclusive prefix is summed
// and passed, the first window with a prefix ends the walk.  A window that is
// not ready yet stops the step; the ready part before it is banked and the step
// repeats from there.  The caller publishes the tile's own inclusive prefix
// (with VT_LB_HELP also those of the aggregate-only tiles summed: "helping").
//
// Aggregates are tile-sized (< 2^16 elements, <= 3 output bytes each), so sums
// over one step's <= 32 * VT_LB_WIN tiles fit in 32 bits (32-bit shuffles, REDUX).
#ifndef VT_LB_WIN
#define VT_LB_WIN 1  // measured: 2 and 4 windows per step are slower (L2 contention)
#endif
// VT_LB_HELP: a look-back also publishes the inclusive prefixes of the
// aggregate-only tiles it summed.  Off: concurrent look-backs walking the same
// tiles stored the same prefixes to the hottest status lines, which every
// poller and publisher hits (measured without: 0.910 -> 0.901 ms cfg2, 1.234 ->
// 1.231 cfg3, 12.16 -> 12.13 cfg5).
#ifndef VT_LB_HELP
#define VT_LB_HELP 0
#endif
#ifndef VT_LB_DELAY
#define VT_LB_DELAY 2000  // ns before the first poll (3000 before the look-back warp took over the copy-out)
#endif
#ifndef VT_LB_SLEEP
#define VT_LB_SLEEP 2000  // ns between polls of a window that is not ready
#endif
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status, unsigned epoch,
                                                      unsigned tile, const Ctl* ctl,
                                                      unsigned long long tile_bytes,
                                                      unsigned long long head) {
  // (One window of 32 status words per step.  The look-back warp also copies
  // the tiles out, and it gets one warp's share of its scheduler's issue slots,
  // so every instruction here delays the hand-back of the staging buffer:
  // 32-bit tags and sums, REDUX instead of shuffle trees, no per-window arrays.)
  const unsigned lane = threadIdx.x & 31;
  const unsigned ep = epoch & 0x3FFF;
  const unsigned tag_agg = 0x4000u | ep, tag_pre = 0x8000u | ep;
  unsigned long long excl = 0;
  int base = (int)tile - 1;  // newest predecessor not yet summed (tiles < 2^31)
#if VT_LB_DELAY
  // the predecessor was taken just before this tile and publishes its
  // aggregate only after its count phase (~4 us): polling before that only
  // loads the status lines (not in the first two waves of tiles: small inputs
  // are latency-bound)
  if (tile >= 2 * gridDim.x) __nanosleep(VT_LB_DELAY);
#endif
  for (bool first = true;; first = false) {
    // a tile behind a known error is dead: give up (its output is never read;
    // the tail of an early-error call waits on these look-backs).  Checked at
    // the start, beside the first status loads (same round trip), and
    // whenever a poll makes no progress (below).
    const unsigned long long err =
        first && lane == 0 ? load_relaxed(const_cast<unsigned long long*>(&ctl->err)) : kNoError;
    const int idx = base - (int)lane;
    const unsigned long long st = idx >= 0 ? load_status(&status[idx]) : 0ull;
    const unsigned tag = (unsigned)(st >> 48);
    const bool pre = idx < 0 || tag == tag_pre;  // before tile 0: prefix 0
    const bool rdy = pre || tag == tag_agg;
    const uint32_t v32 = idx < 0 ? 0u : (uint32_t)st;  // aggregates are tile-sized: 32 bits
    if (first) {
      const unsigned long long e = __shfl_sync(0xffffffffu, err, 0);
      if (e != kNoError && (e + head) / tile_bytes < tile) return ~0ull;
    }
    const unsigned rm = __ballot_sync(0xffffffffu, rdy);
    const unsigned pm = __ballot_sync(0xffffffffu, pre);
    const unsigned run = rm == 0xffffffffu ? 32u : (unsigned)__ffs(~rm) - 1u;
    const unsigned pre_in = pm & (run == 32 ? 0xffffffffu : ((1u << run) - 1u));
    if (pre_in) {
      const unsigned stop = (unsigned)__ffs(pre_in) - 1u;  // nearest inclusive prefix
      const unsigned long long pval =
          __shfl_sync(0xffffffffu, idx < 0 ? 0ull : (st & kValMask), stop);
      const uint32_t s = __reduce_add_sync(0xffffffffu, lane < stop ? v32 : 0u);
      return excl + pval + s;
    }
#ifdef VT_PROBE
    if (lane == 0) atomicAdd(const_cast<unsigned long long*>(&ctl->pad[4]), run > 0 ? (1ull << 32) : 1ull);
#endif
    if (run > 0) {  // no prefix in reach: bank the ready part and walk on
      excl += __reduce_add_sync(0xffffffffu, lane < run ? v32 : 0u);
      base -= (int)run;
      continue;
    }
    // nothing ready yet: give up if an earlier tile failed (our output is dead)
    const unsigned long long e = load_relaxed(const_cast<unsigned long long*>(&ctl->err));
    if (e != kNoError && (e + head) / tile_bytes < tile) return ~0ull;
    // back off: the status lines are hot in L2 (hundreds of look-backs poll
    // them); measured best with a long sleep, the slack is more than a tile
    __nanosleep(VT_LB_SLEEP);
  }
}

// Copies `len` bytes from shared memory `src` (16-byte aligned) to global `dst`
// (any alignment) with aligned 16-byte stores in the body.  Threads
// 0..nthreads-1 participate.  `src` must have >= 16 readable bytes before and
// >= 32 after.
//
// Chunk c of the destination needs source bytes [16c - mis, +16): words
// WS..WS+4 of the two aligned 16-byte source chunks starting at 16(c-1) (+16
// for mis == 0), then a byte funnel shift.  WS and the shift are the same for
// every chunk, so the loop is instantiated per WS.
template <int WS, bool kShift>
__device__ __forceinline__ void copy_chunk(uint8_t* __restrict__ d, uint32_t a, unsigned bs) {
  uint32_t x[8];
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(a));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]) : "r"(a + 16));
  uint4 v;
  if (kShift) {
    v.x = __funnelshift_r(x[WS], x[WS + 1], bs);
    v.y = __funnelshift_r(x[WS + 1], x[WS + 2], bs);
    v.z = __funnelshift_r(x[WS + 2], x[WS + 3], bs);
    v.w = __funnelshift_r(x[WS + 3], x[WS + 4], bs);
  } else {  // source and destination congruent mod 4: whole words
    v.x = x[WS];
    v.y = x[WS + 1];
    v.z = x[WS + 2];
    v.w = x[WS + 3];
  }
  *reinterpret_cast<uint4*>(d) = v;
}

#ifndef VT_COPY_UNROLL
#define VT_COPY_UNROLL 4  // chunks in flight per thread in the copy-out loop (2: +0.6 % on cfg2, r2z)
#endif
template <int WS, bool kShift>
__device__ __forceinline__ void copy_out_ws(uint8_t* __restrict__ dbase, uint32_t sbase,
                                            unsigned mis, unsigned len, unsigned bs,
                                            unsigned nthreads, unsigned tid) {
  const unsigned end = mis + len;
  const unsigned c_end = end >> 4;  // chunks [mis ? 1 : 0, c_end) are whole
  // whole chunks: running addresses with constant strides, two independent
  // chunks per step (more stores in flight)
  const unsigned c0 = (mis ? 1u : 0u) + tid;
  if (c0 < c_end) {
    unsigned n = (c_end - c0 + nthreads - 1) / nthreads;
    uint32_t a = sbase + 16u * c0 - (mis ? 16u : 0u);
    uint8_t* d = dbase + 16u * c0;
    const unsigned step = 16u * nthreads;
    constexpr int kCopyUnroll = VT_COPY_UNROLL;
#pragma unroll kCopyUnroll
    for (; n; n--) {
      copy_chunk<WS, kShift>(d, a, bs);
      a += step;
      d += step;
    }
  }
  // the partial first chunk (bytes [mis, 16)) and last chunk (bytes
  // [16 c_end, end)): one byte per thread, threads 0..15 and 16..31
  const unsigned t = tid;
  if (t < 32) {
    const unsigned pos = t < 16 ? t : 16u * c_end + (t - 16);
    const bool first = t < 16 && mis != 0;
    const bool last = t >= 16 && (end & 15u) != 0 && (c_end > 0 || mis == 0);
    if ((first || last) && pos >= mis && pos < end) {
      uint32_t b;
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(sbase + pos - mis));
      dbase[pos] = (uint8_t)b;
    }
  }
}

__device__ __forceinline__ void copy_out(uint8_t* __restrict__ dst, const uint8_t* src,
                                         unsigned len, unsigned nthreads, unsigned tid) {
  if (len == 0) return;
  const unsigned mis = (unsigned)((uintptr_t)dst & 15);
  uint8_t* dbase = dst - mis;
  const uint32_t sbase = smem_addr(src);
  const unsigned rel = (16u - mis) & 15u;  // (16c - mis) mod 16
  const unsigned bs = (rel & 3u) * 8u;
  // (bs == 0 for every other tile of 2-byte output: those copy whole words
  // without the four funnel shifts per chunk)
  switch ((rel >> 2) | (bs ? 4u : 0u)) {
    case 0: copy_out_ws<0, false>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 1: copy_out_ws<1, false>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 2: copy_out_ws<2, false>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 3: copy_out_ws<3, false>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 4: copy_out_ws<0, true>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 5: copy_out_ws<1, true>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    case 6: copy_out_ws<2, true>(dbase, sbase, mis, len, bs, nthreads, tid); break;
    default: copy_out_ws<3, true>(dbase, sbase, mis, len, bs, nthreads, tid); break;
  }
}

// A lane's 4*NW input bytes at p (16-byte aligned) as NW words w[1..NW], plus
// the word before (w[0]) and after (w[NW+1]) its range: neighbour lanes' words
// by shuffle, lanes 0 and 31 load theirs.  Every lane issues one halo load
// (address selected, no branch), so all loads are in flight together -- a halo
// load behind the shuffles, which wait for the body, would add a second load
// latency to the tile.  p - 4 and p + 4*NW must be readable for lanes 0 / 31.
template <int NW>
__device__ __forceinline__ void load_lane_words(const uint8_t* p, unsigned lane, uint32_t* w) {
  static_assert(NW % 4 == 0, "whole 16-byte loads");
  const uint32_t* hp = reinterpret_cast<const uint32_t*>(lane == 0 ? p - 4 : p + 4 * NW);
  const uint32_t h = __ldg(hp);
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int r = 0; r < NW / 4; r++) {
    const uint4 v = __ldg(q + r);
    w[1 + 4 * r] = v.x;
    w[2 + 4 * r] = v.y;
    w[3 + 4 * r] = v.z;
    w[4 + 4 * r] = v.w;
  }
  const uint32_t pw = __shfl_up_sync(0xffffffffu, w[NW], 1);
  const uint32_t nw = __shfl_down_sync(0xffffffffu, w[1], 1);
  w[0] = lane == 0 ? h : pw;
  w[NW + 1] = lane == 31 ? h : nw;
}

// The same words from a tile prefetched into shared memory (q = the lane's
// first byte; the words before and behind it are in the buffer too).
template <int NW>
__device__ __forceinline__ void load_smem_words(uint32_t q, uint32_t* w) {
  static_assert(NW % 4 == 0, "whole 16-byte loads");
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(q - 4u));
#pragma unroll
  for (int r = 0; r < NW / 4; r++)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[1 + 4 * r]), "=r"(w[2 + 4 * r]), "=r"(w[3 + 4 * r]), "=r"(w[4 + 4 * r])
                 : "r"(q + 16u * r));
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[NW + 1]) : "r"(q + 4u * NW));
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

// Barrier policies for the block-level collectives: the whole CTA, or a named
// barrier over the first N threads (the compute warps of a warp-specialised CTA).
struct SyncAll {
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
template <int ID, int N>
struct SyncNamed {
  __device__ __forceinline__ static void sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
  }
};
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Barrier BASE + (sel mod N) with the id as an immediate (N = 2 or 4; a uniform
// branch picks it).  With an id in a register ptxas cannot tell which barriers
// a kernel uses and books all 16 ("used 16 barriers"), and an SM hands out 64:
// that alone capped the transcode kernels at 4 CTAs per SM whatever their
// registers and shared memory (cudaOccupancyMaxActiveBlocksPerMultiprocessor
// said 4 for a 192-thread, 40-register, 20 KiB variant).
template <int ID, int NT>
__device__ __forceinline__ void bar_sync_imm() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}
template <int ID, int NT>
__device__ __forceinline__ void bar_arrive_imm() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(NT) : "memory");
}
// (VT_BAR_IMM=0, the default: the id stays in a register -- with 56 registers
// per thread the register file caps the kernels at 4 CTAs per SM anyway, and
// the uniform branches cost ~0.5 %.  Shapes with more CTAs per SM need 1; none
// of them was faster, profiles/r02/ab_r3w_occupancy_shapes.txt.)
#ifndef VT_BAR_IMM
#define VT_BAR_IMM 0
#endif
template <int BASE, int N, int NT>
__device__ __forceinline__ void bar_sync_sel(unsigned sel) {
  static_assert(N == 2 || N == 4, "two or four ids");
  sel &= N - 1;
  if (!VT_BAR_IMM) {
    bar_sync(BASE + (int)sel, NT);
    return;
  }
  if (N == 4 && sel >= 2) {
    if (sel == 3) bar_sync_imm<BASE + (N == 4 ? 3 : 1), NT>();
    else bar_sync_imm<BASE + (N == 4 ? 2 : 0), NT>();
  } else {
    if (sel == 1) bar_sync_imm<BASE + 1, NT>();
    else bar_sync_imm<BASE, NT>();
  }
}
template <int BASE, int N, int NT>
__device__ __forceinline__ void bar_arrive_sel(unsigned sel) {
  static_assert(N == 2 || N == 4, "two or four ids");
  sel &= N - 1;
  if (!VT_BAR_IMM) {
    bar_arrive(BASE + (int)sel, NT);
    return;
  }
  if (N == 4 && sel >= 2) {
    if (sel == 3) bar_arrive_imm<BASE + (N == 4 ? 3 : 1), NT>();
    else bar_arrive_imm<BASE + (N == 4 ? 2 : 0), NT>();
  } else {
    if (sel == 1) bar_arrive_imm<BASE + 1, NT>();
    else bar_arrive_imm<BASE, NT>();
  }
}

// ---- row bookkeeping of the barrier-free validate kernels --------------------
// Warp gw takes rows gw, gw + nwarps, ... and stores, per row, its running
// total (inclusive) of the counts of its own rows.  The last CTA of a call with
// an error needs the count of the valid prefix: the rows before the error row
// are, for every warp w, exactly its rows up to its last one before the error
// row, so the sum is one stored running total per warp -- min(erow, nwarps)
// independent loads spread over the CTA (reading every row count, one
// dependent L2 round trip per 256 rows, made a late error cost tens of us).
__device__ __forceinline__ unsigned long long prefix_rows(const unsigned* cum, unsigned long long erow,
                                                          unsigned long long nwarps) {
  if (erow == 0) return 0;
  // warp w's last row before erow: w + nwarps * q0 if w <= (erow - 1) % nwarps,
  // else one round earlier (rows of warps w >= erow do not exist)
  const unsigned long long q0 = (erow - 1) / nwarps, r0 = (erow - 1) - q0 * nwarps;
  const unsigned long long nw = erow < nwarps ? erow : nwarps;
  unsigned long long t = 0;
#pragma unroll 4
  for (unsigned long long w = threadIdx.x; w < nw; w += blockDim.x)
    t += __ldcg(&cum[w + nwarps * (w <= r0 ? q0 : q0 - 1)]);
  return t;
}

// One step of a warp inclusive scan: x += (lane - o)'s x, when that lane exists
// (the shuffle's own in-range predicate guards the add: no compare per step).
__device__ __forceinline__ unsigned scan_step_up(unsigned x, int o) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 y;\n\t"
      "shfl.sync.up.b32 y|p, %0, %1, 0, 0xffffffff;\n\t"
      "@p add.u32 %0, %0, y;\n\t}"
      : "+r"(x)
      : "r"(o));
  return x;
}

// VT_EARLY_PUB: a tile's aggregate goes out before the block scan, not behind
// its two barriers.  Every warp adds its sum (one REDUX) to a shared 64-bit
// word (sum in the low half, arrivals in the high half); the warp that arrives
// last has the tile's total and stores the status word at once, unless the
// total carries an error count (bits kErrShift and up: those tiles publish
// their clipped count later, as before).  Every tile taken after this one
// waits for this store in its look-back, so each cycle it comes earlier is a
// cycle off their copy-out.  The last warp also re-arms the word: the others
// are held by the scan's barrier until it gets there.
#ifndef VT_EARLY_PUB
#define VT_EARLY_PUB 0
#endif
template <int THREADS>
__device__ __forceinline__ void publish_total_early(unsigned v, unsigned long long* word,
                                                    unsigned long long* status, unsigned long long flag,
                                                    unsigned epoch, int err_shift) {
  const unsigned s = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long old = atomicAdd(word, (1ull << 32) | s);
    if ((unsigned)(old >> 32) == THREADS / 32 - 1) {
      const unsigned total = (unsigned)old + s;
      *word = 0;
      if ((total >> err_shift) == 0) store_status(status, pack_status(flag, epoch, total));
    }
  }
}

// Block-wide exclusive scan of one unsigned per thread (THREADS threads).
// kTrailing: end with a barrier so warp_sums can be reused at once; callers
// that pass a barrier before the next scan anyway can drop it.
template <int THREADS, class Sync = SyncAll, bool kTrailing = true>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* warp_sums,
                                                    unsigned& total) {
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) x = scan_step_up(x, o);
  if (lane == 31) warp_sums[wid] = x;
  Sync::sync();
  if (wid == 0) {
    unsigned t = lane < THREADS / 32 ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < THREADS / 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= (unsigned)o) t += y;
    }
    if (lane < THREADS / 32) warp_sums[lane] = t;  // inclusive warp prefixes
  }
  Sync::sync();
  total = warp_sums[THREADS / 32 - 1];
  const unsigned wbase = wid ? warp_sums[wid - 1] : 0u;
  if (kTrailing) Sync::sync();  // warp_sums is reused by the next scan
  return wbase + x - v;
}

// One-barrier form: after the barrier every warp scans the (<= 32) warp sums
// itself with shuffles instead of warp 0 scanning them behind a second barrier.
// The caller must not reuse warp_sums before another barrier.
template <int THREADS, class Sync = SyncAll>
__device__ __forceinline__ unsigned block_excl_scan1(unsigned v, unsigned* warp_sums,
                                                     unsigned& total) {
  constexpr int NW = THREADS / 32;
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  Sync::sync();
  unsigned t = lane < NW ? warp_sums[lane] : 0u;
#pragma unroll
  for (int o = 1; o < NW; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
    if (lane >= (unsigned)o) t += y;
  }
  total = __shfl_sync(0xffffffffu, t, NW - 1);
  const unsigned wbase = __shfl_sync(0xffffffffu, t, (wid + 31) & 31);
  return (wid ? wbase : 0u) + x - v;
}

template <int THREADS, class Sync = SyncAll>
__device__ __forceinline__ unsigned block_min(unsigned v, unsigned* scratch) {
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) scratch[wid] = v;
  Sync::sync();
  unsigned r = scratch[0];
#pragma unroll
  for (int i = 1; i < THREADS / 32; i++) r = min(r, scratch[i]);
  Sync::sync();
  return r;
}

}  // namespace vt

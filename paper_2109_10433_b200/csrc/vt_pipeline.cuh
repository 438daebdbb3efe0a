// vt_pipeline.cuh -- the tile pipeline shared by both transcoding directions.
//
// A Codec supplies the per-tile work:
//   using Args;  (fields: base, head, n, ntiles, epoch, out, status, ctl, res)
//   using TileCount;
//   kTileElems  input elements (bytes / units) per tile
//   kStageBytes largest output of one tile, in bytes
//   kOutBytes   bytes per output element (2 for UTF-16, 1 for UTF-8)
//   kNStage     staging buffers per CTA (1 or 2, see PipeSmem)
//   count<kTranscode, NT, Sync>(a, tile, red, scan, tc, off, agg)
//       load + validate + count the tile; off = this thread's exclusive
//       output offset, agg = the tile's output (elements); errors reported
//       through atomicMin(&ctl->err) and clipped out of the counts
//   emit(a, tc, stage, off, tile, mid)  write this thread's output at stage + off
//
// transcode_body is the kernel body: warp-specialised.  Warps 0..7 count tile
// j and decode it into the staging buffer.  Warp 8 resolves tile j's offset with
// the decoupled look-back (started when tile j was taken) and, once the compute
// warps have decoded it (they arrive on the next tile's GRAB barrier), copies
// the staged tile to global memory itself while the compute warps count tile
// j+1 -- it holds none of the tile's words, so its copy loop has the registers
// the compute warps do not have (VT_LB_COPY; with 0 the compute warps copy tile
// j-1 out between the count and the decode of tile j, the round-1 form).
// Tiles are taken in order, one at a time per CTA.  (Validation and lengths
// need no offsets and use the barrier-free row kernels in k_utf8.cu /
// k_utf16.cu.)
#pragma once

#include <cstddef>
#include <cstdio>

#include "vt_device.cuh"

namespace vt {

// emit word index (of 16) after which the next tile is taken; 16: after the decode
#ifndef VT_GRAB_AT_U8
#define VT_GRAB_AT_U8 16
#endif
#ifndef VT_GRAB_AT_U16
#define VT_GRAB_AT_U16 10  // cfg3 A/B (r1n): 8 1.100, 9 1.087, 10 1.077, 11 1.082, 12 1.081 ms
#endif

// VT_LB_COPY: the look-back warp copies the staged tile out (it holds none of
// the tile's words, so its copy loop has the registers to itself, and the
// compute warps go from count straight to decode)
#ifndef VT_LB_COPY
#define VT_LB_COPY 1
#endif
// VT_BULK_COPY (with VT_LB_COPY, one staging buffer): the staged tile leaves as
// ONE asynchronous bulk copy (cp.async.bulk shared -> global, the TMA unit)
// issued by the look-back warp's leader, not as a copy loop.  A bulk copy needs
// source, destination and size in whole 16-byte chunks, and a tile's output
// starts at any element: so the compute warps wait for the tile's own offset
// before the decode (the look-back of tile j runs while tile j is counted, and
// overlaps the bulk copy of tile j-1) and stage the tile at the phase of its
// global address, (out + excl) & 15.  The look-back warp's lanes store the
// partial chunks at both ends themselves (< 16 bytes each).
#ifndef VT_BULK_COPY
#define VT_BULK_COPY 0
#endif
// VT_PREFETCH (codecs with kPrefetchBytes > 0): the next tile's input arrives in
// shared memory by one bulk copy (TMA unit) while the current tile is decoded.
// Thread 0 takes the next tile right after publishing the aggregate (the
// atomic's round trip overlaps the wait for the staging buffer), starts the
// copy before the decode, and the next count phase reads its words from shared
// memory: neither the tile id nor the input loads are waited for.
#ifndef VT_PREFETCH
#define VT_PREFETCH 0
#endif
#ifndef VT_SCAN1
#define VT_SCAN1 0  // one-barrier block scan (block_excl_scan1)
#endif
// VT_GRAB_EARLY: thread 0 takes the next tile before the copy-out of the
// previous one and publishes it before the "buffer free" barrier, so the
// loop-top barrier goes away (1: the look-back warp still gets the tile after
// the decode; 2: right after that barrier)
#ifndef VT_GRAB_EARLY
#define VT_GRAB_EARLY 0
#endif
// skip the decode and copy-out of tiles behind an error found meanwhile (the
// compute warps' own check: +2% on cfg2, r2h A/B, so off -- dead tiles skip
// their copy-out through the look-back, which gives up on them at once)
#ifndef VT_DEAD_SKIP
#define VT_DEAD_SKIP 0
#endif

#ifndef VT_COMPUTE_THREADS
#define VT_COMPUTE_THREADS 256
#endif
constexpr int kComputeThreads = VT_COMPUTE_THREADS;
constexpr int kPipeBlock = kComputeThreads + 32;
constexpr int BAR_COMPUTE = 1;
constexpr unsigned kSentinel = 0xFFFFFFFFu;
using ComputeSync = SyncNamed<BAR_COMPUTE, kComputeThreads>;

template <class Args>
__device__ __forceinline__ void finalize_if_last(const Args& a, bool transcode,
                                                 unsigned tile_elems) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long e = load_relaxed(&a.ctl->err);
      vt_result r;
      if (transcode) {
        // written = inclusive prefix of the last tile, or of the tile holding
        // the first error (its aggregate stops at that error)
        const unsigned t = e == kNoError ? a.ntiles - 1 : (unsigned)((e + a.head) / tile_elems);
        r.written = load_status(&a.status[t]) & kValMask;
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
      VT_TR_MAX(6);
    }
  }
}

// Next tile for this CTA (called by one thread).  Tiles behind a known error
// are skipped: their output can never be read (the reference stops there too).
template <class Args>
__device__ __forceinline__ unsigned grab_tile(const Args& a, unsigned tile_elems) {
  unsigned t = atomicAdd(&a.ctl->tile_counter, 1u);
  const unsigned long long e = load_relaxed(&a.ctl->err);
  if (t < a.ntiles && e != kNoError && (e + a.head) / tile_elems < t) t = a.ntiles;
  return t;
}

// Staging buffers per CTA (Codec::kNStage):
//   1: tile j-1 is copied out before tile j is decoded into the same buffer
//      (copy, barrier, emit);
//   2: tile j is decoded first and tile j-1 is copied out afterwards, which
//      gives tile j-1's look-back one more decode phase of slack before the
//      compute warps wait for its offset.
// Two buffers fit 4 CTAs per SM only for the UTF-16 -> UTF-8 tile (24 KiB of
// staging); the UTF-8 -> UTF-16 tile needs 32 KiB and uses one (measured: 4
// CTAs with one buffer beat 3 CTAs with two, 1.12 vs 1.18 ms per GiB).
template <class C>
struct PipeSmem {
  // input prefetch (VT_PREFETCH): transaction barrier, the tile the buffer holds
  // (or will hold), the buffer: 16 bytes before the tile, the tile, 16 behind
  alignas(16) unsigned long long mbar;
  unsigned pf_tile, pf_pad;
  alignas(16) uint8_t in[C::kPrefetchBytes > 0 ? C::kPrefetchBytes : 16];
  alignas(16) uint8_t pad0[32];
  alignas(16) uint8_t out[C::kNStage][C::kStageBytes + 48];  // (+16: the staging phase)
  alignas(16) uint8_t pad1[32];
  unsigned scan[kComputeThreads / 32];
  unsigned red[kComputeThreads / 32];
  unsigned tile;
  unsigned dead;  // the tile being decoded lies behind a known error
  unsigned long long err_now;  // thread 0's latest view of the error word
  // hand-off between the compute warps and the look-back warp (rings indexed
  // by the CTA-local tile number, guarded by the named barriers below)
  unsigned lb_tile[4], agg[2];
  unsigned long long excl[2];
  unsigned long long early;  // publish_total_early's sum / arrival word
};

// (vt_device.cuh's staging-store check assumes this tail size)
struct PipeTailProbe {
  static constexpr int kStageBytes = 16, kNStage = 1, kPrefetchBytes = 0;
};
static_assert(offsetof(PipeSmem<PipeTailProbe>, early) + 8 - offsetof(PipeSmem<PipeTailProbe>, scan) ==
                  kPipeTail,
              "PipeSmem tail");

template <class C>
__device__ __forceinline__ void copy_tile_out(const typename C::Args& a, const uint8_t* stage,
                                              unsigned long long excl, unsigned agg,
                                              unsigned nthreads = kComputeThreads,
                                              unsigned tid = threadIdx.x) {
  if (excl == ~0ull) return;  // a tile before this one failed: output is dead
#if VT_CHECKS
  if ((excl + agg) * C::kOutBytes > a.out_cap)
    vt_check_fail("copy-out", excl * C::kOutBytes, (unsigned long long)agg * C::kOutBytes, 0, a.out_cap);
  if (tid == 0) {
    // the staged bytes the copy-out reads lie inside the staging region
    uint32_t dsz;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
    const uint32_t s0 = smem_addr(stage), lo = smem_addr(vt_dyn_smem);
    if (s0 + agg * C::kOutBytes > lo + dsz - kPipeTail)
      vt_check_fail("staged tile", s0, agg * C::kOutBytes, lo, lo + dsz - kPipeTail);
  }
#endif
#ifdef VT_EXP_NOCOPY
  return;
#endif
  copy_out(reinterpret_cast<uint8_t*>(a.out) + excl * C::kOutBytes, stage, agg * C::kOutBytes,
           nthreads, tid);
}

// ---- input prefetch (bulk copy global -> shared with a transaction barrier) ----
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// (one thread) expect `bytes` on the barrier and start the copy that delivers them
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* mbar) {
  const uint32_t m = smem_addr(mbar);
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];" ::"r"(m),
      "r"(bytes), "r"(smem_addr(dst)), "l"(__cvta_generic_to_global(src))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned parity) {
  const uint32_t m = smem_addr(mbar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "VT_MBAR_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra VT_MBAR_WAIT;\n\t}" ::"r"(m),
      "r"(parity)
      : "memory");
}

// Writers of shared memory that an asynchronous (bulk) copy will read: orders
// their generic-proxy stores before the async proxy's reads (with the barrier
// that follows).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// (leader) the bulk copies issued so far have read their shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// The staged tile (at stage + phase, phase = the low four bits of its global
// address) to global memory, by one warp: whole 16-byte chunks as one bulk copy
// (lane 0), the partial chunk before them by lanes 0..15 and the one behind
// them by lanes 16..31, a byte each.
template <class C>
__device__ __forceinline__ void bulk_tile_out(const typename C::Args& a, const uint8_t* stage0,
                                              unsigned long long excl, unsigned agg, unsigned lane) {
  if (excl == ~0ull || agg == 0) return;  // a tile before this one failed: output is dead
#if VT_CHECKS
  if ((excl + agg) * C::kOutBytes > a.out_cap)
    vt_check_fail("copy-out", excl * C::kOutBytes, (unsigned long long)agg * C::kOutBytes, 0, a.out_cap);
#endif
#ifdef VT_EXP_NOCOPY
  return;
#endif
  uint8_t* const d0 = reinterpret_cast<uint8_t*>(a.out) + excl * C::kOutBytes;
  const unsigned len = agg * C::kOutBytes;
  const unsigned phase = (unsigned)((uintptr_t)d0 & 15u);
  // byte positions relative to the 16-byte chunk d0 lies in (= staging offsets)
  const unsigned end = phase + len;
  const unsigned body0 = phase ? 16u : 0u;  // first whole chunk
  const unsigned body1 = end & ~15u;        // behind the last whole chunk
  uint8_t* const dbase = d0 - phase;
  const uint32_t sbase = smem_addr(stage0);
  if (lane == 0 && body1 > body0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                 "cp.async.bulk.commit_group;" ::"l"(__cvta_generic_to_global(dbase + body0)),
                 "r"(sbase + body0), "r"(body1 - body0)
                 : "memory");
  }
  const unsigned tail0 = body1 > body0 ? body1 : body0;
  const unsigned pos = lane < 16 ? lane : tail0 + (lane - 16);
  const bool mine = lane < 16 ? (pos >= phase && pos < (end < body0 ? end : body0)) : pos < end;
  if (mine) {
    uint32_t b;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(sbase + pos));
    dbase[pos] = (uint8_t)b;
  }
}

// Hand-off barriers (all kPipeBlock threads), indexed by the CTA-local tile
// number j:
//   BAR_GRAB + (j & 3): compute warps arrive once tile j's id is in shared
//             memory; the look-back warp waits, then resolves tile j's
//             exclusive prefix while the compute warps count and decode it;
//   BAR_AGG + (j & 1):  compute warps arrive once tile j's aggregate is in
//             shared memory; the look-back warp waits, publishes tile j's
//             inclusive prefix;
//   BAR_DONE + (j & 1): compute warps arrive once tile j is decoded into the
//             staging buffer (VT_LB_COPY); the look-back warp waits, then
//             copies it out;
//   BAR_EXCL + (j & 1): the look-back warp arrives once it has copied tile j
//             out (VT_LB_COPY; otherwise once tile j's offset is in shared
//             memory); the compute warps wait before they decode tile j+1
//             into the same buffer (otherwise: before copying tile j out).
// bar.arrive orders the producer's prior shared-memory writes before the
// consumer's bar.sync returns, and a waiting warp issues nothing (no polling).
// At most one instance per id is pending:
//   AGG(j+2) is arrived at after the compute warps waited for EXCL(j), which
//     the look-back warp arrives at only after its wait on AGG(j);
//   EXCL(j+2) is arrived at after the look-back warp's wait on AGG(j+2), which
//     follows the compute warps' wait on EXCL(j);
//   GRAB(j+4) is arrived at after the compute warps waited for EXCL(j+2) (one
//     buffer) or EXCL(j+1) (two buffers), which the look-back warp arrives at
//     only after its wait on GRAB(j+2) or GRAB(j+1), so after GRAB(j) -- two
//     ids per kind are not enough for GRAB with two buffers, where GRAB(j+2)
//     is arrived at while the look-back warp may still be before GRAB(j+1).
constexpr int BAR_EXCL = 2, BAR_AGG = 4, BAR_GRAB = 8, BAR_DONE = 6;
// (ids as immediates, see bar_sync_sel: the kernel then books 10 or 12 barriers,
// not 16)

#ifdef VT_PHASES
// per-phase cycle totals of warp 0 of every CTA (perf probe): loop-top sync,
// count, EXCL wait, copy-out, post-copy sync, emit, grab; [7] = tiles
__device__ unsigned long long g_phase[8];
// count sub-phases (thread 0, absolute clocks summed): [0] loads arrived,
// [1] classify done; read against the count phase's start/end
__device__ unsigned long long g_phase_sub[4];
// the look-back warp's leader: wait for the staged tile, copy-out, wait for the
// next tile id, look-back, wait for the aggregate + publish; [7] = tiles
__device__ unsigned long long g_phase_lb[8];
#define VT_PHL(i)                                                              \
  do {                                                                         \
    const long long _t = clock64();                                            \
    if (leader) atomicAdd(&g_phase_lb[i], (unsigned long long)(_t - phl_t));   \
    phl_t = _t;                                                                \
  } while (0)
#define VT_PH(i)                                                  \
  do {                                                            \
    const long long _t = clock64();                               \
    if (threadIdx.x == 0) atomicAdd(&g_phase[i], (unsigned long long)(_t - ph_t)); \
    ph_t = _t;                                                    \
  } while (0)
#else
#define VT_PH(i) \
  do {           \
  } while (0)
#define VT_PHL(i) \
  do {            \
  } while (0)
#endif

template <class C>
__device__ __forceinline__ void transcode_body(const typename C::Args& a, PipeSmem<C>& sm) {
  constexpr int NS = C::kNStage;
  static_assert(NS == 1 || NS == 2, "one or two staging buffers");
  // GRAB ids: four in general (see above); with one staging buffer and the
  // plain grab two are enough -- GRAB(j+2) is arrived at after the compute warps
  // waited for EXCL(j), which the look-back warp arrives at after its wait on
  // GRAB(j+1), so GRAB(j) is complete
#ifdef VT_GRAB_IDS
  constexpr int kGrabIds = VT_GRAB_IDS;
#else
  constexpr int kGrabIds = (NS == 1 && !VT_GRAB_EARLY && VT_LB_COPY) ? 2 : 4;
#endif
  if (threadIdx.x == 0) VT_TR_MIN(0);
  if (threadIdx.x >= kComputeThreads) {
    const bool leader = threadIdx.x == kComputeThreads;
#if VT_LB_COPY
    unsigned long long excl_prev = 0;
    unsigned agg_prev = 0;
#endif
#ifdef VT_PHASES
    long long phl_t = clock64();
#endif
    for (unsigned j = 0;; j++) {
#if VT_LB_COPY
      // tile j-1 is staged completely (the compute warps arrive on DONE(j-1)
      // right after its decode, before the next tile's id is known) and its
      // offset was resolved in the previous round: copy it out, then hand the
      // buffer back (EXCL(j-1) = "copy done")
      if (j > 0) {
        bar_sync_sel<BAR_DONE, 2, kPipeBlock>((j - 1));
        VT_PHL(0);
#if VT_BULK_COPY
        bulk_tile_out<C>(a, sm.out[0], excl_prev, agg_prev, threadIdx.x - kComputeThreads);
#else
        copy_tile_out<C>(a, sm.out[(j - 1) % NS], excl_prev, agg_prev, 32u, threadIdx.x - kComputeThreads);
#endif
      }
#endif
      VT_PHL(1);
      bar_sync_sel<BAR_GRAB, kGrabIds, kPipeBlock>(j);
      VT_PHL(2);
      const unsigned tile = sm.lb_tile[j & 3];
      if (tile >= a.ntiles) break;
#if VT_LB_COPY && !VT_BULK_COPY
      // (the compute warps wait for the buffer only after counting tile j; after
      // the CTA's last tile nobody waits, so the arrival comes behind the break)
      if (j > 0) bar_arrive_sel<BAR_EXCL, 2, kPipeBlock>((j - 1));
#endif
      unsigned long long excl = 0;
      if (tile != 0) {
#ifdef VT_PROBE
        const long long t0 = clock64();
#endif
        excl = lookback(a.status, a.epoch, tile, a.ctl, C::kTileElems, a.head);
#ifdef VT_PROBE
        if (leader) {
          atomicAdd(&a.ctl->pad[0], (unsigned long long)(clock64() - t0));
          atomicAdd(&a.ctl->pad[1], 1ull);
        }
#endif
      }
      VT_PHL(3);
      bar_sync_sel<BAR_AGG, 2, kPipeBlock>(j);
      // (the compute warps already published the aggregate, tile 0 its prefix)
      if (leader && tile != 0 && excl != ~0ull)
        store_status(&a.status[tile], pack_status(kFlagPre, a.epoch, excl + sm.agg[j & 1]));
#ifdef VT_TRACE
      if (leader) {
        const unsigned long long e = load_relaxed(&a.ctl->err);
        if (e != kNoError && (e + a.head) / C::kTileElems == tile) VT_TR_MAX(4);
      }
#endif
      if (leader) sm.excl[j & 1] = excl;
      VT_PHL(4);
#ifdef VT_PHASES
      if (leader) atomicAdd(&g_phase_lb[7], 1ull);
#endif
#if VT_LB_COPY
      excl_prev = excl;
      agg_prev = sm.agg[j & 1];
#if VT_BULK_COPY
      // EXCL(j) = tile j's offset is in shared memory AND the bulk copy of tile
      // j-1 (in flight during this look-back) has read the staging buffer
      if (leader) bulk_wait_read();
      __syncwarp();
      bar_arrive_sel<BAR_EXCL, 2, kPipeBlock>(j);
#endif
#else
      bar_arrive_sel<BAR_EXCL, 2, kPipeBlock>(j);
#endif
    }
#if VT_LB_COPY && VT_BULK_COPY
    if (leader) bulk_wait_all();  // (the CTA's shared memory must outlive the last copy)
#endif
  } else {
    // compute warps
    constexpr bool kPF = VT_PREFETCH && C::kPrefetchBytes > 0 && VT_LB_COPY && !VT_BULK_COPY &&
                         NS == 1 && !VT_GRAB_EARLY && !VT_DEAD_SKIP;
    unsigned pf_parity = 0;  // phase of the prefetch barrier the next prefetched tile completes
    if (threadIdx.x == 0) {
      const unsigned t = grab_tile(a, C::kTileElems);
      sm.tile = t;
      sm.lb_tile[0] = t;
      if (kPF) {
        mbar_init(&sm.mbar, 1);
        sm.pf_tile = kSentinel;
      }
      sm.early = 0;
    }
    bar_arrive_imm<BAR_GRAB, kPipeBlock>();
    unsigned j = 0, prev_agg = 0;
#ifdef VT_PHASES
    long long ph_t = clock64();
#endif
    // tile j-1's offset was resolved meanwhile: copy it out
    auto copy_prev = [&]() {
#ifdef VT_PROBE
      const long long t0 = clock64();
#endif
      bar_sync_sel<BAR_EXCL, 2, kPipeBlock>((j - 1));
      VT_PH(2);
#ifdef VT_PROBE
      if (threadIdx.x == 0) {
        atomicAdd(&a.ctl->pad[2], (unsigned long long)(clock64() - t0));
        atomicAdd(&a.ctl->pad[3], 1ull);
      }
#endif
#if !VT_LB_COPY
      copy_tile_out<C>(a, sm.out[(j - 1) % NS], sm.excl[(j - 1) & 1], prev_agg);
#endif
      VT_PH(3);
    };
    while (true) {
      // (early grab: from the third tile on, the tile id was published before
      // the previous tile's buffer-free barrier)
      if (!VT_GRAB_EARLY || NS != 1 || j <= 1) ComputeSync::sync();
      VT_PH(0);
#ifdef VT_PHASES
      if (threadIdx.x == 0) atomicAdd(&g_phase_sub[2], (unsigned long long)ph_t);
#endif
      const unsigned tile = sm.tile;
      if (tile >= a.ntiles) break;
      // a stale error only means a dead tile is processed (its output is
      // dropped at copy-out, its look-back gives up)
      const unsigned long long err_seen = threadIdx.x == 0 ? load_relaxed(&a.ctl->err) : 0ull;
      typename C::TileCount tc;
      unsigned off, agg;
      // (prefetched: the tile's bytes are in, or on their way into, sm.in)
      const bool pf = kPF && sm.pf_tile == tile;
      if (pf) {
        mbar_wait(&sm.mbar, pf_parity);
        pf_parity ^= 1u;
      }
      C::template count<true, kComputeThreads, ComputeSync>(a, tile, sm.red, sm.scan, tc, off, agg,
                                                            pf ? sm.in : nullptr, VT_EARLY_PUB ? &sm.early : nullptr);
#ifdef VT_TRACE
      bool tr_err_tile = false;
      if (threadIdx.x == 0) {
        const unsigned long long e = load_relaxed(&a.ctl->err);
        tr_err_tile = e != kNoError && (e + a.head) / C::kTileElems == tile;
        if (tr_err_tile) VT_TR_MAX(2);
      }
#endif
      if (threadIdx.x == 0) {
        // publish the aggregate right away (tile 0: the inclusive prefix), so
        // other CTAs' look-backs never wait on this CTA's look-back warp
        // (with VT_EARLY_PUB the last warp through the count did it already,
        // except for tiles with an error or an end of the input in them)
        if (!(VT_EARLY_PUB && tc.simple))
          store_status(&a.status[tile], pack_status(tile == 0 ? kFlagPre : kFlagAgg, a.epoch, agg));
        sm.agg[j & 1] = agg;
      }
      unsigned grabbed = 0;
      // prefetch: the next tile is taken now; the atomic's round trip overlaps
      // the wait for the staging buffer
      if (kPF) atom_inc_pinned(&a.ctl->tile_counter, threadIdx.x == 0, grabbed);
      bar_arrive_sel<BAR_AGG, 2, kPipeBlock>(j);
      VT_PH(1);
#ifdef VT_PHASES
      if (threadIdx.x == 0) atomicAdd(&g_phase_sub[3], (unsigned long long)ph_t);
#endif
      bool dead = false;
      const bool early = VT_GRAB_EARLY && NS == 1 && j > 0;
      if (VT_DEAD_SKIP && threadIdx.x == 0) sm.err_now = err_seen;
#if VT_LB_COPY && VT_BULK_COPY
      static_assert(NS == 1 && !VT_GRAB_EARLY && !VT_DEAD_SKIP, "bulk copy-out: one buffer, plain grab");
      // tile j's own offset (the staging phase) and the buffer, both from the
      // look-back warp
      bar_sync_sel<BAR_EXCL, 2, kPipeBlock>(j);
      VT_PH(2);
      VT_PH(3);
      VT_PH(4);
      const unsigned long long excl_j = sm.excl[j & 1];
      // the look-back gave up on tile j: it lies behind an error; its decode
      // and copy-out are skipped
      if (excl_j == ~0ull) {
        dead = true;
        agg = 0;
      }
      const unsigned phase =
          (unsigned)(((uintptr_t)a.out + (uintptr_t)excl_j * (unsigned)C::kOutBytes) & 15u);
#else
      const unsigned phase = 0;
#endif
      if (!(VT_LB_COPY && VT_BULK_COPY) && NS == 1 && j > 0) {
        if (early) atom_inc_pinned(&a.ctl->tile_counter, threadIdx.x == 0, grabbed);
        // a tile behind an error found meanwhile is dead: its output is never
        // read, so its decode and copy-out are skipped (the load's latency
        // hides behind the copy-out; the flag goes out with the barrier below)
        unsigned long long e_now = 0;
        if (VT_DEAD_SKIP && threadIdx.x == 0) e_now = load_relaxed(&a.ctl->err);
        copy_prev();
        if (VT_DEAD_SKIP && threadIdx.x == 0) {
          sm.err_now = e_now;
          sm.dead = e_now != kNoError && (e_now + a.head) / C::kTileElems < tile ? 1u : 0u;
        }
        if (early && threadIdx.x == 0) {
          unsigned t = grabbed;
          if (t < a.ntiles && err_seen != kNoError && (err_seen + a.head) / C::kTileElems < t)
            t = a.ntiles;
          sm.tile = t;
          sm.lb_tile[(j + 1) & 3] = t;
        }
#if !VT_LB_COPY
        ComputeSync::sync();  // the buffer is free (and the next tile id is out)
#endif
        VT_PH(4);
        if (VT_DEAD_SKIP && sm.dead) agg = 0;  // (nothing staged, nothing to copy out)
        // the look-back gave up on tile j-1: it lies behind an error, and so
        // does tile j (taken later): its decode and copy-out are skipped (free:
        // the offset was waited for anyway)
        if (sm.excl[(j - 1) & 1] == ~0ull) {
          dead = true;
          agg = 0;
        }
        if (early && VT_GRAB_EARLY == 2) bar_arrive_sel<BAR_GRAB, kGrabIds, kPipeBlock>((j + 1));
      }
      // thread 0 takes the next tile from inside the decode (the codec says
      // where: Codec::emit calls `grab`); measured per codec, ms/GiB:
      //   UTF-16 -> UTF-8 after word 12 of 16: 1.231 -> 1.220 (after 4 / 8:
      //   1.270, before the decode: 1.261);
      //   UTF-8 -> UTF-16 at the end of the decode (after 12-15: +0.1-0.4 %,
      //   after 4 / 8: +0.9 %, before: +1.7 %)
      auto grab = [&]() {
        if (!early && !kPF) atom_inc_pinned(&a.ctl->tile_counter, threadIdx.x == 0, grabbed);
      };
      if (kPF && threadIdx.x == 0) {
        // the next tile's id is here (or nearly): publish it for the loop top
        // (every compute thread has read sm.tile: they all passed the scan's
        // barriers) and start its input copy; all words of this tile are in
        // registers, so the buffer is free
        unsigned t = grabbed;
        if (t < a.ntiles && err_seen != kNoError && (err_seen + a.head) / C::kTileElems < t) t = a.ntiles;
        const bool fetch = C::prefetchable(a, t);
        if (fetch) fence_proxy_async_smem();  // (the buffer's readers are behind the scan's barriers)
        if (fetch) bulk_load(sm.in, C::prefetch_src(a, t), C::kPrefetchBytes, &sm.mbar);
        sm.pf_tile = fetch ? t : kSentinel;
        sm.tile = t;
        sm.lb_tile[(j + 1) & 3] = t;
      }
#ifndef VT_EXP_NOEMIT
      if (dead || (VT_DEAD_SKIP && NS == 1 && j > 0 && sm.dead))
        grab();
      else
        C::emit(a, tc, sm.out[j % NS] + phase, off, sm.lb_tile[j & 3], grab);
#else
      grab();
#endif
#if VT_LB_COPY
      // tile j is staged: the look-back warp may copy it out now, while thread 0
      // still waits for the next tile's id (the atomic's round trip)
#if VT_BULK_COPY
      fence_proxy_async_smem();
#endif
      bar_arrive_sel<BAR_DONE, 2, kPipeBlock>(j);
#endif
      VT_PH(5);
#ifdef VT_TRACE
      if (tr_err_tile) VT_TR_MAX(3);
#endif
      if (threadIdx.x == 0 && !early && !kPF) {
        // (the error word was read at the top of the tile: one round trip
        // less on the path every warp waits for at the loop-top barrier)
        unsigned t = grabbed;
        const unsigned long long e = VT_DEAD_SKIP ? sm.err_now : err_seen;
        if (t < a.ntiles && e != kNoError && (e + a.head) / C::kTileElems < t) t = a.ntiles;
        sm.tile = t;
        sm.lb_tile[(j + 1) & 3] = t;
      }
      if (!(early && VT_GRAB_EARLY == 2)) bar_arrive_sel<BAR_GRAB, kGrabIds, kPipeBlock>((j + 1));
      VT_PH(6);
#ifdef VT_PHASES
      if (threadIdx.x == 0) atomicAdd(&g_phase[7], 1ull);
#endif
      // two buffers: tile j-1 goes out after tile j was decoded (the loop-top
      // barrier orders this copy before tile j+1 is decoded into its buffer)
      if (NS == 2 && j > 0) copy_prev();
      prev_agg = agg;
      j++;
    }
#if !VT_LB_COPY
    if (j > 0) copy_prev();
#endif
    if (threadIdx.x == 0) VT_TR_MAX(5);
  }
  finalize_if_last(a, true, C::kTileElems);
}

}  // namespace vt

// vt_pipeline.cuh -- the tile pipeline shared by both transcoding directions.
//
// A Codec supplies the per-tile work:
//   using Args;  (fields: base, head, n, ntiles, epoch, out, status, ctl, res)
//   using TileCount;
//   kTileElems  input elements (bytes / units) per tile
//   kStageBytes largest output of one tile, in bytes
//   kOutBytes   bytes per output element (2 for UTF-16, 1 for UTF-8)
//   count<kTranscode, NT, Sync>(a, tile, red, scan, tc, off, agg)
//       load + validate + count the tile; off = this thread's exclusive
//       output offset, agg = the tile's output (elements); errors reported
//       through atomicMin(&ctl->err) and clipped out of the counts
//   emit(a, tc, stage, off)  write this thread's output at stage + off
//
// transcode_body is the kernel body: warp-specialised.  Warps 0..7 count tile
// j and decode it into the staging buffer, then copy it to global memory during
// tile j+1, once warp 8 has resolved its offset with the decoupled look-back
// (started when tile j was taken).  Tiles are taken in order, one at a time per
// CTA.  (Validation and lengths need no offsets and use the barrier-free row
// kernels in k_utf8.cu / k_utf16.cu.)
#pragma once

#include "vt_device.cuh"

namespace vt {

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

// Staging buffers per CTA: 2 would let tile j be decoded while tile j-1 is
// still being copied out; 1 halves the shared memory so 4 CTAs fit per SM
// (measured: 1.12 vs 1.18 ms per GiB, cfg2), at the cost of one more barrier
// per tile.
#ifndef VT_NSTAGE
#define VT_NSTAGE 1
#endif
constexpr int kNStage = VT_NSTAGE;

template <class C>
struct PipeSmem {
  alignas(16) uint8_t pad0[32];
  alignas(16) uint8_t out[kNStage][C::kStageBytes + 32];
  alignas(16) uint8_t pad1[32];
  unsigned scan[kComputeThreads / 32];
  unsigned red[kComputeThreads / 32];
  unsigned tile;
  // hand-off between the compute warps and the look-back warp (2-slot rings
  // indexed by tile parity, guarded by the named barriers below)
  unsigned lb_tile[2], agg[2];
  unsigned long long excl[2];
};

template <class C>
__device__ __forceinline__ void copy_tile_out(const typename C::Args& a, const uint8_t* stage,
                                              unsigned long long excl, unsigned agg) {
  if (excl == ~0ull) return;  // a tile before this one failed: output is dead
#ifdef VT_EXP_NOCOPY
  return;
#endif
  copy_out(reinterpret_cast<uint8_t*>(a.out) + excl * C::kOutBytes, stage, agg * C::kOutBytes,
           kComputeThreads);
}

// Hand-off barriers (all kPipeBlock threads), two ids per kind indexed by the
// CTA-local tile number j & 1:
//   BAR_GRAB: compute warps arrive once tile j's id is in shared memory; the
//             look-back warp waits, then resolves tile j's exclusive prefix
//             while the compute warps count and decode it;
//   BAR_AGG:  compute warps arrive once tile j's aggregate is in shared memory;
//             the look-back warp waits, publishes tile j's inclusive prefix;
//   BAR_EXCL: the look-back warp arrives once tile j's offset is in shared
//             memory; the compute warps wait before copying tile j out (during
//             tile j+1).
// bar.arrive orders the producer's prior shared-memory writes before the
// consumer's bar.sync returns, and a waiting warp issues nothing (no polling).
// At most one instance per id is pending: every arrival for tile j+2 happens
// after the compute warps waited for tile j's offset, which the look-back warp
// only publishes after its waits for tile j completed.
constexpr int BAR_GRAB = 2, BAR_EXCL = 4, BAR_AGG = 6;

template <class C>
__device__ __forceinline__ void transcode_body(const typename C::Args& a, PipeSmem<C>& sm) {
  if (threadIdx.x >= kComputeThreads) {
    const bool leader = threadIdx.x == kComputeThreads;
    for (unsigned j = 0;; j++) {
      bar_sync(BAR_GRAB + (j & 1), kPipeBlock);
      const unsigned tile = sm.lb_tile[j & 1];
      if (tile >= a.ntiles) break;
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
      bar_sync(BAR_AGG + (j & 1), kPipeBlock);
      // (the compute warps already published the aggregate, tile 0 its prefix)
      if (leader && tile != 0 && excl != ~0ull)
        store_status(&a.status[tile], pack_status(kFlagPre, a.epoch, excl + sm.agg[j & 1]));
      if (leader) sm.excl[j & 1] = excl;
      bar_arrive(BAR_EXCL + (j & 1), kPipeBlock);
    }
  } else {
    // compute warps
    if (threadIdx.x == 0) {
      const unsigned t = grab_tile(a, C::kTileElems);
      sm.tile = t;
      sm.lb_tile[0] = t;
    }
    bar_arrive(BAR_GRAB, kPipeBlock);
    unsigned j = 0, prev_agg = 0;
    while (true) {
      ComputeSync::sync();
      const unsigned tile = sm.tile;
      if (tile >= a.ntiles) break;
      typename C::TileCount tc;
      unsigned off, agg;
      C::template count<true, kComputeThreads, ComputeSync>(a, tile, sm.red, sm.scan, tc, off, agg);
      if (threadIdx.x == 0) {
        // publish the aggregate right away (tile 0: the inclusive prefix), so
        // other CTAs' look-backs never wait on this CTA's look-back warp
        store_status(&a.status[tile], pack_status(tile == 0 ? kFlagPre : kFlagAgg, a.epoch, agg));
        sm.agg[j & 1] = agg;
      }
      bar_arrive(BAR_AGG + (j & 1), kPipeBlock);
      if (j > 0) {
        // tile j-1: its offset was resolved meanwhile; copy it out
#ifdef VT_PROBE
        const long long t0 = clock64();
#endif
        bar_sync(BAR_EXCL + ((j - 1) & 1), kPipeBlock);
#ifdef VT_PROBE
        if (threadIdx.x == 0) {
          atomicAdd(&a.ctl->pad[2], (unsigned long long)(clock64() - t0));
          atomicAdd(&a.ctl->pad[3], 1ull);
        }
#endif
        copy_tile_out<C>(a, sm.out[(j - 1) % kNStage], sm.excl[(j - 1) & 1], prev_agg);
        if (kNStage == 1) ComputeSync::sync();
      }
#ifndef VT_EXP_NOEMIT
      C::emit(a, tc, sm.out[j % kNStage], off);
#endif
      if (threadIdx.x == 0) {
        const unsigned t = grab_tile(a, C::kTileElems);
        sm.tile = t;
        sm.lb_tile[(j + 1) & 1] = t;
      }
      bar_arrive(BAR_GRAB + ((j + 1) & 1), kPipeBlock);
      prev_agg = agg;
      j++;
    }
    if (j > 0) {
      bar_sync(BAR_EXCL + ((j - 1) & 1), kPipeBlock);
      copy_tile_out<C>(a, sm.out[(j - 1) % kNStage], sm.excl[(j - 1) & 1], prev_agg);
    }
  }
  finalize_if_last(a, true, C::kTileElems);
}

}  // namespace vt

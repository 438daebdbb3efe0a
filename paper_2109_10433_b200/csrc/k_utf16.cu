// k_utf16.cu -- UTF-16LE -> UTF-8 transcoding (always validating) and UTF-16
// validation / code-point counting on sm_100a.
//
// Replaces the reference's 8-unit register dispatch with its pack tables and
// scalar surrogate fallback (proj/src/utf16_to_utf8.cpp:12-107) and the
// surrogate scan of proj/src/validation.cpp:51-77.  The GPU needs no tables:
// every unit's UTF-8 length is a function of the unit and its neighbours
// (<0x80: 1, <0x800: 2, high surrogate followed by low: 4, the low: 0, other
// BMP: 3) and the first error is the first unit failing the local pairing rule
// (SURVEY.md 8(a) fact C), which is exactly where the scalar decoder
// (proj/src/codec_core.cpp:74-83,106-125) stops.  Same tile pipeline as
// k_utf8.cu: smem staging with a one-unit halo, per-thread lengths, block scan,
// decoupled look-back, encode into smem, aligned 16-byte stores.
#include "vt_device.cuh"
#include "vt_kernels.h"

namespace vt {

constexpr int U16_THREADS = 256;
constexpr int U16_ROWS = 2;
constexpr int U16_ROW = U16_THREADS * 8;      // units per row
constexpr int U16_TILE = U16_ROW * U16_ROWS;  // units per tile
constexpr unsigned kNone16 = 0xFFFFFFFFu;

struct U16Smem {
  alignas(16) uint16_t in[8 + U16_TILE + 8];
  alignas(16) uint8_t out_pad[32];
  alignas(16) uint8_t out[3 * U16_TILE];
  alignas(16) uint8_t out_tail[32];
  unsigned scan[U16_THREADS / 32];
  unsigned red[U16_THREADS / 32];
  unsigned long long excl;
  unsigned tile;
};

__device__ __forceinline__ bool is_hi(unsigned u) { return (u & 0xFC00u) == 0xD800u; }
__device__ __forceinline__ bool is_lo(unsigned u) { return (u & 0xFC00u) == 0xDC00u; }

__device__ __forceinline__ void load_tile16(const U16Args& a, unsigned tile, uint16_t* in_s) {
  // virtual unit v lives at in_s[8 + v - tile*U16_TILE]; chunks are 8 units
  const unsigned long long vbase = (unsigned long long)tile * U16_TILE;
  const unsigned long long vend = a.head + a.n;
  for (int j = threadIdx.x; j < U16_TILE / 8 + 2; j += U16_THREADS) {
    const long long vc = (long long)vbase - 8 + 8LL * j;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (vc >= 0 && (unsigned long long)vc < vend && (unsigned long long)vc + 8 > a.head) {
      v = __ldcs(reinterpret_cast<const uint4*>(a.base + vc));
      if ((unsigned long long)vc < a.head || (unsigned long long)vc + 8 > vend) {
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const unsigned long long pos = (unsigned long long)vc + u;
          if (pos < a.head || pos >= vend) w[u >> 1] &= (u & 1) ? 0x0000FFFFu : 0xFFFF0000u;
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    *reinterpret_cast<uint4*>(in_s + 8 * j) = v;
  }
}

struct Row16 {
  unsigned u[8];
  unsigned prev, next;
  unsigned lo, hi;  // in-input unit positions [lo, hi)
};

__device__ __forceinline__ unsigned utf8_len(const Row16& r, int i) {
  const unsigned u = r.u[i];
  if (u < 0x80u) return 1;
  if (u < 0x800u) return 2;
  if (is_hi(u)) return 4;
  if (is_lo(u)) return 0;
  return 3;
}

__device__ __forceinline__ unsigned first_error16(const Row16& r) {
  unsigned e = kNone16;
#pragma unroll
  for (int i = 7; i >= 0; i--) {
    const unsigned u = r.u[i];
    const unsigned p = i ? r.u[i - 1] : r.prev;
    const unsigned q = i < 7 ? r.u[i + 1] : r.next;
    const bool bad = (is_lo(u) && !is_hi(p)) || (is_hi(u) && !is_lo(q));
    if (bad && (unsigned)i >= r.lo && (unsigned)i < r.hi) e = i;
  }
  return e;
}

template <bool kTranscode>
__global__ void __launch_bounds__(U16_THREADS) utf16_kernel(U16Args a) {
  __shared__ U16Smem sm;
  while (true) {
    if (threadIdx.x == 0) {
      unsigned t = atomicAdd(&a.ctl->tile_counter, 1u);
      const unsigned long long e = load_relaxed(&a.ctl->err);
      if (t < a.ntiles && e != kNoError && (e + a.head) / U16_TILE < t) t = a.ntiles;
      sm.tile = t;
    }
    __syncthreads();
    const unsigned tile = sm.tile;
    if (tile >= a.ntiles) break;
    load_tile16(a, tile, sm.in);
    __syncthreads();

    Row16 row[U16_ROWS];
    unsigned my_err = kNone16;
#pragma unroll
    for (int r = 0; r < U16_ROWS; r++) {
      const uint16_t* p = sm.in + 8 + r * U16_ROW + 8 * threadIdx.x;
      const uint4 v = *reinterpret_cast<const uint4*>(p);
      row[r].u[0] = v.x & 0xFFFF; row[r].u[1] = v.x >> 16;
      row[r].u[2] = v.y & 0xFFFF; row[r].u[3] = v.y >> 16;
      row[r].u[4] = v.z & 0xFFFF; row[r].u[5] = v.z >> 16;
      row[r].u[6] = v.w & 0xFFFF; row[r].u[7] = v.w >> 16;
      row[r].prev = p[-1];
      row[r].next = p[8];
      const long long v0 = (long long)tile * U16_TILE + r * U16_ROW + 8 * threadIdx.x;
      const long long s = (long long)a.head - v0, e = (long long)(a.head + a.n) - v0;
      row[r].lo = (unsigned)max(0LL, min(8LL, s));
      row[r].hi = (unsigned)max((long long)row[r].lo, min(8LL, e));
      const unsigned er = first_error16(row[r]);
      if (er != kNone16 && my_err == kNone16) my_err = r * U16_ROW + 8 * threadIdx.x + er;
    }
    const unsigned tile_err = block_min<U16_THREADS>(my_err, sm.red);
    unsigned cnt[U16_ROWS];
#pragma unroll
    for (int r = 0; r < U16_ROWS; r++) {
      const unsigned start = r * U16_ROW + 8 * threadIdx.x;
      unsigned lim = row[r].hi;
      if (tile_err != kNone16) lim = min(lim, tile_err <= start ? 0u : tile_err - start);
      row[r].hi = max(lim, row[r].lo);
      unsigned c = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        if ((unsigned)i >= row[r].lo && (unsigned)i < row[r].hi)
          c += kTranscode ? utf8_len(row[r], i) : (is_lo(row[r].u[i]) ? 0u : 1u);
      }
      cnt[r] = c;
    }
    if (tile_err != kNone16 && threadIdx.x == 0) {
      const unsigned long long pos = (unsigned long long)tile * U16_TILE + tile_err - a.head;
      atomicMin(&a.ctl->err, pos);
    }
    if (!kTranscode) {
      unsigned total;
      block_excl_scan<U16_THREADS>(cnt[0] + cnt[1], sm.scan, total);
      if (threadIdx.x == 0 && total) atomicAdd(&a.ctl->count, (unsigned long long)total);
      __syncthreads();
      continue;
    }
    unsigned tot0, tot1;
    const unsigned off0 = block_excl_scan<U16_THREADS>(cnt[0], sm.scan, tot0);
    const unsigned off1 = block_excl_scan<U16_THREADS>(cnt[1], sm.scan, tot1) + tot0;
    const unsigned agg = tot0 + tot1;
    if (threadIdx.x < 32) {
      unsigned long long excl = 0;
      if (tile == 0) {
        if (threadIdx.x == 0) store_status(&a.status[0], pack_status(kFlagPre, a.epoch, agg));
      } else {
        if (threadIdx.x == 0) store_status(&a.status[tile], pack_status(kFlagAgg, a.epoch, agg));
        excl = lookback(a.status, a.epoch, tile, a.ctl, U16_TILE, a.head);
        if (threadIdx.x == 0 && excl != ~0ull)
          store_status(&a.status[tile], pack_status(kFlagPre, a.epoch, excl + agg));
      }
      if (threadIdx.x == 0) sm.excl = excl;
    }
#pragma unroll
    for (int r = 0; r < U16_ROWS; r++) {
      uint8_t* d = sm.out + (r ? off1 : off0);
      unsigned q = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        if ((unsigned)i < row[r].lo || (unsigned)i >= row[r].hi) continue;
        const unsigned u = row[r].u[i];
        if (u < 0x80u) {
          d[q++] = (uint8_t)u;
        } else if (u < 0x800u) {
          d[q] = (uint8_t)(0xC0u | (u >> 6));
          d[q + 1] = (uint8_t)(0x80u | (u & 0x3Fu));
          q += 2;
        } else if (is_hi(u)) {
          const unsigned nx = i < 7 ? row[r].u[i + 1] : row[r].next;
          const unsigned cp = 0x10000u + (((u - 0xD800u) << 10) | (nx - 0xDC00u));
          d[q] = (uint8_t)(0xF0u | (cp >> 18));
          d[q + 1] = (uint8_t)(0x80u | ((cp >> 12) & 0x3Fu));
          d[q + 2] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
          d[q + 3] = (uint8_t)(0x80u | (cp & 0x3Fu));
          q += 4;
        } else if (!is_lo(u)) {
          d[q] = (uint8_t)(0xE0u | (u >> 12));
          d[q + 1] = (uint8_t)(0x80u | ((u >> 6) & 0x3Fu));
          d[q + 2] = (uint8_t)(0x80u | (u & 0x3Fu));
          q += 3;
        }
      }
    }
    __syncthreads();
    const unsigned long long excl = sm.excl;
    if (excl != ~0ull) copy_out(a.out + excl, sm.out, agg, U16_THREADS);
    __syncthreads();
  }
  // last CTA writes the result and re-arms the control block
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long e = load_relaxed(&a.ctl->err);
      vt_result r;
      if (kTranscode) {
        const unsigned t = e == kNoError ? a.ntiles - 1 : (unsigned)((e + a.head) / U16_TILE);
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

int launch_utf16(const U16Args& a, bool transcode, int grid, cudaStream_t s) {
  if (transcode)
    utf16_kernel<true><<<grid, U16_THREADS, 0, s>>>(a);
  else
    utf16_kernel<false><<<grid, U16_THREADS, 0, s>>>(a);
  return (int)cudaGetLastError();
}

int occupancy_utf16(bool transcode) {
  int n = 0;
  if (transcode)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf16_kernel<true>, U16_THREADS, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, utf16_kernel<false>, U16_THREADS, 0);
  return n;
}

unsigned tiles_utf16(unsigned long long head, unsigned long long n) {
  const unsigned long long t = (head + n + U16_TILE - 1) / U16_TILE;
  return (unsigned)(t ? t : 1);
}

}  // namespace vt

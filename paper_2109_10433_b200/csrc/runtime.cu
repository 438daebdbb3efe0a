// runtime.cu -- the C ABI of libvtrans_gpu.so (include/vtrans_gpu.h).
//
// Owns per-(device, stream) scratch for the single-pass kernels (control block,
// epoch-tagged tile status array, device result), the per-thread host contexts
// behind the host-pointer entry points (stream, pinned mapped staging, device
// buffers), and the multi-GPU sharder.  No entry point computes anything on the
// CPU: a missing device is an error (VT_E_NODEVICE), never a fallback.
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <deque>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/vtrans_gpu.h"
#include "vt_device.cuh"
#include "vt_kernels.h"

#ifdef VT_TRACE
namespace vt {
int read_trace8(unsigned long long* out16);
int read_trace16(unsigned long long* out16);
}  // namespace vt
extern "C" int vt_debug_trace(int utf16, uint64_t* out16) {
  return utf16 ? vt::read_trace16(reinterpret_cast<unsigned long long*>(out16))
               : vt::read_trace8(reinterpret_cast<unsigned long long*>(out16));
}
#endif
#ifdef VT_PHASES
namespace vt {
int read_phases(unsigned long long* out8);
int read_phases16(unsigned long long* out8);
}  // namespace vt
#endif
extern "C" uint64_t vt_split_point_utf8(const uint8_t* in, uint64_t n, uint64_t cut);
extern "C" uint64_t vt_split_point_utf16(const uint16_t* in, uint64_t n, uint64_t cut);

#ifndef VT_PIPE_BUFS
#define VT_PIPE_BUFS 3
#endif
#ifndef VT_PIPE_CHUNK_MB
#define VT_PIPE_CHUNK_MB 32
#endif

namespace {

std::atomic<uint64_t> g_launches{0};

#define VT_STR2(x) #x
#define VT_STR(x) VT_STR2(x)

#define VT_TRY(expr)                    \
  do {                                  \
    const int rc_ = (int)(expr);        \
    if (rc_ != 0) return rc_;           \
  } while (0)

struct DeviceInfo {
  int sms = 0;
  int occ_u8[2] = {0, 0};
  int occ_u16[2] = {0, 0};
  bool ok = false;
};

std::mutex g_dev_mu;
std::map<int, DeviceInfo> g_devs;

int device_info(int dev, DeviceInfo& out) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_devs.find(dev);
  if (it != g_devs.end()) {
    out = it->second;
    return 0;
  }
  cudaDeviceProp p;
  VT_TRY(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10) return VT_E_ARCH;
  DeviceInfo d;
  d.sms = p.multiProcessorCount;
  d.occ_u8[0] = std::max(1, vt::occupancy_utf8(false));
  d.occ_u8[1] = std::max(1, vt::occupancy_utf8(true));
  d.occ_u16[0] = std::max(1, vt::occupancy_utf16(false));
  d.occ_u16[1] = std::max(1, vt::occupancy_utf16(true));
  // (perf probe: VT_OCC_CAP=k launches the transcode kernels with at most k CTAs per SM)
  if (const char* cap = std::getenv("VT_OCC_CAP")) {
    const int k = std::max(1, std::atoi(cap));
    d.occ_u8[1] = std::min(d.occ_u8[1], k);
    d.occ_u16[1] = std::min(d.occ_u16[1], k);
  }
  if (std::getenv("VT_PRINT_OCC"))
    std::fprintf(stderr, "vtrans: CTAs/SM utf8 validate %d transcode %d, utf16 validate %d transcode %d\n",
                 d.occ_u8[0], d.occ_u8[1], d.occ_u16[0], d.occ_u16[1]);
  d.ok = true;
  g_devs[dev] = d;
  out = d;
  return 0;
}

int current_device(int& dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return VT_E_NODEVICE;
  }
  VT_TRY(cudaGetDevice(&dev));
  return 0;
}

// Scratch for the kernels enqueued on one stream of one device.  Calls on the
// same stream are ordered by the stream, so one scratch serves them all; the
// mutex only guards the host-side bookkeeping (epoch, growth).
struct Scratch {
  std::mutex mu;
  int dev = -1;
  vt::Ctl* ctl = nullptr;
  unsigned long long* status = nullptr;
  size_t status_cap = 0;  // tiles
  unsigned epoch = 0;
  vt_result* d_res = nullptr;  // device result slot for the synchronous API
  vt_result* h_res = nullptr;  // pinned host mirror
  unsigned* rows = nullptr;    // per-row counts of the validate kernels
  size_t rows_cap = 0;
};

// Per-row running totals of the validate kernels (prefix_rows).
int ensure_rows(Scratch& sc, cudaStream_t s, size_t rows) {
  if (rows <= sc.rows_cap) return 0;
  VT_TRY(cudaStreamSynchronize(s));  // the old array may still be in use
  if (sc.rows) VT_TRY(cudaFree(sc.rows));
  const size_t cap = std::max<size_t>(rows, 1u << 19);
  VT_TRY(cudaMalloc(&sc.rows, cap * sizeof(unsigned)));
  sc.rows_cap = cap;
  return 0;
}

// Scratch is keyed by the stream's unique id (cudaStreamGetId), not its handle:
// the special handles (legacy default stream, cudaStreamPerThread) name a
// different real stream in every host thread, and two threads on
// cudaStreamPerThread must not share a control block while their kernels run
// concurrently.  Ids are never reused, so entries of destroyed streams are
// evicted once the table grows past kScratchMax: an entry nobody holds (use
// count 1) is freed after a device synchronize (its last kernels may still be
// in flight on the dead stream).
constexpr size_t kScratchMax = 64;
std::mutex g_scratch_mu;
std::map<std::pair<int, unsigned long long>, std::shared_ptr<Scratch>> g_scratch;

void free_scratch(Scratch& sc) {
  if (sc.ctl) cudaFree(sc.ctl);
  if (sc.status) cudaFree(sc.status);
  if (sc.d_res) cudaFree(sc.d_res);
  if (sc.h_res) cudaFreeHost(sc.h_res);
  if (sc.rows) cudaFree(sc.rows);
  sc.ctl = nullptr;
  sc.status = nullptr;
  sc.d_res = nullptr;
  sc.h_res = nullptr;
  sc.rows = nullptr;
}

// (caller holds g_scratch_mu; `keep` is the entry being handed out)
void evict_idle_scratch(const Scratch* keep) {
  int cur = -1;
  cudaGetDevice(&cur);
  for (auto it = g_scratch.begin(); it != g_scratch.end();) {
    if (it->second.get() != keep && it->second.use_count() == 1) {
      cudaSetDevice(it->second->dev);
      cudaDeviceSynchronize();
      free_scratch(*it->second);
      it = g_scratch.erase(it);
    } else {
      ++it;
    }
  }
  if (cur >= 0) cudaSetDevice(cur);
}

int scratch_for(int dev, cudaStream_t s, std::shared_ptr<Scratch>& out) {
  unsigned long long id = 0;
  VT_TRY(cudaStreamGetId(s, &id));
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  auto& p = g_scratch[{dev, id}];
  if (!p) {
    p = std::make_shared<Scratch>();
    p->dev = dev;
    if (g_scratch.size() > kScratchMax) evict_idle_scratch(p.get());
  }
  out = p;
  return 0;
}

// The kernels' control blocks carry host-side state (the status epoch, grown
// arrays), so a call cannot be recorded into a CUDA graph: every replay would
// reuse one epoch and read stale tile prefixes.  Capture is refused.
int refuse_capture(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  VT_TRY(cudaStreamIsCapturing(s, &st));
  return st == cudaStreamCaptureStatusNone ? 0 : VT_E_ARG;
}

// Ensures capacity for `tiles` status words and returns the epoch to use.
int prepare(Scratch& sc, cudaStream_t s, unsigned tiles, unsigned& epoch) {
  if (!sc.ctl) {
    VT_TRY(cudaMalloc(&sc.ctl, sizeof(vt::Ctl)));
    vt::Ctl init{};
    init.err = vt::kNoError;
    // stream-ordered: a non-blocking stream does not wait for the legacy
    // default stream, where the synchronous forms would be queued
    VT_TRY(cudaMemcpyAsync(sc.ctl, &init, sizeof init, cudaMemcpyHostToDevice, s));
    VT_TRY(cudaStreamSynchronize(s));  // `init` is a host stack object
  }
  if (tiles > sc.status_cap) {
    VT_TRY(cudaStreamSynchronize(s));  // the old array may still be in use
    if (sc.status) VT_TRY(cudaFree(sc.status));
    size_t cap = std::max<size_t>(tiles, 1u << 16);
    VT_TRY(cudaMalloc(&sc.status, cap * sizeof(unsigned long long)));
    VT_TRY(cudaMemsetAsync(sc.status, 0, cap * sizeof(unsigned long long), s));
    sc.status_cap = cap;
    sc.epoch = 0;
  }
  sc.epoch = (sc.epoch + 1) & 0x3FFF;
  if (sc.epoch == 0) {
    // epoch wrapped: clear stale tags so no old status can match a new epoch
    VT_TRY(cudaMemsetAsync(sc.status, 0, sc.status_cap * sizeof(unsigned long long), s));
    sc.epoch = 1;
  }
  epoch = sc.epoch;
  return 0;
}

int grid_for(unsigned tiles, int occ, int sms) {
  const long long g = (long long)occ * sms;
  return (int)std::max(1LL, std::min<long long>(tiles, g));
}

// Enqueues one UTF-8 kernel; the caller holds sc.mu.
int run_utf8_locked(Scratch* sc, const DeviceInfo& di, const uint8_t* d_in, uint64_t n,
                    uint16_t* d_out, vt_result* d_res, cudaStream_t s, int mode,
                    const unsigned* d_skip = nullptr) {
  const bool transcode = mode == vt::kModeTranscode || mode == vt::kModeTranscodeBE ||
                         mode == vt::kModeTranscodeNV;
  if (!d_res || (n && !d_in) || (transcode && n && !d_out)) return VT_E_ARG;
  vt::U8Args a;
  const uintptr_t p = (uintptr_t)d_in;
  a.head = p & 15;
  a.base = reinterpret_cast<const uint8_t*>(p - a.head);
  a.n = n;
  a.ntiles = vt::tiles_utf8(a.head, n);
  static const unsigned dbg = [] {
    const char* e = std::getenv("VT_DEBUG");
    return e ? (unsigned)std::strtoul(e, nullptr, 0) : 0u;
  }();
  a.dbg = dbg;
  a.skip = d_skip;
  a.rows = nullptr;
  a.out_cap = 2 * n;  // the contract: n units
  if (!transcode) {
    const unsigned rows = vt::rows_utf8(a.head, n);
    VT_TRY(ensure_rows(*sc, s, rows));
    a.rows = sc->rows;
  }
  VT_TRY(prepare(*sc, s, a.ntiles, a.epoch));
  a.out = d_out;
  a.status = sc->status;
  a.ctl = sc->ctl;
  a.res = d_res;
  const int grid = grid_for(a.ntiles, di.occ_u8[transcode], di.sms);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_utf8(a, mode, grid, s);
}

int run_utf16_locked(Scratch* sc, const DeviceInfo& di, const uint16_t* d_in, uint64_t n,
                     uint8_t* d_out, vt_result* d_res, cudaStream_t s, int mode) {
  const bool transcode = mode == vt::kModeTranscode || mode == vt::kModeTranscodeBE;
  if (!d_res || (n && !d_in) || (transcode && n && !d_out)) return VT_E_ARG;
  if (((uintptr_t)d_in & 1) != 0) return VT_E_ARG;
  vt::U16Args a;
  const uintptr_t p = (uintptr_t)d_in;
  a.head = (p & 15) >> 1;
  a.base = reinterpret_cast<const uint16_t*>(p - (p & 15));
  a.n = n;
  a.ntiles = vt::tiles_utf16(a.head, n);
  a.rows = nullptr;
  a.out_cap = 3 * n + 16;  // the contract: 3n + 16 bytes
  if (!transcode) {
    const unsigned rows = vt::rows_utf16(a.head, n);
    VT_TRY(ensure_rows(*sc, s, rows));
    a.rows = sc->rows;
  }
  VT_TRY(prepare(*sc, s, a.ntiles, a.epoch));
  a.out = d_out;
  a.status = sc->status;
  a.ctl = sc->ctl;
  a.res = d_res;
  const int grid = grid_for(a.ntiles, di.occ_u16[transcode], di.sms);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_utf16(a, mode, grid, s);
}

struct Target {
  std::shared_ptr<Scratch> hold;  // keeps the entry alive while in use
  Scratch* sc = nullptr;
  DeviceInfo di;
};

int target(cudaStream_t s, Target& t) {
  int dev;
  VT_TRY(current_device(dev));
  VT_TRY(device_info(dev, t.di));
  VT_TRY(refuse_capture(s));
  VT_TRY(scratch_for(dev, s, t.hold));
  t.sc = t.hold.get();
  return 0;
}

int run_utf8(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* d_res, cudaStream_t s,
             int mode) {
  Target t;
  VT_TRY(target(s, t));
  std::lock_guard<std::mutex> lk(t.sc->mu);
  return run_utf8_locked(t.sc, t.di, d_in, n, d_out, d_res, s, mode);
}

int run_utf16(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* d_res, cudaStream_t s,
              int mode) {
  Target t;
  VT_TRY(target(s, t));
  std::lock_guard<std::mutex> lk(t.sc->mu);
  return run_utf16_locked(t.sc, t.di, d_in, n, d_out, d_res, s, mode);
}

// Enqueues through `enqueue(scratch, devinfo, d_res)` and returns the result to
// host memory.  The scratch lock is held throughout, so the scratch's result
// slots are never shared between concurrent callers of one stream.
template <class F>
int sync_result(cudaStream_t s, vt_result* h_res, F&& enqueue) {
  if (!h_res) return VT_E_ARG;
  Target t;
  VT_TRY(target(s, t));
  Scratch* sc = t.sc;
  std::lock_guard<std::mutex> lk(sc->mu);
  if (!sc->d_res) {
    VT_TRY(cudaMalloc(&sc->d_res, sizeof(vt_result)));
    VT_TRY(cudaMallocHost(&sc->h_res, sizeof(vt_result)));
  }
  VT_TRY(enqueue(sc, t.di, sc->d_res));
  VT_TRY(cudaMemcpyAsync(sc->h_res, sc->d_res, sizeof(vt_result), cudaMemcpyDeviceToHost, s));
  VT_TRY(cudaStreamSynchronize(s));
  *h_res = *sc->h_res;
  return 0;
}

// ---- per-thread host contexts for the host-pointer API -----------------------
constexpr uint64_t kZeroCopyMax = 64 * 1024;  // bytes of input

struct HostCtx {
  int dev = -1;
  cudaStream_t stream = nullptr;
  uint8_t* h_in = nullptr;   // pinned, mapped
  uint8_t* h_out = nullptr;  // pinned, mapped
  vt_result* h_res = nullptr;
  vt_result* d_res = nullptr;
  vt_utf8_stream* h_vs = nullptr;  // pinned: streaming-validator state in flight
  vt_utf8_stream* d_vs = nullptr;
  unsigned long long* d_counts = nullptr;  // 4 class counters
  unsigned long long* h_counts = nullptr;
  uint8_t* d_in = nullptr;
  uint8_t* d_out = nullptr;
  size_t d_in_cap = 0, d_out_cap = 0;
  // chunked pipeline (large host-pointer calls): kPipeBufs streams and buffers
  static constexpr int kPipeBufs = VT_PIPE_BUFS;
  cudaStream_t ps[kPipeBufs] = {};
  cudaEvent_t pev[kPipeBufs] = {};
  uint8_t* pd_in[kPipeBufs] = {};
  uint8_t* pd_out[kPipeBufs] = {};
  size_t pd_in_cap = 0, pd_out_cap = 0;
  vt_result* pd_res = nullptr;   // kPipeBufs slots, device
  vt_result* ph_res = nullptr;   // kPipeBufs slots, pinned host
  uint8_t* ph_in[kPipeBufs] = {};   // pinned staging for pageable callers
  uint8_t* ph_out[kPipeBufs] = {};
  size_t ph_in_cap = 0, ph_out_cap = 0;
  ~HostCtx() {
    // process teardown: the driver reclaims everything; avoid CUDA calls here
  }
};

thread_local std::map<int, HostCtx> t_ctx;
// bytes moved host<->device by this thread's host-pointer calls (copies, and
// mapped-memory reads/writes of the zero-copy path)
thread_local uint64_t t_h2d = 0, t_d2h = 0;

int host_ctx(HostCtx*& out) {
  int dev;
  VT_TRY(current_device(dev));
  DeviceInfo di;
  VT_TRY(device_info(dev, di));
  HostCtx& c = t_ctx[dev];
  if (!c.stream) {
    VT_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    VT_TRY(cudaHostAlloc(&c.h_in, kZeroCopyMax + 64, cudaHostAllocMapped));
    VT_TRY(cudaHostAlloc(&c.h_out, 3 * kZeroCopyMax + 64, cudaHostAllocMapped));
    VT_TRY(cudaHostAlloc(&c.h_res, sizeof(vt_result), cudaHostAllocMapped));
    VT_TRY(cudaMalloc(&c.d_res, sizeof(vt_result)));
    VT_TRY(cudaHostAlloc(&c.h_vs, sizeof(vt_utf8_stream), cudaHostAllocDefault));
    VT_TRY(cudaMalloc(&c.d_vs, sizeof(vt_utf8_stream)));
    VT_TRY(cudaHostAlloc(&c.h_counts, 4 * sizeof(unsigned long long), cudaHostAllocDefault));
    VT_TRY(cudaMalloc(&c.d_counts, 4 * sizeof(unsigned long long)));
    c.dev = dev;
  }
  out = &c;
  return 0;
}

int ensure_dev(uint8_t*& p, size_t& cap, size_t need, cudaStream_t s) {
  if (need <= cap) return 0;
  VT_TRY(cudaStreamSynchronize(s));
  if (p) VT_TRY(cudaFree(p));
  size_t c = std::max(need + need / 4, (size_t)1 << 20);
  VT_TRY(cudaMalloc(&p, c));
  cap = c;
  return 0;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_pinned(uint8_t*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return 0;
  if (p) VT_TRY(cudaFreeHost(p));
  VT_TRY(cudaMallocHost(&p, need));
  cap = need;
  return 0;
}

// Host copies between a caller's pageable buffer and the pinned staging of the
// pipelined path, split over a small pool of persistent threads (one thread
// moves ~5-10 GB/s; the pageable drop-in case -- a reference caller passing a
// std::vector -- is bound by these copies, not by PCIe).  The calling thread
// takes part; the pool is never destroyed (its workers idle at exit).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();
    return *p;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < 2 * kPiece || nthreads_ == 0) {
      std::memcpy(dst, src, bytes);
      return;
    }
    auto job = std::make_shared<Job>();
    job->dst = static_cast<uint8_t*>(dst);
    job->src = static_cast<const uint8_t*>(src);
    job->bytes = bytes;
    job->pieces = (bytes + kPiece - 1) / kPiece;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      gen_++;
    }
    cv_.notify_all();
    job->work();
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [&] { return job->done.load() == job->pieces; });
  }

 private:
  static constexpr size_t kPiece = 1u << 20;
  struct Job {
    uint8_t* dst = nullptr;
    const uint8_t* src = nullptr;
    size_t bytes = 0, pieces = 0;
    std::atomic<size_t> next{0}, done{0};
    std::mutex mu;
    std::condition_variable cv;
    void work() {
      size_t k;
      while ((k = next.fetch_add(1)) < pieces) {
        const size_t off = k * kPiece, len = std::min(kPiece, bytes - off);
        std::memcpy(dst + off, src + off, len);
        if (done.fetch_add(1) + 1 == pieces) {
          std::lock_guard<std::mutex> lk(mu);
          cv.notify_all();
        }
      }
    }
  };
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = hw >= 4 ? std::min(7u, hw / 2) : 0u;
    for (unsigned i = 0; i < nthreads_; i++)
      std::thread([this] {
        uint64_t seen = 0;
        for (;;) {
          std::shared_ptr<Job> job;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            job = job_;
          }
          job->work();
        }
      }).detach();
  }
  unsigned nthreads_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  std::shared_ptr<Job> job_;
};

// Input elements per pipeline chunk (VT_PIPE_CHUNK_MB MiB of input).
template <class In>
constexpr uint64_t pipe_chunk() { return ((uint64_t)VT_PIPE_CHUNK_MB << 20) / sizeof(In); }

// Large host-pointer calls: the input is cut at character boundaries into
// 32 MiB chunks (SURVEY.md 8(a) rules D/E, the same split as the sharder) and
// streamed round-robin through three CUDA streams, so host->device copies,
// kernels and device->host copies of neighbouring chunks overlap.
// Per-chunk results combine exactly: written adds up, the first failing
// chunk decides.  Pageable caller buffers go through pinned staging.
template <class In, class Out, class Run, class Split>
int host_transcode_pipelined(HostCtx* c, const In* in, uint64_t n, Out* out,
                             uint64_t out_cap_elems, vt_result* res, Run run, Split split,
                             uint64_t out_mult) {
  const uint64_t C = pipe_chunk<In>();
  std::vector<uint64_t> st{0};
  while (st.back() < n) {
    const uint64_t cut = std::min(n, st.back() + C);
    uint64_t s2 = cut < n ? split(in, n, cut) : n;
    if (s2 <= st.back()) s2 = cut;  // no valid character spans the cut
    st.push_back(s2);
  }
  const size_t K = st.size() - 1;
  const size_t in_cap = (C + 16) * sizeof(In), out_cap = (C * out_mult + 32) * sizeof(Out);
  for (int i = 0; i < HostCtx::kPipeBufs; i++) {
    if (!c->ps[i]) {
      VT_TRY(cudaStreamCreateWithFlags(&c->ps[i], cudaStreamNonBlocking));
      VT_TRY(cudaEventCreateWithFlags(&c->pev[i], cudaEventDisableTiming));
    }
  }
  if (c->pd_in_cap < in_cap || c->pd_out_cap < out_cap) {
    for (int i = 0; i < HostCtx::kPipeBufs; i++) {
      VT_TRY(cudaStreamSynchronize(c->ps[i]));
      if (c->pd_in[i]) VT_TRY(cudaFree(c->pd_in[i]));
      if (c->pd_out[i]) VT_TRY(cudaFree(c->pd_out[i]));
      VT_TRY(cudaMalloc(&c->pd_in[i], in_cap));
      VT_TRY(cudaMalloc(&c->pd_out[i], out_cap));
    }
    c->pd_in_cap = in_cap;
    c->pd_out_cap = out_cap;
  }
  if (!c->pd_res) {
    VT_TRY(cudaMalloc(&c->pd_res, HostCtx::kPipeBufs * sizeof(vt_result)));
    VT_TRY(cudaMallocHost(&c->ph_res, HostCtx::kPipeBufs * sizeof(vt_result)));
  }
  const bool pin_in = host_pinned(in), pin_out = host_pinned(out);
  if (!pin_in)
    for (int i = 0; i < HostCtx::kPipeBufs; i++) {
      size_t cap = c->ph_in_cap;
      VT_TRY(ensure_pinned(c->ph_in[i], cap, in_cap));
      if (i == HostCtx::kPipeBufs - 1) c->ph_in_cap = cap;
    }
  if (!pin_out)
    for (int i = 0; i < HostCtx::kPipeBufs; i++) {
      size_t cap = c->ph_out_cap;
      VT_TRY(ensure_pinned(c->ph_out[i], cap, out_cap));
      if (i == HostCtx::kPipeBufs - 1) c->ph_out_cap = cap;
    }
  auto issue = [&](size_t k) -> int {
    const int b = (int)(k % HostCtx::kPipeBufs);
    cudaStream_t s = c->ps[b];
    const uint64_t len = st[k + 1] - st[k];
    const In* src = in + st[k];
    if (!pin_in) {
      // the staging buffer was last read by chunk k-3's copy, which finished
      // before its result was read
      CopyPool::get().copy(c->ph_in[b], src, len * sizeof(In));
      src = reinterpret_cast<const In*>(c->ph_in[b]);
    }
    VT_TRY(cudaMemcpyAsync(c->pd_in[b], src, len * sizeof(In), cudaMemcpyHostToDevice, s));
    t_h2d += len * sizeof(In);
    t_d2h += sizeof(vt_result);
    VT_TRY(run(reinterpret_cast<const In*>(c->pd_in[b]), len, reinterpret_cast<Out*>(c->pd_out[b]),
               c->pd_res + b, s));
    VT_TRY(cudaMemcpyAsync(c->ph_res + b, c->pd_res + b, sizeof(vt_result),
                           cudaMemcpyDeviceToHost, s));
    VT_TRY(cudaEventRecord(c->pev[b], s));
    return 0;
  };
  // Every exit below drains all pipeline streams first: no copy may still read
  // the caller's input or write the caller's output after the call returns.
  int rc = 0;
  for (size_t k = 0; k < K && k < (size_t)HostCtx::kPipeBufs && rc == 0; k++) rc = issue(k);
  uint64_t written = 0;
  res->error_at = -1;
  res->consumed = n;
  for (size_t k = 0; k < K && rc == 0; k++) {
    const int b = (int)(k % HostCtx::kPipeBufs);
    rc = (int)cudaEventSynchronize(c->pev[b]);
    if (rc) break;
    const vt_result r = c->ph_res[b];
    if (written + r.written > out_cap_elems) {
      rc = VT_E_ARG;
      break;
    }
    t_d2h += r.written * sizeof(Out);
    if (r.written) {
      if (pin_out) {
        rc = (int)cudaMemcpyAsync(out + written, c->pd_out[b], r.written * sizeof(Out),
                                  cudaMemcpyDeviceToHost, c->ps[b]);
      } else {
        rc = (int)cudaMemcpyAsync(c->ph_out[b], c->pd_out[b], r.written * sizeof(Out),
                                  cudaMemcpyDeviceToHost, c->ps[b]);
        if (!rc) rc = (int)cudaStreamSynchronize(c->ps[b]);
        if (!rc) CopyPool::get().copy(out + written, c->ph_out[b], r.written * sizeof(Out));
      }
      if (rc) break;
    }
    written += r.written;
    if (r.error_at >= 0) {
      res->error_at = (int64_t)st[k] + r.error_at;
      res->consumed = (uint64_t)res->error_at;
      break;
    }
    if (k + HostCtx::kPipeBufs < K) rc = issue(k + HostCtx::kPipeBufs);
  }
  for (int i = 0; i < HostCtx::kPipeBufs; i++) {
    const int r2 = (int)cudaStreamSynchronize(c->ps[i]);
    if (!rc) rc = r2;
  }
  res->written = written;
  return rc;
}

template <class In, class Out, class Run>
int host_transcode(const In* in, uint64_t n, Out* out, uint64_t out_cap_elems, vt_result* res,
                   Run run) {
  if (!res || (n && (!in || !out))) return VT_E_ARG;
  HostCtx* c;
  VT_TRY(host_ctx(c));
  const size_t in_bytes = n * sizeof(In);
  if (in_bytes <= kZeroCopyMax) {
    // one launch, no copies: the kernel reads and writes mapped pinned memory
    if (n) std::memcpy(c->h_in, in, in_bytes);
    In* din;
    Out* dout;
    vt_result* dres;
    VT_TRY(cudaHostGetDevicePointer((void**)&din, c->h_in, 0));
    VT_TRY(cudaHostGetDevicePointer((void**)&dout, c->h_out, 0));
    VT_TRY(cudaHostGetDevicePointer((void**)&dres, c->h_res, 0));
    VT_TRY(run(din, n, dout, dres, c->stream));
    VT_TRY(cudaStreamSynchronize(c->stream));
    *res = *c->h_res;
    t_h2d += in_bytes;
    t_d2h += res->written * sizeof(Out) + sizeof(vt_result);
    if (res->written > out_cap_elems) return VT_E_ARG;
    if (res->written) std::memcpy(out, c->h_out, res->written * sizeof(Out));
    return 0;
  }
  if (sizeof(In) == 1)
    return host_transcode_pipelined(c, in, n, out, out_cap_elems, res, run,
                                    [](const In* p, uint64_t m, uint64_t cut) {
                                      return vt_split_point_utf8(
                                          reinterpret_cast<const uint8_t*>(p), m, cut);
                                    },
                                    1);
  return host_transcode_pipelined(c, in, n, out, out_cap_elems, res, run,
                                  [](const In* p, uint64_t m, uint64_t cut) {
                                    return vt_split_point_utf16(
                                        reinterpret_cast<const uint16_t*>(p), m, cut);
                                  },
                                  3);
}

template <class In, class Run>
int host_validate(const In* in, uint64_t n, vt_result* res, Run run) {
  if (!res || (n && !in)) return VT_E_ARG;
  HostCtx* c;
  VT_TRY(host_ctx(c));
  const size_t in_bytes = n * sizeof(In);
  if (in_bytes <= kZeroCopyMax) {
    if (n) std::memcpy(c->h_in, in, in_bytes);
    In* din;
    vt_result* dres;
    VT_TRY(cudaHostGetDevicePointer((void**)&din, c->h_in, 0));
    VT_TRY(cudaHostGetDevicePointer((void**)&dres, c->h_res, 0));
    VT_TRY(run(din, n, dres, c->stream));
    VT_TRY(cudaStreamSynchronize(c->stream));
    *res = *c->h_res;
    return 0;
  }
  VT_TRY(ensure_dev(c->d_in, c->d_in_cap, in_bytes, c->stream));
  VT_TRY(cudaMemcpyAsync(c->d_in, in, in_bytes, cudaMemcpyHostToDevice, c->stream));
  VT_TRY(run(reinterpret_cast<const In*>(c->d_in), n, c->d_res, c->stream));
  VT_TRY(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(vt_result), cudaMemcpyDeviceToHost, c->stream));
  VT_TRY(cudaStreamSynchronize(c->stream));
  *res = *c->h_res;
  return 0;
}

}  // namespace

extern "C" {

int vt_utf8_to_utf16_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* d_res,
                           vt_stream stream) {
  return run_utf8(d_in, n, d_out, d_res, (cudaStream_t)stream, vt::kModeTranscode);
}

int vt_utf16_to_utf8_async(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* d_res,
                           vt_stream stream) {
  return run_utf16(d_in, n, d_out, d_res, (cudaStream_t)stream, vt::kModeTranscode);
}

int vt_validate_utf8_async(const uint8_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream) {
  return run_utf8(d_in, n, nullptr, d_res, (cudaStream_t)stream, vt::kModeValidate);
}

int vt_validate_utf16_async(const uint16_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream) {
  return run_utf16(d_in, n, nullptr, d_res, (cudaStream_t)stream, vt::kModeValidate);
}

int vt_utf8_to_utf16(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* h_res,
                     vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf8_locked(sc, di, d_in, n, d_out, d, s, vt::kModeTranscode);
  });
}

int vt_utf16_to_utf8(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* h_res,
                     vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf16_locked(sc, di, d_in, n, d_out, d, s, vt::kModeTranscode);
  });
}

int vt_validate_utf8(const uint8_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf8_locked(sc, di, d_in, n, nullptr, d, s, vt::kModeValidate);
  });
}

int vt_validate_utf16(const uint16_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf16_locked(sc, di, d_in, n, nullptr, d, s, vt::kModeValidate);
  });
}

// ---- output lengths (vt_utf16_len_from_utf8 / vt_utf8_len_from_utf16)

int vt_utf16_len_from_utf8_async(const uint8_t* d_in, uint64_t n, vt_result* d_res,
                                 vt_stream stream) {
  return run_utf8(d_in, n, nullptr, d_res, (cudaStream_t)stream, vt::kModeLength);
}

int vt_utf8_len_from_utf16_async(const uint16_t* d_in, uint64_t n, vt_result* d_res,
                                 vt_stream stream) {
  return run_utf16(d_in, n, nullptr, d_res, (cudaStream_t)stream, vt::kModeLength);
}

int vt_utf16_len_from_utf8(const uint8_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf8_locked(sc, di, d_in, n, nullptr, d, s, vt::kModeLength);
  });
}

int vt_utf8_len_from_utf16(const uint16_t* d_in, uint64_t n, vt_result* h_res, vt_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return sync_result(s, h_res, [&](Scratch* sc, const DeviceInfo& di, vt_result* d) {
    return run_utf16_locked(sc, di, d_in, n, nullptr, d, s, vt::kModeLength);
  });
}

int vt_host_utf16_len_from_utf8(const uint8_t* in, uint64_t n, int64_t* len) {
  if (!len) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint8_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf8(i, k, nullptr, d, s, vt::kModeLength);
  }));
  *len = r.error_at < 0 ? (int64_t)r.written : -1;
  return 0;
}

int vt_host_utf8_len_from_utf16(const uint16_t* in, uint64_t n, int64_t* len) {
  if (!len) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint16_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf16(i, k, nullptr, d, s, vt::kModeLength);
  }));
  *len = r.error_at < 0 ? (int64_t)r.written : -1;
  return 0;
}

int vt_host_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, vt_result* res) {
  return host_transcode(in, n, out, n, res,
                        [](const uint8_t* i, uint64_t k, uint16_t* o, vt_result* r, cudaStream_t s) {
                          return run_utf8(i, k, o, r, s, vt::kModeTranscode);
                        });
}

int vt_host_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, vt_result* res) {
  return host_transcode(in, n, out, 3 * n + 16, res,
                        [](const uint16_t* i, uint64_t k, uint8_t* o, vt_result* r, cudaStream_t s) {
                          return run_utf16(i, k, o, r, s, vt::kModeTranscode);
                        });
}

int vt_host_validate_utf8(const uint8_t* in, uint64_t n, int64_t* first_err) {
  if (!first_err) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint8_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf8(i, k, nullptr, d, s, vt::kModeValidate);
  }));
  *first_err = r.error_at;
  return 0;
}

int vt_host_validate_utf16(const uint16_t* in, uint64_t n, int64_t* first_err) {
  if (!first_err) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint16_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf16(i, k, nullptr, d, s, vt::kModeValidate);
  }));
  *first_err = r.error_at;
  return 0;
}

int vt_host_count_utf8(const uint8_t* in, uint64_t n, int64_t* count) {
  if (!count) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint8_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf8(i, k, nullptr, d, s, vt::kModeValidate);
  }));
  *count = r.error_at < 0 ? (int64_t)r.written : -1;
  return 0;
}

int vt_host_count_utf16(const uint16_t* in, uint64_t n, int64_t* count) {
  if (!count) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint16_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf16(i, k, nullptr, d, s, vt::kModeValidate);
  }));
  *count = r.error_at < 0 ? (int64_t)r.written : -1;
  return 0;
}

int vt_utf8_to_utf16_nonvalidating_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out,
                                         vt_result* d_res, vt_stream stream) {
  return run_utf8(d_in, n, d_out, d_res, (cudaStream_t)stream, vt::kModeTranscodeNV);
}

int vt_host_utf8_to_utf16_nonvalidating(const uint8_t* in, uint64_t n, uint16_t* out,
                                        vt_result* res) {
  return host_transcode(in, n, out, n, res,
                        [](const uint8_t* i, uint64_t k, uint16_t* o, vt_result* r, cudaStream_t s) {
                          return run_utf8(i, k, o, r, s, vt::kModeTranscodeNV);
                        });
}

int vt_utf8_to_utf16be_async(const uint8_t* d_in, uint64_t n, uint16_t* d_out, vt_result* d_res,
                             vt_stream stream) {
  return run_utf8(d_in, n, d_out, d_res, (cudaStream_t)stream, vt::kModeTranscodeBE);
}

int vt_utf16be_to_utf8_async(const uint16_t* d_in, uint64_t n, uint8_t* d_out, vt_result* d_res,
                             vt_stream stream) {
  return run_utf16(d_in, n, d_out, d_res, (cudaStream_t)stream, vt::kModeTranscodeBE);
}

int vt_validate_utf16be_async(const uint16_t* d_in, uint64_t n, vt_result* d_res, vt_stream stream) {
  return run_utf16(d_in, n, nullptr, d_res, (cudaStream_t)stream, vt::kModeValidateBE);
}

int vt_host_utf8_to_utf16be(const uint8_t* in, uint64_t n, uint16_t* out, vt_result* res) {
  return host_transcode(in, n, out, n, res,
                        [](const uint8_t* i, uint64_t k, uint16_t* o, vt_result* r, cudaStream_t s) {
                          return run_utf8(i, k, o, r, s, vt::kModeTranscodeBE);
                        });
}

int vt_host_utf16be_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, vt_result* res) {
  return host_transcode(in, n, out, 3 * n + 16, res,
                        [](const uint16_t* i, uint64_t k, uint8_t* o, vt_result* r, cudaStream_t s) {
                          return run_utf16(i, k, o, r, s, vt::kModeTranscodeBE);
                        });
}

int vt_host_validate_utf16be(const uint16_t* in, uint64_t n, int64_t* first_err) {
  if (!first_err) return VT_E_ARG;
  vt_result r;
  VT_TRY(host_validate(in, n, &r, [](const uint16_t* i, uint64_t k, vt_result* d, cudaStream_t s) {
    return run_utf16(i, k, nullptr, d, s, vt::kModeValidateBE);
  }));
  *first_err = r.error_at;
  return 0;
}

// harness::transcode_bytes semantics over the GPU entry points (the host only
// looks at the byte-order mark and moves bytes).
int vt_host_transcode_bytes(const uint8_t* in, uint64_t n, int from, int to, int bom,
                            uint8_t* out, uint64_t out_cap, uint64_t* out_len, int* exit_code,
                            int* status, int64_t* error_at) {
  if (!out_len || !exit_code || !status || !error_at || (n && !in) || from < 0 || from > 2 ||
      to < 0 || to > 2 || bom < 0 || bom > 2)
    return VT_E_ARG;
  *out_len = 0;
  *exit_code = 0;
  *status = 0;
  *error_at = -1;
  bool had_bom = false;
  int warn = 0;
  if (from == 0) {
    if (n >= 3 && in[0] == 0xEF && in[1] == 0xBB && in[2] == 0xBF) {
      had_bom = true;
      in += 3;
      n -= 3;
      warn = 0x100;  // "warning: UTF-8 BOM stripped from input"
    }
  } else {
    if (n >= 2) {
      const bool le = in[0] == 0xFF && in[1] == 0xFE, be = in[0] == 0xFE && in[1] == 0xFF;
      if ((le && from == 2) || (be && from == 1)) {
        *exit_code = 1;
        *status = 1;
        return 0;
      }
      if (le || be) {
        had_bom = true;
        in += 2;
        n -= 2;
      }
    }
    if (n % 2) {
      *exit_code = 1;
      *status = 2;
      return 0;
    }
  }
  const bool want_bom = bom == 2 || (bom == 0 && had_bom);
  uint64_t pos = 0;
  auto put_bom = [&]() {
    if (!want_bom) return;
    if (to == 0) {
      out[0] = 0xEF; out[1] = 0xBB; out[2] = 0xBF;
      pos = 3;
    } else if (to == 1) {
      out[0] = 0xFF; out[1] = 0xFE;
      pos = 2;
    } else {
      out[0] = 0xFE; out[1] = 0xFF;
      pos = 2;
    }
  };
  vt_result r;
  if (from == 0) {
    if (to == 0) {
      int64_t e;
      VT_TRY(vt_host_validate_utf8(in, n, &e));
      if (e >= 0) {
        *exit_code = 1;
        *status = 3 | warn;
        *error_at = e;
        return 0;
      }
      if (out_cap < n + 3) return VT_E_ARG;
      put_bom();
      if (n) std::memcpy(out + pos, in, n);
      pos += n;
    } else {
      if (out_cap < 2 * n + 4) return VT_E_ARG;
      put_bom();
      VT_TRY(to == 1 ? vt_host_utf8_to_utf16(in, n, reinterpret_cast<uint16_t*>(out + pos), &r)
                     : vt_host_utf8_to_utf16be(in, n, reinterpret_cast<uint16_t*>(out + pos), &r));
      if (r.error_at >= 0) {
        *exit_code = 1;
        *status = 3 | warn;
        *error_at = r.error_at;
        *out_len = 0;
        return 0;
      }
      pos += 2 * r.written;
    }
  } else {
    const uint64_t units = n / 2;
    // unit loads need 2-byte alignment: realign odd inputs through a copy
    std::vector<uint16_t> tmp;
    const uint16_t* u = reinterpret_cast<const uint16_t*>(in);
    if (((uintptr_t)in & 1) != 0) {
      tmp.resize(units);
      if (units) std::memcpy(tmp.data(), in, n);
      u = tmp.data();
    }
    if (to == 0) {
      if (out_cap < 3 * units + 20) return VT_E_ARG;
      put_bom();
      VT_TRY(from == 1 ? vt_host_utf16_to_utf8(u, units, out + pos, &r)
                       : vt_host_utf16be_to_utf8(u, units, out + pos, &r));
      if (r.error_at >= 0) {
        *exit_code = 1;
        *status = 4;
        *error_at = r.error_at;
        return 0;
      }
      pos += r.written;
    } else {
      int64_t e;
      VT_TRY(from == 1 ? vt_host_validate_utf16(u, units, &e) : vt_host_validate_utf16be(u, units, &e));
      if (e >= 0) {
        *exit_code = 1;
        *status = 4;
        *error_at = e;
        return 0;
      }
      if (out_cap < n + 4) return VT_E_ARG;
      put_bom();
      if (from == to) {
        if (n) std::memcpy(out + pos, u, n);
      } else if (units) {
        // endianness change: byte swap on the GPU
        HostCtx* c;
        VT_TRY(host_ctx(c));
        VT_TRY(ensure_dev(c->d_in, c->d_in_cap, n + 4, c->stream));
        VT_TRY(ensure_dev(c->d_out, c->d_out_cap, n + 4, c->stream));
        VT_TRY(cudaMemcpyAsync(c->d_in, u, n, cudaMemcpyHostToDevice, c->stream));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        VT_TRY(vt::launch_bswap16(reinterpret_cast<const uint16_t*>(c->d_in),
                                  reinterpret_cast<uint16_t*>(c->d_out), units, c->stream));
        VT_TRY(cudaMemcpyAsync(out + pos, c->d_out, n, cudaMemcpyDeviceToHost, c->stream));
        VT_TRY(cudaStreamSynchronize(c->stream));
      }
      pos += n;
    }
  }
  *out_len = pos;
  *status |= warn;
  return 0;
}

int vt_validate_utf8_batch(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           int64_t* d_first_err, vt_stream stream) {
  int dev;
  VT_TRY(current_device(dev));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_validate_utf8_batch(d_data, d_offsets, count, d_first_err,
                                        (cudaStream_t)stream);
}

int vt_utf8_to_utf16_batch(const uint8_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           uint16_t* d_out, vt_result* d_res, int validate, vt_stream stream) {
  if (count && (!d_data || !d_offsets || !d_out || !d_res)) return VT_E_ARG;
  int dev;
  VT_TRY(current_device(dev));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_utf8_to_utf16_batch(d_data, d_offsets, count, d_out, d_res, validate,
                                        (cudaStream_t)stream);
}

int vt_utf16_to_utf8_batch(const uint16_t* d_data, const uint64_t* d_offsets, uint64_t count,
                           uint8_t* d_out, vt_result* d_res, vt_stream stream) {
  if (count && (!d_data || !d_offsets || !d_out || !d_res)) return VT_E_ARG;
  int dev;
  VT_TRY(current_device(dev));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_utf16_to_utf8_batch(d_data, d_offsets, count, d_out, d_res,
                                        (cudaStream_t)stream);
}

int vt_exhaustive_short_verdicts(uint8_t* d_verdicts, vt_stream stream) {
  int dev;
  VT_TRY(current_device(dev));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_exhaustive_short(d_verdicts, (cudaStream_t)stream);
}

// ---- sharder -------------------------------------------------------------------

uint64_t vt_split_point_utf8(const uint8_t* in, uint64_t n, uint64_t cut) {
  // move the cut back to the last non-continuation byte
  // within 3 bytes; if there is none, no valid character spans the cut.
  if (cut == 0 || cut >= n) return cut;
  for (uint64_t k = 0; k <= 3 && k <= cut; k++)
    if ((in[cut - k] & 0xC0) != 0x80) return cut - k;
  return cut;
}

uint64_t vt_split_point_utf16(const uint16_t* in, uint64_t n, uint64_t cut) {
  // fact E: never separate a high surrogate from the low one that follows it
  if (cut == 0 || cut >= n) return cut;
  if ((in[cut] & 0xFC00) == 0xDC00 && (in[cut - 1] & 0xFC00) == 0xD800) return cut - 1;
  return cut;
}

}  // extern "C"

namespace {

// One persistent host thread per device for the host-pointer sharder.  A
// shard's host context (stream, pinned staging, device buffers) belongs to the
// thread that runs it (thread_local HostCtx), so per-call threads would build
// and abandon one per shard per call; these workers keep theirs for the life
// of the process.  The pool is never destroyed (workers idle on a condition
// variable at exit).
class DeviceWorkers {
 public:
  static DeviceWorkers& get() {
    static DeviceWorkers* w = new DeviceWorkers();
    return *w;
  }
  // Runs fn on device dev's worker; the returned job is waited with wait().
  struct Job {
    std::mutex mu;
    std::condition_variable cv;
    bool done = false;
    std::function<void()> fn;
  };
  void submit(int dev, const std::shared_ptr<Job>& job) {
    Worker& w = worker(dev);
    {
      std::lock_guard<std::mutex> lk(w.mu);
      w.q.push_back(job);
    }
    w.cv.notify_one();
  }
  static void wait(const std::shared_ptr<Job>& job) {
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [&] { return job->done; });
  }

 private:
  struct Worker {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::shared_ptr<Job>> q;
    std::thread th;
  };
  std::mutex mu_;
  std::map<int, std::unique_ptr<Worker>> ws_;

  Worker& worker(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    auto& w = ws_[dev];
    if (!w) {
      w.reset(new Worker());
      Worker* wp = w.get();
      wp->th = std::thread([wp, dev] {
        cudaSetDevice(dev);
        for (;;) {
          std::shared_ptr<Job> job;
          {
            std::unique_lock<std::mutex> lk(wp->mu);
            wp->cv.wait(lk, [&] { return !wp->q.empty(); });
            job = wp->q.front();
            wp->q.pop_front();
          }
          job->fn();
          {
            std::lock_guard<std::mutex> lk(job->mu);
            job->done = true;
          }
          job->cv.notify_all();
        }
      });
      wp->th.detach();
    }
    return *w;
  }
};

// Combines per-shard results of consecutive character-boundary shards
// (SURVEY.md 8(a) D/E): output offsets by exclusive scan of `written`, the
// first failing shard decides error_at; shards after it hold no part of the
// defined output.
void combine_shards(const std::vector<uint64_t>& st, const vt_result* rs, int k_n,
                    uint64_t* offsets, vt_result* res) {
  uint64_t written = 0;
  res->error_at = -1;
  res->consumed = st[k_n];
  bool stopped = false;
  for (int k = 0; k < k_n; k++) {
    if (offsets) offsets[k] = written;
    if (stopped) continue;
    written += rs[k].written;
    if (rs[k].error_at >= 0) {
      res->error_at = (int64_t)st[k] + rs[k].error_at;
      res->consumed = (uint64_t)res->error_at;
      stopped = true;
    }
  }
  res->written = written;
}

template <class In, class Out, class Split, class One>
int sharded(const In* in, uint64_t n, Out* out, int ndev, uint64_t mult, vt_result* res,
            Split split, One one) {
  if (!res || (n && (!in || !out))) return VT_E_ARG;
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail == 0) {
    cudaGetLastError();
    return VT_E_NODEVICE;
  }
  // ndev shards; shard k runs on device k % avail (shards sharing a device run
  // one after the other on its worker)
  if (ndev <= 0) ndev = avail;
  std::vector<uint64_t> st(ndev + 1, 0);
  for (int k = 1; k < ndev; k++) st[k] = std::max(st[k - 1], split(in, n, n / ndev * k));
  st[ndev] = n;
  std::vector<vt_result> rs(ndev);
  std::vector<int> rcs(ndev, 0);
  std::vector<std::shared_ptr<DeviceWorkers::Job>> jobs;
  for (int k = 0; k < ndev; k++) {
    auto job = std::make_shared<DeviceWorkers::Job>();
    // shard k's output fits in [mult*st[k], mult*st[k+1]) of the caller's buffer
    job->fn = [&, k] { rcs[k] = one(in + st[k], st[k + 1] - st[k], out + mult * st[k], &rs[k]); };
    DeviceWorkers::get().submit(k % avail, job);
    jobs.push_back(job);
  }
  for (auto& j : jobs) DeviceWorkers::wait(j);
  for (int k = 0; k < ndev; k++)
    if (rcs[k]) return rcs[k];
  std::vector<uint64_t> off(ndev);
  combine_shards(st, rs.data(), ndev, off.data(), res);
  // compact the shards' outputs (in order: a move may overwrite the tail of an
  // earlier shard's source only after that shard moved)
  for (int k = 0; k < ndev && off[k] < res->written; k++)
    if (off[k] != mult * st[k] && rs[k].written)
      std::memmove(out + off[k], out + mult * st[k], rs[k].written * sizeof(Out));
  return 0;
}

// Device-resident shards: per device one library-owned stream and result
// slots; the calling thread enqueues every shard, then waits for all.
struct ShardDev {
  cudaStream_t s = nullptr;
  vt_result* d_res = nullptr;
  vt_result* h_res = nullptr;
  int cap = 0;
};
std::mutex g_shard_mu;
std::map<int, ShardDev> g_shard_dev;

template <class In, class Out, class Async>
int sharded_device(int nshards, const int* dev, const In* const* d_in, const uint64_t* n,
                   Out* const* d_out, vt_result* shard_res, uint64_t* out_offsets, vt_result* res,
                   Async async) {
  if (nshards <= 0 || !dev || !d_in || !n || !d_out || !res) return VT_E_ARG;
  int cur;
  VT_TRY(current_device(cur));
  std::lock_guard<std::mutex> lk(g_shard_mu);
  std::map<int, int> used;  // result slots per device
  std::vector<int> slot(nshards);
  int rc = 0;
  for (int k = 0; k < nshards && !rc; k++) {
    slot[k] = used[dev[k]]++;
    rc = (int)cudaSetDevice(dev[k]);
    if (rc) break;
    ShardDev& sd = g_shard_dev[dev[k]];
    if (!sd.s) rc = (int)cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking);
    if (!rc && sd.cap < nshards) {
      // (all earlier users of this device's slots were waited for)
      if (sd.d_res) cudaFree(sd.d_res);
      if (sd.h_res) cudaFreeHost(sd.h_res);
      rc = (int)cudaMalloc(&sd.d_res, nshards * sizeof(vt_result));
      if (!rc) rc = (int)cudaMallocHost(&sd.h_res, nshards * sizeof(vt_result));
      sd.cap = rc ? 0 : nshards;
    }
    if (!rc) rc = async(d_in[k], n[k], d_out[k], sd.d_res + slot[k], (vt_stream)sd.s);
    if (!rc)
      rc = (int)cudaMemcpyAsync(sd.h_res + slot[k], sd.d_res + slot[k], sizeof(vt_result),
                                cudaMemcpyDeviceToHost, sd.s);
  }
  for (auto& u : used) {  // wait for every device that got work
    cudaSetDevice(u.first);
    const int r2 = (int)cudaStreamSynchronize(g_shard_dev[u.first].s);
    if (!rc) rc = r2;
  }
  cudaSetDevice(cur);
  if (rc) return rc;
  std::vector<uint64_t> st(nshards + 1, 0);
  std::vector<vt_result> rs(nshards);
  for (int k = 0; k < nshards; k++) {
    rs[k] = g_shard_dev[dev[k]].h_res[slot[k]];
    st[k + 1] = st[k] + n[k];
    if (shard_res) shard_res[k] = rs[k];
  }
  combine_shards(st, rs.data(), nshards, out_offsets, res);
  return 0;
}

}  // namespace

extern "C" {

int vt_sharded_utf8_to_utf16(const uint8_t* in, uint64_t n, uint16_t* out, int ndev,
                             vt_result* res) {
  return sharded(in, n, out, ndev, 1, res, vt_split_point_utf8, vt_host_utf8_to_utf16);
}

int vt_sharded_utf16_to_utf8(const uint16_t* in, uint64_t n, uint8_t* out, int ndev,
                             vt_result* res) {
  return sharded(in, n, out, ndev, 3, res, vt_split_point_utf16, vt_host_utf16_to_utf8);
}

int vt_sharded_device_utf8_to_utf16(int nshards, const int* dev, const uint8_t* const* d_in,
                                    const uint64_t* n, uint16_t* const* d_out,
                                    vt_result* shard_res, uint64_t* out_offsets, vt_result* res) {
  return sharded_device(nshards, dev, d_in, n, d_out, shard_res, out_offsets, res,
                        vt_utf8_to_utf16_async);
}

int vt_sharded_device_utf16_to_utf8(int nshards, const int* dev, const uint16_t* const* d_in,
                                    const uint64_t* n, uint8_t* const* d_out,
                                    vt_result* shard_res, uint64_t* out_offsets, vt_result* res) {
  return sharded_device(nshards, dev, d_in, n, d_out, shard_res, out_offsets, res,
                        vt_utf16_to_utf8_async);
}

int vt_gen_sizes(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks, uint64_t* d_sizes,
                 vt_stream stream) {
  if (cfg < 1 || cfg > 5) return VT_E_ARG;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_gen_sizes(cfg, seed, chunk0, nchunks, d_sizes, (cudaStream_t)stream);
}

int vt_gen_write(int cfg, uint64_t seed, uint64_t chunk0, uint64_t nchunks,
                 const uint64_t* d_offsets, uint64_t limit, void* d_out, uint64_t* d_end,
                 vt_stream stream) {
  if (cfg < 1 || cfg > 5) return VT_E_ARG;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return vt::launch_gen_write(cfg, seed, chunk0, nchunks, d_offsets, limit, d_out, d_end,
                              (cudaStream_t)stream);
}

const char* vt_status_string(int status) {
  if (status == 0) return "ok";
  if (status == VT_E_NODEVICE) return "no CUDA device visible (libvtrans_gpu has no CPU fallback)";
  if (status == VT_E_ARG) return "invalid argument";
  if (status == VT_E_ARCH) return "device is not sm_100 (kernels are built for sm_100a only)";
  return cudaGetErrorString((cudaError_t)status);
}

int vt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

uint64_t vt_launch_count(void) { return g_launches.load(); }

// Debug: the 5 probe counters of the control block of (current device, stream).
int vt_debug_probe(vt_stream stream, uint64_t* out5) {
  int dev;
  VT_TRY(current_device(dev));
  std::shared_ptr<Scratch> hold;
  VT_TRY(scratch_for(dev, (cudaStream_t)stream, hold));
  Scratch* sc = hold.get();
  if (!sc->ctl) return VT_E_ARG;
  VT_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  VT_TRY(cudaMemcpy(out5, sc->ctl->pad, 5 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return 0;
}

#ifdef VT_PHASES
int vt_debug_phases(int utf16, uint64_t* out8) {
  return utf16 ? vt::read_phases16(reinterpret_cast<unsigned long long*>(out8))
               : vt::read_phases(reinterpret_cast<unsigned long long*>(out8));
}
#endif

const char* vt_build_info(void) {
  return "libvtrans_gpu sm_100a (nvcc " VT_STR(__CUDACC_VER_MAJOR__) "." VT_STR(
      __CUDACC_VER_MINOR__) ")";
}

// ---- streaming UTF-8 validation ----------------------

void vt_utf8_stream_init(vt_utf8_stream* st) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->error_at = -1;
}

int vt_utf8_stream_ok(const vt_utf8_stream* st) { return st && st->error_at < 0 ? 1 : 0; }

int vt_utf8_stream_finish(const vt_utf8_stream* st) {
  return st && st->error_at < 0 && st->carry_len == 0 ? 1 : 0;
}

int vt_utf8_stream_feed_async(vt_utf8_stream* d_st, const uint8_t* d_chunk, uint64_t n,
                              vt_stream stream) {
  if (!d_st || (n && !d_chunk)) return VT_E_ARG;
  if (n == 0) return 0;
  const cudaStream_t s = (cudaStream_t)stream;
  Target t;
  VT_TRY(target(s, t));
  std::lock_guard<std::mutex> lk(t.sc->mu);
  if (!t.sc->d_res) {
    VT_TRY(cudaMalloc(&t.sc->d_res, sizeof(vt_result)));
    VT_TRY(cudaMallocHost(&t.sc->h_res, sizeof(vt_result)));
  }
  VT_TRY(vt::launch_stream_seam(d_st, d_chunk, n, s));
  VT_TRY(run_utf8_locked(t.sc, t.di, d_chunk, n, nullptr, t.sc->d_res, s, vt::kModeValidate,
                         &d_st->skip));
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return vt::launch_stream_tail(d_st, d_chunk, n, t.sc->d_res, s);
}

int vt_host_utf8_stream_feed(vt_utf8_stream* st, const uint8_t* chunk, uint64_t n) {
  if (!st || (n && !chunk)) return VT_E_ARG;
  if (n == 0) return 0;
  HostCtx* c;
  VT_TRY(host_ctx(c));
  const uint8_t* d_chunk;
  if (n <= kZeroCopyMax) {
    std::memcpy(c->h_in, chunk, n);
    VT_TRY(cudaHostGetDevicePointer((void**)&d_chunk, c->h_in, 0));
  } else {
    VT_TRY(ensure_dev(c->d_in, c->d_in_cap, n, c->stream));
    VT_TRY(cudaMemcpyAsync(c->d_in, chunk, n, cudaMemcpyHostToDevice, c->stream));
    d_chunk = c->d_in;
  }
  *c->h_vs = *st;
  VT_TRY(cudaMemcpyAsync(c->d_vs, c->h_vs, sizeof(vt_utf8_stream), cudaMemcpyHostToDevice,
                         c->stream));
  VT_TRY(vt_utf8_stream_feed_async(c->d_vs, d_chunk, n, (vt_stream)c->stream));
  VT_TRY(cudaMemcpyAsync(c->h_vs, c->d_vs, sizeof(vt_utf8_stream), cudaMemcpyDeviceToHost,
                         c->stream));
  VT_TRY(cudaStreamSynchronize(c->stream));
  *st = *c->h_vs;
  return 0;
}

// ---- character-class counts (harness::compute_stats) -------------------------

int vt_host_utf8_class_counts(const uint8_t* in, uint64_t n, uint64_t counts[4], int* valid) {
  if (!counts || !valid || (n && !in)) return VT_E_ARG;
  for (int i = 0; i < 4; i++) counts[i] = 0;
  *valid = 1;
  if (n == 0) return 0;
  HostCtx* c;
  VT_TRY(host_ctx(c));
  const uint8_t* d;
  if (n <= kZeroCopyMax) {
    std::memcpy(c->h_in, in, n);
    VT_TRY(cudaHostGetDevicePointer((void**)&d, c->h_in, 0));
  } else {
    VT_TRY(ensure_dev(c->d_in, c->d_in_cap, n, c->stream));
    VT_TRY(cudaMemcpyAsync(c->d_in, in, n, cudaMemcpyHostToDevice, c->stream));
    d = c->d_in;
  }
  VT_TRY(run_utf8(d, n, nullptr, c->d_res, c->stream, vt::kModeValidate));
  VT_TRY(cudaMemsetAsync(c->d_counts, 0, 4 * sizeof(unsigned long long), c->stream));
  VT_TRY(vt::launch_utf8_class_counts(d, n, c->d_counts, c->stream));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  VT_TRY(cudaMemcpyAsync(c->h_res, c->d_res, sizeof(vt_result), cudaMemcpyDeviceToHost, c->stream));
  VT_TRY(cudaMemcpyAsync(c->h_counts, c->d_counts, 4 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, c->stream));
  VT_TRY(cudaStreamSynchronize(c->stream));
  if (c->h_res->error_at >= 0) {
    *valid = 0;
    return 0;
  }
  for (int i = 0; i < 4; i++) counts[i] = c->h_counts[i];
  return 0;
}

void vt_host_transfer_counts(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = t_h2d;
  if (d2h) *d2h = t_d2h;
}

}  // extern "C"

// oracle/gen_host.cpp -- TEST / BENCH INFRASTRUCTURE ONLY.
//
// The synthetic BASELINE workloads (paper_2109_10433_b200/csrc/vt_gen.cuh, the
// same header the device generator uses) generated on the host, so that the
// reference arm of bench.py and the CPU baseline leg can build their inputs
// without loading the product library (libvtrans_gpu.so).  Built by
// oracle/Makefile into oracle/lib/libvt_gen.so.
#include <cstdint>
#include <thread>
#include <vector>

#include "../paper_2109_10433_b200/csrc/vt_gen.cuh"

extern "C" {

uint64_t vtg_chunk_draws(int) { return vt::kDraws; }

// One chunk (as vt_gen_host_chunk in the product library).
uint64_t vtg_host_chunk(int cfg, uint64_t seed, uint64_t chunk, void* out, uint64_t cap,
                        uint64_t* first_bad) {
  if (cfg == 3) {
    vt::WriteSink<uint16_t> w{static_cast<uint16_t*>(out), 0, cap};
    vt::gen_chunk(cfg, seed, chunk, w);
    if (first_bad) *first_bad = w.first_bad;
    return w.off;
  }
  vt::WriteSink<uint8_t> w{static_cast<uint8_t*>(out), 0, cap};
  vt::gen_chunk(cfg, seed, chunk, w);
  if (first_bad) *first_bad = w.first_bad;
  return w.off;
}

// The whole stream of `size` elements (bytes; units for cfg 3) from chunk 0 on,
// cut after the last whole character that fits (exactly what the device
// generator writes).  Chunks are sized, then written, in parallel.  Returns
// the number of elements written; *first_bad = first injected error or ~0.
uint64_t vtg_generate(int cfg, uint64_t seed, uint64_t size, void* out, int threads,
                      uint64_t* first_bad) {
  if (threads < 1) threads = 1;
  std::vector<uint64_t> sizes;
  uint64_t total = 0, nchunks = 0;
  while (total < size) {  // size chunks in batches until they cover `size`
    const uint64_t batch = 1024;
    sizes.resize(nchunks + batch);
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; t++)
      ts.emplace_back([&, t] {
        for (uint64_t c = nchunks + t; c < nchunks + batch; c += threads) {
          vt::CountSink cs;
          vt::gen_chunk(cfg, seed, c, cs);
          sizes[c] = cs.n;
        }
      });
    for (auto& th : ts) th.join();
    for (uint64_t c = nchunks; c < nchunks + batch && total < size; c++) total += sizes[c];
    nchunks += batch;
  }
  std::vector<uint64_t> off(nchunks + 1, 0);
  for (uint64_t c = 0; c < nchunks; c++) off[c + 1] = off[c] + sizes[c];
  std::vector<uint64_t> ends(nchunks, 0), bads(nchunks, ~0ull);
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; t++)
    ts.emplace_back([&, t] {
      for (uint64_t c = t; c < nchunks && off[c] < size; c += threads) {
        const uint64_t lim = size - off[c] < sizes[c] ? size - off[c] : sizes[c];
        if (cfg == 3) {
          vt::WriteSink<uint16_t> w{static_cast<uint16_t*>(out) + off[c], 0, lim};
          vt::gen_chunk(cfg, seed, c, w);
          ends[c] = off[c] + w.off;
          if (w.first_bad != ~0ull) bads[c] = off[c] + w.first_bad;
        } else {
          vt::WriteSink<uint8_t> w{static_cast<uint8_t*>(out) + off[c], 0, lim};
          vt::gen_chunk(cfg, seed, c, w);
          ends[c] = off[c] + w.off;
          if (w.first_bad != ~0ull) bads[c] = off[c] + w.first_bad;
        }
      }
    });
  for (auto& th : ts) th.join();
  // the stream ends at the first chunk cut short by `size`
  uint64_t n = 0, fb = ~0ull;
  for (uint64_t c = 0; c < nchunks && off[c] < size; c++) {
    if (fb == ~0ull && bads[c] != ~0ull && bads[c] < ends[c]) fb = bads[c];
    n = ends[c];
    if (ends[c] < off[c] + sizes[c]) break;
  }
  if (first_bad) *first_bad = fb;
  return n;
}

}  // extern "C"

"""Phase stamps of an early-error call (cfg4: first error at ~16 MB of 1 GiB),
from a VT_TRACE build: VT_LIB=tools/variants/traced.so python tools/cfg4_trace.py

Stamps (global timer, ns, relative to the first CTA's start):
  transcode: 1 first error found, 2 the error tile's count done, 3 its
  decode done, 4 its inclusive prefix published, 5 last CTA leaves the tile
  loop, 6 finalize done;  validate: 8 first CTA start, 1 error found, 9 last
  warp leaves the row loop, 10 finalize starts, 11 finalize done."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2109_10433_b200 as vt  # noqa: E402


def trace(L):
    out = (C.c_uint64 * 16)()
    assert L.vt_debug_trace(0, out) == 0
    return list(out)


def main():
    L = vt.lib()
    L.vt_debug_trace.argtypes = [C.c_int, C.c_void_p]
    d, n, bad = vt.generate(4, 1 << 30)
    out = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for m in (bad + (1 << 20), n):
        for rep in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            trace(L)  # re-arm
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = vt.utf8_to_utf16_device(d, m, out)
            b.record()
            torch.cuda.synchronize()
            t = trace(L)
            t0 = t[0]
            rel = {k: (t[k] - t0) / 1e3 for k in (1, 2, 3, 4, 5, 6) if t[k] not in (0, 2**64 - 1)}
            print(f"transcode n={m} {a.elapsed_time(b) * 1e3:.1f} us; stamps (us): " +
                  ", ".join(f"{k}:{v:.1f}" for k, v in rel.items()) + f"  err={r.error_at}", flush=True)
        for rep in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            trace(L)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = vt.validate_utf8_device(d, m)
            b.record()
            torch.cuda.synchronize()
            t = trace(L)
            t0 = t[8]
            rel = {k: (t[k] - t0) / 1e3 for k in (1, 9, 10, 11) if t[k] not in (0, 2**64 - 1)}
            print(f"validate  n={m} {a.elapsed_time(b) * 1e3:.1f} us; stamps (us): " +
                  ", ".join(f"{k}:{v:.1f}" for k, v in rel.items()), flush=True)


if __name__ == "__main__":
    main()

"""Where the time of an early-error call goes (perf probe, BASELINE cfg4).

Times the validating transcode and the validation of the cfg4 stream (first
error at ~16 MB) over buffers of growing length, next to a valid stream of
the same prefix length, each call with a cold L2 (512 MiB written between
calls, outside the events)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2109_10433_b200 as vt  # noqa: E402


def timed(fn, reps=20):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    d, n, bad = vt.generate(4, 1 << 30)
    r = vt.validate_utf8_device(d, n)
    print(f"cfg4: n={n} first error {r.error_at} (generator {bad})", flush=True)
    out = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    res = torch.zeros(3, dtype=torch.int64, device="cuda")
    e = r.error_at
    for m in (e + (1 << 20), e + (16 << 20), 256 << 20, n):
        t1 = timed(lambda: vt.utf8_to_utf16_device(d, m, out, d_res=res))
        t2 = timed(lambda: vt.validate_utf8_device(d, m, d_res=res))
        print(f"cfg4 n={m:>11d}: transcode {t1:8.1f} us   validate {t2:8.1f} us", flush=True)
    v, nv, _ = vt.generate(4, e, seed=44)  # same mix; with seed 44 the first e bytes are valid?
    rv = vt.validate_utf8_device(v, nv)
    if rv.error_at is None:
        t1 = timed(lambda: vt.utf8_to_utf16_device(v, nv, out, d_res=res))
        t2 = timed(lambda: vt.validate_utf8_device(v, nv, d_res=res))
        print(f"valid cfg4-mix prefix n={nv}: transcode {t1:8.1f} us   validate {t2:8.1f} us")
    c2, n2, _ = vt.generate(2, e)
    t1 = timed(lambda: vt.utf8_to_utf16_device(c2, n2, out, d_res=res))
    t2 = timed(lambda: vt.validate_utf8_device(c2, n2, d_res=res))
    print(f"valid cfg2 n={n2}: transcode {t1:8.1f} us   validate {t2:8.1f} us")


if __name__ == "__main__":
    main()

"""Device time of the validate kernels on cfg2 (UTF-8) / cfg3 (UTF-16) and cfg5 (perf helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt

def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

res = torch.zeros(3, dtype=torch.int64, device="cuda")
out = []
for cfg in (2, 5):
    d, n, _ = vt.generate(cfg, 1 << 30)
    out.append(f"cfg{cfg} validate8 {timeit(lambda: vt.validate_utf8_device(d, n, d_res=res)):.4f} ms")
    del d
d, n, _ = vt.generate(3, 1 << 29)
out.append(f"cfg3 validate16 {timeit(lambda: vt.validate_utf16_device(d, n, d_res=res)):.4f} ms")
print("  ".join(out))

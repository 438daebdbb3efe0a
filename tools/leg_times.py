"""Times the kernels per direction on several generated configs (debug/perf helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

res = torch.zeros(3, dtype=torch.int64, device="cuda")
for cfg, size in [(2, 1 << 30), (5, 1 << 30), (4, 1 << 30), (1, 1 << 30)]:
    d, n, _ = vt.generate(cfg, size)
    o16 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    t8 = timeit(lambda: vt.utf8_to_utf16_device(d, n, o16, d_res=res))
    tv = timeit(lambda: vt.validate_utf8_device(d, n, d_res=res))
    r = vt.utf8_to_utf16_device(d, n, o16)
    o8 = torch.empty(3 * r.written + 16, dtype=torch.uint8, device="cuda")
    t16 = timeit(lambda: vt.utf16_to_utf8_device(o16, r.written, o8, d_res=res))
    tv16 = timeit(lambda: vt.validate_utf16_device(o16, r.written, d_res=res))
    print(f"cfg{cfg}: n={n} u8->u16 {t8:.3f} ms ({n/t8/1e6:.0f} GB/s in)  validate8 {tv:.3f} ms  "
          f"u16->u8 {t16:.3f} ms ({2*r.written/t16/1e6:.0f} GB/s in)  validate16 {tv16:.3f} ms  err={r.error_at}",
          flush=True)
    del d, o16, o8

"""Device time of the transcode / validate kernels against input size (perf helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt

def timeit(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000

res = torch.zeros(3, dtype=torch.int64, device="cuda")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, n, _ = vt.generate(cfg, 1 << 30)
o16 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
hot = os.environ.get("HOT")  # keep the GPU busy (clocks up) right before each timing
def warm():
    if hot:
        for _ in range(10): vt.utf8_to_utf16_device(d, n, o16, d_res=res)
for mib in [1, 4, 16, 64, 256, 1024]:
    m = min(n, mib << 20)
    # cut at a character boundary
    while m < n and (int(d[m].item()) & 0xC0) == 0x80: m -= 1
    warm()
    t8 = timeit(lambda: vt.utf8_to_utf16_device(d, m, o16, d_res=res), reps=200)
    warm()
    tv = timeit(lambda: vt.validate_utf8_device(d, m, d_res=res), reps=200)
    print(f"cfg{cfg} {mib:5d} MiB: transcode {t8:8.1f} us ({m / t8 / 1e3:7.1f} GB/s)  validate {tv:8.1f} us ({m / tv / 1e3:7.1f} GB/s)", flush=True)

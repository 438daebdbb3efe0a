"""Device time of both directions on pure-ASCII and pure-CJK text (perf probe: staging-store bank conflicts
depend on the output bytes per thread)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_10433_b200 as vt

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

res = torch.zeros(3, dtype=torch.int64, device="cuda")
n = 1 << 30
rng = np.random.default_rng(1)
for name, make in (("ascii", lambda: rng.integers(0x20, 0x7F, n, dtype=np.uint8)),
                   ("cjk3", lambda: np.tile(np.frombuffer("漢字仮名交".encode(), dtype=np.uint8), n // 15 + 1)[: (n // 15) * 15]),
                   ("latin2", lambda: np.tile(np.frombuffer("éàüñ".encode(), dtype=np.uint8), n // 8)[: (n // 8) * 8])):
    h = make()
    d = torch.from_numpy(h).cuda()
    m = d.numel()
    o16 = torch.empty(m + 8, dtype=torch.int16, device="cuda")
    r = vt.utf8_to_utf16_device(d, m, o16)
    assert r.error_at is None, r
    t8 = timeit(lambda: vt.utf8_to_utf16_device(d, m, o16, d_res=res))
    o8 = torch.empty(3 * r.written + 16, dtype=torch.uint8, device="cuda")
    r2 = vt.utf16_to_utf8_device(o16, r.written, o8)
    assert r2.written == m and torch.equal(o8[:m], d)
    t16 = timeit(lambda: vt.utf16_to_utf8_device(o16, r.written, o8, d_res=res))
    print(f"{name}: u8->u16 {t8:.3f} ms ({m / t8 / 1e6:.0f} GB/s in)  u16->u8 {t16:.3f} ms ({2 * r.written / t16 / 1e6:.0f} GB/s in)", flush=True)
    del d, o16, o8

"""Per-phase cycles of the transcode pipeline (build with -DVT_PHASES; perf helper)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2109_10433_b200 as vt
L = vt.lib(); L.vt_debug_phases.argtypes = [C.c_int, C.c_void_p]
names = ["top-sync", "count", "excl-wait", "copy-out", "post-copy-sync", "emit", "grab"]
res = torch.zeros(3, dtype=torch.int64, device="cuda")
for spec in (sys.argv[1:] or ["2", "3"]):
    cfg, _, sz = spec.partition(":")  # "1:16" = cfg1 at 16 MiB
    cfg = int(cfg)
    size = (int(sz) << 20) if sz else (1 << 30)
    d, n, _ = vt.generate(cfg, size // 2 if cfg == 3 else size)
    if cfg == 3:
        o = torch.empty(3 * n + 16, dtype=torch.uint8, device="cuda")
        run = lambda: vt.utf16_to_utf8_device(d, n, o, d_res=res)
    else:
        o = torch.empty(n + 8, dtype=torch.int16, device="cuda")
        run = lambda: vt.utf8_to_utf16_device(d, n, o, d_res=res)
    for _ in range(3): run()
    torch.cuda.synchronize()
    b0 = np.zeros(20, dtype=np.uint64); L.vt_debug_phases(int(cfg == 3), b0.ctypes.data)
    for _ in range(5): run()
    torch.cuda.synchronize()
    b = np.zeros(20, dtype=np.uint64); L.vt_debug_phases(int(cfg == 3), b.ctypes.data)
    b = (b - b0).astype(np.float64); t = b[7]
    tot = b[:7].sum() / t
    sub = ""
    if b[8] > 0:
        sub = f"  [count: loads {b[1] / t - (b[9] - b[8]) / t - (b[11] - b[9]) / t:.0f}, classify {(b[9] - b[8]) / t:.0f}, scan+publish {(b[11] - b[9]) / t:.0f}]"
    print(sub)
    print(f"cfg{cfg}: cycles per tile (warp 0) total {tot:.0f}: " +
          ", ".join(f"{nm} {b[i] / t:.0f}" for i, nm in enumerate(names)))
    tl = b[19]
    if tl > 0:
        lbn = ["wait-staged", "copy-out", "wait-tile-id", "look-back", "wait-agg+publish"]
        print(f"cfg{cfg}: look-back warp cycles per tile total {b[12:17].sum() / tl:.0f}: " +
              ", ".join(f"{nm} {b[12 + i] / tl:.0f}" for i, nm in enumerate(lbn)))
    del d, o

"""e2e (host pointer) rate of the drop-in C ABI for cfg2 / cfg3 (perf helper)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt
L = vt.lib(); r = vt._CRes()
for cfg, kind in [(2, "u8"), (3, "u16")]:
    d, n, _ = vt.generate(cfg, 1 << 30 if kind == "u8" else 1 << 29)
    if kind == "u8":
        h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True); h_in.copy_(d[:n])
        h_out = torch.empty(n + 8, dtype=torch.int16, pin_memory=True); fn = L.vt_host_utf8_to_utf16; nb = n
    else:
        dd = d.view(torch.int16) if d.dtype != torch.int16 else d
        h_in = torch.empty(n, dtype=torch.int16, pin_memory=True); h_in.copy_(dd[:n])
        h_out = torch.empty(3 * n + 16, dtype=torch.uint8, pin_memory=True); fn = L.vt_host_utf16_to_utf8; nb = 2 * n
    for _ in range(2): assert fn(h_in.data_ptr(), n, h_out.data_ptr(), ctypes.byref(r)) == 0
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); fn(h_in.data_ptr(), n, h_out.data_ptr(), ctypes.byref(r)); ts.append(time.perf_counter() - t0)
    print(f"cfg{cfg} e2e {nb/min(ts)/1e9:.1f} GB/s best, {nb/sorted(ts)[2]/1e9:.1f} median  written={r.written}", flush=True)
    del d, h_in, h_out

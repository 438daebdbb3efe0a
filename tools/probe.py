import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2109_10433_b200 as vt
L = vt.lib(); L.vt_debug_probe.argtypes = [C.c_void_p, C.c_void_p]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
res = torch.zeros(3, dtype=torch.int64, device="cuda")
if cfg == 3:
    d, n, _ = vt.generate(3, 1 << 29)
    o = torch.empty(3 * n + 16, dtype=torch.uint8, device="cuda")
    run = lambda: vt.utf16_to_utf8_device(d, n, o, d_res=res)
else:
    d, n, _ = vt.generate(cfg, 1 << 30)
    o = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    run = lambda: vt.utf8_to_utf16_device(d, n, o, d_res=res)
s = torch.cuda.current_stream()
for _ in range(3): run()
buf = np.zeros(5, dtype=np.uint64); L.vt_debug_probe(s.cuda_stream, buf.ctypes.data); b0 = buf.copy()
for _ in range(5): run()
L.vt_debug_probe(s.cuda_stream, buf.ctypes.data); b = buf - b0
print("lookback avg cycles", b[0] / max(1, b[1]), "n", b[1], " excl-wait avg cycles", b[2] / max(1, b[3]), "n", b[3], "progress steps", int(b[4]) >> 32, "spin steps", int(b[4]) & 0xffffffff)

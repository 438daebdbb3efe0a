"""In-kernel globaltimer timeline of the validate kernel (build with -DVT_TIMELINE; perf helper)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2109_10433_b200 as vt
L = vt.lib(); L.vt_debug_probe.argtypes = [C.c_void_p, C.c_void_p]
res = torch.zeros(3, dtype=torch.int64, device="cuda")
d, n, _ = vt.generate(2, 1 << 20)
s = torch.cuda.current_stream()
for _ in range(3): vt.validate_utf8_device(d, n, d_res=res)
torch.cuda.synchronize()
buf = np.zeros(5, dtype=np.uint64)
for rep in range(3):
    # clear the pads of the last call with a fresh scratch stream each time
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); vt.validate_utf8_device(d, n, stream=st, d_res=res); e1.record(st)
    torch.cuda.synchronize()
    L.vt_debug_probe(st.cuda_stream, buf.ctypes.data)
    first = (~int(buf[0])) & ((1 << 64) - 1)
    print(f"event {e0.elapsed_time(e1) * 1000:.1f} us; CTAs start spread {(int(buf[1]) - first) / 1e3:.1f} us; "
          f"first start -> last end {(int(buf[2]) - first) / 1e3:.1f} us; rule-A {int(buf[4]) >> 32} cycles, generic {int(buf[4]) & 0xffffffff} cycles, masked load {int(buf[3])} cycles")

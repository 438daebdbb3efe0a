import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2109_10433_b200 as vt
d = open(sys.argv[1], "rb").read()
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(d)
d = d[:n]
mode = sys.argv[3] if len(sys.argv) > 3 else "host"
print("n", len(d), "mode", mode, flush=True)
if mode == "host":
    out, r = vt.utf8_to_utf16(d)
elif mode == "validate":
    print(vt.first_error_utf8(d))
else:
    t = torch.frombuffer(bytearray(d), dtype=torch.uint8).cuda()
    o = torch.empty(len(d) + 8, dtype=torch.int16, device="cuda")
    r = vt.utf8_to_utf16_device(t, len(d), o)
print("ok", flush=True)

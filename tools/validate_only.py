"""Runs the UTF-8 and UTF-16 validate kernels on cfg2 / cfg3 (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt
res = torch.zeros(3, dtype=torch.int64, device="cuda")
d, n, _ = vt.generate(2, 1 << 30)
for _ in range(3):
    vt.validate_utf8_device(d, n, d_res=res)
torch.cuda.synchronize()
del d
d, n, _ = vt.generate(3, 1 << 29)
for _ in range(3):
    vt.validate_utf16_device(d, n, d_res=res)
torch.cuda.synchronize()
print("ok")

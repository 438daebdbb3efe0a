import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2109_10433_b200 as vt
d, n, _ = vt.generate(2, 1 << 30)
o = torch.empty(n + 8, dtype=torch.int16, device="cuda")
res = torch.zeros(3, dtype=torch.int64, device="cuda")
for _ in range(3):
    vt.utf8_to_utf16_device(d, n, o, d_res=res)
torch.cuda.synchronize()
print("ok")

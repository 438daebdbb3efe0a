import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2109_10433_b200 as vt
res = torch.zeros(3, dtype=torch.int64, device="cuda")
d, n, _ = vt.generate(2, 1 << 20)
o16 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
for _ in range(3):
    vt.validate_utf8_device(d, n, d_res=res)
    vt.utf8_to_utf16_device(d, n, o16, d_res=res)
torch.cuda.synchronize()
print("ok", n)

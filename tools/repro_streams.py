import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2109_10433_b200 as vt
from oracle_lib import Oracle
O = Oracle()
rng = random.Random(7)
base, _ = vt.generate_host_chunk(5, 7, 0); base = bytes(base)
cases = []
for _ in range(4):
    n = rng.choice([0, 7, 1000, 65_000, 70_000, 300_000, len(base)])
    d = bytearray(base[:n])
    if d and rng.random() < 0.4:
        d[rng.randrange(len(d))] = 0xFF
    cases.append(bytes(d))
for ci, d in enumerate(cases):
    n = len(d)
    want, w = O.utf8_to_utf16(d)
    din = torch.frombuffer(bytearray(d + b"\0"), dtype=torch.uint8).cuda()
    dout = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    r = vt.utf8_to_utf16_device(din, n, dout)
    print(ci, n, "oracle", (w.consumed, w.written, w.error_at), "sync", (r.consumed, r.written, r.error_at))
    for reps in (1, 3):
        for sname in ("default", "new"):
            s = torch.cuda.current_stream() if sname == "default" else torch.cuda.Stream()
            dres = torch.zeros(3, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            for _ in range(reps):
                vt.utf8_to_utf16_device(din, n, dout, stream=s, d_res=dres)
            s.synchronize()
            ra = vt.result_from_device(dres)
            print("   reps", reps, sname, (ra.consumed, ra.written, ra.error_at))
    print("   err pos byte", d[w.error_at:w.error_at+4].hex() if w.error_at is not None else None, "tail", d[-8:].hex())

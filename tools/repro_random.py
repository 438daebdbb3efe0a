"""Replays tests/test_gpu_parity.py::test_random_differential call by call
(debug helper: prints each call before it runs)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2109_10433_b200 as vt  # noqa: E402
from test_gpu_parity import _gen_text  # noqa: E402

rng = np.random.default_rng(20260823)
mixes = [(100, 0, 0, 0), (22, 78, 0, 0), (1, 0, 99, 0), (0, 0, 0, 100), (25, 25, 25, 25), (50, 0, 50, 0)]
for it in range(1500):
    kind = it % 3
    n = int(rng.choice([int(rng.integers(0, 300)), int(rng.integers(0, 40000))]))
    if kind == 0:
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    else:
        data = bytearray(_gen_text(rng, max(1, n // 2), mixes[it % 6]).encode()[:n])
        if kind == 2 and data:
            for _ in range(int(rng.integers(1, 4))):
                data[int(rng.integers(0, len(data)))] ^= 1 << int(rng.integers(0, 8))
        data = bytes(data)
    print(it, kind, len(data), flush=True)
    try:
        out, r = vt.utf8_to_utf16(data)
    except Exception as e:
        print("FAIL utf8_to_utf16", it, e, flush=True)
        open("gpurun_out/repro_case.bin", "wb").write(data)
        raise
    e = vt.first_error_utf8(data)
    if r.error_at is None:
        back, rb = vt.utf16_to_utf8(out)
    u = rng.integers(0, 65536, n // 2, dtype=np.uint16) if kind == 0 else \
        np.frombuffer(data.decode("utf-8", "replace").encode("utf-16-le"), dtype=np.uint16).copy()
    if kind == 2 and len(u):
        u[int(rng.integers(0, len(u)))] ^= 1 << int(rng.integers(0, 16))
    vt.utf16_to_utf8(u)
    vt.validate_utf16(u)
print("all ok")

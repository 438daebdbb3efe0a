"""Small multi-tile workload over every kernel of libvtrans_gpu.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py

Each call is checked against the oracle as well, so a run that completes
without hazards also completed correctly.  Sizes are a few tiles (16 KiB of
input per UTF-8 tile, 8192 units per UTF-16 tile) so the sanitizers finish in
minutes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2109_10433_b200 as vt  # noqa: E402
from oracle_lib import Oracle  # noqa: E402


def same(r, w):
    return (r.consumed, r.written, r.error_at) == (w.consumed, w.written, w.error_at)


def main():
    orc = Oracle()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(7)
    ok = True
    # UTF-8 -> UTF-16: valid multi-tile (cfg2 and the 4-byte-heavy cfg5 mix),
    # then errors in the first tile, a middle tile and the last bytes
    for cfg, size in ((2, 200_000), (5, 150_000), (1, 70_000)):
        d, n, _ = vt.generate(cfg, size)
        host = d[:n].cpu().numpy()
        cases = [host]
        for pos in (3, n // 2, n - 1):
            b = host.copy()
            b[pos] = 0x80 if b[pos] < 0x80 else 0xFF
            cases.append(b)
        for h in cases:
            dd = torch.from_numpy(h).cuda()
            o = torch.zeros(len(h) + 8, dtype=torch.int16, device="cuda")
            r = vt.utf8_to_utf16_device(dd, len(h), o)
            wo, w = orc.utf8_to_utf16(h)
            ok &= same(r, w) and np.array_equal(o[: r.written].cpu().numpy().view(np.uint16), wo)
            ok &= vt.validate_utf8_device(dd, len(h)).error_at == w.error_at
            if w.error_at is None:
                r2 = vt.utf8_to_utf16_nonvalidating_device(dd, len(h), o)
                ok &= same(r2, w)
                o8 = torch.zeros(3 * r.written + 16, dtype=torch.uint8, device="cuda")
                u16 = o[: r.written].clone()
                r3 = vt.utf16_to_utf8_device(u16, r.written, o8)
                ok &= r3.error_at is None and torch.equal(o8[: len(h)].cpu(), torch.from_numpy(h))
    # UTF-16 -> UTF-8 with pairing errors
    d, n, _ = vt.generate(3, 60_000)
    u = d[:n].cpu().numpy().view(np.uint16)
    for pos in (None, 1, n // 3, n - 1):
        x = u.copy()
        if pos is not None:
            x[pos] = 0xDC00
        dd = torch.from_numpy(x.view(np.int16)).cuda()
        o = torch.zeros(3 * len(x) + 16, dtype=torch.uint8, device="cuda")
        r = vt.utf16_to_utf8_device(dd, len(x), o)
        wo, w = orc.utf16_to_utf8(x)
        ok &= same(r, w) and np.array_equal(o[: r.written].cpu().numpy(), wo)
        ok &= vt.validate_utf16_device(dd, len(x)).error_at == w.error_at
    # host-pointer pipeline (several chunks would be 32 MiB each: one chunk here),
    # zero-copy path, UTF-16BE and transcode_bytes
    text = ("aé鏡\U0001F600" * 5000).encode()
    o, r = vt.utf8_to_utf16(text)
    ok &= r.error_at is None and bytes(o.astype("<u2").tobytes()) == text.decode().encode("utf-16-le")
    o8, r8 = vt.utf16_to_utf8(np.frombuffer(text.decode().encode("utf-16-le"), dtype=np.uint16))
    ok &= r8.error_at is None and bytes(o8) == text
    # streaming validator over random chunkings
    sv = vt.Utf8StreamValidator()
    pos = 0
    while pos < len(text):
        k = int(rng.integers(1, 5000))
        sv.feed(text[pos:pos + k])
        pos += k
    ok &= sv.finish()
    # batches
    data, offs = orc.fuzz_cases(11, 3000, 64)
    count = len(offs) - 1
    dd = torch.from_numpy(data).cuda()
    do = torch.from_numpy(offs.view(np.int64)).cuda()
    out = torch.zeros(int(offs[-1]) + 8, dtype=torch.int16, device="cuda")
    res = torch.zeros((count, 3), dtype=torch.int64, device="cuda")
    vt.utf8_to_utf16_batch_device(dd, do, count, out, res)
    _, wres = orc.utf8_to_utf16_batch(data, offs)
    ok &= np.array_equal(res.cpu().numpy(), wres)
    fe = torch.zeros(count, dtype=torch.int64, device="cuda")
    vt.validate_utf8_batch(dd, do, count, fe)
    torch.cuda.synchronize()
    print("SANITIZE WORKLOAD", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

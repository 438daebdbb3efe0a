"""The reference entry points are pure and safe to call concurrently on
disjoint buffers (SURVEY.md 8(b) "Threading").  The GPU
boundary keeps per-thread host contexts and per-(device, stream) scratch: many
host threads calling at once, and one thread driving several streams, must
each get exactly the oracle's answer."""
import random
import threading

import numpy as np
import pytest

import paper_2109_10433_b200 as vt

pytestmark = pytest.mark.gpu


def _cases(seed, count):
    rng = random.Random(seed)
    base, _ = vt.generate_host_chunk(5, seed, 0)
    base = bytes(base)
    out = []
    for _ in range(count):
        n = rng.choice([0, 7, 1000, 65_000, 70_000, 300_000, len(base)])
        d = bytearray(base[:n])
        if d and rng.random() < 0.4:
            d[rng.randrange(len(d))] = 0xFF
        out.append(bytes(d))
    return out


def test_many_host_threads(oracle):
    results, errors = {}, []

    def worker(t):
        try:
            for i, d in enumerate(_cases(100 + t, 12)):
                u16, r = vt.utf8_to_utf16(d)
                u8, r8 = vt.utf16_to_utf8(u16)
                results[(t, i)] = (d, u16, r, u8, r8)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    assert len(results) == 8 * 12
    for (t, i), (d, u16, r, u8, r8) in results.items():
        want16, w = oracle.utf8_to_utf16(d)
        assert (r.consumed, r.written, r.error_at) == (w.consumed, w.written, w.error_at), (t, i)
        assert np.array_equal(u16, want16), (t, i)
        want8, w8 = oracle.utf16_to_utf8(want16)
        assert (r8.written, r8.error_at) == (w8.written, w8.error_at) and bytes(u8) == bytes(want8)


def test_streams_in_flight(oracle, torch):
    """Asynchronous calls on four streams at once, each with its own buffers."""
    cases = _cases(7, 4)
    streams = [torch.cuda.Stream() for _ in cases]
    outs = []
    for d, s in zip(cases, streams):
        n = len(d)
        din = torch.frombuffer(bytearray(d + b"\0"), dtype=torch.uint8).cuda()
        dout = torch.empty(n + 8, dtype=torch.int16, device="cuda")
        dres = torch.zeros(3, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):  # repeated launches reuse the stream's scratch
            vt.utf8_to_utf16_device(din, n, dout, stream=s, d_res=dres)
        outs.append((d, din, dout, dres, s))  # keep din alive until the streams finish
    for d, _din, dout, dres, s in outs:
        s.synchronize()
        r = vt.result_from_device(dres)
        want, w = oracle.utf8_to_utf16(d)
        assert (r.consumed, r.written, r.error_at) == (w.consumed, w.written, w.error_at)
        got = dout[: r.written].cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want)

"""Multi-rank sharding path on CPU: world_size 2 over gloo.

Each rank takes its character-boundary shard (the product's split rule) and
runs a shard transcoder; results are combined with one all_gather of three
integers (paper_2109_10433_b200/sharding.py), exactly as bench.py does across
GPUs.  Here the per-shard transcoder is the CPU oracle (test-only), so the
check is of the split + combine logic the GPUs rely on."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from oracle_lib import Oracle

        from paper_2109_10433_b200 import sharding

        orc = Oracle()
        outs = []
        for data, utf16 in cases:
            fn = orc.utf16_to_utf8 if utf16 else orc.utf8_to_utf16
            out, g, off = sharding.distributed_transcode(data, rank, world, fn, utf16=utf16)
            outs.append((out, (g.consumed, g.written, g.error_at), off))
        q.put((rank, outs))
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding(oracle):
    rng = np.random.default_rng(21)
    cases = []
    for i in range(12):
        text = "".join(chr(int(c)) for c in rng.choice([0x41, 0x7A, 0xE9, 0x93E1, 0x1F600], 300))
        b = bytearray(text.encode())
        if i % 3 == 1:
            b[int(rng.integers(0, len(b)))] = 0xFF
        if i % 3 == 2:
            b[len(b) // 2 + int(rng.integers(-2, 3))] = 0x80  # near the split
        cases.append((np.frombuffer(bytes(b), dtype=np.uint8).copy(), False))
        u = np.frombuffer(text.encode("utf-16-le"), dtype=np.uint16).copy()
        if i % 2:
            u[len(u) // 2] = 0xDC00
        cases.append((u, True))
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for r in got:
        assert not isinstance(got[r], str), got[r]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (data, utf16) in enumerate(cases):
        want_out, want = (oracle.utf16_to_utf8 if utf16 else oracle.utf8_to_utf16)(data)
        g0, g1 = got[0][ci][1], got[1][ci][1]
        assert g0 == g1 == (want.consumed, want.written, want.error_at)
        # concatenating rank outputs at their offsets reproduces the whole output
        out = np.zeros(max(1, want.written + 16), dtype=want_out.dtype)
        for r in range(2):
            o, _, off = got[r][ci]
            k = max(0, min(len(o), want.written - off))
            out[off:off + k] = o[:k]
        assert np.array_equal(out[: want.written], want_out)

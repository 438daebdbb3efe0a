"""Runtime behaviour on the GPU: the host sharder's resource use across calls,
the device-resident sharded entry points against the oracle, per-thread
streams from several host threads, and the refusal of CUDA-graph capture."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2109_10433_b200 as vt

pytestmark = pytest.mark.gpu


def _free_bytes(torch):
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


def test_host_sharder_does_not_leak(torch):
    """100 calls of vt_sharded_utf8_to_utf16 on a 64 MiB input: device memory
    stays within 64 MiB of where it was after the first call (per-call host
    threads used to leave ~288 MiB of buffers per shard behind)."""
    d, n, _ = vt.generate(2, 64 << 20)
    host = d[:n].cpu().numpy()
    out, r = vt.sharded_utf8_to_utf16(host, 4)
    want = vt.utf8_to_utf16_device(d, n, torch.empty(n + 8, dtype=torch.int16, device="cuda"))
    assert (r.consumed, r.written, r.error_at) == (want.consumed, want.written, want.error_at)
    f0 = _free_bytes(torch)
    for _ in range(100):
        _, r2 = vt.sharded_utf8_to_utf16(host, 4)
        assert r2 == r
    f1 = _free_bytes(torch)
    assert f0 - f1 < (64 << 20), (f0 - f1) / 2**20


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_device_sharded_matches_oracle(torch, oracle, cfg):
    """Consecutive character-boundary shards, each a separate device buffer (all
    on cuda:0 here: one GPU per call on this box), transcoded by
    vt_sharded_device_*; outputs concatenated at the returned offsets equal the
    oracle's whole-stream output, the combined result equals its result."""
    d, n, _ = vt.generate(cfg, 24 << 20 if cfg != 3 else 12 << 20)
    host = d[:n].cpu().numpy()
    if cfg == 3:
        host = host.view(np.uint16)
    k = 5
    cuts = [0]
    for i in range(1, k):
        cut = n * i // k
        cuts.append(max(cuts[-1], vt.split_point_utf16(host, cut) if cfg == 3 else vt.split_point_utf8(host, cut)))
    cuts.append(n)
    shards, outs = [], []
    for i in range(k):
        piece = torch.from_numpy(host[cuts[i]:cuts[i + 1]].copy().view(np.int16 if cfg == 3 else np.uint8)).cuda()
        shards.append((piece, cuts[i + 1] - cuts[i]))
        m = cuts[i + 1] - cuts[i]
        outs.append(torch.empty(3 * m + 16 if cfg == 3 else m + 8, dtype=torch.uint8 if cfg == 3 else torch.int16,
                                device="cuda"))
    if cfg == 3:
        g, per, offs = vt.sharded_device_utf16_to_utf8(shards, outs)
        want_out, want = oracle.utf16_to_utf8(host)
    else:
        g, per, offs = vt.sharded_device_utf8_to_utf16(shards, outs)
        want_out, want = oracle.utf8_to_utf16(host)
    assert (g.consumed, g.written, g.error_at) == (want.consumed, want.written, want.error_at)
    got = np.concatenate([outs[i][: per[i].written].cpu().numpy() for i in range(k)])[: g.written]
    assert np.array_equal(got.view(want_out.dtype), want_out)
    assert offs == list(np.concatenate([[0], np.cumsum([p.written for p in per])[:-1]]))


def test_per_thread_streams_from_two_threads(torch):
    """Two host threads enqueue on cudaStreamPerThread (one handle, a different
    real stream in each thread) at the same time; each gets its own control
    block, so both results stay exact."""
    L = vt.lib()
    d, n, _ = vt.generate(2, 16 << 20)
    want = vt.utf8_to_utf16_device(d, n, torch.empty(n + 8, dtype=torch.int16, device="cuda"))
    per_thread = C.c_void_p(2)  # cudaStreamPerThread
    errs = []

    def work():
        try:
            torch.cuda.set_device(0)
            out = torch.empty(n + 8, dtype=torch.int16, device="cuda")
            r = vt._CRes()
            for _ in range(40):
                rc = L.vt_utf8_to_utf16(d.data_ptr(), n, out.data_ptr(), C.byref(r), per_thread)
                assert rc == 0, rc
                assert (r.consumed, r.written, r.error_at) == (want.consumed, want.written, -1)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))
    ts = [threading.Thread(target=work) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs


def test_graph_capture_is_refused(torch):
    """A call recorded into a CUDA graph would replay one status epoch: the
    library refuses capture (VT_E_ARG) instead of returning wrong offsets."""
    d, n, _ = vt.generate(2, 1 << 20)
    out = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    res = torch.zeros(3, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    rc = None
    with torch.cuda.stream(s):
        g.capture_begin()
        try:
            rc = vt.lib().vt_utf8_to_utf16_async(d.data_ptr(), n, out.data_ptr(), res.data_ptr(),
                                                  s.cuda_stream)
        finally:
            g.capture_end()
    assert rc == -2
    # the stream is usable afterwards
    r = vt.utf8_to_utf16_device(d, n, out)
    assert r.error_at is None

"""Batched short strings and the non-validating path
against the oracle.

* A differential fuzz of 10^6 cases shaped like the reference's run_fuzz
  (proj/src/harness.cpp:388-436: random bytes / valid text / valid text with
  one bit flipped, lengths 0..256, seed 20260823) in ONE launch per check:
  validating UTF-8 -> UTF-16, the non-validating decode on the valid cases,
  the round trip back through UTF-16 -> UTF-8, and UTF-16 -> UTF-8 of the
  same bytes read as little-endian units (units_from_bytes,
  proj/src/harness.cpp:179-186) -- the four checks check_utf8_case /
  check_utf16_case make per case, compared per string with the scalar codec.
* The whole-buffer non-validating kernel (vtrans::utf8_to_utf16(...,
  validate=false), proj/src/utf8_to_utf16.cpp:230-239) equals the validating
  one on valid input (cfg1/2/5 shapes), and stays within n units on garbage."""
import numpy as np
import pytest

import paper_2109_10433_b200 as vt

pytestmark = pytest.mark.gpu


def _valid_mask(offsets, written):
    """Positions [off_i, off_i + written_i) of every string, as a mask over the
    packed output (offsets in output elements)."""
    lens = np.diff(offsets).astype(np.int64)
    total = int(offsets[-1])
    sid = np.repeat(np.arange(len(lens)), lens)
    rel = np.arange(total) - offsets[:-1].astype(np.int64)[sid]
    return rel < written[sid]


def _cmp_batch(torch, got_out, got_res, want_out, want_res, offsets, scale=1):
    assert np.array_equal(got_res, want_res), np.nonzero((got_res != want_res).any(axis=1))[0][:10]
    m = _valid_mask(offsets * scale, got_res[:, 1]) if scale == 1 else None
    if scale == 1:
        n = int(offsets[-1])
        assert np.array_equal(got_out[:n][m], want_out[:n][m])
    else:
        # UTF-8 outputs at 3 * offset: expand the per-string windows
        lens = np.diff(offsets).astype(np.int64) * 3
        starts = offsets[:-1].astype(np.int64) * 3
        sid = np.repeat(np.arange(len(lens)), lens)
        pos = np.arange(int(lens.sum())) + np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
        keep = (pos - starts[sid]) < got_res[sid, 1]
        assert np.array_equal(got_out[pos[keep]], want_out[pos[keep]])


def test_batched_fuzz_million_cases(torch, oracle):
    data, offs = oracle.fuzz_cases(20260823, 1_000_000, 256)
    count = len(offs) - 1
    d_data = torch.from_numpy(data).cuda()
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    n = int(offs[-1])
    # 1. validating UTF-8 -> UTF-16
    d_out = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    d_res = torch.zeros((count, 3), dtype=torch.int64, device="cuda")
    before = vt.launch_count()
    vt.utf8_to_utf16_batch_device(d_data, d_offs, count, d_out, d_res, validate=True)
    assert vt.launch_count() - before == 1
    want_out, want_res = oracle.utf8_to_utf16_batch(data, offs)
    got_res = d_res.cpu().numpy()
    _cmp_batch(torch, d_out.cpu().numpy().view(np.uint16), got_res, want_out, want_res, offs)
    valid = want_res[:, 2] < 0
    assert 0.3 < valid.mean() < 0.9  # both kinds of case are well represented
    # 2. non-validating, on the valid cases only (the reference compares it there)
    d_out2 = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    d_res2 = torch.zeros((count, 3), dtype=torch.int64, device="cuda")
    vt.utf8_to_utf16_batch_device(d_data, d_offs, count, d_out2, d_res2, validate=False)
    r2 = d_res2.cpu().numpy()
    assert np.array_equal(r2[valid], want_res[valid])
    m = _valid_mask(offs, np.where(valid, want_res[:, 1], 0))
    assert np.array_equal(d_out2.cpu().numpy().view(np.uint16)[:n][m], want_out[:n][m])
    assert (r2[:, 1] <= np.diff(offs).astype(np.int64)).all()  # bounded on garbage too
    # 3. round trip of the valid cases: their UTF-16 back to UTF-8 is the input
    d_out3 = torch.zeros(3 * n + 16, dtype=torch.uint8, device="cuda")
    d_res3 = torch.zeros((count, 3), dtype=torch.int64, device="cuda")
    # (string i's units live at offs[i] with length written_i: describe them
    # by their own offsets through a packed copy)
    w = np.where(valid, want_res[:, 1], 0).astype(np.uint64)
    uoffs = np.concatenate([[0], np.cumsum(w)]).astype(np.uint64)
    packed = want_out[np.nonzero(_valid_mask(offs, w.astype(np.int64)))[0]]
    d_u16 = torch.from_numpy(packed.view(np.int16).copy()).cuda()
    vt.utf16_to_utf8_batch_device(d_u16, torch.from_numpy(uoffs.view(np.int64)).cuda(), count, d_out3, d_res3)
    r3 = d_res3.cpu().numpy()
    assert (r3[:, 2] < 0).all() and np.array_equal(r3[:, 1], np.where(valid, np.diff(offs).astype(np.int64), 0))
    o3 = d_out3.cpu().numpy()
    for i in np.nonzero(valid)[0][:: 997]:  # sampled byte-for-byte
        a, b = int(offs[i]), int(offs[i + 1])
        s3 = 3 * int(uoffs[i])
        assert bytes(o3[s3: s3 + (b - a)]) == bytes(data[a:b])
    # 4. UTF-16 -> UTF-8 of the bytes read as LE units (odd tail byte dropped)
    units_lens = np.diff(offs) // 2
    uo = np.concatenate([[0], np.cumsum(units_lens)]).astype(np.uint64)
    starts = offs[:-1].astype(np.int64)
    sid = np.repeat(np.arange(count), units_lens.astype(np.int64))
    k = np.arange(int(uo[-1])) - uo[:-1].astype(np.int64)[sid]
    lo = data[starts[sid] + 2 * k].astype(np.uint16)
    hi = data[starts[sid] + 2 * k + 1].astype(np.uint16)
    units = lo | (hi << 8)
    d_units = torch.from_numpy(units.view(np.int16).copy()).cuda()
    d_out4 = torch.zeros(3 * len(units) + 16, dtype=torch.uint8, device="cuda")
    d_res4 = torch.zeros((count, 3), dtype=torch.int64, device="cuda")
    vt.utf16_to_utf8_batch_device(d_units, torch.from_numpy(uo.view(np.int64)).cuda(), count, d_out4, d_res4)
    want4, wres4 = oracle.utf16_to_utf8_batch(units, uo)
    _cmp_batch(torch, d_out4.cpu().numpy(), d_res4.cpu().numpy(), want4, wres4, uo, scale=3)


@pytest.mark.parametrize("cfg", [1, 2, 5])
def test_nonvalidating_equals_validating_on_valid_input(torch, cfg):
    d, n, _ = vt.generate(cfg, (16 << 20) if cfg == 1 else (256 << 20))
    o1 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    o2 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    r1 = vt.utf8_to_utf16_device(d, n, o1)
    r2 = vt.utf8_to_utf16_nonvalidating_device(d, n, o2)
    assert r1.error_at is None and r2 == r1
    assert torch.equal(o1[: r1.written], o2[: r1.written])


def test_nonvalidating_full_size_cfg2(torch):
    d, n, _ = vt.generate(2, 1 << 30)
    o1 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    o2 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    r1 = vt.utf8_to_utf16_device(d, n, o1)
    r2 = vt.utf8_to_utf16_nonvalidating_device(d, n, o2)
    assert r2 == r1 and torch.equal(o1[: r1.written], o2[: r1.written])


def test_nonvalidating_bounded_on_garbage(torch, oracle):
    rng = np.random.default_rng(5)
    for n in (1, 7, 64, 4095, 70001, 1 << 20):
        host = rng.integers(0, 256, n, dtype=np.uint8)
        host[rng.integers(0, n, max(1, n // 7))] = 0xF4  # many 4-byte leads
        d = torch.from_numpy(host).cuda()
        guard = torch.full((n + 4096,), 0x5A5A, dtype=torch.int16, device="cuda")
        r = vt.utf8_to_utf16_nonvalidating_device(d, n, guard)
        assert r.error_at is None and r.consumed == n and r.written <= n
        assert (guard[n:] == 0x5A5A).all()  # nothing written past the capacity
        out, rh = vt.utf8_to_utf16_nonvalidating(host)
        assert rh.written == r.written
    # valid strings through the host form: equal to the validating path
    for text in ["", "a", "é鏡\U0001F600" * 999, "x" * 70000 + "\U00010348"]:
        b = text.encode()
        a1, q1 = vt.utf8_to_utf16(b)
        a2, q2 = vt.utf8_to_utf16_nonvalidating(b)
        assert q1 == q2 and np.array_equal(a1, a2)

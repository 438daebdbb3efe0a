"""GPU parity for SURVEY.md 8(f) row 4: the streaming UTF-8 validator
(vtrans::Utf8BlockValidator, proj/include/vtrans/validation.hpp:15-24, and its
chunked C-ABI form) and the benchmark-record / corpus-statistics producer
(vtrans::harness, proj/include/vtrans/harness.hpp:14-55).

Streaming verdicts and first-error indices are checked against the oracle's
whole-buffer validation of the concatenated chunks; the expected harness
values are the reference's own test expectations (proj/tests/test_harness.cpp,
test_validation.cpp:160-170)."""
import os
import random
import subprocess

import numpy as np
import pytest

import paper_2109_10433_b200 as vt
import paper_2109_10433_b200.harness as h

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _completable(oracle, data) -> bool:
    """Some continuation of `data` is valid UTF-8 (its only defect is a
    sequence cut by the end)."""
    data = bytes(data)
    return oracle.validate_utf8(data) is None or any(
        oracle.validate_utf8(data + bytes([first] + [0x80] * (k - 1))) is None
        for k in (1, 2, 3) for first in (0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF))


def _expect(oracle, data):
    """(error_at, finish) of a stream fed `data`: whole-buffer validation,
    except that a sequence cut by the end is pending, not an error."""
    e = oracle.validate_utf8(data)
    if e is not None and _completable(oracle, data):
        return None, False
    return e, e is None


def _feed_all(data: bytes, cuts):
    v = vt.Utf8StreamValidator()
    prev = 0
    for c in list(cuts) + [len(data)]:
        v.feed(data[prev:c])
        prev = c
    return v


def test_block_validator_matches_whole_buffer(oracle):
    # proj/tests/test_validation.cpp:160-170: 500 x 192 random bytes < 0xF8, 3 blocks of 64
    rng = np.random.default_rng(7)
    for _ in range(500):
        buf = (rng.integers(0, 2**63, 192, dtype=np.uint64) % 0xF8).astype(np.uint8).tobytes()
        v = _feed_all(buf, [64, 128])
        assert v.finish() == (oracle.validate_utf8(buf) is None)
        assert (v.error_at, v.finish()) == _expect(oracle, buf), buf.hex()


SEQS = ["24", "c2a3", "e98fa1", "f0908d88", "e0a080", "ed9fbf", "f48fbfbf", "efbfbf",
        # invalid: overlong, surrogate, > U+10FFFF, truncated, stray, forbidden
        "c0af", "e09f80", "eda080", "f48fbfbf" "f4908080", "e98f41", "80", "f8", "c1bf", "f08f8080"]


def test_every_seam_position(oracle):
    """Each sequence in a valid context, cut at every position (and at every
    pair of positions)."""
    for s in SEQS:
        data = b"ab" + bytes.fromhex(s) + b"\xe9\x8f\xa1z"
        want = oracle.validate_utf8(data)
        for i in range(len(data) + 1):
            v = _feed_all(data, [i])
            assert v.error_at == want and v.finish() == (want is None), (s, i)
            for j in range(i, len(data) + 1):
                v = _feed_all(data, [i, j])
                assert v.error_at == want and v.finish() == (want is None), (s, i, j)


def test_dangling_sequence_is_only_an_error_at_finish(oracle):
    v = vt.Utf8StreamValidator()
    v.feed(b"abc\xf0\x90")
    assert v.ok_so_far() and not v.finish() and v.error_at is None
    v.feed(b"\x8d")
    assert v.ok_so_far() and not v.finish()
    v.feed(b"\x88")
    assert v.ok_so_far() and v.finish() and v.fed == 7
    v.feed(b"\xe0\x9f")  # overlong prefix: an error as soon as it is seen
    assert not v.ok_so_far() and v.error_at == 7
    v.feed(b"valid afterwards")
    assert not v.finish() and v.error_at == 7


def test_random_chunkings(oracle):
    rng = random.Random(11)
    base, _ = vt.generate_host_chunk(4, 4, 0)
    base = bytes(base[:300_000])
    for it in range(60):
        data = bytearray(base[: rng.randrange(1, len(base))])
        for _ in range(rng.randrange(0, 3)):  # mutations
            if data:
                data[rng.randrange(len(data))] = rng.randrange(256)
        data = bytes(data)
        want = _expect(oracle, data)
        k = rng.randrange(0, 12)
        cuts = sorted(rng.randrange(0, len(data) + 1) for _ in range(k))
        v = _feed_all(data, cuts)
        assert (v.error_at, v.finish()) == want, (it, cuts, want, v.error_at)


def test_device_chunks_large(oracle, torch):
    d, n, first = vt.generate(4, 160 << 20)
    host = d[:n].cpu().numpy()
    want = oracle.validate_utf8(host)
    assert want == first and want is not None
    v = vt.Utf8StreamValidator()
    cuts = [0, 5_000_001, 5_000_003, 17 << 20, (17 << 20) + 1, 40 << 20, 90 << 20, n]
    for a, b in zip(cuts, cuts[1:]):
        v.feed(d[a:b])
    assert v.error_at == want and v.fed == n
    # clean prefix before the first error: valid, complete at a boundary
    ok = int(vt.split_point_utf8(host, want))
    v = vt.Utf8StreamValidator()
    for a, b in zip([0, 1 << 20, 3 << 20], [1 << 20, 3 << 20, max(ok, 3 << 20)]):
        v.feed(d[a:b])
    assert v.finish() == (oracle.validate_utf8(host[:ok]) is None)


def test_dropin_block_validator_cxx(tmp_path, oracle):
    """vtrans::Utf8BlockValidator from a C++ program written against the
    reference header: 3 blocks of 64 per case, verdict vs the oracle."""
    rng = np.random.default_rng(5)
    cases = [(rng.integers(0, 2**63, 192, dtype=np.uint64) % 0xF8).astype(np.uint8) for _ in range(200)]
    base, _ = vt.generate_host_chunk(2, 2, 0)
    for k in range(40):
        cases.append(np.frombuffer(bytes(base[k * 192:(k + 1) * 192]), dtype=np.uint8))
    blob = tmp_path / "cases.bin"
    blob.write_bytes(b"".join(c.tobytes() for c in cases))
    src = tmp_path / "blk.cpp"
    src.write_text(r'''
#include "vtrans/validation.hpp"
#include <cstdio>
#include <vector>
int main(int, char** argv) {
  FILE* f = std::fopen(argv[1], "rb");
  std::vector<uint8_t> b(192);
  while (std::fread(b.data(), 1, 192, f) == 192) {
    vtrans::Utf8BlockValidator v;
    for (int k = 0; k < 3; k++) v.feed(b.data() + 64 * k);
    std::printf("%d%d\n", (int)v.ok_so_far(), (int)v.finish());
  }
  return 0;
}
''')
    exe = tmp_path / "blk"
    libdir = os.path.join(os.path.dirname(vt.__file__), "lib")  # the in-tree library (not a VT_LIB variant)
    subprocess.run(["g++", "-std=c++20", "-O1", str(src), "-I", os.path.join(ROOT, "include"), "-L", libdir,
                    "-lvtrans_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(blob)], capture_output=True, text=True, timeout=300).stdout.split()
    assert len(out) == len(cases)
    for c, o in zip(cases, out):
        e = oracle.validate_utf8(c)
        # ok_so_far: no error other than a sequence cut by the end of the data,
        # i.e. some completion makes the whole buffer valid
        completable = _completable(oracle, c.tobytes())
        assert o == ("1" if completable else "0") + ("1" if e is None else "0"), (c.tobytes().hex(), o)


def test_compute_stats_reference_example():
    # proj/tests/test_harness.cpp:70-85
    utf8 = b"a" * 10 + b"\xc2\xa3" * 5 + b"\xe9\x8f\xa1" * 4 + b"\xf0\x90\x8d\x88"
    s = h.compute_stats(utf8)
    assert s.chars == 20
    assert s.pct_1byte == pytest.approx(50.0) and s.pct_2byte == pytest.approx(25.0)
    assert s.pct_3byte == pytest.approx(20.0) and s.pct_4byte == pytest.approx(5.0)
    assert s.avg_bytes_per_char_utf8 == pytest.approx(36.0 / 20.0)
    assert s.avg_bytes_per_char_utf16 == pytest.approx((2.0 * 19 + 4.0) / 20.0)
    assert h.compute_stats(b"\xff") is None
    assert h.compute_stats(b"").chars == 0


@pytest.mark.parametrize("cfg", [1, 2, 5])
def test_class_counts_generated(cfg, oracle):
    data, _ = vt.generate_host_chunk(cfg, cfg, 3)
    a = np.asarray(data, dtype=np.uint8)
    for off in (0, 1, 7):  # the large path needs 16-byte alignment internally
        b = a[off:]
        b = b[: int(vt.split_point_utf8(b, len(b) - 5))]
        b = b[int(vt.split_point_utf8(b, 3)):] if off else b
        want = (int(np.sum(b < 0x80)), int(np.sum((b >= 0xC0) & (b < 0xE0))),
                int(np.sum((b >= 0xE0) & (b < 0xF0))), int(np.sum(b >= 0xF0)))
        assert oracle.validate_utf8(b) is None
        assert vt.utf8_class_counts(b) == want


def test_run_bench_records():
    # proj/tests/test_harness.cpp:34-55
    utf8 = bytes([0x24, 0xC2, 0xA3, 0xE9, 0x8F, 0xA1, 0xF0, 0x90, 0x8D, 0x88])
    recs = h.run_bench("mini", utf8, 50)
    assert len(recs) == 4
    for r in recs:
        assert r.dataset == "mini" and r.chars == 4 and r.reps == 50
        assert r.mean_ns >= r.min_ns and r.gchars_per_sec >= 0.0
        assert r.spread_warning == (r.mean_ns > 0 and (r.mean_ns - r.min_ns) / r.mean_ns > 0.01)
    assert [(r.direction, r.impl) for r in recs] == [
        ("utf8_to_utf16", "gpu"), ("utf8_to_utf16", "gpu-host"),
        ("utf16_to_utf8", "gpu"), ("utf16_to_utf8", "gpu-host")]
    assert recs[0].bytes_in == 10 and recs[0].bytes_out == 10
    assert recs[2].bytes_in == 10 and recs[2].bytes_out == 10


def test_prefix_sweep_cuts_on_character_boundaries():
    # proj/tests/test_harness.cpp:57-68
    utf8 = b"\xe9\x8f\xa1" * 40
    recs = h.run_prefix_sweep("sweep", utf8, budget_seconds=0.01)
    assert recs and recs[0].bytes_in == 15 and recs[0].chars == 5
    assert recs[-1].bytes_in == 120 and recs[-1].chars == 40
    assert all(r.reps > 0 for r in recs)


def test_output_lengths(oracle, torch):
    """vt_utf16_len_from_utf8 / vt_utf8_len_from_utf16: the
    transcoding's `written` without writing output, valid and invalid inputs,
    all alignments."""
    rng = random.Random(3)
    base8, _ = vt.generate_host_chunk(4, 4, 1)
    base8 = bytes(base8[:200_000])
    base16, _ = vt.generate_host_chunk(3, 3, 1)
    base16 = np.asarray(base16[:100_000], dtype=np.uint16)
    for it in range(40):
        d = bytearray(base8[: rng.randrange(0, len(base8))])
        if it % 2 and d:
            d[rng.randrange(len(d))] = rng.choice([0x80, 0xC0, 0xED, 0xFF, 0xF4])
        d = bytes(d)
        _, want = oracle.utf8_to_utf16(d)
        assert vt.utf16_len_from_utf8(d) == (want.written if want.error_at is None else None)
        off = it % 16
        t = torch.zeros(len(d) + 32, dtype=torch.uint8, device="cuda")
        if d:
            t[off:off + len(d)] = torch.frombuffer(bytearray(d), dtype=torch.uint8).cuda()
        r = vt.utf16_len_from_utf8_device(t, len(d), offset=off)
        assert (r.written, r.error_at) == (want.written, want.error_at), it
        u = base16[: rng.randrange(0, len(base16))].copy()
        if it % 2 and len(u):
            u[rng.randrange(len(u))] = rng.choice([0xD800, 0xDC00, 0xDBFF])
        _, w16 = oracle.utf16_to_utf8(u)
        assert vt.utf8_len_from_utf16(u) == (w16.written if w16.error_at is None else None)
        t16 = torch.from_numpy(np.concatenate([np.zeros(8, np.uint16), u]).view(np.int16)).cuda()
        r16 = vt.utf8_len_from_utf16_device(t16, len(u), offset=16)
        assert (r16.written, r16.error_at) == (w16.written, w16.error_at), it

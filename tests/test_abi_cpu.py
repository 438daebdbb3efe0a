"""CPU-side checks of the product library: it loads, exports the whole C ABI,
fails loudly without a GPU, and its host-side logic (split points, the
synthetic workload generator) is right.  No kernel runs here."""
import os
import re

import numpy as np
import pytest

import paper_2109_10433_b200 as vt
from paper_2109_10433_b200 import sharding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    try:
        return vt.device_count() > 0
    except Exception:
        return False


def test_library_exports_every_declared_symbol():
    import ctypes

    hdr = open(os.path.join(ROOT, "include", "vtrans_gpu.h")).read()
    names = sorted(set(re.findall(r"^\s*(?:int|void|uint64_t|const char\*)\s+(vt_\w+)\(", hdr, re.M)))
    assert len(names) >= 28, names
    L = ctypes.CDLL(vt.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_drop_in_cxx_symbols_exported():
    """The vtrans:: entry points a reference user links against
    (proj/include/vtrans/*.hpp) are defined in libvtrans_gpu.so."""
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", vt.LIB_PATH], capture_output=True, text=True).stdout
    for mangled in [
        "_ZN6vtrans13utf8_to_utf16ESt4spanIKhLm18446744073709551615EEPtbPNS_12PathCountersE",
        "_ZN6vtrans13utf8_to_utf16ESt4spanIKhLm18446744073709551615EEbRNS_15TranscodeResultEPNS_12PathCountersE",
        "_ZN6vtrans13utf16_to_utf8ESt4spanIKtLm18446744073709551615EEPh",
        "_ZN6vtrans13utf16_to_utf8ESt4spanIKtLm18446744073709551615EERNS_15TranscodeResultE",
        "_ZN6vtrans13validate_utf8ESt4spanIKhLm18446744073709551615EE",
        "_ZN6vtrans14validate_utf16ESt4spanIKtLm18446744073709551615EE",
        "_ZN6vtrans14active_backendEv",
        "_ZN6vtrans24native_backend_availableEv",
        "_ZN6vtrans22force_emulated_backendEb",
        "_ZN6vtrans18Utf8BlockValidator4feedEPKh",
        "_ZNK6vtrans18Utf8BlockValidator9ok_so_farEv",
        "_ZNK6vtrans18Utf8BlockValidator6finishEv",
    ]:
        assert mangled in out, mangled


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(vt.VtransError, match="no CUDA device"):
        vt.utf8_to_utf16(b"abc")
    with pytest.raises(vt.VtransError):
        vt.utf16_to_utf8([0x41])
    with pytest.raises(vt.VtransError):
        vt.validate_utf8(b"")
    with pytest.raises(vt.VtransError):
        vt.Utf8StreamValidator().feed(b"\xe2\x82")
    with pytest.raises(vt.VtransError):
        vt.utf8_class_counts(b"abc")
    assert vt.device_count() == 0


def test_split_point_rules(oracle):
    """shard results combine exactly to the
    whole-input result (checked with the oracle on CPU)."""
    rng = np.random.default_rng(3)
    for trial in range(400):
        n = int(rng.integers(1, 400))
        if trial % 3 == 0:
            data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        else:
            text = "".join(chr(int(c)) for c in rng.choice([0x41, 0xE9, 0x93E1, 0x1F600, 0x10FFFF], n // 3 + 1))
            data = bytearray(text.encode())
            if trial % 3 == 1 and data:
                data[int(rng.integers(0, len(data)))] ^= 1 << int(rng.integers(0, 8))
            data = bytes(data)
        parts = int(rng.integers(1, 9))
        st = sharding.shard_bounds(data, parts)
        assert st[0] == 0 and st[-1] == len(data) and all(a <= b for a, b in zip(st, st[1:]))
        res = [oracle.utf8_to_utf16(data[st[k]:st[k + 1]]) for k in range(parts)]
        g, offs = sharding.combine(st, [r for _, r in res], len(data))
        want_out, want = oracle.utf8_to_utf16(data)
        assert (g.consumed, g.written, g.error_at) == (want.consumed, want.written, want.error_at)
        cat = np.concatenate([o for o, _ in res] + [np.zeros(0, np.uint16)])[: g.written]
        assert np.array_equal(cat, want_out)

        u = np.frombuffer(data.decode("utf-8", "replace").encode("utf-16-le"), dtype=np.uint16).copy()
        if trial % 2 and len(u):
            u[int(rng.integers(0, len(u)))] = int(rng.choice([0xD800, 0xDC00]))
        st16 = sharding.shard_bounds(u, parts, utf16=True)
        res16 = [oracle.utf16_to_utf8(u[st16[k]:st16[k + 1]]) for k in range(parts)]
        g16, _ = sharding.combine(st16, [r for _, r in res16], len(u))
        w8, want16 = oracle.utf16_to_utf8(u)
        assert (g16.consumed, g16.written, g16.error_at) == (want16.consumed, want16.written, want16.error_at)


CLASS_RANGES = {
    1: [((0x20, 0x7E), 0.90), ((0x80, 0x7FF), 0.10)],
    5: [((0x20, 0x7E), 0.60), ((0x80, 0x7FF), 0.15), ((0x800, 0xFFFF), 0.15), ((0x10000, 0x10FFFF), 0.10)],
}


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generator_chunks(cfg, oracle):
    a, fb = vt.generate_host_chunk(cfg, 7, 3)
    b, fb2 = vt.generate_host_chunk(cfg, 7, 3)
    c, _ = vt.generate_host_chunk(cfg, 8, 3)
    assert np.array_equal(a, b) and fb == fb2 and not np.array_equal(a[:64], c[:64])
    if cfg == 3:
        out, r = oracle.utf16_to_utf8(a)
        assert r.error_at is None
        text = a.astype("<u2").tobytes().decode("utf-16-le")
    else:
        out, r = oracle.utf8_to_utf16(a)
        if cfg == 4:
            assert r.error_at == fb  # None when this chunk has no injection
            return
        assert r.error_at is None
        text = a.tobytes().decode("utf-8")
    cps = np.array([ord(ch) for ch in text])
    assert not ((cps >= 0xD800) & (cps <= 0xDFFF)).any()
    if cfg == 2:
        cjk = ((cps >= 0x4E00) & (cps <= 0x9FFF)).mean()
        asc = ((cps >= 0x20) & (cps <= 0x7E)).mean()
        assert 0.35 < cjk < 0.55 and 0.40 < asc < 0.60, (cjk, asc)  # ~53% ASCII chars
    ranges = CLASS_RANGES.get(3 if cfg == 3 else cfg, CLASS_RANGES.get(5) if cfg == 3 else None)
    if cfg in (1, 3, 5):
        ranges = CLASS_RANGES[1] if cfg == 1 else CLASS_RANGES[5]
        for (lo, hi), p in ranges:
            f = ((cps >= lo) & (cps <= hi)).mean()
            assert abs(f - p) < 0.03, (lo, hi, f, p)


def test_generator_cfg4_injections(oracle):
    """cfg 4: injected sequences are where the reference rule reports the error."""
    found = 0
    for chunk in range(0, 60000, 7):
        a, fb = vt.generate_host_chunk(4, 4, chunk)
        if fb is None:
            continue
        _, r = oracle.utf8_to_utf16(a)
        assert r.error_at == fb, (chunk, fb, r.error_at)
        found += 1
        if found >= 6:
            break
    assert found >= 1

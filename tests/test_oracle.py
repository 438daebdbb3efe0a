"""Pin the C restatement (oracle/vt_oracle.c) before trusting it as the checker.

CPU only.  The oracle is checked against
  * the golden vectors in tests/golden/ (from the reference's own tests and the
    reference library compiled out of tree, see tests/golden/make_golden.py);
  * the compiled reference itself (oracle/_ref), differentially, when present;
  * the local per-byte error rule the GPU kernels rely on,
    which must reproduce the oracle's error_at exactly.
"""
import hashlib

import numpy as np
import pytest

from oracle_lib import Reference


def _u16(hexstr):
    return np.frombuffer(bytes.fromhex(hexstr), dtype="<u2").astype(np.uint16)


def test_oracle_utf8_golden(oracle, golden):
    for c in golden["u8"]:
        data = bytes.fromhex(c["in"])
        out, r = oracle.utf8_to_utf16(data)
        assert (r.consumed, r.written, r.error_at) == (c["consumed"], c["written"], c["error_at"]), c["src"]
        if "out" in c:
            assert [int(x) for x in out] == c["out"], c["src"]
        else:
            assert hashlib.sha1(out.astype("<u2").tobytes()).hexdigest() == c["out_sha1"], c["src"]
        assert (oracle.validate_utf8(data) is None) == c["valid"], c["src"]
        assert oracle.count_utf8(data) == c["count"], c["src"]


def test_oracle_utf16_golden(oracle, golden):
    for c in golden["u16"]:
        units = _u16(c["in"])
        out, r = oracle.utf16_to_utf8(units)
        assert (r.consumed, r.written, r.error_at) == (c["consumed"], c["written"], c["error_at"]), c["src"]
        if "out" in c:
            assert bytes(out).hex() == c["out"], c["src"]
        else:
            assert hashlib.sha1(out.tobytes()).hexdigest() == c["out_sha1"], c["src"]
        assert oracle.validate_utf16(units) == c["validate16"], c["src"]
        assert oracle.count_utf16(units) == c["count"], c["src"]


def test_oracle_encode_kats(oracle, golden):
    k = golden["misc"]["encode"]
    for cp, h in k["utf8"].items():
        assert oracle.encode_utf8(int(cp, 16)).hex() == h
    for cp, u in k["utf16"].items():
        assert oracle.encode_utf16(int(cp, 16)) == u


def test_oracle_exhaustive_short(oracle, golden):
    """acceptance.cpp:138-167 (C3): every 1/2/3-byte input, verdict digest."""
    e = golden["misc"]["exhaustive_short"]
    v = oracle.exhaustive_short_verdicts()
    assert int(v.sum()) == e["valid"]
    assert hashlib.sha256(v.tobytes()).hexdigest() == e["sha256"]


def test_oracle_round_trip_all_scalars(oracle):
    """acceptance.cpp:106-134 (C2) restated over all 1,112,064 scalar values at once."""
    cps = [cp for cp in range(0x110000) if not 0xD800 <= cp <= 0xDFFF]
    text = "".join(map(chr, cps))
    b8 = text.encode("utf-8")
    u16, r = oracle.utf8_to_utf16(b8, threads=4)
    assert r.error_at is None and r.consumed == len(b8)
    assert u16.tobytes() == text.encode("utf-16-le")
    back, r2 = oracle.utf16_to_utf8(u16, threads=4)
    assert r2.error_at is None and back.tobytes() == b8
    assert oracle.count_utf8(b8) == len(cps) == oracle.count_utf16(u16)


def test_oracle_mt_matches_single(oracle):
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(0, 5000))
        data = rng.integers(0x20, 0x7F, n, dtype=np.uint8)
        text = bytearray(data.tobytes())
        # splice in multi-byte characters and an occasional error
        for _ in range(n // 20):
            p = int(rng.integers(0, max(1, len(text))))
            text[p:p] = chr(int(rng.choice([0xE9, 0x93E1, 0x1F600]))).encode()
        if trial % 3 == 0 and text:
            text[int(rng.integers(0, len(text)))] = 0xFF
        a, ra = oracle.utf8_to_utf16(bytes(text))
        b, rb = oracle.utf8_to_utf16(bytes(text), threads=int(rng.integers(2, 9)))
        assert ra == rb and np.array_equal(a, b)
        u = np.frombuffer(bytes(text).decode("utf-8", "replace").encode("utf-16-le"), dtype=np.uint16).copy()
        if trial % 2 and len(u):
            u[int(rng.integers(0, len(u)))] = 0xDC00
        a8, ra8 = oracle.utf16_to_utf8(u)
        b8, rb8 = oracle.utf16_to_utf8(u, threads=int(rng.integers(2, 9)))
        assert ra8 == rb8 and np.array_equal(a8, b8)


# --- the local rules the kernels implement, checked against the oracle -------

def _leadlen(b):
    if b < 0x80:
        return 1
    if b >> 5 == 0b110:
        return 2
    if b >> 4 == 0b1110:
        return 3
    if b >> 3 == 0b11110:
        return 4
    return 1


def rule_a_first_error(data: bytes, oracle):
    """error_at = min i with a failing lead decode at i,
    or a continuation at i not covered by any lead in [i-3, i-1]."""
    n = len(data)
    for i, b in enumerate(data):
        if (b & 0xC0) != 0x80:
            # decode failure at a non-continuation byte (lookahead <= 3)
            if oracle.validate_utf8(data[i:i + _leadlen(b)]) is not None and (
                _leadlen(b) > 1 or b >= 0x80
            ):
                return i
            if _leadlen(b) > 1 and i + _leadlen(b) > n:
                return i
        else:
            if not any(j >= 0 and _leadlen(data[j]) > i - j for j in range(i - 3, i)):
                return i
    return None


def rule_c_first_error(u):
    n = len(u)
    for i in range(n):
        x = int(u[i])
        if 0xDC00 <= x <= 0xDFFF and not (i > 0 and 0xD800 <= int(u[i - 1]) <= 0xDBFF):
            return i
        if 0xD800 <= x <= 0xDBFF and not (i + 1 < n and 0xDC00 <= int(u[i + 1]) <= 0xDFFF):
            return i
    return None


def test_rule_a_matches_oracle(oracle):
    rng = np.random.default_rng(11)
    pool = [0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2, 0xDF, 0xE0,
            0xE1, 0xEC, 0xED, 0xEE, 0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5, 0xF7, 0xF8, 0xFF]
    for trial in range(6000):
        n = int(rng.integers(0, 12))
        data = bytes(int(rng.choice(pool)) for _ in range(n))
        assert rule_a_first_error(data, oracle) == oracle.validate_utf8(data), data.hex()


def test_rule_c_matches_oracle(oracle):
    rng = np.random.default_rng(12)
    pool = np.array([0x41, 0x93E1, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000], dtype=np.uint16)
    for trial in range(4000):
        u = pool[rng.integers(0, len(pool), int(rng.integers(0, 10)))]
        assert rule_c_first_error(u) == oracle.validate_utf16(u)


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")
def test_oracle_vs_compiled_reference(oracle):
    ref = Reference()
    rng = np.random.default_rng(99)
    for trial in range(3000):
        n = int(rng.integers(0, 300))
        if trial % 2:
            data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        else:
            data = "".join(chr(int(c)) for c in rng.integers(0x20, 0x2FFF, n // 2) if not 0xD800 <= c <= 0xDFFF).encode()
            if data and trial % 4 == 0:
                m = bytearray(data)
                m[int(rng.integers(0, len(m)))] ^= 1 << int(rng.integers(0, 8))
                data = bytes(m)
        a, ra = oracle.utf8_to_utf16(data)
        b, rb = ref.utf8_to_utf16(data, validate=True)
        assert ra == rb and np.array_equal(a, b)
        assert (oracle.validate_utf8(data) is None) == ref.validate_utf8(data)
        u = rng.integers(0, 65536, n // 2, dtype=np.uint16)
        a8, ra8 = oracle.utf16_to_utf8(u)
        b8, rb8 = ref.utf16_to_utf8(u)
        assert ra8 == rb8 and np.array_equal(a8, b8)
        assert oracle.validate_utf16(u) == ref.validate_utf16(u)

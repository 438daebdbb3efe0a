"""Generate tests/golden/*.json from the UNMODIFIED reference library.

Run in the build container, where /root/reference exists and
``make -C oracle`` has compiled it out of tree into oracle/_ref/:

    python tests/golden/make_golden.py

Inputs come from two sources:
  * the known-answer vectors of the reference's own tests (cited per case);
  * seeded random cases drawn here (numpy PCG64, seeds below), shaped like the
    reference's differential suites.
Expected results are the reference's scalar codec (the normative oracle,
proj/src/codec_core.cpp:85-125); every case also asserts that the reference's
SIMD driver agrees with it, as its contract says.  Outputs of random cases are
stored as SHA-1 digests to keep the fixture small.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Reference  # noqa: E402


def hx(b) -> str:
    return bytes(b).hex()


def digest(a: np.ndarray) -> str:
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def enc8(cp: int) -> bytes:
    return chr(cp).encode("utf-8", "surrogatepass")


def rand_cp(rng, cls: int) -> int:
    if cls == 0:
        return int(rng.integers(0, 0x80))
    if cls == 1:
        return int(rng.integers(0x80, 0x800))
    if cls == 2:
        while True:
            cp = int(rng.integers(0x800, 0x10000))
            if not 0xD800 <= cp <= 0xDFFF:
                return cp
    return int(rng.integers(0x10000, 0x110000))


def gen_valid_utf8(rng, approx_len: int, weights) -> bytes:
    w = np.asarray(weights, dtype=float)
    w = w / w.sum()
    out = bytearray()
    while len(out) < approx_len:
        out += enc8(rand_cp(rng, int(rng.choice(4, p=w))))
    return bytes(out)


def gen_valid_utf16(rng, approx_units: int, weights) -> list[int]:
    w = np.asarray(weights, dtype=float)
    w = w / w.sum()
    out: list[int] = []
    while len(out) < approx_units:
        cp = rand_cp(rng, int(rng.choice(4, p=w)))
        if cp < 0x10000:
            out.append(cp)
        else:
            v = cp - 0x10000
            out += [0xD800 + (v >> 10), 0xDC00 + (v & 0x3FF)]
    return out


def main() -> None:
    ref = Reference()
    assert ref.native, "reference built without its SSE backend"

    u8_cases: list[dict] = []
    u16_cases: list[dict] = []

    def add8(src: str, data: bytes, full: bool = True) -> None:
        out, r = ref.utf8_to_utf16(data, scalar=True)
        out_simd, r_simd = ref.utf8_to_utf16(data, validate=True)
        assert r == r_simd and np.array_equal(out, out_simd), src
        case = {
            "src": src,
            "in": hx(data),
            "consumed": r.consumed,
            "written": r.written,
            "error_at": r.error_at,
            "valid": ref.validate_utf8(data),
            "count": ref.count_utf8(data),
        }
        if full:
            case["out"] = [int(x) for x in out]
        else:
            case["out_sha1"] = digest(out.astype("<u2"))
        u8_cases.append(case)

    def add16(src: str, units, full: bool = True) -> None:
        a = np.asarray(units, dtype=np.uint16)
        out, r = ref.utf16_to_utf8(a, scalar=True)
        out_simd, r_simd = ref.utf16_to_utf8(a)
        assert r == r_simd and np.array_equal(out, out_simd), src
        case = {
            "src": src,
            "in": hx(a.astype("<u2").tobytes()),
            "consumed": r.consumed,
            "written": r.written,
            "error_at": r.error_at,
            "validate16": ref.validate_utf16(a),
            "count": ref.count_utf16(a),
        }
        if full:
            case["out"] = hx(out)
        else:
            case["out_sha1"] = digest(out)
        u16_cases.append(case)

    # --- known-answer vectors of the reference's own tests ------------------
    add8("test_utf8_to_utf16.cpp:62-70 worked", bytes.fromhex("24c2a3e98fa1f0908d88"))
    add8("test_codec_core.cpp:185-196 error index", bytes.fromhex("41c2a3ff42"))
    for h in ["c0af", "c1bf", "e08080", "e09fbf", "f08fbfbf", "eda080", "edbfbf", "f4908080",
              "f5808080", "ff", "80", "e98f", "c3"]:
        add8("test_codec_core.cpp:139-155 malformed", bytes.fromhex(h))
    for h in ["e0a080", "ed9fbf", "ee8080", "f48fbfbf", "f0908080"]:
        add8("test_codec_core.cpp:157-168 boundary", bytes.fromhex(h))
    for h in ["", "41", "c2a3", "e09fbf", "eda080", "f08fbfbf", "f4908080", "c2", "e98f", "f0908d",
              "4180", "c2a3a3"]:
        add8("test_validation.cpp:57-74 probe", bytes.fromhex(h))
    for pos in [0, 1, 15, 63, 64, 65, 67, 68, 100, 127, 128]:
        b = bytearray(b"a" * 140)
        b[pos] = 0xFF
        add8(f"test_utf8_to_utf16.cpp:159-171 seam {pos}", bytes(b))
    add8("test_utf8_to_utf16.cpp:173-184 truncated final", b"a" * 130 + bytes([0xE9, 0x8F]))
    asc = bytearray(b"q" * 5000)
    for i in range(0, len(asc), 7):
        asc[i] = ord("a") + i % 26
    add8("test_utf8_to_utf16.cpp:72-79 ascii", bytes(asc), full=False)
    seqs = {2: bytes([0xC2, 0xA3]), 3: bytes([0xE9, 0x8F, 0xA1]), 4: bytes([0xF0, 0x90, 0x8D, 0x88])}
    for ln in (2, 3, 4):
        for split in range(1, ln):
            buf = b"a" * (64 - split) + seqs[ln] + b"b" * 40
            add8(f"test_validation.cpp:76-98 straddle {ln}/{split}", buf)
            add8(f"test_validation.cpp:76-98 cut {ln}/{split}", buf[:64])
            bad = bytearray(buf)
            bad[64] = 0x41
            add8(f"test_validation.cpp:76-98 bad {ln}/{split}", bytes(bad))
    pat = bytearray()
    while len(pat) < 300:
        pat += bytes([ord("a"), 0xC2, 0xA3, 0xE9, 0x8F, 0xA1, 0xF0, 0x90, 0x8D, 0x88, ord("b"),
                      ord("c"), 0xD9, 0x84, 0xE4, 0xB8, 0xAD])
    for ln in range(0, 257):
        add8(f"acceptance.cpp:208-229 C5 len {ln}", bytes(pat[:ln]), full=ln <= 64)

    add16("test_utf16_to_utf8.cpp:52-58 worked", [0x0024, 0x00A3, 0x93E1, 0xD801, 0xDC37])
    add16("test_codec_core.cpp:198-205 error index", [0x0041, 0xD800, 0x0042])
    for u in ([0xD800], [0xDC00], [0xD800, 0x0041], [0xDC00, 0xD800], [0xD852, 0xDF62], [], [0x41]):
        add16("test_codec_core.cpp:170-183 / test_utf16_to_utf8.cpp:60-63", u)
    add16("test_utf16_to_utf8.cpp:72-78 straddle", [0x41] * 7 + [0xD852, 0xDF62] + [0x93E1] * 20)
    for pos in [0, 3, 7, 8, 15, 16, 31, 40]:
        v = [0x93E1] * 44
        v[pos] = 0xDC00
        add16(f"test_utf16_to_utf8.cpp:80-92 low {pos}", v)
        v[pos] = 0xD800
        add16(f"test_utf16_to_utf8.cpp:80-92 high {pos}", v)
    add16("test_utf16_to_utf8.cpp:88-92 trailing high", [0x41] * 20 + [0xD800])
    v = [0x41] * 16
    v[7], v[8] = 0xD800, 0xDC00
    add16("test_validation.cpp:143-150 pair 7/8", v)
    v[8] = 0x42
    add16("test_validation.cpp:150-153 unpaired 7", v)
    w = [0x93E1] * 40
    w[33] = 0xDC00
    add16("test_validation.cpp:155-158 lone low 33", w)
    reps = [0x0041, 0x93E1, 0xD800, 0xDBFF, 0xDC00, 0xDFFF]
    for a in reps:
        for b in reps:
            for c in reps:
                add16("test_validation.cpp:125-141 class triple", [a, b, c])
    for ln in range(0, 257):
        units = [[0x0041, 0x93E1, 0xD852, 0xDF62, 0x00E9][i % 5] for i in range(ln)]
        add16(f"acceptance.cpp:231-249 C5 len {ln}", units, full=ln <= 64)

    # --- seeded random differential cases ----------------------------------
    rng = np.random.default_rng(20260823)
    profiles = [(100, 0, 0, 0), (22, 78, 0, 0), (1, 0, 99, 0), (0, 0, 0, 100), (25, 25, 25, 25),
                (50, 0, 50, 0)]
    for i in range(300):
        n = int(rng.integers(0, 401))
        add8("random bytes (cf. test_utf8_to_utf16.cpp:141-157)", rng.integers(0, 256, n, dtype=np.uint8).tobytes(), full=False)
    for i in range(240):
        data = gen_valid_utf8(rng, int(rng.integers(0, 700)), profiles[i % 6])
        add8("valid mix (cf. test_utf8_to_utf16.cpp:114-139)", data, full=False)
        if data:
            m = bytearray(data)
            m[int(rng.integers(0, len(m)))] ^= 1 << int(rng.integers(0, 8))
            add8("mutated mix (cf. test_utf8_to_utf16.cpp:114-139)", bytes(m), full=False)
    for i in range(400):
        n = int(rng.integers(0, 200))
        add16("random units (cf. test_utf16_to_utf8.cpp:94-101)", rng.integers(0, 65536, n, dtype=np.uint16), full=False)
    for i in range(200):
        u = gen_valid_utf16(rng, int(rng.integers(0, 300)), (25, 25, 25, 25))
        add16("valid units (cf. test_utf16_to_utf8.cpp:103-113)", u, full=False)
        if u:
            u = list(u)
            u[int(rng.integers(0, len(u)))] ^= 1 << int(rng.integers(0, 16))
            add16("mutated units (cf. test_utf16_to_utf8.cpp:103-113)", u, full=False)

    # --- harness::transcode_bytes: BOM / endianness policy (test_harness.cpp:87-141)
    tb_cases = []
    samples = [b"", "h\u00e9llo \u93e1 \U00010348".encode(), b"\xef\xbb\xbf" + "ab\u00e9".encode(),
               b"\x41\xc2\xa3\xff\x42"]
    u16s = ["hi \u93e1\U00024b62".encode("utf-16-le"), "hi \u93e1\U00024b62".encode("utf-16-be"),
            b"\xff\xfe" + "x\u00e9".encode("utf-16-le"), b"\xfe\xff" + "x\u00e9".encode("utf-16-be"),
            b"\xff\xfea\x00b", b"\x41\x00\x00\xdc", b"\x00\xd8\x41\x00"]
    for data in samples:
        for to in ("utf8", "utf16le", "utf16be"):
            for bom in ("keep", "strip", "add"):
                code, msg, out = ref.transcode_bytes(data, "utf8", to, bom)
                tb_cases.append({"in": hx(data), "from": "utf8", "to": to, "bom": bom, "exit": code,
                                 "msg": msg, "out": hx(out)})
    for data in u16s:
        for frm in ("utf16le", "utf16be"):
            for to in ("utf8", "utf16le", "utf16be"):
                for bom in ("keep", "strip", "add"):
                    code, msg, out = ref.transcode_bytes(data, frm, to, bom)
                    tb_cases.append({"in": hx(data), "from": frm, "to": to, "bom": bom, "exit": code,
                                     "msg": msg, "out": hx(out)})

    verdicts = ref.exhaustive_short_verdicts()
    exhaustive = {
        "src": "acceptance.cpp:138-167 C3: validate_utf8 over every 1/2/3-byte input",
        "count": int(len(verdicts)),
        "valid": int(verdicts.sum()),
        "sha256": hashlib.sha256(verdicts.tobytes()).hexdigest(),
    }
    kats = {
        "src": "test_codec_core.cpp:55-81 worked encodings, acceptance.cpp:96-102 C1",
        "utf8": {hex(cp): enc8(cp).hex() for cp in [0x24, 0xA3, 0x93E1, 0x10348, 0x10437, 0x24B62]},
        "utf16": {"0x93e1": [0x93E1], "0x10437": [0xD801, 0xDC37], "0x24b62": [0xD852, 0xDF62]},
    }
    with open(os.path.join(HERE, "utf8_to_utf16.json"), "w") as f:
        json.dump(u8_cases, f, separators=(",", ":"))
    with open(os.path.join(HERE, "utf16_to_utf8.json"), "w") as f:
        json.dump(u16_cases, f, separators=(",", ":"))
    with open(os.path.join(HERE, "misc.json"), "w") as f:
        json.dump({"exhaustive_short": exhaustive, "encode": kats, "transcode_bytes": tb_cases}, f,
                  indent=1)
    print(f"{len(u8_cases)} utf8 cases, {len(u16_cases)} utf16 cases, exhaustive valid={exhaustive['valid']}")


if __name__ == "__main__":
    main()

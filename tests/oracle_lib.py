"""ctypes bindings for the TEST-ONLY oracle libraries.

* ``oracle/lib/libvt_oracle.so`` -- the C restatement of the reference scalar
  codec (oracle/vt_oracle.c), always available after ``make -C oracle``.
* ``oracle/_ref/libvtrans_ref.so`` -- the unmodified reference library compiled
  out of tree (oracle/Makefile); present where /root/reference was available
  at build time (and shipped to the GPU box with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "lib", "libvt_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libvtrans_ref.so")
GEN_SO = os.path.join(ROOT, "oracle", "lib", "libvt_gen.so")


class CRes(C.Structure):
    _fields_ = [("consumed", C.c_uint64), ("written", C.c_uint64), ("error_at", C.c_int64)]


@dataclass(frozen=True)
class Result:
    """Python view of vtrans::TranscodeResult (error_at None == empty optional)."""

    consumed: int
    written: int
    error_at: int | None

    @staticmethod
    def of(c: CRes) -> "Result":
        return Result(int(c.consumed), int(c.written), None if c.error_at < 0 else int(c.error_at))


_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)


def _p8(a):
    return a.ctypes.data_as(_u8p)


def _p16(a):
    return a.ctypes.data_as(_u16p)


def ensure_built() -> None:
    if not (os.path.exists(ORACLE_SO) and os.path.exists(GEN_SO)):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)


class _Lib:
    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name, res, *args):
        f = getattr(self.lib, self.prefix + name)
        f.restype = res
        f.argtypes = list(args)
        return f


class Oracle:
    """The C restatement (vt_oracle.c)."""

    def __init__(self):
        ensure_built()
        L = _Lib(ORACLE_SO, "vto_")
        self._u8to16 = L.fn("utf8_to_utf16", None, _u8p, C.c_uint64, _u16p, C.POINTER(CRes))
        self._u16to8 = L.fn("utf16_to_utf8", None, _u16p, C.c_uint64, _u8p, C.POINTER(CRes))
        self._u8to16mt = L.fn("utf8_to_utf16_mt", None, _u8p, C.c_uint64, _u16p, C.c_int, C.POINTER(CRes))
        self._u16to8mt = L.fn("utf16_to_utf8_mt", None, _u16p, C.c_uint64, _u8p, C.c_int, C.POINTER(CRes))
        self._v8 = L.fn("validate_utf8", C.c_int64, _u8p, C.c_uint64)
        self._v16 = L.fn("validate_utf16", C.c_int64, _u16p, C.c_uint64)
        self._c8 = L.fn("count_utf8", C.c_int64, _u8p, C.c_uint64)
        self._c16 = L.fn("count_utf16", C.c_int64, _u16p, C.c_uint64)
        self._exh = L.fn("exhaustive_short_verdicts", C.c_uint64, _u8p)
        self._enc8 = L.fn("encode_utf8", C.c_uint32, C.c_uint32, _u8p)
        self._enc16 = L.fn("encode_utf16", C.c_uint32, C.c_uint32, _u16p)
        self._b8 = L.fn("utf8_to_utf16_batch", None, _u8p, C.c_void_p, C.c_uint64, _u16p, C.c_void_p)
        self._b16 = L.fn("utf16_to_utf8_batch", None, _u16p, C.c_void_p, C.c_uint64, _u8p, C.c_void_p)
        self._fz = L.fn("fuzz_cases", C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _u8p, C.c_void_p,
                        C.c_uint64)

    def fuzz_cases(self, seed: int, count: int, max_len: int):
        """(data, offsets): `count` packed cases shaped like the reference's
        run_fuzz (proj/src/harness.cpp:388-436)."""
        cap = count * (max_len + 8) + 16
        data = np.zeros(cap, dtype=np.uint8)
        offs = np.zeros(count + 1, dtype=np.uint64)
        tot = int(self._fz(seed, count, max_len, _p8(data), offs.ctypes.data, cap))
        assert tot != 0xFFFFFFFFFFFFFFFF
        return data[:tot].copy(), offs

    def utf8_to_utf16_batch(self, data, offsets):
        """Per-string scalar transcoding; outputs at the strings' offsets (units).
        Returns (out, results[count, 3] as int64: consumed, written, error_at)."""
        count = len(offsets) - 1
        out = np.zeros(max(1, int(offsets[-1])) + 8, dtype=np.uint16)
        res = np.zeros((count, 3), dtype=np.int64)
        self._b8(_p8(data), offsets.ctypes.data, count, _p16(out), res.ctypes.data)
        return out, res

    def utf16_to_utf8_batch(self, units, offsets):
        count = len(offsets) - 1
        out = np.zeros(3 * max(1, int(offsets[-1])) + 16, dtype=np.uint8)
        res = np.zeros((count, 3), dtype=np.int64)
        self._b16(_p16(units), offsets.ctypes.data, count, _p8(out), res.ctypes.data)
        return out, res

    def utf8_to_utf16(self, data, threads: int = 1):
        a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        a = np.ascontiguousarray(a, dtype=np.uint8)
        out = np.zeros(len(a) + 8, dtype=np.uint16)
        r = CRes()
        if threads > 1:
            self._u8to16mt(_p8(a), len(a), _p16(out), threads, C.byref(r))
        else:
            self._u8to16(_p8(a), len(a), _p16(out), C.byref(r))
        res = Result.of(r)
        return out[: res.written].copy(), res

    def utf16_to_utf8(self, units, threads: int = 1):
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        out = np.zeros(3 * len(a) + 16, dtype=np.uint8)
        r = CRes()
        if threads > 1:
            self._u16to8mt(_p16(a), len(a), _p8(out), threads, C.byref(r))
        else:
            self._u16to8(_p16(a), len(a), _p8(out), C.byref(r))
        res = Result.of(r)
        return out[: res.written].copy(), res

    def validate_utf8(self, data) -> int | None:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data, dtype=np.uint8)
        e = self._v8(_p8(a), len(a))
        return None if e < 0 else int(e)

    def validate_utf16(self, units) -> int | None:
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        e = self._v16(_p16(a), len(a))
        return None if e < 0 else int(e)

    def count_utf8(self, data) -> int | None:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data, dtype=np.uint8)
        c = self._c8(_p8(a), len(a))
        return None if c < 0 else int(c)

    def count_utf16(self, units) -> int | None:
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        c = self._c16(_p16(a), len(a))
        return None if c < 0 else int(c)

    def exhaustive_short_verdicts(self) -> np.ndarray:
        out = np.zeros(256 + 65536 + 16777216, dtype=np.uint8)
        k = self._exh(_p8(out))
        assert k == len(out)
        return out

    def encode_utf8(self, cp: int) -> bytes:
        b = np.zeros(4, dtype=np.uint8)
        k = self._enc8(cp, _p8(b))
        return bytes(b[:k])

    def encode_utf16(self, cp: int) -> list[int]:
        u = np.zeros(2, dtype=np.uint16)
        k = self._enc16(cp, _p16(u))
        return [int(x) for x in u[:k]]


class Reference:
    """The unmodified reference library (oracle/_ref/libvtrans_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        L = _Lib(REF_SO, "vtr_")
        self._u8to16 = L.fn("utf8_to_utf16", None, _u8p, C.c_uint64, _u16p, C.c_int, C.POINTER(CRes))
        self._u16to8 = L.fn("utf16_to_utf8", None, _u16p, C.c_uint64, _u8p, C.POINTER(CRes))
        self._s8to16 = L.fn("scalar_utf8_to_utf16", None, _u8p, C.c_uint64, _u16p, C.POINTER(CRes))
        self._s16to8 = L.fn("scalar_utf16_to_utf8", None, _u16p, C.c_uint64, _u8p, C.POINTER(CRes))
        self._v8 = L.fn("validate_utf8", C.c_int, _u8p, C.c_uint64)
        self._v16 = L.fn("validate_utf16", C.c_int64, _u16p, C.c_uint64)
        self._c8 = L.fn("count_utf8", C.c_int64, _u8p, C.c_uint64)
        self._c16 = L.fn("count_utf16", C.c_int64, _u16p, C.c_uint64)
        self._exh = L.fn("exhaustive_short_verdicts", C.c_uint64, _u8p)
        self._u8to16mt = L.fn("utf8_to_utf16_mt", None, _u8p, C.c_uint64, _u16p, C.c_int, C.POINTER(CRes))
        self._u16to8mt = L.fn("utf16_to_utf8_mt", None, _u16p, C.c_uint64, _u8p, C.c_int, C.POINTER(CRes))
        self._v8mt = L.fn("validate_utf8_mt", C.c_int, _u8p, C.c_uint64, C.c_int)
        self.native = bool(L.fn("native_backend", C.c_int)())
        self._tb = L.fn("transcode_bytes", C.c_int, _u8p, C.c_uint64, C.c_int, C.c_int, C.c_int, _u8p,
                        C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64)

    def transcode_bytes(self, data: bytes, from_format: str, to_format: str, bom: str = "strip"):
        f = {"utf8": 0, "utf16le": 1, "utf16be": 2}
        b = {"keep": 0, "strip": 1, "add": 2}
        a = np.frombuffer(bytes(data), dtype=np.uint8) if data else np.zeros(1, np.uint8)
        cap = 4 * len(data) + 64
        out = np.zeros(cap, dtype=np.uint8)
        n = C.c_uint64()
        msg = C.create_string_buffer(512)
        code = self._tb(_p8(a), len(data), f[from_format], f[to_format], b[bom], _p8(out), cap, C.byref(n),
                        msg, 512)
        return code, msg.value.decode(), bytes(out[: n.value]) if code == 0 else b""

    def utf8_to_utf16(self, data, validate=True, scalar=False, threads=1, out=None):
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data, dtype=np.uint8)
        if out is None:
            out = np.zeros(len(a) + 8, dtype=np.uint16)
        r = CRes()
        if scalar:
            self._s8to16(_p8(a), len(a), _p16(out), C.byref(r))
        elif threads > 1:
            self._u8to16mt(_p8(a), len(a), _p16(out), threads, C.byref(r))
        else:
            self._u8to16(_p8(a), len(a), _p16(out), int(validate), C.byref(r))
        res = Result.of(r)
        return out[: res.written], res

    def utf16_to_utf8(self, units, scalar=False, threads=1, out=None):
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        if out is None:
            out = np.zeros(3 * len(a) + 16, dtype=np.uint8)
        r = CRes()
        if scalar:
            self._s16to8(_p16(a), len(a), _p8(out), C.byref(r))
        elif threads > 1:
            self._u16to8mt(_p16(a), len(a), _p8(out), threads, C.byref(r))
        else:
            self._u16to8(_p16(a), len(a), _p8(out), C.byref(r))
        res = Result.of(r)
        return out[: res.written], res

    def validate_utf8(self, data, threads=1) -> bool:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data, dtype=np.uint8)
        if threads > 1:
            return bool(self._v8mt(_p8(a), len(a), threads))
        return bool(self._v8(_p8(a), len(a)))

    def validate_utf16(self, units) -> int | None:
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        e = self._v16(_p16(a), len(a))
        return None if e < 0 else int(e)

    def count_utf8(self, data) -> int | None:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data, dtype=np.uint8)
        c = self._c8(_p8(a), len(a))
        return None if c < 0 else int(c)

    def count_utf16(self, units) -> int | None:
        a = np.ascontiguousarray(np.asarray(units, dtype=np.uint16))
        c = self._c16(_p16(a), len(a))
        return None if c < 0 else int(c)

    def exhaustive_short_verdicts(self) -> np.ndarray:
        out = np.zeros(256 + 65536 + 16777216, dtype=np.uint8)
        k = self._exh(_p8(out))
        assert k == len(out)
        return out


class HostGen:
    """The synthetic BASELINE workloads generated on the host from the same
    header as the device generator (oracle/gen_host.cpp -> libvt_gen.so), so
    bench.py's reference arm never loads the product library."""

    def __init__(self):
        ensure_built()
        L = _Lib(GEN_SO, "vtg_")
        self._draws = L.fn("chunk_draws", C.c_uint64, C.c_int)
        self._chunk = L.fn("host_chunk", C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p,
                           C.c_uint64, C.POINTER(C.c_uint64))
        self._gen = L.fn("generate", C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int,
                         C.POINTER(C.c_uint64))

    def chunk(self, cfg: int, seed: int, chunk: int):
        cap = int(self._draws(cfg)) * 64 + 64
        out = np.empty(cap, dtype=np.uint16 if cfg == 3 else np.uint8)
        fb = C.c_uint64()
        k = int(self._chunk(cfg, seed, chunk, out.ctypes.data, cap, C.byref(fb)))
        return out[:k], (None if fb.value == 0xFFFFFFFFFFFFFFFF else int(fb.value))

    def generate(self, cfg: int, size: int, seed: int | None = None, threads: int | None = None):
        """(array, first_injected): the first `size` elements of the stream cut
        after the last whole character, exactly what the device generator
        (paper_2109_10433_b200.generate) writes for chunk0 = 0."""
        seed = cfg if seed is None else seed
        out = np.empty(size + 16, dtype=np.uint16 if cfg == 3 else np.uint8)
        fb = C.c_uint64()
        n = int(self._gen(cfg, seed, size, out.ctypes.data, threads or os.cpu_count() or 1, C.byref(fb)))
        return out[:n], (None if fb.value == 0xFFFFFFFFFFFFFFFF else int(fb.value))

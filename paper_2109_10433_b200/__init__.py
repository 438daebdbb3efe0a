"""B200-native validated UTF-8 <-> UTF-16LE transcoding (arXiv 2109.10433 hot path).

Python face of ``libvtrans_gpu.so`` (built in-tree under ``lib/``), bound with
ctypes to the C ABI declared in ``include/vtrans_gpu.h``.  The host-pointer
functions mirror the reference's entry points (``vtrans::utf8_to_utf16``,
``vtrans::utf16_to_utf8``, ``validate_utf8``, ``validate_utf16``, the code-point
counts) with the same argument meaning, return values and error semantics:
data errors come back in-band in :class:`TranscodeResult`, device failures
raise :class:`VtransError`.  There is no CPU implementation in this package: if
the library or the GPU is missing, calls fail loudly.

The ``*_device`` functions take torch CUDA tensors (device memory and streams
are torch's plumbing) and call the device-pointer ABI directly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libvtrans_gpu.so")
# A/B tooling (tools/ab_*.sh) points VT_LIB at an experimental build of the same
# library instead of overwriting the in-tree product .so.
if os.environ.get("VT_LIB"):
    LIB_PATH = os.path.abspath(os.environ["VT_LIB"])

__all__ = [
    "TranscodeResult", "VtransError", "lib", "utf8_to_utf16", "utf16_to_utf8", "validate_utf8",
    "validate_utf16", "count_utf8", "count_utf16", "utf8_to_utf16_device", "utf16_to_utf8_device",
    "validate_utf8_device", "validate_utf16_device", "validate_utf8_batch",
    "exhaustive_short_verdicts", "sharded_utf8_to_utf16", "sharded_utf16_to_utf8",
    "sharded_device_utf8_to_utf16", "sharded_device_utf16_to_utf8", "utf8_to_utf16_batch_device",
    "utf16_to_utf8_batch_device", "utf8_to_utf16_nonvalidating", "utf8_to_utf16_nonvalidating_device",
    "split_point_utf8", "split_point_utf16", "generate", "launch_count", "device_count",
]


class VtransError(RuntimeError):
    """A device or runtime failure (never a data error)."""


class _CRes(C.Structure):
    _fields_ = [("consumed", C.c_uint64), ("written", C.c_uint64), ("error_at", C.c_int64)]


class _VStream(C.Structure):
    """vt_utf8_stream (include/vtrans_gpu.h)."""
    _fields_ = [("fed", C.c_uint64), ("error_at", C.c_int64), ("carry", C.c_uint8 * 4),
                ("carry_len", C.c_uint32), ("skip", C.c_uint32), ("reserved", C.c_uint32)]


@dataclass(frozen=True)
class TranscodeResult:
    """vtrans::TranscodeResult (proj/include/vtrans/codec_core.hpp:14-21)."""

    consumed: int
    written: int
    error_at: Optional[int]

    def ok(self) -> bool:
        return self.error_at is None

    @staticmethod
    def _of(c: _CRes) -> "TranscodeResult":
        return TranscodeResult(int(c.consumed), int(c.written),
                               None if c.error_at < 0 else int(c.error_at))


_lib = None
_u8p, _u16p, _vp = C.POINTER(C.c_uint8), C.POINTER(C.c_uint16), C.c_void_p


def lib():
    """Loads libvtrans_gpu.so (raises VtransError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise VtransError(f"{LIB_PATH} is missing: run `python -m paper_2109_10433_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "vt_utf8_to_utf16_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_utf16_to_utf8_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_validate_utf8_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
        "vt_validate_utf16_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
        "vt_utf8_to_utf16": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes), _vp]),
        "vt_utf16_to_utf8": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes), _vp]),
        "vt_validate_utf8": (C.c_int, [_vp, C.c_uint64, C.POINTER(_CRes), _vp]),
        "vt_validate_utf16": (C.c_int, [_vp, C.c_uint64, C.POINTER(_CRes), _vp]),
        "vt_host_utf8_to_utf16": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes)]),
        "vt_host_utf16_to_utf8": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes)]),
        "vt_host_validate_utf8": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_host_validate_utf16": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_host_count_utf8": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_host_count_utf16": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_validate_utf8_batch": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp]),
        "vt_utf8_to_utf16be_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_utf16be_to_utf8_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_validate_utf16be_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
        "vt_host_utf8_to_utf16be": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes)]),
        "vt_host_utf16be_to_utf8": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes)]),
        "vt_host_validate_utf16be": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_host_transcode_bytes": (C.c_int, [_vp, C.c_uint64, C.c_int, C.c_int, C.c_int, _vp, C.c_uint64,
                                              C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                              C.POINTER(C.c_int64)]),
        "vt_exhaustive_short_verdicts": (C.c_int, [_vp, _vp]),
        "vt_utf8_to_utf16_batch": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, C.c_int, _vp]),
        "vt_utf16_to_utf8_batch": (C.c_int, [_vp, _vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_utf8_to_utf16_nonvalidating_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp, _vp]),
        "vt_host_utf8_to_utf16_nonvalidating": (C.c_int, [_vp, C.c_uint64, _vp, C.POINTER(_CRes)]),
        "vt_sharded_utf8_to_utf16": (C.c_int, [_vp, C.c_uint64, _vp, C.c_int, C.POINTER(_CRes)]),
        "vt_sharded_utf16_to_utf8": (C.c_int, [_vp, C.c_uint64, _vp, C.c_int, C.POINTER(_CRes)]),
        "vt_sharded_device_utf8_to_utf16": (C.c_int, [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                                      C.POINTER(_CRes)]),
        "vt_sharded_device_utf16_to_utf8": (C.c_int, [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                                      C.POINTER(_CRes)]),
        "vt_split_point_utf8": (C.c_uint64, [_vp, C.c_uint64, C.c_uint64]),
        "vt_split_point_utf16": (C.c_uint64, [_vp, C.c_uint64, C.c_uint64]),
        "vt_gen_sizes": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp]),
        "vt_gen_write": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _vp, C.c_uint64,
                                   _vp, _vp, _vp]),
        "vt_gen_chunk_draws": (C.c_uint64, [C.c_int]),
        "vt_gen_host_chunk": (C.c_uint64, [C.c_int, C.c_uint64, C.c_uint64, _vp, C.c_uint64,
                                           C.POINTER(C.c_uint64)]),
        "vt_utf16_len_from_utf8_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
        "vt_utf8_len_from_utf16_async": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
        "vt_utf16_len_from_utf8": (C.c_int, [_vp, C.c_uint64, C.POINTER(_CRes), _vp]),
        "vt_utf8_len_from_utf16": (C.c_int, [_vp, C.c_uint64, C.POINTER(_CRes), _vp]),
        "vt_host_utf16_len_from_utf8": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_host_utf8_len_from_utf16": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int64)]),
        "vt_utf8_stream_init": (None, [C.POINTER(_VStream)]),
        "vt_utf8_stream_feed_async": (C.c_int, [_vp, _vp, C.c_uint64, _vp]),
        "vt_host_utf8_stream_feed": (C.c_int, [C.POINTER(_VStream), _vp, C.c_uint64]),
        "vt_utf8_stream_ok": (C.c_int, [C.POINTER(_VStream)]),
        "vt_utf8_stream_finish": (C.c_int, [C.POINTER(_VStream)]),
        "vt_host_utf8_class_counts": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_uint64 * 4),
                                                C.POINTER(C.c_int)]),
        "vt_status_string": (C.c_char_p, [C.c_int]),
        "vt_device_count": (C.c_int, []),
        "vt_launch_count": (C.c_uint64, []),
        "vt_host_transfer_counts": (None, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "vt_build_info": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("VT_LIB") and not hasattr(L, name):
            continue  # an older experimental build (A/B tooling) may lack newer entry points
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise VtransError(f"{what}: {lib().vt_status_string(rc).decode()} (status {rc})")


def _bytes_view(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data.view(np.uint8) if data.dtype != np.uint8 else data)
    return np.frombuffer(bytes(data), dtype=np.uint8)


def _units_view(units) -> np.ndarray:
    a = np.asarray(units)
    if a.dtype != np.uint16:
        a = a.astype(np.uint16)
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ---- host-pointer API (the drop-in boundary) --------------------------------

def utf8_to_utf16(data, validate: bool = True) -> tuple[np.ndarray, TranscodeResult]:
    """vtrans::utf8_to_utf16 vector overload (proj/include/vtrans/utf8_to_utf16.hpp:32-33).

    ``validate=False`` runs the non-validating kernel (the reference's
    validate=false path: same result on valid input, unspecified output on
    invalid input)."""
    if not validate:
        return utf8_to_utf16_nonvalidating(data)
    a = _bytes_view(data)
    out = np.empty(len(a) + 8, dtype=np.uint16)
    r = _CRes()
    _check(lib().vt_host_utf8_to_utf16(_ptr(a), len(a), out.ctypes.data, C.byref(r)), "utf8_to_utf16")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def utf16_to_utf8(units) -> tuple[np.ndarray, TranscodeResult]:
    """vtrans::utf16_to_utf8 vector overload (proj/include/vtrans/utf16_to_utf8.hpp:17)."""
    a = _units_view(units)
    out = np.empty(3 * len(a) + 16, dtype=np.uint8)
    r = _CRes()
    _check(lib().vt_host_utf16_to_utf8(_ptr(a), len(a), out.ctypes.data, C.byref(r)), "utf16_to_utf8")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def validate_utf8(data) -> bool:
    """vtrans::validate_utf8 (proj/include/vtrans/validation.hpp:27)."""
    return first_error_utf8(data) is None


def first_error_utf8(data) -> Optional[int]:
    a = _bytes_view(data)
    e = C.c_int64()
    _check(lib().vt_host_validate_utf8(_ptr(a), len(a), C.byref(e)), "validate_utf8")
    return None if e.value < 0 else int(e.value)


def validate_utf16(units) -> Optional[int]:
    """vtrans::validate_utf16 (proj/include/vtrans/validation.hpp:31)."""
    a = _units_view(units)
    e = C.c_int64()
    _check(lib().vt_host_validate_utf16(_ptr(a), len(a), C.byref(e)), "validate_utf16")
    return None if e.value < 0 else int(e.value)


def count_utf8(data) -> Optional[int]:
    """Code points, None when invalid (scalar::count_codepoints_utf8 semantics)."""
    a = _bytes_view(data)
    c = C.c_int64()
    _check(lib().vt_host_count_utf8(_ptr(a), len(a), C.byref(c)), "count_utf8")
    return None if c.value < 0 else int(c.value)


def count_utf16(units) -> Optional[int]:
    a = _units_view(units)
    c = C.c_int64()
    _check(lib().vt_host_count_utf16(_ptr(a), len(a), C.byref(c)), "count_utf16")
    return None if c.value < 0 else int(c.value)


# ---- UTF-16 big-endian and byte-order marks --------------------------------------

def utf16_len_from_utf8(data) -> Optional[int]:
    """UTF-16 units the transcoding of valid UTF-8 writes, None if invalid (GPU)."""
    a = _bytes_view(data)
    n = C.c_int64()
    _check(lib().vt_host_utf16_len_from_utf8(_ptr(a), len(a), C.byref(n)), "utf16_len_from_utf8")
    return None if n.value < 0 else int(n.value)


def utf8_len_from_utf16(units) -> Optional[int]:
    """UTF-8 bytes the transcoding of valid UTF-16 writes, None if invalid (GPU)."""
    a = _units_view(units)
    n = C.c_int64()
    _check(lib().vt_host_utf8_len_from_utf16(_ptr(a), len(a), C.byref(n)), "utf8_len_from_utf16")
    return None if n.value < 0 else int(n.value)


def utf8_to_utf16be(data):
    """UTF-8 -> UTF-16BE units (as host-order uint16 values holding the
    big-endian byte pairs, i.e. ``out.tobytes()`` is the UTF-16BE byte stream)."""
    a = _bytes_view(data)
    out = np.empty(len(a) + 8, dtype=np.uint16)
    r = _CRes()
    _check(lib().vt_host_utf8_to_utf16be(_ptr(a), len(a), out.ctypes.data, C.byref(r)), "utf8_to_utf16be")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def utf16be_to_utf8(units):
    """``units`` holds UTF-16BE byte pairs (e.g. np.frombuffer(be_bytes, np.uint16))."""
    a = _units_view(units)
    out = np.empty(3 * len(a) + 16, dtype=np.uint8)
    r = _CRes()
    _check(lib().vt_host_utf16be_to_utf8(_ptr(a), len(a), out.ctypes.data, C.byref(r)), "utf16be_to_utf8")
    res = TranscodeResult._of(r)
    return out[: res.written], res


FORMATS = {"utf8": 0, "utf16le": 1, "utf16be": 2}
BOM_POLICIES = {"keep": 0, "strip": 1, "add": 2}


def transcode_bytes(data, from_format: str, to_format: str, bom: str = "strip"):
    """harness::transcode_bytes (proj/include/vtrans/harness.hpp:60-69): returns
    (exit_code, message, output bytes) with the reference's codes and messages."""
    a = _bytes_view(data)
    f, t = FORMATS[from_format], FORMATS[to_format]
    cap = 2 * len(a) + 4 if (f == 0 and t != 0) else (3 * (len(a) // 2) + 20 if (f != 0 and t == 0) else len(a) + 4)
    out = np.empty(max(cap, 1), dtype=np.uint8)
    n_out, code, status, err = C.c_uint64(), C.c_int(), C.c_int(), C.c_int64()
    _check(lib().vt_host_transcode_bytes(_ptr(a), len(a), f, t, BOM_POLICIES[bom], out.ctypes.data, len(out),
                                         C.byref(n_out), C.byref(code), C.byref(status), C.byref(err)),
           "transcode_bytes")
    st = status.value & 0xFF
    msg = "warning: UTF-8 BOM stripped from input\n" if status.value & 0x100 else ""
    if st == 1:
        msg = "error: byte-order mark conflicts with declared endianness"
    elif st == 2:
        msg = "error: odd byte count for UTF-16 input"
    elif st == 3:
        msg = f"error: invalid UTF-8 at byte {err.value}"
    elif st == 4:
        msg = f"error: invalid UTF-16 at unit {err.value}"
    return code.value, msg, bytes(out[: n_out.value]) if code.value == 0 else b""


# ---- device-pointer API (torch tensors) --------------------------------------

def _stream_ptr(stream) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def utf8_to_utf16_device(d_in, n: int, d_out, stream=None, d_res=None, offset: int = 0):
    """Transcodes ``n`` bytes at ``d_in.data_ptr() + offset`` into ``d_out``.

    With ``d_res`` (a CUDA tensor of >= 24 bytes) the call is asynchronous and
    returns None; otherwise it waits and returns the TranscodeResult."""
    p = d_in.data_ptr() + offset
    if d_res is not None:
        _check(lib().vt_utf8_to_utf16_async(p, n, d_out.data_ptr(), d_res.data_ptr(),
                                            _stream_ptr(stream)), "utf8_to_utf16_async")
        return None
    r = _CRes()
    _check(lib().vt_utf8_to_utf16(p, n, d_out.data_ptr(), C.byref(r), _stream_ptr(stream)),
           "utf8_to_utf16")
    return TranscodeResult._of(r)


def utf16_to_utf8_device(d_in, n: int, d_out, stream=None, d_res=None, offset: int = 0):
    """``n`` UTF-16 units at ``d_in.data_ptr() + offset`` (bytes) into ``d_out``."""
    p = d_in.data_ptr() + offset
    if d_res is not None:
        _check(lib().vt_utf16_to_utf8_async(p, n, d_out.data_ptr(), d_res.data_ptr(),
                                            _stream_ptr(stream)), "utf16_to_utf8_async")
        return None
    r = _CRes()
    _check(lib().vt_utf16_to_utf8(p, n, d_out.data_ptr(), C.byref(r), _stream_ptr(stream)),
           "utf16_to_utf8")
    return TranscodeResult._of(r)


def validate_utf8_device(d_in, n: int, stream=None, d_res=None, offset: int = 0):
    p = d_in.data_ptr() + offset
    if d_res is not None:
        _check(lib().vt_validate_utf8_async(p, n, d_res.data_ptr(), _stream_ptr(stream)),
               "validate_utf8_async")
        return None
    r = _CRes()
    _check(lib().vt_validate_utf8(p, n, C.byref(r), _stream_ptr(stream)), "validate_utf8")
    return TranscodeResult._of(r)


def validate_utf16_device(d_in, n: int, stream=None, d_res=None, offset: int = 0):
    p = d_in.data_ptr() + offset
    if d_res is not None:
        _check(lib().vt_validate_utf16_async(p, n, d_res.data_ptr(), _stream_ptr(stream)),
               "validate_utf16_async")
        return None
    r = _CRes()
    _check(lib().vt_validate_utf16(p, n, C.byref(r), _stream_ptr(stream)), "validate_utf16")
    return TranscodeResult._of(r)


def utf16_len_from_utf8_device(d_in, n: int, stream=None, offset: int = 0) -> "TranscodeResult":
    """Length of the UTF-16 transcoding of ``n`` bytes on the device: ``written``
    of the valid prefix, ``error_at`` as for validation."""
    r = _CRes()
    _check(lib().vt_utf16_len_from_utf8(d_in.data_ptr() + offset, n, C.byref(r), _stream_ptr(stream)),
           "utf16_len_from_utf8")
    return TranscodeResult._of(r)


def utf8_len_from_utf16_device(d_in, n: int, stream=None, offset: int = 0) -> "TranscodeResult":
    r = _CRes()
    _check(lib().vt_utf8_len_from_utf16(d_in.data_ptr() + offset, n, C.byref(r), _stream_ptr(stream)),
           "utf8_len_from_utf16")
    return TranscodeResult._of(r)


def result_from_device(d_res) -> TranscodeResult:
    """Decodes a device result slot (an int64 CUDA tensor of 3 elements)."""
    v = d_res.cpu().numpy().astype(np.int64)
    return TranscodeResult(int(v[0]), int(v[1]), None if v[2] < 0 else int(v[2]))


def validate_utf8_batch(d_data, d_offsets, count: int, d_first_err, stream=None) -> None:
    _check(lib().vt_validate_utf8_batch(d_data.data_ptr(), d_offsets.data_ptr(), count,
                                        d_first_err.data_ptr(), _stream_ptr(stream)),
           "validate_utf8_batch")


def utf8_to_utf16_batch_device(d_data, d_offsets, count: int, d_out, d_res, validate: bool = True,
                               stream=None) -> None:
    """vt_utf8_to_utf16_batch: string i = d_data[d_offsets[i]:d_offsets[i+1]],
    its units at d_out[d_offsets[i]:], its result in d_res[i] (int64 x3)."""
    _check(lib().vt_utf8_to_utf16_batch(d_data.data_ptr(), d_offsets.data_ptr(), count, d_out.data_ptr(),
                                        d_res.data_ptr(), int(bool(validate)), _stream_ptr(stream)),
           "utf8_to_utf16_batch")


def utf16_to_utf8_batch_device(d_units, d_offsets, count: int, d_out, d_res, stream=None) -> None:
    """vt_utf16_to_utf8_batch: string i's bytes at d_out[3 * d_offsets[i]:]."""
    _check(lib().vt_utf16_to_utf8_batch(d_units.data_ptr(), d_offsets.data_ptr(), count, d_out.data_ptr(),
                                        d_res.data_ptr(), _stream_ptr(stream)), "utf16_to_utf8_batch")


def utf8_to_utf16_nonvalidating(data) -> tuple[np.ndarray, TranscodeResult]:
    """The reference's validate=false path (vt_host_utf8_to_utf16_nonvalidating):
    identical to utf8_to_utf16 on valid input; unspecified output otherwise."""
    a = _bytes_view(data)
    out = np.empty(len(a) + 8, dtype=np.uint16)
    r = _CRes()
    _check(lib().vt_host_utf8_to_utf16_nonvalidating(_ptr(a), len(a), out.ctypes.data, C.byref(r)),
           "utf8_to_utf16_nonvalidating")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def utf8_to_utf16_nonvalidating_device(d_in, n: int, d_out, stream=None, d_res=None):
    if d_res is not None:
        _check(lib().vt_utf8_to_utf16_nonvalidating_async(d_in.data_ptr(), n, d_out.data_ptr(),
                                                          d_res.data_ptr(), _stream_ptr(stream)),
               "utf8_to_utf16_nonvalidating_async")
        return None
    import torch

    res = torch.zeros(3, dtype=torch.int64, device=d_in.device)
    utf8_to_utf16_nonvalidating_device(d_in, n, d_out, stream, res)
    return result_from_device(res)


def exhaustive_short_verdicts(device="cuda"):
    import torch

    out = torch.empty(256 + 65536 + 16777216, dtype=torch.uint8, device=device)
    _check(lib().vt_exhaustive_short_verdicts(out.data_ptr(), _stream_ptr(None)),
           "exhaustive_short_verdicts")
    return out


# ---- multi-GPU sharder ------------------------------------------------------------

def sharded_utf8_to_utf16(data, ndev: int = 0):
    a = _bytes_view(data)
    out = np.empty(len(a) + 8, dtype=np.uint16)
    r = _CRes()
    _check(lib().vt_sharded_utf8_to_utf16(_ptr(a), len(a), out.ctypes.data, ndev, C.byref(r)),
           "sharded_utf8_to_utf16")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def sharded_utf16_to_utf8(units, ndev: int = 0):
    a = _units_view(units)
    out = np.empty(3 * len(a) + 16, dtype=np.uint8)
    r = _CRes()
    _check(lib().vt_sharded_utf16_to_utf8(_ptr(a), len(a), out.ctypes.data, ndev, C.byref(r)),
           "sharded_utf16_to_utf8")
    res = TranscodeResult._of(r)
    return out[: res.written], res


def _sharded_device(fn, what, shards, outs):
    """shards: [(tensor, n)] consecutive character-boundary pieces of one stream,
    each on its own device (tensor.device); outs: output tensors, one per shard."""
    k = len(shards)
    devs = (C.c_int * k)(*[t.device.index for t, _ in shards])
    ins = (C.c_void_p * k)(*[t.data_ptr() for t, _ in shards])
    ns = (C.c_uint64 * k)(*[n for _, n in shards])
    os_ = (C.c_void_p * k)(*[o.data_ptr() for o in outs])
    per = (_CRes * k)()
    offs = (C.c_uint64 * k)()
    r = _CRes()
    _check(fn(k, devs, ins, ns, os_, per, offs, C.byref(r)), what)
    return TranscodeResult._of(r), [TranscodeResult._of(x) for x in per], [int(x) for x in offs]


def sharded_device_utf8_to_utf16(shards, outs):
    """Device-resident shards (vt_sharded_device_utf8_to_utf16): returns
    (combined result, per-shard results, per-shard output offsets)."""
    return _sharded_device(lib().vt_sharded_device_utf8_to_utf16, "sharded_device_utf8_to_utf16",
                           shards, outs)


def sharded_device_utf16_to_utf8(shards, outs):
    return _sharded_device(lib().vt_sharded_device_utf16_to_utf8, "sharded_device_utf16_to_utf8",
                           shards, outs)


def split_point_utf8(data, cut: int) -> int:
    a = _bytes_view(data)
    return int(lib().vt_split_point_utf8(_ptr(a), len(a), cut))


def split_point_utf16(units, cut: int) -> int:
    a = _units_view(units)
    return int(lib().vt_split_point_utf16(_ptr(a), len(a), cut))


# ---- synthetic workloads ------------------------------------------------------------

def generate(cfg: int, size: int, seed: Optional[int] = None, chunk0: int = 0, device="cuda",
             stream=None):
    """Generates configuration ``cfg`` (1-5) of BASELINE.json directly in HBM.

    ``size`` is in bytes for UTF-8 configs and in units for cfg 3 (UTF-16).
    Returns ``(tensor, n, first_injected)``: a uint8 tensor (UTF-8) or int16
    tensor (UTF-16 units) holding exactly ``n`` elements of whole characters,
    n <= size, and for cfg 4 the position of the first injected error (else
    None)."""
    import torch

    seed = cfg if seed is None else seed
    L = lib()
    draws = int(L.vt_gen_chunk_draws(cfg))
    per_draw = {1: 1.1, 2: 3.25, 3: 1.1, 4: 2.5, 5: 1.75}[cfg]
    nchunks = int(size / (draws * per_draw) * 1.08) + 2
    s = _stream_ptr(stream)
    while True:
        sizes = torch.empty(nchunks, dtype=torch.int64, device=device)
        _check(L.vt_gen_sizes(cfg, seed, chunk0, nchunks, sizes.data_ptr(), s), "gen_sizes")
        csum = torch.cumsum(sizes, 0)
        if int(csum[-1]) >= size:
            break
        nchunks = nchunks * 2
    offsets = torch.zeros(nchunks, dtype=torch.int64, device=device)
    offsets[1:] = csum[:-1]
    dtype = torch.int16 if cfg == 3 else torch.uint8
    out = torch.empty(size + 16, dtype=dtype, device=device)
    end = torch.empty(2, dtype=torch.int64, device=device)
    _check(L.vt_gen_write(cfg, seed, chunk0, nchunks, offsets.data_ptr(), size, out.data_ptr(),
                          end.data_ptr(), s), "gen_write")
    e = end.cpu().numpy().view(np.uint64)
    n = int(e[0])
    first_bad = None if int(e[1]) == 0xFFFFFFFFFFFFFFFF else int(e[1])
    return out, n, first_bad


def generate_host_chunk(cfg: int, seed: int, chunk: int) -> tuple[np.ndarray, Optional[int]]:
    """One chunk generated on the CPU (same definition as the device generator)."""
    L = lib()
    cap = int(L.vt_gen_chunk_draws(cfg)) * 64 + 64
    out = np.empty(cap, dtype=np.uint16 if cfg == 3 else np.uint8)
    fb = C.c_uint64()
    k = int(L.vt_gen_host_chunk(cfg, seed, chunk, out.ctypes.data, cap, C.byref(fb)))
    return out[:k], (None if fb.value == 0xFFFFFFFFFFFFFFFF else int(fb.value))


class Utf8StreamValidator:
    """Streaming UTF-8 validation on the GPU: the chunked form of
    vtrans::Utf8BlockValidator (proj/include/vtrans/validation.hpp:15-24).

    Chunks of any length are fed in order (host bytes / numpy arrays, or uint8
    CUDA tensors, which stay on the device); characters may straddle chunk
    seams.  ``ok_so_far()`` and ``finish()`` have the reference's meaning;
    ``error_at`` is the first invalid byte in stream coordinates (what
    whole-buffer validation of the concatenation reports), or None."""

    def __init__(self):
        self._st = _VStream()
        lib().vt_utf8_stream_init(C.byref(self._st))
        self._dev = None

    def feed(self, chunk, n: Optional[int] = None, stream=None) -> None:
        if hasattr(chunk, "is_cuda") and chunk.is_cuda:
            import torch

            n = chunk.numel() if n is None else n
            if self._dev is None:
                self._dev = torch.empty(C.sizeof(_VStream), dtype=torch.uint8, device=chunk.device)
            host = torch.frombuffer(bytearray(bytes(self._st)), dtype=torch.uint8)
            s = stream if stream is not None else torch.cuda.current_stream()
            self._dev.copy_(host, non_blocking=False)
            _check(lib().vt_utf8_stream_feed_async(self._dev.data_ptr(), chunk.data_ptr(), n,
                                                   int(s.cuda_stream)), "utf8_stream_feed")
            s.synchronize()
            C.memmove(C.addressof(self._st), bytes(self._dev.cpu().numpy().tobytes()), C.sizeof(_VStream))
            return
        a = _bytes_view(chunk)
        if n is not None:
            a = a[:n]
        _check(lib().vt_host_utf8_stream_feed(C.byref(self._st), _ptr(a), len(a)), "utf8_stream_feed")

    def ok_so_far(self) -> bool:
        return bool(lib().vt_utf8_stream_ok(C.byref(self._st)))

    def finish(self) -> bool:
        return bool(lib().vt_utf8_stream_finish(C.byref(self._st)))

    @property
    def error_at(self) -> Optional[int]:
        return None if self._st.error_at < 0 else int(self._st.error_at)

    @property
    def fed(self) -> int:
        return int(self._st.fed)


def utf8_class_counts(data) -> Optional[tuple[int, int, int, int]]:
    """Numbers of 1/2/3/4-byte characters of valid UTF-8 (GPU), None if invalid."""
    a = _bytes_view(data)
    counts = (C.c_uint64 * 4)()
    valid = C.c_int()
    _check(lib().vt_host_utf8_class_counts(_ptr(a), len(a), C.byref(counts), C.byref(valid)),
           "utf8_class_counts")
    return tuple(int(x) for x in counts) if valid.value else None


def host_transfer_counts() -> tuple[int, int]:
    """(H2D, D2H) bytes moved so far by this thread's host-pointer transcoding calls."""
    a, b = C.c_uint64(), C.c_uint64()
    lib().vt_host_transfer_counts(C.byref(a), C.byref(b))
    return int(a.value), int(b.value)


def launch_count() -> int:
    """Kernels launched by libvtrans_gpu in this process so far."""
    return int(lib().vt_launch_count())


def device_count() -> int:
    return int(lib().vt_device_count())

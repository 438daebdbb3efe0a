"""GPU producer of the reference's benchmark records and corpus statistics.

Mirrors ``vtrans::harness`` (proj/include/vtrans/harness.hpp:14-55,
proj/src/harness.cpp:14-200): the same ``BenchRecord`` fields and JSON / CSV
formats, ``run_bench`` with four records per call and ``run_prefix_sweep``
cutting prefixes on character boundaries, ``compute_stats`` with the same
percentages.  The implementations timed are this package's GPU paths:

  ``impl == "gpu"``       device-resident buffers (C ABI device pointers),
                          CUDA-event timed, one kernel per rep;
  ``impl == "gpu-host"``  the drop-in host-pointer call (H2D + kernel + D2H),
                          wall-clock timed like the reference.

(the reference's two impls are "simd" and "scalar", both on the CPU).
Gchar/s = chars / min_ns, the spread flag is set when (mean - min) / mean
exceeds 1 % (proj/src/harness.cpp:35-49).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import (_CRes, _bytes_view, _check, _ptr, count_utf8, lib, utf8_class_counts, utf8_to_utf16)


@dataclass
class BenchRecord:
    dataset: str = ""
    direction: str = ""  # utf8_to_utf16 | utf16_to_utf8
    impl: str = ""       # gpu | gpu-host
    chars: int = 0
    bytes_in: int = 0
    bytes_out: int = 0
    reps: int = 0
    min_ns: int = 0
    mean_ns: float = 0.0
    gchars_per_sec: float = 0.0
    spread_warning: bool = False


def _fmt(x: float) -> str:
    """A double as std::ostream prints it by default (%g, 6 significant digits)."""
    return format(float(x), "g")


def to_json(r: BenchRecord) -> str:
    return (f'{{"dataset":"{r.dataset}","direction":"{r.direction}","impl":"{r.impl}",'
            f'"chars":{r.chars},"bytes_in":{r.bytes_in},"bytes_out":{r.bytes_out},"reps":{r.reps},'
            f'"min_ns":{r.min_ns},"mean_ns":{_fmt(r.mean_ns)},"gchars_per_sec":{_fmt(r.gchars_per_sec)},'
            f'"spread_warning":{"true" if r.spread_warning else "false"}}}')


def csv_header() -> str:
    return ("dataset,direction,impl,chars,bytes_in,bytes_out,reps,min_ns,mean_ns,gchars_per_sec,"
            "spread_warning")


def to_csv(r: BenchRecord) -> str:
    return (f"{r.dataset},{r.direction},{r.impl},{r.chars},{r.bytes_in},{r.bytes_out},{r.reps},"
            f"{r.min_ns},{_fmt(r.mean_ns)},{_fmt(r.gchars_per_sec)},{'true' if r.spread_warning else 'false'}")


def make_record(dataset, direction, impl, chars, bytes_in, bytes_out, reps, min_ns, mean_ns) -> BenchRecord:
    """proj/src/harness.cpp:35-49."""
    r = BenchRecord(dataset, direction, impl, int(chars), int(bytes_in), int(bytes_out), int(reps),
                    int(min_ns), float(mean_ns))
    r.gchars_per_sec = chars / min_ns if min_ns > 0 else 0.0
    r.spread_warning = mean_ns > 0 and (mean_ns - min_ns) / mean_ns > 0.01
    return r


def _time_host(reps: int, fn) -> tuple[int, float]:
    if reps == 0:
        return 0, 0.0
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        ts.append(time.perf_counter_ns() - t0)
    return min(ts), sum(ts) / reps


def _time_device(reps: int, fn) -> tuple[int, float]:
    import torch

    if reps == 0:
        return 0, 0.0
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = [max(1, int(round(a.elapsed_time(b) * 1e6))) for a, b in ev]
    return min(ts), sum(ts) / reps


def _bench_pair(dataset, utf8: np.ndarray, chars: int, reps: int, records: list) -> None:
    import torch

    L = lib()
    u16, res = utf8_to_utf16(utf8)
    n8, n16 = len(utf8), len(u16)
    b8, b16 = n8, 2 * n16
    dev = torch.device("cuda")
    d8 = torch.from_numpy(utf8.copy()).to(dev) if n8 else torch.empty(1, dtype=torch.uint8, device=dev)
    d16 = torch.from_numpy(u16.view(np.int16).copy()).to(dev) if n16 else torch.empty(1, dtype=torch.int16, device=dev)
    o16 = torch.empty(n8 + 8, dtype=torch.int16, device=dev)
    o8 = torch.empty(3 * n16 + 16, dtype=torch.uint8, device=dev)
    d_res = torch.zeros(3, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    h16 = np.empty(n8 + 8, dtype=np.uint16)
    h8 = np.empty(3 * n16 + 16, dtype=np.uint8)
    r = _CRes()

    def dev8():
        _check(L.vt_utf8_to_utf16_async(d8.data_ptr(), n8, o16.data_ptr(), d_res.data_ptr(), s), "bench")

    def host8():
        _check(L.vt_host_utf8_to_utf16(_ptr(utf8), n8, _ptr(h16), C.byref(r)), "bench")

    def dev16():
        _check(L.vt_utf16_to_utf8_async(d16.data_ptr(), n16, o8.data_ptr(), d_res.data_ptr(), s), "bench")

    def host16():
        _check(L.vt_host_utf16_to_utf8(_ptr(u16), n16, _ptr(h8), C.byref(r)), "bench")

    for direction, impl, bi, bo, fn, timer in [
            ("utf8_to_utf16", "gpu", b8, b16, dev8, _time_device),
            ("utf8_to_utf16", "gpu-host", b8, b16, host8, _time_host),
            ("utf16_to_utf8", "gpu", b16, b8, dev16, _time_device),
            ("utf16_to_utf8", "gpu-host", b16, b8, host16, _time_host)]:
        mn, mean = timer(reps, fn)
        records.append(make_record(dataset, direction, impl, chars, bi, bo, reps, mn, mean))


def run_bench(dataset: str, utf8, reps: int) -> list[BenchRecord]:
    """Both directions, both GPU impls, over valid UTF-8 content
    (proj/src/harness.cpp:101-126); allocation outside the timed region."""
    a = _bytes_view(utf8)
    chars = count_utf8(a) or 0
    records: list[BenchRecord] = []
    _bench_pair(dataset, a, chars, reps, records)
    return records


def run_prefix_sweep(dataset: str, utf8, budget_seconds: float = 0.2) -> list[BenchRecord]:
    """Speed versus length (proj/src/harness.cpp:128-170): prefixes of 16, 32,
    64, ... bytes and the whole input, each backed up to a character boundary
    and re-transcoded (host-pointer drop-in, UTF-8 -> UTF-16) until the time
    budget is spent."""
    a = _bytes_view(utf8)
    L = lib()
    out16 = np.empty(len(a) + 8, dtype=np.uint16)
    budget_ns = int(budget_seconds * 1e9)
    lens = []
    ln = 16
    while ln < len(a):
        lens.append(ln)
        ln *= 2
    if len(a):
        lens.append(len(a))
    records = []
    r = _CRes()
    for ln in lens:
        cut = ln
        while 0 < cut < len(a) and (a[cut] & 0xC0) == 0x80:
            cut -= 1
        prefix = a[:cut]
        chars = count_utf8(prefix) or 0
        mn, total, reps = None, 0, 0
        while total < budget_ns:
            t0 = time.perf_counter_ns()
            _check(L.vt_host_utf8_to_utf16(_ptr(prefix), cut, _ptr(out16), C.byref(r)), "sweep")
            dt = time.perf_counter_ns() - t0
            mn = dt if mn is None else min(mn, dt)
            total += dt
            reps += 1
        records.append(make_record(f"{dataset}:{cut}", "utf8_to_utf16", "gpu-host", chars, cut, 0,
                                   reps, mn, total / reps))
    return records


@dataclass
class CorpusStats:
    avg_bytes_per_char_utf8: float = 0.0
    avg_bytes_per_char_utf16: float = 0.0
    pct_1byte: float = 0.0
    pct_2byte: float = 0.0
    pct_3byte: float = 0.0
    pct_4byte: float = 0.0
    chars: int = 0


def compute_stats(utf8) -> Optional[CorpusStats]:
    """Per-character length histogram over valid UTF-8 (GPU class counts);
    None when invalid (proj/include/vtrans/harness.hpp:47-55)."""
    a = _bytes_view(utf8)
    c = utf8_class_counts(a)
    if c is None:
        return None
    chars = sum(c)
    s = CorpusStats(chars=chars)
    if chars:
        s.pct_1byte, s.pct_2byte, s.pct_3byte, s.pct_4byte = (100.0 * k / chars for k in c)
        s.avg_bytes_per_char_utf8 = len(a) / chars
        s.avg_bytes_per_char_utf16 = (2.0 * (chars - c[3]) + 4.0 * c[3]) / chars
    return s

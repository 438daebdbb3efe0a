"""Benchmark of the validated UTF-8 <-> UTF-16LE hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Default workload (BASELINE.json configs[1], "cfg2"): 1 GiB of valid UTF-8,
CJK-heavy (75% U+4E00-9FFF, 20% ASCII events with runs, 5% U+0080-07FF),
seeded and generated directly in HBM (synthetic stand-in for the paper's
corpora).  A step is one validating UTF-8 -> UTF-16LE transcode of the whole
input through the device-pointer C ABI (vt_utf8_to_utf16_async): one kernel
launch.  The 1 GiB input is larger than the 126 MB L2, so no flush is needed
between steps.  Other configs can be measured with --config (1, 3, 4, 5; 3 is
UTF-16LE -> UTF-8, 5 the 4 GiB round trip UTF-8 -> UTF-16 -> UTF-8).

Metric: input GB/s (aggregate over GPUs) with Gchar/s and the HBM roofline
fraction of the kernel beside it.  Multi-GPU (torchrun, one process per GPU):
weak scaling, each rank transcodes its own slice of the stream (disjoint chunk
ranges); no data-path collective, timing is the max over ranks.

``--impl reference`` times the reference's own CPU implementation (the
unmodified library compiled out of tree into oracle/_ref, SIMD path, on
character-boundary shards over all host threads) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# cfg: (description, input elements (bytes; units for cfg 3), direction)
CONFIGS = {
    1: ("cfg1: UTF-8->UTF-16LE validating, 16 MiB, 90% U+0020-007E / 10% U+0080-07FF", 16 << 20, "u8"),
    2: ("cfg2: UTF-8->UTF-16LE validating, 1 GiB, 75% U+4E00-9FFF / 20% ASCII (runs) / 5% U+0080-07FF",
        1 << 30, "u8"),
    3: ("cfg3: UTF-16LE->UTF-8, 1 GiB of UTF-16 (2^29 units), 60/15/15/10% 1/2/3/4-byte classes", 1 << 29,
        "u16"),
    4: ("cfg4: UTF-8->UTF-16LE validating, 1 GiB, 25/25/25/25% + ~1 error per 64 MiB", 1 << 30, "u8"),
    5: ("cfg5: round trip UTF-8->UTF-16LE->UTF-8, 4 GiB per GPU, cfg-3 mix", 4 << 30, "rt"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU works."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        busy = [r for r in self.rows if r[2].isdigit() and int(r[2]) > 0] or self.rows
        sm = [int(r[0]) for r in busy if r[0].isdigit()]
        mx = [int(r[1]) for r in self.rows if r[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(busy)}


def _char_boundary(host, m, kind):
    """Largest whole-character prefix length <= m."""
    if kind == "u16":
        if m < len(host) and 0xDC00 <= int(host[m]) <= 0xDFFF:
            m -= 1
        return m
    while 0 < m < len(host) and (host[m] & 0xC0) == 0x80:
        m -= 1
    return m


def cpu_reference_runner(kind):
    """The reference CPU path (oracle/_ref, SIMD, sharded) or, if that build is
    missing, the oracle port.  Returns (run(host, threads) -> result, kind)."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference

    if Reference.available():
        impl, ck = Reference(), "reference"
    else:
        impl, ck = Oracle(), "port"
    bufs = {}

    def run(host, threads):
        if kind == "u16":
            out = bufs.get(len(host))
            if out is None and ck == "reference":
                out = bufs[len(host)] = np.empty(3 * len(host) + 16, dtype=np.uint8)
            if ck == "reference":
                return impl.utf16_to_utf8(host, threads=threads, out=out)[1]
            return impl.utf16_to_utf8(host, threads=threads)[1]
        out = bufs.get(len(host))
        if out is None and ck == "reference":
            out = bufs[len(host)] = np.empty(len(host) + 8, dtype=np.uint16)
        if ck == "reference":
            return impl.utf8_to_utf16(host, threads=threads, out=out)[1]
        return impl.utf8_to_utf16(host, threads=threads)[1]

    return run, ck


def host_input(cfg, size):
    """The workload generated on the host by the test-side build of the same
    generator header (oracle/lib/libvt_gen.so): the reference arm never loads
    the product library."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import HostGen

    return HostGen().generate(cfg, size)[0]


def cpu_info():
    """nproc, CPU model and machine (an aarch64 host would run the
    reference's emulated vector backend, proj/include/vtrans/vec128.hpp:7-10)."""
    import platform

    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model, "machine": platform.machine()}


# bounded CPU sample per step for the round trip (4 GiB x 2 legs is minutes of CPU work)
RT_CPU_SAMPLE = 512 << 20


def cpu_reference_sample(cfg, host):
    """The reference CPU path for config `cfg` on `host` (the config's whole
    input; cfg5: a bounded prefix for the two-leg round trip).  Returns
    (run(sample, threads) -> result, sample, kind, description, check(result))."""
    import numpy as np

    kind = CONFIGS[cfg][2]
    if kind != "rt":
        run, ck = cpu_reference_runner(kind)
        return run, host, ck, f"whole cfg{cfg} input ({host.nbytes} bytes) per step", lambda r: None
    m = _char_boundary(host, RT_CPU_SAMPLE, "u8")
    sample = np.ascontiguousarray(host[:m])
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle, Reference

    ck = "reference" if Reference.available() else "port"
    impl = Reference() if ck == "reference" else Oracle()
    out16 = np.empty(len(sample) + 8, dtype=np.uint16)
    out8 = np.empty(3 * len(sample) + 16, dtype=np.uint8)

    def run(h, t):
        if ck == "reference":
            _, r1 = impl.utf8_to_utf16(h, threads=t, out=out16)
            o8, r2 = impl.utf16_to_utf8(out16[: r1.written], threads=t, out=out8)
        else:
            o16, r1 = impl.utf8_to_utf16(h, threads=t)
            o8, r2 = impl.utf16_to_utf8(o16, threads=t)
            out8[: len(o8)] = o8
        return r2

    def check(r):
        assert r.error_at is None and r.written == sample.nbytes
        assert np.array_equal(out8[: sample.nbytes], sample), "CPU round trip not byte-equal"
    desc = (f"round trip 8->16->8 on the first {sample.nbytes} bytes of the cfg5 stream per step "
            f"(bounded CPU sample), byte-equal checked")
    return run, sample, ck, desc, check


def run_reference_arm(args, rank):
    """--impl reference: the reference's own CPU implementation on this box
    (oracle/_ref: the unmodified library compiled out of tree; SIMD path on
    character-boundary shards over all host threads), on the same workload,
    config, metric and unit as the GPU arm.  Rank 0 only."""
    if rank != 0:
        return None
    desc, size, kind = CONFIGS[args.config]
    host = host_input(args.config, size)
    in_bytes = host.nbytes
    threads = os.cpu_count() or 1
    run, sample, ck, sample_desc, check = cpu_reference_sample(args.config, host)
    for _ in range(args.warmup):
        r = run(sample, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = run(sample, threads)
        times.append(time.perf_counter() - t0)
    check(r)
    t = sum(times) / len(times)
    gbs = sample.nbytes / t / 1e9
    line = {
        "metric": METRICS[kind], "value": round(gbs, 4), "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16" if kind == "u16" else "u8", "data": DATA,
        "config": bench_config(args.config, in_bytes),
        "parallelism": f"cpu x{threads} threads (character-boundary shards)",
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": ck,
                         "sample": sample_desc + f", reference SIMD path on {threads} character-boundary shards",
                         **cpu_info()},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"consumed": r.consumed, "written": r.written, "error_at": r.error_at},
    }
    return line


METRICS = {"u8": "input GB/s (validated UTF-8 -> UTF-16LE)", "u16": "input GB/s (UTF-16LE -> UTF-8)",
           "rt": "input GB/s (UTF-8 -> UTF-16LE -> UTF-8 round trip)"}
DATA = "synthetic (seeded splitmix64 chunk generator, BASELINE cfg shape; corpora absent)"


def bench_config(cfg, in_bytes):
    """The workload-defining config dict, identical in both arms."""
    return {"workload": CONFIGS[cfg][0], "input_bytes_per_gpu": int(in_bytes)}


def timed_steps_flushed(step, steps, stream, flush, torch):
    """Device time (ms) of `steps` calls, each bracketed by its own events on the
    launching stream, with an L2 flush (a write of a buffer larger than L2)
    between the calls and outside the events."""
    evs = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs)


def combine_over_ranks(dist, device, res, n, in_bytes):
    """The sharder's host combine across ranks (sharding.combine):
    each rank holds one character-boundary shard of the job's stream; three
    integers per rank are gathered (not data), the first failing shard decides
    error_at and written, and the input bytes add up.  Works over NCCL
    (device "cuda") or gloo (device "cpu", tests/test_bench_dist.py)."""
    import numpy as np
    import torch

    from paper_2109_10433_b200 import TranscodeResult, sharding

    world = dist.get_world_size()
    mine = torch.tensor([res.consumed, res.written, -1 if res.error_at is None else res.error_at, n,
                         in_bytes], dtype=torch.int64, device=device)
    allr = [torch.zeros(5, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allr, mine)
    rows = [[int(v) for v in x.cpu().tolist()] for x in allr]
    starts = np.concatenate([[0], np.cumsum([r[3] for r in rows])]).tolist()
    rs = [TranscodeResult(r[0], r[1], None if r[2] < 0 else r[2]) for r in rows]
    gres, _ = sharding.combine(starts, rs, starts[-1])
    return gres, sum(r[4] for r in rows)


def round_trip_weak(vt, torch, dist, rank, world, steps, peak):
    """BASELINE cfg5 beside the headline line, at the same N: every rank holds
    its own 4 GiB character-boundary shard of the cfg5 stream (disjoint chunk
    ranges), converts UTF-8 -> UTF-16LE -> UTF-8 on its GPU and checks the result
    equals its input byte for byte; per-rank results combine on the host
    (combine_over_ranks).  Weak scaling: the shard size is fixed per GPU.
    Device time with CUDA events, max over ranks."""
    size = CONFIGS[5][1]
    d_in, n, _ = vt.generate(5, size, chunk0=rank * 1_000_000)
    d16 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
    r16 = vt.utf8_to_utf16_device(d_in, n, d16)
    d8 = torch.empty(3 * r16.written + 16, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    ra = torch.zeros(3, dtype=torch.int64, device="cuda")
    rb = torch.zeros(3, dtype=torch.int64, device="cuda")

    def step():
        vt.utf8_to_utf16_device(d_in, n, d16, stream=stream, d_res=ra)
        vt.utf16_to_utf8_device(d16, r16.written, d8, stream=stream, d_res=rb)
    for _ in range(3):
        step()
    k = max(3, min(steps, 10))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    r1, r2 = vt.result_from_device(ra), vt.result_from_device(rb)
    equal = bool(r1.error_at is None and r2.error_at is None and r2.written == n
                 and torch.equal(d8[:n], d_in[:n]))
    ok = torch.tensor([1 if equal else 0], device="cuda")
    gres, total_in = r1, n
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        gres, total_in = combine_over_ranks(dist, "cuda", r1, n, n)
    out = {"workload": CONFIGS[5][0], "input_bytes_per_gpu": n, "utf16_units_per_gpu": r16.written,
           "ms_per_step": round(ms, 4), "steps": k,
           "value": round(total_in / (ms / 1e3) / 1e9, 2), "unit": "GB/s (aggregate UTF-8 input)",
           "per_gpu_gbs": round(n / (ms / 1e3) / 1e9, 2),
           "roofline_frac": round((2 * n + 4 * r16.written) / (ms / 1e3) / 1e9 / peak, 4),
           "byte_equal_all_ranks": bool(ok.item()),
           "combined_first_leg": {"consumed": gres.consumed, "written": gres.written,
                                  "error_at": gres.error_at}}
    del d_in, d16, d8
    torch.cuda.empty_cache()
    return out


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) without a launcher: one process per GPU under
    torch.distributed.run on 127.0.0.1, as the driver launches it.  Fails
    loudly when fewer than N GPUs are visible (the GPU arm only: the reference
    arm runs on rank 0's host cores and the other ranks exit at once)."""
    import socket

    if args.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible", file=sys.stderr)
            return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-rt", action="store_true", help="skip the cfg5 round-trip line beside cfg2")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        line = run_reference_arm(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch

    import paper_2109_10433_b200 as vt

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    desc, size, kind = CONFIGS[args.config]
    gen_cfg = args.config
    # each rank its own slice of the stream: disjoint chunk ranges
    d_in, n, first_bad = vt.generate(gen_cfg, size, chunk0=rank * 1_000_000)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    d_res = torch.zeros(3, dtype=torch.int64, device="cuda")
    d_res2 = torch.zeros(3, dtype=torch.int64, device="cuda")
    if kind == "u16":
        d_out = torch.empty(3 * n + 16, dtype=torch.uint8, device="cuda")
        in_bytes = 2 * n

        def step():
            vt.utf16_to_utf8_device(d_in, n, d_out, stream=stream, d_res=d_res)
        kernel = "vt::utf16_transcode_kernel"
    elif kind == "u8":
        d_out = torch.empty(n + 8, dtype=torch.int16, device="cuda")
        in_bytes = n

        def step():
            vt.utf8_to_utf16_device(d_in, n, d_out, stream=stream, d_res=d_res)
        kernel = "vt::utf8_transcode_kernel"
    else:  # round trip: the UTF-16 length is known from one warm-up pass
        d16 = torch.empty(n + 8, dtype=torch.int16, device="cuda")
        r16 = vt.utf8_to_utf16_device(d_in, n, d16)
        n16 = r16.written
        d_out = torch.empty(3 * n16 + 16, dtype=torch.uint8, device="cuda")
        in_bytes = n

        def step():
            vt.utf8_to_utf16_device(d_in, n, d16, stream=stream, d_res=d_res)
            vt.utf16_to_utf8_device(d16, n16, d_out, stream=stream, d_res=d_res2)
        kernel = "vt::utf8_transcode_kernel + vt::utf16_transcode_kernel"

    # inputs that fit the 126 MB L2 (cfg1), or of which a call reads only the
    # prefix up to its first error (cfg4, ~16 MB): L2 flushed between timed
    # steps by writing a buffer larger than L2, outside the per-step events
    flush = (torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
             if in_bytes < (256 << 20) or args.config == 4 else None)
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        t_end = time.time() + 0.6  # keep the GPU busy long enough for nvidia-smi to see it
        while time.time() < t_end:
            step()
            torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = vt.launch_count()
        if flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        else:
            ms = timed_steps_flushed(step, args.steps, stream, flush, torch)
        launches = vt.launch_count() - launches0
        if dist:
            dist.barrier()
    res = vt.result_from_device(d_res)
    if kind == "rt":
        res2 = vt.result_from_device(d_res2)
        assert res2.error_at is None and res2.written == n and torch.equal(d_out[:n], d_in[:n]), \
            "round trip did not reproduce the input"
    ms_max = ms
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        gres, total_in = combine_over_ranks(dist, "cuda", res, n, in_bytes)
    else:
        gres = res
        total_in = in_bytes
    per_step_ms = ms_max / args.steps
    if kind == "u16":
        chars = vt.validate_utf16_device(d_in, n).written
        # a call that stops at an error only has to read up to it
        alg_bytes = 2 * (n if res.error_at is None else res.error_at) + res.written
    elif kind == "u8":
        chars = vt.validate_utf8_device(d_in, n).written
        alg_bytes = (n if res.error_at is None else res.error_at) + 2 * res.written
    else:
        chars = vt.validate_utf8_device(d_in, n).written
        alg_bytes = 2 * n + 4 * res.written  # 8->16 (n + 2 u16) + 16->8 (2 u16 + n)
    if dist:
        c = torch.tensor([chars], device="cuda")
        dist.all_reduce(c)
        chars = int(c.item())
    value = total_in / (per_step_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (ms / args.steps / 1e3) / 1e9
    line = {
        "metric": METRICS[kind],
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(per_step_ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16" if kind == "u16" else "u8",
        "data": DATA + ", generated in HBM",
        "config": bench_config(args.config, in_bytes),
        "output_elems_per_gpu": res.written,
        "chars_total": chars,
        "l2": ("input > 126 MB L2: no flush between steps" if flush is None
               else "L2 flushed (512 MiB write) between timed steps, each step timed "
                    "by its own events (the bytes a call reads fit L2)"),
        "parallelism": f"{world} character-boundary shards, one per GPU (no collective)" if world > 1
        else "single GPU",
        "gchars_per_s": round(chars / (per_step_ms / 1e3) / 1e9, 2),
        "result": {"consumed": gres.consumed, "written": gres.written, "error_at": gres.error_at},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "kernel": kernel,
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if kind in ("u8", "u16"):
        # validation-only throughput on the same input (read-only,
        # algorithmic bytes = the input), device-timed like the main number
        vfn = vt.validate_utf16_device if kind == "u16" else vt.validate_utf8_device
        vres = torch.zeros(3, dtype=torch.int64, device="cuda")
        for _ in range(3):
            vfn(d_in, n, stream=stream, d_res=vres)
        if flush is None:
            v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            v0.record(stream)
            for _ in range(args.steps):
                vfn(d_in, n, stream=stream, d_res=vres)
            v1.record(stream)
            torch.cuda.synchronize()
            vms = v0.elapsed_time(v1) / args.steps
        else:
            vms = timed_steps_flushed(lambda: vfn(d_in, n, stream=stream, d_res=vres), args.steps,
                                      stream, flush, torch) / args.steps
        vbytes = in_bytes if res.error_at is None else (2 if kind == "u16" else 1) * res.error_at
        line["validate"] = {"kernel": "vt::utf16_validate_rows_kernel" if kind == "u16"
                            else "vt::utf8_validate_rows_kernel",
                            "ms_per_step": round(vms, 4), "input_gbs": round(in_bytes / vms / 1e6, 1),
                            "roofline_frac": round(vbytes / vms / 1e6 / peak, 4)}
    tr = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr):
        with open(tr) as f:
            t = json.load(f).get(f"cfg{args.config}")
        if t:
            line["roofline"]["traffic"] = t["dram_bytes_per_launch"]
            line["roofline"]["traffic_source"] = t["source"]

    if not args.no_e2e and kind != "rt":
        # end to end through the drop-in (host-pointer) C ABI: pinned host input,
        # H2D + kernel + D2H of result and output inside the timed region; every
        # rank on its own slice, the slowest rank's time for the whole job
        import ctypes

        L = vt.lib()
        r = vt._CRes()
        if kind == "u8":
            h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            h_in.copy_(d_in[:n])
            h_out = torch.empty(n + 8, dtype=torch.int16, pin_memory=True)
            fn, elem_out = L.vt_host_utf8_to_utf16, 2
        else:
            h_in = torch.empty(n, dtype=torch.int16, pin_memory=True)
            h_in.copy_(d_in[:n])
            h_out = torch.empty(3 * n + 16, dtype=torch.uint8, pin_memory=True)
            fn, elem_out = L.vt_host_utf16_to_utf8, 1

        def e2e_step():
            rc = fn(h_in.data_ptr(), n, h_out.data_ptr(), ctypes.byref(r))
            assert rc == 0, rc
        for _ in range(2):
            e2e_step()
        k = max(3, min(args.steps, 10))
        if dist:
            dist.barrier()
        x0 = vt.host_transfer_counts()
        t0 = time.perf_counter()
        for _ in range(k):
            e2e_step()
        dt = (time.perf_counter() - t0) / k
        x1 = vt.host_transfer_counts()
        assert r.written == res.written and r.error_at == (-1 if res.error_at is None else res.error_at)
        # bytes actually moved per step (a call stops early behind an error)
        h2d, d2h = (x1[0] - x0[0]) // k, (x1[1] - x0[1]) // k
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
            b = torch.tensor([h2d, d2h], dtype=torch.int64, device="cuda")
            dist.all_reduce(b)
            h2d, d2h = int(b[0].item()), int(b[1].item())
        # the same call on pageable buffers (a reference-style caller passing a
        # std::vector): the library stages through its own pinned buffers
        p_in = h_in.numpy().copy()
        p_out = np.empty(h_out.numel() * h_out.element_size(), dtype=np.uint8)
        fn(p_in.ctypes.data, n, p_out.ctypes.data, ctypes.byref(r))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k):
            rc = fn(p_in.ctypes.data, n, p_out.ctypes.data, ctypes.byref(r))
            assert rc == 0, rc
        dtp = (time.perf_counter() - t0) / k
        if dist:
            t = torch.tensor([dtp], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dtp = float(t.item())
        if rank == 0:
            line["e2e"] = {"value": round(total_in / dt / 1e9, 3), "unit": "GB/s",
                           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                           "api": f"{fn.__name__} (drop-in boundary), pinned host buffers"
                                  + (f", {world} ranks, max over ranks" if world > 1 else ""),
                           "ms_per_step": round(dt * 1e3, 3),
                           "pageable": {"value": round(total_in / dtp / 1e9, 3), "unit": "GB/s",
                                        "ms_per_step": round(dtp * 1e3, 3),
                                        "api": f"{fn.__name__}, pageable (numpy) host buffers"}}

    if args.config == 2 and not args.no_rt:
        line["round_trip_cfg5"] = round_trip_weak(vt, torch, dist, rank, world, args.steps, peak)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host = d_in[:n].cpu().numpy()
        if kind == "u16":
            host = host.view(np.uint16)
        threads = os.cpu_count() or 1
        run, sample, ck, sample_desc, check = cpu_reference_sample(args.config, host)
        best, cres = None, None
        for _ in range(3):
            t0 = time.perf_counter()
            cres = run(sample, threads)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        check(cres)
        if kind != "rt":
            assert cres.written == res.written and cres.error_at == res.error_at, "CPU baseline disagrees"
        single = ""
        if kind != "rt":
            # the reference's own design point: one thread, on a 64 MiB prefix
            m = _char_boundary(sample, (64 << 20) // sample.itemsize, kind)
            t0 = time.perf_counter()
            run(sample[:m], 1)
            single = round(m * sample.itemsize / (time.perf_counter() - t0) / 1e9, 3)
        line["cpu_baseline"] = {
            "value": round(sample.nbytes / best / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": ck,
            "sample": f"{sample_desc}; reference SIMD path (oracle/_ref, -O3 SSE4.1) on {threads} "
                      f"character-boundary shards, best of 3"
                      + (f"; 1 thread on a 64 MiB prefix: {single} GB/s" if single else ""),
            **({"single_thread_gbs": single} if single else {}),
            **cpu_info(),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

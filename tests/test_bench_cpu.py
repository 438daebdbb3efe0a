"""bench.py's host logic on CPU: the reference arm's isolation from the product
library, the `--gpus N` launcher, the cross-rank combine over gloo (world size
2), and the config dict both arms print."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_generator_matches_product_generator():
    """oracle/lib/libvt_gen.so (the reference arm's input) and the product
    library's host generator produce the same chunks, and the whole-stream
    generator cuts exactly where the concatenated chunks would."""
    import paper_2109_10433_b200 as vt
    from oracle_lib import HostGen

    g = HostGen()
    for cfg in (1, 2, 3, 4, 5):
        for c in (0, 1, 77):
            a, fa = g.chunk(cfg, cfg, c)
            b, fb = vt.generate_host_chunk(cfg, cfg, c)
            assert np.array_equal(a, b) and fa == fb, (cfg, c)
    for cfg, size in ((2, 1 << 20), (3, 300_001), (4, 1 << 22)):
        whole, _ = g.generate(cfg, size, threads=3)
        parts, total, c = [], 0, 0
        while total < size:
            x = g.chunk(cfg, cfg, c)[0]
            parts.append(x)
            total += len(x)
            c += 1
        cat = np.concatenate(parts)
        assert len(whole) <= size and np.array_equal(whole, cat[: len(whole)])
        nxt = cat[len(whole)]  # the cut is at a character start, and the next one does not fit
        if cfg == 3:
            assert not (0xDC00 <= int(nxt) <= 0xDFFF)
        else:
            assert (int(nxt) & 0xC0) != 0x80


def test_reference_arm_never_maps_the_product_library():
    code = (
        "import sys, json; sys.path.insert(0, %r); sys.argv=['bench.py'];\n"
        "import bench, argparse\n"
        "a = argparse.Namespace(config=1, steps=1, warmup=0, gpus=1)\n"
        "line = bench.run_reference_arm(a, 0)\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'line': line, 'product': 'libvtrans_gpu.so' in maps,\n"
        "                  'gen': 'libvt_gen.so' in maps}))\n" % ROOT)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert not out["product"], "the reference arm loaded libvtrans_gpu.so"
    assert out["gen"]
    line = out["line"]
    assert line["impl"] == "reference" and line["result"]["error_at"] is None
    import bench

    assert line["config"] == bench.bench_config(1, line["config"]["input_bytes_per_gpu"])
    assert set(line["config"]) == {"workload", "input_bytes_per_gpu"}
    for k in ("nproc", "cpu_model", "machine"):
        assert k in line["cpu_baseline"]


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` without a launcher starts two ranks under
    torch.distributed.run; for the reference arm rank 0 alone prints."""
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"


def test_gpus_flag_fails_loudly_without_gpus():
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert p.returncode != 0 and "GPU(s) visible" in p.stderr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _combine_worker(rank, world, port, per_rank, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        import bench
        from paper_2109_10433_b200 import TranscodeResult

        outs = []
        for case in per_rank:
            consumed, written, err, n, nbytes = case[rank]
            g, total = bench.combine_over_ranks(dist, "cpu", TranscodeResult(consumed, written, err), n, nbytes)
            outs.append(((g.consumed, g.written, g.error_at), total))
        q.put((rank, outs))
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_combine_over_ranks_gloo():
    """The cross-rank combine bench.py runs over NCCL, here over gloo with two
    ranks: shard sizes add up, the first failing shard decides error_at."""
    cases = [
        [(100, 90, None, 100, 100), (50, 40, None, 50, 50)],   # both valid
        [(100, 90, None, 100, 100), (7, 5, 7, 50, 50)],        # error in shard 1
        [(30, 20, 30, 100, 100), (7, 5, 7, 50, 50)],           # errors in both: shard 0 wins
        [(0, 0, None, 0, 0), (9, 9, None, 9, 18)],             # empty shard
    ]
    want = [((150, 130, None), 150), ((107, 95, 107), 150), ((30, 20, 30), 150), ((9, 9, None), 18)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_combine_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(got[r], str), got[r]
        assert got[r] == want, (r, got[r])

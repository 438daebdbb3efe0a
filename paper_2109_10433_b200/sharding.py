"""Character-boundary sharding across ranks (one process per GPU).

The transcoding path partitions: shards split at character boundaries are
independent, so N GPUs need no data-path
collective.  A rank transcodes its shard on its own GPU; the only exchange is
three integers per rank to combine the results, the same combine the in-process
sharder does in C++ (runtime.cu `sharded`):
  * output offsets = exclusive scan of the per-shard `written`;
  * the first shard (in order) with an error decides the global result:
    error_at = shard start + local error_at, written = sum of earlier shards'
    written + local written, consumed = error_at.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from . import TranscodeResult, split_point_utf16, split_point_utf8


def shard_bounds(data, parts: int, utf16: bool = False) -> list[int]:
    """Shard starts (plus the end) for ``parts`` shards of ``data``."""
    n = len(data)
    split = split_point_utf16 if utf16 else split_point_utf8
    st = [0]
    for k in range(1, parts):
        st.append(max(st[-1], split(data, n // parts * k)))
    st.append(n)
    return st


def combine(starts: Sequence[int], results: Sequence[TranscodeResult], n: int) -> tuple[TranscodeResult, list[int]]:
    """Combines per-shard results; returns the global result and the output
    offset of every shard (shards after the first failing one hold no part of
    the defined output; their offsets point past it)."""
    offsets, acc = [], 0
    for r in results:
        offsets.append(acc)
        acc += r.written
    for k, r in enumerate(results):
        if r.error_at is not None:
            e = starts[k] + r.error_at
            return TranscodeResult(e, offsets[k] + r.written, e), offsets
    return TranscodeResult(n, acc, None), offsets


def distributed_transcode(data, rank: int, world: int, shard_fn: Callable, utf16: bool = False,
                          group=None) -> tuple[np.ndarray, TranscodeResult, int]:
    """Runs ``shard_fn(shard) -> (out, TranscodeResult)`` on this rank's shard
    and combines the results across ranks with one all_gather of 3 integers.

    Returns (this rank's output, the global result, this rank's output offset).
    ``shard_fn`` is the GPU path in production and may be any implementation
    of the same contract in tests."""
    import torch
    import torch.distributed as dist

    st = shard_bounds(data, world, utf16)
    out, r = shard_fn(data[st[rank]:st[rank + 1]])
    mine = torch.tensor([r.consumed, r.written, -1 if r.error_at is None else r.error_at],
                        dtype=torch.int64)
    allr = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, mine, group=group)
    res = [TranscodeResult(int(t[0]), int(t[1]), None if int(t[2]) < 0 else int(t[2])) for t in allr]
    g, offsets = combine(st, res, len(data))
    return out, g, offsets[rank]

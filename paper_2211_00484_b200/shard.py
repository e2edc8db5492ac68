"""Stream sharding across GPUs (one process per GPU).

Streams are independent — the reference's batching-transparency property
(search_test.cpp:169-187, fsa_search_test.cpp:364-393) — so a batch splits by
streams with no exchange during decoding.  The only collective is the final
result gather (``gather_results``), which moves ragged int32 tokens and fp64
scores to rank 0 (<= B*(4T+8) bytes).
"""
from __future__ import annotations

import numpy as np


def shard_ranges(frame_splits, world: int, balance: str = "frames"):
    """Contiguous stream ranges [(b0, b1)] per rank.

    balance="frames" cuts where the cumulative frame count crosses r/world of
    the total, so ranks get similar work for ragged T; "streams" cuts evenly
    by stream count."""
    fs = np.asarray(frame_splits, dtype=np.int64)
    B = len(fs) - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    if balance == "streams" or fs[-1] == 0:
        cuts = [B * r // world for r in range(world + 1)]
    else:
        total = fs[-1]
        cuts = [0]
        for r in range(1, world):
            cuts.append(int(np.searchsorted(fs, total * r / world, side="left")))
        cuts.append(B)
        for r in range(1, world + 1):  # monotone
            cuts[r] = max(cuts[r], cuts[r - 1])
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def local_batch(enc, frame_splits, rank: int, world: int, balance: str = "frames"):
    """This rank's (enc rows, rebased frame_splits, (b0, b1))."""
    fs = np.asarray(frame_splits, dtype=np.int32)
    b0, b1 = shard_ranges(fs, world, balance)[rank]
    r0, r1 = int(fs[b0]), int(fs[b1])
    return enc[r0:r1], (fs[b0 : b1 + 1] - fs[b0]).astype(np.int32), (b0, b1)


def gather_results(tokens, scores, group=None, dst: int = 0):
    """Gathers per-rank ragged token lists and scores on rank `dst` in rank
    order (== global stream order for contiguous shards).  Returns
    (tokens, scores) on dst and (None, None) elsewhere."""
    import torch.distributed as dist

    obj = (tokens, None if scores is None else np.asarray(scores).tolist())
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return tokens, scores
    out = [None] * dist.get_world_size(group) if dist.get_rank(group) == dst else None
    dist.gather_object(obj, out, dst=dst, group=group)
    if out is None:
        return None, None
    toks, scs = [], []
    for t, s in out:
        toks.extend(t)
        if s is not None:
            scs.extend(s)
    return toks, (np.asarray(scs) if scores is not None else None)

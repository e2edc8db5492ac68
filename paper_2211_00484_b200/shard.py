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


def plan_streams(world: int, rank: int, batch: int, scaling: str = "weak"):
    """Global stream range [g0, g1) decoded by `rank`.

    weak:   every rank decodes `batch` streams of its own (global streams
            rank*batch .. rank*batch + batch - 1); the whole job is
            world*batch streams.
    strong: the job is `batch` streams in total, cut into contiguous
            near-equal shards (the reference CLI's parallel_for over
            utterances, tools/rnnt_main.cpp:131-158, split across GPUs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if scaling == "weak":
        return rank * batch, (rank + 1) * batch
    if scaling == "strong":
        return batch * rank // world, batch * (rank + 1) // world
    raise ValueError(f"unknown scaling mode {scaling!r}")


def gather_flat(out_splits, tokens, scores, device=None, group=None, dst: int = 0):
    """Final result gather of the flat C-ABI result form: each rank holds
    (out_splits[b+1], tokens[n], scores[b]) of its contiguous shard; rank
    `dst` receives the concatenation in rank order (== global stream order)
    as numpy arrays, other ranks get (None, None, None).

    Tensor collectives only (all_gather of the sizes, then of padded int32 /
    fp64 buffers), so it runs over NCCL (device tensors, NVLink) as well as
    gloo (CPU tensors).  This is the only collective of the decode path."""
    import torch
    import torch.distributed as dist

    osp = np.asarray(out_splits, np.int64)
    tok = np.asarray(tokens, np.int32)[: int(osp[-1])]
    sc = np.asarray(scores, np.float64)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return osp.astype(np.int32), tok, sc
    world = dist.get_world_size(group)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    sizes = torch.tensor([len(sc), len(tok)], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [tuple(int(v) for v in s.cpu()) for s in all_sizes]
    mb = max(1, max(s[0] for s in all_sizes))
    mt = max(1, max(s[1] for s in all_sizes))
    # one int32 buffer per rank: [lengths (mb) | tokens (mt)], one fp64 buffer of scores
    ibuf = torch.zeros(mb + mt, dtype=torch.int32, device=dev)
    ibuf[: len(sc)] = torch.from_numpy(np.diff(osp).astype(np.int32))
    ibuf[mb : mb + len(tok)] = torch.from_numpy(tok)
    fbuf = torch.zeros(mb, dtype=torch.float64, device=dev)
    fbuf[: len(sc)] = torch.from_numpy(sc)
    ig = [torch.empty_like(ibuf) for _ in range(world)]
    fg = [torch.empty_like(fbuf) for _ in range(world)]
    dist.all_gather(ig, ibuf, group=group)
    dist.all_gather(fg, fbuf, group=group)
    if dist.get_rank(group) != dst:
        return None, None, None
    lens, toks, scs = [], [], []
    for (nb, nt), ib, fb in zip(all_sizes, ig, fg):
        ib, fb = ib.cpu().numpy(), fb.cpu().numpy()
        lens.append(ib[:nb])
        toks.append(ib[mb : mb + nt])
        scs.append(fb[:nb])
    lens = np.concatenate(lens)
    osp_all = np.zeros(len(lens) + 1, np.int32)
    osp_all[1:] = np.cumsum(lens)
    return osp_all, np.concatenate(toks).astype(np.int32), np.concatenate(scs)

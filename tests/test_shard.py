"""Multi-GPU host logic on CPU: world_size-2 gloo processes shard a batch by
streams, decode their shard independently, and gather on rank 0; the result
must equal the single-process decode (shard transparency).  The per-rank
decoder here is the oracle (no GPU in CI); on GPUs it is librnntg (bench.py,
tests/test_gpu_parity.py::test_shard_transparency_gpu)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2211_00484_b200.shard import local_batch, shard_ranges


def test_shard_ranges_cover_and_balance():
    fs = np.concatenate([[0], np.cumsum([10, 0, 30, 5, 5, 50, 1])]).astype(np.int32)
    for world in (1, 2, 3, 4, 8):
        for bal in ("frames", "streams"):
            r = shard_ranges(fs, world, bal)
            assert r[0][0] == 0 and r[-1][1] == len(fs) - 1
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    r = shard_ranges(np.arange(0, 1001, 100), 2)
    assert r == [(0, 5), (5, 10)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ret):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2211_00484_b200.shard import gather_results
    from tests import helpers as H

    m = H.ref().model(6, 6, 16, 64, 16, 9, -0.5)
    Ts = [3, 0, 7, 12, 1, 9, 4]
    _, enc, fs = H.frames(m, Ts, seed0=33)
    le, lfs, _ = local_batch(enc, fs, rank, world)
    toks, sc = H.orc().beam(m.w, le, lfs, beam=3, threads=1)
    gt, gs = gather_results(toks, sc)
    if rank == 0:
        want, wsc = H.orc().beam(m.w, enc, fs, beam=3, threads=1)
        ret.put((gt == want, bool(np.array_equal(gs, wsc))))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_transparency():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == (True, True)


def test_plan_streams_weak_and_strong():
    from paper_2211_00484_b200.shard import plan_streams

    assert [plan_streams(4, r, 1024, "weak") for r in range(4)] == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    strong = [plan_streams(8, r, 1024, "strong") for r in range(8)]
    assert strong[0] == (0, 128) and strong[-1] == (896, 1024)
    assert all(a[1] == b[0] for a, b in zip(strong, strong[1:]))
    odd = [plan_streams(3, r, 10, "strong") for r in range(3)]
    assert odd == [(0, 3), (3, 6), (6, 10)]
    with pytest.raises(ValueError):
        plan_streams(2, 2, 8)


def _gather_worker(rank, world, port, ret):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2211_00484_b200.shard import gather_flat, plan_streams

    # bench.py's rank logic: strong split of 7 streams, ragged token lists
    g0, g1 = plan_streams(world, rank, 7, "strong")
    lists = [[g * 10 + j for j in range(g % 3)] for g in range(g0, g1)]
    osp = np.zeros(len(lists) + 1, np.int32)
    osp[1:] = np.cumsum([len(x) for x in lists])
    tok = np.array([t for x in lists for t in x] + [-1, -1], np.int32)  # capacity beyond osp[-1]
    sc = np.arange(g0, g1, dtype=np.float64) * 0.5
    a, b, c = gather_flat(osp, tok, sc)
    if rank == 0:
        ret.put((a.tolist(), b.tolist(), c.tolist()))
    else:
        ret.put(None if a is None else "leak")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_flat():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = [r for r in res if r is not None]
    assert len(res) == 1 and res[0] != "leak"
    osp, tok, sc = res[0]
    lists = [[g * 10 + j for j in range(g % 3)] for g in range(7)]
    assert osp == [0] + np.cumsum([len(x) for x in lists]).tolist()
    assert tok == [t for x in lists for t in x]
    assert sc == [g * 0.5 for g in range(7)]


def test_bench_relaunches_under_torchrun():
    import bench

    cmd = bench.torchrun_cmd(["--gpus", "4", "--steps", "2"], 4)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]

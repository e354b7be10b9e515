"""Multi-process (world size 2, gloo, CPU) tests of the frame sharder and
the tile gather.  The per-rank compute is replaced by a deterministic CPU
stand-in (tiles derived from the block coordinates), so the test exercises
exactly the host-side distribution logic the GPU bench uses."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2204_14193_b200 import sharding


def _fake_tiles(frames_offset, local_blocks):
    b = local_blocks.astype(np.int64)
    g = (b[:, 0] + frames_offset) * 7919 + b[:, 1] * 31 + b[:, 2]
    return (g[:, None, None] + np.arange(16 * 16).reshape(1, 16, 16)) % 251


def _worker(rank, world, port, blocks, n_frames, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = sharding.shard_blocks(blocks, n_frames, rank, world)
    tiles = _fake_tiles(sh.f0, sh.blocks).astype(np.uint8)
    out = sharding.gather_tiles(sh, tiles, len(blocks))
    # the one-box path: every rank stores its slice into one shared host buffer
    path = os.path.join("/dev/shm", f"fse_test_tiles_{port}")
    if rank == 0:
        buf = sharding.HostTileBuffer(path, (len(blocks), 16, 16), torch.uint8, create=True, pin=False)
    dist.barrier()
    if rank != 0:
        buf = sharding.HostTileBuffer(path, (len(blocks), 16, 16), torch.uint8, create=False, pin=False)
    lo, hi = sharding.contiguous_range(sh)
    buf.slice(lo, hi).copy_(torch.from_numpy(tiles))
    dist.barrier()
    if rank == 0:
        q.put((out, buf.numpy().copy()))
        buf.close(unlink=True)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_gather_matches_single_process(world):
    import paper_2204_14193_b200 as fse

    n_frames = 5
    blocks = fse.frames_pattern(n_frames, 270, 480, 16, 0.05, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, blocks, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    out, shared = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = _fake_tiles(0, blocks).astype(np.uint8)
    assert np.array_equal(out, ref)
    assert np.array_equal(shared, ref)


def test_frame_ranges_balanced_and_cover():
    for n in [1, 7, 64, 256]:
        for w in [1, 2, 3, 4, 8]:
            rs = [sharding.frame_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_shard_blocks_rebases_frames():
    blocks = np.array([[0, 0, 0], [1, 16, 16], [2, 32, 0], [3, 0, 48]], np.int32)
    s = sharding.shard_blocks(blocks, 4, 1, 2)
    assert (s.f0, s.f1) == (2, 4)
    assert np.array_equal(s.index, [2, 3])
    assert np.array_equal(s.blocks, [[0, 32, 0], [1, 0, 48]])
    with pytest.raises(ValueError):
        sharding.assemble([np.zeros((1, 2, 2))], [np.array([0])], 2)


def test_weak_scaling_shards_keep_the_n1_share():
    """bench.py's default (weak scaling): rank r of N conceals frames
    256 r .. 256 r + 255 of an N x 256-frame job, and every frame's loss
    pattern is the same at every N (per-frame seeds)."""
    import importlib.util
    import os as _os

    import paper_2204_14193_b200 as fse

    spec = importlib.util.spec_from_file_location(
        "bench", _os.path.join(_os.path.dirname(_os.path.dirname(__file__)), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    per, H, W = 3, 270, 480
    base = fse.frames_pattern(per, H, W, 16, 0.05, seed=5)
    for world in [1, 2, 4, 8]:
        n = bench.job_frames(per, world, "weak")
        assert n == per * world and bench.job_frames(per, world, "strong") == per
        job = fse.frames_pattern(n, H, W, 16, 0.05, seed=5)
        assert np.array_equal(job[job[:, 0] < per], base)
        for r in range(world):
            sh = sharding.shard_blocks(job, n, r, world)
            assert (sh.f0, sh.n_frames) == (per * r, per)
            assert np.array_equal(sh.blocks[:, 0], job[job[:, 0] // per == r][:, 0] - per * r)

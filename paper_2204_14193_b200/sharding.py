"""Multi-GPU frame sharding.

Lost blocks are independent given the immutable input frames (SPEC.md:220,
358), so the path shards with no collective: rank r of W conceals the
contiguous frame range [r*F/W, (r+1)*F/W) on its own GPU (one process per
GPU, torch.distributed only for rendezvous / timing / the optional tile
gather).  The only data crossing ranks is the reconstructed tiles, and only
if the caller wants them on one rank (`gather_tiles`).

Host-side logic only; the per-rank compute is harness.Concealer /
harness.ConcealPlan on that rank's device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    f0: int  # first frame (inclusive)
    f1: int  # last frame (exclusive)
    index: np.ndarray  # positions of this shard's blocks in the global block list
    blocks: np.ndarray  # (n, 3) (frame - f0, top, left), the shard's local block list

    @property
    def n_frames(self) -> int:
        return self.f1 - self.f0


def frame_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced frame range of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return n_frames * rank // world, n_frames * (rank + 1) // world


def shard_blocks(blocks: np.ndarray, n_frames: int, rank: int, world: int) -> Shard:
    """Split a global (frame, top, left) block list by frame range."""
    b = np.asarray(blocks, np.int32).reshape(-1, 3)
    f0, f1 = frame_range(n_frames, rank, world)
    idx = np.nonzero((b[:, 0] >= f0) & (b[:, 0] < f1))[0]
    local = b[idx].copy()
    local[:, 0] -= f0
    return Shard(rank, world, f0, f1, idx, local)


def assemble(shards_tiles, shards_index, n_blocks: int) -> np.ndarray:
    """Place per-shard tiles back into global block order."""
    first = next(t for t in shards_tiles if t is not None)
    out = np.empty((n_blocks,) + tuple(first.shape[1:]), first.dtype)
    seen = np.zeros(n_blocks, bool)
    for t, i in zip(shards_tiles, shards_index):
        out[i] = t
        seen[i] = True
    if not seen.all():
        raise ValueError("shards do not cover every block")
    return out


def gather_tiles(shard: Shard, tiles: np.ndarray, n_blocks: int, dst: int = 0):
    """Gather every rank's host tiles to rank `dst` over the default process
    group (gloo or nccl via object collectives; tiles are small: 256 B per
    16x16 u8 block).  Returns the global tile array on `dst`, None elsewhere."""
    import torch.distributed as dist

    payload = (shard.index, np.ascontiguousarray(tiles))
    if dist.get_world_size() == 1:
        return assemble([payload[1]], [payload[0]], n_blocks)
    objs = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    dist.gather_object(payload, objs, dst=dst)
    if dist.get_rank() != dst:
        return None
    return assemble([o[1] for o in objs], [o[0] for o in objs], n_blocks)

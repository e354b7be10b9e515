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


def contiguous_range(shard: Shard) -> tuple[int, int]:
    """[lo, hi) of the shard's blocks in the global list (frame-ordered
    block lists give every rank one contiguous range)."""
    idx = shard.index
    if len(idx) == 0:
        return 0, 0
    lo, hi = int(idx[0]), int(idx[-1]) + 1
    if hi - lo != len(idx):
        raise ValueError("shard blocks are not contiguous in the global list (sort blocks by frame)")
    return lo, hi


class HostTileBuffer:
    """One host tile buffer for every GPU of the box.

    A file in /dev/shm holds the (n_blocks, B, B) tiles in global block
    order.  Each rank maps it (torch.from_file, shared) and page-locks its
    mapping (cudaHostRegister), so a rank's kernel stores its shard's tiles
    straight into its slice of the one buffer (ConcealPlan.run with host
    tiles): the gather costs no collective and no extra copy.  Rank 0 creates
    the file; `open` on the other ranks after a barrier.  `pin=False` (CPU
    tests) skips the page-locking."""

    def __init__(self, path: str, shape, dtype, create: bool, pin: bool = True):
        import torch

        self.path = path
        self.shape = tuple(int(x) for x in shape)
        numel = int(np.prod(self.shape))
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        if create:
            with open(path, "wb") as fh:
                fh.truncate(max(nbytes, 1))
        self.tensor = torch.from_file(path, shared=True, size=max(numel, 1), dtype=dtype)[:numel].view(self.shape)
        self.registered = False
        if pin and nbytes:
            rc = torch.cuda.cudart().cudaHostRegister(self.tensor.data_ptr(), nbytes, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister of the shared tile buffer failed ({rc})")
            self.registered = True
        self.nbytes = nbytes

    def slice(self, lo: int, hi: int):
        return self.tensor[lo:hi]

    def numpy(self) -> np.ndarray:
        return self.tensor.numpy()

    def close(self, unlink: bool = False):
        import os

        import torch

        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.tensor.data_ptr())
            self.registered = False
        self.tensor = None
        if unlink:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass


def gather_tiles(shard: Shard, tiles, n_blocks: int, dst: int = 0):
    """Gather every rank's tiles to rank `dst` over the default process group
    as tensors (gloo: CPU tensors, nccl: device tensors), each rank's block
    indices first, then its tiles padded to the largest shard.  Returns the
    global (n_blocks, ...) numpy array on `dst`, None elsewhere.  On one box
    `HostTileBuffer` needs no collective at all; this is the general path."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(tiles))
    world = dist.get_world_size()
    if world == 1:
        return assemble([t.numpy()], [shard.index], n_blocks)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x.item()) for x in sizes]
    cap = max(sizes)
    row = tuple(t.shape[1:])
    pad_t = torch.zeros((cap,) + row, dtype=t.dtype, device=dev)
    pad_t[: t.shape[0]] = t.to(dev)
    pad_i = torch.full((cap,), -1, dtype=torch.int64, device=dev)
    pad_i[: t.shape[0]] = torch.as_tensor(shard.index, dtype=torch.int64).to(dev)
    me = dist.get_rank()
    gt = [torch.empty_like(pad_t) for _ in range(world)] if me == dst else None
    gi = [torch.empty_like(pad_i) for _ in range(world)] if me == dst else None
    dist.gather(pad_i, gi, dst=dst)
    dist.gather(pad_t, gt, dst=dst)
    if me != dst:
        return None
    return assemble([x[:k].cpu().numpy() for x, k in zip(gt, sizes)],
                    [x[:k].cpu().numpy() for x, k in zip(gi, sizes)], n_blocks)

"""Image-level concealment: the north-star entry point on the GPU.

The reference specifies, but does not ship, an image harness
(SPEC.md:296-365): for every lost B x B block cut the F x F window centred
on it, build the mask with the support ring clipped to the image
(`build_mask(..., valid_rect=image)`), run cFSE, write Re{g} of the loss
pixels back (clamped to [0, 255] for 8-bit images).  Here that loop is one
persistent CUDA launch over all blocks of all frames:

  ConcealPlan  -- host planner (native, libfse_b200: geometry classes of the
                  clipped support, rounds of same-class blocks) + per-class
                  weight spectra on the device; `run(frames)` launches the
                  fused kernel on device-resident frames and writes tiles.
  Concealer    -- host frames in, host tiles out: frames stream to the GPU in
                  chunks on a copy stream while the previous chunk computes,
                  tiles come back on the same pipeline (pinned buffers).
  conceal      -- SPEC.md:332-340 convenience form on one image + pattern.
  psnr, loss_pattern -- SPEC.md:341-356 evaluation helpers.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError

_DTYPES = {np.dtype(np.uint8): _lib.FSE_U8, np.dtype(np.float32): _lib.FSE_F32,
           np.dtype(np.float64): _lib.FSE_F64}
_TILE = {"u8": _lib.FSE_U8, "f32": _lib.FSE_F32, "f64": _lib.FSE_F64}


def _torch_dtype_code(t) -> int:
    import torch

    return {torch.uint8: _lib.FSE_U8, torch.float32: _lib.FSE_F32,
            torch.float64: _lib.FSE_F64}[t.dtype]


@dataclass(frozen=True)
class Geometry:
    """Block size B, support ring width `border`, FFT window F (centred)."""

    B: int = 16
    border: int = 16
    F: int = 64


class ConcealPlan:
    """A reusable schedule for one loss pattern over frames of size H x W.

    blocks: int array (n, 3) = (frame, top, left) or (n, 2) = (top, left)
    for a single frame.  precision "fp32" uses the fused register-resident
    kernel (F in {32, 64, 128}); "fp64" the reference-exact per-window path.
    algorithm "rfse" runs the conjugate-pair variant (rfse.py; fused in fp32,
    per window in fp64); basis_target as in FseConfig.
    """

    def __init__(self, blocks, H: int, W: int, geometry: Geometry = Geometry(), *,
                 rho_hat: float = 0.8, gamma: float = 0.2, iterations: int = 100,
                 precision: str = "fp32", algorithm: str = "cfse", basis_target=None,
                 stream=None):
        torch = _lib.require_cuda()
        b = np.asarray(blocks, dtype=np.int32)
        if b.ndim != 2 or b.shape[1] not in (2, 3):
            raise ConfigError(f"blocks must be (n, 2) or (n, 3), got {b.shape}")
        if b.shape[1] == 2:
            b = np.concatenate([np.zeros((b.shape[0], 1), np.int32), b], axis=1)
        self.blocks = np.ascontiguousarray(b)
        self.H, self.W, self.geometry = int(H), int(W), geometry
        if algorithm not in ("cfse", "rfse"):
            raise ConfigError(f"algorithm must be 'cfse' or 'rfse', got {algorithm!r}")
        self.algorithm = algorithm
        self.iterations = int(basis_target) if basis_target is not None else int(iterations)
        self.precision = precision
        self.device = torch.cuda.current_device()
        prec = _lib.FSE_PREC_F32 if precision == "fp32" else _lib.FSE_PREC_F64
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().fse_plan_create_ex(
            ctypes.byref(h), self.blocks.ctypes.data_as(ctypes.c_void_p), self.blocks.shape[0],
            self.H, self.W, geometry.B, geometry.border, geometry.F, float(rho_hat), float(gamma),
            int(iterations), prec, _lib.FSE_ALG_RFSE if algorithm == "rfse" else _lib.FSE_ALG_CFSE,
            -1 if basis_target is None else int(basis_target), _lib.stream_ptr(stream)))
        self._h = h
        info = _lib.PlanInfo()
        _lib.check(_lib.lib().fse_plan_get_info(self._h, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _lib.PlanInfo._fields_}

    @property
    def n_blocks(self) -> int:
        return self.blocks.shape[0]

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().fse_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, frames, tiles=None, *, tile_dtype: str = "u8", trace: bool = False, stream=None):
        """Conceal every planned block of device-resident `frames`
        ((n_frames, H, W) or (H, W) CUDA tensor, u8/f32/f64, rows may be
        padded: the row pitch is taken from the tensor stride).  Returns
        the (n_blocks, B, B) tiles tensor (and a trace dict if `trace`).

        `tiles` may be a pinned (page-locked) host tensor: the kernel then
        stores each finished tile straight into host memory over the
        host link (mapped pinned memory, unified addressing), so the tiles
        are on the host when the stream reaches this point -- no separate
        device-to-host copy."""
        import torch

        if not (frames.is_cuda or frames.is_pinned()):
            raise ValueError("ConcealPlan.run needs device frames or page-locked host frames "
                             "(pageable host frames: use Concealer)")
        f3 = frames if frames.ndim == 3 else frames[None]
        if f3.shape[1] != self.H or f3.shape[2] != self.W or f3.stride(2) != 1:
            raise ValueError(f"frames {tuple(f3.shape)} do not match plan {self.H}x{self.W}")
        B = self.geometry.B
        tdt = {"u8": torch.uint8, "f32": torch.float32, "f64": torch.float64}[tile_dtype]
        if tiles is None:
            tiles = torch.empty((self.n_blocks, B, B), dtype=tdt,
                                device=f3.device if f3.is_cuda else torch.device("cuda", self.device))
        elif (tuple(tiles.shape) != (self.n_blocks, B, B) or tiles.dtype != tdt
              or not tiles.is_contiguous()):
            raise ValueError(f"tiles must be a contiguous {tdt} tensor of shape "
                             f"{(self.n_blocks, B, B)}, got {tiles.dtype} {tuple(tiles.shape)}")
        elif not (tiles.is_cuda or tiles.is_pinned()):
            raise ValueError("tiles must live on the device or in pinned host memory")
        tr = None
        if trace:
            it = self.iterations
            ft = torch.float32 if self.precision == "fp32" else torch.float64
            tr = dict(uv=torch.empty((self.n_blocks, it, 2), dtype=torch.int32, device=f3.device),
                      c=torch.empty((self.n_blocks, it, 2), dtype=ft, device=f3.device),
                      e=torch.empty((self.n_blocks, it), dtype=ft, device=f3.device))
        _lib.check(_lib.lib().fse_plan_run(
            self._h, _lib.ptr(f3), _torch_dtype_code(f3), f3.stride(1), f3.stride(0), f3.shape[0],
            _lib.ptr(tiles), _TILE[tile_dtype], _lib.ptr(tr["uv"]) if tr else None,
            _lib.ptr(tr["c"]) if tr else None, _lib.ptr(tr["e"]) if tr else None,
            _lib.stream_ptr(stream)))
        return (tiles, tr) if trace else tiles


class Concealer:
    """Host frames -> host tiles with copy/compute overlap.

    Frames are split into chunks of `chunk_frames` (default 4, or 2 for at
    most 32 frames); each chunk has its own
    plan (built once here: the geometry tables are prebuilt, as a decoder
    would keep them for a fixed loss pattern).  `run(host_frames)` copies
    chunk k+1 host->device on a copy stream while chunk k runs, and copies
    each chunk's tiles device->host as soon as they are ready.  Host input
    should be pinned (`pin()`), so the copies are true DMA.
    """

    def __init__(self, blocks, n_frames: int, H: int, W: int, geometry: Geometry = Geometry(), *,
                 rho_hat: float = 0.8, gamma: float = 0.2, iterations: int = 100,
                 precision: str = "fp32", chunk_frames=None, frame_dtype=np.uint8,
                 tile_dtype: str = "u8", algorithm: str = "cfse", basis_target=None,
                 tile_path: str = "host"):
        torch = _lib.require_cuda()
        b = np.asarray(blocks, np.int32).reshape(-1, 3)
        order = np.argsort(b[:, 0], kind="stable")
        self.order = order
        self.identity_order = bool(np.array_equal(order, np.arange(len(order))))
        b = b[order]
        self.n_frames, self.H, self.W, self.geometry = n_frames, H, W, geometry
        self.tile_dtype = tile_dtype
        self.frame_dtype = np.dtype(frame_dtype)
        if chunk_frames is None:
            # measured (config 5 frames, one B200): 4-frame chunks best at 256
            # frames per GPU; at 32 frames per GPU (8-GPU share) 2-frame chunks
            # expose less of the first copy (e2e 6.67 vs 5.98 M blocks/s with 8)
            chunk_frames = 2 if n_frames <= 32 else 4
        self.chunks = []
        # the first chunk is one frame: its copy is the only one nothing overlaps
        bounds = [0] + list(range(1 if chunk_frames > 1 and n_frames > 1 else chunk_frames,
                                  n_frames, chunk_frames)) + [n_frames]
        for f0, f1 in zip(bounds[:-1], bounds[1:]):
            lo, hi = np.searchsorted(b[:, 0], [f0, f1])
            cb = b[lo:hi].copy()
            cb[:, 0] -= f0
            plan = ConcealPlan(cb, H, W, geometry, rho_hat=rho_hat, gamma=gamma,
                               iterations=iterations, precision=precision, algorithm=algorithm,
                               basis_target=basis_target) if hi > lo else None
            self.chunks.append((f0, f1, int(lo), int(hi), plan))
        tdt = {"u8": torch.uint8, "f32": torch.float32, "f64": torch.float64}[tile_dtype]
        tt = torch.from_numpy(np.zeros((), self.frame_dtype)).dtype
        self.n_blocks = b.shape[0]
        self.nbuf = 4
        self.dev_frames = [torch.empty((chunk_frames, H, W), dtype=tt, device="cuda")
                           for _ in range(min(self.nbuf, len(self.chunks)))]
        # tiles: by default each kernel stores its tiles straight into the
        # pinned host buffer (zero-copy, see ConcealPlan.run); tile_path="copy"
        # keeps device tiles and copies each chunk's tiles back instead
        if tile_path not in ("host", "copy"):
            raise ConfigError(f"tile_path must be 'host' or 'copy', got {tile_path!r}")
        self.tile_path = tile_path
        self.dev_tiles = (torch.empty((self.n_blocks, geometry.B, geometry.B), dtype=tdt, device="cuda")
                          if tile_path == "copy" else None)
        self.host_tiles = torch.empty((self.n_blocks, geometry.B, geometry.B), dtype=tdt).pin_memory()
        self.copy_stream = torch.cuda.Stream()
        # two compute streams: chunk k+1's persistent kernel fills the SMs
        # freed by chunk k's tail instead of waiting for it
        self.compute_streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    @staticmethod
    def pin(frames: np.ndarray):
        import torch

        return torch.from_numpy(np.ascontiguousarray(frames)).pin_memory()

    def h2d_bytes(self) -> int:
        return self.n_frames * self.H * self.W * self.frame_dtype.itemsize

    def d2h_bytes(self) -> int:
        return self.host_tiles.numel() * self.host_tiles.element_size()

    def run(self, host_frames, copy: bool = False, out=None) -> np.ndarray:
        """host_frames: pinned torch tensor (n_frames, H, W).  Returns the
        tiles in the caller's block order.  When the caller's blocks are
        already in frame order (the usual case) the result is a view of the
        pinned tile buffer, valid until the next run (copy=True detaches it).

        `out`: optional pinned host tensor (n_blocks, B, B) of the tile
        dtype (e.g. one rank's slice of a host buffer shared by every GPU of
        the box) that receives the tiles instead of the internal buffer;
        needs blocks in frame order.  Returns out.numpy()."""
        import torch

        dst = self._dst(out)
        self._enqueue(host_frames, dst)
        for ks in self.compute_streams:
            ks.synchronize()
        return self._result(dst, copy)

    def capture(self, host_frames, out=None):
        """Record the whole pipeline for these buffers (pinned host frames, and
        `out` or the internal tile buffer) as one CUDA graph and return a
        callable that replays it: each call conceals the current contents of
        `host_frames` with a single graph launch instead of one host round of
        copies and launches per chunk, and returns the tiles as `run` does.
        For decoders that refill the same pinned frame buffer every batch."""
        import torch

        dst = self._dst(out)
        self.run(host_frames, out=out)  # warm-up: function attributes, tensor maps
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        side = (self.copy_stream, *self.compute_streams)
        with torch.cuda.graph(graph, stream=cap):
            for s in side:  # fork the side streams from the capture stream ...
                s.wait_stream(cap)
            self._enqueue(host_frames, dst)
            for s in side:  # ... and join them back
                cap.wait_stream(s)

        def replay(copy: bool = False) -> np.ndarray:  # holds the graph alive
            graph.replay()
            torch.cuda.current_stream().synchronize()
            return self._result(dst, copy)

        return replay

    def _dst(self, out):
        dst = self.host_tiles
        if out is not None:
            if not self.identity_order:
                raise ValueError("out= needs the block list in frame order")
            if tuple(out.shape) != tuple(dst.shape) or out.dtype != dst.dtype or not out.is_pinned():
                raise ValueError(f"out must be a pinned {dst.dtype} tensor of shape {tuple(dst.shape)}")
            dst = out
        return dst

    def _result(self, dst, copy: bool) -> np.ndarray:
        tiles = dst.numpy()
        if self.identity_order:
            return tiles.copy() if copy else tiles
        res = np.empty(tiles.shape, tiles.dtype)
        res[self.order] = tiles
        return res

    def _enqueue(self, host_frames, dst) -> None:
        """Queue every chunk's H2D copy and kernel on the copy / compute streams."""
        import torch

        cs = self.copy_stream
        nb = len(self.dev_frames)
        done = [None] * len(self.chunks)  # compute-done event per chunk (frees its buffer)
        for i, (f0, f1, lo, hi, plan) in enumerate(self.chunks):
            buf = self.dev_frames[i % nb]
            with torch.cuda.stream(cs):
                if i >= nb:
                    cs.wait_event(done[i - nb])  # the buffer's previous chunk has finished
                buf[: f1 - f0].copy_(host_frames[f0:f1], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(cs)
            ks = self.compute_streams[i % 2]
            with torch.cuda.stream(ks):
                ks.wait_event(ready)
                if plan is not None:
                    if self.dev_tiles is None:  # kernel stores tiles into pinned host memory
                        plan.run(buf[: f1 - f0], dst[lo:hi], tile_dtype=self.tile_dtype, stream=ks)
                    else:
                        plan.run(buf[: f1 - f0], self.dev_tiles[lo:hi], tile_dtype=self.tile_dtype,
                                 stream=ks)
                        dst[lo:hi].copy_(self.dev_tiles[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(ks)
                done[i] = ev


def conceal_frames(frames, blocks, geometry: Geometry = Geometry(), *, rho_hat=0.8, gamma=0.2,
                   iterations=100, precision="fp32", tile_dtype="u8", algorithm="cfse",
                   basis_target=None):
    """One-shot form: device or host frames, returns tiles (same side)."""
    import torch

    on_host = isinstance(frames, np.ndarray)
    f = torch.from_numpy(np.ascontiguousarray(frames)).cuda() if on_host else frames
    f3 = f if f.ndim == 3 else f[None]
    plan = ConcealPlan(blocks, f3.shape[1], f3.shape[2], geometry, rho_hat=rho_hat, gamma=gamma,
                       iterations=iterations, precision=precision, algorithm=algorithm,
                       basis_target=basis_target)
    tiles = plan.run(f3, tile_dtype=tile_dtype)
    return tiles.cpu().numpy() if on_host else tiles


def write_tiles(image: np.ndarray, blocks, tiles: np.ndarray, B: int) -> np.ndarray:
    """Return a copy of `image` ((H, W) or (nf, H, W)) with the tiles written
    into their loss blocks (only loss samples change)."""
    out = np.array(image, copy=True)
    o3 = out if out.ndim == 3 else out[None]
    b = np.asarray(blocks, np.int32)
    if b.shape[1] == 2:
        b = np.concatenate([np.zeros((b.shape[0], 1), np.int32), b], 1)
    for k, (f, t, l) in enumerate(b):
        o3[f, t:t + B, l:l + B] = tiles[k]
    return out


def conceal(image: np.ndarray, pattern, config, geometry: Geometry = Geometry()):
    """conceal every block of `pattern` ((n, 2) top-left
    corners) in `image` (H x W).  Returns (concealed image, tiles): for 8-bit
    images Re{g} is clamped to [0, 255] and rounded; float images get the
    unclamped model.  `config` is an FseConfig (rho_hat, gamma, loop_bound,
    precision, algorithm -- cfse or rfse; fft_dims must equal (F, F))."""
    if tuple(config.fft_dims) != (geometry.F, geometry.F):
        raise ConfigError(f"fft_dims {config.fft_dims} != window {geometry.F}")
    img = np.asarray(image)
    tdt = "u8" if img.dtype == np.uint8 else ("f64" if config.precision == "fp64" else "f32")
    rfse = config.algorithm == "rfse"
    tiles = conceal_frames(img, pattern, geometry, rho_hat=config.rho_hat, gamma=config.gamma,
                           iterations=config.iterations if rfse else config.loop_bound,
                           precision=config.precision, tile_dtype=tdt, algorithm=config.algorithm,
                           basis_target=config.basis_target if rfse else None)
    return write_tiles(img, pattern, tiles, geometry.B), tiles


def psnr(original: np.ndarray, reconstructed: np.ndarray, blocks, B: int) -> float:
    """10 log10(255^2 / MSE), MSE pooled over the loss pixels only
    (SPEC.md:341-356).  Returns +inf for a perfect reconstruction."""
    o = np.asarray(original, np.float64)
    r = np.asarray(reconstructed, np.float64)
    o3, r3 = (o, r) if o.ndim == 3 else (o[None], r[None])
    b = np.asarray(blocks, np.int32)
    if b.shape[1] == 2:
        b = np.concatenate([np.zeros((b.shape[0], 1), np.int32), b], 1)
    if b.shape[0] == 0:
        raise ConfigError("no loss samples")
    se = 0.0
    for f, t, l in b:
        d = o3[f, t:t + B, l:l + B] - r3[f, t:t + B, l:l + B]
        se += float(np.sum(d * d))
    mse = se / (b.shape[0] * B * B)
    return math.inf if mse == 0 else 10.0 * math.log10(255.0 ** 2 / mse)


def psnr_tiles(truth_tiles: np.ndarray, tiles: np.ndarray) -> float:
    d = np.asarray(truth_tiles, np.float64) - np.asarray(tiles, np.float64)
    mse = float(np.mean(d * d))
    return math.inf if mse == 0 else 10.0 * math.log10(255.0 ** 2 / mse)


def grid_pattern(H: int, W: int, block: int, stride: int, support: int, seed: int = 0) -> np.ndarray:
    """SPEC.md:318-324 `generate_pattern`: a deterministic grid of isolated
    B x B losses every `stride` pixels; the seed only shifts the grid phase
    (phase = support + seed mod (stride - block - 2 support + 1)).  512x512,
    stride 64, seed 0 -> 64 blocks at (16 + 64 i, 16 + 64 j)."""
    if stride < block + 2 * support:
        raise ConfigError(f"stride {stride} < block + 2*support = {block + 2 * support} (losses not isolated)")
    span = stride - block - 2 * support + 1
    ph = support + (int(seed) % span)
    tops = range(ph, H - block + 1, stride)
    lefts = range(ph, W - block + 1, stride)
    return np.array([(t, l) for t in tops for l in lefts], np.int32).reshape(-1, 2)


def loss_pattern(H: int, W: int, B: int, count: int, seed: int) -> np.ndarray:
    """Seeded isolated-block loss pattern (native fse_loss_pattern): random
    sequential selection on the B x B grid, no two chosen blocks 8-adjacent.
    Returns (k, 2) int32 top-left corners in row-major order."""
    out = np.empty((max(count, 0), 2), np.int32)
    k = _lib.lib().fse_loss_pattern(int(H), int(W), int(B), int(count), int(seed) & (2 ** 64 - 1),
                                    out.ctypes.data_as(ctypes.c_void_p))
    _lib.check(min(k, 0))
    return out[:k]


def loss_pattern_fraction(H: int, W: int, B: int, fraction: float, seed: int) -> np.ndarray:
    """Pattern with round(fraction * full-grid-blocks) lost blocks."""
    n = int(round(fraction * (H // B) * (W // B)))
    return loss_pattern(H, W, B, n, seed)


def frames_pattern(n_frames: int, H: int, W: int, B: int, fraction: float, seed: int) -> np.ndarray:
    """(n, 3) = (frame, top, left) for n_frames frames, one seeded pattern per frame."""
    parts = []
    for f in range(n_frames):
        p = loss_pattern_fraction(H, W, B, fraction, seed * 1000003 + f)
        parts.append(np.concatenate([np.full((p.shape[0], 1), f, np.int32), p], 1))
    return np.concatenate(parts, 0) if parts else np.zeros((0, 3), np.int32)

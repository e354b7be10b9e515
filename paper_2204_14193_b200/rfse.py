"""Real-valued (conjugate-pair) frequency-selective extrapolation on the GPU.

Mirror of the reference module `fse.rfse` (/root/reference/pkg/src/fse/
rfse.py): the paper's comparison variant.  Each iteration selects the
conjugate pair {phi_(u,v), conj(phi)} with the largest exact energy decrease
(per-bin 2x2 Gram solve with variable denominators, self-conjugate bins as a
single real atom), so the model stays real.  Computed by
`fse_extrapolate_rfse` (csrc/generic.cu `rfse_iterate`), fp64 by default with
the reference's operation order.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .cfse import _as_signal, _prec, _validate
from .errors import ConfigError
from .types import ExtrapolationResult, FseConfig, IterationRecord
from .weighting import AreaMask, build_mask

__all__ = ["extrapolate_rfse", "extrapolate_rfse_batch", "RfsePlan", "conceal_frames_rfse"]


def _bounds(config: FseConfig):
    # rfse.py:182-187
    if config.basis_target is not None:
        return config.basis_target, config.basis_target
    return config.iterations, 2 * config.iterations + 1


def extrapolate_rfse_batch(signals, labels, config: FseConfig, *, want_model=False, stream=None):
    """Batched rFSE over (n, M, N) windows; labels shared (M, N) or (n, M, N).
    Returns CUDA tensors: reconstructed, model, us, vs, cs, es, selfs (n,
    max_iters, valid up to counts), counts, tallies, status."""
    torch = _lib.require_cuda()
    s = torch.as_tensor(signals, dtype=torch.float64).cuda().contiguous()
    if s.ndim == 2:
        s = s[None]
    lab = torch.as_tensor(np.asarray(labels, np.int8) if not torch.is_tensor(labels) else labels,
                          dtype=torch.int8).cuda().contiguous()
    n, M, N = s.shape
    lstride = 0 if lab.ndim == 2 else M * N
    max_iters, stop = _bounds(config)
    dev = s.device
    k = max(max_iters, 1)
    rec = torch.empty_like(s)
    model = torch.empty((n, M, N), dtype=torch.complex128, device=dev) if want_model else None
    us = torch.empty((n, k), dtype=torch.int64, device=dev)
    vs = torch.empty_like(us)
    cs = torch.empty((n, k), dtype=torch.complex128, device=dev)
    es = torch.empty((n, k), dtype=torch.float64, device=dev)
    selfs = torch.empty((n, k), dtype=torch.int32, device=dev)
    counts = torch.empty((n,), dtype=torch.int32, device=dev)
    tallies = torch.empty((n,), dtype=torch.int32, device=dev)
    status = torch.empty((n,), dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().fse_extrapolate_rfse(
        n, M, N, _prec(config), _lib.ptr(s), _lib.ptr(lab), lstride, float(config.rho_hat),
        float(config.gamma), max_iters, stop, _lib.ptr(rec), _lib.ptr(model), _lib.ptr(us),
        _lib.ptr(vs), _lib.ptr(cs), _lib.ptr(es), _lib.ptr(selfs), _lib.ptr(counts),
        _lib.ptr(tallies), _lib.ptr(status), _lib.stream_ptr(stream)))
    st = status.cpu().numpy()
    if (st == 1).any():
        raise ConfigError("total support weight is numerically zero (empty support)")
    if (st == 2).any():
        raise ConfigError("support area is degenerate for pairwise selection "
                          "(conjugate atoms nearly parallel under the weight)")
    return dict(reconstructed=rec, model=model, us=us, vs=vs, cs=cs, es=es, selfs=selfs,
                counts=counts, tallies=tallies, status=status)


def extrapolate_rfse(signal, mask: AreaMask, config: FseConfig) -> ExtrapolationResult:
    """rfse.py:170-210: same validation as cFSE, trace with self_conjugate
    flags, basis_count = tally (2 per pair, 1 per self-conjugate atom)."""
    s = _as_signal(signal)
    _validate(s, mask, config)
    if s.ndim != 2:  # rfse.py -> cfse.py:36-40 via _prepare: the signal must be fft_dims
        raise ConfigError(f"signal shape {s.shape} does not match configured FFT dims {config.fft_dims}")
    # latency path (as cfse.extrapolate_cfse): every output in one device
    # buffer, one copy to pinned host memory
    torch = _lib.require_cuda()
    M, N = s.shape
    MN = M * N
    max_iters, stop = _bounds(config)
    k = max(max_iters, 1)
    # recon f64 | model c128 | us i64 | vs i64 | cs c128 | es f64 | selfs i32 | counts, tallies, status i32
    sizes = [8 * MN, 16 * MN, 8 * k, 8 * k, 16 * k, 8 * k, ((4 * k + 7) // 8) * 8, 8, 8, 8]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    dev = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
    sd = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(mask.labels, np.int8)).cuda()
    p = [dev.data_ptr() + int(o) for o in offs[:-1]]
    _lib.check(_lib.lib().fse_extrapolate_rfse(
        1, M, N, _prec(config), sd.data_ptr(), lab.data_ptr(), 0, float(config.rho_hat),
        float(config.gamma), max_iters, stop, *p, _lib.stream_ptr(None)))
    host = _lib.pinned_staging(int(offs[-1]))
    host.copy_(dev)  # synchronous: waits for the kernel
    raw = host.numpy()

    def part(i, dt, n):
        return np.frombuffer(raw, dtype=dt, count=n, offset=int(offs[i])).copy()

    st = int(part(9, np.int32, 1)[0])
    if st == 1:
        raise ConfigError("total support weight is numerically zero (empty support)")
    if st == 2:
        raise ConfigError("support area is degenerate for pairwise selection "
                          "(conjugate atoms nearly parallel under the weight)")
    cnt = int(part(7, np.int32, 1)[0])
    us, vs = part(2, np.int64, k)[:cnt], part(3, np.int64, k)[:cnt]
    cs, es = part(4, np.complex128, k)[:cnt], part(5, np.float64, k)[:cnt]
    sf = part(6, np.int32, k)[:cnt]
    trace = [IterationRecord(index=i, frequency=(int(us[i]), int(vs[i])), coefficient=complex(cs[i]),
                             residual_energy=float(es[i]), self_conjugate=bool(sf[i]))
             for i in range(cnt)]
    return ExtrapolationResult(reconstructed=part(0, np.float64, MN).reshape(M, N),
                               model=part(1, np.complex128, MN).reshape(M, N), trace=trace,
                               basis_count=int(part(8, np.int32, 1)[0]))



class RfsePlan:
    """Image-level rFSE: windows centred on each block (valid_rect = image),
    as harness.ConcealPlan does for cFSE.  Windows and masks are cut on the
    host (this is the comparison path, not the throughput path) and the
    extrapolation runs batched on the GPU."""

    def __init__(self, blocks, H, W, geometry, *, rho_hat=0.8, gamma=0.2, basis_target=None,
                 iterations=100, precision="fp64"):
        b = np.asarray(blocks, np.int32)
        if b.shape[1] == 2:
            b = np.concatenate([np.zeros((b.shape[0], 1), np.int32), b], 1)
        self.blocks, self.H, self.W, self.geo = b, H, W, geometry
        self.config = FseConfig(rho_hat=rho_hat, gamma=gamma, iterations=max(iterations, 1),
                                fft_dims=(geometry.F, geometry.F), algorithm="rfse",
                                basis_target=basis_target, precision=precision)
        F, B, off = geometry.F, geometry.B, (geometry.F - geometry.B) // 2
        self.labels = np.stack([build_mask((F, F), (off, off, B, B), geometry.border,
                                           (-(t - off), -(l - off), H, W)).labels
                                for _, t, l in b]) if len(b) else np.zeros((0, F, F), np.int8)

    def windows(self, frames):
        fr = frames if frames.ndim == 3 else frames[None]
        F, B = self.geo.F, self.geo.B
        off = (F - B) // 2
        out = np.zeros((len(self.blocks), F, F), np.float64)
        for k, (f, t, l) in enumerate(self.blocks):
            wt, wl = t - off, l - off
            y0, y1, x0, x1 = max(0, wt), min(self.H, wt + F), max(0, wl), min(self.W, wl + F)
            out[k, y0 - wt:y1 - wt, x0 - wl:x1 - wl] = fr[f, y0:y1, x0:x1]
        return out

    def run(self, frames):
        """frames: host numpy or CUDA tensor; returns (n, B, B) f64 tiles on the device."""
        import torch

        fr = frames.cpu().numpy() if torch.is_tensor(frames) else np.asarray(frames)
        win = self.windows(fr)
        out = extrapolate_rfse_batch(win, self.labels, self.config)
        F, B = self.geo.F, self.geo.B
        off = (F - B) // 2
        return out["reconstructed"][:, off:off + B, off:off + B]


def conceal_frames_rfse(frames, blocks, geometry, *, rho_hat=0.8, gamma=0.2, basis_target=None,
                        iterations=100, precision="fp64"):
    H, W = np.asarray(frames).shape[-2:]
    plan = RfsePlan(blocks, H, W, geometry, rho_hat=rho_hat, gamma=gamma, basis_target=basis_target,
                    iterations=iterations, precision=precision)
    return plan.run(frames).cpu().numpy()

"""Parity gates of SURVEY.md 8(c) -- TEST INFRASTRUCTURE ONLY.

Used by tests/ and by bench.py's parity sample (outside the timed region) to
check the CUDA path's tiles against the CPU oracle; never imported by the
product package.
"""
import numpy as np

from . import oracle as orc


def window_of(frame: np.ndarray, top: int, left: int, F: int, B: int, border: int):
    """SPEC.md:332-340 window + mask (valid_rect = image), via the oracle."""
    H, W = frame.shape
    off = (F - B) // 2
    wt, wl = top - off, left - off
    s = np.zeros((F, F), np.float64)
    y0, y1, x0, x1 = max(0, wt), min(H, wt + F), max(0, wl), min(W, wl + F)
    s[y0 - wt:y1 - wt, x0 - wl:x1 - wl] = frame[y0:y1, x0:x1]
    lab = orc.build_mask((F, F), (off, off, B, B), border, (-wt, -wl, H, W))
    return s, lab


def fp32_gate(frames, blocks, tiles_gpu, traces_gpu, F, B, border, rho, gamma, iters,
              px_tol=0.5, psnr_tol=0.01, truth=None, log=None):
    """The north-star fp32 gate: per block max |dpx| <= px_tol except
    certified near-ties, and pooled PSNR within psnr_tol dB.

    Every block over px_tol is certified from the fp64 oracle state at its
    first canonical divergence (oracle.divergence_certificate):
      strict   the fp64 relative |R_w|^2 gap between the fp64 pick and the
               fp32 pick is < 1e-6;
      bounded  the fp64 amplitude gap |R[top]| - |R[pick]| is at most twice
               the fp32 run's residual error measured on that block (the
               largest |R32 - R64| over its selections up to the divergence):
               the two bins are tied to within the fp32 arithmetic's own
               measured error, so any fp32 implementation may pick either.
    Anything else fails.  Returns a stats dict listing every outlier."""
    fr = frames if frames.ndim == 3 else frames[None]
    ref = orc.conceal_blocks(fr, blocks, B, border, F, rho, gamma, iters)
    g = np.asarray(tiles_gpu, np.float64)
    dev = np.abs(g - ref).reshape(len(blocks), -1).max(axis=1)
    # a non-finite tile is a failure, never an outlier to certify
    nonfinite = [(int(k), "non-finite tile") for k in np.nonzero(~np.isfinite(dev))[0]]
    assert not nonfinite, f"fp32 tiles with NaN/Inf: {nonfinite[:10]}"
    bad = np.nonzero(dev > px_tol)[0]
    outliers, failed = [], []
    for k in bad:
        f, t, l = blocks[k]
        s, lab = window_of(fr[f].astype(np.float64), t, l, F, B, border)
        o = orc.extrapolate(s, lab, rho, gamma, iters)
        tr = traces_gpu(k) if traces_gpu else None
        assert tr is not None, f"block {k} off by {dev[k]:.3f} and no trace to certify it"
        at = orc.first_divergence((o["us"], o["vs"], o["cs"]), tr, F, F)
        if at is None:
            failed.append((int(k), float(dev[k]), "identical selections"))
            continue
        cert = orc.divergence_certificate(s, lab, rho, gamma, at, tr)
        row = dict(block=int(k), dev=float(dev[k]), **cert)
        outliers.append(row)
        if not (cert["strict"] or cert["bounded"]):
            failed.append((int(k), float(dev[k]), cert))
    stats = dict(n=len(blocks), max_dev=float(dev.max()) if len(dev) else 0.0,
                 over=len(bad), strict=sum(r["strict"] for r in outliers),
                 bounded=sum((not r["strict"]) and r["bounded"] for r in outliers),
                 outliers=outliers)
    if truth is not None:
        cl = lambda x: np.clip(x, 0, 255)
        p_ref = psnr_tiles(truth, cl(ref))
        p_gpu = psnr_tiles(truth, cl(g))
        stats.update(psnr_ref=p_ref, psnr_gpu=p_gpu, psnr_delta=p_gpu - p_ref)
    if log:
        log_stats(log, stats)
    assert not failed, f"uncertified fp32 outliers: {failed}"
    if truth is not None:
        assert abs(stats["psnr_delta"]) <= psnr_tol, (stats["psnr_ref"], stats["psnr_gpu"])
    return stats


def first_rfse_divergence(trace_a, trace_b):
    """First iteration whose (u, v) differ (rFSE traces carry the canonical
    pair member already, rfse.py:113-121); None if identical."""
    ua, va = np.asarray(trace_a[0]), np.asarray(trace_a[1])
    ub, vb = np.asarray(trace_b[0]), np.asarray(trace_b[1])
    n = min(len(ua), len(ub))
    d = np.nonzero((ua[:n] != ub[:n]) | (va[:n] != vb[:n]))[0]
    if d.size:
        return int(d[0])
    return None if len(ua) == len(ub) else n


def rfse_gate(frames, blocks, tiles_gpu, traces_gpu, F, B, border, rho, gamma, iters,
              basis_target=None, px_tol=0.5, log=None):
    """fp32 rFSE gate against the fp64 rFSE oracle (oracle/cfse_oracle.c,
    restating rfse.py:37-210): per block max |dpx| <= px_tol except
    certified near-ties (oracle.rfse_divergence_certificate: strict =
    criterion gap < 1e-6 relative at the first differing selection; bounded
    = gap within twice the fp32 run's measured criterion error).  traces_gpu(k)
    -> (us, vs, cs) of the fp32 run, trimmed to its executed iterations."""
    fr = frames if frames.ndim == 3 else frames[None]
    ref = orc.conceal_blocks_rfse(fr, blocks, B, border, F, rho, gamma, iters, basis_target)
    g = np.asarray(tiles_gpu, np.float64)
    dev = np.abs(g - ref).reshape(len(blocks), -1).max(axis=1)
    nonfinite = [(int(k), "non-finite tile") for k in np.nonzero(~np.isfinite(dev))[0]]
    assert not nonfinite, f"fp32 rFSE tiles with NaN/Inf: {nonfinite[:10]}"
    outliers, failed = [], []
    for k in np.nonzero(dev > px_tol)[0]:
        f, t, l = blocks[k]
        s, lab = window_of(fr[f].astype(np.float64), t, l, F, B, border)
        o = orc.extrapolate_rfse(s, lab, rho, gamma, iters, basis_target)
        tr = traces_gpu(k)
        at = first_rfse_divergence((o["us"], o["vs"]), tr)
        if at is None or at >= len(tr[0]):
            failed.append((int(k), float(dev[k]), "no selection divergence"))
            continue
        cert = orc.rfse_divergence_certificate(s, lab, rho, gamma, at, tr)
        outliers.append(dict(block=int(k), dev=float(dev[k]), **cert))
        if not (cert["strict"] or cert["bounded"]):
            failed.append((int(k), float(dev[k]), cert))
    stats = dict(n=len(blocks), max_dev=float(dev.max()) if len(dev) else 0.0,
                 over=int((dev > px_tol).sum()), strict=sum(r["strict"] for r in outliers),
                 bounded=sum((not r["strict"]) and r["bounded"] for r in outliers), outliers=outliers)
    if log:
        log_stats(log, stats)
    assert not failed, f"uncertified fp32 rFSE outliers: {failed}"
    return stats


def psnr_tiles(truth, tiles) -> float:
    """Pooled PSNR over loss pixels: 10 log10(255^2 / MSE)."""
    d = np.asarray(truth, np.float64) - np.asarray(tiles, np.float64)
    mse = float(np.mean(d * d))
    return float("inf") if mse == 0 else 10.0 * np.log10(255.0 ** 2 / mse)


def log_stats(name, stats):
    """Append a parity record to $FSE_PARITY_LOG (JSON lines) when set."""
    import json
    import os
    path = os.environ.get("FSE_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(dict(test=name, **stats), default=float) + "\n")

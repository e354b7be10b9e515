"""Window / mask helpers shared by the parity tests (test-side only)."""
import numpy as np

from oracle import oracle as orc


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
              px_tol=0.5, psnr_tol=0.01, tie_tol=1e-4, truth=None):
    """The north-star fp32 gate: per block max |dpx| <= px_tol except
    certified near-ties, and pooled PSNR within psnr_tol dB.  A block is a
    certified near-tie when, at the first canonical divergence, the fp32
    run's selected bin has |R_w|^2 within a relative tie_tol of the fp64
    maximum (oracle.pick_deficit): both choices are greedy-optimal to
    within fp32 accumulated error (near-ties below fp32
    resolution are unavoidable for any fp32 implementation).  Returns a
    stats dict (raises AssertionError on failure)."""
    fr = frames if frames.ndim == 3 else frames[None]
    ref = orc.conceal_blocks(fr, blocks, B, border, F, rho, gamma, iters)
    g = np.asarray(tiles_gpu, np.float64)
    dev = np.abs(g - ref).reshape(len(blocks), -1).max(axis=1)
    bad = np.nonzero(dev > px_tol)[0]
    certified = []
    for k in bad:
        f, t, l = blocks[k]
        s, lab = window_of(fr[f].astype(np.float64), t, l, F, B, border)
        o = orc.extrapolate(s, lab, rho, gamma, iters)
        tr = traces_gpu(k) if traces_gpu else None
        assert tr is not None, f"block {k} off by {dev[k]:.3f} and no trace to certify it"
        at = orc.first_divergence((o["us"], o["vs"], o["cs"]), tr, F, F)
        assert at is not None, f"block {k}: identical selections yet off by {dev[k]:.3f} px"
        gap = orc.pick_deficit(s, lab, rho, gamma, at, tr)
        assert gap < tie_tol, f"block {k}: off by {dev[k]:.3f} px, divergence at {at} deficit {gap:.2e}"
        certified.append((int(k), float(dev[k]), int(at), float(gap)))
    stats = dict(n=len(blocks), max_dev=float(dev.max()) if len(dev) else 0.0,
                 over=len(bad), certified=certified)
    if truth is not None:
        from paper_2204_14193_b200.harness import psnr_tiles
        cl = lambda x: np.clip(x, 0, 255)
        p_ref = psnr_tiles(truth, cl(ref))
        p_gpu = psnr_tiles(truth, cl(g))
        stats.update(psnr_ref=p_ref, psnr_gpu=p_gpu)
        assert abs(p_ref - p_gpu) <= psnr_tol, (p_ref, p_gpu)
    return stats

"""Generate golden vectors by running the REFERENCE cFSE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference package `fse` (cfse.py / weighting.py /
types.py), runs `extrapolate_cfse` on seeded windows cut from the synthetic
1/f^2 fields of paper_2204_14193_b200.synth, and stores inputs + outputs as
compressed .npz fixtures next to this script.  Nothing here is written by
hand: every number in the fixtures comes from the reference.  The GPU box
does not have /root/reference; tests only read the .npz files.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ.get("FSE_REFERENCE_SRC", "/root/reference/pkg/src"))

from fse.cfse import _prepare, extrapolate_cfse  # noqa: E402  (reference)
from fse.rfse import extrapolate_rfse  # noqa: E402
from fse.types import FseConfig  # noqa: E402
from fse.weighting import AreaMask, build_mask  # noqa: E402

from paper_2204_14193_b200.synth import field  # noqa: E402


def window(img, top, left, F, B, border):
    """F x F window centred on the B x B block, image pixels
    inside, 0 outside; valid_rect = image in window coordinates."""
    H, W = img.shape
    off = (F - B) // 2
    wt, wl = top - off, left - off
    s = np.zeros((F, F), np.float64)
    y0, y1 = max(0, wt), min(H, wt + F)
    x0, x1 = max(0, wl), min(W, wl + F)
    s[y0 - wt:y1 - wt, x0 - wl:x1 - wl] = img[y0:y1, x0:x1]
    mask = build_mask((F, F), (off, off, B, B), border, valid_rect=(-wt, -wl, H, W))
    return s, mask


def run(s, mask, rho, gamma, iters, basis_target=None, keep_spectra=False, keep_model=False):
    M, N = s.shape
    cfg = FseConfig(rho_hat=rho, gamma=gamma, iterations=iters, fft_dims=(M, N),
                    basis_target=basis_target)
    res = extrapolate_cfse(s, mask, cfg)
    rec = dict(
        signal=s, labels=mask.labels, rho=rho, gamma=gamma,
        iterations=cfg.loop_bound,
        recon_loss=res.reconstructed[mask.loss],
        us=np.array([t.frequency[0] for t in res.trace], np.int64),
        vs=np.array([t.frequency[1] for t in res.trace], np.int64),
        cs=np.array([t.coefficient for t in res.trace], np.complex128),
        es=np.array([t.residual_energy for t in res.trace], np.float64),
    )
    _, w, W, w00, R_w, e0 = _prepare(s, mask, cfg)
    rec["w00"] = w00
    rec["e0"] = e0
    if keep_spectra:
        rec["R_w"] = R_w
        rec["W"] = W
        rec["w"] = w
    if keep_model:
        rec["model"] = res.model
    return rec


def run_rfse(s, mask, rho, gamma, iters, basis_target=None):
    M, N = s.shape
    cfg = FseConfig(rho_hat=rho, gamma=gamma, iterations=iters, fft_dims=(M, N), algorithm="rfse",
                    basis_target=basis_target)
    res = extrapolate_rfse(s, mask, cfg)
    _, w, W, w00, R_w, e0 = _prepare(s, mask, cfg)
    return dict(
        signal=s, labels=mask.labels, rho=rho, gamma=gamma, iterations=iters,
        basis_target=-1 if basis_target is None else basis_target,
        recon_loss=res.reconstructed[mask.loss], tally=res.basis_count, w00=w00, e0=e0,
        us=np.array([t.frequency[0] for t in res.trace], np.int64),
        vs=np.array([t.frequency[1] for t in res.trace], np.int64),
        cs=np.array([t.coefficient for t in res.trace], np.complex128),
        es=np.array([t.residual_energy for t in res.trace], np.float64),
        selfs=np.array([t.self_conjugate for t in res.trace], np.int32),
    )


def save(name, cases):
    out = {}
    for i, c in enumerate(cases):
        for k, v in c.items():
            out[f"{i:03d}_{k}"] = np.asarray(v)
    out["n"] = np.asarray(len(cases))
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, len(cases), "cases")


def main():
    rho, gamma = 0.8, 0.5

    # config 1: 256x256 fp64 field, one block at the centre (120,120)
    img1 = field(256, 256, seed=1)
    s, m = window(img1, 120, 120, 64, 16, 16)
    save("config1.npz", [run(s, m, rho, gamma, 100, keep_spectra=True, keep_model=True)])

    # 64x64 / 16 / 16 windows from a 512x512 field (config 2 geometry),
    # interior + clipped (corner, edges), I = 100 and 200
    img2 = field(512, 512, seed=2)
    pos = [(32 * i, 32 * j) for i, j in
           [(0, 0), (0, 5), (5, 0), (3, 3), (7, 9), (12, 4), (15, 15), (9, 14), (4, 11), (10, 10)]]
    pos += [(496, 496), (496, 128)]
    cases = []
    for k, (t, l) in enumerate(pos):
        s, m = window(img2, t, l, 64, 16, 16)
        cases.append(run(s, m, rho, gamma, 200 if k % 4 == 3 else 100, keep_spectra=(k < 2)))
    save("win64.npz", cases)

    # 32x32 / 8 / 8 (config 4a geometry)
    img4 = field(512, 512, seed=4)
    cases = []
    for (t, l) in [(0, 0), (16, 256), (240, 0), (128, 128), (304, 400), (504, 504), (64, 32), (200, 480)]:
        s, m = window(img4, t, l, 32, 8, 8)
        cases.append(run(s, m, rho, gamma, 100, keep_spectra=(t == 128)))
    save("win32.npz", cases)

    # 128x128 / 32 / 16 (config 4b geometry)
    img5 = field(512, 512, seed=5)
    cases = []
    for (t, l) in [(0, 0), (192, 256), (448, 64)]:
        s, m = window(img5, t, l, 128, 32, 16)
        cases.append(run(s, m, rho, gamma, 100))
    save("win128.npz", cases)

    # small random instances (SPEC.md:266-294 / acceptance criterion 1 sizes)
    rng = np.random.default_rng(7)
    cases = []
    for k in range(12):
        M = [8, 12, 16][k % 3]
        N = [8, 12, 16, 10][k % 4]
        s = rng.uniform(0, 255, (M, N))
        loss = rng.uniform(size=(M, N)) < 0.25
        pad = (rng.uniform(size=(M, N)) < 0.1) & ~loss
        mask = AreaMask.from_loss(loss, pad)
        cases.append(run(s, mask, 0.8, 0.2, 40, keep_spectra=(k < 3)))
    # basis_target = 0 (types.py:55-60): transforms only, loss -> 0
    s, m = window(img2, 160, 160, 64, 16, 16)
    cases.append(run(s, m, rho, gamma, 100, basis_target=0))
    # basis_target overriding iterations
    cases.append(run(s, m, rho, gamma, 100, basis_target=7))
    # constant signal: c = gamma * const
    s = np.full((64, 64), 200.0)
    cases.append(run(s, build_mask((64, 64), (24, 24, 16, 16), 16), 0.8, 0.2, 1))
    cases.append(run(s, build_mask((64, 64), (24, 24, 16, 16), 16), 0.8, 0.2, 200))
    save("small.npz", cases)

    # rFSE (rfse.py:170-210), the paper's comparison variant
    rng = np.random.default_rng(17)
    cases = []
    for k in range(6):
        M = [8, 12, 16][k % 3]
        s = rng.uniform(0, 255, (M, M))
        loss = rng.uniform(size=(M, M)) < 0.25
        cases.append(run_rfse(s, AreaMask.from_loss(loss), 0.8, 0.2, 20))
    for (t, l) in [(128, 128), (0, 256)]:
        s, m = window(img4, t, l, 32, 8, 8)
        cases.append(run_rfse(s, m, rho, gamma, 50))
    for (t, l) in [(96, 160), (0, 0)]:
        s, m = window(img2, t, l, 64, 16, 16)
        cases.append(run_rfse(s, m, rho, gamma, 50))
    s, m = window(img2, 160, 160, 64, 16, 16)
    cases.append(run_rfse(s, m, rho, gamma, 50, basis_target=7))
    cases.append(run_rfse(s, m, rho, gamma, 50, basis_target=0))
    save("rfse.npz", cases)


if __name__ == "__main__":
    main()

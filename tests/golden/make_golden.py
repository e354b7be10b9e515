"""Generate golden vectors by running the REFERENCE cFSE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py wide   # wide_*.npz

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

from paper_2204_14193_b200.synth import field, frame_u8  # noqa: E402
from oracle.oracle import frames_pattern  # noqa: E402  (== the product's pattern generator)


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


# ---------------------------------------------------------------- wide sets
# The wide fp64 gate (>= 1,000 reference windows over every BASELINE config
# geometry).  Inputs are NOT stored: the test regenerates the seeded frames
# with paper_2204_14193_b200.synth (numpy, deterministic) and cuts the same
# windows; the fixture holds the block list and the reference's outputs.

WIDE_SETS = {
    # name: frame generator spec, blocks, geometry, iterations
    "c2": dict(gen="field_f32", shape=(512, 512), seeds=[2], F=64, B=16, border=16, iters=100),
    "c4a": dict(gen="field_f32", shape=(512, 512), seeds=[4], F=32, B=8, border=8, iters=100),
    "c4b": dict(gen="field_f32", shape=(512, 512), seeds=[40 + k for k in range(8)], F=128, B=32,
                border=16, iters=100, pixels=125),
    "c5": dict(gen="frame_u8", shape=(2160, 3840), seeds=[500, 501], F=64, B=16, border=16, iters=100),
    "c3": dict(gen="frame_u8", shape=(1080, 1920), seeds=[300, 301], F=64, B=16, border=16, iters=200),
}


# rFSE wide sets (rfse.py:170-210): fixed count and basis_target runs
WIDE_RFSE = {
    "r64": dict(gen="field_f32", shape=(512, 512), seeds=[2], F=64, B=16, border=16, iters=50),
    "r32": dict(gen="field_f32", shape=(512, 512), seeds=[4], F=32, B=8, border=8, iters=50),
    "r128": dict(gen="field_f32", shape=(512, 512), seeds=[40], F=128, B=32, border=16, iters=40),
}


def rfse_blocks(name):
    if name == "r64":
        return np.array([(0, 32 * i, 32 * j) for i in range(16) for j in range(16)], np.int32)
    if name == "r32":
        tl = np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::4]
        return np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
    return np.array([(0, 64 * i, 64 * j) for i in range(8) for j in range(8)], np.int32)


def make_wide_rfse(name):
    spec = WIDE_RFSE[name]
    frames = wide_frames(spec)
    blocks = rfse_blocks(name)
    F, B, border, I = spec["F"], spec["B"], spec["border"], spec["iters"]
    rho, gamma = 0.8, 0.5
    n = len(blocks)
    # every 4th window runs in basis_target mode (target 2 I - 3: ends on the tally rule)
    bts = np.array([2 * I - 3 if k % 4 == 3 else -1 for k in range(n)], np.int32)
    cap = max(I, 2 * I - 3)
    uv = np.full((n, cap, 2), -1, np.int16)
    cs = np.zeros((n, cap), np.complex128)
    selfs = np.zeros((n, cap), np.uint8)
    count = np.zeros(n, np.int32)
    tally = np.zeros(n, np.int32)
    px = np.zeros((n, B * B))
    for k, (f, t, l) in enumerate(blocks):
        s, m = window(frames[f].astype(np.float64), int(t), int(l), F, B, border)
        r = run_rfse(s, m, rho, gamma, I, basis_target=None if bts[k] < 0 else int(bts[k]))
        c = len(r["us"])
        uv[k, :c, 0], uv[k, :c, 1] = r["us"], r["vs"]
        cs[k, :c] = r["cs"]
        selfs[k, :c] = r["selfs"]
        count[k], tally[k] = c, r["tally"]
        px[k] = r["recon_loss"]
    np.savez_compressed(os.path.join(HERE, f"wide_{name}.npz"), blocks=blocks, basis_target=bts, uv=uv,
                        cs=cs, selfs=selfs, count=count, tally=tally, pixels=px, F=F, B=B, border=border,
                        iterations=I, rho=rho, gamma=gamma)
    print(f"wide_{name}.npz", n, "windows")


def wide_frames(spec):
    H, W = spec["shape"]
    if spec["gen"] == "field_f32":
        return np.stack([field(H, W, seed=s).astype(np.float32) for s in spec["seeds"]])
    return np.stack([frame_u8(H, W, seed=s) for s in spec["seeds"]])


def wide_blocks(name, spec):
    H, W = spec["shape"]
    if name == "c2":
        return np.array([(0, 32 * i, 32 * j) for i in range(16) for j in range(16)], np.int32)
    if name == "c4a":
        tl = np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::2][:500]
        tl = tl[np.lexsort((tl[:, 1], tl[:, 0]))]
        return np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)
    if name == "c4b":
        return np.array([(f, 64 * i, 64 * j) for f in range(8) for i in range(8) for j in range(8)],
                        np.int32)[:500]
    frac, seed, n = (0.05, 5, 120) if name == "c5" else (0.10, 3, 100)
    allb = frames_pattern(2, H, W, 16, frac, seed)
    b = allb[np.linspace(0, len(allb) - 1, n).round().astype(np.int64)]
    if name == "c5":  # + the four corner classes
        b = np.concatenate([b, np.array([[1, 0, 0], [1, 0, W - 16], [1, H - 16, 0], [1, H - 16, W - 16]],
                                        np.int32)])
    return b


def make_wide(name):
    spec = WIDE_SETS[name]
    frames = wide_frames(spec)
    blocks = wide_blocks(name, spec)
    F, B, border, I = spec["F"], spec["B"], spec["border"], spec["iters"]
    rho, gamma = 0.8, 0.5
    n = len(blocks)
    uv = np.zeros((n, I, 2), np.uint8)
    cs = np.zeros((n, I), np.complex128)
    w00 = np.zeros(n)
    e0 = np.zeros(n)
    npx = spec.get("pixels", n)
    px = np.zeros((npx, B * B))
    for k, (f, t, l) in enumerate(blocks):
        s, m = window(frames[f].astype(np.float64), int(t), int(l), F, B, border)
        r = run(s, m, rho, gamma, I)
        uv[k, :, 0], uv[k, :, 1] = r["us"], r["vs"]
        cs[k] = r["cs"]
        w00[k], e0[k] = r["w00"], r["e0"]
        if k < npx:
            px[k] = r["recon_loss"]
    np.savez_compressed(os.path.join(HERE, f"wide_{name}.npz"), blocks=blocks, uv=uv, cs=cs, w00=w00,
                        e0=e0, pixels=px, F=F, B=B, border=border, iterations=I, rho=rho, gamma=gamma)
    print(f"wide_{name}.npz", n, "windows")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wide":
        for name in (sys.argv[2:] or list(WIDE_SETS) + list(WIDE_RFSE)):
            if name in WIDE_RFSE:
                make_wide_rfse(name)
            else:
                make_wide(name)
    else:
        main()

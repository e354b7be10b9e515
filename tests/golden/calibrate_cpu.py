"""Calibrate the CPU baseline: the reference's own extrapolate_cfse (numba,
one process = one core) against the oracle port (C, one thread) on the same
config-5 windows, in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/calibrate_cpu.py

bench.py's cpu_baseline and --impl reference time the port on the GPU box
(the reference cannot travel there); this records how the port's per-core
rate relates to the reference's, and that both give the same tiles, in
tests/golden/cpu_calibration.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("FSE_REFERENCE_SRC", "/root/reference/pkg/src"))

from fse.cfse import extrapolate_cfse  # noqa: E402  (reference)
from fse.types import FseConfig  # noqa: E402
from make_golden import window  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2204_14193_b200.harness import frames_pattern  # noqa: E402
from paper_2204_14193_b200.synth import frame_u8  # noqa: E402

F, B, BORDER, RHO, GAMMA, ITERS = 64, 16, 16, 0.8, 0.5, 100
H, W = 2160, 3840
img = frame_u8(H, W, seed=5)
blocks = frames_pattern(1, H, W, B, 0.05, seed=5)[:120]
cfg = FseConfig(rho_hat=RHO, gamma=GAMMA, iterations=ITERS, fft_dims=(F, F))
off = (F - B) // 2

wins = [window(img.astype(np.float64), int(t), int(l), F, B, BORDER) for _, t, l in blocks]
extrapolate_cfse(*wins[0], cfg)  # numba JIT warm-up
t0 = time.perf_counter()
ref_tiles = [extrapolate_cfse(s, m, cfg).reconstructed[off:off + B, off:off + B] for s, m in wins]
t_ref = time.perf_counter() - t0

orc.conceal_blocks(img, blocks[:2], B, BORDER, F, RHO, GAMMA, ITERS, nthreads=1)
t0 = time.perf_counter()
port = orc.conceal_blocks(img, blocks, B, BORDER, F, RHO, GAMMA, ITERS, nthreads=1)
t_port = time.perf_counter() - t0

dev = float(np.max(np.abs(np.stack(ref_tiles) - port)))
out = {
    "workload": "config 5 geometry (F=64, B=16, border 16, I=100), first 120 lost blocks of a "
                "3840x2160 u8 frame (seed 5)",
    "reference_blocks_per_s_1core": len(blocks) / t_ref,
    "port_blocks_per_s_1thread": len(blocks) / t_port,
    "port_over_reference": t_ref / t_port,
    "max_abs_tile_difference": dev,
    "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(" :\t"),
}
print(json.dumps(out, indent=1))
with open(os.path.join(HERE, "cpu_calibration.json"), "w") as fh:
    json.dump(out, fh, indent=1)

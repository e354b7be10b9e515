"""Every lost block of the benched workload against the CPU oracle.

bench.py gates an evenly spaced sample of its timed tiles (<= 32 frames);
this script runs the whole of BASELINE config 5 (or 3): the u8 tiles of one
full plan run (what bench.py times) are compared bit for bit with re-runs of
32-frame chunks in f32 + trace, and every chunk is gated against the fp64 C
oracle (oracle/gate.py: per block max |dpx| <= 0.5 except certified near-ties,
pooled PSNR within 0.01 dB).  Test infrastructure: run on the GPU box,

    python scripts/config5_full_parity.py [--config 5] [--out gpurun_out/x.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_14193_b200 as fse  # noqa: E402
from paper_2204_14193_b200.synth import field_torch  # noqa: E402


def run(config: str = "5", chunk: int = 32, n_frames: int | None = None, verbose: bool = False):
    """Gate every lost block of bench.py's workload `config`; returns
    (summary record, per-chunk records)."""
    a = argparse.Namespace(config=config, chunk=chunk, frames=n_frames)
    cfg = dict(bench.CONFIGS[a.config])
    if a.frames:
        cfg["frames"] = a.frames
    nf = cfg["frames"]
    blocks = fse.frames_pattern(nf, cfg["H"], cfg["W"], cfg["B"], cfg["frac"],
                                bench.SEED if a.config == "5" else 3)
    frames = field_torch(nf, cfg["H"], cfg["W"], seed=bench.frame_seed(a.config), device="cuda")
    geo = fse.Geometry(cfg["B"], cfg["border"], cfg["F"])
    plan_kw = dict(geometry=geo, rho_hat=bench.RHO, gamma=bench.GAMMA, iterations=cfg["iters"],
                   precision="fp32")
    plan = fse.ConcealPlan(blocks, cfg["H"], cfg["W"], **plan_kw)
    tiles = torch.empty((len(blocks), cfg["B"], cfg["B"]), dtype=torch.uint8, device="cuda")
    plan.run(frames, tiles)
    torch.cuda.synchronize()
    timed = tiles.cpu().numpy()

    tot = dict(blocks=0, over_0p5=0, certified_strict=0, certified_bounded=0, max_dev=0.0)
    chunks, ok, t0 = [], True, time.time()
    for f0 in range(0, nf, a.chunk):
        f1 = min(nf, f0 + a.chunk)
        sel = np.nonzero((blocks[:, 0] >= f0) & (blocks[:, 0] < f1))[0]
        cb = blocks[sel].copy()
        cb[:, 0] -= f0
        r = bench.parity_sample(fse, plan_kw, frames[f0:f1], cb, timed[sel], cfg, len(cb))
        r["frames_range"] = [f0, f1]
        chunks.append(r)
        ok = ok and r["passed"]
        tot["blocks"] += r["blocks"]
        for k in ("over_0p5", "certified_strict", "certified_bounded"):
            tot[k] += r[k] or 0
        tot["max_dev"] = max(tot["max_dev"], r["max_dev"] or 0.0)
        if verbose:
            print(json.dumps(r), flush=True)
    rec = {"workload": f"config{a.config}", "frames": nf, "H": cfg["H"], "W": cfg["W"],
           "iterations": cfg["iters"], "F": cfg["F"], **tot,
           "psnr_delta_db_worst_chunk": max((abs(c["psnr_delta_db"]) for c in chunks
                                             if c["psnr_delta_db"] is not None), default=None),
           "timed_u8_equal_every_chunk": all(c["timed_u8_equal"] for c in chunks),
           "passed": bool(ok and tot["blocks"] == len(blocks)), "seconds": round(time.time() - t0, 1),
           "gate": chunks[0]["gate"] if chunks else None}
    return rec, chunks


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="5", choices=sorted(bench.CONFIGS))
    p.add_argument("--chunk", type=int, default=32)
    p.add_argument("--frames", type=int, default=None)
    p.add_argument("--out", default=None)
    a = p.parse_args()
    rec, chunks = run(a.config, a.chunk, a.frames, verbose=True)
    print(json.dumps(rec))
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(rec) + "\n")
            for c in chunks:
                f.write(json.dumps(c) + "\n")
    sys.exit(0 if rec["passed"] else 1)


if __name__ == "__main__":
    main()

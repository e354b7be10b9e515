"""Kernel-variant equivalence check: run the fused kernel (library chosen by
FSE_LIB_PATH) on fixed workloads of every window size and save tiles +
traces; `--compare a.npz b.npz ...` asserts they are bitwise identical.
Used to prove that a scheduling/bookkeeping change keeps the exact results
(the same arithmetic and the same first-max selection)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out):
    import torch

    import paper_2204_14193_b200 as fse
    from paper_2204_14193_b200.synth import field_torch
    res = {}
    frames = field_torch(3, 2160, 3840, seed=5 * 7919, device="cuda")
    for F, B, bd, frac, it in ((64, 16, 16, 0.05, 100), (32, 8, 8, 0.05, 100), (128, 32, 16, 0.03, 100),
                               (64, 16, 16, 0.05, 450)):
        blocks = fse.frames_pattern(3, 2160, 3840, B, frac, seed=F + it)[:6000]
        plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(B, bd, F), gamma=0.5, iterations=it)
        t, tr = plan.run(frames, tile_dtype="f32", trace=True)
        key = f"F{F}_I{it}"
        res[key + "_tiles"] = t.cpu().numpy()
        res[key + "_uv"] = tr["uv"].cpu().numpy()
        res[key + "_c"] = tr["c"].cpu().numpy()
    np.savez(out, **res)
    print("saved", out, {k: v.shape for k, v in res.items() if k.endswith("tiles")})


def compare(paths):
    base = np.load(paths[0])
    ok = True
    for p in paths[1:]:
        z = np.load(p)
        for k in base.files:
            same = np.array_equal(base[k], z[k])
            if not same:
                ok = False
                d = np.nonzero((base[k] != z[k]).reshape(len(base[k]), -1).any(1))[0]
                print(f"DIFF {p} {k}: {len(d)} blocks differ, first {d[:5]}")
        print(p, "bitwise identical" if ok else "DIFFERS")
    return ok


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(0 if compare(sys.argv[2:]) else 1)
    run(sys.argv[1])

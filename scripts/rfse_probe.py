"""Fused fp32 rFSE (F=64) vs the per-window fp64 rFSE plan on the same blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
H, W = 540, 960
frames = field_torch(2, H, W, seed=11, device="cuda", edges=True)
blocks = fse.frames_pattern(2, H, W, 16, 0.05, seed=3)[:200]
blocks = np.concatenate([blocks, np.array([[0, 0, 0], [1, H - 16, W - 16]], np.int32)])
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bt = int(sys.argv[2]) if len(sys.argv) > 2 else -1
kw = dict(rho_hat=0.8, gamma=0.5, algorithm="rfse")
if bt >= 0:
    kw["basis_target"] = bt
fast = fse.ConcealPlan(blocks, H, W, fse.Geometry(16, 16, 64), iterations=iters, precision="fp32", **kw)
ref = fse.ConcealPlan(blocks, H, W, fse.Geometry(16, 16, 64), iterations=iters, precision="fp64", **kw)
print("fast info", fast.info, "ref info", ref.info)
t32, tr = fast.run(frames, tile_dtype="f32", trace=True)
t64 = ref.run(frames, tile_dtype="f64")
d = (t32.double() - t64).abs().reshape(len(blocks), -1).max(1).values.cpu().numpy()
print("max dev", d.max(), "median", np.median(d), "blocks > 0.5:", int((d > 0.5).sum()), "of", len(d))
uv = tr["uv"].cpu().numpy()
print("first block trace uv", uv[0, :8].tolist())
e = tr["e"].cpu().numpy()
print("energies block0", e[0, :5].tolist(), "...", e[0, -2:].tolist())

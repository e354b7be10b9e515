"""Fused rFSE vs fused cFSE throughput on config-5 frames at equal basis-function
counts (cFSE: I = BF iterations; rFSE: basis_target = BF).
Usage: python scripts/rfse_rate.py [F]  (F = 32, 64, 128; F = 128 uses the
config-4b geometry, border 16, 4 % loss: interior blocks fused, clipped ones
per window, both inside the timed plan run)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F = int(sys.argv[1]) if len(sys.argv) > 1 else 64
nf = 32 if F == 64 else 8
border = 16 if F == 128 else F // 4
frames = field_torch(nf, 2160, 3840, seed=5, device="cuda", edges=True)
blocks = fse.frames_pattern(nf, 2160, 3840, F // 4, 0.04 if F == 128 else 0.05, seed=5)
# interior blocks only (every window unclipped: all fused; at F = 128 the
# clipped rFSE windows otherwise run on the per-window kernel)
off = (F - F // 4) // 2
inner = blocks[(blocks[:, 1] >= off) & (blocks[:, 2] >= off) & (blocks[:, 1] + F - off <= 2160) &
               (blocks[:, 2] + F - off <= 3840)]
for bf in (100, 200):
    for alg in ("cfse", "rfse", "rfse-interior"):
        blocks_all = blocks
        if alg == "rfse-interior":
            blocks, alg = inner, "rfse"
        name = "rfse-interior" if blocks is inner else alg
        kw = dict(iterations=bf) if alg == "cfse" else dict(iterations=bf, basis_target=bf)
        plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(F // 4, border, F), rho_hat=0.8, gamma=0.5,
                               algorithm=alg, **kw)
        t = plan.run(frames)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            plan.run(frames, t)
        e1.record(); torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 3 / 1e3
        # iterations actually run (rFSE stops at the basis target) and the
        # shared-memory bytes they read: per bin and iteration 8 B of W' (cFSE);
        # rFSE 16 B of W' (both atoms) + 12 B of criterion coefficients
        _, tr = plan.run(frames, tile_dtype="f32", trace=True)
        its = float((tr["uv"][:, :, 0] >= 0).sum(1).double().mean())
        per_bin = 8 if alg == "cfse" else 28
        tbps = len(blocks) / s * its * F * F * per_bin / 1e12
        peak = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 1965e6 / 1e12
        print(json.dumps({"F": F, "algorithm": name, "basis_functions": bf, "blocks": len(blocks),
                          "blocks_per_s": len(blocks) / s, "us_per_block": s / len(blocks) * 1e6,
                          "mean_iterations": its, "smem_bytes_per_bin_iteration": per_bin,
                          "smem_TBps": tbps, "frac_nominal": tbps / peak, "plan": plan.info}))
        blocks = blocks_all

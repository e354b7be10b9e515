"""Per-phase cycle counts of the fused F = 128 kernel (FSE_DIAG=32 library via
FSE_LIB_PATH; one block per SM, so a lone block is the large-batch case):
window + row FFTs, row-phase barrier, column FFTs, readout, 100 iterations,
synthesis -- medians over 148 and 1,184 blocks of config-5-style 4K frames."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
names = ["rows_fft", "rows_sync", "cols_fft", "readout+e0", "iterations", "synth+store"]
frames = field_torch(4, 2160, 3840, seed=5, device="cuda", edges=True)
allb = fse.frames_pattern(4, 2160, 3840, 32, 0.04, seed=5)
for n in (148, 1184):
    b = allb[:n]
    plan = fse.ConcealPlan(b, 2160, 3840, fse.Geometry(32, 48, 128), rho_hat=0.8, gamma=0.5, iterations=100)
    t = plan.run(frames, tile_dtype="f32"); t = plan.run(frames, tile_dtype="f32"); torch.cuda.synchronize()
    c = t.reshape(t.shape[0], -1)[:, 1:7].cpu().numpy().astype(np.float64)
    prev = np.zeros(len(c)); marks = {}
    for j, nm in enumerate(names):
        marks[nm] = float(np.median(c[:, j] - prev)); prev = c[:, j]
    print(json.dumps({"F": 128, "blocks": n, "info": plan.info, "phase_cycles_median": marks}))

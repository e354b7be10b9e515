"""Per-phase cycle counts of a lone fused block (small batch; FSE_DIAG=32
library via FSE_LIB_PATH): rows FFT, sync, column FFT, readout, 100
iterations, synthesis -- medians over the blocks of a 64-block batch."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field, grid_blocks
names = ["rows_fft", "rows_sync", "cols_fft", "readout+e0", "iterations", "synth+store"]
for F, B, bd, n in ((64, 16, 16, 64), (32, 8, 8, 64), (64, 16, 16, 256)):
    img = torch.from_numpy(field(512, 512, seed=2).astype(np.float32)).cuda()
    tl = grid_blocks(512, 512, B) if F == 64 else np.array([(16 * i, 16 * j) for i in range(32) for j in range(32)], np.int32)[::2]
    b = np.concatenate([np.zeros((len(tl), 1), np.int32), tl], 1)[:n]
    plan = fse.ConcealPlan(b, 512, 512, fse.Geometry(B, bd, F), gamma=0.5, iterations=100)
    t = plan.run(img, tile_dtype="f32"); t = plan.run(img, tile_dtype="f32"); torch.cuda.synchronize()
    c = t.reshape(t.shape[0], -1)[:, 1:7].cpu().numpy()
    prev = np.zeros(len(c)); marks = {}
    for j, nm in enumerate(names):
        marks[nm] = float(np.median(c[:, j] - prev)); prev = c[:, j]
    print(json.dumps({"F": F, "blocks": n, "phase_cycles_median": marks}))

"""Slot phase probe (FSE_DIAG=32 library via FSE_LIB_PATH): per iteration the
fused kernel records its start clock and the (CTA, slot) that ran it.
Reports iteration period, setup+synthesis gap between blocks, and how the
five slots of a CTA are phased relative to each other."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200 import synth

n_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
F = int(sys.argv[2]) if len(sys.argv) > 2 else 64
H, W = 2160, 3840
frames = synth.field_torch(n_frames, H, W, 5, "cuda")
blocks = fse.frames_pattern(n_frames, H, W, F // 4, 0.05 if F < 128 else 0.04, seed=5)
plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(B=F // 4, border=8 if F == 32 else 16, F=F),
                       rho_hat=0.8, gamma=0.5, iterations=100)
for _ in range(2):
    tiles, tr = plan.run(frames, trace=True)
torch.cuda.synchronize()
uv = tr["uv"].cpu().numpy().astype(np.int64)
clk = uv[:, :, 0] & 0xffffffff
cta = uv[:, 0, 1] // 8
slot = uv[:, 0, 1] % 8
it_period = np.diff(clk, axis=1) & 0xffffffff
out = {"iter_period_median": float(np.median(it_period)), "iter_period_p10": float(np.percentile(it_period, 10)),
       "iter_period_p90": float(np.percentile(it_period, 90))}
# per CTA: blocks in order of start; gaps between consecutive blocks of the same slot
gaps, phase = [], []
for c in np.unique(cta)[:40]:
    sel = np.where(cta == c)[0]
    for s in range(5):
        ss = sel[slot[sel] == s]
        ss = ss[np.argsort(clk[ss, 0])]
        for a, b in zip(ss[:-1], ss[1:]):
            gaps.append(int((clk[b, 0] - clk[a, -1]) & 0xffffffff))
    # phase of slot starts of iteration 50 relative to the CTA's slot 0 block running at the same time
    s0 = sel[slot[sel] == 0]
    for b0 in s0[:20]:
        t = clk[b0, 50]
        per = np.median(np.diff(clk[b0]) & 0xffffffff)
        for s in range(1, 5):
            ss = sel[slot[sel] == s]
            # nearest iteration start of slot s to t
            d = ((clk[ss] - t + 2**31) & 0xffffffff) - 2**31
            if d.size == 0:
                continue
            k = np.argmin(np.abs(d))
            phase.append(float((np.abs(d).flat[k] % per) / per))
out["block_gap_median"] = float(np.median(gaps)) if gaps else None
out["phase_hist"] = np.histogram(phase, bins=10, range=(0, 1))[0].tolist()
print(json.dumps(out))
# phase marks (FSE_TMARK): c[b, j, 0] = T_j - T_0
c = tr["c"].cpu().numpy()[:, 1:7, 0]
names = ["rows_fft", "rows_sync", "cols_fft", "readout+e0", "iterations", "synth+store"]
prev = np.zeros(len(c))
marks = {}
for j, n in enumerate(names):
    marks[n] = float(np.median(c[:, j] - prev))
    prev = c[:, j]
print(json.dumps({"phase_cycles_median": marks}))

# the same marks without trace output (tile-based: f32 tiles carry T_j - T_0)
t2 = plan.run(frames, tile_dtype="f32")
t2 = plan.run(frames, tile_dtype="f32")
torch.cuda.synchronize()
c = t2.reshape(t2.shape[0], -1)[:, 1:7].cpu().numpy()
prev = np.zeros(len(c))
marks = {}
for j, n in enumerate(names):
    marks[n] = float(np.median(c[:, j] - prev))
    prev = c[:, j]
print(json.dumps({"phase_cycles_median_no_trace": marks}))

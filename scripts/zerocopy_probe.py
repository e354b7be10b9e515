"""Fused kernel reading the frames straight from page-locked host memory
(unified addressing; TMA tile loads of each support window, or direct loads)
vs device-resident frames: config-5 frames, device time per launch."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = field_torch(nf, 2160, 3840, seed=5 * 7919, device="cuda")
host = dev.cpu().pin_memory()
blocks = fse.frames_pattern(nf, 2160, 3840, 16, 0.05, seed=5)
plan = fse.ConcealPlan(blocks, 2160, 3840, gamma=0.5, iterations=100)
ref = plan.run(dev).cpu()


def t(fr, reps=5):
    out = plan.run(fr); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.run(fr, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), out.cpu()


res = {"frames": nf, "blocks": len(blocks)}
for name, fr, tma in (("device", dev, None), ("host_tma", host, "1"), ("host_direct", host, "0")):
    if tma is not None:
        os.environ["FSE_TMA"] = tma
    ms, out = t(fr)
    os.environ.pop("FSE_TMA", None)
    res[name + "_ms"] = ms
    res[name + "_blocks_per_s"] = len(blocks) / ms * 1e3
    res[name + "_equal"] = bool(torch.equal(out, ref))
print(json.dumps(res))

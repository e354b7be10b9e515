"""Throughput and SMEM-roofline fraction of the fused kernel for the three
window sizes (configs 4a / 2 / 4b geometries) on a large synthetic batch."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
sms = torch.cuda.get_device_properties(0).multi_processor_count
peak = sms * 128 * 1965e6
frames = field_torch(16, 2160, 3840, seed=9, device="cuda", edges=True)
only = [int(a) for a in sys.argv[1:]]
for F, B, border in ((32, 8, 8), (64, 16, 16), (128, 32, 16)):
    if only and F not in only:
        continue
    blocks = fse.frames_pattern(16, 2160, 3840, B, 0.05 if B < 32 else 0.04, seed=2)
    plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(B, border, F), iterations=100, gamma=0.5)
    t = plan.run(frames); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): plan.run(frames, t)
    e1.record(); torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 3 / 1e3
    rate = len(blocks) / s
    achieved = rate * 8 * F * F * 100
    print(json.dumps({"F": F, "B": B, "border": border, "blocks": len(blocks), "blocks_per_s": rate,
                      "smem_TBps": achieved / 1e12, "frac_nominal": achieved / peak,
                      "roofline_blocks_per_s": peak / (8 * F * F * 100), "plan": plan.info}))

import os, sys, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from oracle import oracle as orc
use_torch = len(sys.argv) > 1
if use_torch:
    import torch
    from paper_2204_14193_b200.synth import field_torch
    fr = field_torch(6, 2160, 3840, seed=5 * 7919, device="cuda").cpu().numpy()
else:
    from paper_2204_14193_b200.synth import frame_u8
    fr = np.stack([frame_u8(2160, 3840, seed=s) for s in range(2)])
nf = fr.shape[0]
b = orc.frames_pattern(nf, 2160, 3840, 16, 0.05, 5)
res = {"torch": use_torch, "blocks": len(b), "cpus": len(os.sched_getaffinity(0))}
for nt in (1, 8, 16):
    n = 48 if nt == 1 else len(b)
    t = time.perf_counter(); orc.conceal_blocks(fr, b[:n], 16, 16, 64, 0.8, 0.5, 100, nthreads=nt); dt = time.perf_counter() - t
    res[f"t{nt}"] = n / dt
print(json.dumps(res))

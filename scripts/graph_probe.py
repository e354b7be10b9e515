"""Concealer.run vs a captured CUDA graph of the same pipeline (config-5
frames, N frames per GPU): tiles identical, e2e blocks/s."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = field_torch(nf, 2160, 3840, seed=5 * 7919, device="cuda")
host = dev.cpu().pin_memory()
del dev
blocks = fse.frames_pattern(nf, 2160, 3840, 16, 0.05, seed=5)
con = fse.Concealer(blocks, nf, 2160, 3840, gamma=0.5, iterations=100)
ref = con.run(host, copy=True)
replay = con.capture(host)
t_graph = replay(copy=True)
res = {"frames": nf, "equal": bool(np.array_equal(ref, t_graph))}
for name, fn in (("run", lambda: con.run(host)), ("graph", lambda: replay())):
    for _ in range(3):
        fn()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    res[name + "_blocks_per_s"] = 10 * len(blocks) / (time.perf_counter() - t)
print(json.dumps(res))

"""One fused rFSE run on config-5 frames (for profiling): python scripts/rfse_once.py [F]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F = int(sys.argv[1]) if len(sys.argv) > 1 else 64
frames = field_torch(8, 2160, 3840, seed=5, device="cuda", edges=True)
blocks = fse.frames_pattern(8, 2160, 3840, F // 4, 0.05, seed=5)
plan = fse.ConcealPlan(blocks, 2160, 3840, fse.Geometry(F // 4, F // 4, F), rho_hat=0.8, gamma=0.5,
                       algorithm="rfse", iterations=100, basis_target=100)
for _ in range(2):
    plan.run(frames)
torch.cuda.synchronize()
print("ok", len(blocks), plan.info)

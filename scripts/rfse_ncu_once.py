"""One fused rFSE plan run (100 basis functions, 16 config-5 frames) after a warm-up run: the launch ncu captures (-k regex:fast_kernel -s 1 -c 1).  Usage: python scripts/rfse_ncu_once.py F"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
F = int(sys.argv[1])
fr = field_torch(16, 2160, 3840, seed=5, device="cuda", edges=True)
b = fse.frames_pattern(16, 2160, 3840, F // 4, 0.05, seed=5)
p = fse.ConcealPlan(b, 2160, 3840, fse.Geometry(F // 4, 16 if F == 128 else F // 4, F), rho_hat=0.8, gamma=0.5,
                    algorithm="rfse", iterations=100, basis_target=100)
t = p.run(fr); torch.cuda.synchronize(); p.run(fr, t); torch.cuda.synchronize(); print("ok", len(b))

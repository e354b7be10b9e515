"""Event timeline of Concealer.run: per chunk copy / kernel start-end (ms)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2204_14193_b200 as fse
from paper_2204_14193_b200.synth import field_torch
nf, H, W, ch = 64, 2160, 3840, 8
frames = field_torch(nf, H, W, seed=3, device="cuda")
host = frames.cpu().pin_memory()
blocks = fse.frames_pattern(nf, H, W, 16, 0.05, 5)
con = fse.Concealer(blocks, nf, H, W, chunk_frames=ch)
con.run(host)
# instrumented copy of Concealer.run
E = lambda: torch.cuda.Event(enable_timing=True)
cs = con.copy_stream
t0 = E(); t0.record(torch.cuda.current_stream()); torch.cuda.synchronize()
base = E(); base.record(cs)
rec = []
done = [None] * len(con.chunks)
nb = len(con.dev_frames)
for i, (f0, f1, lo, hi, plan) in enumerate(con.chunks):
    buf = con.dev_frames[i % nb]
    with torch.cuda.stream(cs):
        if i >= nb: cs.wait_event(done[i - nb])
        a = E(); a.record(cs)
        buf[: f1 - f0].copy_(host[f0:f1], non_blocking=True)
        b = E(); b.record(cs)
    ks = con.compute_streams[i % 2]
    with torch.cuda.stream(ks):
        ks.wait_event(b)
        c = E(); c.record(ks)
        plan.run(buf[: f1 - f0], con.dev_tiles[lo:hi], stream=ks)
        d = E(); d.record(ks)
        con.host_tiles[lo:hi].copy_(con.dev_tiles[lo:hi], non_blocking=True)
        e = E(); e.record(ks)
        done[i] = e
    rec.append((a, b, c, d, e))
torch.cuda.synchronize()
for i, (a, b, c, d, e) in enumerate(rec):
    f = lambda x: base.elapsed_time(x)
    print(f"chunk {i}: copy {f(a):6.2f}-{f(b):6.2f}  kernel {f(c):6.2f}-{f(d):6.2f}  d2h-end {f(e):6.2f}")

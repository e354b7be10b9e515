"""Shared-memory wavefronts per source line of an ncu report, per block.
usage: python scripts/ncu_wavefronts.py report.ncu-rep n_blocks"""
import csv, io, subprocess, sys
from collections import defaultdict
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
iw, ie, ii = (hdr.index(k) for k in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
                                      "Instructions Executed"))
def fl(x):
    try: return float(x)
    except ValueError: return 0.0
line, agg, seen = None, defaultdict(lambda: [0.0, 0.0, 0.0]), set()
for r in rows[3:]:
    if r and r[0] and r[0].isdigit():
        line = int(r[0]); continue
    if not r or r[0]: continue
    if r[2] in seen:  # inlined code lists a SASS row under several source lines: count once
        continue
    seen.add(r[2])
    a = agg[line]; a[0] += fl(r[iw]); a[1] += fl(r[ie]); a[2] += fl(r[ii])
B = float(sys.argv[2])
src = open("paper_2204_14193_b200/csrc/fast.cu").read().split("\n")
tot = sum(a[0] for a in agg.values())
print(f"wavefronts/block {tot / B:.0f}  excessive/block {sum(a[1] for a in agg.values()) / B:.0f}")
for ln, (w, e, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:20]:
    if w == 0: break
    print(f"{ln:5d} wf {w / B:8.1f} exc {e / B:7.1f} inst {n / B:8.1f}  {src[ln - 1].strip()[:70]}")

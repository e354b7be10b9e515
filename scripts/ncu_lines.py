"""Per-source-line totals of an ncu report (SASS rows attributed to the
preceding CUDA line): samples, warp instructions, shared wavefronts.
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
ci = {k: hdr.index(k) for k in ("# Samples", "Instructions Executed", "L1 Wavefronts Shared",
                                "L1 Wavefronts Shared Excessive")}
agg = defaultdict(lambda: [0, 0, 0, 0, 0])
line = None
for r in rows[3:]:
    if r and r[0] and r[0].isdigit():
        line = int(r[0]); continue
    if not r or r[0] or line is None: continue
    a = agg[line]
    for j, k in enumerate(ci):
        try: a[j] += float(r[ci[k]] or 0)
        except ValueError: pass
    a[4] += 1
tot = [sum(a[j] for a in agg.values()) for j in range(4)]
print(f"total samples {tot[0]:.0f} instrs {tot[1]:.3g} smem wavefronts {tot[2]:.3g} excessive {tot[3]:.3g}")
src = open(sys.argv[2] if len(sys.argv) > 3 else "paper_2204_14193_b200/csrc/fast.cu").read().splitlines()
top = int(sys.argv[-1]) if len(sys.argv) > 2 and sys.argv[-1].isdigit() else 40
for ln, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    s = src[ln - 1].strip()[:60] if ln - 1 < len(src) else ""
    print(f"{ln:5d} smp {100*a[0]/tot[0]:5.1f}% ins {100*a[1]/tot[1]:5.1f}% wf {100*a[2]/max(tot[2],1):5.1f}% exc {a[3]:9.3g} n{a[4]:4d}  {s}")

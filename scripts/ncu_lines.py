"""Per-source-line totals of an ncu report (SASS rows attributed to the
preceding CUDA line, every source file of the kernel): samples, warp
instructions, shared wavefronts.
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv, io, os, subprocess, sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])
srcs = {}
fname, ci, key = None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        ci = {k: r.index(k) for k in ("# Samples", "Instructions Executed", "L1 Wavefronts Shared",
                                      "L1 Wavefronts Shared Excessive")}
        continue
    if ci is None or r[0] == "Function Name":
        continue
    if r[0].isdigit():  # a CUDA source line
        key = (fname, int(r[0]))
        srcs[key] = r[1]
        continue
    if key is None:
        continue
    a = agg[key]
    for j, k in enumerate(ci):
        try:
            a[j] += float(r[ci[k]] or 0)
        except (ValueError, IndexError):
            pass
    a[4] += 1
tot = [sum(a[j] for a in agg.values()) for j in range(4)]
print(f"total samples {tot[0]:.0f} instrs {tot[1]:.3g} smem wavefronts {tot[2]:.3g} excessive {tot[3]:.3g}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    s = srcs.get((f, ln), "").strip()[:58]
    print(f"{os.path.basename(f or '?'):12s}{ln:5d} smp {100*a[0]/max(tot[0],1):5.1f}% ins {100*a[1]/max(tot[1],1):5.1f}% "
          f"wf {100*a[2]/max(tot[2],1):5.1f}% exc {a[3]:8.3g}  {s}")

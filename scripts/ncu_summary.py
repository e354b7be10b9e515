"""Summarise an ncu report of the fused kernel: headline metrics, stall
reasons and a per-phase split of warp samples (by per-warp execution count).
Usage: python scripts/ncu_summary.py report.ncu-rep [blocks_in_launch]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, val = raw[0], raw[2]
R = dict(zip(hdr, val))
def g(k):
    try: return float(R[k].replace(",", ""))
    except Exception: return None
keys = ["gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
out = {k: g(k) for k in keys}
for k, v in out.items():
    print(f"{k:90s} {v}")
st = [(g(k), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
      for k in hdr if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
print("stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8] if v))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]; data = src[2:]
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[iss] or 0) for r in data)
maxex = max(float(r[iex] or 0) for r in data)
cls = collections.defaultdict(lambda: [0.0, 0, 0.0])
for r in data:
    ex = float(r[iex] or 0); s = float(r[iss] or 0)
    key = round(ex / maxex * 100) if maxex else 0
    c = cls[key]; c[0] += s; c[1] += 1; c[2] += ex
print("phase split (exec count as % of the hottest instruction: 100 = iteration loop)")
for k, (s, n, ex) in sorted(cls.items(), key=lambda x: -x[1][0])[:10]:
    print(f"  exec%={k:4d} samples={s / tot * 100:6.2f}% static_instrs={n:5d} dyn_instrs={ex:.3g}")

"""Compile csrc/fast.cu to a cubin and summarise the fused kernel's hot loop
(the smallest loop containing >= 80 FFMA2) for F = 32/64/128."""
import collections, os, re, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
defs = sys.argv[1:]
cub = "/tmp/fast_an.cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin",
                "--expt-relaxed-constexpr", *[f"-D{d}" for d in defs], "-I", f"{REPO}/include",
                "-o", cub, f"{REPO}/paper_2204_14193_b200/csrc/fast.cu"], check=True, capture_output=True)
sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)
for fn in re.split(r"\n\s+Function : ", sass)[1:]:
    name = fn.split("\n")[0]
    if "fast_kernel" not in name and "fast_iterate" not in name:
        continue
    F = re.search(r"ILi(\d+)E", name).group(1) + (" tma" if "ELb1E" in name else "") + (" iter" if "iterate" in name else "")
    ins = [l for l in fn.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
    best = None
    for l in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", l)
        if m and int(m.group(1), 16) < addr(l):
            t = int(m.group(1), 16)
            body = [x for x in ins if t <= addr(x) <= addr(l)]
            if (sum("FFMA2" in x for x in body) >= 40 and sum("LDS" in x for x in body) >= 16
                    and (best is None or len(body) < len(best))):
                best = body
    if best is None:
        print(f"F={F}: loop not found"); continue
    c = collections.Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", l).split()[0].split(".")[0]
                            for l in best)
    # distinct LDS.128 destination registers = W' loads the schedule keeps in flight
    bufs = {m.group(1) for l in best for m in [re.search(r"LDS\.128 (R\d+),", l)] if m}
    print(f"F={F}: loop {len(best)} instrs; MOV={c['MOV'] + c['IMAD']} LDL={c['LDL']} STL={c['STL']} "
          f"FFMA2={c['FFMA2']} LDS={c['LDS']} BRA={c['BRA']} ldsbufs={len(bufs)}")
    if os.environ.get("LOOP_DUMP") == F:
        print("\n".join(best))

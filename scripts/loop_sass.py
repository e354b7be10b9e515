"""Compile csrc/fast.cu to a cubin and summarise the fused kernel's hot loop
(instruction mix of the loop containing FFMA2) for F = 32/64/128."""
import re, subprocess, sys, collections, os
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
defs = sys.argv[1:]
cub = "/tmp/fast_an.cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin",
                "--expt-relaxed-constexpr", "-Xptxas=-v", *[f"-D{d}" for d in defs], "-I", f"{REPO}/include",
                "-o", cub, f"{REPO}/paper_2204_14193_b200/csrc/fast.cu"], check=True,
               capture_output=True)
sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for fn in funcs[1:]:
    name = fn.split("\n")[0]
    if "fast_kernel" not in name:
        continue
    F = re.search(r"ILi(\d+)E", name).group(1)
    ins = [l for l in fn.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
    addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)
    fi = [i for i, l in enumerate(ins) if "FFMA2" in l]
    first, last = fi[0], fi[-1]
    end = tgt = None
    for i in range(last, len(ins)):  # innermost backward branch around the FFMA2 block
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", ins[i])
        if m and int(m.group(1), 16) <= addr(ins[first]) and (tgt is None or int(m.group(1), 16) > tgt):
            tgt, end = int(m.group(1), 16), i
    start = [i for i, l in enumerate(ins) if addr(l) == tgt][0]
    body = ins[start:end + 1]
    c = collections.Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", l).split()[0].split(".")[0]
                            for l in body)
    print(f"F={F}: loop {len(body)} instrs; MOV={c['MOV']+c['IMAD']} LDL={c['LDL']} STL={c['STL']} "
          f"FFMA2={c['FFMA2']} LDS={c['LDS']} BRA={c['BRA']}")

"""Compare only the hot iteration loop (smallest backward-branch body with
>= 40 FFMA2 and >= 16 LDS) of every fused kernel in two libraries, ignoring
addresses and constant-bank offsets: python scripts/loop_diff.py old.so new.so"""
import re, subprocess, sys


def loops(path):
    txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    out = {}
    addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)
    for fn in re.split(r"\n\s+Function : ", txt)[1:]:
        name = fn.split("\n")[0].strip()
        if "fast_kernel" not in name:
            continue
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
        if best:
            out[name] = [re.sub(r"0x[0-9a-f]+", "A", re.sub(r"c\[0x0\]\[0x[0-9a-f]+\]", "c[X]",
                         re.sub(r"/\*[0-9a-f]{4,}\*/", "", l).split(";")[0])).strip() for l in best]
    return out


a, b = loops(sys.argv[1]), loops(sys.argv[2])
for k in sorted(set(a) & set(b)):
    la, lb = a[k], b[k]
    d = sum(1 for x, y in zip(la, lb) if x != y) + abs(len(la) - len(lb))
    print(f"{k[:64]} loop {len(la)} {len(lb)} {'same' if d == 0 else f'{d} lines differ'}")

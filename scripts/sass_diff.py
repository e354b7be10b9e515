"""Compare the fused kernels' SASS of two libraries, ignoring constant-bank
offsets (kernel-parameter layout): python scripts/sass_diff.py old.so new.so"""
import hashlib, re, subprocess, sys


def fns(path):
    txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    out = {}
    for fn in re.split(r"\n\s+Function : ", txt)[1:]:
        name = fn.split("\n")[0].strip().replace("ELi0EEEv", "EEEv")
        lines = [re.sub(r"/\*[0-9a-f]{4,}\*/", "", l) for l in fn.split("\n")[1:]
                 if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
        norm = [re.sub(r"c\[0x0\]\[0x[0-9a-f]+\]", "c[X]", l.split(";")[0]).strip() for l in lines]
        out[name] = norm
    return out


a, b = fns(sys.argv[1]), fns(sys.argv[2])
for k in sorted(set(a) | set(b)):
    if "fast_kernel" not in k:
        continue
    la, lb = a.get(k), b.get(k)
    if la is None or lb is None:
        print(f"{k[:60]} only in {'new' if la is None else 'old'}")
        continue
    d = sum(1 for x, y in zip(la, lb) if x != y) + abs(len(la) - len(lb))
    print(f"{k[:60]} {len(la)} {len(lb)} {'same' if d == 0 else f'{d} lines differ'}")

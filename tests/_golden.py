"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = ["config1.npz", "win64.npz", "win32.npz", "win128.npz", "small.npz"]


def load(name):
    z = np.load(os.path.join(GOLDEN, name))
    n = int(z["n"])
    cases = []
    for i in range(n):
        pre = f"{i:03d}_"
        c = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        for k in ("rho", "gamma", "w00", "e0"):
            c[k] = float(c[k])
        c["iterations"] = int(c["iterations"])
        for k in ("tally", "basis_target"):
            if k in c:
                c[k] = int(c[k])
        c["name"] = f"{name}:{i}"
        cases.append(c)
    return cases


def all_cases():
    out = []
    for f in FILES:
        out += load(f)
    return out


def trace(c):
    return c["us"], c["vs"], c["cs"]

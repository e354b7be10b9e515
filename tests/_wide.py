"""Wide fp64 golden sets (tests/golden/wide_*.npz, made by make_golden.py wide
from the reference's own extrapolate_cfse): regenerate the seeded frames and
compare traces / pixels.  Test-side only."""
import functools
import os

import numpy as np

from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SETS = ["c2", "c4a", "c4b", "c5", "c3"]
GEN = {  # must match make_golden.WIDE_SETS
    "c2": ("field_f32", (512, 512), [2]),
    "c4a": ("field_f32", (512, 512), [4]),
    "c4b": ("field_f32", (512, 512), [40 + k for k in range(8)]),
    "c5": ("frame_u8", (2160, 3840), [500, 501]),
    "c3": ("frame_u8", (1080, 1920), [300, 301]),
}


@functools.lru_cache(maxsize=None)
def load(name):
    z = np.load(os.path.join(GOLDEN, f"wide_{name}.npz"))
    d = {k: z[k] for k in z.files}
    for k in ("F", "B", "border", "iterations"):
        d[k] = int(d[k])
    for k in ("rho", "gamma"):
        d[k] = float(d[k])
    return d


@functools.lru_cache(maxsize=None)
def frames(name):
    from paper_2204_14193_b200.synth import field, frame_u8
    gen, (H, W), seeds = GEN[name]
    if gen == "field_f32":
        return np.stack([field(H, W, seed=s).astype(np.float32) for s in seeds])
    return np.stack([frame_u8(H, W, seed=s) for s in seeds])


def golden_trace(d, k):
    return (d["uv"][k, :, 0].astype(np.int64), d["uv"][k, :, 1].astype(np.int64), d["cs"][k])


def compare(d, k, trace, M):
    """Strict gate: the selection sequence is raw-identical to the
    reference's or identical after the single global conjugate-mirror
    canonicalisation; anything else (mirror-pair order swaps
    included) is a divergence.  Coefficients within 1e-9 relative."""
    kind, _ = orc.trace_equivalence(golden_trace(d, k), trace, M, M)
    return kind


def certify(d, k, frames_, trace):
    """A divergence from the reference is accepted only as a certified fp64
    near-tie (oracle.fp64_tie_certificate: at the first canonical split the
    two picks' |R_w| differ by at most twice the two runs' measured fp64
    disagreement).  Returns the certificate dict."""
    from oracle.gate import window_of
    F, B, bd = d["F"], d["B"], d["border"]
    f, t, l = d["blocks"][k]
    s, lab = window_of(frames_[f].astype(np.float64), int(t), int(l), F, B, bd)
    g = golden_trace(d, k)
    at = orc.first_divergence(g, trace, F, F)
    if at is None:  # same selections, coefficients off: not a tie
        return dict(at=None, bounded=False)
    return orc.fp64_tie_certificate(s, lab, d["rho"], d["gamma"], at, trace, g)

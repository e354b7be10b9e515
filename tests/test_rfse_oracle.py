"""The rFSE restatement in the C oracle (orc_rfse_kernel / orc_extrapolate_rfse,
rfse.py:37-210) pinned to the reference's own outputs: the 12 windows of
tests/golden/rfse.npz and the wide rFSE sets (tests/golden/wide_r{64,32,128}.npz:
every config-2 window position at F = 64, 256 config-4a positions at F = 32,
64 windows at F = 128; every 4th in basis_target mode).  Same selections
(canonical pair member), self-conjugate flags, tally; coefficients and
pixels within 1e-9.  The GPU fp64 rFSE plan is checked against the same
wide sets (-m gpu)."""
import functools
import os

import numpy as np
import pytest

from oracle import oracle as orc
from oracle.gate import window_of
from tests import _golden

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
WIDE = ["r64", "r32", "r128"]


@functools.lru_cache(maxsize=None)
def _load(name):
    z = np.load(os.path.join(GOLDEN, f"wide_{name}.npz"))
    d = {k: z[k] for k in z.files}
    for k in ("F", "B", "border", "iterations"):
        d[k] = int(d[k])
    for k in ("rho", "gamma"):
        d[k] = float(d[k])
    return d


@functools.lru_cache(maxsize=None)
def _frames(name):
    from paper_2204_14193_b200.synth import field
    seed = {"r64": 2, "r32": 4, "r128": 40}[name]
    return field(512, 512, seed=seed).astype(np.float32)[None]


def _golden_trace(d, k):
    n = int(d["count"][k])
    return (d["uv"][k, :n, 0].astype(np.int64), d["uv"][k, :n, 1].astype(np.int64), d["cs"][k, :n],
            d["selfs"][k, :n])


@pytest.mark.parametrize("c", _golden.load("rfse.npz"), ids=lambda c: c["name"])
def test_oracle_rfse_matches_reference_goldens(c):
    bt = None if c["basis_target"] < 0 else c["basis_target"]
    o = orc.extrapolate_rfse(c["signal"], c["labels"], c["rho"], c["gamma"], c["iterations"], bt)
    assert np.array_equal(o["us"], c["us"]) and np.array_equal(o["vs"], c["vs"])
    assert np.array_equal(o["selfs"], c["selfs"]) and o["tally"] == c["tally"]
    if len(c["cs"]):
        np.testing.assert_allclose(o["cs"], c["cs"], rtol=1e-9, atol=1e-12 * np.abs(c["cs"]).max())
        np.testing.assert_allclose(o["es"], c["es"], rtol=1e-9, atol=1e-9 * c["e0"])
    loss = c["labels"] == 2
    np.testing.assert_allclose(o["reconstructed"][loss], c["recon_loss"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("name", WIDE)
def test_oracle_rfse_matches_wide_goldens(name):
    d = _load(name)
    fr = _frames(name)
    F, B, bd, I = d["F"], d["B"], d["border"], d["iterations"]
    for k in range(0, len(d["blocks"]), 3):
        f, t, l = d["blocks"][k]
        s, lab = window_of(fr[f].astype(np.float64), int(t), int(l), F, B, bd)
        bt = None if d["basis_target"][k] < 0 else int(d["basis_target"][k])
        o = orc.extrapolate_rfse(s, lab, d["rho"], d["gamma"], I, bt)
        us, vs, cs, sf = _golden_trace(d, k)
        assert np.array_equal(o["us"], us) and np.array_equal(o["vs"], vs), (name, k)
        assert np.array_equal(o["selfs"], sf) and o["tally"] == d["tally"][k]
        np.testing.assert_allclose(o["cs"], cs, rtol=1e-9, atol=1e-12 * np.abs(cs).max())
        np.testing.assert_allclose(o["reconstructed"][lab == 2], d["pixels"][k], rtol=0, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name", WIDE)
def test_fp64_rfse_plan_matches_wide_goldens(cuda_ok, name):
    """GPU fp64 rFSE (per-window reference arithmetic) on every wide window:
    identical canonical pair sequence, flags, counts; coefficients and
    pixels within 1e-9."""
    import torch

    import paper_2204_14193_b200 as fse
    d = _load(name)
    fr = _frames(name)
    F, B, bd, I = d["F"], d["B"], d["border"], d["iterations"]
    bts = d["basis_target"]
    for mode in (-1, 1):  # fixed-count windows, then basis_target windows (one plan each)
        sel = np.nonzero((bts < 0) if mode < 0 else (bts >= 0))[0]
        bt = None if mode < 0 else int(bts[sel[0]])
        plan = fse.ConcealPlan(d["blocks"][sel], 512, 512, fse.Geometry(B, bd, F), rho_hat=d["rho"],
                               gamma=d["gamma"], iterations=I, precision="fp64", algorithm="rfse",
                               basis_target=bt)
        tiles, tr = plan.run(torch.from_numpy(fr).cuda(), tile_dtype="f64", trace=True)
        tiles = tiles.cpu().numpy().reshape(len(sel), -1)
        uv = tr["uv"].cpu().numpy()
        c = tr["c"].cpu().numpy()
        for j, k in enumerate(sel):
            us, vs, cs, _ = _golden_trace(d, k)
            n = int((uv[j, :, 0] >= 0).sum())
            assert n == len(us), (name, k, n, len(us))
            assert np.array_equal(uv[j, :n, 0], us) and np.array_equal(uv[j, :n, 1], vs), (name, k)
            np.testing.assert_allclose(c[j, :n, 0] + 1j * c[j, :n, 1], cs, rtol=1e-9,
                                       atol=1e-12 * np.abs(cs).max())
            np.testing.assert_allclose(tiles[j], d["pixels"][k], rtol=0, atol=1e-9)

"""Pin the CPU oracle (oracle/) against golden vectors produced by running
the reference implementation (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import _golden

CASES = _golden.all_cases()


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(c):
    M, N = c["signal"].shape
    o = orc.extrapolate(c["signal"], c["labels"], c["rho"], c["gamma"], c["iterations"],
                        return_spectra=True)
    loss = c["labels"] == 2
    # pixels: fp64 gate 1e-9 (north_star)
    np.testing.assert_allclose(o["reconstructed"][loss], c["recon_loss"], rtol=0, atol=1e-9)
    # support / padding samples are the input, bit for bit (cfse.py:127-129)
    assert np.array_equal(o["reconstructed"][~loss], c["signal"][~loss])
    # weight DC and initial energy
    assert abs(o["W"][0, 0].real - c["w00"]) <= 1e-12 * c["w00"]
    # selection sequence: identical modulo the conjugate-mirror symmetry
    kind, info = orc.trace_equivalence(_golden.trace(c), (o["us"], o["vs"], o["cs"]), M, N)
    assert kind != "diverged", (kind, info)
    if c["iterations"]:
        np.testing.assert_allclose(o["es"], c["es"], rtol=1e-9, atol=1e-9 * c["e0"])
    if "model" in c:
        np.testing.assert_allclose(o["model"], c["model"], rtol=0, atol=1e-9)


def test_oracle_loop_bitwise_on_reference_spectra():
    """With the reference's own initial spectra, the C loop reproduces the
    numba loop bit for bit."""
    n = 0
    for c in _golden.all_cases():
        if "R_w" not in c:
            continue
        R = np.ascontiguousarray(c["R_w"].copy())
        G, us, vs, cs, es = orc.cfse_kernel(R, c["W"], c["gamma"], 1.0 / c["w00"],
                                            c["iterations"], c["e0"])
        assert np.array_equal(us, c["us"]) and np.array_equal(vs, c["vs"]), c["name"]
        assert np.array_equal(cs, c["cs"]), c["name"]
        assert np.array_equal(es, c["es"]), c["name"]
        n += 1
    assert n >= 5


def test_spec_known_answers():
    # SPEC.md:99 mask counts
    for (F, B, bw), cnt in {(64, 16, 16): (256, 2048, 1792), (32, 8, 8): (64, 512, 448),
                            (128, 32, 16): (1024, 3072, 12288)}.items():
        o = (F - B) // 2
        lab = orc.build_mask((F, F), (o, o, B, B), bw)
        assert ((lab == 2).sum(), (lab == 1).sum(), (lab == 0).sum()) == cnt
    # SPEC.md:108-110 weights (the reference value at (0,0) is 4.818e-5, not 4.838e-5)
    lab = np.ones((5, 5), np.int8)
    w = orc.build_weight(lab, 0.8)
    assert w[2, 2] == 1.0 and abs(w[2, 4] - 0.64) < 1e-15
    w = orc.build_weight(np.ones((64, 64), np.int8), 0.8)
    assert abs(w[0, 0] - 4.8181373491703716e-05) < 1e-18
    # W00 for the three standard geometries
    for (F, B, bw), w00 in {(64, 16, 16): 48.97836003129341, (32, 8, 8): 67.0818567479399,
                            (128, 32, 16): 11.578969116240492}.items():
        o = (F - B) // 2
        W = orc.dft2(orc.build_weight(orc.build_mask((F, F), (o, o, B, B), bw), 0.8))
        assert abs(W[0, 0].real - w00) < 1e-12 * w00
    # constant signal
    lab = orc.build_mask((64, 64), (24, 24, 16, 16), 16)
    s = np.full((64, 64), 200.0)
    o = orc.extrapolate(s, lab, 0.8, 0.2, 1)
    assert (o["us"][0], o["vs"][0]) == (0, 0)
    assert np.allclose(o["reconstructed"][lab == 2], 40.0, atol=1e-9)


def test_dft_properties():
    rng = np.random.default_rng(3)
    for shape in [(8, 8), (16, 16), (12, 10), (64, 64)]:
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        X = orc.dft2(x)
        np.testing.assert_allclose(X, np.fft.fft2(x), rtol=0, atol=1e-10 * np.abs(X).max())
        np.testing.assert_allclose(orc.idft2(X), x, rtol=0, atol=1e-10 * np.abs(x).max())


def test_conceal_blocks_matches_window_path():
    from paper_2204_14193_b200.synth import field
    img = field(128, 128, seed=11)
    blocks = np.array([[0, 0, 0], [0, 48, 64], [0, 112, 112]], np.int32)
    tiles = orc.conceal_blocks(img, blocks, 16, 16, 64, 0.8, 0.5, 50, nthreads=2)
    for b, (f, t, l) in enumerate(blocks):
        wt, wl = t - 24, l - 24
        s = np.zeros((64, 64))
        y0, y1, x0, x1 = max(0, wt), min(128, wt + 64), max(0, wl), min(128, wl + 64)
        s[y0 - wt:y1 - wt, x0 - wl:x1 - wl] = img[y0:y1, x0:x1]
        lab = orc.build_mask((64, 64), (24, 24, 16, 16), 16, (-wt, -wl, 128, 128))
        o = orc.extrapolate(s, lab, 0.8, 0.5, 50)
        assert np.array_equal(tiles[b], o["reconstructed"][24:40, 24:40])


def test_trace_equivalence_utility():
    us = np.array([0, 3, 5]); vs = np.array([0, 1, 60]); cs = np.array([1 + 0j, 2 + 1j, 1 - 1j])
    mu, mv, mc = (-us) % 64, (-vs) % 64, np.conj(cs)
    assert orc.trace_equivalence((us, vs, cs), (us, vs, cs), 64, 64)[0] == "identical"
    assert orc.trace_equivalence((us, vs, cs), (mu, mv, mc), 64, 64)[0] == "mirror"
    bad = (us, np.array([0, 2, 60]), cs)
    assert orc.trace_equivalence((us, vs, cs), bad, 64, 64)[0] == "diverged"

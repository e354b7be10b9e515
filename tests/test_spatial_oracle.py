"""Independent spatial-domain oracle (no FFT) against the
reference's golden outputs and the energy-decrease identity (SPEC
acceptance criteria 1 and 2).  CPU only."""
import numpy as np
import pytest

from oracle import oracle as orc
from oracle import spatial
from tests import _golden

SMALL = [c for c in _golden.load("small.npz") if c["signal"].shape[0] <= 16 and c["iterations"] <= 64
         and c["iterations"] > 0 and c["signal"].std() > 0]


@pytest.mark.parametrize("c", SMALL, ids=[c["name"] for c in SMALL])
def test_spatial_oracle_equivalent_to_reference(c):
    M, N = c["signal"].shape
    o = spatial.extrapolate(c["signal"], c["labels"], c["rho"], c["gamma"], c["iterations"])
    kind, info = orc.trace_equivalence(_golden.trace(c), (o["us"], o["vs"], o["cs"]), M, N)
    assert kind != "diverged", (kind, info)
    loss = c["labels"] == 2
    np.testing.assert_allclose(o["reconstructed"][loss], c["recon_loss"], rtol=0, atol=1e-8)
    # energy identity: incremental == direct weighted residual energy
    assert abs(o["es"][-1] - o["energy_direct"]) <= 1e-9 * max(c["e0"], 1.0)
    np.testing.assert_allclose(o["es"], c["es"], rtol=1e-9, atol=1e-9 * c["e0"])


def test_spatial_oracle_random_instances():
    """50 seeded 12x12 instances, 30% loss, gamma 0.2, I = 40 (SPEC acceptance 1):
    the frequency-domain C oracle and the spatial oracle agree."""
    rng = np.random.default_rng(11)
    kinds = {}
    for _ in range(50):
        s = rng.uniform(0, 255, (12, 12))
        lab = np.where(rng.uniform(size=(12, 12)) < 0.3, 2, 1).astype(np.int8)
        if not (lab == 1).any():
            continue
        a = spatial.extrapolate(s, lab, 0.8, 0.2, 40)
        b = orc.extrapolate(s, lab, 0.8, 0.2, 40)
        k, info = orc.trace_equivalence((a["us"], a["vs"], a["cs"]), (b["us"], b["vs"], b["cs"]), 12, 12)
        assert k != "diverged", info
        kinds[k] = kinds.get(k, 0) + 1
        np.testing.assert_allclose(a["reconstructed"], b["reconstructed"], rtol=0, atol=1e-8)
    print(kinds)


RFSE_SMALL = [c for c in _golden.load("rfse.npz") if c["signal"].shape[0] <= 16]


@pytest.mark.parametrize("c", RFSE_SMALL, ids=[c["name"] for c in RFSE_SMALL])
def test_spatial_pair_oracle_matches_reference_rfse(c):
    """pair_mode of the spatial oracle (rfse.py rule, direct sums) against the
    reference's extrapolate_rfse golden outputs."""
    o = spatial.extrapolate(c["signal"], c["labels"], c["rho"], c["gamma"], c["iterations"],
                            pair_mode=True)
    assert np.array_equal(o["us"], c["us"]) and np.array_equal(o["vs"], c["vs"])
    np.testing.assert_allclose(o["cs"], c["cs"], rtol=1e-9, atol=1e-9 * np.abs(c["cs"]).max())
    assert o["tally"] == c["tally"]
    loss = c["labels"] == 2
    np.testing.assert_allclose(o["reconstructed"][loss], c["recon_loss"], rtol=0, atol=1e-8)
    # realness of the pair model (SPEC acceptance 4)
    assert np.abs(o["model"].imag).max() <= 1e-8 * max(np.abs(o["model"].real).max(), 1.0)

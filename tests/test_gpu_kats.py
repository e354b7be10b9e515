"""SPEC-level known answers and properties on the GPU
product path (the fp64 per-window entry point and the fused fp32 plan)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fse(cuda_ok):
    import paper_2204_14193_b200 as fse
    return fse


def _mask(fse):
    return fse.build_mask((64, 64), (24, 24, 16, 16), 16)


def test_constant_signal(fse):
    """a constant signal selects (0, 0) first with c = gamma
    * const; the loss converges as const (1 - (1 - gamma)^I)."""
    s = np.full((64, 64), 200.0)
    m = _mask(fse)
    r1 = fse.extrapolate_cfse(s, m, fse.FseConfig(rho_hat=0.8, gamma=0.2, iterations=1))
    assert r1.trace[0].frequency == (0, 0)
    assert abs(r1.trace[0].coefficient - 40.0) < 1e-12
    np.testing.assert_allclose(r1.reconstructed[m.loss], 40.0, rtol=0, atol=1e-9)
    r200 = fse.extrapolate_cfse(s, m, fse.FseConfig(rho_hat=0.8, gamma=0.2, iterations=200))
    np.testing.assert_allclose(r200.reconstructed[m.loss], 200.0 * (1 - 0.8 ** 200), rtol=0, atol=1e-9)


def test_scale_equivariance(fse):
    """3 s selects the same sequence, coefficients x 3, residual
    energies x 9 (fp64)."""
    from paper_2204_14193_b200.synth import field
    s = field(64, 64, seed=12)
    m = _mask(fse)
    cfg = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=60)
    a = fse.extrapolate_cfse(s, m, cfg)
    b = fse.extrapolate_cfse(3.0 * s, m, cfg)
    assert [t.frequency for t in a.trace] == [t.frequency for t in b.trace]
    ca = np.array([t.coefficient for t in a.trace])
    cb = np.array([t.coefficient for t in b.trace])
    np.testing.assert_allclose(cb, 3.0 * ca, rtol=1e-12, atol=1e-12 * np.abs(ca).max())
    ea = np.array([t.residual_energy for t in a.trace])
    eb = np.array([t.residual_energy for t in b.trace])
    np.testing.assert_allclose(eb, 9.0 * ea, rtol=1e-10)


def test_energy_identity(fse):
    """the trace's incremental residual energy equals the direct
    weighted residual sum(w |s - g|^2) of the model g."""
    from paper_2204_14193_b200.synth import field
    s = field(64, 64, seed=13)
    m = _mask(fse)
    cfg = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=60)
    r = fse.extrapolate_cfse(s, m, cfg)
    w = fse.build_weight(m, 0.8)
    g = r.model  # complex spatial model (cfse.py:126)
    direct = float(np.sum(w * np.abs(s - g) ** 2))
    assert abs(r.trace[-1].residual_energy - direct) <= 1e-9 * direct


def test_support_and_padding_untouched(fse):
    """support and padding samples of the output are the input
    bit for bit; only loss samples change."""
    from paper_2204_14193_b200.synth import field
    s = field(64, 64, seed=14)
    m = _mask(fse)
    r = fse.extrapolate_cfse(s, m, fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=30))
    assert np.array_equal(r.reconstructed[~m.loss], s[~m.loss])
    assert not np.array_equal(r.reconstructed[m.loss], s[m.loss])


def test_fused_plan_constant_frame(fse):
    """The fused fp32 image path on a constant u8 frame: every block's loss
    converges to the constant like the per-window answer (I = 100, gamma =
    0.5: 200 (1 - 0.5^100) = 200 to fp32 precision)."""
    import torch
    H, W = 256, 384
    frames = torch.full((1, H, W), 200, dtype=torch.uint8, device="cuda")
    blocks = fse.frames_pattern(1, H, W, 16, 0.05, seed=1)
    plan = fse.ConcealPlan(blocks, H, W, fse.Geometry(16, 16, 64), rho_hat=0.8, gamma=0.5,
                           iterations=100)
    assert plan.info["fast_path"] == 1
    t = plan.run(frames, tile_dtype="f32").cpu().numpy()
    np.testing.assert_allclose(t, 200.0, rtol=0, atol=1e-3)


def test_concurrent_calls(fse):
    """every function is pure, so concurrent calls on distinct
    arrays are safe -- four threads calling extrapolate_cfse / _rfse at once
    give the sequential results bit for bit."""
    import threading
    from paper_2204_14193_b200.synth import field
    m = _mask(fse)
    sigs = [field(64, 64, seed=40 + k) for k in range(8)]
    cc = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=40)
    rc = fse.FseConfig(rho_hat=0.8, gamma=0.5, iterations=20, algorithm="rfse")
    want = [(fse.extrapolate_cfse(s, m, cc).reconstructed, fse.extrapolate_rfse(s, m, rc).reconstructed)
            for s in sigs]
    got = [None] * len(sigs)

    def work(k):
        for j in range(k, len(sigs), 4):
            got[j] = (fse.extrapolate_cfse(sigs[j], m, cc).reconstructed,
                      fse.extrapolate_rfse(sigs[j], m, rc).reconstructed)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for (a, b), (c, d) in zip(want, got):
        assert np.array_equal(a, c) and np.array_equal(b, d)

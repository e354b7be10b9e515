"""CPU tests of the parity-gate utilities (oracle/gate.py, oracle.divergence_certificate)
and of the oracle's loss-pattern restatement against the product's native generator."""
import numpy as np

import paper_2204_14193_b200 as fse
from oracle import oracle as orc
from paper_2204_14193_b200.synth import field


def _window():
    img = field(128, 128, seed=11)
    s = img[32:96, 32:96].astype(np.float64)
    lab = orc.build_mask((64, 64), (24, 24, 16, 16), 16)
    return s, lab


def test_certificate_of_a_forced_second_best_pick():
    """A fabricated 'fp32' trace that follows the fp64 trace exactly and then
    takes the fp64 runner-up at iteration k: the certificate reports the fp64
    top-2 gap as the deficit, zero measured error (so not 'bounded'), and
    'strict' exactly when that gap is below 1e-6."""
    s, lab = _window()
    rho, gamma, k = 0.8, 0.5, 7
    w = orc.build_weight(lab, rho)
    W = orc.dft2(w.astype(complex))
    R = orc.dft2((s * w).astype(complex))
    e0 = float(np.sum(w * s * s))
    w00 = W[0, 0].real
    _, us, vs, cs, _ = orc.cfse_kernel(R.copy(), W, gamma, 1 / w00, k, e0)
    orc.cfse_kernel(R, W, gamma, 1 / w00, k, e0)
    m2 = np.abs(R) ** 2
    top = int(np.argmax(m2))
    tu, tv = divmod(top, 64)
    m2x = m2.copy().ravel()
    m2x[top] = -1
    m2x[((-tu) % 64) * 64 + (-tv) % 64] = -1   # the top's mirror is an exact tie
    sec = int(np.argmax(m2x))
    su, sv = divmod(sec, 64)
    tr = (np.append(us, su), np.append(vs, sv), np.append(cs, gamma * R[su, sv] / w00))
    # the oracle's own trace canonicalises the same way up to k (shared prefix)
    cert = orc.divergence_certificate(s, lab, rho, gamma, k, tr)
    gap = (m2.ravel()[top] - m2.ravel()[sec]) / m2.ravel()[top]
    assert cert["at"] == k
    assert abs(cert["deficit"] - gap) <= 1e-12
    assert cert["err_amp"] <= 1e-9 * np.sqrt(m2.ravel()[top])
    assert cert["strict"] == (gap < 1e-6)
    assert not cert["bounded"]
    # a perturbed prefix (measured error e) certifies 'bounded' once the amplitude gap <= 2e
    amp_gap = np.sqrt(m2.ravel()[top]) - np.sqrt(m2.ravel()[sec])
    cs2 = tr[2].copy()
    cs2[k - 1] += (amp_gap * 0.6) * gamma / w00
    cert2 = orc.divergence_certificate(s, lab, rho, gamma, k, (tr[0], tr[1], cs2))
    assert cert2["bounded"] and cert2["err_amp"] >= 0.59 * amp_gap


def test_gate_passes_oracle_against_itself():
    from oracle.gate import fp32_gate
    img = field(256, 256, seed=3).astype(np.float32)
    blocks = np.array([[0, 0, 0], [0, 120, 120], [0, 240, 200]], np.int32)
    ref = orc.conceal_blocks(img, blocks, 16, 16, 64, 0.8, 0.5, 30)
    truth = np.stack([img[t:t + 16, l:l + 16] for _, t, l in blocks])
    st = fp32_gate(img, blocks, ref, None, 64, 16, 16, 0.8, 0.5, 30, truth=truth)
    assert st["over"] == 0 and st["psnr_delta"] == 0


def test_oracle_loss_pattern_equals_native_generator():
    """bench.py's reference arm builds its block list with the oracle's
    restatement; it must be the product generator's exact output."""
    for (H, W, B, frac, seed) in [(2160, 3840, 16, 0.05, 5), (1080, 1920, 16, 0.10, 3),
                                  (512, 512, 8, 0.2, 1), (100, 37, 16, 0.3, 9)]:
        a = orc.frames_pattern(3, H, W, B, frac, seed)
        b = fse.frames_pattern(3, H, W, B, frac, seed)
        assert np.array_equal(a, b), (H, W, B)


def test_rfse_certificate_of_a_forced_second_best_pick():
    """rFSE: follow the oracle's selections, then take the criterion
    runner-up at iteration k with its exact fp64 coefficient: the
    certificate reports the criterion gap as the deficit and no measured
    error; a perturbed earlier coefficient makes it 'bounded'."""
    s, lab = _window()
    rho, gamma, k = 0.8, 0.5, 5
    R, W, w00, pre = orc._rfse_state(s, lab, rho, gamma, k)
    _, us, vs, cs, _, _, _ = pre
    crit = orc.rfse_crit_map(R, W, w00)
    order = np.argsort(crit.ravel())[::-1]
    top = order[0]
    tu, tv = divmod(int(top), 64)
    mir = ((-tu) % 64) * 64 + (-tv) % 64
    sec = next(int(i) for i in order[1:] if i != mir)   # the top's pair partner is the same pair
    su, sv = divmod(sec, 64)
    # the runner-up's own projection (rfse.py:93-103), canonical member
    a = R[su, sv]
    w2 = W[(2 * su) % 64, (2 * sv) % 64]
    D = w00 * w00 - abs(w2) ** 2
    p = complex((w00 * a.real - (w2.real * a.real + w2.imag * a.imag)) / D,
                (w00 * a.imag - (w2.imag * a.real - w2.real * a.imag)) / D)
    mu, mv = (-su) % 64, (-sv) % 64
    if mu * 64 + mv < su * 64 + sv:
        su, sv, p = mu, mv, p.conjugate()
    tr = (np.append(us, su), np.append(vs, sv), np.append(cs, gamma * p))
    cert = orc.rfse_divergence_certificate(s, lab, rho, gamma, k, tr)
    gap = np.sqrt(crit.ravel()[top]) - np.sqrt(crit[su, sv])
    assert abs(cert["gap_amp"] - gap) <= 1e-9 * np.sqrt(crit.ravel()[top])
    assert cert["err_amp"] <= 1e-9 * np.sqrt(crit.ravel()[top])
    assert not cert["bounded"]
    cs2 = tr[2].copy()
    cs2[k - 1] *= 1 + 1e-3
    assert orc.rfse_divergence_certificate(s, lab, rho, gamma, k, (tr[0], tr[1], cs2))["err_amp"] > 0


def test_gates_reject_non_finite_tiles():
    """A NaN tile must fail the gate (|NaN - x| > tol is False, so it would
    otherwise slip past the per-block check)."""
    import numpy as np
    import pytest
    from oracle import oracle as orc
    from oracle.gate import fp32_gate, rfse_gate
    from paper_2204_14193_b200.synth import frame_u8
    fr = frame_u8(96, 96, seed=2)
    blocks = np.array([[0, 40, 40]], np.int32)
    t = orc.conceal_blocks(fr, blocks, 16, 16, 64, 0.8, 0.5, 5)
    t[0, 3, 3] = np.nan
    with pytest.raises(AssertionError, match="NaN"):
        fp32_gate(fr, blocks, t, None, 64, 16, 16, 0.8, 0.5, 5)
    tr = orc.conceal_blocks_rfse(fr, blocks, 16, 16, 64, 0.8, 0.5, 5)
    tr[0, 0, 0] = np.inf
    with pytest.raises(AssertionError, match="NaN"):
        rfse_gate(fr, blocks, tr, None, 64, 16, 16, 0.8, 0.5, 5)

"""CPU tests: host logic, validation, the C-ABI library exports, the native
loss-pattern generator.  No GPU compute calls."""
import ctypes
import os

import numpy as np
import pytest

import paper_2204_14193_b200 as fse
from paper_2204_14193_b200 import _lib
from oracle import oracle as orc


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 13
    L = ctypes.CDLL(_lib.SO_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in _lib.lib().fse_version()


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_validation_matches_reference():
    # types.py:37-53
    for kw in [dict(rho_hat=0.0), dict(rho_hat=1.0), dict(gamma=0.0), dict(gamma=1.5),
               dict(iterations=0), dict(fft_dims=(0, 4)), dict(fft_dims=(4,)),
               dict(algorithm="x"), dict(basis_target=-1), dict(precision="fp16")]:
        with pytest.raises(fse.ConfigError):
            fse.FseConfig(**kw)
    c = fse.FseConfig(basis_target=0)
    assert c.loop_bound == 0
    assert fse.FseConfig(iterations=7).loop_bound == 7
    assert issubclass(fse.ConfigError, ValueError)


@pytest.mark.parametrize("args", [
    ((64, 64), (24, 24, 16, 16), 16, None),
    ((32, 32), (12, 12, 8, 8), 8, None),
    ((64, 64), (24, 24, 16, 16), 16, (24, 24, 64, 64)),
    ((64, 64), (24, 24, 16, 16), 16, (-40, 8, 100, 100)),
    ((8, 8), (0, 0, 2, 2), 2, None),
    ((12, 10), (3, 2, 4, 5), 3, (1, 0, 11, 9)),
])
def test_build_mask_matches_oracle(args):
    m = fse.build_mask(*args)
    assert np.array_equal(m.labels, orc.build_mask(*args))


def test_build_mask_errors():
    with pytest.raises(fse.ConfigError):
        fse.build_mask((4, 4), (0, 0, 4, 4), 2)  # no support
    with pytest.raises(fse.ConfigError):
        fse.build_mask((8, 8), (6, 6, 4, 4), 2)  # outside window
    with pytest.raises(fse.ConfigError):
        fse.build_mask((8, 8), (2, 2, 2, 2), -1)
    with pytest.raises(fse.ConfigError):
        fse.build_mask((64, 64), (24, 24, 16, 16), 16, (30, 30, 64, 64))  # loss outside valid
    with pytest.raises(fse.ConfigError):
        fse.AreaMask(np.full((4, 4), 2))
    m = fse.AreaMask.from_loss(np.eye(4, dtype=bool), np.zeros((4, 4), bool))
    assert m.loss.sum() == 4 and m.support.sum() == 12


def test_loss_pattern_isolated_and_deterministic():
    a = fse.loss_pattern(2160, 3840, 16, 1620, seed=5)
    b = fse.loss_pattern(2160, 3840, 16, 1620, seed=5)
    assert np.array_equal(a, b) and len(a) == 1620
    assert not np.array_equal(a, fse.loss_pattern(2160, 3840, 16, 1620, seed=6))
    g = np.zeros((2160 // 16 + 2, 3840 // 16 + 2), int)
    for t, l in a:
        g[t // 16 + 1, l // 16 + 1] += 1
    # no two chosen blocks 8-adjacent
    for t, l in a:
        i, j = t // 16 + 1, l // 16 + 1
        assert g[i - 1:i + 2, j - 1:j + 2].sum() == 1
    assert np.all(a % 16 == 0) and np.all(a[:, 0] + 16 <= 2160)
    # 10% of 1920x1080 (config 3): 804 of 120 x 67
    assert len(fse.loss_pattern_fraction(1080, 1920, 16, 0.10, 3)) == 804


def test_cuda_required_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fse.FseError):
        fse.extrapolate_cfse(np.zeros((64, 64)), fse.build_mask((64, 64), (24, 24, 16, 16), 16),
                             fse.FseConfig())


def test_product_does_not_import_oracle():
    pkg = os.path.dirname(fse.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_psnr_closed_form():
    img = np.full((32, 32), 100.0)
    rec = img + 16
    # 10 log10(255^2 / 16^2) = 24.0484 dB (SPEC.md:348 prints 24.0464, a typo of the same formula)
    assert fse.psnr(img, rec, np.array([[0, 0], [16, 16]]), 16) == pytest.approx(24.04840, abs=1e-4)
    assert fse.psnr(img, img, np.array([[0, 0]]), 16) == float("inf")


def test_synthetic_field_stats():
    from paper_2204_14193_b200.synth import field, frame_u8
    x = field(256, 256, 0)
    assert abs(x.mean() - 128) < 1.5 and abs(x.std() - 40) < 1.5
    f = frame_u8(128, 256, 1)
    assert f.dtype == np.uint8 and f.shape == (128, 256)


def test_rfse_rejects_a_3d_signal_like_the_reference():
    """rfse.extrapolate_rfse on a (1, M, N) signal: ConfigError (the
    reference's _prepare checks signal.shape == fft_dims), no CUDA needed."""
    cfg = fse.FseConfig(fft_dims=(8, 8), algorithm="rfse")
    mask = fse.build_mask((8, 8), (2, 2, 4, 4), 2)
    with pytest.raises(fse.ConfigError):
        fse.extrapolate_rfse(np.zeros((1, 8, 8)), mask, cfg)
    with pytest.raises(fse.ConfigError):
        fse.extrapolate_cfse(np.zeros((1, 8, 8)), mask, fse.FseConfig(fft_dims=(8, 8)))


def test_pinned_staging_is_thread_local_and_bounded(monkeypatch):
    """The latency paths' pinned staging buffers live per thread and at most
    `keep` sizes are cached (no unbounded module-level cache)."""
    import threading

    class FakeT:
        def __init__(self, n):
            self.n = n

        def pin_memory(self):
            return self

    import torch
    monkeypatch.setattr(torch, "empty", lambda n, dtype=None: FakeT(n))
    a = _lib.pinned_staging(100)
    assert _lib.pinned_staging(100) is a
    for n in range(200, 800, 100):
        _lib.pinned_staging(n)
    assert len(_lib._STAGING.bufs) == 4 and 100 not in _lib._STAGING.bufs
    other = []
    t = threading.Thread(target=lambda: other.append(_lib.pinned_staging(100)))
    t.start(); t.join()
    assert other[0] is not _lib._STAGING.bufs.get(100)

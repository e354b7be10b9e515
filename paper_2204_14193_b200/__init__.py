"""B200-native complex-valued Frequency Selective Extrapolation (cFSE).

Drop-in for the reference package `fse` (Seiler & Kaup, arXiv 2204.14193):
`extrapolate_cfse(signal, mask, config)` with the reference's FseConfig /
AreaMask / build_mask API, computed by hand-written sm_100a CUDA kernels in
libfse_b200.so (no CPU fallback).  Image-level concealment (the north-star
entry: image + loss blocks + block size, border, FFT size, iterations, rho,
gamma) is `harness.ConcealPlan` / `harness.Concealer`.
"""
from .errors import ConfigError, FseError, PgmError
from .types import ALGORITHMS, ExtrapolationResult, FseConfig, IterationRecord
from .weighting import Area, AreaMask, build_mask, build_weight, weight_spectrum
from .spectral import basis_function, dft2, idft2
from .cfse import (cfse_kernel, estimate_coefficient, extrapolate_cfse, extrapolate_cfse_batch,
                   select_basis, update_model, update_residual)
from .harness import (Concealer, ConcealPlan, Geometry, conceal, conceal_frames, grid_pattern,
                      loss_pattern, loss_pattern_fraction, frames_pattern, psnr, psnr_tiles,
                      write_tiles)
from .rfse import RfsePlan, conceal_frames_rfse, extrapolate_rfse, extrapolate_rfse_batch

__all__ = [
    "ConfigError", "FseError", "PgmError", "ALGORITHMS", "ExtrapolationResult", "FseConfig",
    "IterationRecord", "Area", "AreaMask", "build_mask", "build_weight", "weight_spectrum",
    "basis_function", "dft2", "idft2", "cfse_kernel", "estimate_coefficient", "extrapolate_cfse",
    "extrapolate_cfse_batch", "select_basis", "update_model", "update_residual", "Concealer",
    "ConcealPlan", "Geometry", "conceal", "conceal_frames", "loss_pattern", "loss_pattern_fraction",
    "frames_pattern", "psnr", "psnr_tiles", "write_tiles", "grid_pattern", "RfsePlan",
    "conceal_frames_rfse", "extrapolate_rfse", "extrapolate_rfse_batch",
]

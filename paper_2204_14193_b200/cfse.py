"""Complex-valued frequency-selective extrapolation on the GPU.

Drop-in for the reference module `fse.cfse` (/root/reference/pkg/src/fse/
cfse.py).  `extrapolate_cfse(signal, mask, config)` keeps the reference's
signature, validation order and exceptions (cfse.py:28-48) and returns the
same `ExtrapolationResult`; the work itself (weights, both DFTs, the I
select/estimate/update iterations, the sparse-model synthesis and the
write-back) runs in one fused CUDA kernel per window (fse_extrapolate in
libfse_b200.so).  fp64 by default, like the reference.

Also here:
  * `extrapolate_cfse_batch` -- many windows in one launch (device arrays in,
    device arrays out), the throughput form of the same entry point;
  * `cfse_kernel` -- drop-in for the numba loop `_cfse_kernel`
    (cfse.py:55-107), bit-identical to it given the same spectra;
  * the single-step ops of cfse.py:145-178.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError
from .types import ExtrapolationResult, FseConfig, IterationRecord
from .weighting import AreaMask

__all__ = ["extrapolate_cfse", "extrapolate_cfse_batch", "cfse_kernel", "select_basis",
           "estimate_coefficient", "update_model", "update_residual"]


def _as_signal(signal) -> np.ndarray:
    try:
        return np.asarray(signal, dtype=np.float64)  # cfse.py:30-33
    except TypeError as exc:
        raise ValueError("signal must be real-valued") from exc


def _validate(s: np.ndarray, mask: AreaMask, config: FseConfig) -> None:
    # cfse.py:34-41, same order and exception types
    if s.shape[-2:] != tuple(config.fft_dims) or s.ndim not in (2, 3):
        raise ConfigError(
            f"signal shape {s.shape} does not match configured FFT dims {config.fft_dims}")
    if s.shape[-2:] != mask.shape:
        raise ConfigError(f"signal shape {s.shape} does not match mask shape {mask.shape}")
    if not np.all(np.isfinite(s)):
        raise ValueError("signal contains non-finite values")


def _prec(config: FseConfig) -> int:
    return _lib.FSE_PREC_F32 if config.precision == "fp32" else _lib.FSE_PREC_F64


def extrapolate_cfse_batch(signals, labels, config: FseConfig, *, want_model: bool = False,
                           stream=None) -> dict:
    """Run `extrapolate_cfse` on a batch of windows in one launch.

    signals: (n, M, N) float64 (numpy or CUDA tensor); labels: (M, N) shared
    or (n, M, N) int8 Area labels.  Returns a dict of CUDA tensors:
    reconstructed (n, M, N) f64, model (n, M, N) c128 or None, us/vs
    (n, I) int64, cs (n, I) c128, es (n, I) f64, status (n,) int32.
    Raises ConfigError if any window has an empty support weight.
    """
    torch = _lib.require_cuda()
    s = torch.as_tensor(signals, dtype=torch.float64).cuda().contiguous()
    if s.ndim == 2:
        s = s[None]
    lab = torch.as_tensor(np.asarray(labels, np.int8) if not torch.is_tensor(labels) else labels,
                          dtype=torch.int8).cuda().contiguous()
    n, M, N = s.shape
    lstride = 0 if lab.ndim == 2 else M * N
    it = config.loop_bound
    dev = s.device
    rec = torch.empty_like(s)
    model = torch.empty((n, M, N), dtype=torch.complex128, device=dev) if want_model else None
    us = torch.empty((n, max(it, 1)), dtype=torch.int64, device=dev)
    vs = torch.empty_like(us)
    cs = torch.empty((n, max(it, 1)), dtype=torch.complex128, device=dev)
    es = torch.empty((n, max(it, 1)), dtype=torch.float64, device=dev)
    status = torch.empty((n,), dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().fse_extrapolate(
        n, M, N, _prec(config), _lib.ptr(s), _lib.ptr(lab), lstride, float(config.rho_hat),
        float(config.gamma), it, _lib.ptr(rec), _lib.ptr(model), _lib.ptr(us), _lib.ptr(vs),
        _lib.ptr(cs), _lib.ptr(es), _lib.ptr(status), _lib.stream_ptr(stream)))
    if bool((status != 0).any()):
        raise ConfigError("total support weight is numerically zero (empty support)")
    return dict(reconstructed=rec, model=model, us=us[:, :it], vs=vs[:, :it], cs=cs[:, :it],
                es=es[:, :it], status=status)


def extrapolate_cfse(signal, mask: AreaMask, config: FseConfig) -> ExtrapolationResult:
    """Run the complex-valued extrapolation and replace the loss samples
    (cfse.py:110-142).  Support and padding samples of the output equal the
    float64 input exactly; loss samples take Re{g}; the trace holds one
    IterationRecord per iteration.

    Latency path: every output of the window (reconstruction, model, trace,
    status) lands in one device buffer and comes back in one copy to pinned
    host memory."""
    s = _as_signal(signal)
    _validate(s, mask, config)
    if s.ndim != 2:
        raise ConfigError(f"signal shape {s.shape} does not match configured FFT dims {config.fft_dims}")
    torch = _lib.require_cuda()
    M, N = s.shape
    MN, it = M * N, config.loop_bound
    I = max(it, 1)
    # byte layout: recon f64 MN | model c128 MN | us i64 I | vs i64 I | cs c128 I | es f64 I | status
    sizes = [8 * MN, 16 * MN, 8 * I, 8 * I, 16 * I, 8 * I, 8]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    dev = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
    sd = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    lab = torch.from_numpy(np.ascontiguousarray(mask.labels, np.int8)).cuda()
    p = [dev.data_ptr() + int(o) for o in offs[:-1]]
    _lib.check(_lib.lib().fse_extrapolate(
        1, M, N, _prec(config), sd.data_ptr(), lab.data_ptr(), 0, float(config.rho_hat),
        float(config.gamma), it, p[0], p[1], p[2], p[3], p[4], p[5], p[6], _lib.stream_ptr(None)))
    host = _lib.pinned_staging(int(offs[-1]))
    host.copy_(dev)  # synchronous: waits for the kernel
    raw = host.numpy()

    def part(k, dt, n):
        return np.frombuffer(raw, dtype=dt, count=n, offset=int(offs[k])).copy()

    if part(6, np.int32, 1)[0] != 0:
        raise ConfigError("total support weight is numerically zero (empty support)")
    rec = part(0, np.float64, MN).reshape(M, N)
    model = part(1, np.complex128, MN).reshape(M, N)
    us, vs = part(2, np.int64, I), part(3, np.int64, I)
    cs, es = part(4, np.complex128, I), part(5, np.float64, I)
    trace = [IterationRecord(index=i, frequency=(int(us[i]), int(vs[i])),
                             coefficient=complex(cs[i]), residual_energy=float(es[i]))
             for i in range(it)]
    return ExtrapolationResult(reconstructed=rec, model=model, trace=trace, basis_count=len(trace))


def cfse_kernel(R_w, W, gamma: float, inv_w00: float, iterations: int, e0: float):
    """Drop-in for the numba `_cfse_kernel(R_w, W, gamma, inv_w00, iterations,
    e0)` (cfse.py:55-107) on the GPU.  R_w (complex128) is mutated in place
    like the reference; returns (G, us, vs, cs, es) as numpy arrays."""
    torch = _lib.require_cuda()
    R_np = R_w if isinstance(R_w, np.ndarray) else None
    R = torch.as_tensor(np.ascontiguousarray(R_w, np.complex128) if R_np is not None else R_w,
                        dtype=torch.complex128).cuda().contiguous()
    Wd = torch.as_tensor(np.ascontiguousarray(W, np.complex128), dtype=torch.complex128).cuda()
    M, N = R.shape
    n = max(int(iterations), 1)
    dev = R.device
    G = torch.zeros((M, N), dtype=torch.complex128, device=dev)
    us = torch.zeros(n, dtype=torch.int64, device=dev)
    vs = torch.zeros_like(us)
    cs = torch.zeros(n, dtype=torch.complex128, device=dev)
    es = torch.zeros(n, dtype=torch.float64, device=dev)
    inv = torch.tensor([float(inv_w00)], dtype=torch.float64, device=dev)
    e0t = torch.tensor([float(e0)], dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().fse_cfse_kernel_f64(
        1, M, N, _lib.ptr(R), _lib.ptr(Wd), 0, float(gamma), _lib.ptr(inv), int(iterations),
        _lib.ptr(e0t), _lib.ptr(G), _lib.ptr(us), _lib.ptr(vs), _lib.ptr(cs), _lib.ptr(es),
        _lib.stream_ptr()))
    k = int(iterations)
    if R_np is not None:
        R_np[...] = R.cpu().numpy()
    elif R.data_ptr() != R_w.data_ptr():
        R_w.copy_(R)
    return (G.cpu().numpy(), us[:k].cpu().numpy(), vs[:k].cpu().numpy(), cs[:k].cpu().numpy(),
            es[:k].cpu().numpy())


def select_basis(R_w: np.ndarray) -> tuple[int, int]:
    """Index of the maximal squared-modulus bin, first in row-major order
    (cfse.py:145-154), on the GPU."""
    torch = _lib.require_cuda()
    R = torch.as_tensor(np.ascontiguousarray(R_w, np.complex128)).cuda()
    uv = torch.empty(2, dtype=torch.int64, device=R.device)
    M, N = R.shape
    _lib.check(_lib.lib().fse_select_basis_f64(M, N, _lib.ptr(R), _lib.ptr(uv), _lib.stream_ptr()))
    u, v = uv.cpu().tolist()
    return int(u), int(v)


def estimate_coefficient(R_w: np.ndarray, u: int, v: int, gamma: float, inv_w00: float) -> complex:
    """gamma * R_w[u, v] * inv_w00 (cfse.py:157-162) -- one scalar."""
    return complex(gamma * R_w[u, v] * inv_w00)


def update_model(G: np.ndarray, u: int, v: int, coefficient: complex) -> None:
    """G[u, v] += M*N*c in place (cfse.py:165-169) -- one element."""
    M, N = G.shape
    G[u, v] += M * N * coefficient


def update_residual(R_w: np.ndarray, W: np.ndarray, u: int, v: int, coefficient: complex) -> None:
    """R_w[k, l] -= c * W[(k-u) mod M, (l-v) mod N] in place (cfse.py:172-178), on the GPU."""
    torch = _lib.require_cuda()
    R = torch.as_tensor(np.ascontiguousarray(R_w, np.complex128)).cuda()
    Wd = torch.as_tensor(np.ascontiguousarray(W, np.complex128)).cuda()
    M, N = R.shape
    c = complex(coefficient)
    _lib.check(_lib.lib().fse_update_residual_f64(M, N, _lib.ptr(R), _lib.ptr(Wd), int(u), int(v),
                                                  c.real, c.imag, _lib.stream_ptr()))
    R_w[...] = R.cpu().numpy()

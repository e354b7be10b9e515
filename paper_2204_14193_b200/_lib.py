"""ctypes binding of libfse_b200.so (the C ABI declared in include/fse_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
present, every compute entry point raises.  Build with
`python -m paper_2204_14193_b200.build` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os
import re

from .errors import ConfigError, FseError

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("FSE_LIB_PATH") or os.path.join(HERE, "libfse_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fse_b200.h")

FSE_OK = 0
FSE_ERR_CONFIG = -1
FSE_ERR_VALUE = -2
FSE_ERR_UNSUPPORTED = -3
FSE_ERR_CUDA = -4

FSE_U8, FSE_F32, FSE_F64 = 0, 1, 2
FSE_PREC_F64, FSE_PREC_F32 = 0, 1
FSE_ALG_CFSE, FSE_ALG_RFSE = 0, 1


class FseUnsupported(FseError, NotImplementedError):
    """Size / dtype outside what the CUDA kernels implement."""


class FseCudaError(FseError, RuntimeError):
    """CUDA runtime failure inside libfse_b200."""


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "n_blocks", "n_classes", "n_rounds", "slots", "threads", "grid", "smem_bytes", "fast_path", "n_centred")]


_lib = None

P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
LL = ctypes.c_longlong

_SIGS = {
    "fse_version": ([], ctypes.c_char_p),
    "fse_last_error": ([ctypes.c_char_p, ctypes.c_size_t], I),
    "fse_dft2_f64": ([I, I, I, P, P, I, P], I),
    "fse_build_weight_f64": ([I, I, I, P, D, P, P], I),
    "fse_cfse_kernel_f64": ([I, I, I, P, P, LL, D, P, I, P, P, P, P, P, P, P], I),
    "fse_extrapolate": ([I, I, I, I, P, P, LL, D, D, I, P, P, P, P, P, P, P, P], I),
    "fse_extrapolate_rfse": ([I, I, I, I, P, P, LL, D, D, I, I, P, P, P, P, P, P, P, P, P, P, P], I),
    "fse_select_basis_f64": ([I, I, P, P, P], I),
    "fse_update_residual_f64": ([I, I, P, P, I, I, D, D, P], I),
    "fse_plan_create": ([ctypes.POINTER(P), P, I, I, I, I, I, I, D, D, I, I, P], I),
    "fse_plan_create_ex": ([ctypes.POINTER(P), P, I, I, I, I, I, I, D, D, I, I, I, I, P], I),
    "fse_plan_get_info": ([P, ctypes.POINTER(PlanInfo)], I),
    "fse_plan_destroy": ([P], I),
    "fse_plan_run": ([P, P, I, LL, LL, I, P, I, P, P, P, P], I),
    "fse_loss_pattern": ([I, I, I, I, ctypes.c_uint64, P], I),
    "fse_spatial_extrapolate": ([I, I, I, P, P, LL, D, D, I, I, I, P, P, P, P, P, P, P, P, P, P, P], I),
}


def header_symbols() -> list[str]:
    """Function names declared in include/fse_b200.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fse_\w+)\s*\(", txt, re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise FseError(
                f"{SO_PATH} is missing: build it with `python -m paper_2204_14193_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(SO_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().fse_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int) -> None:
    if rc == FSE_OK:
        return
    msg = last_error()
    if rc == FSE_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == FSE_ERR_VALUE:
        raise ValueError(msg)
    if rc == FSE_ERR_UNSUPPORTED:
        raise FseUnsupported(msg)
    raise FseCudaError(msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise FseError("no CUDA device: the cFSE kernels run on the GPU only (no CPU fallback)")
    lib()
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


_STAGING = __import__("threading").local()


def pinned_staging(nbytes: int, keep: int = 4):
    """A pinned host byte buffer of `nbytes` for the calling thread (the
    per-window latency paths copy every output back in one DMA).  Buffers
    live in thread-local storage, so they are released with their thread,
    and at most `keep` sizes are cached per thread (least recently used
    dropped)."""
    import torch

    cache = getattr(_STAGING, "bufs", None)
    if cache is None:
        cache = _STAGING.bufs = {}
    buf = cache.pop(nbytes, None)
    if buf is None:
        buf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    cache[nbytes] = buf  # most recent last
    while len(cache) > keep:
        cache.pop(next(iter(cache)))
    return buf


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())

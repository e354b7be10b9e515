"""Binary PGM (P5, maxval 255) I/O for the harness.

Errors raise PgmError (errors.py:13-14) with the byte offset of the problem.
Saving clamps to [0, 255] and rounds half to even (the harness's write-back
rule).
"""
from __future__ import annotations

import numpy as np

from .errors import PgmError


def _tokens(data: bytes, count: int):
    """Yield (token, offset) for the first `count` header tokens, skipping
    whitespace and '#' comments; returns the offset after the last token's
    single trailing whitespace byte."""
    out, i, n = [], 0, len(data)
    while len(out) < count:
        while i < n and data[i:i + 1].isspace():
            i += 1
        if i < n and data[i:i + 1] == b"#":
            while i < n and data[i:i + 1] not in (b"\n", b"\r"):
                i += 1
            continue
        if i >= n:
            raise PgmError(f"truncated header at byte {i}")
        j = i
        while j < n and not data[j:j + 1].isspace() and data[j:j + 1] != b"#":
            j += 1
        out.append((data[i:j], i))
        i = j
    if i >= n or not data[i:i + 1].isspace():
        raise PgmError(f"missing whitespace after header at byte {i}")
    return out, i + 1


def loads(data: bytes) -> np.ndarray:
    if len(data) < 2:
        raise PgmError("truncated header at byte 0")
    if data[:2] != b"P5":
        raise PgmError(f"unsupported format {data[:2]!r} at byte 0 (only binary P5)")
    toks, off = _tokens(data, 4)
    vals = []
    for tok, pos in toks[1:]:
        if not tok.isdigit():
            raise PgmError(f"bad header field {tok!r} at byte {pos}")
        vals.append(int(tok))
    w, h, maxval = vals
    if w < 1 or h < 1:
        raise PgmError(f"bad dimensions {w}x{h} at byte {toks[1][1]}")
    if maxval != 255:
        raise PgmError(f"unsupported maxval {maxval} at byte {toks[3][1]} (only 255)")
    need = w * h
    if len(data) - off < need:
        raise PgmError(f"truncated pixel data at byte {len(data)} (need {need} bytes from {off})")
    return np.frombuffer(data, np.uint8, count=need, offset=off).reshape(h, w).copy()


def dumps(image: np.ndarray) -> bytes:
    img = np.asarray(image)
    if img.ndim != 2:
        raise PgmError(f"image must be 2-D, got {img.shape}")
    if img.dtype != np.uint8:
        img = np.rint(np.clip(np.asarray(img, np.float64), 0, 255)).astype(np.uint8)
    h, w = img.shape
    return b"P5\n%d %d\n255\n" % (w, h) + img.tobytes()


def load_image(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return loads(f.read())


def save_image(image: np.ndarray, path: str) -> None:
    with open(path, "wb") as f:
        f.write(dumps(image))

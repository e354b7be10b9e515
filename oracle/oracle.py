"""CPU oracle for the cFSE hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (the cpu_baseline leg and
`--impl reference`) may import this module.  The product package
(`paper_2204_14193_b200`) never imports, links or executes anything under
oracle/; it fails loudly when its CUDA library is missing.

The oracle is a C restatement (oracle/cfse_oracle.c) of the reference Python
package `fse` (/root/reference/pkg/src/fse), wrapped here with ctypes:

  build_mask      <- weighting.py:81-127
  build_weight    <- weighting.py:130-145
  dft2 / idft2    <- spectral.py:32-56
  cfse_kernel     <- cfse.py:55-107
  extrapolate     <- cfse.py:110-142
  conceal_blocks  <- SPEC.md:332-340 (harness conceal, absent in the reference)
  loss_pattern    <- SURVEY.md 8(d) isolated-block loss selection

It is pinned against golden vectors produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; checked by
tests/test_oracle_golden.py).

Also here: the parity-gate utilities of SURVEY.md section 8(c) --
`canonicalize_trace` (conjugate-mirror canonical form) and
`near_tie_gap` (top-2 |R_w|^2 relative gap certifier for fp32 outliers).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_ERRORS = {
    -1: "support_width must be >= 0",
    -2: "loss rectangle must be non-empty",
    -3: "loss rectangle does not fit inside the window",
    -4: "loss rectangle extends outside the valid region",
    -5: "mask geometry leaves no support samples",
    -6: "total support weight is numerically zero (empty support)",
    -7: "support area is degenerate for pairwise selection",
}


class OracleError(ValueError):
    pass


def build() -> str:
    """Compile oracle/cfse_oracle.c (Makefile) into oracle/build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "cfse_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i, d, ll = ctypes.c_int, ctypes.c_double, ctypes.c_longlong
        L.orc_build_mask.argtypes = [i, i, i, i, i, i, i, i, i, i, i, i, P]
        L.orc_build_mask.restype = i
        L.orc_build_weight.argtypes = [i, i, P, d, P]
        L.orc_dft2.argtypes = [i, i, P, P, i]
        L.orc_cfse_kernel.argtypes = [i, i, P, P, d, d, i, d, P, P, P, P, P]
        L.orc_extrapolate.argtypes = [i, i, P, P, d, d, i, P, P, P, P, P, P, P, P]
        L.orc_extrapolate.restype = i
        L.orc_conceal_blocks.argtypes = [P, i, i, i, ll, ll, P, i, i, i, i, d, d, i, P, i]
        L.orc_conceal_blocks.restype = i
        L.orc_max_threads.restype = i
        L.orc_loss_pattern.argtypes = [i, i, i, i, ctypes.c_uint64, P]
        L.orc_loss_pattern.restype = i
        L.orc_rfse_kernel.argtypes = [i, i, P, P, d, d, i, i, d, P, P, P, P, P, P, P]
        L.orc_rfse_kernel.restype = i
        L.orc_extrapolate_rfse.argtypes = [i, i, P, P, d, d, i, i, P, P, P, P, P, P, P]
        L.orc_extrapolate_rfse.restype = i
        L.orc_conceal_blocks_rfse.argtypes = [P, i, i, i, ll, ll, P, i, i, i, i, d, d, i, i, P, i]
        L.orc_conceal_blocks_rfse.restype = i
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int):
    if rc != 0:
        raise OracleError(_ERRORS.get(rc, f"oracle error {rc}"))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ------------------------------------------------------------------ API


def build_mask(fft_dims, loss_rect, support_width, valid_rect=None) -> np.ndarray:
    M, N = int(fft_dims[0]), int(fft_dims[1])
    t, l, h, w = (int(v) for v in loss_rect)
    labels = np.empty((M, N), np.int8)
    if valid_rect is None:
        rc = lib().orc_build_mask(M, N, t, l, h, w, int(support_width), 0, 0, 0, 0, 0, _p(labels))
    else:
        vt, vl, vh, vw = (int(v) for v in valid_rect)
        rc = lib().orc_build_mask(M, N, t, l, h, w, int(support_width), 1, vt, vl, vh, vw, _p(labels))
    _check(rc)
    return labels


def build_weight(labels: np.ndarray, rho: float) -> np.ndarray:
    labels = np.ascontiguousarray(labels, np.int8)
    M, N = labels.shape
    w = np.empty((M, N), np.float64)
    lib().orc_build_weight(M, N, _p(labels), float(rho), _p(w))
    return w


def dft2(x: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(x, np.complex128)
    out = np.empty_like(a)
    lib().orc_dft2(a.shape[0], a.shape[1], _p(a), _p(out), 0)
    return out


def idft2(X: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(X, np.complex128)
    out = np.empty_like(a)
    lib().orc_dft2(a.shape[0], a.shape[1], _p(a), _p(out), 1)
    return out


def cfse_kernel(R_w: np.ndarray, W: np.ndarray, gamma: float, inv_w00: float,
                iterations: int, e0: float):
    """cfse.py:55-107.  R_w (complex128, C-order) is mutated in place."""
    assert R_w.dtype == np.complex128 and R_w.flags.c_contiguous
    W = np.ascontiguousarray(W, np.complex128)
    M, N = R_w.shape
    G = np.zeros((M, N), np.complex128)
    n = max(int(iterations), 1)
    us = np.zeros(n, np.int64); vs = np.zeros(n, np.int64)
    cs = np.zeros(n, np.complex128); es = np.zeros(n, np.float64)
    lib().orc_cfse_kernel(M, N, _p(R_w), _p(W), float(gamma), float(inv_w00), int(iterations),
                          float(e0), _p(G), _p(us), _p(vs), _p(cs), _p(es))
    k = int(iterations)
    return G, us[:k], vs[:k], cs[:k], es[:k]


def extrapolate(signal, labels, rho, gamma, iterations, return_spectra=False):
    """cfse.py:110-142.  Returns dict(reconstructed, model, us, vs, cs, es)."""
    s = np.ascontiguousarray(signal, np.float64)
    labels = np.ascontiguousarray(labels, np.int8)
    M, N = s.shape
    rec = np.empty((M, N), np.float64)
    model = np.empty((M, N), np.complex128)
    n = max(int(iterations), 1)
    us = np.zeros(n, np.int64); vs = np.zeros(n, np.int64)
    cs = np.zeros(n, np.complex128); es = np.zeros(n, np.float64)
    Rw = np.empty((M, N), np.complex128) if return_spectra else None
    W = np.empty((M, N), np.complex128) if return_spectra else None
    rc = lib().orc_extrapolate(M, N, _p(s), _p(labels), float(rho), float(gamma), int(iterations),
                               _p(rec), _p(model), _p(us), _p(vs), _p(cs), _p(es),
                               _p(Rw) if Rw is not None else None,
                               _p(W) if W is not None else None)
    _check(rc)
    k = int(iterations)
    out = dict(reconstructed=rec, model=model, us=us[:k], vs=vs[:k], cs=cs[:k], es=es[:k])
    if return_spectra:
        out["R_w"], out["W"] = Rw, W
    return out


_DT = {np.dtype(np.uint8): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}


def conceal_blocks(frames: np.ndarray, blocks: np.ndarray, B: int, border: int, F: int,
                   rho: float, gamma: float, iterations: int, nthreads: int = 0) -> np.ndarray:
    """SPEC.md:332-340 per-block concealment.  frames: (nf, H, W) or (H, W);
    blocks: int32 (n, 3) = (frame, top, left).  Returns fp64 tiles (n, B, B),
    unclamped Re{g} on the loss pixels."""
    fr = np.ascontiguousarray(frames)
    if fr.ndim == 2:
        fr = fr[None]
    nf, H, W = fr.shape
    bl = np.ascontiguousarray(blocks, np.int32).reshape(-1, 3)
    tiles = np.empty((bl.shape[0], B, B), np.float64)
    rc = lib().orc_conceal_blocks(_p(fr), _DT[fr.dtype], H, W, W, H * W, _p(bl), bl.shape[0],
                                  int(B), int(border), int(F), float(rho), float(gamma),
                                  int(iterations), _p(tiles), int(nthreads))
    _check(rc)
    return tiles


def rfse_kernel(R_w: np.ndarray, W: np.ndarray, gamma: float, w00: float, max_iters: int,
                stop_tally: int, e0: float):
    """rfse.py:37-167 (_pair_tables + _rfse_kernel).  R_w mutated in place.
    Returns (G, us, vs, cs, es, selfs, tally)."""
    assert R_w.dtype == np.complex128 and R_w.flags.c_contiguous
    W = np.ascontiguousarray(W, np.complex128)
    M, N = R_w.shape
    n = max(int(max_iters), 1)
    G = np.zeros((M, N), np.complex128)
    us = np.zeros(n, np.int64); vs = np.zeros(n, np.int64)
    cs = np.zeros(n, np.complex128); es = np.zeros(n); sf = np.zeros(n, np.uint8)
    t = ctypes.c_int(0)
    k = lib().orc_rfse_kernel(M, N, _p(R_w), _p(W), float(gamma), float(w00), int(max_iters),
                              int(stop_tally), float(e0), _p(G), _p(us), _p(vs), _p(cs), _p(es), _p(sf),
                              ctypes.byref(t))
    if k < 0:
        _check(k)
    return G, us[:k], vs[:k], cs[:k], es[:k], sf[:k], int(t.value)


def extrapolate_rfse(signal, labels, rho, gamma, iterations, basis_target=None):
    """rfse.py:170-210.  Returns dict(reconstructed, us, vs, cs, es, selfs, tally)."""
    s = np.ascontiguousarray(signal, np.float64)
    labels = np.ascontiguousarray(labels, np.int8)
    M, N = s.shape
    bt = -1 if basis_target is None else int(basis_target)
    n = max(int(iterations) if bt < 0 else bt, 1)
    rec = np.empty((M, N))
    us = np.zeros(n, np.int64); vs = np.zeros(n, np.int64)
    cs = np.zeros(n, np.complex128); es = np.zeros(n); sf = np.zeros(n, np.uint8)
    t = ctypes.c_int(0)
    k = lib().orc_extrapolate_rfse(M, N, _p(s), _p(labels), float(rho), float(gamma), int(iterations), bt,
                                   _p(rec), _p(us), _p(vs), _p(cs), _p(es), _p(sf), ctypes.byref(t))
    if k < 0:
        _check(k)
    return dict(reconstructed=rec, us=us[:k], vs=vs[:k], cs=cs[:k], es=es[:k], selfs=sf[:k],
                tally=int(t.value))


def conceal_blocks_rfse(frames: np.ndarray, blocks: np.ndarray, B: int, border: int, F: int,
                        rho: float, gamma: float, iterations: int, basis_target=None,
                        nthreads: int = 0) -> np.ndarray:
    """conceal_blocks with rFSE (rfse.py:170-210) per window."""
    fr = np.ascontiguousarray(frames)
    if fr.ndim == 2:
        fr = fr[None]
    nf, H, W = fr.shape
    bl = np.ascontiguousarray(blocks, np.int32).reshape(-1, 3)
    tiles = np.empty((bl.shape[0], B, B), np.float64)
    rc = lib().orc_conceal_blocks_rfse(_p(fr), _DT[fr.dtype], H, W, W, H * W, _p(bl), bl.shape[0],
                                       int(B), int(border), int(F), float(rho), float(gamma),
                                       int(iterations), -1 if basis_target is None else int(basis_target),
                                       _p(tiles), int(nthreads))
    _check(rc)
    return tiles


def loss_pattern(H: int, W: int, B: int, count: int, seed: int) -> np.ndarray:
    """SURVEY.md 8(d) isolated-block loss selection (orc_loss_pattern);
    (k, 2) int32 (top, left), row-major."""
    out = np.empty((max(int(count), 1), 2), np.int32)
    k = lib().orc_loss_pattern(int(H), int(W), int(B), int(count), int(seed) & (2 ** 64 - 1), _p(out))
    if k < 0:
        raise OracleError("bad loss-pattern geometry")
    return out[:k]


def frames_pattern(n_frames: int, H: int, W: int, B: int, fraction: float, seed: int) -> np.ndarray:
    """(n, 3) = (frame, top, left), one pattern per frame with
    round(fraction * grid blocks) losses (the product's frames_pattern)."""
    n = int(round(fraction * (H // B) * (W // B)))
    parts = []
    for f in range(n_frames):
        p = loss_pattern(H, W, B, n, seed * 1000003 + f)
        parts.append(np.concatenate([np.full((p.shape[0], 1), f, np.int32), p], 1))
    return np.concatenate(parts, 0) if parts else np.zeros((0, 3), np.int32)


# ------------------------------------------------------- parity utilities


def canonicalize_trace(us, vs, cs, M: int, N: int):
    """Conjugate-mirror canonical form of a cFSE trace.

    Let nu* be the first iteration whose (u, v) is not self-conjugate, i.e.
    (2u mod M, 2v mod N) != (0, 0).  If the row-major index of the mirror
    ((-u) mod M, (-v) mod N) is smaller than that of (u, v) at nu*, map every
    (u, v) to its mirror and every c to conj(c).  For real input this is an
    exact symmetry of the problem: Re{g} is invariant.
    """
    us = np.asarray(us, np.int64); vs = np.asarray(vs, np.int64)
    cs = np.asarray(cs, np.complex128)
    selfc = ((2 * us) % M == 0) & ((2 * vs) % N == 0)
    idx = np.nonzero(~selfc)[0]
    if idx.size == 0:
        return us.copy(), vs.copy(), cs.copy()
    k = idx[0]
    mu, mv = (-us[k]) % M, (-vs[k]) % N
    if mu * N + mv < us[k] * N + vs[k]:
        return (-us) % M, (-vs) % N, np.conj(cs)
    return us.copy(), vs.copy(), cs.copy()


def first_divergence(trace_a, trace_b, M, N):
    """Index of the first differing canonical selection (None if identical)."""
    ua, va, _ = canonicalize_trace(*trace_a, M, N)
    ub, vb, _ = canonicalize_trace(*trace_b, M, N)
    n = min(len(ua), len(ub))
    diff = np.nonzero((ua[:n] != ub[:n]) | (va[:n] != vb[:n]))[0]
    if diff.size:
        return int(diff[0])
    return None if len(ua) == len(ub) else n


def trace_equivalence(trace_a, trace_b, M: int, N: int, ctol: float = 1e-9,
                      noise_floor: float = 1e-10):
    """Compare two cFSE traces modulo the exact conjugate-mirror symmetry.

    Returns (kind, info): kind is "identical" (raw traces equal), "mirror"
    (equal after the global canonicalisation of `canonicalize_trace`),
    "mirror-swaps" (equal except at points where the residual was
    (near-)Hermitian and the two runs picked a bin and its mirror in the
    opposite order or switched to the mirror trajectory -- each such point is
    an fp64 tie between (u,v) and (-u,-v)), or "diverged" with info["at"] the
    first iteration that is neither.  Coefficients are compared (conjugated
    where mirrored) with relative tolerance `ctol` on the matched entries.
    """
    ua, va, ca = (np.asarray(x) for x in trace_a)
    ub, vb, cb = (np.asarray(x) for x in trace_b)
    if len(ua) != len(ub):
        return "diverged", {"at": min(len(ua), len(ub))}
    scale = max(1e-300, float(np.max(np.abs(ca))) if len(ca) else 1.0)
    small = np.nonzero(np.abs(ca) < noise_floor * scale)[0]
    if small.size:
        cut = int(small[0])
        ua, va, ca, ub, vb, cb = ua[:cut], va[:cut], ca[:cut], ub[:cut], vb[:cut], cb[:cut]

    def mir(u, v):
        return (-u) % M, (-v) % N

    def ceq(x, y):
        return abs(x - y) <= ctol * max(abs(x), abs(y), 1e-12 * scale)

    if np.array_equal(ua, ub) and np.array_equal(va, vb):
        ok = all(ceq(x, y) for x, y in zip(ca, cb))
        return ("identical" if ok else "diverged"), {"at": None if ok else -1}
    a = canonicalize_trace(ua, va, ca, M, N)
    b = canonicalize_trace(ub, vb, cb, M, N)
    if np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]):
        ok = all(ceq(x, y) for x, y in zip(a[2], b[2]))
        return ("mirror" if ok else "diverged"), {"at": None if ok else -1}
    flipped = False
    flips = 0
    k = 0
    n = len(ua)
    while k < n:
        bu, bv, bc = int(ub[k]), int(vb[k]), complex(cb[k])
        if flipped:
            bu, bv = mir(bu, bv)
            bc = bc.conjugate()
        au, av, ac = int(ua[k]), int(va[k]), complex(ca[k])
        if (au, av) == (bu, bv):
            if ceq(ac, bc):
                k += 1
                continue
            return "diverged", {"at": k, "flips": flips}
        if (au, av) == mir(bu, bv):
            # order swap of a mirror pair: a = (X, X*), b = (X*, X)
            if k + 1 < n:
                nu, nv, nc = int(ub[k + 1]), int(vb[k + 1]), complex(cb[k + 1])
                if flipped:
                    nu, nv = mir(nu, nv)
                    nc = nc.conjugate()
                if ((int(ua[k + 1]), int(va[k + 1])) == (bu, bv) and (nu, nv) == (au, av)
                        and ceq(ac, nc) and ceq(complex(ca[k + 1]), bc)):
                    flips += 1
                    k += 2
                    continue
            # switch to the mirror trajectory from here on
            flipped = not flipped
            flips += 1
            bu, bv = mir(bu, bv)
            bc = bc.conjugate()
            if ceq(ac, bc):
                k += 1
                continue
        return "diverged", {"at": k, "flips": flips}
    return "mirror-swaps", {"flips": flips}


def pick_deficit(signal, labels, rho, gamma, upto: int, trace_other) -> float:
    """Certify an fp32 divergence: step the fp64 oracle to iteration `upto`
    (the first canonical divergence from `trace_other`) and return
    (max|R_w|^2 - |R_w[pick]|^2) / max|R_w|^2, where pick is the other run's
    selection at `upto` mapped into the oracle's (possibly mirrored) frame.
    A small value means the other run chose a bin that is, within its own
    arithmetic's precision, as good as the maximum -- a near-tie."""
    s = np.asarray(signal, np.float64)
    w = build_weight(labels, rho)
    W = dft2(w.astype(np.complex128))
    R = dft2((s * w).astype(np.complex128))
    e0 = float(np.sum(w * s * s))
    M, N = R.shape
    n = max(upto + 1, 1)
    R0 = R.copy()
    _, ous, ovs, ocs, _ = cfse_kernel(R0, W, gamma, 1.0 / W[0, 0].real, n, e0)
    oc = canonicalize_trace(ous, ovs, ocs, M, N)
    mirrored = not np.array_equal(oc[0], ous)
    gu, gv, _ = canonicalize_trace(*trace_other, M, N)
    pu, pv = int(gu[upto]), int(gv[upto])
    if mirrored:
        pu, pv = (-pu) % M, (-pv) % N
    if upto > 0:
        cfse_kernel(R, W, gamma, 1.0 / W[0, 0].real, upto, e0)
    m2 = R.real ** 2 + R.imag ** 2
    top = float(m2.max())
    return float((top - m2[pu, pv]) / top) if top > 0 else 0.0


def divergence_certificate(signal, labels, rho, gamma, upto: int, trace_fp32) -> dict:
    """Evidence for an fp32 run that left the fp64 selection sequence at
    iteration `upto` (its first canonical divergence from the oracle).

    The fp64 oracle is stepped to `upto`; in its state R64:
      top      max |R64|^2 (the fp64 pick),
      pick     |R64|^2 at the fp32 run's pick (mapped into the oracle's
               canonical frame),
      deficit  (top - pick) / top,
      gap_amp  |R64[top]| - |R64[pick]| (amplitude gap; >= 0),
      err_amp  the fp32 run's measured residual error: the largest
               |R32 - R64| over the bins both runs selected before `upto`
               (|c32 - c64| * w00 / gamma, c = gamma R / w00, cfse.py:85)
               and at the fp32 pick itself at `upto`
               (|c32[upto] w00 / gamma - R64[pick]|).
    The fp32 run can rank the two bins the other way only if its errors at
    them sum to at least gap_amp; `err_amp` is the size of those errors as
    measured on this block.  `bounded` = gap_amp <= 2 err_amp.
    `strict` = deficit < 1e-6 (top-2 relative gap < 1e-6).
    """
    s = np.asarray(signal, np.float64)
    w = build_weight(labels, rho)
    W = dft2(w.astype(np.complex128))
    R = dft2((s * w).astype(np.complex128))
    e0 = float(np.sum(w * s * s))
    M, N = R.shape
    w00 = W[0, 0].real
    n = max(upto + 1, 1)
    _, ous, ovs, ocs, _ = cfse_kernel(R.copy(), W, gamma, 1.0 / w00, n, e0)
    ocu, ocv, occ = canonicalize_trace(ous, ovs, ocs, M, N)
    mirrored = not (np.array_equal(ocu, ous) and np.array_equal(ocv, ovs))
    gu, gv, gc = canonicalize_trace(*trace_fp32, M, N)
    if upto > 0:
        cfse_kernel(R, W, gamma, 1.0 / w00, upto, e0)
    pu, pv = int(gu[upto]), int(gv[upto])
    # R in the canonical frame: Rc[u, v] = conj(R[-u, -v]) when mirrored
    r_pick = np.conj(R[(-pu) % M, (-pv) % N]) if mirrored else R[pu, pv]
    m2 = R.real ** 2 + R.imag ** 2
    top = float(m2.max())
    pick = float(abs(r_pick) ** 2)
    scale = w00 / gamma
    err = [abs(complex(gc[k]) - complex(occ[k])) * scale for k in range(upto)]
    err.append(abs(complex(gc[upto]) * scale - complex(r_pick)))
    err_amp = float(max(err))
    gap_amp = float(np.sqrt(top) - np.sqrt(pick))
    deficit = float((top - pick) / top) if top > 0 else 0.0
    return dict(at=int(upto), deficit=deficit, gap_amp=gap_amp, err_amp=err_amp,
                strict=bool(deficit < 1e-6), bounded=bool(gap_amp <= 2.0 * err_amp))


def fp64_tie_certificate(signal, labels, rho, gamma, upto: int, trace_a, trace_b) -> dict:
    """Evidence for two fp64 runs (e.g. the GPU reference-arithmetic path and
    the reference itself) whose canonical selection sequences first differ
    at iteration `upto`.  The oracle is stepped to `upto` (its state stands
    in for both runs' common fp64 state) and compares the two picks:
      gap_amp  | |R[pick_a]| - |R[pick_b]| |,
      err_amp  the measured disagreement of the two runs before the split:
               max over the shared selections of |c_a - c_b| w00 / gamma
               (c = gamma R / w00, cfse.py:85), and at `upto` each run's own
               |R| estimate against the oracle's.
    `bounded` = gap_amp <= 2 err_amp: the two bins are tied below the
    runs' own fp64 rounding disagreement, so either pick is correct fp64."""
    s = np.asarray(signal, np.float64)
    w = build_weight(labels, rho)
    W = dft2(w.astype(np.complex128))
    R = dft2((s * w).astype(np.complex128))
    e0 = float(np.sum(w * s * s))
    M, N = R.shape
    w00 = W[0, 0].real
    _, ous, ovs, ocs, _ = cfse_kernel(R.copy(), W, gamma, 1.0 / w00, max(upto, 1), e0)
    mirrored = not np.array_equal(canonicalize_trace(ous, ovs, ocs, M, N)[0], ous) if upto else False
    if upto > 0:
        cfse_kernel(R, W, gamma, 1.0 / w00, upto, e0)
    au, av, ac = canonicalize_trace(*trace_a, M, N)
    bu, bv, bc = canonicalize_trace(*trace_b, M, N)

    def r_at(u, v):  # R in the canonical frame
        return np.conj(R[(-u) % M, (-v) % N]) if mirrored else R[u, v]

    ra, rb = r_at(int(au[upto]), int(av[upto])), r_at(int(bu[upto]), int(bv[upto]))
    scale = w00 / gamma
    err = [abs(complex(ac[k]) - complex(bc[k])) * scale for k in range(upto)]
    err += [abs(complex(ac[upto]) * scale - complex(ra)), abs(complex(bc[upto]) * scale - complex(rb))]
    err_amp = float(max(err))
    gap_amp = float(abs(abs(ra) - abs(rb)))
    top = float(np.max(R.real ** 2 + R.imag ** 2))
    return dict(at=int(upto), gap_amp=gap_amp, err_amp=err_amp, rel_gap=gap_amp / np.sqrt(top),
                bounded=bool(gap_amp <= 2.0 * err_amp))


def _rfse_state(signal, labels, rho, gamma, upto):
    s = np.asarray(signal, np.float64)
    w = build_weight(labels, rho)
    W = dft2(w.astype(np.complex128))
    R = dft2((s * w).astype(np.complex128))
    e0 = float(np.sum(w * s * s))
    w00 = W[0, 0].real
    pre = rfse_kernel(R, W, gamma, w00, upto, 2 * upto + 1, e0) if upto > 0 else None
    return R, W, w00, pre


def rfse_crit_map(R, W, w00):
    """The pair-selection criterion of every bin (rfse.py:83-111)."""
    M, N = R.shape
    W2 = W[np.ix_((2 * np.arange(M)) % M, (2 * np.arange(N)) % N)]
    selfc = ((2 * np.arange(M)) % M == 0)[:, None] & ((2 * np.arange(N)) % N == 0)[None, :]
    D = w00 * w00 - np.abs(W2) ** 2
    a = R
    nr = w00 * a.real - (W2.real * a.real + W2.imag * a.imag)
    ni = w00 * a.imag - (W2.imag * a.real - W2.real * a.imag)
    with np.errstate(divide="ignore", invalid="ignore"):
        crit = 2.0 * (nr / D * a.real + ni / D * a.imag)
    return np.where(selfc, a.real * a.real / w00, crit)


def rfse_crit_of_coefficient(c, u, v, W, w00, gamma):
    """The criterion value a selection's coefficient implies: p = c / gamma is
    the joint projection, and crit = 2 p^T adj(A) p with A the pair Gram
    matrix (= p_re^2 w00 for a self-conjugate bin)."""
    M, N = W.shape
    p = complex(c) / gamma
    if (2 * u) % M == 0 and (2 * v) % N == 0:
        return p.real * p.real * w00
    w2 = W[(2 * u) % M, (2 * v) % N]
    return 2.0 * (p.real ** 2 * (w00 + w2.real) + 2 * p.real * p.imag * w2.imag
                  + p.imag ** 2 * (w00 - w2.real))


def rfse_divergence_certificate(signal, labels, rho, gamma, upto: int, trace_fp32) -> dict:
    """rFSE analogue of divergence_certificate, in amplitude units: the fp64
    oracle is stepped to `upto` (the fp32 run's first differing selection);
    with q = sqrt(criterion) (the pair criterion is a quadratic form of the
    residual, so q is linear in it, like |R_w| for cFSE):
      deficit   (crit_top - crit_pick) / crit_top at the fp64 state,
      gap_amp   q_top - q_pick,
      err_amp   the fp32 run's measured error in the same units: the largest
                |q(c32) - q(c64)| over the shared selections (q implied by
                the coefficient, rfse_crit_of_coefficient) and at the fp32
                pick itself.
    strict: deficit < 1e-6; bounded: gap_amp <= 2 err_amp."""
    R, W, w00, pre = _rfse_state(signal, labels, rho, gamma, upto)
    us32, vs32, cs32 = (np.asarray(x) for x in trace_fp32[:3])
    crit = rfse_crit_map(R, W, w00)
    top = float(np.max(crit))
    pu, pv = int(us32[upto]), int(vs32[upto])
    pick = float(crit[pu, pv])
    q = lambda x: float(np.sqrt(max(x, 0.0)))
    err = []
    if pre is not None:
        _, ous, ovs, ocs, _, _, _ = pre
        for k in range(upto):
            u, v = int(ous[k]), int(ovs[k])
            err.append(abs(q(rfse_crit_of_coefficient(cs32[k], u, v, W, w00, gamma))
                           - q(rfse_crit_of_coefficient(ocs[k], u, v, W, w00, gamma))))
    err.append(abs(q(rfse_crit_of_coefficient(cs32[upto], pu, pv, W, w00, gamma)) - q(pick)))
    err_amp = float(max(err))
    gap_amp = q(top) - q(pick)
    deficit = (top - pick) / top if top > 0 else 0.0
    return dict(at=int(upto), deficit=float(deficit), gap_amp=gap_amp, err_amp=err_amp,
                strict=bool(deficit < 1e-6), bounded=bool(gap_amp <= 2.0 * err_amp))


def near_tie_gap(signal, labels, rho, gamma, upto: int) -> float:
    """Step the fp64 oracle `upto` iterations, then return the relative gap
    between the two largest |R_w|^2 values at that point (the selection the
    fp32 path diverged on).  A gap < 1e-6 certifies an fp32 near-tie."""
    s = np.asarray(signal, np.float64)
    w = build_weight(labels, rho)
    W = dft2(w.astype(np.complex128))
    w00 = W[0, 0].real
    R = dft2((s * w).astype(np.complex128))
    e0 = float(np.sum(w * s * s))
    if upto > 0:
        cfse_kernel(R, W, gamma, 1.0 / w00, upto, e0)
    m2 = (R.real ** 2 + R.imag ** 2).ravel()
    # the mirror of the top bin has (up to rounding) the same magnitude while
    # R_w is still Hermitian; exclude it so the gap measures a real near-tie
    M, N = R.shape
    top = int(np.argmax(m2))
    u, v = divmod(top, N)
    mir = ((-u) % M) * N + ((-v) % N)
    m2s = m2.copy()
    m2s[top] = -1.0
    if mir != top and abs(m2[mir] - m2[top]) <= 1e-9 * m2[top]:
        m2s[mir] = -1.0
    second = float(np.max(m2s))
    return float((m2[top] - second) / m2[top]) if m2[top] > 0 else 0.0

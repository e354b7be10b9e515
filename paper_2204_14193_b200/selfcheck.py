"""Independent equivalence self-check (the SPEC's `oracle` module and
`cmd_selfcheck`, SPEC.md:266-294, 413 -- the reference package ships
neither).

`spatial_extrapolate` runs the spatial-domain brute-force matching pursuit
on the GPU (csrc/spatial.cu via the C ABI): no FFT and no frequency-domain
residual; every projection is the direct double sum of Eq. (9).  Its
selections, coefficients and pixels are compared with the production
frequency-domain path (`extrapolate_cfse` / `extrapolate_rfse`) on seeded
random instances (SPEC: 12 x 12, 30 % loss, gamma 0.2, rho 0.8, I = 40),
together with the energy-decrease identity (trace energy vs the directly
evaluated weighted residual energy).  Nothing here reads the test oracle
under oracle/: this is the shipped check.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError
from .types import FseConfig
from .weighting import AreaMask


def spatial_extrapolate(signal, mask: AreaMask, config: FseConfig, pair_mode: bool = False) -> dict:
    """Brute-force spatial matching pursuit of one window (M, N <= 32).
    Returns dict(reconstructed, us, vs, cs, es, es_direct, selfs, tally)."""
    torch = _lib.require_cuda()
    s = np.ascontiguousarray(signal, np.float64)
    M, N = s.shape
    if (M, N) != tuple(config.fft_dims):
        raise ConfigError(f"signal shape {s.shape} does not match configured FFT dims {config.fft_dims}")
    bt = -1 if config.basis_target is None else int(config.basis_target)
    cap = max(bt if (pair_mode and bt >= 0) else config.loop_bound, 1)
    dev = "cuda"
    sd = torch.from_numpy(s).to(dev)
    lab = torch.from_numpy(np.ascontiguousarray(mask.labels, np.int8)).to(dev)
    rec = torch.empty((M, N), dtype=torch.float64, device=dev)
    us = torch.zeros(cap, dtype=torch.int64, device=dev)
    vs = torch.zeros_like(us)
    cs = torch.zeros(cap, dtype=torch.complex128, device=dev)
    es = torch.zeros(cap, dtype=torch.float64, device=dev)
    ed = torch.zeros_like(es)
    sf = torch.zeros(cap, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    tal = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().fse_spatial_extrapolate(
        1, M, N, _lib.ptr(sd), _lib.ptr(lab), 0, float(config.rho_hat), float(config.gamma),
        config.loop_bound if not pair_mode else config.iterations, int(pair_mode), bt if pair_mode else -1,
        _lib.ptr(rec), _lib.ptr(us), _lib.ptr(vs), _lib.ptr(cs), _lib.ptr(es), _lib.ptr(ed), _lib.ptr(sf),
        _lib.ptr(cnt), _lib.ptr(tal), _lib.ptr(st), _lib.stream_ptr(None)))
    status = int(st.item())
    if status == 1:
        raise ConfigError("total support weight is numerically zero (empty support)")
    if status == 2:
        raise ConfigError("support area is degenerate for pairwise selection")
    k = int(cnt.item())
    return dict(reconstructed=rec.cpu().numpy(), us=us[:k].cpu().numpy(), vs=vs[:k].cpu().numpy(),
                cs=cs[:k].cpu().numpy(), es=es[:k].cpu().numpy(), es_direct=ed[:k].cpu().numpy(),
                selfs=sf[:k].cpu().numpy(), tally=int(tal.item()))


def canonical(us, vs, cs, M: int, N: int):
    """Conjugate-mirror canonical form of a cFSE trace: at
    the first selection that is not self-conjugate, if the mirror
    ((-u) mod M, (-v) mod N) has the smaller row-major index, mirror every
    selection and conjugate every coefficient (an exact symmetry for real
    input: Re{g} is unchanged)."""
    us, vs, cs = np.asarray(us, np.int64), np.asarray(vs, np.int64), np.asarray(cs, np.complex128)
    nsc = np.nonzero(((2 * us) % M != 0) | ((2 * vs) % N != 0))[0]
    if nsc.size:
        k = nsc[0]
        if ((-us[k]) % M) * N + (-vs[k]) % N < us[k] * N + vs[k]:
            return (-us) % M, (-vs) % N, np.conj(cs)
    return us, vs, cs


def _trace(r):
    us = np.array([t.frequency[0] for t in r.trace], np.int64)
    vs = np.array([t.frequency[1] for t in r.trace], np.int64)
    cs = np.array([t.coefficient for t in r.trace], np.complex128)
    es = np.array([t.residual_energy for t in r.trace], np.float64)
    return us, vs, cs, es


def instances(seed: int = 0, n: int = 50, size: int = 12, loss: float = 0.3):
    """SPEC.md:277 instances: uniform [0, 255) signals, random loss masks."""
    rng = np.random.default_rng(seed)
    for _ in range(n):
        s = rng.uniform(0.0, 255.0, (size, size))
        lo = rng.uniform(size=(size, size)) < loss
        if lo.all() or not lo.any():
            lo[0, 0] = not lo[0, 0]
        yield s, AreaMask.from_loss(lo)


def run(seed: int = 0, n: int = 50, size: int = 12, iterations: int = 40, gamma: float = 0.2,
        rho: float = 0.8, tol: float = 1e-9):
    """Oracle equivalence (cFSE and rFSE) and energy identities on seeded
    instances.  Returns a list of (name, passed, detail)."""
    from .cfse import extrapolate_cfse
    from .rfse import extrapolate_rfse

    results = []
    kinds = {"identical": 0, "mirror": 0, "diverged": 0}
    dev_px = dev_c = dev_e = dev_id = 0.0
    rf_ok, rf_px, rf_n = 0, 0.0, 0
    cfg = FseConfig(rho_hat=rho, gamma=gamma, iterations=iterations, fft_dims=(size, size))
    cfg_r = FseConfig(rho_hat=rho, gamma=gamma, iterations=iterations, fft_dims=(size, size), algorithm="rfse")
    for s, mask in instances(seed, n, size):
        r = extrapolate_cfse(s, mask, cfg)
        o = spatial_extrapolate(s, mask, cfg)
        us, vs, cs, es = _trace(r)
        scale = max(float(np.max(np.abs(cs))), 1e-300)
        e0 = float(np.sum(np.where(mask.labels == 1, 1.0, 0.0) * s * s)) or 1.0
        dev_id = max(dev_id, float(np.max(np.abs(o["es"] - o["es_direct"]))) / e0)
        if np.array_equal(us, o["us"]) and np.array_equal(vs, o["vs"]):
            kind, oc = "identical", o["cs"]
        else:
            a, b = canonical(us, vs, cs, size, size), canonical(o["us"], o["vs"], o["cs"], size, size)
            same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            kind, cs, oc = ("mirror", a[2], b[2]) if same else ("diverged", cs, o["cs"])
        kinds[kind] += 1
        if kind != "diverged":
            dev_c = max(dev_c, float(np.max(np.abs(cs - oc))) / scale)
            dev_e = max(dev_e, float(np.max(np.abs(es - o["es"]))) / e0)
            loss = mask.loss
            dev_px = max(dev_px, float(np.max(np.abs(r.reconstructed[loss] - o["reconstructed"][loss]))))
        try:
            rr = extrapolate_rfse(s, mask, cfg_r)
            ro = spatial_extrapolate(s, mask, cfg_r, pair_mode=True)
        except ConfigError:
            continue  # degenerate pair geometry: both paths reject it
        rf_n += 1
        rus = np.array([t.frequency for t in rr.trace], np.int64).reshape(-1, 2)
        same = (len(rus) == len(ro["us"]) and np.array_equal(rus[:, 0], ro["us"])
                and np.array_equal(rus[:, 1], ro["vs"]) and rr.basis_count == ro["tally"])
        if same:
            rcs = np.array([t.coefficient for t in rr.trace])
            sc = max(float(np.max(np.abs(rcs))), 1e-300) if len(rcs) else 1.0
            same = float(np.max(np.abs(rcs - ro["cs"]), initial=0.0)) <= tol * sc
            rf_px = max(rf_px, float(np.max(np.abs(rr.reconstructed[mask.loss] - ro["reconstructed"][mask.loss]))))
        rf_ok += bool(same)
    results.append(("cFSE oracle equivalence: selection sequence identical or global mirror",
                    kinds["diverged"] == 0, dict(kinds)))
    results.append(("cFSE coefficients within 1e-9 relative", dev_c <= tol, dev_c))
    results.append(("cFSE trace energies within 1e-9 of the oracle's", dev_e <= tol, dev_e))
    results.append(("cFSE loss pixels within 1e-9", dev_px <= tol, dev_px))
    results.append(("energy-decrease identity (tracked vs direct spatial) within 1e-9", dev_id <= tol, dev_id))
    results.append(("rFSE oracle equivalence: pair sequence, tally, coefficients 1e-9",
                    rf_ok == rf_n, f"{rf_ok}/{rf_n}"))
    results.append(("rFSE loss pixels within 1e-9", rf_px <= tol, rf_px))
    return results

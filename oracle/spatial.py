"""Spatial-domain brute-force matching pursuit -- TEST INFRASTRUCTURE ONLY.

Restates the SPEC's `oracle` module: no FFT anywhere; every
projection is the direct double sum of Eq. (9),
    p_(k,l) = sum_{m,n} w[m,n] r[m,n] conj(phi_(k,l)[m,n]) / sum w,
(the denominator is W[0,0] because |phi| = 1), selection by Eq. (10)
(argmax |p|^2 W00 == argmax |R_w|^2, shared row-major-first tie rule),
coefficient c = gamma p (Eq. 13), and the residual / model updates of
Eqs. (14), (17) applied in the spatial domain.  Cost O(I M^2 N^2): for the
small instances of acceptance criterion 1 (M, N <= 16, I <= 64).

`pair_mode=True` mirrors the reference's rFSE pair rule (rfse.py:37-167):
joint projection onto {phi, conj(phi)} with the per-bin 2x2 Gram solve,
self-conjugate bins handled as a single real atom.
"""
from __future__ import annotations

import numpy as np


def _atoms(M: int, N: int) -> np.ndarray:
    """phi[(k,l), m, n] = exp(2j pi (k m / M + l n / N)) as an (MN, M, N) array."""
    m = np.arange(M)[:, None]
    n = np.arange(N)[None, :]
    k = np.arange(M)[:, None, None, None]
    l = np.arange(N)[None, :, None, None]
    ph = np.exp(2j * np.pi * (k * m[None, None] / M + l * n[None, None] / N))
    return ph.reshape(M * N, M, N)


def weights(labels: np.ndarray, rho: float) -> np.ndarray:
    M, N = labels.shape
    dm = np.arange(M)[:, None] - (M - 1) / 2.0
    dn = np.arange(N)[None, :] - (N - 1) / 2.0
    w = rho ** np.hypot(dm, dn)
    return np.where(labels == 1, w, 0.0)


def extrapolate(signal, labels, rho, gamma, iterations, pair_mode=False, max_size=32):
    s = np.asarray(signal, np.float64)
    M, N = s.shape
    if M > max_size or N > max_size:
        raise ValueError("spatial oracle is O(I M^2 N^2); size guard exceeded")
    w = weights(labels, rho)
    W00 = w.sum()
    phi = _atoms(M, N)
    r = s.astype(np.complex128).copy()  # residual over the whole window (w masks it)
    g = np.zeros((M, N), np.complex128)
    us, vs, cs, es = [], [], [], []
    E = float(np.sum(w * np.abs(r) ** 2))
    tally = 0
    for _ in range(iterations):
        proj = np.einsum("kmn,mn->k", np.conj(phi), w * r) / W00  # p_(k,l), Eq. (9)
        if not pair_mode:
            crit = np.abs(proj) ** 2 * W00  # Eq. (10)
            kbest = int(np.argmax(crit))  # first max, row-major
            u, v = divmod(kbest, N)
            c = gamma * proj[kbest]  # Eq. (13)
            g += c * phi[kbest]  # Eq. (14)
            r -= c * phi[kbest]  # Eq. (17)
            E -= gamma * (2 - gamma) * abs(proj[kbest]) ** 2 * W00
            tally += 1
        else:
            # rfse.py:82-121: joint projection on {phi_kl, conj(phi_kl)}
            R_w = proj * W00  # = R_w[k, l] of the frequency-domain loop
            best, bk, bp = -1.0, 0, 0j
            bself = True
            for kk in range(M * N):
                k, l = divmod(kk, N)
                a = R_w[kk]
                if (2 * k) % M == 0 and (2 * l) % N == 0:
                    pr = a.real / W00
                    crit = a.real * pr
                    if crit > best:
                        best, bk, bp, bself = crit, kk, complex(pr, 0.0), True
                else:
                    W2 = np.sum(w * np.exp(-2j * np.pi * (2 * k * np.arange(M)[:, None] / M
                                                         + 2 * l * np.arange(N)[None, :] / N)))
                    D = W00 * W00 - abs(W2) ** 2
                    nr = W00 * a.real - (W2.real * a.real + W2.imag * a.imag)
                    ni = W00 * a.imag - (W2.imag * a.real - W2.real * a.imag)
                    pr, pi = nr / D, ni / D
                    crit = 2.0 * (pr * a.real + pi * a.imag)
                    if crit > best:
                        best, bk, bp, bself = crit, kk, complex(pr, pi), False
            u, v = divmod(bk, N)
            if not bself:
                mu, mv = (-u) % M, (-v) % N
                if mu * N + mv < u * N + v:
                    u, v, bp = mu, mv, bp.conjugate()
            c = gamma * bp
            kk = u * N + v
            if bself:
                g += c * phi[kk]
                r -= c * phi[kk]
                tally += 1
            else:
                mk = ((-u) % M) * N + ((-v) % N)
                g += c * phi[kk] + np.conj(c) * phi[mk]
                r -= c * phi[kk] + np.conj(c) * phi[mk]
                tally += 2
            E -= gamma * (2 - gamma) * best
        us.append(u); vs.append(v); cs.append(c); es.append(E)
    rec = s.copy()
    loss = labels == 2
    rec[loss] = g.real[loss]
    return dict(reconstructed=rec, model=g, us=np.array(us, np.int64), vs=np.array(vs, np.int64),
                cs=np.array(cs, np.complex128), es=np.array(es), tally=tally,
                energy_direct=float(np.sum(w * np.abs(r) ** 2)))

/*
 * cfse_oracle.c -- CPU restatement of the reference cFSE path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the CPU baseline timed by bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline leg / --impl reference)
 * may load it.  The product package never links or calls it.
 *
 * Every function restates the reference Python package `fse` (mounted at
 * /root/reference/pkg/src/fse) in plain C, fp64, single thread per window:
 *
 *   orc_build_mask      <- weighting.py:81-127   (build_mask)
 *   orc_build_weight    <- weighting.py:130-145  (build_weight)
 *   orc_dft2            <- spectral.py:32-56     (dft2 / idft2 = numpy pocketfft
 *                          convention: unnormalised forward, 1/(MN) inverse)
 *   orc_cfse_kernel     <- cfse.py:55-107        (_cfse_kernel, numba loop)
 *   orc_extrapolate     <- cfse.py:28-52,110-142 (_prepare + extrapolate_cfse)
 *   orc_conceal_blocks  <- SPEC.md:332-340       (harness `conceal`: centred
 *                          F x F window, valid_rect = image, write Re{g})
 *   orc_rfse_kernel     <- rfse.py:37-167        (_pair_tables + _rfse_kernel)
 *   orc_extrapolate_rfse<- rfse.py:170-210       (extrapolate_rfse)
 *   orc_conceal_blocks_rfse                      (conceal with rFSE)
 *   orc_loss_pattern    <- SURVEY.md 8(d)        (seeded isolated-block loss
 *                          selection; the bench's reference-arm block list)
 *
 * Arithmetic order in orc_cfse_kernel follows the numba loop exactly with
 * no FMA contraction (compile with -ffp-contract=off): c = (gamma*a)*inv_w00,
 * p = (c.re*W.re - c.im*W.im, c.re*W.im + c.im*W.re), R -= p, |x|^2 =
 * re*re + im*im, strict '>' row-major scan starting at best = -1.0.
 *
 * The FFT is a textbook radix-2 Cooley-Tukey (direct DFT for other sizes);
 * it is NOT bit-identical to pocketfft, so selection sequences are compared
 * after conjugate-mirror canonicalisation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { AREA_PADDING = 0, AREA_SUPPORT = 1, AREA_LOSS = 2 };

/* ---------------------------------------------------------------- masks */

/* weighting.py:81-127.  Returns 0 on success, negative on ConfigError:
 * -1 support_width < 0, -2 empty loss rect, -3 loss rect outside window,
 * -4 loss rect outside valid region, -5 no support samples. */
int orc_build_mask(int M, int N, int top, int left, int height, int width,
                   int support_width, int has_valid, int vt, int vl, int vh,
                   int vw, int8_t *labels) {
  if (support_width < 0) return -1;
  if (height < 1 || width < 1) return -2;
  if (top < 0 || left < 0 || top + height > M || left + width > N) return -3;
  memset(labels, AREA_PADDING, (size_t)M * N);
  int rt = top - support_width < 0 ? 0 : top - support_width;
  int rl = left - support_width < 0 ? 0 : left - support_width;
  int rb = top + height + support_width > M ? M : top + height + support_width;
  int rr = left + width + support_width > N ? N : left + width + support_width;
  for (int m = rt; m < rb; ++m)
    for (int n = rl; n < rr; ++n) labels[(size_t)m * N + n] = AREA_SUPPORT;
  if (has_valid) {
    int v0 = vt < 0 ? 0 : vt, v1 = vt + vh > M ? M : vt + vh;
    int h0 = vl < 0 ? 0 : vl, h1 = vl + vw > N ? N : vl + vw;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        int valid = (m >= v0 && m < v1 && n >= h0 && n < h1);
        if (!valid) labels[(size_t)m * N + n] = AREA_PADDING;
      }
    for (int m = top; m < top + height; ++m)
      for (int n = left; n < left + width; ++n)
        if (!(m >= v0 && m < v1 && n >= h0 && n < h1)) return -4;
  }
  for (int m = top; m < top + height; ++m)
    for (int n = left; n < left + width; ++n) labels[(size_t)m * N + n] = AREA_LOSS;
  for (size_t i = 0; i < (size_t)M * N; ++i)
    if (labels[i] == AREA_SUPPORT) return 0;
  return -5;
}

/* weighting.py:130-145: w = rho ** hypot(m-(M-1)/2, n-(N-1)/2) on support. */
void orc_build_weight(int M, int N, const int8_t *labels, double rho, double *w) {
  for (int m = 0; m < M; ++m) {
    double dm = (double)m - (M - 1) / 2.0;
    for (int n = 0; n < N; ++n) {
      double dn = (double)n - (N - 1) / 2.0;
      double v = pow(rho, hypot(dm, dn));
      w[(size_t)m * N + n] = labels[(size_t)m * N + n] == AREA_SUPPORT ? v : 0.0;
    }
  }
}

/* ------------------------------------------------------------------ FFT */

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* In-place 1-D transform of n complex values at stride `st` (in complex
 * units).  sign = -1 forward, +1 inverse (unscaled). */
static void fft1d(double *x, int n, int st, int sign, double *tmp) {
  for (int i = 0; i < n; ++i) {
    tmp[2 * i] = x[2 * (size_t)i * st];
    tmp[2 * i + 1] = x[2 * (size_t)i * st + 1];
  }
  if (is_pow2(n)) {
    /* bit reversal */
    for (int i = 1, j = 0; i < n; ++i) {
      int bit = n >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) {
        double a = tmp[2 * i], b = tmp[2 * i + 1];
        tmp[2 * i] = tmp[2 * j]; tmp[2 * i + 1] = tmp[2 * j + 1];
        tmp[2 * j] = a; tmp[2 * j + 1] = b;
      }
    }
    for (int len = 2; len <= n; len <<= 1) {
      int half = len >> 1;
      for (int k = 0; k < half; ++k) {
        double ang = sign * 2.0 * M_PI * (double)k / (double)len;
        double wr = cos(ang), wi = sin(ang);
        for (int i = 0; i < n; i += len) {
          double *a = tmp + 2 * (i + k), *b = tmp + 2 * (i + k + half);
          double tr = b[0] * wr - b[1] * wi, ti = b[0] * wi + b[1] * wr;
          b[0] = a[0] - tr; b[1] = a[1] - ti;
          a[0] = a[0] + tr; a[1] = a[1] + ti;
        }
      }
    }
    for (int i = 0; i < n; ++i) {
      x[2 * (size_t)i * st] = tmp[2 * i];
      x[2 * (size_t)i * st + 1] = tmp[2 * i + 1];
    }
  } else {
    /* direct DFT with exact index reduction (k*m mod n) */
    double *out = tmp + 2 * n;
    for (int k = 0; k < n; ++k) {
      double sr = 0, si = 0;
      for (int m = 0; m < n; ++m) {
        int j = (int)(((long long)k * m) % n);
        double ang = sign * 2.0 * M_PI * (double)j / (double)n;
        double wr = cos(ang), wi = sin(ang);
        sr += tmp[2 * m] * wr - tmp[2 * m + 1] * wi;
        si += tmp[2 * m] * wi + tmp[2 * m + 1] * wr;
      }
      out[2 * k] = sr; out[2 * k + 1] = si;
    }
    for (int i = 0; i < n; ++i) {
      x[2 * (size_t)i * st] = out[2 * i];
      x[2 * (size_t)i * st + 1] = out[2 * i + 1];
    }
  }
}

/* spectral.py:32-56.  in/out interleaved complex M x N (may alias). */
void orc_dft2(int M, int N, const double *in, double *out, int inverse) {
  size_t mn = (size_t)M * N;
  if (out != in) memcpy(out, in, mn * 2 * sizeof(double));
  int L = M > N ? M : N;
  double *tmp = (double *)malloc(sizeof(double) * 4 * (size_t)L);
  int sign = inverse ? +1 : -1;
  for (int m = 0; m < M; ++m) fft1d(out + 2 * (size_t)m * N, N, 1, sign, tmp);
  for (int n = 0; n < N; ++n) fft1d(out + 2 * (size_t)n, M, N, sign, tmp);
  free(tmp);
  if (inverse) {
    double s = 1.0 / (double)mn;
    for (size_t i = 0; i < 2 * mn; ++i) out[i] *= s;
  }
}

/* --------------------------------------------------------- cFSE loop */

/* cfse.py:55-107.  R (c128 M x N) is mutated in place; G zero-initialised
 * here.  Trace arrays have `iters` entries. */
void orc_cfse_kernel(int M, int N, double *R, const double *W, double gamma,
                     double inv_w00, int iters, double e0, double *G,
                     int64_t *us, int64_t *vs, double *cs, double *es) {
  size_t mn = (size_t)M * N;
  double dmn = (double)mn;
  if (G) memset(G, 0, sizeof(double) * 2 * mn);
  double damp = gamma * (2.0 - gamma);
  double e = e0;
  for (int it = 0; it < iters; ++it) {
    double best = -1.0;
    int bu = 0, bv = 0;
    for (int k = 0; k < M; ++k)
      for (int l = 0; l < N; ++l) {
        const double *x = R + 2 * ((size_t)k * N + l);
        double m2 = x[0] * x[0] + x[1] * x[1];
        if (m2 > best) { best = m2; bu = k; bv = l; }
      }
    int u = bu, v = bv;
    double ar = R[2 * ((size_t)u * N + v)], ai = R[2 * ((size_t)u * N + v) + 1];
    /* c = gamma * rw_uv * inv_w00 (numba: real*complex promotes the real) */
    double t_r = gamma * ar - 0.0 * ai, t_i = gamma * ai + 0.0 * ar;
    double cr = t_r * inv_w00 - t_i * 0.0, ci = t_i * inv_w00 + t_r * 0.0;
    if (G) {
      double gr = dmn * cr - 0.0 * ci, gi = dmn * ci + 0.0 * cr;
      G[2 * ((size_t)u * N + v)] += gr;
      G[2 * ((size_t)u * N + v) + 1] += gi;
    }
    for (int k = 0; k < M; ++k) {
      int ks = k - u;
      if (ks < 0) ks += M;
      for (int l = 0; l < N; ++l) {
        int ls = l - v;
        if (ls < 0) ls += N;
        const double *w = W + 2 * ((size_t)ks * N + ls);
        double pr = cr * w[0] - ci * w[1];
        double pi = cr * w[1] + ci * w[0];
        double *x = R + 2 * ((size_t)k * N + l);
        x[0] = x[0] - pr;
        x[1] = x[1] - pi;
      }
    }
    e -= damp * (ar * ar + ai * ai) * inv_w00;
    us[it] = u; vs[it] = v;
    cs[2 * it] = cr; cs[2 * it + 1] = ci;
    es[it] = e;
  }
}

/* cfse.py:28-52 (_prepare) + 110-142 (extrapolate_cfse).
 * s: real M x N; recon: real M x N; model (nullable): c128 M x N.
 * Returns 0, or -6 for "total support weight is numerically zero". */
int orc_extrapolate(int M, int N, const double *s, const int8_t *labels,
                    double rho, double gamma, int iters, double *recon,
                    double *model, int64_t *us, int64_t *vs, double *cs,
                    double *es, double *Rw_out, double *W_out) {
  size_t mn = (size_t)M * N;
  double *w = (double *)malloc(sizeof(double) * mn);
  double *W = (double *)malloc(sizeof(double) * 2 * mn);
  double *R = (double *)malloc(sizeof(double) * 2 * mn);
  double *G = (double *)malloc(sizeof(double) * 2 * mn);
  orc_build_weight(M, N, labels, rho, w);
  for (size_t i = 0; i < mn; ++i) { W[2 * i] = w[i]; W[2 * i + 1] = 0.0; }
  orc_dft2(M, N, W, W, 0);
  double w00 = W[0];
  if (w00 <= 1e-12 * (double)M * (double)N) {
    free(w); free(W); free(R); free(G);
    return -6;
  }
  double e0 = 0.0;
  for (size_t i = 0; i < mn; ++i) {
    R[2 * i] = s[i] * w[i]; R[2 * i + 1] = 0.0;
    e0 += w[i] * s[i] * s[i];
  }
  orc_dft2(M, N, R, R, 0);
  if (Rw_out) memcpy(Rw_out, R, sizeof(double) * 2 * mn);
  if (W_out) memcpy(W_out, W, sizeof(double) * 2 * mn);
  orc_cfse_kernel(M, N, R, W, gamma, 1.0 / w00, iters, e0, G, us, vs, cs, es);
  orc_dft2(M, N, G, G, 1); /* g = idft2(G) */
  for (size_t i = 0; i < mn; ++i)
    recon[i] = labels[i] == AREA_LOSS ? G[2 * i] : s[i];
  if (model) memcpy(model, G, sizeof(double) * 2 * mn);
  free(w); free(W); free(R); free(G);
  return 0;
}

/* ------------------------------------------------------ image harness */

static double pix(const void *frames, int dtype, size_t idx) {
  switch (dtype) {
    case 0: return (double)((const uint8_t *)frames)[idx];
    case 1: return (double)((const float *)frames)[idx];
    default: return ((const double *)frames)[idx];
  }
}

/* SPEC.md:332-340 (conceal): for each block (frame, top, left) cut the F x F
 * window centred on the B x B loss block, valid_rect = image in window
 * coordinates, run extrapolate, write Re{g} of the loss pixels to tiles
 * (nblocks x B x B, unclamped fp64).  Blocks are independent
 * and run on `nthreads` OpenMP threads.  Returns 0 or the first error. */
int orc_conceal_blocks(const void *frames, int dtype, int H, int Wd,
                       long long pitch, long long frame_stride,
                       const int32_t *blocks, int nblocks, int B, int border,
                       int F, double rho, double gamma, int iters,
                       double *tiles, int nthreads) {
  int off = (F - B) / 2;
  int err = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    size_t mn = (size_t)F * F;
    double *s = (double *)malloc(sizeof(double) * mn);
    double *rec = (double *)malloc(sizeof(double) * mn);
    int8_t *lab = (int8_t *)malloc(mn);
    int64_t *us = (int64_t *)malloc(sizeof(int64_t) * (iters > 0 ? iters : 1));
    int64_t *vs = (int64_t *)malloc(sizeof(int64_t) * (iters > 0 ? iters : 1));
    double *cs = (double *)malloc(sizeof(double) * 2 * (iters > 0 ? iters : 1));
    double *es = (double *)malloc(sizeof(double) * (iters > 0 ? iters : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int b = 0; b < nblocks; ++b) {
      int f = blocks[3 * b], top = blocks[3 * b + 1], left = blocks[3 * b + 2];
      int wt = top - off, wl = left - off;
      int rc = orc_build_mask(F, F, off, off, B, B, border, 1, -wt, -wl, H, Wd, lab);
      if (rc == 0) {
        const size_t fbase = (size_t)f * (size_t)frame_stride;
        for (int m = 0; m < F; ++m)
          for (int n = 0; n < F; ++n) {
            int y = wt + m, x = wl + n;
            s[(size_t)m * F + n] = (y >= 0 && y < H && x >= 0 && x < Wd)
                                       ? pix(frames, dtype, fbase + (size_t)y * pitch + x)
                                       : 0.0;
          }
        rc = orc_extrapolate(F, F, s, lab, rho, gamma, iters, rec, NULL, us, vs, cs, es,
                             NULL, NULL);
      }
      if (rc != 0) {
#ifdef _OPENMP
#pragma omp critical
#endif
        { if (!err) err = rc; }
        continue;
      }
      for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j)
          tiles[(size_t)b * B * B + (size_t)i * B + j] = rec[(size_t)(off + i) * F + off + j];
    }
    free(s); free(rec); free(lab); free(us); free(vs); free(cs); free(es);
  }
  return err;
}

/* ------------------------------------------------------------ rFSE */

/* rfse.py:37-55 (_pair_tables) + 56-167 (_rfse_kernel), numba order.
 * R (c128 M x N) mutated in place; W the weight spectrum; w00 = W[0,0].re.
 * Runs until `max_iters` iterations or the basis-function tally reaches
 * `stop_tally`.  Trace arrays hold max_iters entries; returns the count
 * executed (*tally = basis functions), or -7 when the pair Gram
 * determinant is degenerate (ConfigError, rfse.py:50-54).  G nullable. */
int orc_rfse_kernel(int M, int N, double *R, const double *W, double gamma,
                    double w00, int max_iters, int stop_tally, double e0,
                    double *G, int64_t *us, int64_t *vs, double *cs,
                    double *es, uint8_t *selfs, int *tally_out) {
  size_t mn = (size_t)M * N;
  double dmn = (double)mn;
  double *W2 = (double *)malloc(sizeof(double) * 2 * mn);
  double *D = (double *)malloc(sizeof(double) * mn);
  uint8_t *sc = (uint8_t *)malloc(mn);
  for (int k = 0; k < M; ++k)
    for (int l = 0; l < N; ++l) {
      size_t i = (size_t)k * N + l;
      int k2 = (2 * k) % M, l2 = (2 * l) % N;
      const double *w2 = W + 2 * ((size_t)k2 * N + l2);
      W2[2 * i] = w2[0]; W2[2 * i + 1] = w2[1];
      sc[i] = (k2 == 0 && l2 == 0);
      D[i] = w00 * w00 - (w2[0] * w2[0] + w2[1] * w2[1]);
      if (!sc[i] && D[i] <= 1e-9 * w00 * w00) {
        free(W2); free(D); free(sc);
        return -7;
      }
    }
  if (G) memset(G, 0, sizeof(double) * 2 * mn);
  double damp = gamma * (2.0 - gamma), e = e0;
  int count = 0, tally = 0;
  while (count < max_iters && tally < stop_tally) {
    double best = -1.0, bpr = 0.0, bpi = 0.0;
    int bu = 0, bv = 0, bself = 1;
    for (int k = 0; k < M; ++k)
      for (int l = 0; l < N; ++l) {
        size_t i = (size_t)k * N + l;
        double ar = R[2 * i], ai = R[2 * i + 1];
        if (sc[i]) {
          double pr = ar / w00, crit = ar * pr;
          if (crit > best) { best = crit; bu = k; bv = l; bpr = pr; bpi = 0.0; bself = 1; }
        } else {
          double w2r = W2[2 * i], w2i = W2[2 * i + 1];
          double nr = w00 * ar - (w2r * ar + w2i * ai);
          double ni = w00 * ai - (w2i * ar - w2r * ai);
          double d = D[i];
          double pr = nr / d, pi = ni / d;
          double crit = 2.0 * (pr * ar + pi * ai);
          if (crit > best) { best = crit; bu = k; bv = l; bpr = pr; bpi = pi; bself = 0; }
        }
      }
    int u = bu, v = bv;
    if (!bself) {
      int mu = (M - u) % M, mv = (N - v) % N;
      if (mu * N + mv < u * N + v) { u = mu; v = mv; bpi = -bpi; }
    }
    /* c = gamma * complex(bpr, bpi) */
    double cr = gamma * bpr - 0.0 * bpi, ci = gamma * bpi + 0.0 * bpr;
    if (G) {
      G[2 * ((size_t)u * N + v)] += dmn * cr - 0.0 * ci;
      G[2 * ((size_t)u * N + v) + 1] += dmn * ci + 0.0 * cr;
    }
    if (bself) {
      for (int k = 0; k < M; ++k) {
        int ks = k - u;
        if (ks < 0) ks += M;
        for (int l = 0; l < N; ++l) {
          int ls = l - v;
          if (ls < 0) ls += N;
          const double *w = W + 2 * ((size_t)ks * N + ls);
          double *x = R + 2 * ((size_t)k * N + l);
          x[0] = x[0] - (cr * w[0] - ci * w[1]);
          x[1] = x[1] - (cr * w[1] + ci * w[0]);
        }
      }
      tally += 1;
    } else {
      int mu = (M - u) % M, mv = (N - v) % N;
      double ccr = cr, cci = -ci;
      if (G) {
        G[2 * ((size_t)mu * N + mv)] += dmn * ccr - 0.0 * cci;
        G[2 * ((size_t)mu * N + mv) + 1] += dmn * cci + 0.0 * ccr;
      }
      for (int k = 0; k < M; ++k) {
        int ks = k - u, ks2 = k - mu;
        if (ks < 0) ks += M;
        if (ks2 < 0) ks2 += M;
        for (int l = 0; l < N; ++l) {
          int ls = l - v, ls2 = l - mv;
          if (ls < 0) ls += N;
          if (ls2 < 0) ls2 += N;
          const double *w = W + 2 * ((size_t)ks * N + ls);
          const double *w2 = W + 2 * ((size_t)ks2 * N + ls2);
          double *x = R + 2 * ((size_t)k * N + l);
          /* (R - c W) - conj(c) W' */
          double t0 = x[0] - (cr * w[0] - ci * w[1]);
          double t1 = x[1] - (cr * w[1] + ci * w[0]);
          x[0] = t0 - (ccr * w2[0] - cci * w2[1]);
          x[1] = t1 - (ccr * w2[1] + cci * w2[0]);
        }
      }
      tally += 2;
    }
    e -= damp * best;
    us[count] = u; vs[count] = v;
    cs[2 * count] = cr; cs[2 * count + 1] = ci;
    es[count] = e;
    selfs[count] = (uint8_t)bself;
    ++count;
  }
  free(W2); free(D); free(sc);
  if (tally_out) *tally_out = tally;
  return count;
}

/* rfse.py:170-210 (extrapolate_rfse): _prepare, pair tables, loop, Re{idft2}
 * on the loss.  basis_target < 0: fixed count `iters`; else max_iters =
 * stop_tally = basis_target.  Returns the iteration count (>= 0) or a
 * negative error (-6 empty support, -7 degenerate pairs). */
int orc_extrapolate_rfse(int M, int N, const double *s, const int8_t *labels,
                         double rho, double gamma, int iters, int basis_target,
                         double *recon, int64_t *us, int64_t *vs, double *cs,
                         double *es, uint8_t *selfs, int *tally) {
  size_t mn = (size_t)M * N;
  double *w = (double *)malloc(sizeof(double) * mn);
  double *W = (double *)malloc(sizeof(double) * 2 * mn);
  double *R = (double *)malloc(sizeof(double) * 2 * mn);
  double *G = (double *)malloc(sizeof(double) * 2 * mn);
  orc_build_weight(M, N, labels, rho, w);
  for (size_t i = 0; i < mn; ++i) { W[2 * i] = w[i]; W[2 * i + 1] = 0.0; }
  orc_dft2(M, N, W, W, 0);
  double w00 = W[0];
  int rc;
  if (w00 <= 1e-12 * (double)M * (double)N) {
    rc = -6;
  } else {
    double e0 = 0.0;
    for (size_t i = 0; i < mn; ++i) {
      R[2 * i] = s[i] * w[i]; R[2 * i + 1] = 0.0;
      e0 += w[i] * s[i] * s[i];
    }
    orc_dft2(M, N, R, R, 0);
    int max_it = basis_target >= 0 ? basis_target : iters;
    int stop = basis_target >= 0 ? basis_target : 2 * iters + 1;
    rc = orc_rfse_kernel(M, N, R, W, gamma, w00, max_it, stop, e0, G, us, vs, cs, es, selfs, tally);
    if (rc >= 0) {
      orc_dft2(M, N, G, G, 1);
      for (size_t i = 0; i < mn; ++i) recon[i] = labels[i] == AREA_LOSS ? G[2 * i] : s[i];
    }
  }
  free(w); free(W); free(R); free(G);
  return rc;
}

/* rFSE per-block concealment (as orc_conceal_blocks). */
int orc_conceal_blocks_rfse(const void *frames, int dtype, int H, int Wd,
                            long long pitch, long long frame_stride,
                            const int32_t *blocks, int nblocks, int B, int border,
                            int F, double rho, double gamma, int iters, int basis_target,
                            double *tiles, int nthreads) {
  int off = (F - B) / 2;
  int err = 0;
  int cap = basis_target >= 0 ? basis_target : iters;
  if (cap < 1) cap = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    size_t mn = (size_t)F * F;
    double *s = (double *)malloc(sizeof(double) * mn);
    double *rec = (double *)malloc(sizeof(double) * mn);
    int8_t *lab = (int8_t *)malloc(mn);
    int64_t *us = (int64_t *)malloc(sizeof(int64_t) * cap);
    int64_t *vs = (int64_t *)malloc(sizeof(int64_t) * cap);
    double *cs = (double *)malloc(sizeof(double) * 2 * cap);
    double *es = (double *)malloc(sizeof(double) * cap);
    uint8_t *sf = (uint8_t *)malloc(cap);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int b = 0; b < nblocks; ++b) {
      int f = blocks[3 * b], top = blocks[3 * b + 1], left = blocks[3 * b + 2];
      int wt = top - off, wl = left - off, tally = 0;
      int rc = orc_build_mask(F, F, off, off, B, B, border, 1, -wt, -wl, H, Wd, lab);
      if (rc == 0) {
        const size_t fbase = (size_t)f * (size_t)frame_stride;
        for (int m = 0; m < F; ++m)
          for (int n = 0; n < F; ++n) {
            int y = wt + m, x = wl + n;
            s[(size_t)m * F + n] = (y >= 0 && y < H && x >= 0 && x < Wd)
                                       ? pix(frames, dtype, fbase + (size_t)y * pitch + x)
                                       : 0.0;
          }
        rc = orc_extrapolate_rfse(F, F, s, lab, rho, gamma, iters, basis_target, rec, us, vs, cs,
                                  es, sf, &tally);
        if (rc > 0) rc = 0;
      }
      if (rc != 0) {
#ifdef _OPENMP
#pragma omp critical
#endif
        { if (!err) err = rc; }
        continue;
      }
      for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j)
          tiles[(size_t)b * B * B + (size_t)i * B + j] = rec[(size_t)(off + i) * F + off + j];
    }
    free(s); free(rec); free(lab); free(us); free(vs); free(cs); free(es); free(sf);
  }
  return err;
}

/* ---------------------------------------------------- loss pattern */

/* Seeded isolated-block loss selection of SURVEY.md 8(d) (the same
 * generator the product's fse_loss_pattern implements, restated here so
 * the reference arm of bench.py builds its block list without the product
 * library): Fisher-Yates shuffle of the (H/B) x (W/B) block grid driven by
 * splitmix64(seed), then random-sequential selection rejecting any block
 * 8-adjacent to one already chosen, up to `count` blocks; output sorted
 * row-major as (top, left) pairs.  Returns the number selected. */
static uint64_t orc_splitmix64(uint64_t *x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int orc_cmp_pair(const void *a, const void *b) {
  const int32_t *x = (const int32_t *)a, *y = (const int32_t *)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

int orc_loss_pattern(int H, int W, int B, int count, uint64_t seed, int32_t *top_left) {
  if (H < 1 || W < 1 || B < 1 || count < 0) return -1;
  int gh = H / B, gw = W / B, n = gh * gw, k = 0;
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  uint8_t *taken = (uint8_t *)calloc(n > 0 ? n : 1, 1);
  for (int i = 0; i < n; ++i) perm[i] = i;
  uint64_t s = seed;
  for (int i = n - 1; i > 0; --i) {
    int j = (int)(orc_splitmix64(&s) % (uint64_t)(i + 1));
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  for (int t = 0; t < n && k < count; ++t) {
    int c = perm[t], gy = c / gw, gx = c % gw, ok = 1;
    for (int dy = -1; dy <= 1 && ok; ++dy)
      for (int dx = -1; dx <= 1 && ok; ++dx) {
        int y = gy + dy, x = gx + dx;
        if (y >= 0 && y < gh && x >= 0 && x < gw && taken[y * gw + x]) ok = 0;
      }
    if (!ok) continue;
    taken[c] = 1;
    top_left[2 * k] = gy * B;
    top_left[2 * k + 1] = gx * B;
    ++k;
  }
  qsort(top_left, (size_t)k, 2 * sizeof(int32_t), orc_cmp_pair);
  free(perm); free(taken);
  return k;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

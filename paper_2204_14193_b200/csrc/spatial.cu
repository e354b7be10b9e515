// spatial.cu -- spatial-domain brute-force matching pursuit on the GPU: the
// package's own independent equivalence check (the
// `oracle` module, used by `fse selfcheck`).
//
// No FFT and no frequency-domain residual anywhere: every iteration projects
// the spatial residual r onto every atom by the direct double sum of Eq. (9),
//     p_(k,l) = sum_{m,n} w[m,n] r[m,n] conj(phi_(k,l)[m,n]) / sum w,
// phi_(k,l)[m,n] = exp(2 pi i (k m / M + l n / N)) from exact integer-reduced
// twiddle tables, selects by Eq. (10) (argmax |p|^2 W00 == argmax |R_w|^2,
// first maximum in row-major order -- the documented tie rule, shared by
// contract), sets c = gamma p (Eq. 13) and applies the model / residual
// updates of Eqs. (14) and (17) in the spatial domain.  pair_mode mirrors the
// rFSE pair rule (rfse.py:37-167): joint projection onto {phi, conj(phi)}
// with the 2x2 Gram determinant W00^2 - |W2|^2, W2[k,l] the spatial sum of
// w exp(-2 pi i (2 k m / M + 2 l n / N)); self-conjugate atoms as one real
// atom; the pair represented by its smaller row-major member.
// Cost O(I M^2 N^2): instances up to 32 x 32 (a self-check, not a path).
#include <float.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace fse {

constexpr int kSpThreads = 256;

__global__ void __launch_bounds__(kSpThreads) spatial_kernel(SpatialArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int M = a.M, N = a.N, MN = M * N, win = blockIdx.x;
  double2 *twM = (double2 *)sm;  // exp(+2 pi i j / M)
  double2 *twN = twM + M;
  double2 *r = twN + N;          // spatial residual (complex)
  double2 *g = r + MN;           // model
  double2 *p = g + MN;           // projections
  double2 *W2 = p + MN;          // pair Gram couplings (pair mode)
  double *w = (double *)(W2 + MN);
  double *red = w + MN;          // 2 x (kSpThreads / 32) reduction slots
  int *redi = (int *)(red + 2 * (kSpThreads / 32));
  const double *s = a.signal + (size_t)win * MN;
  const int8_t *lab = a.labels + (size_t)win * a.labels_stride;
  const int tid = threadIdx.x;

  for (int j = tid; j < M; j += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * j / M, &sn, &cs);
    twM[j] = make_double2(cs, sn);
  }
  for (int j = tid; j < N; j += blockDim.x) {
    double sn, cs;
    sincospi(2.0 * j / N, &sn, &cs);
    twN[j] = make_double2(cs, sn);
  }
  for (int i = tid; i < MN; i += blockDim.x) {
    const int m = i / N, n = i - m * N;
    const double dm = (double)m - (M - 1) / 2.0, dn = (double)n - (N - 1) / 2.0;
    w[i] = lab[i] == kSupport ? pow(a.rho, hypot(dm, dn)) : 0.0;  // weighting.py:130-145
    r[i] = make_double2(lab[i] == kSupport ? s[i] : 0.0, 0.0);
    g[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  // W00 = sum w and the initial weighted energy sum w |r|^2 (one thread: exact, deterministic)
  __shared__ double sW00, sE;
  if (tid == 0) {
    double t = 0.0, e = 0.0;
    for (int i = 0; i < MN; ++i) { t += w[i]; e += w[i] * r[i].x * r[i].x; }
    sW00 = t;
    sE = e;
  }
  __syncthreads();
  const double W00 = sW00;
  if (W00 <= 1e-12 * (double)MN) {
    if (tid == 0) a.status[win] = 1;
    return;
  }
  // phi_(k,l)[m,n] = twM[(k m) mod M] * twN[(l n) mod N]
  auto atom = [&](int k, int l, int m, int n) -> double2 {
    const double2 x = twM[(k * m) % M], y = twN[(l * n) % N];
    return make_double2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
  };
  if (a.pair_mode) {
    int bad = 0;
    for (int b = tid; b < MN; b += blockDim.x) {
      const int k = b / N, l = b - k * N;
      double sr = 0.0, si = 0.0;
      for (int i = 0; i < MN; ++i) {
        const int m = i / N, n = i - m * N;
        const double2 ph = atom((2 * k) % M, (2 * l) % N, m, n);  // exp(+...), conj below
        sr += w[i] * ph.x;
        si -= w[i] * ph.y;
      }
      W2[b] = make_double2(sr, si);
      const bool selfc = (2 * k) % M == 0 && (2 * l) % N == 0;
      if (!selfc && W00 * W00 - (sr * sr + si * si) <= 1e-9 * W00 * W00) bad = 1;
    }
    if (__syncthreads_or(bad)) {
      if (tid == 0) a.status[win] = 2;
      return;
    }
  }
  double E = sE;
  const double damp = a.gamma * (2.0 - a.gamma);
  int count = 0, tally = 0;
  const int max_it = a.iterations, stop = a.pair_mode ? a.stop_tally : 2 * max_it + 1;
  while (count < max_it && tally < stop) {
    // Eq. (9): every projection by direct summation
    for (int b = tid; b < MN; b += blockDim.x) {
      const int k = b / N, l = b - k * N;
      double sr = 0.0, si = 0.0;
      for (int i = 0; i < MN; ++i) {
        const int m = i / N, n = i - m * N;
        const double2 ph = atom(k, l, m, n);
        const double xr = w[i] * r[i].x, xi = w[i] * r[i].y;
        sr += xr * ph.x + xi * ph.y;  // (xr + i xi) * conj(ph)
        si += xi * ph.x - xr * ph.y;
      }
      p[b] = make_double2(sr / W00, si / W00);
    }
    __syncthreads();
    // Eq. (10) / rfse pair criterion; first maximum in row-major order
    double best = -1.0;
    int bi = 0;
    for (int b = tid; b < MN; b += blockDim.x) {
      const int k = b / N, l = b - k * N;
      double crit;
      if (!a.pair_mode) {
        crit = (p[b].x * p[b].x + p[b].y * p[b].y) * W00;
      } else {
        const double ar = p[b].x * W00, ai = p[b].y * W00;  // = R_w[k, l]
        if ((2 * k) % M == 0 && (2 * l) % N == 0) {
          crit = ar * (ar / W00);
        } else {
          const double2 q = W2[b];
          const double D = W00 * W00 - (q.x * q.x + q.y * q.y);
          const double pr = (W00 * ar - (q.x * ar + q.y * ai)) / D;
          const double pi = (W00 * ai - (q.y * ar - q.x * ai)) / D;
          crit = 2.0 * (pr * ar + pi * ai);
        }
      }
      if (crit > best) { best = crit; bi = b; }
    }
    for (int o = 16; o; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_combine(best, bi, v2, i2);
    }
    if ((tid & 31) == 0) { red[tid >> 5] = best; redi[tid >> 5] = bi; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q) argmax_combine(best, bi, red[q], redi[q]);
      red[2 * (kSpThreads / 32) - 1] = best;
      redi[kSpThreads / 32] = bi;
    }
    __syncthreads();
    best = red[2 * (kSpThreads / 32) - 1];
    bi = redi[kSpThreads / 32];
    int u = bi / N, v = bi - (bi / N) * N;
    const bool selfc = !a.pair_mode || ((2 * u) % M == 0 && (2 * v) % N == 0);
    double cr, ci;
    if (!a.pair_mode) {
      cr = a.gamma * p[bi].x;  // Eq. (13)
      ci = a.gamma * p[bi].y;
    } else {
      const double ar = p[bi].x * W00, ai = p[bi].y * W00;
      double pr, pi;
      if (selfc) {
        pr = ar / W00;
        pi = 0.0;
      } else {
        const double2 q = W2[bi];
        const double D = W00 * W00 - (q.x * q.x + q.y * q.y);
        pr = (W00 * ar - (q.x * ar + q.y * ai)) / D;
        pi = (W00 * ai - (q.y * ar - q.x * ai)) / D;
        const int mu = (M - u) % M, mv = (N - v) % N;
        if (mu * N + mv < u * N + v) { u = mu; v = mv; pi = -pi; }  // canonical member
      }
      cr = a.gamma * pr;
      ci = a.gamma * pi;
    }
    __syncthreads();  // every thread has read p[bi] / red
    // Eqs. (14), (17): g += c phi (+ conj(c) conj(phi) for a pair), r -= the same
    for (int i = tid; i < MN; i += blockDim.x) {
      const int m = i / N, n = i - m * N;
      const double2 ph = atom(u, v, m, n);
      double dr = cr * ph.x - ci * ph.y, di = cr * ph.y + ci * ph.x;
      if (!selfc) di = 0.0, dr *= 2.0;  // c phi + conj(c phi) = 2 Re{c phi}
      g[i].x += dr; g[i].y += di;
      r[i].x -= dr; r[i].y -= di;
    }
    __syncthreads();
    if (tid == 0) {
      E -= damp * best;  // the decrease identity (cfse.py:101 / rfse.py:147)
      double Ed = 0.0;   // and the directly evaluated weighted residual energy
      for (int i = 0; i < MN; ++i) Ed += w[i] * (r[i].x * r[i].x + r[i].y * r[i].y);
      const size_t o = (size_t)win * max_it + count;
      a.us[o] = u;
      a.vs[o] = v;
      a.cs[2 * o] = cr;
      a.cs[2 * o + 1] = ci;
      a.es[o] = E;
      a.es_direct[o] = Ed;
      if (a.selfs) a.selfs[o] = selfc ? 1 : 0;
    }
    tally += selfc ? 1 : 2;
    ++count;
    __syncthreads();
  }
  for (int i = tid; i < MN; i += blockDim.x)
    a.recon[(size_t)win * MN + i] = lab[i] == kLoss ? g[i].x : s[i];
  if (tid == 0) {
    a.status[win] = 0;
    if (a.counts) a.counts[win] = count;
    if (a.tallies) a.tallies[win] = tally;
  }
}

size_t spatial_smem_bytes(int M, int N) {
  const size_t MN = (size_t)M * N;
  return (size_t)(M + N) * sizeof(double2) + 4 * MN * sizeof(double2) + MN * sizeof(double) +
         2 * (kSpThreads / 32) * sizeof(double) + (kSpThreads / 32 + 1) * sizeof(int) + 64;
}

cudaError_t launch_spatial(const SpatialArgs &a, cudaStream_t st) {
  if (a.count <= 0) return cudaSuccess;
  const size_t sm = spatial_smem_bytes(a.M, a.N);
  cudaError_t e = cudaFuncSetAttribute(spatial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  spatial_kernel<<<a.count, kSpThreads, sm, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fse

// generic.cu -- any-size cFSE kernels (fp64 reference-exact path).
//
// One CTA per window.  This is the drop-in for the reference's per-window
// entry point `extrapolate_cfse` (cfse.py:110-142) and for the numba loop
// `_cfse_kernel` (cfse.py:55-107): it accepts any M x N (the reference does;
// the SPEC oracle tests use 8x8 .. 16x16), computes in fp64 by default, and
// its iteration loop uses the reference's unfused IEEE operation order so
// identical spectra give bit-identical traces.  The throughput path for the
// image-level configs is fast.cu.
//
// Per window (all on device):
//   w      = rho^hypot(m-(M-1)/2, n-(N-1)/2) on support   weighting.py:130-145
//   W, R_w = DFT(w), DFT(s*w)                              cfse.py:43-50
//            (one complex DFT of z = w + i*kappa*s*w, kappa a power of two,
//             unpacked with the two-real-signals identity, which makes both
//             spectra exactly Hermitian -- see DESIGN.md "mirror ties")
//   I iterations of argmax / coefficient / residual update cfse.py:67-105
//   g      = sum_nu c_nu exp(+2 pi i (u m / M + v n / N))  cfse.py:126 (idft2
//            of the sparse G, evaluated directly)
//   recon  = s on support/padding, Re{g} on loss           cfse.py:127-129
#include <float.h>
#include <limits.h>
#include <math_constants.h>
#include <stdio.h>

#include "common.cuh"
#include "dft.cuh"
#include "kernels.h"

namespace fse {

constexpr int kGenThreads = 512;
constexpr size_t kCandBytes = 2 * (kGenThreads / 32) * sizeof(double4);  // cfse_iterate_reg slots

// block-wide maximum of v (every thread gets it)
__device__ double block_max(double v, double *red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// block-wide maximum of mx and sum of sm in one reduction (every thread gets
// both; the sum's association order is that of block_sum)
__device__ void block_max_sum(double &mx, double &sm, double *red) {
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = mx; red[32 + (threadIdx.x >> 5)] = sm; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool v = threadIdx.x < (blockDim.x >> 5);
    mx = v ? red[threadIdx.x] : 0.0;
    sm = v ? red[32 + threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    if (threadIdx.x == 0) { red[0] = mx; red[32] = sm; }
  }
  __syncthreads();
  mx = red[0];
  sm = red[32];
  __syncthreads();
}

// max |x[i]| over the samples with lab[i] == keep (all when lab is null)
__device__ double block_max_abs(const double *x, int n, double *red, const int8_t *lab = nullptr,
                                int keep = 0) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!lab || lab[i] == keep) v = fmax(v, fabs(x[i]));
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

__device__ double block_sum(double v, double *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

__device__ __forceinline__ double weight_at(int m, int n, int M, int N, double rho) {
  // weighting.py:140-143: rho ** hypot(m - (M-1)/2, n - (N-1)/2)
  double dm = (double)m - (M - 1) / 2.0, dn = (double)n - (N - 1) / 2.0;
  return pow(rho, hypot(dm, dn));
}

// Unpack Z = DFT(w + i*kappa*sw) into W = DFT(w) (-> Wd) and DFT(sw) (in
// place in Z).  Each mirror pair (k, -k) is owned by one thread, so both
// outputs are exactly Hermitian: W[-k] == conj(W[k]) bit for bit.
__device__ void unpack_two_real(double2 *Z, double2 *Wd, int M, int N, double inv_kappa) {
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) {
    int k = i / N, l = i - k * N;
    int mk = k ? M - k : 0, ml = l ? N - l : 0;
    int j = mk * N + ml;
    if (i > j) continue;
    double2 zi = Z[i], zj = Z[j];
    double2 wi = make_double2((zi.x + zj.x) * 0.5, (zi.y - zj.y) * 0.5);
    double2 wj = make_double2((zj.x + zi.x) * 0.5, (zj.y - zi.y) * 0.5);
    double2 si = make_double2((zi.y + zj.y) * 0.5 * inv_kappa, (zj.x - zi.x) * 0.5 * inv_kappa);
    double2 sj = make_double2((zj.y + zi.y) * 0.5 * inv_kappa, (zi.x - zj.x) * 0.5 * inv_kappa);
    Wd[i] = wi;
    Wd[j] = wj;
    Z[i] = si;
    Z[j] = sj;
  }
}

// ------------------------------------------------------------ iteration
// Block-wide argmax of (value, index), first max in row-major order.
template <typename T>
__device__ void block_argmax(T &best, int &bi, T *sv, int *si) {
  for (int o = 16; o; o >>= 1) {
    T v2 = __shfl_xor_sync(0xffffffffu, best, o);
    int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_combine(best, bi, v2, i2);
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : (T)-2.0;
    bi = lane < nw ? si[lane] : INT_MAX;
    for (int o = 16; o; o >>= 1) {
      T v2 = __shfl_xor_sync(0xffffffffu, best, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_combine(best, bi, v2, i2);
    }
  }
}

// The reference loop (cfse.py:67-105), arithmetic in T with unfused IEEE
// ops.  R is mutated in place.  Trace goes to global (us, vs, cs, es) and,
// when G != null, the dense model spectrum is accumulated (cfse.py:88).
template <typename T>
__device__ void cfse_iterate(Cplx<T> *R, const Cplx<T> *W, int M, int N, T gamma, T inv_w00,
                             int iterations, double e0, int64_t *us, int64_t *vs, double *cs,
                             double *es, double *G, T *sv, int *si, double4 *bcast) {
  typedef Ieee<T> F;
  const int MN = M * N;
  const T damp = F::mul(gamma, F::sub((T)2.0, gamma));
  T e = (T)e0;
  // pass 0: scan only
  T best = (T)-1.0;
  int bi = 0;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    Cplx<T> x = R[i];
    T m2 = F::add(F::mul(x.re, x.re), F::mul(x.im, x.im));
    if (m2 > best) { best = m2; bi = i; }
  }
  for (int it = 0; it < iterations; ++it) {
    block_argmax(best, bi, sv, si);
    if (threadIdx.x == 0) {
      Cplx<T> a = R[bi];
      bcast[0] = make_double4((double)a.re, (double)a.im, (double)best, __longlong_as_double((long long)bi));
    }
    __syncthreads();
    double4 b = bcast[0];
    const int idx = (int)__double_as_longlong(b.w);
    const T ar = (T)b.x, ai = (T)b.y;
    const int u = idx / N, v = idx - u * N;
    // c = gamma * rw_uv * inv_w00 (cfse.py:85): (gamma*a)*inv_w00
    const T cr = F::mul(F::mul(gamma, ar), inv_w00);
    const T ci = F::mul(F::mul(gamma, ai), inv_w00);
    if (threadIdx.x == 0) {
      // e -= damp * |rw_uv|^2 * inv_w00 (cfse.py:101)
      T m2 = F::add(F::mul(ar, ar), F::mul(ai, ai));
      e = F::sub(e, F::mul(F::mul(damp, m2), inv_w00));
      us[it] = u;
      vs[it] = v;
      cs[2 * it] = (double)cr;
      cs[2 * it + 1] = (double)ci;
      es[it] = (double)e;
      if (G) {  // G[u,v] += mn * c (cfse.py:88)
        double mn = (double)MN;
        G[2 * idx] = __dadd_rn(G[2 * idx], __dmul_rn(mn, (double)cr));
        G[2 * idx + 1] = __dadd_rn(G[2 * idx + 1], __dmul_rn(mn, (double)ci));
      }
    }
    if (it + 1 == iterations) break;
    // residual update (cfse.py:91-99) fused with the next pass's scan
    best = (T)-1.0;
    bi = 0;
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      int k = i / N, l = i - k * N;
      int ks = k - u, ls = l - v;
      if (ks < 0) ks += M;
      if (ls < 0) ls += N;
      Cplx<T> w = W[ks * N + ls], x = R[i];
      T pr = F::sub(F::mul(cr, w.re), F::mul(ci, w.im));
      T pi = F::add(F::mul(cr, w.im), F::mul(ci, w.re));
      x.re = F::sub(x.re, pr);
      x.im = F::sub(x.im, pi);
      R[i] = x;
      T m2 = F::add(F::mul(x.re, x.re), F::mul(x.im, x.im));
      if (m2 > best) { best = m2; bi = i; }
    }
    __syncthreads();  // bcast / sv reuse
  }
  __syncthreads();
}

// cfse_iterate with the residual spectrum in registers (windows of up to
// kGenThreads * BPT bins: every size up to 64 x 64): thread t owns bins
// t + kGenThreads j, j < BPT, in the same increasing order as the shared-
// memory loop, so per-thread first maxima and every IEEE op are identical
// (bit-exact); only W' is read from shared memory.  The block argmax is
// latency-lean: a non-negative |R|^2 orders like its bit pattern, so a warp
// finds its (value, first index) with two or three REDUX ops; the owning
// lane publishes (value, index, R) to a double-buffered candidate slot; after
// one barrier every warp merges the 16 candidates the same way and reads the
// winner's residual with two shuffles.  Same total order as cfse.py:68-79
// (larger |R|^2, then smaller row-major index).
template <typename T> struct Key;
template <> struct Key<double> {
  static FSE_DEV unsigned hi(double v) { return (unsigned)__double2hiint(v); }
  static FSE_DEV unsigned lo(double v) { return (unsigned)__double2loint(v); }
};
template <> struct Key<float> {
  static FSE_DEV unsigned hi(float v) { return __float_as_uint(v); }
  static FSE_DEV unsigned lo(float) { return 0u; }
};

// first maximum over the warp of (v >= 0, idx) for lanes with `valid`;
// returns the winning index (0xffffffff when no lane is valid)
template <typename T> FSE_DEV unsigned warp_first_max(T v, unsigned idx, bool valid) {
  const unsigned h = valid ? Key<T>::hi(v) : 0u;
  const unsigned l = valid ? Key<T>::lo(v) : 0u;
  const unsigned wh = __reduce_max_sync(0xffffffffu, h);
  unsigned wl = 0u;
  if (sizeof(T) == 8) wl = __reduce_max_sync(0xffffffffu, h == wh ? l : 0u);
  return __reduce_min_sync(0xffffffffu, valid && h == wh && l == wl ? idx : 0xffffffffu);
}

// warp_first_max with the winner's lane: one REDUX on the high key word and
// a ballot settle the common case (a single lane holds the largest high
// word); only exact high-word ties take the full (lo word, index) path.
// The same total order as warp_first_max.
template <typename T>
FSE_DEV unsigned warp_first_max_lane(T v, unsigned idx, bool valid, int &lane_out) {
  const unsigned h = valid ? Key<T>::hi(v) : 0u;
  const unsigned wh = __reduce_max_sync(0xffffffffu, h);
  const unsigned tie = __ballot_sync(0xffffffffu, valid && h == wh);
  if (__popc(tie) == 1) {
    lane_out = __ffs(tie) - 1;
    return __shfl_sync(0xffffffffu, idx, lane_out);
  }
  const unsigned l = valid ? Key<T>::lo(v) : 0u;
  unsigned wl = 0u;
  if (sizeof(T) == 8) wl = __reduce_max_sync(0xffffffffu, h == wh ? l : 0u);
  const unsigned widx = __reduce_min_sync(0xffffffffu, valid && h == wh && l == wl ? idx : 0xffffffffu);
  lane_out = __ffs(__ballot_sync(0xffffffffu, valid && idx == widx)) - 1;
  return widx;
}

// one vector load of a complex value (16 B for double: LDS.128, not two LDS.64)
FSE_DEV Cplx<double> load_cplx(const Cplx<double> *p) {
  const double2 v = *(const double2 *)p;
  return {v.x, v.y};
}
FSE_DEV Cplx<float> load_cplx(const Cplx<float> *p) {
  const float2 v = *(const float2 *)p;
  return {v.x, v.y};
}

// floor(i / n) for 0 <= i < 2^24, n >= 1 (float reciprocal + one correction)
FSE_DEV int div_small(int i, int n, float rn) {
  int q = __float2int_rz((float)i * rn);
  q -= q * n > i;
  q += (q + 1) * n <= i;
  return q;
}

template <typename T, int BPT>
__device__ void cfse_iterate_reg(const Cplx<T> *R0, const Cplx<T> *W, int M, int N, T gamma,
                                 T inv_w00, int iterations, double e0, int64_t *us, int64_t *vs,
                                 double *cs, double *es, double4 *cand) {
  typedef Ieee<T> F;
  constexpr int NW = kGenThreads / 32;
  const int MN = M * N, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const float rn = 1.0f / (float)N;
  const T damp = F::mul(gamma, F::sub((T)2.0, gamma));
  T e = (T)e0;
  Cplx<T> R[BPT];
  int kk[BPT], ll[BPT];
  T best = (T)-1.0, bre = (T)0.0, bim = (T)0.0;
  int bi = 0;
#pragma unroll
  for (int j = 0; j < BPT; ++j) {  // pass 0: load + scan
    const int i = tid + kGenThreads * j;
    kk[j] = i / N;
    ll[j] = i - kk[j] * N;
    if (i < MN) {
      R[j] = R0[i];
      T m2 = F::add(F::mul(R[j].re, R[j].re), F::mul(R[j].im, R[j].im));
      if (m2 > best) { best = m2; bi = i; bre = R[j].re; bim = R[j].im; }
    }
  }
  for (int it = 0; it < iterations; ++it) {
    double4 *slot = cand + (it & 1) * NW;
    const bool have = best >= (T)0;
    const unsigned widx = warp_first_max<T>(best, (unsigned)bi, have);
    if (have && (unsigned)bi == widx)
      slot[w] = make_double4((double)best, __longlong_as_double((long long)bi), (double)bre, (double)bim);
    if (lane == 0 && widx == 0xffffffffu)
      slot[w] = make_double4(-1.0, __longlong_as_double(-1ll), 0.0, 0.0);
    __syncthreads();
    const double4 c4 = lane < NW ? slot[lane] : make_double4(-1.0, __longlong_as_double(-1ll), 0.0, 0.0);
    const unsigned cidx = (unsigned)__double_as_longlong(c4.y);
    const unsigned gidx = warp_first_max<T>((T)c4.x, cidx, c4.x >= 0.0);
    const int ow = __ffs(__ballot_sync(0xffffffffu, lane < NW && cidx == gidx)) - 1;
    const T ar = (T)__shfl_sync(0xffffffffu, c4.z, ow);
    const T ai = (T)__shfl_sync(0xffffffffu, c4.w, ow);
    const int idx = (int)gidx;
    const int u = div_small(idx, N, rn), v = idx - u * N;
    // c = gamma * rw_uv * inv_w00 (cfse.py:85): (gamma*a)*inv_w00
    const T cr = F::mul(F::mul(gamma, ar), inv_w00);
    const T ci = F::mul(F::mul(gamma, ai), inv_w00);
    if (tid == 0) {
      // e -= damp * |rw_uv|^2 * inv_w00 (cfse.py:101)
      T m2 = F::add(F::mul(ar, ar), F::mul(ai, ai));
      e = F::sub(e, F::mul(F::mul(damp, m2), inv_w00));
      us[it] = u;
      vs[it] = v;
      cs[2 * it] = (double)cr;
      cs[2 * it + 1] = (double)ci;
      es[it] = (double)e;
    }
    if (it + 1 == iterations) break;
    // residual update (cfse.py:91-99) fused with the next pass's scan
    best = (T)-1.0;
    bi = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int i = tid + kGenThreads * j;
      if (i < MN) {
        int ks = kk[j] - u, ls = ll[j] - v;
        if (ks < 0) ks += M;
        if (ls < 0) ls += N;
        const Cplx<T> wv = load_cplx(W + ks * N + ls);
        Cplx<T> x = R[j];
        T pr = F::sub(F::mul(cr, wv.re), F::mul(ci, wv.im));
        T pi = F::add(F::mul(cr, wv.im), F::mul(ci, wv.re));
        x.re = F::sub(x.re, pr);
        x.im = F::sub(x.im, pi);
        R[j] = x;
        T m2 = F::add(F::mul(x.re, x.re), F::mul(x.im, x.im));
        if (m2 > best) { best = m2; bi = i; bre = x.re; bim = x.im; }
      }
    }
    // no trailing barrier: the candidate slots are double-buffered
  }
  __syncthreads();
}

// cfse_iterate_reg for windows that tile the CTA exactly (MN = 512 BPT,
// N | 512, M and N powers of two: every BASELINE size up to 64 x 64).
// Thread t owns bins t + 512 j: column l = t mod N for every j, rows
// k0 + (512/N) j.  W' comes from a row-extended table Wx = [W; W] (2M rows,
// built here in the caller's free buffer `wx`), so the shifted bins of a
// thread are one base address plus immediate strides -- no per-bin index
// arithmetic or wrap, no per-bin bounds branch.  Same per-thread scan order,
// IEEE ops and block reduction as cfse_iterate_reg (bit-identical results).
template <typename T, int BPT>
__device__ void cfse_iterate_tile(const Cplx<T> *R0, const Cplx<T> *W, Cplx<T> *wx, int M, int N, T gamma,
                                  T inv_w00, int iterations, double e0, int64_t *us, int64_t *vs,
                                  double *cs, double *es, double4 *cand) {
  typedef Ieee<T> F;
  constexpr int NW = kGenThreads / 32;
  const int MN = M * N, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int logN = __ffs(N) - 1;
  const T damp = F::mul(gamma, F::sub((T)2.0, gamma));
  T e = (T)e0;
  Cplx<T> R[BPT];
  T best = (T)-1.0, bre = (T)0.0, bim = (T)0.0;
  int bi = 0;
#pragma unroll
  for (int j = 0; j < BPT; ++j) {  // pass 0: load + scan
    const int i = tid + kGenThreads * j;
    R[j] = R0[i];
    T m2 = F::add(F::mul(R[j].re, R[j].re), F::mul(R[j].im, R[j].im));
    if (m2 > best) { best = m2; bi = i; bre = R[j].re; bim = R[j].im; }
  }
  __syncthreads();  // R0 may alias wx
  for (int i = tid; i < 2 * MN; i += kGenThreads) {
    const Cplx<T> x = W[i & (MN - 1)];
    wx[i] = x;
  }
  __syncthreads();
  const int k0 = tid >> logN, l0 = tid & (N - 1);
#ifdef FSE_GCLK
  long long ck[6] = {0, 0, 0, 0, 0, 0}, cl = clock64();
#define FSE_LCLK(j) do { const long long c2 = clock64(); ck[j] += c2 - cl; cl = c2; } while (0)
#else
#define FSE_LCLK(j) ((void)0)
#endif
  for (int it = 0; it < iterations; ++it) {
    double4 *slot = cand + (it & 1) * NW;
    int wl_own;
    warp_first_max_lane<T>(best, (unsigned)bi, true, wl_own);
    FSE_LCLK(0);
    if (lane == wl_own)
      slot[w] = make_double4((double)best, __longlong_as_double((long long)bi), (double)bre, (double)bim);
    FSE_LCLK(1);
    __syncthreads();
    FSE_LCLK(2);
    const double4 c4 = lane < NW ? slot[lane] : make_double4(-1.0, __longlong_as_double(-1ll), 0.0, 0.0);
    const unsigned cidx = (unsigned)__double_as_longlong(c4.y);
    int ow;
    const unsigned gidx = warp_first_max_lane<T>((T)c4.x, cidx, c4.x >= 0.0, ow);
    const T ar = (T)__shfl_sync(0xffffffffu, c4.z, ow);
    const T ai = (T)__shfl_sync(0xffffffffu, c4.w, ow);
    const int u = (int)gidx >> logN, v = (int)gidx & (N - 1);
    // c = gamma * rw_uv * inv_w00 (cfse.py:85): (gamma*a)*inv_w00
    const T cr = F::mul(F::mul(gamma, ar), inv_w00);
    const T ci = F::mul(F::mul(gamma, ai), inv_w00);
    FSE_LCLK(3);
    if (tid == 0) {
      // e -= damp * |rw_uv|^2 * inv_w00 (cfse.py:101)
      T m2 = F::add(F::mul(ar, ar), F::mul(ai, ai));
      e = F::sub(e, F::mul(F::mul(damp, m2), inv_w00));
      us[it] = u;
      vs[it] = v;
      cs[2 * it] = (double)cr;
      cs[2 * it + 1] = (double)ci;
      es[it] = (double)e;
    }
    if (it + 1 == iterations) break;
    // residual update (cfse.py:91-99) fused with the next pass's scan:
    // bin j of this thread reads Wx[((k0 - u) mod M + (512/N) j) N + (l0 - v) mod N]
    const Cplx<T> *wp = wx + ((((k0 - u) & (M - 1)) << logN) + ((l0 - v) & (N - 1)));
    best = (T)-1.0;
    bi = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      FSE_CHECK((wp - wx) + kGenThreads * j < 2 * MN);
      const Cplx<T> wv = load_cplx(wp + kGenThreads * j);
      Cplx<T> x = R[j];
      T pr = F::sub(F::mul(cr, wv.re), F::mul(ci, wv.im));
      T pi = F::add(F::mul(cr, wv.im), F::mul(ci, wv.re));
      x.re = F::sub(x.re, pr);
      x.im = F::sub(x.im, pi);
      R[j] = x;
      T m2 = F::add(F::mul(x.re, x.re), F::mul(x.im, x.im));
      const bool gt = m2 > best;
      best = gt ? m2 : best;
      bi = gt ? tid + kGenThreads * j : bi;
      bre = gt ? x.re : bre;
      bim = gt ? x.im : bim;
    }
    FSE_LCLK(4);
    // no trailing barrier: the candidate slots are double-buffered
  }
#ifdef FSE_GCLK
  if (tid == 0 && blockIdx.x == 0)
    printf("iteration phases (thread 0, cycles/iter): warp argmax %lld, publish %lld, barrier %lld, merge+c %lld, update+scan %lld\n",
           ck[0] / iterations, ck[1] / iterations, ck[2] / iterations, ck[3] / iterations, ck[4] / iterations);
#endif
#undef FSE_LCLK
  __syncthreads();
}

// rFSE loop (rfse.py:58-167): per iteration a scan of every bin with the
// joint projection onto the conjugate pair {phi, conj(phi)} (variable
// denominators D = w00^2 - |W[2k,2l]|^2, self-conjugate bins on their own
// branch), selection of the maximal exact energy decrease, canonical pair
// member, and a two-term residual update.  Unfused IEEE ops in the numba
// order, so fp64 results are bit-identical given the same spectra.
template <typename T>
__device__ void rfse_iterate(Cplx<T> *R, const Cplx<T> *W, int M, int N, T gamma, T w00,
                             int max_iters, int stop_tally, double e0, int64_t *us, int64_t *vs,
                             double *cs, double *es, int32_t *selfs, int32_t *out_count,
                             int32_t *out_tally, T *sv, int *si, double4 *bcast) {
  typedef Ieee<T> F;
  const int MN = M * N;
  const T damp = F::mul(gamma, F::sub((T)2.0, gamma));
  const T w00sq = F::mul(w00, w00);
  T e = (T)e0;
  int count = 0, tally = 0;
  while (count < max_iters && tally < stop_tally) {
    T best = (T)-1.0;
    int bi = 0;
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      const int k = i / N, l = i - k * N;
      const Cplx<T> a = R[i];
      T crit;
      if ((2 * k) % M == 0 && (2 * l) % N == 0) {
        const T pr = F::div(a.re, w00);
        crit = F::mul(a.re, pr);
      } else {
        const Cplx<T> w2 = W[((2 * k) % M) * N + (2 * l) % N];
        const T nr = F::sub(F::mul(w00, a.re), F::add(F::mul(w2.re, a.re), F::mul(w2.im, a.im)));
        const T ni = F::sub(F::mul(w00, a.im), F::sub(F::mul(w2.im, a.re), F::mul(w2.re, a.im)));
        const T d = F::sub(w00sq, F::add(F::mul(w2.re, w2.re), F::mul(w2.im, w2.im)));
        const T pr = F::div(nr, d), pi = F::div(ni, d);
        crit = F::mul((T)2.0, F::add(F::mul(pr, a.re), F::mul(pi, a.im)));
      }
      if (crit > best) { best = crit; bi = i; }
    }
    block_argmax(best, bi, sv, si);
    if (threadIdx.x == 0) bcast[0] = make_double4((double)best, 0.0, 0.0, __longlong_as_double((long long)bi));
    __syncthreads();
    const double4 b0 = bcast[0];
    const int idx = (int)__double_as_longlong(b0.w);
    const T bestv = (T)b0.x;
    int u = idx / N, v = idx - u * N;
    const bool bself = (2 * u) % M == 0 && (2 * v) % N == 0;
    // the projection of the winner, recomputed by every thread (identical ops)
    T bpr, bpi;
    {
      const Cplx<T> a = R[idx];
      if (bself) {
        bpr = F::div(a.re, w00);
        bpi = (T)0.0;
      } else {
        const Cplx<T> w2 = W[((2 * u) % M) * N + (2 * v) % N];
        const T nr = F::sub(F::mul(w00, a.re), F::add(F::mul(w2.re, a.re), F::mul(w2.im, a.im)));
        const T ni = F::sub(F::mul(w00, a.im), F::sub(F::mul(w2.im, a.re), F::mul(w2.re, a.im)));
        const T d = F::sub(w00sq, F::add(F::mul(w2.re, w2.re), F::mul(w2.im, w2.im)));
        bpr = F::div(nr, d);
        bpi = F::div(ni, d);
      }
    }
    __syncthreads();  // everyone has read R[idx] before it is updated
    int mu = (M - u) % M, mv = (N - v) % N;
    if (!bself && mu * N + mv < u * N + v) {  // canonical member (rfse.py:111-121)
      const int tu = u, tv = v;
      u = mu; v = mv; mu = tu; mv = tv;
      bpi = -bpi;
    }
    const T cr = F::mul(gamma, bpr), ci = F::mul(gamma, bpi);  // gamma * complex(bpr, bpi)
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      const int k = i / N, l = i - k * N;
      int ks = k - u, ls = l - v;
      if (ks < 0) ks += M;
      if (ls < 0) ls += N;
      const Cplx<T> w1 = W[ks * N + ls];
      Cplx<T> x = R[i];
      // t1 = c * W[ks, ls]
      const T t1r = F::sub(F::mul(cr, w1.re), F::mul(ci, w1.im));
      const T t1i = F::add(F::mul(cr, w1.im), F::mul(ci, w1.re));
      x.re = F::sub(x.re, t1r);
      x.im = F::sub(x.im, t1i);
      if (!bself) {
        int ks2 = k - mu, ls2 = l - mv;
        if (ks2 < 0) ks2 += M;
        if (ls2 < 0) ls2 += N;
        const Cplx<T> w2 = W[ks2 * N + ls2];
        // t2 = conj(c) * W[ks2, ls2]
        const T t2r = F::sub(F::mul(cr, w2.re), F::mul(-ci, w2.im));
        const T t2i = F::add(F::mul(cr, w2.im), F::mul(-ci, w2.re));
        x.re = F::sub(x.re, t2r);
        x.im = F::sub(x.im, t2i);
      }
      R[i] = x;
    }
    e = F::sub(e, F::mul(damp, bestv));
    if (threadIdx.x == 0) {
      us[count] = u;
      vs[count] = v;
      cs[2 * count] = (double)cr;
      cs[2 * count + 1] = (double)ci;
      es[count] = (double)e;
      selfs[count] = bself ? 1 : 0;
    }
    tally += bself ? 1 : 2;
    ++count;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_count = count;
    *out_tally = tally;
  }
  __syncthreads();
}

// ------------------------------------------------------- extrapolation
struct GenLayout {
  bool smem;
  size_t smem_bytes, ws_per_window;
  size_t off_A, off_B, off_R, off_W;  // byte offsets inside the buffer region
};

static GenLayout gen_layout(int M, int N, int precision) {
  GenLayout L{};
  size_t MN = (size_t)M * N;
  size_t fixed = (size_t)(M + N) * sizeof(double2) * 2 + 64 * sizeof(double) + 64 * sizeof(int) + 64 +
                 kCandBytes;
  fixed = (fixed + 255) & ~(size_t)255;
  size_t big = 2 * MN * sizeof(double2);
  if (precision == 1) big += 2 * MN * sizeof(float2);
  L.off_A = 0;
  L.off_B = MN * sizeof(double2);
  if (precision == 1) {
    L.off_R = 2 * MN * sizeof(double2);
    L.off_W = L.off_R + MN * sizeof(float2);
  } else {
    L.off_R = L.off_A;
    L.off_W = L.off_B;
  }
  if (fixed + big <= 200 * 1024) {
    L.smem = true;
    L.smem_bytes = fixed + big;
    L.ws_per_window = 0;
  } else {
    L.smem = false;
    L.smem_bytes = fixed;
    L.ws_per_window = (big + 255) & ~(size_t)255;
  }
  return L;
}

size_t generic_workspace_bytes(int count, int M, int N, int precision) {
  GenLayout L = gen_layout(M, N, precision);
  return L.ws_per_window * (size_t)count;
}

// FSE_GDIAG=k diagnostic builds: return after setup phase k (timing only);
// FSE_GCLK: thread 0 of window 0 prints the clock at every phase boundary
#ifdef FSE_GDIAG
#define FSE_GSTOP(k) \
  if ((k) == FSE_GDIAG) return
#elif defined(FSE_GCLK)
#define FSE_GSTOP(k)                                                        \
  do {                                                                      \
    if (threadIdx.x == 0) gclk[(k)] = clock64() - gclk0;                    \
    if ((k) == 7 && threadIdx.x == 0 && blockIdx.x == 0)                    \
      for (int q = 0; q < 8; ++q) printf("phase %d clock %lld\n", q, gclk[q]); \
  } while (0)
#else
#define FSE_GSTOP(k) ((void)0)
#endif

// SMEM: the window's work arrays live in shared memory (L.smem); a separate
// instantiation so every access to them compiles to LDS/STS rather than
// generic loads
template <typename T, int ALG, bool SMEM>
__global__ void __launch_bounds__(kGenThreads) extrapolate_kernel(GenArgs a, GenLayout L,
                                                                   char *workspace) {
  extern __shared__ __align__(16) char smem[];
  const int M = a.M, N = a.N, MN = M * N;
  const int win = blockIdx.x;
  double2 *twM = (double2 *)smem;           // forward tables exp(-2 pi i j / n)
  double2 *twN = twM + M;
  double2 *twMp = twN + N;                  // inverse tables exp(+2 pi i j / n)
  double2 *twNp = twMp + M;
  double *red = (double *)(twNp + N);
  int *redi = (int *)(red + 64);
  double4 *bcast = (double4 *)(redi + 64);
  double4 *cand = (double4 *)((char *)bcast + 64);  // 2 x 16 warp candidates
  size_t fixed = (size_t)(M + N) * sizeof(double2) * 2 + 64 * sizeof(double) + 64 * sizeof(int) + 64 +
                 kCandBytes;
  fixed = (fixed + 255) & ~(size_t)255;
  char *region = SMEM ? smem + fixed : workspace + (size_t)win * L.ws_per_window;
  double2 *A = (double2 *)(region + L.off_A);
  double2 *Bf = (double2 *)(region + L.off_B);
  Cplx<T> *R = (Cplx<T> *)(region + L.off_R);
  Cplx<T> *Wt = (Cplx<T> *)(region + L.off_W);

#ifdef FSE_GCLK
  const long long gclk0 = clock64();
  __shared__ long long gclk[8];
#endif
  const bool img = a.frames != nullptr;
  const double *s = img ? nullptr : a.signal + (size_t)win * MN;
  int wt = 0, wl = 0, off = 0;
  size_t fbase = 0;
  if (img) {
    off = (M - a.B) / 2;
    fbase = (size_t)a.blocks[3 * win] * (size_t)a.frame_stride;
    wt = a.blocks[3 * win + 1] - off;
    wl = a.blocks[3 * win + 2] - off;
  }
  // window sample i (image mode: from the frame, 0 outside it)
  auto sval = [&](int i) -> double {
    if (!img) return s[i];
    const int m = i / N, n = i - m * N, y = wt + m, x = wl + n;
    if (y < 0 || y >= a.H || x < 0 || x >= a.W) return 0.0;
    const size_t o = fbase + (size_t)y * a.pitch + x;
    return a.dtype == 0 ? (double)((const uint8_t *)a.frames)[o]
                        : a.dtype == 1 ? (double)((const float *)a.frames)[o] : ((const double *)a.frames)[o];
  };
  // output of window sample i: recon (every sample) or, in image mode, the
  // loss tile (u8: clamp + round half even)
  auto put = [&](int i, double v, bool loss) {
    if (!img) {
      a.recon[(size_t)win * MN + i] = loss ? v : s[i];
      return;
    }
    if (!loss) return;
    const int m = i / N, n = i - m * N;
    FSE_CHECK(m >= off && m < off + a.B && n >= off && n < off + a.B);
    const size_t o = (size_t)win * a.B * a.B + (size_t)(m - off) * a.B + (n - off);
    if (a.tile_dtype == 0)
      ((uint8_t *)a.tiles)[o] = (uint8_t)__double2int_rn(fmin(fmax(v, 0.0), 255.0));
    else if (a.tile_dtype == 1)
      ((float *)a.tiles)[o] = (float)v;
    else
      ((double *)a.tiles)[o] = v;
  };
  const int8_t *lab =
      a.labels + (size_t)(a.label_index ? a.label_index[win] : win) * a.labels_stride;
  int64_t *us = a.us + (size_t)win * a.iterations;
  int64_t *vs = a.vs + (size_t)win * a.iterations;
  double *cs = a.cs + (size_t)win * 2 * a.iterations;
  double *es = a.es + (size_t)win * a.iterations;

  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    twM[j] = twiddle(j, M, -1);
    twMp[j] = twiddle(j, M, +1);
  }
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    twN[j] = twiddle(j, N, -1);
    twNp[j] = twiddle(j, N, +1);
  }
  FSE_GSTOP(0);
  // kappa = 2^-e with max|s| = f 2^e, f in [0.5, 1): balances the two real
  // signals packed into one complex DFT; scaling by a power of two is exact.
  // Only support samples enter the transforms: loss / padding samples have
  // w = 0, so this equals the reference for finite input, and a non-finite
  // value in the lost block (common for decoded frames) cannot leak into
  // the window through 0 * NaN.
  // one pass over the window: w, s*w (unscaled) into A, max |s| over the
  // support and e0 = sum w s^2 (cfse.py:51); then one joint reduction and
  // the exact power-of-two scaling of the packed signal
  double smax = 0.0, e0p = 0.0;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    int m = i / N, n = i - m * N;
    const bool sup = lab[i] == kSupport;
    double w = !sup ? 0.0 : a.wtab ? a.wtab[(size_t)a.label_index[win] * a.labels_stride + i]
                                   : weight_at(m, n, M, N, a.rho);
    const double si = sup ? sval(i) : 0.0;
    smax = fmax(smax, fabs(si));
    A[i] = make_double2(w, si * w);
    e0p += w * si * si;
  }
  double e0 = e0p;
  block_max_sum(smax, e0, red);  // includes barriers
  FSE_GSTOP(1);
  int ex = 0;
  if (smax > 0.0) frexp(smax, &ex);
  const double kappa = ldexp(1.0, -ex), inv_kappa = ldexp(1.0, ex);
  for (int i = threadIdx.x; i < MN; i += blockDim.x) A[i].y *= kappa;  // exact
  __syncthreads();
  FSE_GSTOP(2);
  // power-of-two sizes: in-place radix-2 FFTs (log-depth, a few us for 64 x
  // 64); other sizes: the separable direct DFT
  const int logM = ilog2_pow2(M), logN = ilog2_pow2(N);
  const bool pow2 = logM >= 0 && logN >= 0;
  if (M == 64 && N == 64 && blockDim.x == 512) {  // register radix-8 x 8, Bf as exchange
    fft64_axis(A, Bf, false, false, twN);
    fft64_axis(A, Bf, true, false, twM);
  } else if (pow2) {
    if (N > 1) fft_axis(A, logN, logM, 1, N, twN);
    if (M > 1) fft_axis(A, logM, logN, N, 1, twM);
  } else {
    dft_rows(A, Bf, M, N, twN);
    __syncthreads();
    dft_cols(Bf, A, M, N, twM);
    __syncthreads();
  }
  unpack_two_real(A, Bf, M, N, inv_kappa);  // Bf = W, A = R_w
  FSE_GSTOP(3);
  __syncthreads();
  const double w00 = Bf[0].x;
  // rejected windows still write their output: the input outside the loss,
  // NaN on it (never stale memory).  Plans reject these geometries at
  // creation; the per-window status reports them to the direct API.
  if (w00 <= 1e-12 * (double)M * (double)N) {  // cfse.py:47-48
    for (int i = threadIdx.x; i < MN; i += blockDim.x) put(i, CUDART_NAN, lab[i] == kLoss);
    if (threadIdx.x == 0) a.status[win] = 1;
    return;
  }
  if (ALG == 1) {
    // rfse.py:50-54: pair Gram determinant must not be (nearly) singular
    int bad = 0;
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      const int k = i / N, l = i - k * N;
      if ((2 * k) % M == 0 && (2 * l) % N == 0) continue;
      const double2 w2 = Bf[((2 * k) % M) * N + (2 * l) % N];
      const double D = w00 * w00 - (w2.x * w2.x + w2.y * w2.y);
      if (D <= 1e-9 * w00 * w00) bad = 1;
    }
    if (__syncthreads_or(bad)) {
      for (int i = threadIdx.x; i < MN; i += blockDim.x) put(i, CUDART_NAN, lab[i] == kLoss);
      if (threadIdx.x == 0) a.status[win] = 2;
      return;
    }
  }
  if (threadIdx.x == 0) a.status[win] = 0;
  const double inv_w00 = 1.0 / w00;
  if (sizeof(T) == sizeof(float)) {
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      R[i].re = (T)A[i].x; R[i].im = (T)A[i].y;
      Wt[i].re = (T)Bf[i].x; Wt[i].im = (T)Bf[i].y;
    }
    __syncthreads();
  }
  int n_it = a.iterations;
  FSE_GSTOP(4);
  // the exactly-tiling register loop: MN = 512 BPT, N | 512, powers of two;
  // its row-extended W' table goes to the (then free) A buffer, which holds
  // 2 MN complex values for either precision (A + Bf for fp64)
  const int tile_bpt = pow2 && (MN % kGenThreads) == 0 && N <= kGenThreads ? MN / kGenThreads : 0;
  if (ALG == 0 && (tile_bpt == 8 || tile_bpt == 4 || tile_bpt == 2)) {
    Cplx<T> *wx = (Cplx<T> *)A;
    if (tile_bpt == 8)
      cfse_iterate_tile<T, 8>(R, Wt, wx, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, cand);
    else if (tile_bpt == 4)
      cfse_iterate_tile<T, 4>(R, Wt, wx, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, cand);
    else
      cfse_iterate_tile<T, 2>(R, Wt, wx, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, cand);
  } else if (ALG == 0 && MN <= kGenThreads * 8) {
    cfse_iterate_reg<T, 8>(R, Wt, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, cand);
  } else if (ALG == 0) {
    cfse_iterate<T>(R, Wt, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, nullptr,
                    (T *)red, redi, bcast);
  } else {
    rfse_iterate<T>(R, Wt, M, N, (T)a.gamma, (T)w00, a.iterations, a.stop_tally, e0, us, vs, cs, es,
                    a.selfs + (size_t)win * a.iterations, a.counts + win, a.tallies + win, (T *)red,
                    redi, bcast);
    n_it = a.counts[win];
  }
  // synthesis g = idft2(G) (cfse.py:126): G[u,v] += MN c in iteration order
  // (cfse.py:88; rFSE also adds MN conj(c) at the mirror bin, rfse.py:128-
  // 145), then inverse FFTs and 1/(MN) -- or, for other sizes, the direct
  // sum g = sum c e^{+2 pi i (u m/M + v n/N)} over the trace
  double *model = a.model ? a.model + (size_t)win * 2 * MN : nullptr;
  FSE_GSTOP(5);
  if (pow2 && img && !model && M == N && (kGenThreads % (a.B * a.B)) == 0) {
    // image mode needs Re{g} on the B x B loss tile only: a direct sum over
    // the trace there is ~10x cheaper than the inverse 2-D FFT of G.  TPP
    // threads per pixel split the iterations (strided) and meet by shuffles;
    // e^{2 pi i (u m + v n) / M} is one table lookup (M == N)
    __syncthreads();  // trace (global, written by thread 0) visible
    // stage (u, v, c, pair factor) in shared memory with one coalesced pass:
    // the sum below then reads broadcasts, not serial L2 round trips
    const bool staged = (size_t)n_it * sizeof(double4) <= (size_t)MN * sizeof(double2);
    double4 *tr4 = (double4 *)Bf;
    if (staged) {
      for (int it = threadIdx.x; it < n_it; it += blockDim.x) {
        const double f = (ALG == 1 && !a.selfs[(size_t)win * a.iterations + it]) ? 2.0 : 1.0;
        FSE_CHECK((it + 1) * sizeof(double4) <= (size_t)MN * sizeof(double2));
        tr4[it] = make_double4(cs[2 * it] * f, cs[2 * it + 1] * f, (double)us[it], (double)vs[it]);
      }
      __syncthreads();
    }
    const int BB = a.B * a.B, TPP = kGenThreads / BB;  // power of two (B is), <= 32 for B >= 4
    const int px = threadIdx.x / TPP, sub = threadIdx.x - px * TPP;
    const int m = off + px / a.B, n = off + px % a.B;
    double g = 0.0;
#pragma unroll 4
    for (int it = sub; it < n_it; it += TPP) {
      double4 t4;
      if (staged) {
        t4 = tr4[it];
      } else {
        const double f = (ALG == 1 && !a.selfs[(size_t)win * a.iterations + it]) ? 2.0 : 1.0;
        t4 = make_double4(cs[2 * it] * f, cs[2 * it + 1] * f, (double)us[it], (double)vs[it]);
      }
      const double2 ph = twMp[((int)t4.z * m + (int)t4.w * n) & (M - 1)];
      g += t4.x * ph.x - t4.y * ph.y;  // Re{c phi} (x2 for a conjugate pair)
    }
    for (int o = TPP >> 1; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if (sub == 0) put(m * N + n, g, true);
    FSE_GSTOP(6);
    FSE_GSTOP(7);
    return;
  }
  if (pow2) {
    __syncthreads();  // trace (global, written by thread 0) visible; A and Bf free
    // stage the trace in shared memory (Bf) with one coalesced pass, so the
    // in-order scatter below reads broadcasts instead of L2 round trips
    const bool staged = (size_t)n_it * 24 <= (size_t)MN * sizeof(double2);
    double2 *tc = (double2 *)Bf;
    int *ti = (int *)(tc + n_it), *tsf = ti + n_it;
    if (staged)
      for (int it = threadIdx.x; it < n_it; it += blockDim.x) {
        tc[it] = make_double2(cs[2 * it], cs[2 * it + 1]);
        ti[it] = (int)us[it] * N + (int)vs[it];
        tsf[it] = ALG == 1 ? a.selfs[(size_t)win * a.iterations + it] : 1;
      }
    for (int i = threadIdx.x; i < MN; i += blockDim.x) A[i] = make_double2(0.0, 0.0);
    __syncthreads();
    const double dmn = (double)MN;
    for (int it = 0; it < n_it; ++it) {  // each bin accumulated by one thread, in order
      const int idx = staged ? ti[it] : (int)us[it] * N + (int)vs[it];
      const double2 c = staged ? tc[it] : make_double2(cs[2 * it], cs[2 * it + 1]);
      const double cr = c.x, ci = c.y;
      FSE_CHECK(idx >= 0 && idx < MN);
      if ((idx & (kGenThreads - 1)) == (int)threadIdx.x) {
        A[idx].x = __dadd_rn(A[idx].x, __dmul_rn(dmn, cr));
        A[idx].y = __dadd_rn(A[idx].y, __dmul_rn(dmn, ci));
      }
      if (ALG == 1 && !(staged ? tsf[it] : a.selfs[(size_t)win * a.iterations + it])) {
        const int u = idx / N, v = idx - u * N;
        const int mi = ((M - u) & (M - 1)) * N + ((N - v) & (N - 1));
        if ((mi & (kGenThreads - 1)) == (int)threadIdx.x) {
          A[mi].x = __dadd_rn(A[mi].x, __dmul_rn(dmn, cr));
          A[mi].y = __dadd_rn(A[mi].y, __dmul_rn(dmn, -ci));
        }
      }
    }
    __syncthreads();
    if (M == 64 && N == 64 && blockDim.x == 512) {  // W no longer needed: Bf is the exchange
      fft64_axis(A, Bf, false, true, twN);
      fft64_axis(A, Bf, true, true, twM);
    } else {
      if (N > 1) fft_axis(A, logN, logM, 1, N, twNp);
      if (M > 1) fft_axis(A, logM, logN, N, 1, twMp);
    }
    FSE_GSTOP(6);
    const double sc = 1.0 / dmn;
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      const double gr = A[i].x * sc;
      if (model) { model[2 * i] = gr; model[2 * i + 1] = A[i].y * sc; }
      put(i, gr, lab[i] == kLoss);
    }
    FSE_GSTOP(7);
    return;
  }
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    const bool loss = lab[i] == kLoss;
    if (!loss && !model) { put(i, 0.0, false); continue; }
    int m = i / N, n = i - m * N;
    double gr = 0.0, gi = 0.0;
    for (int it = 0; it < n_it; ++it) {
      int u = (int)us[it], v = (int)vs[it];
      // (u, m < M <= 4096: the products fit 32 bits)
      double2 p = twMp[(u * m) % M], q = twNp[(v * n) % N];
      double pr = p.x * q.x - p.y * q.y, pi = p.x * q.y + p.y * q.x;
      double cr = cs[2 * it], ci = cs[2 * it + 1];
      gr += cr * pr - ci * pi;
      gi += cr * pi + ci * pr;
      if (ALG == 1 && !a.selfs[(size_t)win * a.iterations + it]) {
        // the conjugate member: conj(c) * phi_(-u,-v) = conj(c * phi_(u,v))
        gr += cr * pr - ci * pi;
        gi -= cr * pi + ci * pr;
      }
    }
    if (model) { model[2 * i] = gr; model[2 * i + 1] = gi; }
    put(i, gr, loss);
  }
}

cudaError_t launch_generic_extrapolate(const GenArgs &a, void *workspace, cudaStream_t st) {
  GenLayout L = gen_layout(a.M, a.N, a.precision);
  if (a.count <= 0) return cudaSuccess;
  cudaError_t e;
  auto launch = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)L.smem_bytes);
    if (e2 != cudaSuccess) return e2;
    kern<<<a.count, kGenThreads, L.smem_bytes, st>>>(a, L, (char *)workspace);
    return cudaGetLastError();
  };
  if (L.smem) {
    if (a.algorithm == 1)
      e = a.precision == 1 ? launch(extrapolate_kernel<float, 1, true>) : launch(extrapolate_kernel<double, 1, true>);
    else
      e = a.precision == 1 ? launch(extrapolate_kernel<float, 0, true>) : launch(extrapolate_kernel<double, 0, true>);
  } else {
    if (a.algorithm == 1)
      e = a.precision == 1 ? launch(extrapolate_kernel<float, 1, false>) : launch(extrapolate_kernel<double, 1, false>);
    else
      e = a.precision == 1 ? launch(extrapolate_kernel<float, 0, false>) : launch(extrapolate_kernel<double, 0, false>);
  }
  return e;
}

// --------------------------------------------- drop-in for _cfse_kernel
__global__ void __launch_bounds__(kGenThreads)
    cfse_kernel_f64(int M, int N, double *R, const double *W, long long w_stride, double gamma,
                    const double *inv_w00, int iterations, const double *e0, double *G, int64_t *us,
                    int64_t *vs, double *cs, double *es) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ double4 bcast[1];
  const int win = blockIdx.x, MN = M * N;
  Cplx<double> *Rw = (Cplx<double> *)(R + (size_t)win * 2 * MN);
  const Cplx<double> *Ww = (const Cplx<double> *)(W + (size_t)win * 2 * w_stride);
  double *Gw = G ? G + (size_t)win * 2 * MN : nullptr;
  if (Gw)
    for (int i = threadIdx.x; i < 2 * MN; i += blockDim.x) Gw[i] = 0.0;
  __syncthreads();
  cfse_iterate<double>(Rw, Ww, M, N, gamma, inv_w00[win], iterations, e0[win],
                       us + (size_t)win * iterations, vs + (size_t)win * iterations,
                       cs + (size_t)win * 2 * iterations, es + (size_t)win * iterations, Gw, sv, si,
                       bcast);
  // the reference applies the last residual update too (R_w is mutated in
  // place and visible to the caller, cfse.py:91-99)
  if (iterations > 0) {
    const int idx = (int)(us[(size_t)win * iterations + iterations - 1] * N +
                          vs[(size_t)win * iterations + iterations - 1]);
    const int u = idx / N, v = idx - u * N;
    const double cr = cs[(size_t)win * 2 * iterations + 2 * (iterations - 1)];
    const double ci = cs[(size_t)win * 2 * iterations + 2 * (iterations - 1) + 1];
    typedef Ieee<double> F;
    for (int i = threadIdx.x; i < MN; i += blockDim.x) {
      int k = i / N, l = i - k * N;
      int ks = k - u, ls = l - v;
      if (ks < 0) ks += M;
      if (ls < 0) ls += N;
      Cplx<double> w = Ww[ks * N + ls], x = Rw[i];
      double pr = F::sub(F::mul(cr, w.re), F::mul(ci, w.im));
      double pi = F::add(F::mul(cr, w.im), F::mul(ci, w.re));
      Rw[i].re = F::sub(x.re, pr);
      Rw[i].im = F::sub(x.im, pi);
    }
  }
}

cudaError_t launch_cfse_kernel_f64(int count, int M, int N, double *R, const double *W,
                                   long long w_stride, double gamma, const double *inv_w00,
                                   int iterations, const double *e0, double *G, int64_t *us,
                                   int64_t *vs, double *cs, double *es, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  cfse_kernel_f64<<<count, kGenThreads, 0, s>>>(M, N, R, W, w_stride, gamma, inv_w00, iterations,
                                                e0, G, us, vs, cs, es);
  return cudaGetLastError();
}

// ------------------------------------------------------------ dft2 / idft2
__global__ void __launch_bounds__(kGenThreads)
    dft2_kernel(int M, int N, const double *in, double *out, int inverse, double *tmp) {
  extern __shared__ __align__(16) char smem[];
  double2 *twM = (double2 *)smem, *twN = twM + M;
  const int sign = inverse ? +1 : -1;
  for (int j = threadIdx.x; j < M; j += blockDim.x) twM[j] = twiddle(j, M, sign);
  for (int j = threadIdx.x; j < N; j += blockDim.x) twN[j] = twiddle(j, N, sign);
  __syncthreads();
  const size_t MN = (size_t)M * N;
  const double2 *src = (const double2 *)in + blockIdx.x * MN;
  double2 *t = (double2 *)tmp + blockIdx.x * MN;
  double2 *dst = (double2 *)out + blockIdx.x * MN;
  dft_rows(src, t, M, N, twN);
  __syncthreads();
  dft_cols(t, dst, M, N, twM);
  if (inverse) {
    __syncthreads();
    const double sc = 1.0 / (double)MN;
    for (size_t i = threadIdx.x; i < MN; i += blockDim.x) {
      double2 x = dst[i];
      dst[i] = make_double2(x.x * sc, x.y * sc);
    }
  }
}

cudaError_t launch_dft2_f64(int count, int M, int N, const double *in, double *out, int inverse,
                            double *tmp, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  size_t sm = (size_t)(M + N) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(dft2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dft2_kernel<<<count, kGenThreads, sm, s>>>(M, N, in, out, inverse, tmp);
  return cudaGetLastError();
}

__global__ void build_weight_kernel(int M, int N, const int8_t *labels, double rho, double *w,
                                    long long total) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int r = (int)(i % ((long long)M * N));
  int m = r / N, n = r - m * N;
  w[i] = labels[i] == kSupport ? weight_at(m, n, M, N, rho) : 0.0;
}

cudaError_t launch_build_weight_f64(int count, int M, int N, const int8_t *labels, double rho,
                                    double *w, cudaStream_t s) {
  long long total = (long long)count * M * N;
  if (total <= 0) return cudaSuccess;
  build_weight_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(M, N, labels, rho, w, total);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kGenThreads)
    select_basis_kernel(int M, int N, const double *R, int64_t *uv) {
  __shared__ double sv[32];
  __shared__ int si[32];
  typedef Ieee<double> F;
  double best = -1.0;
  int bi = 0;
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) {
    double re = R[2 * i], im = R[2 * i + 1];
    double m2 = F::add(F::mul(re, re), F::mul(im, im));
    if (m2 > best) { best = m2; bi = i; }
  }
  block_argmax(best, bi, sv, si);
  if (threadIdx.x == 0) { uv[0] = bi / N; uv[1] = bi % N; }
}

cudaError_t launch_select_basis_f64(int M, int N, const double *R, int64_t *uv, cudaStream_t s) {
  select_basis_kernel<<<1, kGenThreads, 0, s>>>(M, N, R, uv);
  return cudaGetLastError();
}

__global__ void update_residual_kernel(int M, int N, double *R, const double *W, int u, int v,
                                       double cr, double ci) {
  typedef Ieee<double> F;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  int k = i / N, l = i - k * N;
  int ks = k - u, ls = l - v;
  ks %= M; if (ks < 0) ks += M;
  ls %= N; if (ls < 0) ls += N;
  double wr = W[2 * (ks * N + ls)], wi = W[2 * (ks * N + ls) + 1];
  double pr = F::sub(F::mul(cr, wr), F::mul(ci, wi));
  double pi = F::add(F::mul(cr, wi), F::mul(ci, wr));
  R[2 * i] = F::sub(R[2 * i], pr);
  R[2 * i + 1] = F::sub(R[2 * i + 1], pi);
}

cudaError_t launch_update_residual_f64(int M, int N, double *R, const double *W, int u, int v,
                                       double cr, double ci, cudaStream_t s) {
  int n = M * N;
  update_residual_kernel<<<(n + 255) / 256, 256, 0, s>>>(M, N, R, W, u, v, cr, ci);
  return cudaGetLastError();
}

// ---------------------------------------------------- image-level helpers
__global__ void pack_trace_kernel(const int64_t *us, const int64_t *vs, const double *cs,
                                  const double *es, const int32_t *counts, int n, int It,
                                  int32_t *uv, void *c, void *e, int c64) {
  const long long total = (long long)n * It;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int w = (int)(i / It), it = (int)(i - (long long)w * It);
    const bool used = !counts || it < counts[w];
    uv[2 * i] = used ? (int32_t)us[i] : -1;
    uv[2 * i + 1] = used ? (int32_t)vs[i] : -1;
    const double re = used ? cs[2 * i] : 0.0, im = used ? cs[2 * i + 1] : 0.0;
    const double en = used ? es[i] : 0.0;
    if (c64) {
      ((double *)c)[2 * i] = re; ((double *)c)[2 * i + 1] = im; ((double *)e)[i] = en;
    } else {
      ((float *)c)[2 * i] = (float)re; ((float *)c)[2 * i + 1] = (float)im; ((float *)e)[i] = (float)en;
    }
  }
}

cudaError_t launch_pack_trace(const int64_t *us, const int64_t *vs, const double *cs,
                              const double *es, const int32_t *counts, int n, int It,
                              int32_t *uv, void *c, void *e, int c64, cudaStream_t s) {
  const long long total = (long long)n * It;
  if (total <= 0) return cudaSuccess;
  const int grid = (int)std::min<long long>((total + 255) / 256, 4096);
  pack_trace_kernel<<<grid, 256, 0, s>>>(us, vs, cs, es, counts, n, It, uv, c, e, c64);
  return cudaGetLastError();
}

}  // namespace fse

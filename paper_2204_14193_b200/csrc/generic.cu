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

#include "common.cuh"
#include "dft.cuh"
#include "kernels.h"

namespace fse {

constexpr int kGenThreads = 512;

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
// memory loop, so per-thread first maxima, the block reduction and every
// IEEE op are identical (bit-exact); only W' is read from shared memory.
// The winner's residual value travels with the reduction, so one barrier
// per iteration publishes (value, index).
template <typename T>
__device__ void argmax_combine_v(T &v, int &i, T &re, T &im, T v2, int i2, T re2, T im2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; re = re2; im = im2; }
}

template <typename T, int BPT>
__device__ void cfse_iterate_reg(const Cplx<T> *R0, const Cplx<T> *W, int M, int N, T gamma,
                                 T inv_w00, int iterations, double e0, int64_t *us, int64_t *vs,
                                 double *cs, double *es, double *red) {
  typedef Ieee<T> F;
  static_assert(kGenThreads / 32 * 2 * sizeof(double2) <= 64 * sizeof(double), "winner slots");
  const int MN = M * N, tid = threadIdx.x;
  // the warp winners: (value re, im) and (|R|^2, index), 16 warps
  double2 *wa = (double2 *)red, *wb = wa + kGenThreads / 32;
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
  const int w = tid >> 5, lane = tid & 31;
  for (int it = 0; it < iterations; ++it) {
    for (int o = 16; o; o >>= 1) {
      const T v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      const T r2 = __shfl_xor_sync(0xffffffffu, bre, o), m2 = __shfl_xor_sync(0xffffffffu, bim, o);
      argmax_combine_v(best, bi, bre, bim, v2, i2, r2, m2);
    }
    if (lane == 0) {
      wa[w] = make_double2((double)bre, (double)bim);
      wb[w] = make_double2((double)best, __longlong_as_double((long long)bi));
    }
    __syncthreads();
    // every thread merges the 16 warp winners with the same total order
    // (larger |R|^2, then smaller index)
    T bv = (T)wb[0].x, ar = (T)wa[0].x, ai = (T)wa[0].y;
    int bidx = (int)__double_as_longlong(wb[0].y);
#pragma unroll 4
    for (int q = 1; q < kGenThreads / 32; ++q) {
      const double2 ca = wa[q], cb = wb[q];
      argmax_combine_v(bv, bidx, ar, ai, (T)cb.x, (int)__double_as_longlong(cb.y), (T)ca.x, (T)ca.y);
    }
    const int idx = bidx;
    const int u = idx / N, v = idx - u * N;
    const T cr = F::mul(F::mul(gamma, ar), inv_w00);
    const T ci = F::mul(F::mul(gamma, ai), inv_w00);
    if (tid == 0) {
      T m2 = F::add(F::mul(ar, ar), F::mul(ai, ai));
      e = F::sub(e, F::mul(F::mul(damp, m2), inv_w00));
      us[it] = u;
      vs[it] = v;
      cs[2 * it] = (double)cr;
      cs[2 * it + 1] = (double)ci;
      es[it] = (double)e;
    }
    if (it + 1 == iterations) break;
    best = (T)-1.0;
    bi = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int i = tid + kGenThreads * j;
      if (i < MN) {
        int ks = kk[j] - u, ls = ll[j] - v;
        if (ks < 0) ks += M;
        if (ls < 0) ls += N;
        const Cplx<T> wv = W[ks * N + ls];
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
    __syncthreads();  // winner slots reuse
  }
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
  size_t fixed = (size_t)(M + N) * sizeof(double2) * 2 + 64 * sizeof(double) + 64 * sizeof(int) + 64;
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

template <typename T, int ALG>
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
  size_t fixed = (size_t)(M + N) * sizeof(double2) * 2 + 64 * sizeof(double) + 64 * sizeof(int) + 64;
  fixed = (fixed + 255) & ~(size_t)255;
  char *region = L.smem ? smem + fixed : workspace + (size_t)win * L.ws_per_window;
  double2 *A = (double2 *)(region + L.off_A);
  double2 *Bf = (double2 *)(region + L.off_B);
  Cplx<T> *R = (Cplx<T> *)(region + L.off_R);
  Cplx<T> *Wt = (Cplx<T> *)(region + L.off_W);

  const double *s = a.signal + (size_t)win * MN;
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
  // kappa = 2^-e with max|s| = f 2^e, f in [0.5, 1): balances the two real
  // signals packed into one complex DFT; scaling by a power of two is exact.
  // Only support samples enter the transforms: loss / padding samples have
  // w = 0, so this equals the reference for finite input, and a non-finite
  // value in the lost block (common for decoded frames) cannot leak into
  // the window through 0 * NaN.
  double smax = block_max_abs(s, MN, red, lab, kSupport);
  int ex = 0;
  if (smax > 0.0) frexp(smax, &ex);
  const double kappa = ldexp(1.0, -ex), inv_kappa = ldexp(1.0, ex);
  double e0p = 0.0;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    int m = i / N, n = i - m * N;
    const bool sup = lab[i] == kSupport;
    double w = sup ? weight_at(m, n, M, N, a.rho) : 0.0;
    const double si = sup ? s[i] : 0.0;
    double sw = si * w;
    A[i] = make_double2(w, sw * kappa);
    e0p += w * si * si;  // np.sum(w * s * s), cfse.py:51
  }
  const double e0 = block_sum(e0p, red);  // includes barrier
  dft_rows(A, Bf, M, N, twN);
  __syncthreads();
  dft_cols(Bf, A, M, N, twM);
  __syncthreads();
  unpack_two_real(A, Bf, M, N, inv_kappa);  // Bf = W, A = R_w
  __syncthreads();
  const double w00 = Bf[0].x;
  // rejected windows still write their output: the input outside the loss,
  // NaN on it (never stale memory).  Plans reject these geometries at
  // creation; the per-window status reports them to the direct API.
  double *rec_out = a.recon + (size_t)win * MN;
  if (w00 <= 1e-12 * (double)M * (double)N) {  // cfse.py:47-48
    for (int i = threadIdx.x; i < MN; i += blockDim.x) rec_out[i] = lab[i] == kLoss ? CUDART_NAN : s[i];
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
      for (int i = threadIdx.x; i < MN; i += blockDim.x) rec_out[i] = lab[i] == kLoss ? CUDART_NAN : s[i];
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
  if (ALG == 0 && MN <= kGenThreads * 8) {
    cfse_iterate_reg<T, 8>(R, Wt, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, red);
  } else if (ALG == 0) {
    cfse_iterate<T>(R, Wt, M, N, (T)a.gamma, (T)inv_w00, a.iterations, e0, us, vs, cs, es, nullptr,
                    (T *)red, redi, bcast);
  } else {
    rfse_iterate<T>(R, Wt, M, N, (T)a.gamma, (T)w00, a.iterations, a.stop_tally, e0, us, vs, cs, es,
                    a.selfs + (size_t)win * a.iterations, a.counts + win, a.tallies + win, (T *)red,
                    redi, bcast);
    n_it = a.counts[win];
  }
  // synthesis g = sum c e^{+2 pi i (u m/M + v n/N)} and write-back
  double *rec = a.recon + (size_t)win * MN;
  double *model = a.model ? a.model + (size_t)win * 2 * MN : nullptr;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    const bool loss = lab[i] == kLoss;
    if (!loss && !model) { rec[i] = s[i]; continue; }
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
    rec[i] = loss ? gr : s[i];
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
  if (a.algorithm == 1)
    e = a.precision == 1 ? launch(extrapolate_kernel<float, 1>) : launch(extrapolate_kernel<double, 1>);
  else
    e = a.precision == 1 ? launch(extrapolate_kernel<float, 0>) : launch(extrapolate_kernel<double, 0>);
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
__global__ void gather_windows_kernel(const void *frames, int dtype, long long pitch,
                                      long long frame_stride, int H, int W, const int32_t *blocks,
                                      int F, int B, double *windows) {
  const int b = blockIdx.x;
  const int f = blocks[3 * b], top = blocks[3 * b + 1], left = blocks[3 * b + 2];
  const int off = (F - B) / 2, wt = top - off, wl = left - off;
  double *dst = windows + (size_t)b * F * F;
  for (int i = threadIdx.x; i < F * F; i += blockDim.x) {
    int m = i / F, n = i - m * F, y = wt + m, x = wl + n;
    double v = 0.0;
    if (y >= 0 && y < H && x >= 0 && x < W) {
      size_t idx = (size_t)f * frame_stride + (size_t)y * pitch + x;
      v = dtype == 0 ? (double)((const uint8_t *)frames)[idx]
                     : dtype == 1 ? (double)((const float *)frames)[idx] : ((const double *)frames)[idx];
    }
    dst[i] = v;
  }
}

cudaError_t launch_gather_windows(const void *frames, int dtype, long long pitch,
                                  long long frame_stride, int H, int W, const int32_t *blocks,
                                  int n, int F, int B, double *windows, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  gather_windows_kernel<<<n, 256, 0, s>>>(frames, dtype, pitch, frame_stride, H, W, blocks, F, B,
                                          windows);
  return cudaGetLastError();
}

__global__ void extract_tiles_kernel(const double *recon, int F, int B, void *tiles, int tile_dtype) {
  const int b = blockIdx.x, off = (F - B) / 2;
  for (int i = threadIdx.x; i < B * B; i += blockDim.x) {
    int r = i / B, c = i - r * B;
    double v = recon[(size_t)b * F * F + (size_t)(off + r) * F + off + c];
    size_t o = (size_t)b * B * B + i;
    if (tile_dtype == 0) {
      double cl = fmin(fmax(v, 0.0), 255.0);
      ((uint8_t *)tiles)[o] = (uint8_t)__double2int_rn(cl);
    } else if (tile_dtype == 1) {
      ((float *)tiles)[o] = (float)v;
    } else {
      ((double *)tiles)[o] = v;
    }
  }
}

cudaError_t launch_extract_tiles(const double *recon, int n, int F, int B, void *tiles,
                                 int tile_dtype, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  extract_tiles_kernel<<<n, 256, 0, s>>>(recon, F, B, tiles, tile_dtype);
  return cudaGetLastError();
}

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

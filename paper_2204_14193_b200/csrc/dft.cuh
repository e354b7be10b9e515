// dft.cuh -- separable direct DFT passes (fp64), shared by generic.cu and fast.cu.
#pragma once
#include "common.cuh"

namespace fse {

// ----------------------------------------------------------- DFT passes
// Separable direct DFT with exact integer index reduction; tw* tables hold
// exp(sign 2 pi i j / n).  Row pass: dst[m][l] = sum_n src[m][n] twN[l n % N].
inline __device__ void dft_rows(const double2 *src, double2 *dst, int M, int N, const double2 *twN) {
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) {
    int m = i / N, l = i - m * N;
    const double2 *row = src + (size_t)m * N;
    double sr = 0.0, si = 0.0;
    int j = 0;
    for (int n = 0; n < N; ++n) {
      double2 x = row[n], t = twN[j];
      sr += x.x * t.x - x.y * t.y;
      si += x.x * t.y + x.y * t.x;
      j += l;
      if (j >= N) j -= N;
    }
    dst[i] = make_double2(sr, si);
  }
}

// Column pass: dst[k][l] = sum_m src[m][l] twM[k m % M].
inline __device__ void dft_cols(const double2 *src, double2 *dst, int M, int N, const double2 *twM) {
  for (int i = threadIdx.x; i < M * N; i += blockDim.x) {
    int k = i / N, l = i - k * N;
    double sr = 0.0, si = 0.0;
    int j = 0;
    for (int m = 0; m < M; ++m) {
      double2 x = src[(size_t)m * N + l], t = twM[j];
      sr += x.x * t.x - x.y * t.y;
      si += x.x * t.y + x.y * t.x;
      j += k;
      if (j >= M) j -= M;
    }
    dst[i] = make_double2(sr, si);
  }
}

// ------------------------------------------------------------ radix-2 FFT
// In-place radix-2 FFTs (decimation in time) of length L = 2^logL along one
// axis of an array, batched over the other axis (2^logB transforms): element
// j of transform b sits at A[b * bs + j * es].  tw holds exp(sign 2 pi i j /
// L), j < L (exact twiddles from sincospi), so forward / inverse is the
// table.  Every thread of the block participates; barriers between stages.
// Rows (es = 1) map consecutive threads to consecutive butterflies, columns
// (es > 1) to consecutive transforms (conflict-free shared accesses); all
// index math is shifts and masks (sizes are powers of two, offsets < 2^31).
inline __device__ void fft_axis(double2 *A, int logL, int logB, int es, int bs, const double2 *tw) {
  const int L = 1 << logL, tot = L << logB;
  const bool rows = es == 1;
  for (int t = threadIdx.x; t < tot; t += blockDim.x) {
    const int b = rows ? t >> logL : t & ((1 << logB) - 1);
    const int j = rows ? t & (L - 1) : t >> logB;
    const int r = (int)(__brev((unsigned)j) >> (32 - logL));
    if (j < r) {
      double2 *p = A + b * bs;
      const double2 x = p[j * es];
      p[j * es] = p[r * es];
      p[r * es] = x;
    }
  }
  __syncthreads();
  const int nb = tot >> 1;
  for (int st = 1; st <= logL; ++st) {
    const int half = 1 << (st - 1);
#pragma unroll 4
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int b = rows ? t >> (logL - 1) : t & ((1 << logB) - 1);
      const int q = rows ? t & ((L >> 1) - 1) : t >> logB;
      const int k = q & (half - 1), i0 = ((q >> (st - 1)) << st) + k;
      const double2 w = tw[k << (logL - st)];
      double2 *p = A + b * bs;
      const double2 x0 = p[i0 * es], x1 = p[(i0 + half) * es];
      const double2 y = make_double2(w.x * x1.x - w.y * x1.y, w.x * x1.y + w.y * x1.x);
      p[i0 * es] = make_double2(x0.x + y.x, x0.y + y.y);
      p[(i0 + half) * es] = make_double2(x0.x - y.x, x0.y - y.y);
    }
    __syncthreads();
  }
}


// ------------------------------------------------ 64-point register FFT
// Length-64 FFTs along one axis of a 64 x 64 fp64 array, all 64 transforms
// of the axis at once by 512 threads (8 per transform): radix 8 x 8 with
// the 8 values of each lane in registers, one exchange through X (4096
// entries, XOR-swizzled so both exchange phases are conflict-free) -- the
// whole pass moves 4 x 64 KB through shared memory instead of 7 x 160 KB
// for radix 2.  cols: transforms run down the columns; inverse: conj in,
// conj out (unnormalised inverse).  tw = exp(-2 pi i j / 64), j < 64.
FSE_DEV double2 dcadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
FSE_DEV double2 dcsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
FSE_DEV double2 dcmi(double2 a) { return make_double2(a.y, -a.x); }  // -i a
FSE_DEV double2 dcmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
FSE_DEV void ddft8(double2 (&x)[8]) {
  const double s = 0.70710678118654752440;
  double2 a0 = dcadd(x[0], x[4]), a4 = dcsub(x[0], x[4]);
  double2 a1 = dcadd(x[1], x[5]), a5 = dcsub(x[1], x[5]);
  double2 a2 = dcadd(x[2], x[6]), a6 = dcsub(x[2], x[6]);
  double2 a3 = dcadd(x[3], x[7]), a7 = dcsub(x[3], x[7]);
  a5 = make_double2(s * (a5.x + a5.y), s * (a5.y - a5.x));   // * e^{-i pi/4}
  a6 = dcmi(a6);                                              // * -i
  a7 = make_double2(s * (a7.y - a7.x), -s * (a7.x + a7.y));   // * e^{-3i pi/4}
  double2 b0 = dcadd(a0, a2), b2 = dcsub(a0, a2), b1 = dcadd(a1, a3), b3 = dcmi(dcsub(a1, a3));
  double2 b4 = dcadd(a4, a6), b6 = dcsub(a4, a6), b5 = dcadd(a5, a7), b7 = dcmi(dcsub(a5, a7));
  x[0] = dcadd(b0, b1); x[4] = dcsub(b0, b1); x[2] = dcadd(b2, b3); x[6] = dcsub(b2, b3);
  x[1] = dcadd(b4, b5); x[5] = dcsub(b4, b5); x[3] = dcadd(b6, b7); x[7] = dcsub(b6, b7);
}

inline __device__ void fft64_axis(double2 *A, double2 *X, bool cols, bool inverse, const double2 *tw) {
  const int t = threadIdx.x;  // 512 threads
  // transform f, lane q: rows -> f = t >> 3, q = t & 7; cols -> f = t & 63, q = t >> 6
  const int f = cols ? (t & 63) : (t >> 3), q = cols ? (t >> 6) : (t & 7);
  // element n of transform f
  auto at = [&](int n) -> double2 & {
    FSE_CHECK(n >= 0 && n < 64 && f >= 0 && f < 64);
    return cols ? A[n * 64 + f] : A[f * 64 + n];
  };
  // exchange slot of (q1, k1) of transform f
  auto ex = [&](int q1, int k1) -> double2 & {
    return cols ? X[(q1 * 8 + k1) * 64 + f] : X[f * 64 + q1 * 8 + (k1 ^ q1)];
  };
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 x = at(q + 8 * k);
    v[k] = inverse ? make_double2(x.x, -x.y) : x;
  }
  ddft8(v);  // over k: v[k1] = sum_k x[q + 8 k] w8^{k k1}
#pragma unroll
  for (int k1 = 1; k1 < 8; ++k1) v[k1] = dcmul(v[k1], tw[q * k1]);
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) ex(q, k1) = v[k1];
  __syncthreads();
#pragma unroll
  for (int q1 = 0; q1 < 8; ++q1) v[q1] = ex(q1, q);  // this lane is k1 = q now
  ddft8(v);  // over q1: X[q + 8 k2] = v[k2]
  __syncthreads();
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) at(q + 8 * k2) = inverse ? make_double2(v[k2].x, -v[k2].y) : v[k2];
  __syncthreads();
}

inline __device__ int ilog2_pow2(int n) { return (n > 0 && (n & (n - 1)) == 0) ? __ffs(n) - 1 : -1; }

}  // namespace fse

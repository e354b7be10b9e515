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

}  // namespace fse

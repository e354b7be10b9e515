// common.cuh -- shared device helpers for the cFSE kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FSE_DEV __device__ __forceinline__

// FSE_CHECKS builds (tests only): device-side bounds checks on the shared and
// global indices of the kernels (compute-sanitizer is closed on this pool).
#ifdef FSE_CHECKS
#include <cassert>
#define FSE_CHECK(cond) assert(cond)
#else
#define FSE_CHECK(cond) ((void)0)
#endif

namespace fse {

constexpr int kPadding = 0;
constexpr int kSupport = 1;
constexpr int kLoss = 2;

// Unfused IEEE arithmetic (numba's complex ops are plain fmul/fsub/fadd with
// no FMA contraction).  The intrinsics below are
// never contracted by nvcc, whatever -fmad says.
template <typename T> struct Ieee;
template <> struct Ieee<double> {
  static FSE_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
  static FSE_DEV double add(double a, double b) { return __dadd_rn(a, b); }
  static FSE_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
  static FSE_DEV double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Ieee<float> {
  static FSE_DEV float mul(float a, float b) { return __fmul_rn(a, b); }
  static FSE_DEV float add(float a, float b) { return __fadd_rn(a, b); }
  static FSE_DEV float sub(float a, float b) { return __fsub_rn(a, b); }
  static FSE_DEV float div(float a, float b) { return __fdiv_rn(a, b); }
};

template <typename T> struct Cplx { T re, im; };

// exp(sign * 2 pi i * j / n), j in [0, n): exact argument reduction by the
// caller (j is an integer index), sincospi for a correctly rounded-ish angle.
FSE_DEV double2 twiddle(int j, int n, int sign) {
  double s, c;
  sincospi(2.0 * (double)j / (double)n, &s, &c);
  return make_double2(c, sign < 0 ? -s : s);
}

// (value, index) argmax combine: larger value wins, equal values -> smaller
// row-major index (the reference's first-max scan, cfse.py:68-79).
template <typename T>
FSE_DEV void argmax_combine(T &v, int &i, T v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

FSE_DEV unsigned lane_id() { return threadIdx.x & 31u; }

}  // namespace fse

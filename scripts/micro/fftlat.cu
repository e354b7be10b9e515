// clock64 timing of fft_axis (csrc/dft.cuh) on one CTA of 512 threads,
// 64 x 64 fp64 complex array in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2204_14193_b200/csrc/dft.cuh"
using namespace fse;

__global__ void k(double2 *out, long long *cyc) {
  extern __shared__ double2 sm[];
  double2 *A = sm, *twN = sm + 4096, *twM = twN + 64;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) A[i] = make_double2(i % 7, i % 5);
  for (int j = threadIdx.x; j < 64; j += blockDim.x) { twN[j] = twiddle(j, 64, -1); twM[j] = twN[j]; }
  __syncthreads();
  long long t0 = clock64();
  fft_axis(A, 6, 6, 1, 64, twN);
  long long t1 = clock64();
  fft_axis(A, 6, 6, 64, 1, twM);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = A[i];
}

int main() {
  double2 *o; long long *c;
  cudaMalloc(&o, 4096 * 16); cudaMalloc(&c, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  for (int r = 0; r < 3; ++r) {
    k<<<1, 512, (4096 + 128) * 16>>>(o, c);
    long long h[2];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("rows %lld cycles, cols %lld cycles\n", h[0], h[1]);
  }
  return 0;
}

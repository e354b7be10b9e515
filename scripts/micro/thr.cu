// Throughput: 512 threads x 8 independent chains of DFMA / FFMA / DADD, one CTA.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T *out, long long *cyc, int n) {
  T a[8];
  for (int j = 0; j < 8; ++j) a[j] = out[j] + threadIdx.x;
  const T y = (T)1.0000001, z = (T)0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = a[j] * y + z;
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  T s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  out[8 + threadIdx.x] = s;
}
int main() {
  double *o; long long *c;
  cudaMalloc(&o, 8 * 2048); cudaMalloc(&c, 64); cudaMemset(o, 0, 8 * 2048);
  int n = 2000;
  for (int r = 0; r < 2; ++r) {
    long long h;
    k<double><<<1, 512>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fp64: %.2f DFMA per clk per SM\n", 512.0 * 8 * n / h);
    k<float><<<1, 512>>>((float *)o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fp32: %.2f FFMA per clk per SM\n", 512.0 * 8 * n / h);
  }
  return 0;
}

// Latency microbenchmarks on one SM (clock64 deltas): dependent DFMA / FFMA /
// DMUL chains, dependent LDS.128 pointer chase, __syncthreads with 512
// threads, fp64 sincospi, generic vs shared loads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, long long *cyc, int n) {
  __shared__ double2 sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = make_double2(i, 1.0); idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = out[0] + threadIdx.x, y = 1.0000001;
  float fx = (float)x, fy = 1.0000001f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) fx = fmaf(fx, fy, 0.5f);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t3 = clock64();
  int j = threadIdx.x & 1023;
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t5 = clock64();
  double s = 0, c = 0;
  for (int i = 0; i < 64; ++i) { double a, b; sincospi(2.0 * (i + x * 1e-30) / 64.0, &a, &b); s += a; c += b; }
  long long t6 = clock64();
  double2 acc = make_double2(0, 0);
  int jj = threadIdx.x;
  for (int i = 0; i < n; ++i) { double2 v = sm[jj]; acc.x += v.x; jj = ((int)v.y + jj) & 1023; }
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
  }
  out[1 + threadIdx.x] = x + fx + j + s + c + acc.x;
}

int main() {
  double *o; long long *c;
  cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  cudaMemset(o, 0, 8 * 1024);
  int n = 1000;
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(o, c, n);
    long long h[7];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads %d: per op cycles: dfma %.1f ffma %.1f dmul %.1f lds-chase %.1f bar %.1f sincospi(64 calls) %.0f per call; lds.128+dadd chain %.1f\n",
           threads, h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / 64.0, h[6] / (double)n);
  }
  return 0;
}

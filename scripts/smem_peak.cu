// Microbenchmarks for the roofline denominators of the fused cFSE kernel:
//   lds128      : pure shared-memory read bandwidth (LDS.128, conflict-free)
//   lds_ffma2   : LDS.128 + the loop's 6 packed FP32 ops per 16 B (no argmax)
//   lds_full    : + the loop's 5 ALU ops per 16 B (first-max bookkeeping)
//   ffma2       : packed FP32 FMA throughput
// One CTA per SM x 640 / 512 threads with 16 pairs per thread, and x 384
// threads with 32 pairs per thread (the F=64 kernel's current occupancy).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_peak smem_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

template <int mode, int NPR = 16>
__global__ void __launch_bounds__(NPR == 16 ? 640 : 384, 1) lds128(float4 *out) {
  extern __shared__ float4 sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = tid & 31, w = tid >> 5;
  float2 acc[NPR], acc2[NPR];
  for (int p = 0; p < NPR; ++p) { acc[p] = make_float2(p, 1); acc2[p] = make_float2(1, p); }
  float best = -1.f, bx = 0.f;
  int bp = 0;
  const float c0 = 0.001f * tid, c1 = 0.002f;
  for (int it = 0; it < ITERS; ++it) {
    const float4 *base = sm + ((w * 16 + it) & 63) * 64 + ((lane + it) & 63);
#pragma unroll
    for (int p = 0; p < NPR; ++p) {
      float4 v;
      if (mode == 3) {  // the same 16 B as two LDS.64 from planar halves
        const float2 *b2 = (const float2 *)sm + 2 * (((w * 16 + it) & 63) * 64 + ((lane + it) & 63));
        float2 lo = b2[(p & 7) * 128 + (p >> 3) * 64];
        float2 hi = b2[(p & 7) * 128 + (p >> 3) * 64 + 8192 / 2];
        v = make_float4(lo.x, lo.y, hi.x, hi.y);
      } else {
        v = base[(p & 7) * 64 + ((p >> 3) & 1) * 32 + (p >> 4) * 512];
      }
      if (mode >= 1) {
        float2 wr = make_float2(v.x, v.y), wi = make_float2(v.z, v.w);
        acc[p] = __ffma2_rn(wr, make_float2(-c0, -c0), acc[p]);
        acc[p] = __ffma2_rn(wi, make_float2(c1, c1), acc[p]);
        acc2[p] = __ffma2_rn(wi, make_float2(-c0, -c0), acc2[p]);
        acc2[p] = __ffma2_rn(wr, make_float2(-c1, -c1), acc2[p]);
        float2 mg = __ffma2_rn(acc2[p], acc2[p], __fmul2_rn(acc[p], acc[p]));
        if (mode == 2) {
          float m = fmaxf(mg.x, mg.y);
          if (m > best) { best = m; bp = p; bx = mg.x; }
        } else {
          best += mg.x;
        }
      } else {
        acc[p].x += v.x + v.w;
        acc[p].y += v.y + v.z;
      }
    }
  }
  float s = best + bx + bp;
  for (int p = 0; p < NPR; ++p) s += acc[p].x + acc[p].y + acc2[p].x + acc2[p].y;
  if (s == 12345.f) out[tid] = make_float4(s, 0, 0, 0);
}

// pure read bandwidth at 8 B and 4 B per lane (same bytes per iteration)
template <int BYTES>
__global__ void __launch_bounds__(640, 1) ldsw(float4 *out) {
  extern __shared__ float4 sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = tid & 31, w = tid >> 5;
  float a = 0.f, b = 0.f;
  constexpr int PER = 16 * 16 / BYTES;  // loads per iteration (256 B per lane)
  for (int it = 0; it < ITERS; ++it) {
    if (BYTES == 8) {
      const float2 *base = (const float2 *)sm + ((w * 16 + it) & 63) * 128 + ((lane + it) & 63);
#pragma unroll
      for (int p = 0; p < PER; ++p) { float2 v = base[(p & 15) * 128 + (p >> 4) * 64]; a += v.x; b += v.y; }
    } else {
      const float *base = (const float *)sm + ((w * 16 + it) & 63) * 256 + ((lane + it) & 127);
#pragma unroll
      for (int p = 0; p < PER; ++p) { float v = base[(p & 31) * 256 + (p >> 5) * 128]; a += v; }
    }
  }
  if (a + b == 12345.f) out[tid] = make_float4(a, b, 0, 0);
}

__global__ void ffma2k(float2 *out) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x, i);
  const float2 b = make_float2(0.999f, 0.998f), c = make_float2(0.001f, 0.002f);
  for (int it = 0; it < ITERS * 4; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) out[threadIdx.x] = make_float2(s, 0);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float4 *out;
  cudaMalloc(&out, 1 << 20);
  void (*kern[4])(float4 *) = {lds128<0>, lds128<1>, lds128<2>, lds128<3>};
  for (auto k : kern) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *names[] = {"lds128", "lds128+6ffma2", "lds128+6ffma2+argmax", "2xlds64+6ffma2"};
  for (int threads : {512, 640}) {
    for (int mode = 0; mode < 4; ++mode) {
      kern[mode]<<<sms, threads, 131072>>>(out);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) kern[mode]<<<sms, threads, 131072>>>(out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
      double bytes = 5.0 * sms * threads * (double)ITERS * 16 * 16;
      double tbs = bytes / (ms * 1e-3) / 1e12;
      printf("{\"test\": \"%s\", \"threads\": %d, \"smem_TBps\": %.3f, \"bytes_per_clk_per_sm\": %.1f}\n",
             names[mode], threads, tbs, tbs * 1e12 / sms / (clk * 1e3));
    }
  }
  {  // 384 threads x 32 pairs (F=64 kernel occupancy): LDS.128 + mix, + argmax
    void (*k32[3])(float4 *) = {lds128<0, 32>, lds128<1, 32>, lds128<2, 32>};
    const char *n32[] = {"lds128_p32", "lds128+6ffma2_p32", "lds128+6ffma2+argmax_p32"};
    for (int mode = 0; mode < 3; ++mode) {
      cudaFuncSetAttribute(k32[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
      k32[mode]<<<sms, 384, 131072>>>(out);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k32[mode]<<<sms, 384, 131072>>>(out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
      double bytes = 5.0 * sms * 384 * (double)ITERS * 32 * 16;
      double tbs = bytes / (ms * 1e-3) / 1e12;
      printf("{\"test\": \"%s\", \"threads\": 384, \"smem_TBps\": %.3f, \"bytes_per_clk_per_sm\": %.1f}\n",
             n32[mode], tbs, tbs * 1e12 / sms / (clk * 1e3));
    }
  }
  cudaFuncSetAttribute(ldsw<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(ldsw<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int bw : {8, 4}) {
    auto k = bw == 8 ? ldsw<8> : ldsw<4>;
    k<<<sms, 640, 131072>>>(out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<sms, 640, 131072>>>(out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 5.0 * sms * 640 * (double)ITERS * 256;
    double tbs = bytes / (ms * 1e-3) / 1e12;
    printf("{\"test\": \"lds%d\", \"threads\": 640, \"smem_TBps\": %.3f, \"bytes_per_clk_per_sm\": %.1f}\n",
           bw * 8, tbs, tbs * 1e12 / sms / (clk * 1e3));
  }
  ffma2k<<<sms * 4, 512>>>((float2 *)out);
  cudaEventRecord(e0);
  ffma2k<<<sms * 4, 512>>>((float2 *)out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = (double)sms * 4 * 512 * ITERS * 4 * 8 * 4;  // 2 FMAs x 2 flops per FFMA2
  printf("{\"test\": \"ffma2\", \"fp32_TFLOPs\": %.2f, \"flops_per_clk_per_sm\": %.1f, \"sm_clock_mhz_attr\": %d}\n",
         flops / (ms * 1e-3) / 1e12, flops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  return 0;
}

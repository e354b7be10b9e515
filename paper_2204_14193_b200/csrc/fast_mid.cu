// fast_mid.cu -- latency build of the fused kernel for mid-size F = 64 cFSE
// plans (one wave of five blocks per SM): 32 bins per thread, four warps per
// block, five blocks per CTA (384 blocks 131 -> 112 us; DESIGN 4.2).  Same
// source as fast.cu, compiled into fse::s32 (see fast_small.cu).
#define FSE_FAST_NS s32
#define FSE_FAST_ONLY64 1
#define FSE_BPT64 32
#define FSE_SLOTS64 5
#define FSE_GROUPMAX64 0
#define FSE_PREFETCH64 2
#define FSE_SYN_GT 16  // synthesis on the throughput build's thread layout: same pixels bit for bit
#include "fast.cu"

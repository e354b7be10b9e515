// fast_small.cu -- latency build of the fused kernel for small F = 64 cFSE
// plans (at most two blocks per SM): 16 bins per thread, eight warps per
// block, two blocks per CTA.  A lone block's iteration is dependency-bound
// (each warp alone on its SM sub-partition), so spreading its 4096 bins over
// four times the warps shortens the scan more than the eight-warp argmax
// merge lengthens the tail: 256 blocks (config 2) 112 -> 91 us, 64 blocks
// 106 -> 79 us (DESIGN 4.2, profiles/r02/batch_sweep.jsonl).  The same
// source as fast.cu, compiled into fse::s16 with these knobs; the planner
// (api.cpp) picks it by block count.
#define FSE_FAST_NS s16
#define FSE_FAST_ONLY64 1
#define FSE_BPT64 16
#define FSE_SLOTS64 2
#define FSE_GROUPMAX64 0
#define FSE_PREFETCH64 2
#define FSE_SYN_GT 16  // synthesis on the throughput build's thread layout: same pixels bit for bit
#include "fast.cu"

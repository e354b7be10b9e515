// fast.cu -- fused, register-resident fp32 cFSE kernel for F in {32,64,128}.
//
// One lost block per "slot" (a group of NT = F*F/BPT threads holding BPT
// spectrum bins each in registers: BPT = 32 at F=32, 64 at F=64/128); S
// slots per CTA share one shared-memory copy of their geometry class's
// weight spectrum W; one CTA per SM, persistent over a list of same-class
// rounds.
//
// Per block (all on chip):
//   load   s*w of the support window (TMA-staged u8 tile or direct loads)  cfse.py:50
//   FFT    real-input half-spectrum 2-D FFT in the slot's shared scratch   cfse.py:50
//   R_w -> registers, exactly Hermitian by construction
//   I x { R_w -= c W[k-u, l-v]  (FFMA2 on SoA bin pairs, W' from a
//                                row-extended shared table: one LDS.128
//                                per bin pair, no index wrap arithmetic)
//         |R_w|^2, per-thread first max, warp REDUX max/min, cross-warp
//         exchange through shared memory + named barrier
//         c = gamma/W00 * R_w[u,v] }                                cfse.py:67-105
//   synth  Re{sum c e^{+2 pi i (u m + v n)/F}} on the B x B loss pixels,
//          clamp/round to u8 (or f32/f64) tile                      cfse.py:126-129
//
// Bin -> thread mapping (slot thread st = 32 w + lane): warp w owns rows
// [w*RPW, (w+1)*RPW), lane owns columns lane + 32 h (h < CPL = F/32).  The
// BPT bins of a thread form BPT/2 SoA pairs (a, b), consecutive in the
// thread's row-major scan order (RPW = BPT/CPL):
//   F=32 : a = (2p, lane),                  b = (2p+1, lane)
//   F=64 : a = (RPW w + p, lane),           b = a + (0, 32)
//   F=128: a = (RPW w + p/2, lane+64(p&1)), b = a + (0, 32)
//
// Compile-time knobs (defaults = the measured best on config 5; each was
// A/B-measured with scripts/gpu_ab.sh, results in DESIGN.md section 4):
//   FSE_BPT32 / FSE_BPT64 / FSE_BPT128  bins per thread (32 / 64 / 64)
//   FSE_SLOTS64 / FSE_SLOTS32  blocks per CTA at F=64 / 32 (6 / 20)
//   FSE_PREFETCH / FSE_PREFETCH64 / FSE_PREFETCH128  table loads issued this
//                           many pairs ahead (2 / 2 / 0 = left to ptxas)
//   FSE_GROUPMAX32/64/128   first-max tracked per group of bin pairs (0 / 2 / 0)
//   FSE_GMAX3               group's last value inside the running FMNMX3 (1)
//   FSE_RESOLVE_SEL / FSE_IDXSHFL  F=64 tail: select-tree group resolution, whole-index shuffle (1 / 1)
//   FSE_CHAINS64 / FSE_CHAINS128  independent first-max chains (1 / 1)
//   FSE_XTREE               F=128 warp-candidate merge in registers (0)
//   FSE_MAX3 / FSE_PACKKEY  alternative first-max trackers (1 / 0)
//   FSE_RSYM / FSE_RTWIST   centred-frame rFSE at F=32/64; F=64 twisted pairs (1 / 1)
//   FSE_SYN_GT              synthesis threads per coefficient group (0 = all;
//                           16 in the F=64 latency builds: the throughput layout)
//   FSE_DIAG                diagnostic builds (bit 32: per-phase clock probe)
//   FSE_CHECKS              device asserts on every shared/global index
//   FSE_FAST_NS             latency builds (fast_small.cu): this file compiled
//                           again into fse::FSE_FAST_NS with other F=64 knobs,
//                           F=64 cFSE only (FSE_FAST_ONLY64)
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "common.cuh"
#include "dft.cuh"
#include "kernels.h"

namespace fse {
#ifdef FSE_FAST_NS
namespace FSE_FAST_NS {
#endif

template <int F> struct FG {
  static constexpr int LOG = F == 32 ? 5 : F == 64 ? 6 : 7;
#ifndef FSE_BPT64
#define FSE_BPT64 64  // F=64: 64 bins per thread, two warps per block (measured +9 % over 32)
#endif
#ifndef FSE_BPT128
#define FSE_BPT128 64  // F=128: 256 threads per block (+4.5 % over 32)
#endif
#ifndef FSE_BPT32
#define FSE_BPT32 32  // F=32: one warp per block (16: two warps, the latency build)
#endif
  static constexpr int BPT = F == 64 ? FSE_BPT64 : F == 128 ? FSE_BPT128 : FSE_BPT32;  // bins per thread
  static constexpr int NP = BPT / 2;      // SoA bin pairs per thread
  static constexpr int NT = F * F / BPT;  // threads per slot
  static constexpr int NW = NT / 32;      // warps per slot
  static constexpr int CPL = F / 32;      // columns per lane
  static constexpr int RPW = BPT / CPL;   // rows per warp
#ifndef FSE_SLOTS64
#define FSE_SLOTS64 6  // 6 x 64 threads, 168 registers (7 spills)
#endif
#ifndef FSE_SLOTS32
#define FSE_SLOTS32 20
#endif
  static constexpr int S = F == 32 ? FSE_SLOTS32 : F == 64 ? FSE_SLOTS64 : 1;
  static constexpr int CTA = NT * S;      // threads per CTA
  static constexpr bool PLANAR = F == 128;  // planar re/im table (pair table would not fit)
  // rows of the row-extended table: the thread walks rows rowoff + step*p
  static constexpr int TROWS = F == 32 ? F + 31 : F + RPW - 1;
  // class region: the complex W' table or the centred-frame Q table (below),
  // whichever is larger
  static constexpr size_t CPLX_BYTES =
      PLANAR ? (size_t)TROWS * F * 2 * sizeof(float) : (size_t)TROWS * F * sizeof(float4);
  static constexpr size_t SYM_BYTES =
      F == 128 ? (size_t)(2 * F - 1) * F * sizeof(float)
               : (size_t)(F == 32 ? 62 : 2 * F - 1) * (F == 32 ? 63 : F + 31) * sizeof(float2);
  static constexpr size_t TABLE_BYTES = ((CPLX_BYTES > SYM_BYTES ? CPLX_BYTES : SYM_BYTES) + 15) & ~(size_t)15;
  // real half-spectrum FFT scratch: max(F/2 x (F+1), F x (F/2+1)) complex
  static constexpr size_t SCRATCH = (((size_t)F * (F / 2 + 1) * sizeof(float2) + 15) & ~(size_t)15);
  static constexpr int B = F / 4;  // loss block edge (the planner's fast-path condition)
  // synthesis: SG groups of threads split the coefficients; their partial
  // pixel sums meet in a reduction buffer at the end of the scratch
  static constexpr int SG = F == 32 ? 1 : 4;
  static constexpr size_t SYN_RED = SG > 1 ? (size_t)SG * B * B * sizeof(float) : 0;
  // iterations whose trace (16 B) and synthesis coefficients (16 B) fit the scratch
  static constexpr int TRACE_CAP = (int)((SCRATCH - SYN_RED) / 32);
  // TMA window bytes (u8 support box: 32x24, 48x48, 64x64 at the configs)
  static constexpr size_t STAGE = F == 32 ? 1024 : F == 64 ? 2560 : 4096;
  // the length-F FFTs of the setup: QT lanes per FFT, VPT values per lane
  static constexpr int QT = F == 128 ? 8 : F / 8;
  static constexpr int VPT = F / QT;
  // transforms per lane group and pass: every row pair / column in one pass
  static constexpr int NFT = (F / 2) / (NT / QT);
  static constexpr size_t REGION = TABLE_BYTES;
  // centred-frame real table (mirror-symmetric classes): F = 32 / 64, SYM_R
  // x SYM_C float2 entries, rows i = r - (F - 1), columns j = c - (F - 1);
  // F = 128, SYM_R x F floats, columns j mod F (signs in the coefficients)
  static constexpr int SYM_R = F == 32 ? 62 : 2 * F - 1;
  static constexpr int SYM_C = F == 32 ? 63 : F == 64 ? F + 31 : F;
  static_assert((size_t)SYM_R * SYM_C * (PLANAR ? sizeof(float) : sizeof(float2)) <= TABLE_BYTES,
                "Q table fits");
};


FSE_DEV float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// acc = a * b + acc with the accumulator as a read-write PTX operand.  With
// the intrinsic form ptxas writes the result into the (dead) W' register
// pair and pays ~30 MOVs per iteration to rotate the loop-carried spectrum
// back into place; the tied operand keeps it in place.
FSE_DEV void ffma2_acc(float2 &acc, float2 a, float b) {
  unsigned long long r, x;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  unsigned long long bb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(x), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(r));
}
// acc = a * b + acc, b a register pair (per-member coefficients)
FSE_DEV void ffma2_acc2(float2 &acc, float2 a, float2 b) {
  unsigned long long r, x, bb;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(x), "l"(bb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(r));
}
FSE_DEV float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

#if FSE_DIAG & 32
// timing probe (scripts/slot_phase.py): phase timestamps of the current
// block by slot thread 0, written over the first trace coefficients after
// the block as T_j - T_0, j = 1..6
#define FSE_TMARK(j) (tmk[j] = (unsigned)clock())
#else
#define FSE_TMARK(j) ((void)0)
#endif

// three-input maximum (FMNMX3, sm_100)
FSE_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
#ifndef FSE_MAX3
// FMNMX3 running maximum: one op fewer per pair and one op on the loop-carried
// chain.  With the complex-table loop it measured -3 % (F=64); with the
// centred-frame loop +1.7 % (config 5), +3.6 % (F=32), +-0 (F=128)
#define FSE_MAX3 1
#endif
// first-max tracker step over bin pair p with |R|^2 = (mg.x, mg.y): the
// larger value strictly above the running maximum wins, member a on equal
// values (bxs keeps member a's value to resolve the member afterwards)
FSE_DEV void first_max(float &bst, int &bps, float &bxs, float2 mg, int p) {
#if FSE_MAX3
  const float nb = fmax3(bst, mg.x, mg.y);  // the running maximum is the only dependent op
  if (nb > bst) { bps = p; bxs = mg.x; }
  bst = nb;
#else
  const float m = fmaxf(mg.x, mg.y);
  if (m > bst) { bst = m; bps = p; bxs = mg.x; }
#endif
}

// Exchange-buffer accesses through 32-bit shared-window addresses (the two
// buffers differ in one address bit, so switching is an XOR).
FSE_DEV uint4 lds128u(unsigned addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
FSE_DEV void sts128u(unsigned addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// bytes per slot region: [stage] scratch | exchange x 2 | red[16] | mbarrier
template <int F> constexpr size_t slot_stride(bool tma) {
  return ((tma ? FG<F>::STAGE : 0) + FG<F>::SCRATCH + 2 * FG<F>::NW * sizeof(uint4) + 64 + 16 +
          511) & ~(size_t)511;
}

// 16-byte shared load at a 32-bit shared-window address (hot loop only)
FSE_DEV float4 lds128f(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// rFSE (conjugate-pair) variant of the fused kernel, F = 64 only: four
// blocks per CTA (the pair tables take the shared memory of two slots).
// Per class, after the W' table: RA4[r][c] = (A_a, A_b, C_a, C_b) and
// RA2[r][c] = (-D_a, -D_b) for the pair (r, c), (r, c + 32), c < 32, with
// the pair selection criterion of bin k written as a quadratic form of
// a = R_w[k]:  crit = A a.re^2 + C a.im^2 - D a.re a.im  (rfse.py:86-111).
// F = 32: sixteen one-warp blocks per CTA (the rFSE loop state needs up to
// 128 registers), tables for bins (2p, c), (2p + 1, c) of pair p, column c.
// F = 128: one block per CTA.  Its pair-criterion coefficients depend on the
// doubled frequency only: per doubled row (64) and lane, the lane's two
// doubled columns -- centred frame (alpha, beta), 32 KB; complex frame (A, C,
// -D), 48 KB -- a table each block copies into the tail of its FFT scratch
// after the setup (the W' / Q table fills the class region).
template <int F> constexpr int rf_slots() { return F == 32 ? 16 : F == 64 ? 4 : 1; }
// pair-criterion tables: F^2 / 2 bin pairs x (float4 + float2); F = 128 the
// centred alpha | beta halves, 64 doubled rows x 32 lanes x float2 each
template <int F> constexpr size_t rf_t2_bytes() {
  return F == 128 ? (size_t)64 * 32 * (sizeof(float4) + sizeof(float2))
                  : (size_t)F * F / 2 * (sizeof(float4) + sizeof(float2));
}
template <int F, int ALG> struct KS {  // per-algorithm launch shape
  static constexpr int S = ALG ? rf_slots<F>() : FG<F>::S;
  static constexpr int CTA = FG<F>::NT * S;
  static constexpr size_t REGION =
      ALG && F != 128 ? FG<F>::TABLE_BYTES + rf_t2_bytes<F>() : FG<F>::REGION;
};

FSE_DEV float lds32f(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
FSE_DEV float2 lds64f(unsigned addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

template <int F> struct SlotPtrs {
  float2 *scratch;  // F x F (non-alias) -- FFT, then trace
  uint4 *xch;       // 2 x NW candidates
  float4 *trace;    // iteration trace (u|v<<16, c.re, c.im, e)
  float *red;       // small reduction scratch
};

template <int F> FSE_DEV void slot_sync(int slot) {
  if (FG<F>::NW == 1) {
    __syncwarp();
  } else if (FG<F>::S == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(FG<F>::NT) : "memory");
  }
}

// ----------------------------------------------------- TMA + mbarrier
FSE_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
FSE_DEV void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
// one thread: expect `bytes` and start the 3-D tile load (OOB elements -> 0)
FSE_DEV void tma_window(void *dst, const CUtensorMap *map, uint64_t *bar, unsigned bytes, int x, int y,
                        int z) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
FSE_DEV void mbar_wait(uint64_t *bar, int phase) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

FSE_DEV float load_px(const void *frames, int dtype, size_t idx) {
#if FSE_DIAG & 4
  return 100.f + (float)(idx & 7);
#endif
  if (dtype == 0) return (float)__ldg((const uint8_t *)frames + idx);
  if (dtype == 1) return __ldg((const float *)frames + idx);
  return (float)__ldg((const double *)frames + idx);
}

// row-major bin index of pair p, member mem (0 = a, 1 = b) for thread (w, lane)
template <int F> FSE_DEV int bin_index(int w, int lane, int p, int mem) {
  if (F == 32) return (FG<32>::RPW * w + 2 * p + mem) * 32 + lane;
  if (F == 64) return (FG<64>::RPW * w + p) * 64 + lane + 32 * mem;
  return (FG<128>::RPW * w + (p >> 1)) * 128 + lane + 64 * (p & 1) + 32 * mem;
}

// the pair index / member / owning lane of a bin owned by warp w (uniform)
template <int F> FSE_DEV void decode_bin(int idx, int w, int &p, int &mem, int &lane) {
  if (F == 32) {
    int row = idx >> 5;
    p = (row - FG<32>::RPW * w) >> 1; mem = row & 1; lane = idx & 31;
  } else if (F == 64) {
    int row = idx >> 6;
    p = row - FG<64>::RPW * w; mem = (idx >> 5) & 1; lane = idx & 31;
  } else {
    int row = idx >> 7, c = idx & 127;
    p = 2 * (row - FG<128>::RPW * w) + (c >> 6); mem = (c >> 5) & 1; lane = c & 31;
  }
}

#define FSE_PICK(P)                                  \
  case P:                                            \
    if constexpr (P < NP) {                          \
      re = mem ? Rre[P].y : Rre[P].x;                \
      im = mem ? Rim[P].y : Rim[P].x;                \
    }                                                \
    break;

// Value of bin (pair p, member mem) of this thread; p is warp-uniform, so
// the switch is a uniform indirect branch (one BRX jump table: every case
// present, p < NP promised), not a select chain.
template <int NP>
FSE_DEV void pick_bin(const float2 (&Rre)[NP], const float2 (&Rim)[NP], int p, int mem, float &re,
                      float &im) {
  // exactly NP cases (empty extra cases would deepen the branch tree)
  if constexpr (NP > 16) {
    switch (p) {
      FSE_PICK(0) FSE_PICK(1) FSE_PICK(2) FSE_PICK(3) FSE_PICK(4) FSE_PICK(5) FSE_PICK(6)
      FSE_PICK(7) FSE_PICK(8) FSE_PICK(9) FSE_PICK(10) FSE_PICK(11) FSE_PICK(12) FSE_PICK(13)
      FSE_PICK(14) FSE_PICK(15) FSE_PICK(16) FSE_PICK(17) FSE_PICK(18) FSE_PICK(19) FSE_PICK(20)
      FSE_PICK(21) FSE_PICK(22) FSE_PICK(23) FSE_PICK(24) FSE_PICK(25) FSE_PICK(26) FSE_PICK(27)
      FSE_PICK(28) FSE_PICK(29) FSE_PICK(30) FSE_PICK(31)
      default:
        __builtin_unreachable();
    }
  } else {
    switch (p) {
      FSE_PICK(0) FSE_PICK(1) FSE_PICK(2) FSE_PICK(3) FSE_PICK(4) FSE_PICK(5) FSE_PICK(6)
      FSE_PICK(7) FSE_PICK(8) FSE_PICK(9) FSE_PICK(10) FSE_PICK(11) FSE_PICK(12) FSE_PICK(13)
      FSE_PICK(14) FSE_PICK(15)
      default:
        __builtin_unreachable();
    }
  }
}

#ifndef FSE_GROUPMAX32
#define FSE_GROUPMAX32 FSE_GROUPMAX
#endif
#ifndef FSE_GROUPMAX64
#ifdef FSE_GROUPMAX
#define FSE_GROUPMAX64 FSE_GROUPMAX
#else
// F=64: groups of 2 bin pairs (with the centred-frame loop: 7.88 -> 8.21 M
// blocks/s on config 5 at a table prefetch depth of 4; with the FMNMX3 group
// step (FSE_GMAX3) the best depth is 2 again: 8.36 M; bitwise identical tiles
// and traces throughout)
#define FSE_GROUPMAX64 2
#endif
#endif
#ifndef FSE_RTWIST
// F=64 centred rFSE: "twisted" register pairs A = (re_a, im_b), B = (im_a, re_b)
// so the pair criterion alpha re^2 + beta im^2 (member b: alpha and beta
// swapped, its doubled column wraps) is alpha A^2 + beta B^2 with scalar
// coefficients: one LDS.64 (alpha, beta) per pair instead of an LDS.128
#define FSE_RTWIST 1
#endif
#ifndef FSE_PREFETCH64
#define FSE_PREFETCH64 2  // F=64 table-load prefetch depth (4 before the FMNMX3 group step)
#endif
#ifndef FSE_GROUPMAX128
#define FSE_GROUPMAX128 FSE_GROUPMAX
#endif
#ifndef FSE_GROUPMAX
// first-max tracking per group of GM bin pairs: the group's maximum by a
// three-input max tree (2 GM values, ~GM ops), then one compare + two
// selects against the running maximum -- ~1.75 ALU ops per pair at GM = 4
// instead of 5 for a per-pair tracker.  The exact first bin inside the
// winning group is resolved after the warp maximum is known (bitwise the
// same |R|^2 ops as the scan; scripts/ab_bitwise.py: identical tiles and
// traces).  Measured slower at every size (config 5: 7.07 -> 6.29 M
// blocks/s at GM = 4, 5.64 at GM = 8; F = 128: 1.20 -> 1.13 M): the longer
// per-iteration tail costs more than the ALU ops it saves.  0 = per pair.
#define FSE_GROUPMAX 0
#endif

// |R|^2 of the SoA pair p (the scan's exact instruction sequence)
template <int NP> FSE_DEV float2 mag2(const float2 (&Rre)[NP], const float2 (&Rim)[NP], int p) {
  float2 mg = __fmul2_rn(Rre[p], Rre[p]);
  return __ffma2_rn(Rim[p], Rim[p], mg);
}

// maximum of the 2 GM |R|^2 values of a group (exact: returns one input)
template <int GM> FSE_DEV float group_max(const float (&v)[2 * GM]) {
  if constexpr (GM == 4) {
    return fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmaxf(v[6], v[7]));
  } else if constexpr (GM == 2) {
    return fmaxf(fmax3(v[0], v[1], v[2]), v[3]);
  } else {
    float t = v[0];
#pragma unroll
    for (int i = 1; i < 2 * GM; ++i) t = fmaxf(t, v[i]);
    return t;
  }
}

#ifndef FSE_GMAX3
// 1: the running maximum takes the group's last value in its FMNMX3 (one op on
// the loop-carried chain, one ALU op fewer per group); 0: group maximum, then
// compare and select against the running maximum.  Same result either way.
#define FSE_GMAX3 1  // F=64 config 5: 8.15 -> 8.36 M blocks/s (bitwise identical)
#endif
// first-max step over a completed group g: bst = max(bst, group), bg = g when
// the group holds a value strictly above the previous maximum
template <int GM> FSE_DEV void group_step(const float (&v)[2 * GM], float &bst, int &bg, int g) {
  if constexpr (FSE_GMAX3 && GM == 2) {
    const float nb = fmax3(fmax3(v[0], v[1], v[2]), v[3], bst);
    if (nb > bst) bg = g;
    bst = nb;
  } else if constexpr (FSE_GMAX3 && GM == 4) {
    const float nb = fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmax3(v[6], v[7], bst));
    if (nb > bst) bg = g;
    bst = nb;
  } else {
    const float t = group_max<GM>(v);
    if (t > bst) { bst = t; bg = g; }
  }
}

// copy group G0's GM SoA pairs out of the spectrum registers
template <int GM, int G0, int NP>
FSE_DEV void group_copy(const float2 (&Rre)[NP], const float2 (&Rim)[NP], float2 (&gr)[GM],
                        float2 (&gi)[GM]) {
#pragma unroll
  for (int q = 0; q < GM; ++q) {
    gr[q] = Rre[G0 * GM + q];
    gi[q] = Rim[G0 * GM + q];
  }
}

#define FSE_RG(G0)                                                 \
  case G0:                                                        \
    if constexpr (G0 < NG) group_copy<GM, G0, NP>(Rre, Rim, gr, gi); \
    break;

// The first (pair, member) of group g whose |R|^2 equals target, and its
// value.  g must be warp-uniform (a uniform jump, like pick_bin); |R|^2 is
// recomputed with the scan's exact instruction sequence.
template <int NP, int GM>
FSE_DEV void resolve_group(const float2 (&Rre)[NP], const float2 (&Rim)[NP], int g, float target,
                           int &pp, int &mm, float &re, float &im) {
  constexpr int NG = NP / GM;
  static_assert(NG * GM == NP && NG <= 16, "groups tile the pairs");
  float2 gr[GM], gi[GM];
  if constexpr (NG <= 4) {
    switch (g) { FSE_RG(0) FSE_RG(1) FSE_RG(2) FSE_RG(3) default: __builtin_unreachable(); }
  } else if constexpr (NG <= 8) {
    switch (g) {
      FSE_RG(0) FSE_RG(1) FSE_RG(2) FSE_RG(3) FSE_RG(4) FSE_RG(5) FSE_RG(6) FSE_RG(7)
      default: __builtin_unreachable();
    }
  } else {
    switch (g) {
      FSE_RG(0) FSE_RG(1) FSE_RG(2) FSE_RG(3) FSE_RG(4) FSE_RG(5) FSE_RG(6) FSE_RG(7)
      FSE_RG(8) FSE_RG(9) FSE_RG(10) FSE_RG(11) FSE_RG(12) FSE_RG(13) FSE_RG(14) FSE_RG(15)
      default: __builtin_unreachable();
    }
  }
#ifndef FSE_RESOLVE_SEL
// 1: GM = 2 resolution as a two-level select tree instead of four overwrite passes (14 ops
// for 26 on the per-iteration serial tail; config 5: 8.37 -> 8.59 M blocks/s, bitwise identical)
#define FSE_RESOLVE_SEL 1
#endif
  if constexpr (FSE_RESOLVE_SEL && GM == 2) {
    // the caller's lane holds target in this group, so the fourth value needs no test
    const float2 m0 = __ffma2_rn(gi[0], gi[0], __fmul2_rn(gr[0], gr[0]));
    const float2 m1 = __ffma2_rn(gi[1], gi[1], __fmul2_rn(gr[1], gr[1]));
    const bool e0 = m0.x == target, e1 = m0.y == target, e2 = m1.x == target;
    const bool lo = e0 || e1;
    const float ra = e0 ? gr[0].x : gr[0].y, rb = e2 ? gr[1].x : gr[1].y;
    const float ia = e0 ? gi[0].x : gi[0].y, ib = e2 ? gi[1].x : gi[1].y;
    re = lo ? ra : rb;
    im = lo ? ia : ib;
    const int k = lo ? (e0 ? 0 : 1) : (e2 ? 2 : 3);
    pp = g * GM + (k >> 1);
    mm = k & 1;
    return;
  }
  // scan backwards so the first match in (pair, member) order is kept
  pp = g * GM;
  mm = 0;
  re = gr[0].x;
  im = gi[0].x;
#pragma unroll
  for (int q = GM - 1; q >= 0; --q) {
    const float2 mg = __ffma2_rn(gi[q], gi[q], __fmul2_rn(gr[q], gr[q]));
    if (mg.y == target) { pp = g * GM + q; mm = 1; re = gr[q].y; im = gi[q].y; }
    if (mg.x == target) { pp = g * GM + q; mm = 0; re = gr[q].x; im = gi[q].x; }
  }
}
#undef FSE_RG

// ------------------------------------------------ radix-8 register FFT
FSE_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
FSE_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
FSE_DEV float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
FSE_DEV float2 cmi(float2 a) { return make_float2(a.y, -a.x); }  // -i * a

// In-register forward DFT-8 (natural order in and out).
FSE_DEV void dft8(float2 (&x)[8]) {
  const float s = 0.70710678118654752f;
  float2 a0 = cadd(x[0], x[4]), a4 = csub(x[0], x[4]);
  float2 a1 = cadd(x[1], x[5]), a5 = csub(x[1], x[5]);
  float2 a2 = cadd(x[2], x[6]), a6 = csub(x[2], x[6]);
  float2 a3 = cadd(x[3], x[7]), a7 = csub(x[3], x[7]);
  a5 = make_float2(s * (a5.x + a5.y), s * (a5.y - a5.x));    // * e^{-i pi/4}
  a6 = cmi(a6);                                               // * -i
  a7 = make_float2(s * (a7.y - a7.x), -s * (a7.x + a7.y));    // * e^{-3i pi/4}
  float2 b0 = cadd(a0, a2), b2 = csub(a0, a2), b1 = cadd(a1, a3), b3 = cmi(csub(a1, a3));
  float2 b4 = cadd(a4, a6), b6 = csub(a4, a6), b5 = cadd(a5, a7), b7 = cmi(csub(a5, a7));
  x[0] = cadd(b0, b1); x[4] = csub(b0, b1); x[2] = cadd(b2, b3); x[6] = csub(b2, b3);
  x[1] = cadd(b4, b5); x[5] = csub(b4, b5); x[3] = cadd(b6, b7); x[7] = csub(b6, b7);
}

FSE_DEV void dft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
  float2 a0 = cadd(x0, x2), a2 = csub(x0, x2), a1 = cadd(x1, x3), a3 = cmi(csub(x1, x3));
  x0 = cadd(a0, a1); x1 = cadd(a2, a3); x2 = csub(a0, a1); x3 = csub(a2, a3);
}

// In-register forward DFT-16 (4 x 4), natural order in and out.
FSE_DEV void dft16(float2 (&x)[16], const float2 *tw, int twstep) {
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4(x[b], x[b + 4], x[b + 8], x[b + 12]);
#pragma unroll
  for (int b = 1; b < 4; ++b)
#pragma unroll
    for (int c = 1; c < 4; ++c) x[b + 4 * c] = cmul(x[b + 4 * c], tw[b * c * twstep]);
  float2 y[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float2 a0 = x[4 * c], a1 = x[4 * c + 1], a2 = x[4 * c + 2], a3 = x[4 * c + 3];
    dft4(a0, a1, a2, a3);
    y[c] = a0; y[c + 4] = a1; y[c + 8] = a2; y[c + 12] = a3;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = y[k];
}

// Length-F forward FFT by a group of QT lanes of one warp.  Lane t holds
// x[t + QT k] (k < VPT) in v.  F = 32, 64: radix 8 x (F/8) (QT = F/8 lanes,
// 8 values each); F = 128: radix 16 x 8 (8 lanes, 16 values each).  One
// exchange through `ex` (element (q1, t) at ex[(q1 * QT + t) * es]); on
// return v[i] holds X[group_out<F>(t, i)].
template <int F, int NF>
FSE_DEV void group_fft(float2 (&v)[NF][FG<F>::VPT], float2 *const (&ex)[NF], int es, const float2 *tw,
                       int t) {
  constexpr int QT = FG<F>::QT;
  // NF independent transforms per lane group share the two warp syncs (and
  // their latencies overlap).  Exchange slot of element (q1, t): XOR-swizzled
  // within each row of QT so both the writes (fixed q1, lanes t) and the
  // transposed reads (fixed k, lanes t reading row q1 = t) hit distinct banks.
  auto X = [&](int f, int q1, int tt) -> float2 & {
    return ex[f][(q1 * QT + (tt ^ (q1 & (QT - 1)))) * es];
  };
  if constexpr (F == 128) {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      dft16(v[f], tw, F / 16);
#pragma unroll
      for (int q1 = 1; q1 < 16; ++q1) v[f][q1] = cmul(v[f][q1], tw[t * q1]);
#pragma unroll
      for (int q1 = 0; q1 < 16; ++q1) X(f, q1, t) = v[f][q1];
    }
    __syncwarp();
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float2 y[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) y[k] = X(f, t + 8 * h, k);
        dft8(y);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[f][8 * h + k] = y[k];
      }
  } else {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      dft8(v[f]);
#pragma unroll
      for (int q1 = 1; q1 < 8; ++q1) v[f][q1] = cmul(v[f][q1], tw[t * q1]);
#pragma unroll
      for (int q1 = 0; q1 < 8; ++q1) X(f, q1, t) = v[f][q1];
    }
    __syncwarp();
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      if (QT == 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[f][k] = X(f, t, k);
        dft8(v[f]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[f][k] = X(f, t, k);
          v[f][4 + k] = X(f, t + 4, k);
        }
        dft4(v[f][0], v[f][1], v[f][2], v[f][3]);
        dft4(v[f][4], v[f][5], v[f][6], v[f][7]);
      }
    }
  }
  __syncwarp();
}

// output index of v[i] after group_fft for lane t
template <int F> FSE_DEV int group_out(int t, int i) {
  if (F == 128) return (i < 8) ? t + 16 * i : (t + 8) + 16 * (i - 8);
  if (F == 64) return t + 8 * i;
  return (i < 4) ? t + 8 * i : (t + 4) + 8 * (i - 4);
}

// Cooperative copy of one class's table (global -> shared), 16 B per op.
FSE_DEV void copy_table(void *dst, const void *src, size_t bytes, int tid, int nthr) {
  const uint4 *s = (const uint4 *)src;
  uint4 *d = (uint4 *)dst;
  for (size_t i = tid; i < bytes / 16; i += nthr) d[i] = __ldg(s + i);
}

// TMA = true: u8 frames, each block's support window staged in shared memory
// by a tensor-map load prefetched during the slot's previous block; TMA =
// false: direct bounds-checked loads.  Separate instantiations keep each
// variant's registers for its own path.
template <int F, bool TMA, int ALG>
__global__ void __launch_bounds__(KS<F, ALG>::CTA, 1)
    fast_kernel(FastArgs a, int iter_cap, const __grid_constant__ CUtensorMap tmap) {
  typedef FG<F> G;
  static_assert(ALG == 0 || F == 32 || F == 64 || F == 128, "fused window sizes");
  constexpr int NS = KS<F, ALG>::S;  // blocks (slots) per CTA
  extern __shared__ __align__(16) char smem[];
  char *region = smem;
  float2 *syn_tw = (float2 *)(smem + KS<F, ALG>::REGION);  // exp(+2 pi i j / F), j < F
  float2 *fft_tw = syn_tw + F;                     // exp(-2 pi i j / F), j < F
  float2 *rot_tw = fft_tw + F;                     // exp(+i pi j (F - 1) / F), j < 2F
  // slot regions 512-byte aligned: TMA destinations (128 B) and the
  // exchange double buffer (aligned to its size, <= 512 B)
  char *slots_base = (char *)(((uintptr_t)(rot_tw + 2 * F) + 511) & ~(uintptr_t)511);
  constexpr size_t STG = TMA ? G::STAGE : 0;  // the direct-load variant keeps no staging area
  constexpr size_t slot_bytes = slot_stride<F>(TMA);

  const int tid = threadIdx.x;
  const int slot = tid / G::NT, st = tid - slot * G::NT;
  const int w = st >> 5, lane = st & 31;
  char *sb = slots_base + slot * slot_bytes;
  SlotPtrs<F> sp;
  sp.scratch = (float2 *)(sb + STG);
  sp.xch = (uint4 *)(sb + STG + G::SCRATCH);
  sp.red = (float *)(sp.xch + 2 * G::NW);
  uint64_t *const mbar = (uint64_t *)((char *)sp.red + 64);  // TMA completion barrier
  int *const tphase = (int *)(mbar + 1);                      // its expected phase
  sp.trace = (float4 *)sp.scratch;  // the FFT scratch holds the trace after setup
  if (a.trace_scratch)  // more iterations than the shared trace holds: per-slot global scratch
    sp.trace = a.trace_scratch + ((size_t)blockIdx.x * NS + slot) * 2 * a.iterations;

  for (int j = tid; j < F; j += blockDim.x) {
    double s, c;
    sincospi(2.0 * j / F, &s, &c);
    syn_tw[j] = make_float2((float)c, (float)s);
    fft_tw[j] = make_float2((float)c, (float)-s);
  }
  for (int j = tid; j < 2 * F; j += blockDim.x) {
    double s, c;
    sincospi((double)((j * (F - 1)) % (2 * F)) / F, &s, &c);
    rot_tw[j] = make_float2((float)c, (float)s);
  }
  if constexpr (TMA) {
    if (st == 0) {
      mbar_init(mbar);
      *tphase = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // issue the TMA load of the support window of this slot's block in round rnd
  auto prefetch = [&](int rnd) {
    if constexpr (!TMA) return;
    if (st != 0 || rnd >= a.n_rounds) return;
    const int nb = __ldg(a.rounds + (size_t)rnd * NS + slot);
    if (nb < 0) return;
    const int o = (F - a.B) / 2 - a.box_off;  // image offset of the box from the block
    tma_window(sb, &tmap, mbar, (unsigned)(a.box_w * a.box_h), __ldg(a.blocks + 3 * nb + 2) - o,
               __ldg(a.blocks + 3 * nb + 1) - o, __ldg(a.blocks + 3 * nb));
  };
  prefetch(blockIdx.x);

  const int off = (F - a.B) / 2;
  int loaded = -1;
#if FSE_DIAG & 32
  unsigned tmk[7];
#endif
  for (int round = blockIdx.x; round < a.n_rounds; round += gridDim.x) {
    const int cls = __ldg(a.round_class + round);
    if (cls != loaded) {
      __syncthreads();
      // (rFSE at F = 128: the W' / Q table only; the criterion table goes to
      // the scratch per block)
      copy_table(region, (const char *)a.table + (size_t)cls * a.table_bytes,
                 ALG && F == 128 ? G::TABLE_BYTES : a.table_bytes, tid, blockDim.x);
      __syncthreads();
      loaded = cls;
    }
    // centred frame: the class's weights are mirror-symmetric and its table
    // is the real Q (see the iteration section); uniform over the CTA
    const bool sym = a.class_sym && __ldg(a.class_sym + cls);
    const int b = __ldg(a.rounds + (size_t)round * NS + slot);
    if (b < 0) {  // idle this round: keep the slot's prefetch chain going
      if constexpr (TMA) prefetch(round + gridDim.x);
      continue;
    }
    if constexpr (TMA) mbar_wait(mbar, *tphase);
    FSE_TMARK(0);

    // ---------------------------------------------------------- load s*w
    FSE_CHECK(b < a.n_blocks && cls < a.n_classes);
    const int fidx = __ldg(a.blocks + 3 * b), top = __ldg(a.blocks + 3 * b + 1),
              left = __ldg(a.blocks + 3 * b + 2);
    const int wt = top - off, wl = left - off;
    const float *wtab = a.wtab + (size_t)cls * F * F;
    const size_t fbase = (size_t)fidx * (size_t)a.frame_stride;
    float e0p = 0.f;
    float2 Rre[G::NP], Rim[G::NP];
    {
      // Real-input 2-D FFT, half spectrum:
      //   rows   -- row pairs packed as one complex row, z_j = x_2j + i x_2j+1,
      //             one length-F FFT per pair (only pairs meeting the support);
      //   columns -- columns 1..F/2-1 of the untangled row spectra, plus
      //             columns 0 and F/2 packed as one complex column;
      //   the other half follows from X[k][l] = conj(X[-k][-l]), so R_w is
      //   exactly Hermitian by construction.
      // Each length-F FFT runs in the registers of QT lanes (radix 8 x F/8,
      // or 16 x 8 for F = 128) with one shared-memory exchange (group_fft).
      constexpr int Q = G::QT, VPT = G::VPT, NG = G::NT / Q, H = F / 2, ZS = F + 1, XS = H + 1,
                    CP = H / NG;
      const int g = st / Q, t = st - (st / Q) * Q;
      float2 *S = sp.scratch;
      const int4 rect = __ldg((const int4 *)a.support_rect + cls);  // (r0, c0, r1, c1)
      const int j0 = rect.x >> 1, j1 = (rect.z + 1) >> 1;
      const bool inside8 = a.dtype == 0 && wt >= 0 && wl >= 0 && wt + F <= a.H && wl + F <= a.W;
      // Group g transforms row pairs j = g + NG f (f < NFT): every row pair in
      // one pass; pairs outside the support rows [j0, j1) transform zeros.
      constexpr int NFT = G::NFT;
      static_assert(NFT * NG == H, "row pairs per pass");
      float2 v[NFT][VPT];
      float2 *rows[NFT];
#pragma unroll
      for (int fi = 0; fi < NFT; ++fi) {
        const int j = g + NG * fi;
        rows[fi] = S + j * ZS;
        const bool act = j >= j0 && j < j1;
        const int y0 = wt + 2 * j;
        if constexpr (TMA) {
          // support window staged by TMA (zeros outside the image)
          const uint8_t *stage = (const uint8_t *)sb;
          const int br = 2 * j - a.box_off;
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            const int n = t + Q * k, bc = n - a.box_off;
            float xe = 0.f, xo = 0.f;
            if (act && (unsigned)bc < (unsigned)a.box_w) {
              if ((unsigned)br < (unsigned)a.box_h) {
                const float s = (float)stage[br * a.box_w + bc];
                xe = s * __ldg(wtab + (2 * j) * F + n);
                e0p += xe * s;
              }
              if ((unsigned)(br + 1) < (unsigned)a.box_h) {
                const float s = (float)stage[(br + 1) * a.box_w + bc];
                xo = s * __ldg(wtab + (2 * j + 1) * F + n);
                e0p += xo * s;
              }
            }
            v[fi][k] = make_float2(xe, xo);
          }
        } else if (inside8) {
          // u8 frame, window inside the image: no bounds checks, one base
          // pointer per row and immediate offsets (w = 0 outside the
          // support, and a u8 sample is finite, so s * w needs no mask)
          const uint8_t *p0 = (const uint8_t *)a.frames + fbase + (size_t)y0 * a.pitch + wl + t;
          const uint8_t *p1 = p0 + a.pitch;
          const float *w0 = wtab + (2 * j) * F + t, *w1 = w0 + F;
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            float xe = 0.f, xo = 0.f;
            if (act) {
              const float se = (float)__ldg(p0 + Q * k), so = (float)__ldg(p1 + Q * k);
              xe = se * __ldg(w0 + Q * k);
              xo = so * __ldg(w1 + Q * k);
              e0p += xe * se;
              e0p += xo * so;
            }
            v[fi][k] = make_float2(xe, xo);
          }
        } else {
          // weights and pixels are loaded independently (in-bounds pixels
          // unconditionally) so a cold window costs one memory round trip,
          // not two dependent ones; samples off the support (w = 0, e.g. a
          // NaN-filled lost block) are zeroed by a select, not multiplied
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            const int n = t + Q * k, x = wl + n;
            float xe = 0.f, xo = 0.f;
            if (act && x >= 0 && x < a.W) {
              const float we = __ldg(wtab + (2 * j) * F + n), wo = __ldg(wtab + (2 * j + 1) * F + n);
              const bool ie = y0 >= 0 && y0 < a.H, io = y0 + 1 >= 0 && y0 + 1 < a.H;
              const float se = ie ? load_px(a.frames, a.dtype, fbase + (size_t)y0 * a.pitch + x) : 0.f;
              const float so = io ? load_px(a.frames, a.dtype, fbase + (size_t)(y0 + 1) * a.pitch + x) : 0.f;
              if (we != 0.f) {
                xe = se * we;
                e0p += xe * se;
              }
              if (wo != 0.f) {
                xo = so * wo;
                e0p += xo * so;
              }
            }
            v[fi][k] = make_float2(xe, xo);
          }
        }
      }
#if FSE_DIAG & 16
      if (false)
#endif
      {
        group_fft<F, NFT>(v, rows, 1, fft_tw, t);
#pragma unroll
        for (int fi = 0; fi < NFT; ++fi)
#pragma unroll
          for (int i = 0; i < VPT; ++i) {
            FSE_CHECK((g + NG * fi) * ZS + group_out<F>(t, i) < (int)(G::SCRATCH / sizeof(float2)));
            rows[fi][group_out<F>(t, i)] = v[fi][i];
          }
      }
      slot_sync<F>(slot);
      FSE_TMARK(1);
      if constexpr (TMA) {
        if (st == 0) *tphase ^= 1;  // every thread of the slot has waited
        prefetch(round + gridDim.x);  // the staged window has been consumed
      }
      float2 cin[CP][VPT];
#pragma unroll
      for (int pass = 0; pass < CP; ++pass) {
        const int c = g + pass * NG;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          const int m = t + Q * k, j = m >> 1, odd = m & 1;
          float2 y = make_float2(0.f, 0.f);
          if (j >= j0 && j < j1) {
            if (c == 0) {
              const float2 z0 = S[j * ZS], zh = S[j * ZS + H];
              y = odd ? make_float2(z0.y, zh.y) : make_float2(z0.x, zh.x);
            } else {
              const float2 zl = S[j * ZS + c], zm = S[j * ZS + F - c];
              y = odd ? make_float2((zl.y + zm.y) * 0.5f, (zm.x - zl.x) * 0.5f)
                      : make_float2((zl.x + zm.x) * 0.5f, (zl.y - zm.y) * 0.5f);
            }
          }
          cin[pass][k] = y;
        }
      }
      slot_sync<F>(slot);  // the row spectra are consumed; reuse as X
      FSE_TMARK(2);
#if FSE_DIAG & 16
      if (false)
#endif
      {
        float2 *cols[CP];
#pragma unroll
        for (int pass = 0; pass < CP; ++pass) cols[pass] = S + g + pass * NG;
        group_fft<F, CP>(cin, cols, XS, fft_tw, t);
#pragma unroll
        for (int pass = 0; pass < CP; ++pass) {
          const int c = g + pass * NG;
#pragma unroll
          for (int i = 0; i < VPT; ++i) {
            FSE_CHECK(group_out<F>(t, i) * XS + c < (int)(G::SCRATCH / sizeof(float2)));
            S[group_out<F>(t, i) * XS + c] = cin[pass][i];
          }
        }
      }
      slot_sync<F>(slot);
      FSE_TMARK(3);
      // untangle the packed real columns 0 and F/2 in place (column F/2 of
      // the scratch is free): thread r <= F/2 owns rows r and -r
      if (st <= H) {
        const int r = st, rm = (F - r) & (F - 1);
        const float2 yk = S[r * XS], ym = S[rm * XS];
        const float2 x0 = make_float2((yk.x + ym.x) * 0.5f, (yk.y - ym.y) * 0.5f);
        const float2 xh = make_float2((yk.y + ym.y) * 0.5f, (ym.x - yk.x) * 0.5f);
        S[r * XS] = x0;
        S[r * XS + H] = xh;
        if (rm != r) {
          S[rm * XS] = make_float2(x0.x, -x0.y);
          S[rm * XS + H] = make_float2(xh.x, -xh.y);
        }
      }
      slot_sync<F>(slot);
      // X[r][c] = S[r][c] for c <= F/2, else conj(S[-r][F - c])
      auto bin = [&](int r, int c) -> float2 {
        const bool lo = c <= H;
        const float2 z = S[lo ? r * XS + c : ((F - r) & (F - 1)) * XS + (F - c)];
        return make_float2(z.x, lo ? z.y : -z.y);
      };
#pragma unroll
      for (int p = 0; p < G::NP; ++p) {
        const int ia = bin_index<F>(w, lane, p, 0), ib = bin_index<F>(w, lane, p, 1);
        float2 xa = bin(ia >> G::LOG, ia & (F - 1)), xb = bin(ib >> G::LOG, ib & (F - 1));
        if (sym) {  // R~[k][l] = R_w[k][l] e^{+i pi (k + l)(F - 1) / F}
          const float2 ra = rot_tw[(ia >> G::LOG) + (ia & (F - 1))], rb = rot_tw[(ib >> G::LOG) + (ib & (F - 1))];
          xa = make_float2(xa.x * ra.x - xa.y * ra.y, xa.x * ra.y + xa.y * ra.x);
          xb = make_float2(xb.x * rb.x - xb.y * rb.y, xb.x * rb.y + xb.y * rb.x);
        }
        // an arithmetic op gives each SoA pair a fresh, aligned register
        // pair (plain copies let the allocator split the pairs and pay MOVs
        // around every FFMA2 of the hot loop)
        const bool tw = FSE_RTWIST && ALG == 1 && F == 64 && sym;  // twisted pairs (rFSE loop)
        Rre[p] = __fadd2_rn(make_float2(xa.x, tw ? xb.y : xb.x), make_float2(0.f, 0.f));
        Rim[p] = __fadd2_rn(make_float2(xa.y, tw ? xb.x : xb.y), make_float2(0.f, 0.f));
      }
    }
    // e0 = sum w s^2 (slot reduction; trace energies only)
    for (int o = 16; o; o >>= 1) e0p += __shfl_xor_sync(0xffffffffu, e0p, o);
    if (lane == 0) sp.red[w] = e0p;
    slot_sync<F>(slot);  // scratch is free from here on (trace area)
    FSE_TMARK(4);

    // ------------------------------------------------------- iterations
    // Loop state is kept minimal (the spectrum takes 64 of the 96 registers):
    // the selection as one row-major index, the exchange buffer as a 32-bit
    // shared address; slot thread 0 records (index, R_w[u,v]) only -- the
    // coefficients, energies and trace outputs are derived after the loop.
    const float ginv = a.gamma * __ldg(a.inv_w00 + cls);
    int nit = a.iterations;  // iterations run (rFSE: fewer when the tally target is met)
    float cre = 0.f, cim = 0.f;
    unsigned gidx = 0;
    unsigned xc = (unsigned)__cvta_generic_to_shared(sp.xch);
    const int rowbase = w * G::RPW;
    // Loop-invariant address terms, passed through an identity shuffle so
    // ptxas keeps them in registers instead of re-deriving them from the
    // thread/CTA ids (S2R/S2UR) at the latency-critical start of every
    // iteration: kpos = (first row of the warp) * F | lane, and the table's
    // 32-bit shared-window address.
    const unsigned kpos = __shfl_sync(0xffffffffu, (unsigned)(rowbase * F) | (unsigned)lane, lane);
    const unsigned tbase =
        __shfl_sync(0xffffffffu, (unsigned)__cvta_generic_to_shared(region), lane);

    if constexpr (ALG == 0) {
    auto iterate = [&](auto symc) {
    constexpr bool SY = decltype(symc)::value;
#pragma unroll 1
    for (int it = 0; it < a.iterations; ++it) {
#if FSE_DIAG & 32
      const unsigned clk0 = (unsigned)clock();
#endif
      const int rowoff = (rowbase - (int)(gidx >> G::LOG)) & (F - 1);
      (void)rowoff;
#ifndef FSE_CHAINS64
#define FSE_CHAINS64 1
#endif
      // CH independent first-max trackers over consecutive pair ranges
      // (shorter dependent compare/select chains), merged in order below;
      // measured best: 1 (2 helped the 32-bins-per-thread F = 64 variant)
#ifndef FSE_XTREE
// F=128 warp-candidate merge: 1 = every lane reads all 8 candidates and
// merges in registers (+0.6 % with the complex-table loop), 0 = one REDUX
// pair over a lane-per-warp load (+4.8 % with the centred-frame loop)
#define FSE_XTREE 0
#endif
#ifndef FSE_CHAINS128
#define FSE_CHAINS128 1
#endif
#ifndef FSE_CHAINS32
#define FSE_CHAINS32 1
#endif
      constexpr int CH = F == 64 ? FSE_CHAINS64 : F == 128 ? FSE_CHAINS128 : FSE_CHAINS32;
      float bst[CH], bxs[CH];
      int bps[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) { bst[c] = -1.f; bxs[c] = 0.f; bps[c] = c * (G::NP / CH); }
#ifndef FSE_PACKKEY
// 1: the first-max tracker keeps one packed key per thread -- |R|^2 bits with
// the low log2(F) bits replaced by the bin's rank (4 ops per pair instead of
// 5; F=64 loop 569 -> 521 instructions, +3.3 % on config 5).  Selection then
// resolves |R|^2 to 2^-17 relative (ties by row-major index), below fp32's
// accumulated noise but above exact first-max: config 3 gained one certified
// near-tie (2 of 402 blocks, PSNR delta 2e-4 dB).  Off: exact fp32 first max.
#define FSE_PACKKEY 0
#endif
      constexpr bool PK = FSE_PACKKEY && !G::PLANAR && CH == 1;
      constexpr int GM = PK ? 0 : F == 32 ? FSE_GROUPMAX32 : F == 64 ? FSE_GROUPMAX64 : FSE_GROUPMAX128;
      static_assert(GM == 0 || (CH == 1 && G::NP % GM == 0), "group tracker: one chain, whole groups");
      float gv[GM > 0 ? 2 * GM : 2];  // the current group's |R|^2 values
      int bg = 0;                     // GM: the thread's first group holding its maximum
      (void)gv;
      (void)bg;
      unsigned bkey = 0u;  // PK: truncated |R|^2 bits | (NP-1-p) << 1 | member a
      // (the mask laundered through a shuffle stays a register operand, so
      // clear-and-insert is one LOP3 with the rank as its immediate)
      // (from the runtime window size, so that it is not an immediate:
      // ~(F - 1) clears the rank bits, 2 NP <= F)
      const unsigned kmask = PK ? 0u - (unsigned)a.F : 0u;
      if constexpr (!G::PLANAR && SY) {
        // Centred frame (mirror-symmetric weights: every interior block).
        // With w[m][n] = w[F-1-m][n] = w[m][F-1-n], W[k][l] = A(k) A(l) Q(k, l)
        // with A(k) = e^{-i pi k (F-1)/F} and Q real, anti-periodic
        // (Q(i + F, j) = -Q(i, j)).  In the frame R~[k][l] = R_w[k][l] /
        // (A(k) A(l)) the update R_w[k] -= c W[k - (u,v)] becomes
        // R~[k] -= c~ Q(k - (u,v)), c~ = gamma R~[u,v] / W00, and |R~| = |R_w|:
        // one real table value per bin (one LDS.64 and two FFMA2 per bin pair
        // instead of an LDS.128 and four FFMA2).  Entry (i, j) of the table
        // holds the pair (Q(i, j), Q(i + di, j + dj)), rows / columns from
        // -(F-1): no wrap arithmetic and no sign flips in the walk.
#ifndef FSE_PREFETCH
#define FSE_PREFETCH 2
#endif
        constexpr int PD = F == 64 ? FSE_PREFETCH64 : FSE_PREFETCH;
        constexpr unsigned RSB = (F == 32 ? 2u : 1u) * (unsigned)G::SYM_C * 8u;  // bytes per pair step
        // entry of (row rowbase - u, column lane - v): with kpos = rowbase F + lane
        // and gidx = u F + v, (rowbase - u + F - 1) SYM_C + lane - v + F - 1 =
        // kpos - gidx + (SYM_C - F)(rowbase - u) + (F - 1)(SYM_C + 1)
        const unsigned tq =
            tbase + ((kpos - gidx + (unsigned)(G::SYM_C - F) * ((kpos >> G::LOG) - (gidx >> G::LOG)) +
                      (unsigned)((F - 1) * (G::SYM_C + 1)))
                     << 3);
        float2 qbuf[PD > 0 ? PD : 1];
#pragma unroll
        for (int d = 0; d < PD; ++d) qbuf[d] = lds64f(tq + (unsigned)d * RSB);
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          FSE_CHECK((tq - tbase) / 8 + (unsigned)p * (RSB / 8) < (unsigned)(G::SYM_R * G::SYM_C));
          float2 qv;
          if constexpr (PD > 0) {
            qv = qbuf[p % PD];
            if (p + PD < G::NP) qbuf[p % PD] = lds64f(tq + (unsigned)(p + PD) * RSB);
          } else {
            qv = lds64f(tq + (unsigned)p * RSB);
          }
          ffma2_acc(Rre[p], qv, -cre);
          ffma2_acc(Rim[p], qv, -cim);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const int ch = p / (G::NP / CH);
          (void)ch;
#if FSE_DIAG & 2
          bst[ch] = fmax3(bst[ch], mg.x, mg.y);
#else
          if constexpr (PK) {
            const unsigned ka = (__float_as_uint(mg.x) & kmask) | (unsigned)(((G::NP - 1 - p) << 1) | 1);
            const unsigned kb = (__float_as_uint(mg.y) & kmask) | (unsigned)((G::NP - 1 - p) << 1);
            bkey = max(bkey, max(ka, kb));
          } else if constexpr (GM > 0) {
            gv[2 * (p % GM)] = mg.x;
            gv[2 * (p % GM) + 1] = mg.y;
            if (p % GM == GM - 1) group_step<GM>(gv, bst[0], bg, p / GM);
          } else {
            first_max(bst[ch], bps[ch], bxs[ch], mg, p);
          }
#endif
        }
      } else if constexpr (!G::PLANAR) {
        // table index (rowoff, coloff) = ((rowbase - u) mod F, (lane - v) mod F)
        constexpr unsigned RM = (unsigned)(F - 1) << G::LOG;
        const unsigned tp =
            tbase + ((((kpos - (gidx & RM)) & RM) | ((kpos - gidx) & (unsigned)(F - 1))) << 4);
#ifndef FSE_PREFETCH
#define FSE_PREFETCH 2
#endif
        // W' loads issued PD pairs ahead of their use (0: left to ptxas).  Without
        // it ptxas may keep only two load buffers in flight when registers are
        // tight, exposing the shared-memory latency (measured -10%).
        constexpr int PD = F == 64 ? FSE_PREFETCH64 : FSE_PREFETCH;
        float4 wbuf[PD > 0 ? PD : 1];
#pragma unroll
        for (int d = 0; d < PD; ++d) wbuf[d] = lds128f(tp + (unsigned)((F == 32 ? 2 * d : d) * F * 16));
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          FSE_CHECK(rowoff + (F == 32 ? 2 * p : p) < G::TROWS);
          float4 wv;
          if constexpr (PD > 0) {
            wv = wbuf[p % PD];
            if (p + PD < G::NP)
              wbuf[p % PD] = lds128f(tp + (unsigned)((F == 32 ? 2 * (p + PD) : p + PD) * F * 16));
          } else {
            wv = lds128f(tp + (unsigned)((F == 32 ? 2 * p : p) * F * 16));
          }
          const float2 wr = make_float2(wv.x, wv.y), wi = make_float2(wv.z, wv.w);
          ffma2_acc(Rre[p], wr, -cre);
          ffma2_acc(Rre[p], wi, cim);
          ffma2_acc(Rim[p], wi, -cre);
          ffma2_acc(Rim[p], wr, -cim);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const int ch = p / (G::NP / CH);
          (void)ch;
#if FSE_DIAG & 2
          bst[ch] = fmax3(bst[ch], mg.x, mg.y);
#else
          if constexpr (PK) {
            static_assert(!PK || 2 * G::NP <= F, "rank bits fit under the mask");
            const unsigned ka = (__float_as_uint(mg.x) & kmask) | (unsigned)(((G::NP - 1 - p) << 1) | 1);
            const unsigned kb = (__float_as_uint(mg.y) & kmask) | (unsigned)((G::NP - 1 - p) << 1);
            bkey = max(bkey, max(ka, kb));
          } else if constexpr (GM > 0) {
            gv[2 * (p % GM)] = mg.x;
            gv[2 * (p % GM) + 1] = mg.y;
            if (p % GM == GM - 1) group_step<GM>(gv, bst[0], bg, p / GM);
          } else {
            first_max(bst[ch], bps[ch], bxs[ch], mg, p);
          }
#endif
        }
      } else if constexpr (SY) {
        // centred frame at F = 128: scalar table T[i + F - 1][c] = Q(i, c),
        // c = (l - v) mod F; the column sign sgn(l - v) of each of the
        // thread's four columns goes into its coefficient pair
        const float *Tq = (const float *)region;
        const int v = (int)(gidx & (F - 1));
        int co[4];
        float sg[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          co[h] = (lane + 32 * h - v) & (F - 1);
          sg[h] = lane + 32 * h < v ? -1.f : 1.f;
        }
        const float2 cr2[2] = {make_float2(-cre * sg[0], -cre * sg[1]), make_float2(-cre * sg[2], -cre * sg[3])};
        const float2 ci2[2] = {make_float2(-cim * sg[0], -cim * sg[1]), make_float2(-cim * sg[2], -cim * sg[3])};
        const int rq = rowbase - (int)(gidx >> G::LOG) + F - 1;
#ifndef FSE_PREFETCH128
#define FSE_PREFETCH128 0  // explicit table-load prefetch depth (0: left to ptxas)
#endif
        constexpr int PQ = FSE_PREFETCH128;
        auto ldq = [&](int pp) {
          const int r = (rq + (pp >> 1)) * F, q = pp & 1;
          FSE_CHECK(rq + (pp >> 1) < G::SYM_R);
          return make_float2(Tq[r + co[2 * q]], Tq[r + co[2 * q + 1]]);
        };
        float2 qb[PQ > 0 ? PQ : 1];
#pragma unroll
        for (int d = 0; d < PQ; ++d) qb[d] = ldq(d);
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          const int q = p & 1;
          float2 qv;
          if constexpr (PQ > 0) {
            constexpr int PQ1 = PQ > 0 ? PQ : 1;
            qv = qb[p % PQ1];
            if (p + PQ < G::NP) qb[p % PQ1] = ldq(p + PQ);
          } else {
            qv = ldq(p);
          }
          ffma2_acc2(Rre[p], qv, cr2[q]);
          ffma2_acc2(Rim[p], qv, ci2[q]);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const int ch = p / (G::NP / CH);
          if constexpr (GM > 0) {
            gv[2 * (p % GM)] = mg.x;
            gv[2 * (p % GM) + 1] = mg.y;
            if (p % GM == GM - 1) group_step<GM>(gv, bst[0], bg, p / GM);
          } else {
            first_max(bst[ch], bps[ch], bxs[ch], mg, p);
          }
        }
      } else {
        const float *Tre = (const float *)region;
        const float *Tim = Tre + G::TROWS * F;
        int co[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) co[h] = (lane + 32 * h - (int)(gidx & (F - 1))) & (F - 1);
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          const int r = (rowoff + (p >> 1)) * F;
          const int q = 2 * (p & 1);
          FSE_CHECK(rowoff + (p >> 1) < G::TROWS);
          const float2 wr = make_float2(Tre[r + co[q]], Tre[r + co[q + 1]]);
          const float2 wi = make_float2(Tim[r + co[q]], Tim[r + co[q + 1]]);
          ffma2_acc(Rre[p], wr, -cre);
          ffma2_acc(Rre[p], wi, cim);
          ffma2_acc(Rim[p], wi, -cre);
          ffma2_acc(Rim[p], wr, -cim);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const int ch = p / (G::NP / CH);
          if constexpr (GM > 0) {
            gv[2 * (p % GM)] = mg.x;
            gv[2 * (p % GM) + 1] = mg.y;
            if (p % GM == GM - 1) group_step<GM>(gv, bst[0], bg, p / GM);
          } else {
            first_max(bst[ch], bps[ch], bxs[ch], mg, p);
          }
        }
      }
      float best = bst[0], bx = bxs[0];
      int bp = bps[0];
#pragma unroll
      for (int c = 1; c < CH; ++c)
        if (bst[c] > best) { best = bst[c]; bp = bps[c]; bx = bxs[c]; }
      // thread's first max (member a wins ties inside the pair)
      const int myidx = PK ? bin_index<F>(w, lane, G::NP - 1 - (int)((bkey >> 1) & (unsigned)(G::NP - 1)),
                                          (bkey & 1u) ? 0 : 1)
                           : bin_index<F>(w, lane, bp, bx >= best ? 0 : 1);
      const unsigned key = PK ? (bkey & kmask) : __float_as_uint(best);  // best >= 0: monotone as unsigned
      const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
      int pw, mw, ow;
      float are, aim;
      if constexpr (GM > 0) {
        // Lanes holding the warp maximum, one at a time (usually one; a
        // conjugate-mirror tie can give two): broadcast the lane's group, all
        // lanes run the (then uniform) resolution on their own registers, and
        // the lane's first bin equal to the maximum and its value are read
        // back; the smallest row-major index wins the warp.
        unsigned cand = __ballot_sync(0xffffffffu, key == wmax);
        const float wbest = __uint_as_float(wmax);
        unsigned widx = 0xffffffffu;
        are = 0.f;
        aim = 0.f;
        do {
          const int L = __ffs(cand) - 1;
          cand &= cand - 1;
          const int gL = __shfl_sync(0xffffffffu, bg, L);
          int pp, mm;
          float re = 0.f, im = 0.f;
          resolve_group<G::NP, GM>(Rre, Rim, gL, wbest, pp, mm, re, im);
#ifndef FSE_IDXSHFL
// 1 (F = 64): the candidate lane's bin index is shuffled whole instead of rebuilt from
// (warp, lane, pair, member): no S2R of the thread index on the tail (8.59 -> 8.78 M)
#define FSE_IDXSHFL 1
#endif
          unsigned idx;
          if constexpr (FSE_IDXSHFL && F == 64 && !G::PLANAR) {
            // F = 64: bin (pair p, member m) of a thread is kpos + 64 p + 32 m = kpos + 32 (2 p + m)
            idx = __shfl_sync(0xffffffffu, kpos + ((unsigned)((pp << 1) | mm) << 5), L);
          } else {
            const int pm = __shfl_sync(0xffffffffu, (pp << 1) | mm, L);
            idx = (unsigned)bin_index<F>(w, L, pm >> 1, pm & 1);
          }
          re = __shfl_sync(0xffffffffu, re, L);
          im = __shfl_sync(0xffffffffu, im, L);
          if (idx < widx) { widx = idx; are = re; aim = im; }
        } while (cand);
        gidx = widx;
        (void)pw; (void)mw; (void)ow;
      } else {
      const unsigned widx = __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
      decode_bin<F>((int)widx, w, pw, mw, ow);
      FSE_CHECK(pw >= 0 && pw < G::NP && ow >= 0 && ow < 32);
      pick_bin<G::NP>(Rre, Rim, pw, mw, are, aim);
      are = __shfl_sync(0xffffffffu, are, ow);
      aim = __shfl_sync(0xffffffffu, aim, ow);
      gidx = widx;
      }
      const unsigned widx = gidx;
#if FSE_DIAG & 1
      if (false) {
#else
      if (G::NW > 1) {
#endif
        if (lane == 0)
          sts128u(xc + 16u * w, make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim)));
        slot_sync<F>(slot);
        if constexpr (G::NW == 2) {
          // two warps: compare with the other warp's candidate in registers
          // (same total order -- larger |R|^2, then smaller index -- in both)
          const uint4 o = lds128u(xc + 16u * (unsigned)(w ^ 1));
          const bool take = o.x > wmax || (o.x == wmax && o.y < widx);
          if (take) {
            gidx = o.y;
            are = __uint_as_float(o.z);
            aim = __uint_as_float(o.w);
          }
        } else if (FSE_XTREE) {
          // every lane reads all NW candidates (broadcast loads) and merges
          // them pairwise in registers; warp w owns rows [w RPW, (w+1) RPW),
          // so on equal |R|^2 the lower warp holds the smaller index and the
          // left operand wins ties
          uint4 cd[G::NW];
#pragma unroll
          for (int j = 0; j < G::NW; ++j) cd[j] = lds128u(xc + 16u * (unsigned)j);
#pragma unroll
          for (int s = 1; s < G::NW; s *= 2)
#pragma unroll
            for (int j = 0; j + s < G::NW; j += 2 * s)
              if (cd[j + s].x > cd[j].x) cd[j] = cd[j + s];
          gidx = cd[0].y;
          are = __uint_as_float(cd[0].z);
          aim = __uint_as_float(cd[0].w);
        } else {
        const uint4 cnd = lane < G::NW ? lds128u(xc + 16u * lane) : make_uint4(0u, 0xffffffffu, 0u, 0u);
        const unsigned gkey = __reduce_max_sync(0xffffffffu, cnd.x);
        gidx = __reduce_min_sync(0xffffffffu, cnd.x == gkey ? cnd.y : 0xffffffffu);
        const int wl = (int)(gidx / (unsigned)(G::RPW * F));
        are = __shfl_sync(0xffffffffu, __uint_as_float(cnd.z), wl);
        aim = __shfl_sync(0xffffffffu, __uint_as_float(cnd.w), wl);
        }
        xc ^= (unsigned)(G::NW * sizeof(uint4));  // the other buffer next time
      }
      cre = ginv * are;
      cim = ginv * aim;
      if (st == 0) {
        FSE_CHECK(a.trace_scratch || it < G::TRACE_CAP);
#if FSE_DIAG & 32
        sp.trace[it] = make_float4(__uint_as_float(gidx), are, aim, __uint_as_float(clk0));
#else
        sp.trace[it] = make_float4(__uint_as_float(gidx), are, aim, 0.f);
#endif
      }
    }
    };  // iterate
    // one loop per table kind (a branch inside the loop made ptxas spill)
    if (sym) iterate(std::true_type{});
    else iterate(std::false_type{});
    } else if constexpr (F == 128) {
      // ------------------------- rFSE at F = 128 in the centred frame
      // (interior classes; rfse.py:69-160).  With R~ = R_w / phi (phi(k) =
      // A(k) A(l), see the cFSE centred loop) and W[2k] = phi(k)^2 Q(2k), the
      // pair criterion 2 (p.re a.re + p.im a.im) of rfse.py:93-103 is
      //   crit = alpha R~.re^2 + beta R~.im^2,
      //   alpha = 2 / (W00 + Q(2k)), beta = 2 / (W00 - Q(2k)),
      // the joint projection is p~ = (R~.re / (W00 + Q2), R~.im / (W00 - Q2))
      // = (alpha, beta) R~ / 2, and the pair update R_w -= c W[k - s] +
      // conj(c) W[k - m] (m the mirror bin) becomes R~ -= c~ Q(k - s) +
      // sg conj(c~) Q(k - m) with c~ = gamma p~ (c = c~ phi(s), restored
      // after the loop) and the sign sg below.  A
      // self-conjugate bin (2k = 0 mod F: s in {0, F/2}^2, phi(s) in {1, i,
      // -1}) has crit = a.re^2 / W00 with a = phi R~: (alpha, beta) = (1/W00,
      // 0) for real phi, (0, 1/W00) for imaginary phi, p~ = (alpha, beta) R~.
      // alpha and beta depend on (2k mod F, 2l mod F): the table holds them
      // at the doubled row 2 r2 (r2 < 64) and the lane's doubled columns
      // (2 lane, 2 lane + 64); a doubled row or column that wraps past F
      // flips the sign of Q(2k), i.e. swaps alpha and beta.
      const unsigned crit_base = smem_u32(sp.scratch) + (unsigned)(G::SCRATCH - rf_t2_bytes<F>());
      {
        const char *src = (const char *)a.table + (size_t)cls * a.table_bytes + G::TABLE_BYTES;
        const int n16 = (int)((sym ? 64 * 32 * 2 * sizeof(float2) : rf_t2_bytes<F>()) / 16);
        for (int i = st; i < n16; i += G::NT)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(crit_base + 16u * (unsigned)i),
                       "l"(src + 16 * (size_t)i)
                       : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
        slot_sync<F>(slot);
      }
      constexpr unsigned HALF = 64u * 32u * (unsigned)sizeof(float2);  // alpha half | beta half
      // this warp's entries: doubled row of row r = rowbase + rr is (r mod 64)
      // (rows >= 64 wrap: alpha <-> beta); pair p = 2 rr + q, q = 1 for the
      // lane's columns + 64 (their doubled columns wrap: swap again)
      if (sym) {
      const unsigned cw = __shfl_sync(0xffffffffu, crit_base + (unsigned)((((rowbase & 63) * 32) + lane) * 8), lane);
      const unsigned pA = w >= 4 ? cw + HALF : cw, pB = w >= 4 ? cw : cw + HALF;
      const float *Tq = (const float *)region;
      unsigned midx = 0;             // bin of the previous pick's second atom
      float c2re = 0.f, c2im = 0.f;  // its coefficient (conj c~, or 0 after a self-conjugate pick)
      int tally = 0;
      nit = 0;
#pragma unroll 1
      for (int it = 0; it < a.iterations && tally < a.stop_tally; ++it) {
        const int v1 = (int)(gidx & (F - 1)), v2 = (int)(midx & (F - 1));
        int co1[4], co2[4];
        float s1[4], s2[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          co1[h] = (lane + 32 * h - v1) & (F - 1);
          co2[h] = (lane + 32 * h - v2) & (F - 1);
          s1[h] = lane + 32 * h < v1 ? -1.f : 1.f;
          s2[h] = lane + 32 * h < v2 ? -1.f : 1.f;
        }
        const float2 a1r[2] = {make_float2(-cre * s1[0], -cre * s1[1]), make_float2(-cre * s1[2], -cre * s1[3])};
        const float2 a1i[2] = {make_float2(-cim * s1[0], -cim * s1[1]), make_float2(-cim * s1[2], -cim * s1[3])};
        const float2 a2r[2] = {make_float2(-c2re * s2[0], -c2re * s2[1]), make_float2(-c2re * s2[2], -c2re * s2[3])};
        const float2 a2i[2] = {make_float2(-c2im * s2[0], -c2im * s2[1]), make_float2(-c2im * s2[2], -c2im * s2[3])};
        const int rq1 = rowbase - (int)(gidx >> G::LOG) + F - 1, rq2 = rowbase - (int)(midx >> G::LOG) + F - 1;
        float bst = -1.f, bxs = 0.f;
        int bps = 0;
        float2 xa = make_float2(0.f, 0.f), xb = xa;
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          const int q = p & 1, rr = p >> 1;
          const int r1 = (rq1 + rr) * F, r2 = (rq2 + rr) * F;
          FSE_CHECK(rq1 + rr < G::SYM_R && rq2 + rr < G::SYM_R);
          const float2 q1 = make_float2(Tq[r1 + co1[2 * q]], Tq[r1 + co1[2 * q + 1]]);
          const float2 q2 = make_float2(Tq[r2 + co2[2 * q]], Tq[r2 + co2[2 * q + 1]]);
          ffma2_acc2(Rre[p], q1, a1r[q]);
          ffma2_acc2(Rim[p], q1, a1i[q]);
          ffma2_acc2(Rre[p], q2, a2r[q]);
          ffma2_acc2(Rim[p], q2, a2i[q]);
          if (q == 0) {
            xa = lds64f(pA + (unsigned)(rr * 256));
            xb = lds64f(pB + (unsigned)(rr * 256));
          }
          const float2 al = q ? xb : xa, be = q ? xa : xb;
          const float2 t1 = fmul2(al, Rre[p]), t2 = fmul2(be, Rim[p]);
          float2 cr = fmul2(t1, Rre[p]);
          cr = ffma2(t2, Rim[p], cr);
          first_max(bst, bps, bxs, cr, p);
        }
        const int myidx = bin_index<F>(w, lane, bps, bxs >= bst ? 0 : 1);
        const unsigned key = __float_as_uint(fmaxf(bst, 0.f));  // crit >= 0: monotone as unsigned
        const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
        const unsigned widx = __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
        int pw, mw, ow;
        decode_bin<F>((int)widx, w, pw, mw, ow);
        float are, aim;
        pick_bin<G::NP>(Rre, Rim, pw, mw, are, aim);
        are = __shfl_sync(0xffffffffu, are, ow);
        aim = __shfl_sync(0xffffffffu, aim, ow);
        // the 8 warp candidates: (crit, index) max, first index on ties
        if (lane == 0) sts128u(xc + 16u * w, make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim)));
        slot_sync<F>(slot);
        const uint4 cnd = lane < G::NW ? lds128u(xc + 16u * lane) : make_uint4(0u, 0xffffffffu, 0u, 0u);
        const unsigned gkey = __reduce_max_sync(0xffffffffu, cnd.x);
        gidx = __reduce_min_sync(0xffffffffu, cnd.x == gkey ? cnd.y : 0xffffffffu);
        const int wl = (int)(gidx / (unsigned)(G::RPW * F));
        are = __shfl_sync(0xffffffffu, __uint_as_float(cnd.z), wl);
        aim = __shfl_sync(0xffffffffu, __uint_as_float(cnd.w), wl);
        xc ^= (unsigned)(G::NW * sizeof(uint4));
        // joint projection of the chosen bin from its (alpha, beta)
        const unsigned u = gidx >> G::LOG, v = gidx & (F - 1);
        const bool self = ((2 * u) & (F - 1)) == 0 && ((2 * v) & (F - 1)) == 0;
        const unsigned ea = crit_base + (((u & 63u) * 32u + (v & 31u)) * 8u) + ((v >> 5) & 1u) * 4u;
        float al = lds32f(ea), be = lds32f(ea + HALF);
        if ((u >= 64u) != (((v >> 6) & 1u) != 0u)) {
          const float t = al;
          al = be;
          be = t;
        }
        const float fac = self ? 1.f : 0.5f;
        float pr = fac * al * are, pi = fac * be * aim;
        // The mirror member m = (-u, -v) mod F: conj(phi(m)) = sg phi(s) with
        // sg = (-1)^([u != 0] + [v != 0]) (A(F - x) = -conj(A(x))), so its
        // centred projection is sg conj(p~) and the second atom, read at the
        // shift m, carries sg conj(c~).  The pair is represented by its
        // smaller row-major member (rfse.py:113-121).
        const float sg = ((u != 0u) != (v != 0u)) ? -1.f : 1.f;
        unsigned mi = (((F - u) & (F - 1)) << G::LOG) | ((F - v) & (F - 1));
        if (!self && mi < gidx) {
          const unsigned t = gidx;
          gidx = mi;
          mi = t;
          pr = sg * pr;
          pi = -sg * pi;
        }
        midx = self ? gidx : mi;
        cre = a.gamma * pr;
        cim = a.gamma * pi;
        c2re = self ? 0.f : sg * cre;
        c2im = self ? 0.f : -sg * cim;
        tally += self ? 1 : 2;
        if (st == 0) {
          FSE_CHECK(a.trace_scratch || (unsigned)it * 16u < (unsigned)(G::SCRATCH - rf_t2_bytes<F>()));
          sp.trace[it] = make_float4(__uint_as_float(gidx | (self ? 0x80000000u : 0u)), cre, cim,
                                     __uint_as_float(gkey));
        }
        nit = it + 1;
      }
      } else {
        // Complex frame (clipped classes): the reference's quadratic form
        // crit = A a.re^2 + C a.im^2 - D a.re a.im (rfse.py:93-103) with
        // (A, C, -D) at the doubled frequency -- in this frame W[2k] needs no
        // sign, and the lane's four columns share the two doubled columns
        // (2 lane, 2 lane + 64) -- from the 48 KB scratch table (float4 (A_c1,
        // A_c2, C_c1, C_c2) half, float2 (-D_c1, -D_c2) half); the update reads
        // the planar W' table at both atoms' shifts (rows row-extended, columns
        // mod F), the mirror atom with conj(c); the winner's projection uses
        // W[2u, 2v] and the reference's divisions (fast path).
        const unsigned cw4 = __shfl_sync(0xffffffffu, crit_base + (unsigned)((((rowbase & 63) * 32) + lane) * 16), lane);
        const unsigned cw2 = cw4 + 64u * 32u * 16u - (unsigned)((((rowbase & 63) * 32) + lane) * 8);
        const float *Tre = (const float *)region;
        const float *Tim = Tre + G::TROWS * F;
        const float w00 = 1.f / __ldg(a.inv_w00 + cls);
        unsigned midx = 0;
        float c2re = 0.f, c2im = 0.f;
        int tally = 0;
        nit = 0;
#pragma unroll 1
        for (int it = 0; it < a.iterations && tally < a.stop_tally; ++it) {
          int co1[4], co2[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            co1[h] = (lane + 32 * h - (int)(gidx & (F - 1))) & (F - 1);
            co2[h] = (lane + 32 * h - (int)(midx & (F - 1))) & (F - 1);
          }
          const int ro1 = (rowbase - (int)(gidx >> G::LOG)) & (F - 1);
          const int ro2 = (rowbase - (int)(midx >> G::LOG)) & (F - 1);
          float bst = -1.f, bxs = 0.f;
          int bps = 0;
          float4 e4 = make_float4(0.f, 0.f, 0.f, 0.f);
          float2 e2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < G::NP; ++p) {
            const int q = 2 * (p & 1), rr = p >> 1;
            const int r1 = (ro1 + rr) * F, r2 = (ro2 + rr) * F;
            FSE_CHECK(ro1 + rr < G::TROWS && ro2 + rr < G::TROWS);
            const float2 wr = make_float2(Tre[r1 + co1[q]], Tre[r1 + co1[q + 1]]);
            const float2 wi = make_float2(Tim[r1 + co1[q]], Tim[r1 + co1[q + 1]]);
            const float2 qr = make_float2(Tre[r2 + co2[q]], Tre[r2 + co2[q + 1]]);
            const float2 qi = make_float2(Tim[r2 + co2[q]], Tim[r2 + co2[q + 1]]);
            ffma2_acc(Rre[p], wr, -cre);
            ffma2_acc(Rre[p], wi, cim);
            ffma2_acc(Rim[p], wi, -cre);
            ffma2_acc(Rim[p], wr, -cim);
            ffma2_acc(Rre[p], qr, -c2re);
            ffma2_acc(Rre[p], qi, c2im);
            ffma2_acc(Rim[p], qi, -c2re);
            ffma2_acc(Rim[p], qr, -c2im);
            if (q == 0) {
              e4 = lds128f(cw4 + (unsigned)(rr * 32 * 16));
              e2 = lds64f(cw2 + (unsigned)(rr * 32 * 8));
            }
            float2 t1 = fmul2(make_float2(e4.x, e4.y), Rre[p]);
            t1 = ffma2(e2, Rim[p], t1);
            const float2 t2 = fmul2(make_float2(e4.z, e4.w), Rim[p]);
            float2 cr = fmul2(t1, Rre[p]);
            cr = ffma2(t2, Rim[p], cr);
            first_max(bst, bps, bxs, cr, p);
          }
          const int myidx = bin_index<F>(w, lane, bps, bxs >= bst ? 0 : 1);
          const unsigned key = __float_as_uint(fmaxf(bst, 0.f));  // monotone as unsigned
          const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
          const unsigned widx = __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
          int pw, mw, ow;
          decode_bin<F>((int)widx, w, pw, mw, ow);
          float are, aim;
          pick_bin<G::NP>(Rre, Rim, pw, mw, are, aim);
          are = __shfl_sync(0xffffffffu, are, ow);
          aim = __shfl_sync(0xffffffffu, aim, ow);
          if (lane == 0) sts128u(xc + 16u * w, make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim)));
          slot_sync<F>(slot);
          const uint4 cnd = lane < G::NW ? lds128u(xc + 16u * lane) : make_uint4(0u, 0xffffffffu, 0u, 0u);
          const unsigned gkey = __reduce_max_sync(0xffffffffu, cnd.x);
          gidx = __reduce_min_sync(0xffffffffu, cnd.x == gkey ? cnd.y : 0xffffffffu);
          const int wl = (int)(gidx / (unsigned)(G::RPW * F));
          are = __shfl_sync(0xffffffffu, __uint_as_float(cnd.z), wl);
          aim = __shfl_sync(0xffffffffu, __uint_as_float(cnd.w), wl);
          xc ^= (unsigned)(G::NW * sizeof(uint4));
          // joint projection of the chosen bin (rfse.py:93-103)
          const unsigned u = gidx >> G::LOG, v = gidx & (F - 1);
          const bool self = ((2 * u) & (F - 1)) == 0 && ((2 * v) & (F - 1)) == 0;
          float pr, pi;
          if (self) {
            pr = __fdividef(are, w00);
            pi = 0.f;
          } else {
            const int wi2 = (int)((((2 * u) & (F - 1)) * F) + ((2 * v) & (F - 1)));
            const float wx = Tre[wi2], wy = Tim[wi2];
            const float nr = w00 * are - (wx * are + wy * aim);
            const float ni = w00 * aim - (wy * are - wx * aim);
            const float d = w00 * w00 - (wx * wx + wy * wy);
            const float rd = __fdividef(1.f, d);
            pr = nr * rd;
            pi = ni * rd;
          }
          unsigned mi = (((F - u) & (F - 1)) << G::LOG) | ((F - v) & (F - 1));
          if (!self && mi < gidx) {  // canonical member (rfse.py:113-121)
            const unsigned t = gidx;
            gidx = mi;
            mi = t;
            pi = -pi;
          }
          midx = self ? gidx : mi;
          cre = a.gamma * pr;
          cim = a.gamma * pi;
          c2re = self ? 0.f : cre;
          c2im = self ? 0.f : -cim;
          tally += self ? 1 : 2;
          if (st == 0) {
            FSE_CHECK(a.trace_scratch || (unsigned)it * 16u < (unsigned)(G::SCRATCH - rf_t2_bytes<F>()));
            sp.trace[it] = make_float4(__uint_as_float(gidx | (self ? 0x80000000u : 0u)), cre, cim,
                                       __uint_as_float(gkey));
          }
          nit = it + 1;
        }
      }
    } else {
      // ---------------------------------------- rFSE (rfse.py:69-160)
      // The selection scans the joint projection of every bin onto its
      // conjugate pair (crit, a quadratic form of R_w[k] with per-bin
      // coefficients from the shared pair tables); the winner's projection
      // (p_re, p_im) follows from its residual and W[2u, 2v] with the
      // reference's divisions; a pair pick updates R_w with both atoms,
      // R_w -= c W[k - p] + conj(c) W[k + p], a self-conjugate pick with one.
      const float w00 = 1.f / __ldg(a.inv_w00 + cls);
      const unsigned rt4 = __shfl_sync(
          0xffffffffu,
          (unsigned)__cvta_generic_to_shared(region + G::TABLE_BYTES) + (unsigned)(rowbase * 32 + lane) * 16u,
          lane);
      const unsigned rt2 = __shfl_sync(
          0xffffffffu,
          (unsigned)__cvta_generic_to_shared(region + G::TABLE_BYTES + F * F / 2 * sizeof(float4)) +
              (unsigned)(rowbase * 32 + lane) * 8u,
          lane);
#ifndef FSE_RSYM
#define FSE_RSYM 1  // centred-frame rFSE for mirror-symmetric classes at F = 32 / 64
#endif
      if (FSE_RSYM && sym) {
        // Centred frame (interior classes), as the F = 128 rFSE loop: crit =
        // alpha R~.re^2 + beta R~.im^2 with per-bin (alpha, beta) in the
        // pair-criterion table's place (one float4 (alpha_a, alpha_b,
        // beta_a, beta_b) per bin pair, doubled-frequency wraps already
        // applied), the update reads the real Q pair table (one LDS.64 per
        // atom) at both atoms' shifts, the mirror atom with sg conj(c~).
        constexpr unsigned RSB = (F == 32 ? 2u : 1u) * (unsigned)G::SYM_C * 8u;  // bytes per pair step
        const unsigned crit0 = (unsigned)__cvta_generic_to_shared(region + G::TABLE_BYTES);
        constexpr bool TW = FSE_RTWIST && F == 64;
        // twisted layout: (alpha, beta) per (row, lane), 8 B entries
        const unsigned rt2c = __shfl_sync(0xffffffffu, crit0 + (unsigned)(rowbase * 32 + lane) * 8u, lane);
        unsigned midx = 0;
        float c2re = 0.f, c2im = 0.f;
        int tally = 0;
        nit = 0;
#pragma unroll 1
        for (int it = 0; it < a.iterations && tally < a.stop_tally; ++it) {
          const unsigned k0 = kpos + (unsigned)(G::SYM_C - F) * (kpos >> G::LOG) + (unsigned)((F - 1) * (G::SYM_C + 1));
          const unsigned tq1 = tbase + ((k0 - gidx - (unsigned)(G::SYM_C - F) * (gidx >> G::LOG)) << 3);
          const unsigned tq2 = tbase + ((k0 - midx - (unsigned)(G::SYM_C - F) * (midx >> G::LOG)) << 3);
          const float2 k1a = make_float2(-cre, -cim), k1b = make_float2(-cim, -cre);
          const float2 k2a = make_float2(-c2re, -c2im), k2b = make_float2(-c2im, -c2re);
          float bst = -1.f, bxs = 0.f;
          int bps = 0;
#pragma unroll
          for (int p = 0; p < G::NP; ++p) {
            FSE_CHECK((tq1 - tbase) / 8 + (unsigned)p * (RSB / 8) < (unsigned)(G::SYM_R * G::SYM_C));
            FSE_CHECK((tq2 - tbase) / 8 + (unsigned)p * (RSB / 8) < (unsigned)(G::SYM_R * G::SYM_C));
            const float2 q1 = lds64f(tq1 + (unsigned)p * RSB), q2 = lds64f(tq2 + (unsigned)p * RSB);
            float2 cr;
            if constexpr (TW) {
              // A = (re_a, im_b) -= (c.re, c.im) q, B = (im_a, re_b) -= (c.im, c.re) q
              ffma2_acc2(Rre[p], q1, k1a);
              ffma2_acc2(Rim[p], q1, k1b);
              ffma2_acc2(Rre[p], q2, k2a);
              ffma2_acc2(Rim[p], q2, k2b);
              const float2 ab = lds64f(rt2c + (unsigned)(p * 32 * 8));  // (alpha, beta) of member a
              const float2 t1 = fmul2(Rre[p], Rre[p]), t2 = fmul2(Rim[p], Rim[p]);
              cr = fmul2(t1, make_float2(ab.x, ab.x));
              cr = ffma2(t2, make_float2(ab.y, ab.y), cr);
            } else {
              ffma2_acc(Rre[p], q1, -cre);
              ffma2_acc(Rim[p], q1, -cim);
              ffma2_acc(Rre[p], q2, -c2re);
              ffma2_acc(Rim[p], q2, -c2im);
              const float4 ab = lds128f(rt4 + (unsigned)(p * 32 * 16));  // (alpha_a, alpha_b, beta_a, beta_b)
              const float2 t1 = fmul2(make_float2(ab.x, ab.y), Rre[p]);
              const float2 t2 = fmul2(make_float2(ab.z, ab.w), Rim[p]);
              cr = fmul2(t1, Rre[p]);
              cr = ffma2(t2, Rim[p], cr);
            }
            first_max(bst, bps, bxs, cr, p);
          }
          const int myidx = bin_index<F>(w, lane, bps, bxs >= bst ? 0 : 1);
          const unsigned key = __float_as_uint(fmaxf(bst, 0.f));  // monotone as unsigned
          const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
          const unsigned widx =
              __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
          int pw, mw, ow;
          decode_bin<F>((int)widx, w, pw, mw, ow);
          float are, aim;
          pick_bin<G::NP>(Rre, Rim, pw, mw, are, aim);
          if (TW && mw) {  // twisted pairs hold member b as (im, re)
            const float t = are;
            are = aim;
            aim = t;
          }
          are = __shfl_sync(0xffffffffu, are, ow);
          aim = __shfl_sync(0xffffffffu, aim, ow);
          gidx = widx;
          unsigned gkey = wmax;
          if constexpr (G::NW == 2) {
            if (lane == 0)
              sts128u(xc + 16u * w, make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim)));
            slot_sync<F>(slot);
            const uint4 o = lds128u(xc + 16u * (unsigned)(w ^ 1));
            if (o.x > wmax || (o.x == wmax && o.y < widx)) {
              gidx = o.y;
              gkey = o.x;
              are = __uint_as_float(o.z);
              aim = __uint_as_float(o.w);
            }
            xc ^= (unsigned)(G::NW * sizeof(uint4));
          }
          // (alpha, beta) of the chosen bin: its table entry and member
          const unsigned u = gidx >> G::LOG, v = gidx & (F - 1);
          const bool self = ((2 * u) & (F - 1)) == 0 && ((2 * v) & (F - 1)) == 0;
          const unsigned ent = F == 32 ? (u >> 1) * 32u + v : u * 32u + (v & 31u);
          const bool mb = F == 32 ? (u & 1u) != 0u : ((v >> 5) & 1u) != 0u;
          float wal, wbe;
          if constexpr (TW) {  // (alpha, beta) of member a; member b swaps them
            const float2 e2 = lds64f(crit0 + ent * 8u);
            wal = mb ? e2.y : e2.x;
            wbe = mb ? e2.x : e2.y;
          } else {
            const float4 e4 = lds128f(crit0 + ent * 16u);
            wal = mb ? e4.y : e4.x;
            wbe = mb ? e4.w : e4.z;
          }
          const float fac = self ? 1.f : 0.5f;
          float pr = fac * wal * are, pi = fac * wbe * aim;
          const float sg = ((u != 0u) != (v != 0u)) ? -1.f : 1.f;
          unsigned mi = (((F - u) & (F - 1)) << G::LOG) | ((F - v) & (F - 1));
          if (!self && mi < gidx) {  // canonical member (rfse.py:113-121)
            const unsigned t = gidx;
            gidx = mi;
            mi = t;
            pr = sg * pr;
            pi = -sg * pi;
          }
          midx = self ? gidx : mi;
          cre = a.gamma * pr;
          cim = a.gamma * pi;
          c2re = self ? 0.f : sg * cre;
          c2im = self ? 0.f : -sg * cim;
          tally += self ? 1 : 2;
          if (st == 0)
            sp.trace[it] = make_float4(__uint_as_float(gidx | (self ? 0x80000000u : 0u)), cre, cim,
                                       __uint_as_float(gkey));
          nit = it + 1;
        }
      } else {
      unsigned midx = 0;            // bin of the previous pick's second atom
      float c2re = 0.f, c2im = 0.f;  // its coefficient (conj c, or 0 after a self-conjugate pick)
      int tally = 0;
      nit = 0;
#pragma unroll 1
      for (int it = 0; it < a.iterations && tally < a.stop_tally; ++it) {
        constexpr unsigned RM = (unsigned)(F - 1) << G::LOG;
        const unsigned tp =
            tbase + ((((kpos - (gidx & RM)) & RM) | ((kpos - gidx) & (unsigned)(F - 1))) << 4);
        const unsigned tq =
            tbase + ((((kpos - (midx & RM)) & RM) | ((kpos - midx) & (unsigned)(F - 1))) << 4);
        float best = -1.f, bx = 0.f;
        int bp = 0;
#pragma unroll
        for (int p = 0; p < G::NP; ++p) {
          const unsigned po = (unsigned)((F == 32 ? 2 * p : p) * F * 16);  // the pair's table row
          const float4 wv = lds128f(tp + po);
          const float4 wq = lds128f(tq + po);
          const float2 wr = make_float2(wv.x, wv.y), wi = make_float2(wv.z, wv.w);
          const float2 qr = make_float2(wq.x, wq.y), qi = make_float2(wq.z, wq.w);
          ffma2_acc(Rre[p], wr, -cre);
          ffma2_acc(Rre[p], wi, cim);
          ffma2_acc(Rim[p], wi, -cre);
          ffma2_acc(Rim[p], wr, -cim);
          ffma2_acc(Rre[p], qr, -c2re);
          ffma2_acc(Rre[p], qi, c2im);
          ffma2_acc(Rim[p], qi, -c2re);
          ffma2_acc(Rim[p], qr, -c2im);
          // crit = A re^2 + C im^2 - D re im = re (A re - D im) + im (C im)
          const float4 b4 = lds128f(rt4 + (unsigned)(p * 32 * 16));  // (A_a, A_b, C_a, C_b)
          const float2 dd = lds64f(rt2 + (unsigned)(p * 32 * 8));     // (-D_a, -D_b)
          float2 t1 = fmul2(make_float2(b4.x, b4.y), Rre[p]);
          t1 = ffma2(dd, Rim[p], t1);
          const float2 t2 = fmul2(make_float2(b4.z, b4.w), Rim[p]);
          float2 cr2 = fmul2(t1, Rre[p]);
          cr2 = ffma2(t2, Rim[p], cr2);
          const float m = fmaxf(cr2.x, cr2.y);
          if (m > best) { best = m; bp = p; bx = cr2.x; }
        }
        const int myidx = bin_index<F>(w, lane, bp, bx >= best ? 0 : 1);
        const unsigned key = __float_as_uint(fmaxf(best, 0.f));  // monotone as unsigned
        const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
        const unsigned widx =
            __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
        int pw, mw, ow;
        decode_bin<F>((int)widx, w, pw, mw, ow);
        float are, aim;
        pick_bin<G::NP>(Rre, Rim, pw, mw, are, aim);
        are = __shfl_sync(0xffffffffu, are, ow);
        aim = __shfl_sync(0xffffffffu, aim, ow);
        gidx = widx;
        unsigned gkey = wmax;
        if constexpr (G::NW == 2) {
          if (lane == 0)
            sts128u(xc + 16u * w, make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim)));
          slot_sync<F>(slot);
          const uint4 o = lds128u(xc + 16u * (unsigned)(w ^ 1));
          if (o.x > wmax || (o.x == wmax && o.y < widx)) {
            gidx = o.y;
            gkey = o.x;
            are = __uint_as_float(o.z);
            aim = __uint_as_float(o.w);
          }
          xc ^= (unsigned)(G::NW * sizeof(uint4));
        }
        // joint projection of the chosen bin (rfse.py:93-103)
        const unsigned u = gidx >> G::LOG, v = gidx & (F - 1);
        const bool self = ((2 * u) & (F - 1)) == 0 && ((2 * v) & (F - 1)) == 0;
        float pr, pi;
        // (fast-path divisions: an IEEE '/' calls a slow-path subroutine whose
        // calling convention makes ptxas move the spectrum registers each iteration)
        if (self) {
          pr = __fdividef(are, w00);
          pi = 0.f;
        } else {
          // W[2u, 2v]: member a of the W' table entry (row 2u, column 2v)
          const float4 e = lds128f(tbase + ((((2 * u) & (F - 1)) * F + ((2 * v) & (F - 1))) << 4));
          const float nr = w00 * are - (e.x * are + e.z * aim);
          const float ni = w00 * aim - (e.z * are - e.x * aim);
          const float d = w00 * w00 - (e.x * e.x + e.z * e.z);
          const float rd = __fdividef(1.f, d);
          pr = nr * rd;
          pi = ni * rd;
        }
        // the pair is represented by its smaller row-major member (rfse.py:113-121)
        unsigned mi = (((F - u) & (F - 1)) << G::LOG) | ((F - v) & (F - 1));
        if (!self && mi < gidx) {
          const unsigned t = gidx;
          gidx = mi;
          mi = t;
          pi = -pi;
        }
        midx = self ? gidx : mi;
        cre = a.gamma * pr;
        cim = a.gamma * pi;
        c2re = self ? 0.f : cre;
        c2im = self ? 0.f : -cim;
        tally += self ? 1 : 2;
        if (st == 0)
          sp.trace[it] = make_float4(__uint_as_float(gidx | (self ? 0x80000000u : 0u)), cre, cim,
                                     __uint_as_float(gkey));
        nit = it + 1;
      }
      }
    }
    slot_sync<F>(slot);
    FSE_TMARK(5);

    // ------------------------------------ coefficients, trace, synthesis
    // trace[it] = (index, R_w[u,v]) -> (u | v << 16, c, |R_w[u,v]|^2), and
    // cq[it] = (c, c2) as (re, re2, -im, -im2) with c2 = c e^{2 pi i u (B/2) / F}
    // for the second pixel row of the synthesis (below)
    // (rFSE: trace[it] = (index | self << 31, c, criterion); a pair pick
    // contributes c phi + conj(c) phi*, i.e. twice Re{c phi} on real pixels)
    float4 *const cq = sp.trace + a.iterations;
    for (int k = st; k < (ALG ? nit : a.iterations); k += G::NT) {
      const float4 tr = sp.trace[k];
      float cr, ci, aux, fac = 1.f;
      unsigned gi = __float_as_uint(tr.x);
      if constexpr (ALG == 0) {
        cr = ginv * tr.y;
        ci = ginv * tr.z;
        aux = tr.y * tr.y + tr.z * tr.z;
        if (sym) {  // back from the centred frame: c = c~ e^{-i pi (u + v)(F - 1) / F}
          const float2 r = rot_tw[(gi >> G::LOG) + (gi & (F - 1))];
          const float c0 = cr;
          cr = c0 * r.x + ci * r.y;
          ci = ci * r.x - c0 * r.y;
        }
      } else {
        fac = (gi >> 31) ? 1.f : 2.f;
        gi &= 0x7fffffffu;
        cr = tr.y;
        ci = tr.z;
        aux = __uint_as_float(__float_as_uint(tr.w));
        if (sym) {  // back from the centred frame: c = c~ phi(u, v)
          const float2 r = rot_tw[(gi >> G::LOG) + (gi & (F - 1))];
          const float c0 = cr;
          cr = c0 * r.x + ci * r.y;
          ci = ci * r.x - c0 * r.y;
        }
      }
      const unsigned tu = gi >> G::LOG;
      sp.trace[k] = make_float4(__uint_as_float(tu | ((gi & (F - 1)) << 16)), cr, ci, aux);
      const float2 om = syn_tw[(tu * (G::B / 2)) & (F - 1)];
      cq[k] = make_float4(fac * cr, fac * (cr * om.x - ci * om.y), -fac * ci,
                          -fac * (cr * om.y + ci * om.x));
#if FSE_DIAG & 32
      sp.trace[k].w = tr.w;
#endif
    }
    slot_sync<F>(slot);
    if (a.trace_uv) {  // trace outputs; energies e_t = e_{t-1} - gamma (2 - gamma) |R_w[u,v]|^2 / W00
      if (st == 0) {
        // cFSE: e -= gamma (2 - gamma) |R_w[u,v]|^2 / W00;  rFSE: e -= gamma (2 - gamma) crit
        const float dinv = ALG == 0 ? a.gamma * (2.f - a.gamma) * __ldg(a.inv_w00 + cls)
                                    : a.gamma * (2.f - a.gamma);
        float e = 0.f;
        for (int k = 0; k < G::NW; ++k) e += sp.red[k];
        for (int it = 0; it < a.iterations; ++it) {
          const size_t o = (size_t)b * a.iterations + it;
          if (ALG == 1 && it >= nit) {  // rFSE stopped at the tally target: unused entries
            a.trace_uv[2 * o] = -1;
            a.trace_uv[2 * o + 1] = -1;
            a.trace_c[2 * o] = 0.f;
            a.trace_c[2 * o + 1] = 0.f;
            a.trace_e[o] = e;
            continue;
          }
          const float4 tr = sp.trace[it];
          const unsigned uv = __float_as_uint(tr.x);
          e -= dinv * tr.w;
#if FSE_DIAG & 32
          // timing probe: iteration start clock, CTA/slot
          a.trace_uv[2 * o] = (int)__float_as_uint(tr.w);
          a.trace_uv[2 * o + 1] = (int)(blockIdx.x * 8 + slot);
          a.trace_e[o] = 0.f;
#else
          a.trace_uv[2 * o] = (int)(uv & 0xffffu);
          a.trace_uv[2 * o + 1] = (int)(uv >> 16);
          a.trace_e[o] = e;
#endif
          a.trace_c[2 * o] = tr.y;
          a.trace_c[2 * o + 1] = tr.z;
        }
      }
    }
    // Synthesis.  The slot's threads form SG groups; group sg sums the
    // coefficients it = sg (mod SG) (short dependent chains), thread gt of a
    // group owns PP pixel pairs (m, n), (m + B/2, n) with m = m0 + RS k.  The
    // two pixels of a pair differ in phase by u (B/2) / F = u / 8 turns, so
    // one twiddle lookup serves both:
    //   g(m, n)       += Re{c  t},   t = e^{2 pi i (u m + v n) / F}
    //   g(m + B/2, n) += Re{c2 t},  c2 = c e^{2 pi i u (B/2) / F}.
    // (the two-warp F=32 latency build: the first warp alone, exactly as the
    // one-warp build, so both give the same pixels)
#ifndef FSE_SYN_GT
// synthesis threads per coefficient group; the F=64 latency builds set the
// throughput build's 16, so their synthesis runs exactly its code on the same
// threads' worth of pixels (bit-identical tiles) while the other warps wait
#define FSE_SYN_GT 0
#endif
    constexpr int GT0 = G::NT / G::SG < G::B * G::B / 2 ? G::NT / G::SG : G::B * G::B / 2;
    constexpr int BB = G::B * G::B, SG = G::SG, GT = FSE_SYN_GT > 0 && FSE_SYN_GT < GT0 ? FSE_SYN_GT : GT0,
                  PP = BB / GT / 2, RS = GT / G::B;
    static_assert(PP * GT * 2 == BB, "pixel pairs cover the block");
    const bool syn = st < SG * GT;
    const int sg = st / GT, gt = st - sg * GT;
    const int pm = off + gt / G::B, pn = off + gt % G::B;
    float2 g[PP];  // (pixel (m, n), pixel (m + B/2, n)) of pair k
#pragma unroll
    for (int k = 0; k < PP; ++k) g[k] = make_float2(0.f, 0.f);
#if FSE_DIAG & 8
    if (false)
#endif
#pragma unroll 2
    for (int it = sg; syn && it < (ALG ? nit : a.iterations); it += SG) {
      const unsigned uv = __float_as_uint(((const float *)sp.trace)[4 * it]);
      const float4 c4 = cq[it];
      const float2 cr = make_float2(c4.x, c4.y), ci = make_float2(c4.z, c4.w);
      const int tu = (int)(uv & 0xffffu), j0 = tu * pm + (int)(uv >> 16) * pn;
      // twiddles of the thread's rows m0 + RS k by recurrence t_{k+1} = t_k w,
      // w = e^{2 pi i u RS / F}: two lookups per coefficient instead of PP
      float2 t = syn_tw[j0 & (F - 1)];
      const float2 wv = syn_tw[(tu * RS) & (F - 1)];
      const float2 wa = make_float2(wv.x, wv.y), wb = make_float2(-wv.y, wv.x);
#pragma unroll
      for (int k = 0; k < PP; ++k) {
        g[k] = ffma2(cr, make_float2(t.x, t.x), g[k]);
        g[k] = ffma2(ci, make_float2(t.y, t.y), g[k]);
        if (k + 1 < PP) t = ffma2(make_float2(t.y, t.y), wb, fmul2(make_float2(t.x, t.x), wa));
      }
    }
    auto store_px = [&](int q, float gk) {
      const size_t o = (size_t)b * BB + (size_t)q;
      FSE_CHECK(b < a.n_blocks && q < BB);
      if (a.tile_dtype == 0) {
        ((uint8_t *)a.tiles)[o] = (uint8_t)__float2int_rn(fminf(fmaxf(gk, 0.f), 255.f));
      } else if (a.tile_dtype == 1) {
        ((float *)a.tiles)[o] = gk;
      } else {
        ((double *)a.tiles)[o] = (double)gk;
      }
    };
    if constexpr (SG > 1) {
      float *red = (float *)((char *)sp.scratch + G::SCRATCH - G::SYN_RED);
      if (syn) {
#pragma unroll
        for (int k = 0; k < PP; ++k) {
          red[sg * BB + gt + GT * k] = g[k].x;
          red[sg * BB + gt + GT * k + BB / 2] = g[k].y;
        }
      }
      slot_sync<F>(slot);
#pragma unroll
      for (int q = st; q < BB; q += G::NT) {
        float s = red[q];
#pragma unroll
        for (int s2 = 1; s2 < SG; ++s2) s += red[s2 * BB + q];
        store_px(q, s);
      }
    } else if (syn) {
#pragma unroll
      for (int k = 0; k < PP; ++k) {
        store_px(gt + GT * k, g[k].x);
        store_px(gt + GT * k + BB / 2, g[k].y);
      }
    }
    slot_sync<F>(slot);  // trace / scratch reuse by the next block
#if FSE_DIAG & 32
    FSE_TMARK(6);
    if (st == 0 && a.trace_c)
      for (int j = 1; j < 7 && j < a.iterations; ++j)
        a.trace_c[2 * ((size_t)b * a.iterations + j)] = (float)(tmk[j] - tmk[0]);
    if (st == 0 && !a.trace_c && a.tile_dtype == 1)  // no trace: marks over the f32 tile
      for (int j = 1; j < 7; ++j) ((float *)a.tiles)[(size_t)b * G::B * G::B + j] = (float)(tmk[j] - tmk[0]);
#endif
  }
}



template <int F, int ALG = 0> static size_t fast_smem(int iter_cap) {
  (void)iter_cap;
  return KS<F, ALG>::REGION + 4 * (size_t)F * sizeof(float2) + 512 +
         KS<F, ALG>::S * slot_stride<F>(true);
}

bool fast_config(int F, int iterations, int sm_count, FastConfig *cfg, int algorithm) {
  size_t smem, tb;
  int S;
#ifdef FSE_FAST_ONLY64
  if (F != 64 || algorithm != 0) return false;
#endif
#ifdef FSE_FAST_ONLY32
  if (F != 32 || algorithm != 0) return false;
#endif
  if (algorithm == 1) {  // fused rFSE: F = 32, 64; F = 128 centred-frame classes only
    if (F != 32 && F != 64 && F != 128) return false;
    // (F = 128: the trace must also stay clear of the criterion table in the
    // scratch tail during the iterations)
    constexpr int cap128 = (int)((FG<128>::SCRATCH - rf_t2_bytes<128>()) / 16) < FG<128>::TRACE_CAP
                               ? (int)((FG<128>::SCRATCH - rf_t2_bytes<128>()) / 16)
                               : FG<128>::TRACE_CAP;
    cfg->global_trace = iterations > (F == 32 ? FG<32>::TRACE_CAP : F == 64 ? FG<64>::TRACE_CAP : cap128);
    smem = F == 32 ? fast_smem<32, 1>(0) : F == 64 ? fast_smem<64, 1>(0) : fast_smem<128, 1>(0);
    if (smem > 227 * 1024) return false;
    cfg->slots = F == 32 ? rf_slots<32>() : F == 64 ? rf_slots<64>() : rf_slots<128>();
    cfg->threads = F == 32 ? KS<32, 1>::CTA : F == 64 ? KS<64, 1>::CTA : KS<128, 1>::CTA;
    cfg->smem_bytes = (int)smem;
    cfg->grid = sm_count;
    cfg->table_bytes = F == 32   ? FG<32>::TABLE_BYTES + rf_t2_bytes<32>()
                       : F == 64 ? FG<64>::TABLE_BYTES + rf_t2_bytes<64>()
                                 : FG<128>::TABLE_BYTES + rf_t2_bytes<128>();
    return true;
  }
  switch (F) {
    case 32:
      cfg->global_trace = iterations > FG<32>::TRACE_CAP;
      smem = fast_smem<32>(0); tb = FG<32>::TABLE_BYTES; S = FG<32>::S;
      break;
    case 64:
      cfg->global_trace = iterations > FG<64>::TRACE_CAP;
      smem = fast_smem<64>(0); tb = FG<64>::TABLE_BYTES; S = FG<64>::S;
      break;
    case 128: {
      cfg->global_trace = iterations > FG<128>::TRACE_CAP;
      smem = fast_smem<128>(0); tb = FG<128>::TABLE_BYTES; S = FG<128>::S;
      break;
    }
    default:
      return false;
  }
  if (smem > 227 * 1024) return false;
  cfg->slots = S;
  cfg->threads = F == 32 ? FG<32>::CTA : F == 64 ? FG<64>::CTA : FG<128>::CTA;
  cfg->smem_bytes = (int)smem;
  cfg->grid = sm_count;
  cfg->table_bytes = tb;
  return true;
}

template <int F, int ALG> static cudaError_t launch_fast_t(const FastArgs &a, const FastConfig &cfg,
                                                          const CUtensorMap *tmap, cudaStream_t s) {
  auto kern = tmap ? fast_kernel<F, true, ALG> : fast_kernel<F, false, ALG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       cfg.smem_bytes);
  if (e != cudaSuccess) return e;
  int grid = cfg.grid < a.n_rounds ? cfg.grid : a.n_rounds;
  if (grid <= 0) return cudaSuccess;
  CUtensorMap none;
  memset(&none, 0, sizeof none);
  kern<<<grid, cfg.threads, cfg.smem_bytes, s>>>(a, 0, tmap ? *tmap : none);
  return cudaGetLastError();
}

cudaError_t launch_fast(const FastArgs &a, const FastConfig &cfg, const CUtensorMap *tmap,
                        cudaStream_t s) {
#if defined(FSE_FAST_ONLY64)
  return a.F == 64 && a.algorithm == 0 ? launch_fast_t<64, 0>(a, cfg, tmap, s) : cudaErrorInvalidValue;
#elif defined(FSE_FAST_ONLY32)
  return a.F == 32 && a.algorithm == 0 ? launch_fast_t<32, 0>(a, cfg, tmap, s) : cudaErrorInvalidValue;
#else
  if (a.algorithm == 1)
    return a.F == 64    ? launch_fast_t<64, 1>(a, cfg, tmap, s)
           : a.F == 32  ? launch_fast_t<32, 1>(a, cfg, tmap, s)
           : a.F == 128 ? launch_fast_t<128, 1>(a, cfg, tmap, s)
                        : cudaErrorInvalidValue;
  switch (a.F) {
    case 32: return launch_fast_t<32, 0>(a, cfg, tmap, s);
    case 64: return launch_fast_t<64, 0>(a, cfg, tmap, s);
    case 128: return launch_fast_t<128, 0>(a, cfg, tmap, s);
  }
  return cudaErrorInvalidValue;
#endif
}

size_t fast_stage_bytes(int F) {
  return F == 32 ? FG<32>::STAGE : F == 64 ? FG<64>::STAGE : F == 128 ? FG<128>::STAGE : 0;
}

// ---------------------------------------------------------- class setup
// One CTA per geometry class: w, W = DFT(w) (fp64, symmetrised), fp32
// tables in the fast kernel's layout.

__global__ void __launch_bounds__(512) class_setup_kernel(ClassSetupArgs a) {
  extern __shared__ __align__(16) char smem[];
  const int F = a.F, FF = F * F, c = blockIdx.x;
  double2 *tw = (double2 *)smem;
  for (int j = threadIdx.x; j < F; j += blockDim.x) tw[j] = twiddle(j, F, -1);
  const int8_t *lab = a.labels + (size_t)c * FF;
  double *w64 = a.w64 + (size_t)c * FF;
  double2 *W = (double2 *)a.W64 + (size_t)c * FF;
  double2 *T = (double2 *)a.tmp + (size_t)c * FF;
  for (int i = threadIdx.x; i < FF; i += blockDim.x) {
    const int m = i / F, n = i - m * F;
    double dm = (double)m - (F - 1) / 2.0, dn = (double)n - (F - 1) / 2.0;
    double w = lab[i] == kSupport ? pow(a.rho, hypot(dm, dn)) : 0.0;
    w64[i] = w;
    a.wtab[(size_t)c * FF + i] = (float)w;
    W[i] = make_double2(w, 0.0);
  }
  __syncthreads();
  dft_rows(W, T, F, F, tw);
  __syncthreads();
  dft_cols(T, W, F, F, tw);
  __syncthreads();
  // exact Hermitian symmetrisation (w is real)
  for (int i = threadIdx.x; i < FF; i += blockDim.x) {
    const int k = i / F, l = i - k * F;
    const int j = ((F - k) % F) * F + (F - l) % F;
    if (i > j) continue;
    double2 x = W[i], y = W[j];
    double re = (x.x + y.x) * 0.5, im = (x.y - y.y) * 0.5;
    W[i] = make_double2(re, im);
    W[j] = make_double2(re, -im);
  }
  __syncthreads();
  if (threadIdx.x == 0) a.w00[c] = W[0].x;
  if (a.dmin) {
    // rFSE pair Gram determinant check (rfse.py:47-55), for every rFSE plan:
    // min over non-self-conjugate bins of (W00^2 - |W[2k, 2l]|^2) / W00^2
    __shared__ double red[512];
    const double w00 = W[0].x;
    double dmin = 1e300;
    for (int i = threadIdx.x; i < FF; i += blockDim.x) {
      const int k = i / F, l = i - k * F;
      const int r2 = (2 * k) % F, c2 = (2 * l) % F;
      if (r2 == 0 && c2 == 0) continue;
      const double2 w2 = W[r2 * F + c2];
      dmin = fmin(dmin, (w00 * w00 - (w2.x * w2.x + w2.y * w2.y)) / (w00 * w00));
    }
    red[threadIdx.x] = dmin;
    __syncthreads();
    for (int s2 = blockDim.x / 2; s2 > 0; s2 >>= 1) {
      if ((int)threadIdx.x < s2) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s2]);
      __syncthreads();
    }
    if (threadIdx.x == 0) a.dmin[c] = red[0];
  }
  if (!a.fast_table) return;
  char *tab = (char *)a.fast_table + (size_t)c * a.fast_table_bytes;
  if (a.sym && a.sym[c]) {
    // Centred frame (mirror-symmetric weights, see the kernel's iteration
    // section): Q0[k][l] = W[k][l] e^{+i pi (k + l)(F - 1) / F} is real, and
    // Q(i, j) = sgn(i) sgn(j) Q0[i mod F][j mod F] for |i|, |j| < F.  Entry
    // (r, c) = (Q(i, j), Q(i + di, j + dj)), i = r - (F - 1), j = c - (F - 1),
    // (di, dj) = the offset of member b of a thread's bin pair.
    for (int i = threadIdx.x; i < FF; i += blockDim.x) {
      const int k = i / F, l = i - k * F;
      double sn, cs;
      sincospi((double)(((k + l) * (F - 1)) % (2 * F)) / F, &sn, &cs);
      T[i].x = W[i].x * cs - W[i].y * sn;
    }
    __syncthreads();
    auto q = [&](int i, int j) -> float {
      double sg = 1.0;
      if (i < 0) { i += F; sg = -sg; } else if (i >= F) { i -= F; sg = -sg; }
      if (j < 0) { j += F; sg = -sg; } else if (j >= F) { j -= F; sg = -sg; }
      return (float)(sg * T[i * F + j].x);
    };
    if (F == 128) {
      float *Tq = (float *)tab;
      for (int i = threadIdx.x; i < FG<128>::SYM_R * F; i += blockDim.x) {
        const int r = i / F, cc = i - r * F;
        Tq[i] = q(r - (F - 1), cc);
      }
      if (a.rfse) {
        // centred rFSE criterion table (the kernel's F = 128 rFSE loop):
        // alpha = 2 / (W00 + Q0), beta = 2 / (W00 - Q0) at the doubled
        // frequency (2 r2, 2 lane + 64 h); (1 / W00, 0) at (0, 0), the
        // self-conjugate bins.  alpha half, then beta half.
        const double w00 = W[0].x;
        float2 *CA = (float2 *)(tab + FG<128>::TABLE_BYTES), *CB = CA + 64 * 32;
        for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
          const int r2 = i >> 5, ln = i & 31;
          double al[2], be[2];
          for (int h = 0; h < 2; ++h) {
            const int k2 = 2 * r2, l2 = 2 * ln + 64 * h;
            const double q0 = T[k2 * F + l2].x;
            if (k2 == 0 && l2 == 0) {
              al[h] = 1.0 / w00;
              be[h] = 0.0;
            } else {
              al[h] = 2.0 / (w00 + q0);
              be[h] = 2.0 / (w00 - q0);
            }
          }
          CA[i] = make_float2((float)al[0], (float)al[1]);
          CB[i] = make_float2((float)be[0], (float)be[1]);
        }
      }
      return;
    }
    const int R = F == 32 ? FG<32>::SYM_R : FG<64>::SYM_R, C = F == 32 ? FG<32>::SYM_C : FG<64>::SYM_C;
    const int di = F == 32 ? 1 : 0, dj = F == 32 ? 0 : 32;
    float2 *E = (float2 *)tab;
    for (int i = threadIdx.x; i < R * C; i += blockDim.x) {
      const int r = i / C, cc = i - r * C, qi = r - (F - 1), qj = cc - (F - 1);
      E[i] = make_float2(q(qi, qj), q(qi + di, qj + dj));
    }
    if (a.rfse) {
      // centred rFSE criterion (the kernel's centred rFSE loop): per bin
      // pair of the thread layout (as the complex path's A4 entries)
      // (alpha_a, alpha_b, beta_a, beta_b), alpha = 2 / (W00 + s Q0), beta =
      // 2 / (W00 - s Q0) at the doubled frequency, s = -1 per doubled row or
      // column that wraps past F; self-conjugate bins (1 / W00, 0), swapped
      // when s = -1 (exactly the bins whose phase factor is imaginary)
      const double w00 = W[0].x;
      float4 *A4 = (float4 *)(tab + (F == 32 ? FG<32>::TABLE_BYTES : FG<64>::TABLE_BYTES));
      for (int i = threadIdx.x; i < FF / 2; i += blockDim.x) {
        const int r = i >> 5, cc = i & 31;
        double al[2], be[2];
        for (int h = 0; h < 2; ++h) {
          const int br = F == 32 ? 2 * r + h : r, bc = F == 32 ? cc : cc + 32 * h;
          const int r2 = 2 * br, c2 = 2 * bc;
          const bool flip = (r2 >= F) != (c2 >= F);
          const int k2 = r2 % F, l2 = c2 % F;
          double x, y;
          if (k2 == 0 && l2 == 0) {
            x = 1.0 / w00;
            y = 0.0;
          } else {
            const double q0 = T[k2 * F + l2].x;
            x = 2.0 / (w00 + q0);
            y = 2.0 / (w00 - q0);
          }
          al[h] = flip ? y : x;
          be[h] = flip ? x : y;
        }
        if (FSE_RTWIST && F == 64)  // twisted loop: member a's (alpha, beta) only
          ((float2 *)A4)[i] = make_float2((float)al[0], (float)be[0]);
        else
          A4[i] = make_float4((float)al[0], (float)al[1], (float)be[0], (float)be[1]);
      }
    }
    return;
  }
  if (F == 128) {
    const int TR = FG<128>::TROWS;
    float *Tre = (float *)tab, *Tim = Tre + TR * F;
    for (int i = threadIdx.x; i < TR * F; i += blockDim.x) {
      const int r = i / F, q = i - r * F;
      double2 x = W[(r % F) * F + q];
      Tre[i] = (float)x.x;
      Tim[i] = (float)x.y;
    }
    if (a.rfse) {
      // complex-frame rFSE criterion at the doubled frequency (2 r2, 2 lane +
      // 64 h): A = 2 (W00 - W2.re) / Dt, C = 2 (W00 + W2.re) / Dt, D = 4 W2.im /
      // Dt, Dt = W00^2 - |W2|^2; (1 / W00, 0, 0) at (0, 0) (rfse.py:86-111)
      const double w00 = W[0].x;
      float4 *C4 = (float4 *)(tab + FG<128>::TABLE_BYTES);
      float2 *C2 = (float2 *)(tab + FG<128>::TABLE_BYTES + 64 * 32 * sizeof(float4));
      for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
        const int r2 = i >> 5, ln = i & 31;
        double qa[2], qc[2], qd[2];
        for (int h = 0; h < 2; ++h) {
          const int k2 = 2 * r2, l2 = 2 * ln + 64 * h;
          if (k2 == 0 && l2 == 0) {
            qa[h] = 1.0 / w00;
            qc[h] = 0.0;
            qd[h] = 0.0;
          } else {
            const double2 w2 = W[k2 * F + l2];
            const double d = w00 * w00 - (w2.x * w2.x + w2.y * w2.y);
            qa[h] = 2.0 * (w00 - w2.x) / d;
            qc[h] = 2.0 * (w00 + w2.x) / d;
            qd[h] = 4.0 * w2.y / d;
          }
        }
        C4[i] = make_float4((float)qa[0], (float)qa[1], (float)qc[0], (float)qc[1]);
        C2[i] = make_float2((float)-qd[0], (float)-qd[1]);
      }
    }
  } else {
    const int TR = F == 32 ? FG<32>::TROWS : FG<64>::TROWS;
    float4 *T4 = (float4 *)tab;
    for (int i = threadIdx.x; i < TR * F; i += blockDim.x) {
      const int r = i / F, q = i - r * F;
      double2 x0 = W[(r % F) * F + q], x1;
      if (F == 32) x1 = W[((r + 1) % F) * F + q];
      else x1 = W[(r % F) * F + (q + 32) % F];
      T4[i] = make_float4((float)x0.x, (float)x1.x, (float)x0.y, (float)x1.y);
    }
    if (a.rfse && (F == 64 || F == 32)) {
      // rFSE pair tables (rfse.py:40-55, 86-111): the pair criterion
      // 2 (p.re a.re + p.im a.im) with p = [[W00 - W2.re, -W2.im], [-W2.im,
      // W00 + W2.re]] a / Dt, Dt = W00^2 - |W2|^2, W2 = W[2k, 2l], is
      // crit = A a.re^2 + C a.im^2 - D a.re a.im with A = 2 (W00 - W2.re) / Dt,
      // C = 2 (W00 + W2.re) / Dt, D = 4 W2.im / Dt; a self-conjugate bin
      // (crit = a.re^2 / W00) has A = 1 / W00, C = D = 0.
      // Entry i = (r, c) of the thread layout (32 columns): bins (r, c) and
      // (r, c + 32) at F = 64; bins (2r, c) and (2r + 1, c) at F = 32.
      const double w00 = W[0].x;
      const size_t TB = F == 32 ? FG<32>::TABLE_BYTES : FG<64>::TABLE_BYTES;
      float4 *A4 = (float4 *)(tab + TB);
      float2 *A2 = (float2 *)(tab + TB + (size_t)FF / 2 * sizeof(float4));
      for (int i = threadIdx.x; i < FF / 2; i += blockDim.x) {
        const int r = i >> 5, c = i & 31;
        double qa[2], qc[2], qd[2];
        for (int h = 0; h < 2; ++h) {
          const int br = F == 32 ? 2 * r + h : r, bc = F == 32 ? c : c + 32 * h;
          const int r2 = (2 * br) % F, c2 = (2 * bc) % F;
          if (r2 == 0 && c2 == 0) {
            qa[h] = 1.0 / w00;
            qc[h] = 0.0;
            qd[h] = 0.0;
          } else {
            const double2 w2 = W[r2 * F + c2];
            const double d = w00 * w00 - (w2.x * w2.x + w2.y * w2.y);
            qa[h] = 2.0 * (w00 - w2.x) / d;
            qc[h] = 2.0 * (w00 + w2.x) / d;
            qd[h] = 4.0 * w2.y / d;
          }
        }
        A4[i] = make_float4((float)qa[0], (float)qa[1], (float)qc[0], (float)qc[1]);
        A2[i] = make_float2((float)-qd[0], (float)-qd[1]);
      }
    }
  }
}

cudaError_t launch_class_setup(const ClassSetupArgs &a, cudaStream_t s) {
  if (a.n_classes <= 0) return cudaSuccess;
  size_t sm = (size_t)a.F * sizeof(double2);
  class_setup_kernel<<<a.n_classes, 512, sm, s>>>(a);
  return cudaGetLastError();
}

#ifdef FSE_FAST_NS
}  // namespace FSE_FAST_NS
#endif
}  // namespace fse

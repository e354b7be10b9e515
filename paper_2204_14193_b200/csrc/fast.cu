// fast.cu -- fused, register-resident fp32 cFSE kernel for F in {32,64,128}.
//
// One lost block per "slot" (a group of NT = F*F/32 threads, i.e. 32
// spectrum bins per thread held in registers); S slots per CTA share one
// shared-memory copy of their geometry class's weight spectrum W; one CTA
// per SM, persistent over a list of same-class rounds.
//
// Per block (all on chip):
//   load   s*w of the support ring from the frame (u8/f32/f64)   cfse.py:50
//   FFT    in-place radix-2 2-D FFT in the slot's shared scratch cfse.py:50
//   R_w -> registers, exactly Hermitian ((X[k] + conj X[-k]) / 2)
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
// 32 bins of a thread form 16 SoA pairs (a, b), consecutive in the thread's
// row-major scan order:
//   F=32 : a = (2p, lane),            b = (2p+1, lane)
//   F=64 : a = (16w+p, lane),         b = (16w+p, lane+32)
//   F=128: a = (8w+p/2, lane+64(p&1)), b = a + (0, 32)
#include "common.cuh"
#include "dft.cuh"
#include "kernels.h"

namespace fse {

template <int F> struct FG {
  static constexpr int LOG = F == 32 ? 5 : F == 64 ? 6 : 7;
  static constexpr int NT = F * F / 32;   // threads per slot
  static constexpr int NW = NT / 32;      // warps per slot
  static constexpr int CPL = F / 32;      // columns per lane
  static constexpr int RPW = 32 / CPL;    // rows per warp
  static constexpr int S = F == 32 ? 16 : F == 64 ? 4 : 1;
  static constexpr int CTA = NT * S;      // 512
  static constexpr bool PLANAR = F == 128;  // planar re/im table (pair table would not fit)
  static constexpr bool ALIAS = F == 128;   // FFT scratch and table share one region
  // rows of the row-extended table: the thread walks rows rowoff + step*p
  static constexpr int TROWS = F == 32 ? F + 31 : F == 64 ? F + 15 : F + 7;
  static constexpr size_t TABLE_BYTES =
      PLANAR ? (size_t)TROWS * F * 2 * sizeof(float) : (size_t)TROWS * F * sizeof(float4);
  static constexpr size_t SCRATCH = (size_t)F * F * sizeof(float2);
  static constexpr size_t REGION = ALIAS ? (TABLE_BYTES > SCRATCH ? TABLE_BYTES : SCRATCH) : TABLE_BYTES;
};

FSE_DEV float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
FSE_DEV float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

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

FSE_DEV float load_px(const void *frames, int dtype, size_t idx) {
  if (dtype == 0) return (float)__ldg((const uint8_t *)frames + idx);
  if (dtype == 1) return __ldg((const float *)frames + idx);
  return (float)__ldg((const double *)frames + idx);
}

// row-major bin index of pair p, member mem (0 = a, 1 = b) for thread (w, lane)
template <int F> FSE_DEV int bin_index(int w, int lane, int p, int mem) {
  if (F == 32) return (2 * p + mem) * 32 + lane;
  if (F == 64) return (16 * w + p) * 64 + lane + 32 * mem;
  return (8 * w + (p >> 1)) * 128 + lane + 64 * (p & 1) + 32 * mem;
}

// the pair index / member / owning lane of a bin owned by warp w (uniform)
template <int F> FSE_DEV void decode_bin(int idx, int w, int &p, int &mem, int &lane) {
  if (F == 32) {
    int row = idx >> 5;
    p = row >> 1; mem = row & 1; lane = idx & 31;
  } else if (F == 64) {
    int row = idx >> 6;
    p = row - 16 * w; mem = (idx >> 5) & 1; lane = idx & 31;
  } else {
    int row = idx >> 7, c = idx & 127;
    p = 2 * (row - 8 * w) + (c >> 6); mem = (c >> 5) & 1; lane = c & 31;
  }
}

#define FSE_PICK(P)                 \
  case P:                           \
    rr = Rre[P];                    \
    ri = Rim[P];                    \
    break;

// warp-uniform p: one indirect branch instead of a 16-way select chain
FSE_DEV void pick_pair(const float2 (&Rre)[16], const float2 (&Rim)[16], int p, float2 &rr,
                       float2 &ri) {
  switch (p) {
    FSE_PICK(0) FSE_PICK(1) FSE_PICK(2) FSE_PICK(3) FSE_PICK(4) FSE_PICK(5) FSE_PICK(6)
    FSE_PICK(7) FSE_PICK(8) FSE_PICK(9) FSE_PICK(10) FSE_PICK(11) FSE_PICK(12) FSE_PICK(13)
    FSE_PICK(14) default: rr = Rre[15]; ri = Rim[15]; break;
  }
}

// In-place radix-2 DIT 2-D FFT of the slot's F x F scratch (input stored in
// bit-reversed row and column order), forward kernel exp(-2 pi i / F).
template <int F>
FSE_DEV void slot_fft(float2 *S, const float2 *tw, int st, int slot) {
  constexpr int HALF = F / 2;
  // rows
#pragma unroll 1
  for (int lh = 0; lh < FG<F>::LOG; ++lh) {
    const int half = 1 << lh;
#pragma unroll 4
    for (int t = st; t < F * HALF; t += FG<F>::NT) {
      const int row = t / HALF, j = t - row * HALF;
      const int k = j & (half - 1);
      const int i0 = ((j >> lh) << (lh + 1)) + k, i1 = i0 + half;
      const float2 w = tw[k << (FG<F>::LOG - 1 - lh)];
      float2 a = S[row * F + i0], b = S[row * F + i1];
      float2 x = make_float2(b.x * w.x - b.y * w.y, b.x * w.y + b.y * w.x);
      S[row * F + i0] = make_float2(a.x + x.x, a.y + x.y);
      S[row * F + i1] = make_float2(a.x - x.x, a.y - x.y);
    }
    slot_sync<F>(slot);
  }
  // columns (consecutive threads -> consecutive columns: conflict-free)
#pragma unroll 1
  for (int lh = 0; lh < FG<F>::LOG; ++lh) {
    const int half = 1 << lh;
#pragma unroll 4
    for (int t = st; t < F * HALF; t += FG<F>::NT) {
      const int col = t & (F - 1), j = t >> FG<F>::LOG;
      const int k = j & (half - 1);
      const int i0 = ((j >> lh) << (lh + 1)) + k, i1 = i0 + half;
      const float2 w = tw[k << (FG<F>::LOG - 1 - lh)];
      float2 a = S[i0 * F + col], b = S[i1 * F + col];
      float2 x = make_float2(b.x * w.x - b.y * w.y, b.x * w.y + b.y * w.x);
      S[i0 * F + col] = make_float2(a.x + x.x, a.y + x.y);
      S[i1 * F + col] = make_float2(a.x - x.x, a.y - x.y);
    }
    slot_sync<F>(slot);
  }
}

// Cooperative copy of one class's table (global -> shared), 16 B per op.
FSE_DEV void copy_table(void *dst, const void *src, size_t bytes, int tid, int nthr) {
  const uint4 *s = (const uint4 *)src;
  uint4 *d = (uint4 *)dst;
  for (size_t i = tid; i < bytes / 16; i += nthr) d[i] = __ldg(s + i);
}

template <int F>
__global__ void __launch_bounds__(512, 1) fast_kernel(FastArgs a, int iter_cap) {
  typedef FG<F> G;
  extern __shared__ __align__(16) char smem[];
  char *region = smem;
  float2 *syn_tw = (float2 *)(smem + G::REGION);  // exp(+2 pi i j / F), j < F
  float2 *fft_tw = syn_tw + F;                     // exp(-2 pi i j / F), j < F/2
  char *slots_base = (char *)(fft_tw + F / 2);
  const size_t slot_bytes =
      (G::ALIAS ? 0 : G::SCRATCH) + 2 * G::NW * sizeof(uint4) + 64 +
      (G::ALIAS ? (size_t)iter_cap * sizeof(float4) : 0);

  const int tid = threadIdx.x;
  const int slot = tid / G::NT, st = tid - slot * G::NT;
  const int w = st >> 5, lane = st & 31;
  char *sb = slots_base + slot * slot_bytes;
  SlotPtrs<F> sp;
  sp.scratch = G::ALIAS ? (float2 *)region : (float2 *)sb;
  sp.xch = (uint4 *)(sb + (G::ALIAS ? 0 : G::SCRATCH));
  sp.red = (float *)(sp.xch + 2 * G::NW);
  sp.trace = G::ALIAS ? (float4 *)((char *)sp.red + 64) : (float4 *)sp.scratch;

  for (int j = tid; j < F; j += blockDim.x) {
    double s, c;
    sincospi(2.0 * j / F, &s, &c);
    syn_tw[j] = make_float2((float)c, (float)s);
    if (j < F / 2) fft_tw[j] = make_float2((float)c, (float)-s);
  }
  __syncthreads();

  const int off = (F - a.B) / 2;
  int loaded = -1;
  for (int round = blockIdx.x; round < a.n_rounds; round += gridDim.x) {
    const int cls = __ldg(a.round_class + round);
    if (!G::ALIAS && cls != loaded) {
      __syncthreads();
      copy_table(region, (const char *)a.table + (size_t)cls * a.table_bytes, a.table_bytes, tid,
                 blockDim.x);
      __syncthreads();
      loaded = cls;
    }
    const int b = __ldg(a.rounds + (size_t)round * G::S + slot);
    if (G::S == 1 && b < 0) continue;  // uniform for a single slot
    if (b < 0) continue;

    // ---------------------------------------------------------- load s*w
    const int fidx = __ldg(a.blocks + 3 * b), top = __ldg(a.blocks + 3 * b + 1),
              left = __ldg(a.blocks + 3 * b + 2);
    const int wt = top - off, wl = left - off;
    const float *wtab = a.wtab + (size_t)cls * F * F;
    const size_t fbase = (size_t)fidx * (size_t)a.frame_stride;
    float e0p = 0.f;
    for (int i = st; i < F * F; i += G::NT) {
      const int m = i >> G::LOG, n = i & (F - 1);
      const int y = wt + m, x = wl + n;
      const float wv = __ldg(wtab + i);
      float v = 0.f;
      if (wv != 0.f && y >= 0 && y < a.H && x >= 0 && x < a.W) {
        const float s = load_px(a.frames, a.dtype, fbase + (size_t)y * a.pitch + x);
        v = s * wv;
        e0p += v * s;
      }
      const int rm = __brev(m) >> (32 - G::LOG), rn = __brev(n) >> (32 - G::LOG);
      sp.scratch[rm * F + rn] = make_float2(v, 0.f);
    }
    slot_sync<F>(slot);
    slot_fft<F>(sp.scratch, fft_tw, st, slot);

    // ------------------------------- R_w -> registers, exactly Hermitian
    float2 Rre[16], Rim[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      float2 xa, xb, ma, mb;
      {
        const int ia = bin_index<F>(w, lane, p, 0), ib = bin_index<F>(w, lane, p, 1);
        const int ra = ia >> G::LOG, ca = ia & (F - 1), rb = ib >> G::LOG, cb = ib & (F - 1);
        xa = sp.scratch[ia];
        xb = sp.scratch[ib];
        ma = sp.scratch[((F - ra) & (F - 1)) * F + ((F - ca) & (F - 1))];
        mb = sp.scratch[((F - rb) & (F - 1)) * F + ((F - cb) & (F - 1))];
      }
      Rre[p] = make_float2((xa.x + ma.x) * 0.5f, (xb.x + mb.x) * 0.5f);
      Rim[p] = make_float2((xa.y - ma.y) * 0.5f, (xb.y - mb.y) * 0.5f);
    }
    // e0 = sum w s^2 (slot reduction; trace energies only)
    for (int o = 16; o; o >>= 1) e0p += __shfl_xor_sync(0xffffffffu, e0p, o);
    if (lane == 0) sp.red[w] = e0p;
    slot_sync<F>(slot);  // scratch is free from here on (trace area)
    float e = 0.f;
    if (st == 0)
      for (int k = 0; k < G::NW; ++k) e += sp.red[k];

    if (G::ALIAS) {  // single slot: bring the class table into the region
      copy_table(region, (const char *)a.table + (size_t)cls * a.table_bytes, a.table_bytes, tid,
                 blockDim.x);
      __syncthreads();
    }

    // ------------------------------------------------------- iterations
    const float ginv = a.gamma * __ldg(a.inv_w00 + cls);
    const float dinv = a.gamma * (2.f - a.gamma) * __ldg(a.inv_w00 + cls);
    float cre = 0.f, cim = 0.f;
    int u = 0, v = 0, parity = 0;
    const int rowbase = w * G::RPW;
#pragma unroll 1
    for (int it = 0; it < a.iterations; ++it) {
      const int rowoff = (rowbase - u) & (F - 1);
      float best = -1.f, bx = 0.f;
      int bp = 0;
      if (!G::PLANAR) {
        const int coloff = (lane - v) & (F - 1);
        const float4 *tp = (const float4 *)region + rowoff * F + coloff;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const float4 wv = tp[(F == 32 ? 2 * p : p) * F];
          const float2 wr = make_float2(wv.x, wv.y), wi = make_float2(wv.z, wv.w);
          Rre[p] = ffma2(wr, make_float2(-cre, -cre), Rre[p]);
          Rre[p] = ffma2(wi, make_float2(cim, cim), Rre[p]);
          Rim[p] = ffma2(wi, make_float2(-cre, -cre), Rim[p]);
          Rim[p] = ffma2(wr, make_float2(-cim, -cim), Rim[p]);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const float m = fmaxf(mg.x, mg.y);
          if (m > best) { best = m; bp = p; bx = mg.x; }
        }
      } else {
        const float *Tre = (const float *)region;
        const float *Tim = Tre + G::TROWS * F;
        int co[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) co[h] = (lane + 32 * h - v) & (F - 1);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int r = (rowoff + (p >> 1)) * F;
          const int q = 2 * (p & 1);
          const float2 wr = make_float2(Tre[r + co[q]], Tre[r + co[q + 1]]);
          const float2 wi = make_float2(Tim[r + co[q]], Tim[r + co[q + 1]]);
          Rre[p] = ffma2(wr, make_float2(-cre, -cre), Rre[p]);
          Rre[p] = ffma2(wi, make_float2(cim, cim), Rre[p]);
          Rim[p] = ffma2(wi, make_float2(-cre, -cre), Rim[p]);
          Rim[p] = ffma2(wr, make_float2(-cim, -cim), Rim[p]);
          float2 mg = fmul2(Rre[p], Rre[p]);
          mg = ffma2(Rim[p], Rim[p], mg);
          const float m = fmaxf(mg.x, mg.y);
          if (m > best) { best = m; bp = p; bx = mg.x; }
        }
      }
      // thread's first max (member a wins ties inside the pair)
      const int myidx = bin_index<F>(w, lane, bp, bx >= best ? 0 : 1);
      const unsigned key = __float_as_uint(best);  // best >= 0: monotone as unsigned
      const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
      const unsigned widx = __reduce_min_sync(0xffffffffu, key == wmax ? (unsigned)myidx : 0xffffffffu);
      int pw, mw, ow;
      decode_bin<F>((int)widx, w, pw, mw, ow);
      float2 rr, ri;
      pick_pair(Rre, Rim, pw, rr, ri);
      float are = __shfl_sync(0xffffffffu, mw ? rr.y : rr.x, ow);
      float aim = __shfl_sync(0xffffffffu, mw ? ri.y : ri.x, ow);
      unsigned gidx = widx, gkey = wmax;
      if (G::NW > 1) {
        uint4 *xc = sp.xch + parity * G::NW;
        if (lane == 0) xc[w] = make_uint4(wmax, widx, __float_as_uint(are), __float_as_uint(aim));
        slot_sync<F>(slot);
        const uint4 cnd = lane < G::NW ? xc[lane] : make_uint4(0u, 0xffffffffu, 0u, 0u);
        gkey = __reduce_max_sync(0xffffffffu, cnd.x);
        gidx = __reduce_min_sync(0xffffffffu, cnd.x == gkey ? cnd.y : 0xffffffffu);
        const int wl = (int)(gidx / (unsigned)(G::RPW * F));
        are = __shfl_sync(0xffffffffu, __uint_as_float(cnd.z), wl);
        aim = __shfl_sync(0xffffffffu, __uint_as_float(cnd.w), wl);
        parity ^= 1;
      }
      u = (int)(gidx >> G::LOG);
      v = (int)(gidx & (F - 1));
      cre = ginv * are;
      cim = ginv * aim;
      if (st == 0) {
        e -= dinv * (are * are + aim * aim);
        sp.trace[it] = make_float4(__uint_as_float((unsigned)u | ((unsigned)v << 16)), cre, cim, e);
        if (a.trace_uv) {
          const size_t o = (size_t)b * a.iterations + it;
          a.trace_uv[2 * o] = u;
          a.trace_uv[2 * o + 1] = v;
          a.trace_c[2 * o] = cre;
          a.trace_c[2 * o + 1] = cim;
          a.trace_e[o] = e;
        }
      }
      (void)gkey;
    }
    slot_sync<F>(slot);

    // ------------------------------------------------ synthesis + store
    constexpr int PX = 2;  // (F/4)^2 / NT loss pixels per thread
    float g[PX];
    int pm[PX], pn[PX];
#pragma unroll
    for (int k = 0; k < PX; ++k) {
      const int q = st + k * G::NT;
      pm[k] = off + q / a.B;
      pn[k] = off + q % a.B;
      g[k] = 0.f;
    }
#pragma unroll 2
    for (int it = 0; it < a.iterations; ++it) {
      const float4 tr = sp.trace[it];
      const unsigned uv = __float_as_uint(tr.x);
      const int tu = (int)(uv & 0xffffu), tv = (int)(uv >> 16);
#pragma unroll
      for (int k = 0; k < PX; ++k) {
        const float2 t = syn_tw[(tu * pm[k] + tv * pn[k]) & (F - 1)];
        g[k] = fmaf(tr.y, t.x, g[k]);
        g[k] = fmaf(-tr.z, t.y, g[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < PX; ++k) {
      const size_t o = (size_t)b * a.B * a.B + (size_t)(pm[k] - off) * a.B + (pn[k] - off);
      if (a.tile_dtype == 0) {
        ((uint8_t *)a.tiles)[o] = (uint8_t)__float2int_rn(fminf(fmaxf(g[k], 0.f), 255.f));
      } else if (a.tile_dtype == 1) {
        ((float *)a.tiles)[o] = g[k];
      } else {
        ((double *)a.tiles)[o] = (double)g[k];
      }
    }
    slot_sync<F>(slot);  // trace / scratch reuse by the next block
  }
}

template <int F> static size_t fast_smem(int iter_cap) {
  typedef FG<F> G;
  size_t slot_bytes = (G::ALIAS ? 0 : G::SCRATCH) + 2 * G::NW * sizeof(uint4) + 64 +
                      (G::ALIAS ? (size_t)iter_cap * sizeof(float4) : 0);
  return G::REGION + (size_t)F * sizeof(float2) + (size_t)(F / 2) * sizeof(float2) +
         G::S * slot_bytes;
}

bool fast_config(int F, int iterations, int sm_count, FastConfig *cfg) {
  size_t smem, tb;
  int S;
  switch (F) {
    case 32:
      if (iterations > 32 * 32 / 2) return false;
      smem = fast_smem<32>(0); tb = FG<32>::TABLE_BYTES; S = FG<32>::S;
      break;
    case 64:
      if (iterations > 64 * 64 / 2) return false;
      smem = fast_smem<64>(0); tb = FG<64>::TABLE_BYTES; S = FG<64>::S;
      break;
    case 128:
      smem = fast_smem<128>(iterations); tb = FG<128>::TABLE_BYTES; S = FG<128>::S;
      break;
    default:
      return false;
  }
  if (smem > 227 * 1024) return false;
  cfg->slots = S;
  cfg->threads = 512;
  cfg->smem_bytes = (int)smem;
  cfg->grid = sm_count;
  cfg->table_bytes = tb;
  return true;
}

template <int F> static cudaError_t launch_fast_t(const FastArgs &a, const FastConfig &cfg,
                                                 cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(fast_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       cfg.smem_bytes);
  if (e != cudaSuccess) return e;
  int grid = cfg.grid < a.n_rounds ? cfg.grid : a.n_rounds;
  if (grid <= 0) return cudaSuccess;
  fast_kernel<F><<<grid, cfg.threads, cfg.smem_bytes, s>>>(a, F == 128 ? a.iterations : 0);
  return cudaGetLastError();
}

cudaError_t launch_fast(const FastArgs &a, const FastConfig &cfg, cudaStream_t s) {
  switch (a.F) {
    case 32: return launch_fast_t<32>(a, cfg, s);
    case 64: return launch_fast_t<64>(a, cfg, s);
    case 128: return launch_fast_t<128>(a, cfg, s);
  }
  return cudaErrorInvalidValue;
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
  if (!a.fast_table) return;
  char *tab = (char *)a.fast_table + (size_t)c * a.fast_table_bytes;
  if (F == 128) {
    const int TR = F + 7;
    float *Tre = (float *)tab, *Tim = Tre + TR * F;
    for (int i = threadIdx.x; i < TR * F; i += blockDim.x) {
      const int r = i / F, q = i - r * F;
      double2 x = W[(r % F) * F + q];
      Tre[i] = (float)x.x;
      Tim[i] = (float)x.y;
    }
  } else {
    const int TR = F == 32 ? F + 31 : F + 15;
    float4 *T4 = (float4 *)tab;
    for (int i = threadIdx.x; i < TR * F; i += blockDim.x) {
      const int r = i / F, q = i - r * F;
      double2 x0 = W[(r % F) * F + q], x1;
      if (F == 32) x1 = W[((r + 1) % F) * F + q];
      else x1 = W[(r % F) * F + (q + 32) % F];
      T4[i] = make_float4((float)x0.x, (float)x1.x, (float)x0.y, (float)x1.y);
    }
  }
}

cudaError_t launch_class_setup(const ClassSetupArgs &a, cudaStream_t s) {
  if (a.n_classes <= 0) return cudaSuccess;
  size_t sm = (size_t)a.F * sizeof(double2);
  class_setup_kernel<<<a.n_classes, 512, sm, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fse

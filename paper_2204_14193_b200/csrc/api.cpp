// api.cpp -- C ABI (include/fse_b200.h): validation, the block planner
// (geometry classes, rounds), workspace management and kernel launches.
//
// Reference interfaces replaced (file:line under /root/reference/pkg/src/fse):
//   fse_dft2_f64          spectral.py:32-56   (np.fft.fft2 / ifft2)
//   fse_build_weight_f64  weighting.py:130-145
//   fse_cfse_kernel_f64   cfse.py:55-107      (numba _cfse_kernel)
//   fse_extrapolate       cfse.py:110-142     (extrapolate_cfse)
//   fse_select_basis_f64  cfse.py:145-154
//   fse_update_residual_f64 cfse.py:172-178
//   fse_plan_*            SPEC.md:332-340     (image-level conceal; absent in
//                                              the reference package)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <array>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/fse_b200.h"
#include "kernels.h"

#include <mutex>

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(FSE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call)                                      \
  do {                                                \
    cudaError_t _e = (call);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

int check_dims(int M, int N) {
  if (M < 1 || N < 1 || M > 4096 || N > 4096)
    return fail(FSE_ERR_UNSUPPORTED, "dims %dx%d outside [1, 4096]", M, N);
  return FSE_OK;
}

int check_rho_gamma(double rho, double gamma) {
  // types.py:41-44
  if (!(rho > 0.0 && rho < 1.0)) return fail(FSE_ERR_CONFIG, "rho_hat must be in (0, 1), got %g", rho);
  if (!(gamma > 0.0 && gamma <= 1.0)) return fail(FSE_ERR_CONFIG, "gamma must be in (0, 1], got %g", gamma);
  return FSE_OK;
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

}  // namespace

struct fse_plan {
  int n_blocks = 0, H = 0, W = 0, B = 0, border = 0, F = 0, iterations = 0, precision = 0;
  int algorithm = 0, stop_tally = 0;  // rFSE: stop a block at this basis-function tally
  double rho = 0, gamma = 0;
  int n_classes = 0, n_rounds = 0;
  bool fast = false;
  int variant = 0;  // fused-kernel build: 0 fast.cu, 1 fast_mid.cu (s32), 2 fast_small.cu (s16)
  bool tma_aligned = true;  // every window box starts on a 16-byte column (TMA legal)
  int max_frame = -1;       // largest frame index of the block list
  fse::FastConfig cfg{};
  // device
  int32_t *blocks = nullptr, *rounds = nullptr, *round_class = nullptr, *block_class = nullptr;
  int32_t *rects = nullptr;  // n_classes x (r0, c0, r1, c1): clipped support rectangle
  int32_t *class_sym = nullptr;  // n_classes: fused-kernel table in the centred frame (real Q)
  int n_sym = 0;                 // classes with the centred-frame table
  int8_t *labels = nullptr;
  float *wtab = nullptr, *inv_w00 = nullptr;
  void *table = nullptr;
  float4 *trace_scratch = nullptr;
  double *W64 = nullptr, *w64 = nullptr, *w00 = nullptr, *tmp = nullptr;
  // f64 path workspace
  int chunk = 0;
  double *cs = nullptr, *es = nullptr;
  int64_t *us = nullptr, *vs = nullptr;
  int32_t *status = nullptr;
  int32_t *selfs = nullptr, *counts = nullptr, *tallies = nullptr;  // generic rFSE outputs
  void *gen_ws = nullptr;
  std::vector<void *> owned;

  template <typename T> cudaError_t alloc(T **p, size_t n) {
    cudaError_t e = cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) owned.push_back((void *)*p);
    return e;
  }
  ~fse_plan() {
    for (void *p : owned) cudaFree(p);
  }
};

extern "C" {

const char *fse_version(void) { return "fse_b200 0.1 (sm_100a)"; }

int fse_last_error(char *buf, size_t len) {
  if (!buf || !len) return (int)g_err.size();
  snprintf(buf, len, "%s", g_err.c_str());
  return (int)g_err.size();
}

int fse_dft2_f64(int count, int M, int N, const double *in, double *out, int inverse, void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (count <= 0) return FSE_OK;
  if (!in || !out) return fail(FSE_ERR_VALUE, "null pointer");
  double *tmp = nullptr;
  CK(cudaMallocAsync((void **)&tmp, (size_t)count * M * N * 2 * sizeof(double), S(stream)));
  cudaError_t e = fse::launch_dft2_f64(count, M, N, in, out, inverse, tmp, S(stream));
  cudaFreeAsync(tmp, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dft2");
  return FSE_OK;
}

int fse_build_weight_f64(int count, int M, int N, const int8_t *labels, double rho, double *w,
                         void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (!(rho > 0.0 && rho < 1.0)) return fail(FSE_ERR_CONFIG, "rho_hat must be in (0, 1), got %g", rho);
  CK(fse::launch_build_weight_f64(count, M, N, labels, rho, w, S(stream)));
  return FSE_OK;
}

int fse_cfse_kernel_f64(int count, int M, int N, double *R_w, const double *W, long long w_stride,
                        double gamma, const double *inv_w00, int iterations, const double *e0,
                        double *G, int64_t *us, int64_t *vs, double *cs, double *es, void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (iterations < 0) return fail(FSE_ERR_CONFIG, "iterations must be >= 0");
  if (count <= 0) return FSE_OK;
  if (iterations == 0) {
    if (G) CK(cudaMemsetAsync(G, 0, (size_t)count * M * N * 2 * sizeof(double), S(stream)));
    return FSE_OK;
  }
  CK(fse::launch_cfse_kernel_f64(count, M, N, R_w, W, w_stride, gamma, inv_w00, iterations, e0, G,
                                 us, vs, cs, es, S(stream)));
  return FSE_OK;
}

int fse_extrapolate(int count, int M, int N, int precision, const double *signal,
                    const int8_t *labels, long long labels_stride, double rho, double gamma,
                    int iterations, double *recon, double *model, int64_t *us, int64_t *vs,
                    double *cs, double *es, int32_t *status, void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (int r = check_rho_gamma(rho, gamma)) return r;
  if (iterations < 0) return fail(FSE_ERR_CONFIG, "iterations must be >= 0");
  if (precision != FSE_PREC_F64 && precision != FSE_PREC_F32)
    return fail(FSE_ERR_UNSUPPORTED, "precision %d", precision);
  if (count <= 0) return FSE_OK;
  if (!signal || !labels || !recon || !status || (iterations > 0 && (!us || !vs || !cs || !es)))
    return fail(FSE_ERR_VALUE, "null pointer");
  const int chunk = 2048;
  for (int c0 = 0; c0 < count; c0 += chunk) {
    int n = std::min(chunk, count - c0);
    fse::GenArgs a{};
    a.count = n; a.M = M; a.N = N; a.iterations = iterations; a.precision = precision;
    a.rho = rho; a.gamma = gamma;
    a.signal = signal + (size_t)c0 * M * N;
    a.labels = labels + (size_t)c0 * labels_stride;
    a.labels_stride = labels_stride;
    a.label_index = nullptr;
    a.recon = recon + (size_t)c0 * M * N;
    a.model = model ? model + (size_t)c0 * 2 * M * N : nullptr;
    a.us = us ? us + (size_t)c0 * iterations : nullptr;
    a.vs = vs ? vs + (size_t)c0 * iterations : nullptr;
    a.cs = cs ? cs + (size_t)c0 * 2 * iterations : nullptr;
    a.es = es ? es + (size_t)c0 * iterations : nullptr;
    a.status = status + c0;
    size_t ws = fse::generic_workspace_bytes(n, M, N, precision);
    void *wsp = nullptr;
    if (ws) CK(cudaMallocAsync(&wsp, ws, S(stream)));
    cudaError_t e = fse::launch_generic_extrapolate(a, wsp, S(stream));
    if (wsp) cudaFreeAsync(wsp, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "extrapolate");
  }
  return FSE_OK;
}

int fse_extrapolate_rfse(int count, int M, int N, int precision, const double *signal,
                         const int8_t *labels, long long labels_stride, double rho, double gamma,
                         int max_iters, int stop_tally, double *recon, double *model, int64_t *us,
                         int64_t *vs, double *cs, double *es, int32_t *selfs, int32_t *counts,
                         int32_t *tallies, int32_t *status, void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (int r = check_rho_gamma(rho, gamma)) return r;
  if (max_iters < 0 || stop_tally < 0) return fail(FSE_ERR_CONFIG, "iterations must be >= 0");
  if (precision != FSE_PREC_F64 && precision != FSE_PREC_F32)
    return fail(FSE_ERR_UNSUPPORTED, "precision %d", precision);
  if (count <= 0) return FSE_OK;
  if (!signal || !labels || !recon || !status || !counts || !tallies ||
      (max_iters > 0 && (!us || !vs || !cs || !es || !selfs)))
    return fail(FSE_ERR_VALUE, "null pointer");
  const int chunk = 2048;
  for (int c0 = 0; c0 < count; c0 += chunk) {
    int n = std::min(chunk, count - c0);
    fse::GenArgs a{};
    a.count = n; a.M = M; a.N = N; a.iterations = max_iters; a.precision = precision;
    a.rho = rho; a.gamma = gamma; a.algorithm = 1; a.stop_tally = stop_tally;
    a.signal = signal + (size_t)c0 * M * N;
    a.labels = labels + (size_t)c0 * labels_stride;
    a.labels_stride = labels_stride;
    a.recon = recon + (size_t)c0 * M * N;
    a.model = model ? model + (size_t)c0 * 2 * M * N : nullptr;
    a.us = us ? us + (size_t)c0 * max_iters : nullptr;
    a.vs = vs ? vs + (size_t)c0 * max_iters : nullptr;
    a.cs = cs ? cs + (size_t)c0 * 2 * max_iters : nullptr;
    a.es = es ? es + (size_t)c0 * max_iters : nullptr;
    a.selfs = selfs ? selfs + (size_t)c0 * max_iters : nullptr;
    a.counts = counts + c0;
    a.tallies = tallies + c0;
    a.status = status + c0;
    size_t ws = fse::generic_workspace_bytes(n, M, N, precision);
    void *wsp = nullptr;
    if (ws) CK(cudaMallocAsync(&wsp, ws, S(stream)));
    cudaError_t e = fse::launch_generic_extrapolate(a, wsp, S(stream));
    if (wsp) cudaFreeAsync(wsp, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "extrapolate_rfse");
  }
  return FSE_OK;
}

int fse_select_basis_f64(int M, int N, const double *R, int64_t *uv, void *stream) {
  if (int r = check_dims(M, N)) return r;
  CK(fse::launch_select_basis_f64(M, N, R, uv, S(stream)));
  return FSE_OK;
}

int fse_update_residual_f64(int M, int N, double *R, const double *W, int u, int v, double c_re,
                            double c_im, void *stream) {
  if (int r = check_dims(M, N)) return r;
  CK(fse::launch_update_residual_f64(M, N, R, W, u, v, c_re, c_im, S(stream)));
  return FSE_OK;
}

// ------------------------------------------------------------- planner

int fse_plan_create(fse_plan **out, const int32_t *blocks, int n_blocks, int H, int W, int B,
                    int border, int F, double rho, double gamma, int iterations, int precision,
                    void *stream) {
  return fse_plan_create_ex(out, blocks, n_blocks, H, W, B, border, F, rho, gamma, iterations,
                            precision, FSE_ALG_CFSE, -1, stream);
}

int fse_plan_create_ex(fse_plan **out, const int32_t *blocks, int n_blocks, int H, int W, int B,
                       int border, int F, double rho, double gamma, int iterations, int precision,
                       int algorithm, int basis_target, void *stream) {
  if (!out) return fail(FSE_ERR_VALUE, "null plan pointer");
  if (algorithm != FSE_ALG_CFSE && algorithm != FSE_ALG_RFSE)
    return fail(FSE_ERR_CONFIG, "algorithm must be cfse (0) or rfse (1), got %d", algorithm);
  // basis_target (types.py:55-60, rfse.py:184-189): cFSE runs that many
  // iterations; rFSE stops once its basis-function tally reaches it
  if (basis_target >= 0) {
    if (algorithm == FSE_ALG_CFSE) iterations = basis_target;
  }
  *out = nullptr;
  if (int r = check_rho_gamma(rho, gamma)) return r;
  if (iterations < 0) return fail(FSE_ERR_CONFIG, "iterations must be >= 0, got %d", iterations);
  if (border < 0) return fail(FSE_ERR_CONFIG, "support_width must be >= 0, got %d", border);
  if (B < 1 || F < B || ((F - B) & 1))
    return fail(FSE_ERR_CONFIG, "need 1 <= B <= F and F - B even (B=%d, F=%d)", B, F);
  if (H < 1 || W < 1) return fail(FSE_ERR_CONFIG, "frame %dx%d", H, W);
  if (n_blocks < 0 || (n_blocks > 0 && !blocks)) return fail(FSE_ERR_VALUE, "bad block list");
  if (precision != FSE_PREC_F64 && precision != FSE_PREC_F32)
    return fail(FSE_ERR_UNSUPPORTED, "precision %d", precision);
  if (int r = check_dims(F, F)) return r;

  std::unique_ptr<fse_plan> p(new fse_plan());
  p->n_blocks = n_blocks; p->H = H; p->W = W; p->B = B; p->border = border; p->F = F;
  p->iterations = iterations; p->precision = precision; p->rho = rho; p->gamma = gamma;
  p->algorithm = algorithm;
  if (algorithm == FSE_ALG_RFSE) {
    if (basis_target >= 0) {
      p->iterations = iterations = basis_target;
      p->stop_tally = basis_target;
    } else {
      p->stop_tally = 2 * iterations + 1;  // fixed-count mode (unreachable tally)
    }
  }
  const int off = (F - B) / 2;

  // geometry classes: the clipped support rectangle (build_mask with
  // valid_rect = image, weighting.py:105-117) identifies the mask
  std::map<uint64_t, int> cls_of;
  std::vector<std::array<int, 4>> rects;
  std::vector<int32_t> bclass(n_blocks);
  for (int b = 0; b < n_blocks; ++b) {
    const int top = blocks[3 * b + 1], left = blocks[3 * b + 2];
    if (blocks[3 * b] < 0) return fail(FSE_ERR_VALUE, "block %d: negative frame index", b);
    p->max_frame = std::max(p->max_frame, (int)blocks[3 * b]);
    if (top < 0 || left < 0 || top + B > H || left + B > W)
      return fail(FSE_ERR_CONFIG,
                  "block %d: loss rectangle (%d, %d, %d, %d) extends outside the %dx%d image", b, top,
                  left, B, B, H, W);
    const int wt = top - off, wl = left - off;
    const int r0 = std::max({0, off - border, -wt}), r1 = std::min({F, off + B + border, H - wt});
    const int c0 = std::max({0, off - border, -wl}), c1 = std::min({F, off + B + border, W - wl});
    const uint64_t key = ((uint64_t)r0 << 48) | ((uint64_t)c0 << 32) | ((uint64_t)r1 << 16) | (uint64_t)c1;
    auto it = cls_of.find(key);
    int c;
    if (it == cls_of.end()) {
      c = (int)rects.size();
      cls_of.emplace(key, c);
      rects.push_back({r0, c0, r1, c1});
    } else {
      c = it->second;
    }
    bclass[b] = c;
    // TMA box start column (left - off + box_off) must be 16-byte aligned
    if ((left - off + std::max(0, off - border)) % 16 != 0) p->tma_aligned = false;
  }
  const int nc = (int)rects.size();
  p->n_classes = nc;
  std::vector<int8_t> labels((size_t)std::max(nc, 1) * F * F, 0);
  for (int c = 0; c < nc; ++c) {
    int8_t *L = labels.data() + (size_t)c * F * F;
    int nsup = 0;
    for (int m = rects[c][0]; m < rects[c][2]; ++m)
      for (int n = rects[c][1]; n < rects[c][3]; ++n) {
        const bool loss = m >= off && m < off + B && n >= off && n < off + B;
        L[m * F + n] = loss ? 2 : 1;
        nsup += !loss;
      }
    for (int m = off; m < off + B; ++m)
      for (int n = off; n < off + B; ++n) L[m * F + n] = 2;
    if (nsup == 0) return fail(FSE_ERR_CONFIG, "mask geometry leaves no support samples");
  }

  cudaStream_t st = S(stream);
  const size_t FF = (size_t)F * F;
  CK(p->alloc(&p->blocks, (size_t)n_blocks * 3));
  CK(p->alloc(&p->block_class, (size_t)n_blocks));
  CK(p->alloc(&p->labels, labels.size()));
  CK(p->alloc(&p->rects, (size_t)std::max(nc, 1) * 4));
  if (nc) CK(cudaMemcpyAsync(p->rects, rects.data(), (size_t)nc * 4 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CK(p->alloc(&p->wtab, (size_t)nc * FF));
  CK(p->alloc(&p->inv_w00, (size_t)nc));
  CK(p->alloc(&p->W64, (size_t)nc * FF * 2));
  CK(p->alloc(&p->w64, (size_t)nc * FF));
  CK(p->alloc(&p->w00, (size_t)nc));
  CK(p->alloc(&p->tmp, (size_t)nc * FF * 2));
  if (n_blocks) {
    CK(cudaMemcpyAsync(p->blocks, blocks, (size_t)n_blocks * 3 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p->block_class, bclass.data(), (size_t)n_blocks * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(p->labels, labels.data(), labels.size(), cudaMemcpyHostToDevice, st));

  // Centred frame (fast.cu): a class whose label map is mirror-symmetric in
  // both axes (every unclipped window) has real centred weight spectra; the
  // fused kernels then iterate on one real table value per bin (cFSE) or
  // per atom and bin (rFSE).  FSE_SYM=0 keeps every class on the complex W'
  // table.
  std::vector<int32_t> symc(std::max(nc, 1), 0);
  for (int c = 0; c < nc; ++c) {
    const int8_t *L = labels.data() + (size_t)c * F * F;
    bool ok = true;
    for (int m = 0; ok && m < F; ++m)
      for (int n = 0; ok && n < F; ++n)
        ok = L[m * F + n] == L[(F - 1 - m) * F + n] && L[m * F + n] == L[m * F + (F - 1 - n)];
    symc[c] = ok;
  }
  const char *sym_env = getenv("FSE_SYM");
  const bool sym_allowed = !(sym_env && atoi(sym_env) == 0);
  p->fast = precision == FSE_PREC_F32 &&
            fse::fast_config(F, iterations, sm_count(), &p->cfg, algorithm) &&
            B * B == 2 * (F * F / 32) && iterations > 0;
  // Small F = 64 cFSE plans are latency-bound (each block's 100 dependent
  // iterations, its warps alone on their SM sub-partitions): spread each
  // block over more warps while the plan still fits one wave of the build's
  // slots -- up to 2 blocks per SM the 8-warp build (fast_small.cu), up to
  // 3 the 4-warp build (fast_mid.cu; measured equal at 3.5, 2 % slower at
  // 3.5-5), beyond that the 2-warp throughput build.  All three give the
  // same tiles and traces bit for bit.  FSE_VARIANT=0/1/2 forces one.
  if (p->fast && F == 64 && algorithm == FSE_ALG_CFSE) {
    const int sm = sm_count();
    const char *venv = getenv("FSE_VARIANT");
    int v = venv ? atoi(venv) : n_blocks <= 2 * sm ? 2 : n_blocks <= 3 * sm ? 1 : 0;
    fse::FastConfig vc{};
    if (v == 2 && fse::s16::fast_config(F, iterations, sm, &vc, algorithm)) {
      p->variant = 2;
      p->cfg = vc;
    } else if (v == 1 && fse::s32::fast_config(F, iterations, sm, &vc, algorithm)) {
      p->variant = 1;
      p->cfg = vc;
    }
  }
  double *dmin_dev = nullptr;  // rfse.py:47-55 degeneracy check, every rFSE plan
  if (algorithm == FSE_ALG_RFSE) CK(p->alloc(&dmin_dev, (size_t)std::max(nc, 1)));
  if (p->fast) CK(p->alloc((char **)&p->table, (size_t)nc * p->cfg.table_bytes));
  if (p->fast && p->cfg.global_trace)
    CK(p->alloc(&p->trace_scratch, (size_t)p->cfg.grid * p->cfg.slots * 2 * iterations));

  std::vector<int32_t> sym(std::max(nc, 1), 0);
  for (int c = 0; c < nc; ++c) {
    sym[c] = p->fast && symc[c] && sym_allowed;
    p->n_sym += sym[c];
  }
  CK(p->alloc(&p->class_sym, (size_t)std::max(nc, 1)));
  CK(cudaMemcpyAsync(p->class_sym, sym.data(), (size_t)std::max(nc, 1) * sizeof(int32_t),
                     cudaMemcpyHostToDevice, st));
  fse::ClassSetupArgs ca{};
  ca.sym = p->class_sym;
  ca.n_classes = nc; ca.F = F; ca.rho = rho; ca.labels = p->labels; ca.W64 = p->W64;
  ca.w64 = p->w64; ca.wtab = p->wtab; ca.fast_table = p->fast ? p->table : nullptr;
  ca.fast_table_bytes = p->fast ? p->cfg.table_bytes : 0; ca.w00 = p->w00; ca.tmp = p->tmp;
  ca.rfse = p->fast && algorithm == FSE_ALG_RFSE; ca.dmin = dmin_dev;
  CK(p->variant == 2   ? fse::s16::launch_class_setup(ca, st)
     : p->variant == 1 ? fse::s32::launch_class_setup(ca, st)
                       : fse::launch_class_setup(ca, st));
  std::vector<double> w00(nc), dmin(nc, 1.0);
  if (nc) CK(cudaMemcpyAsync(w00.data(), p->w00, nc * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (nc && dmin_dev)
    CK(cudaMemcpyAsync(dmin.data(), dmin_dev, nc * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int c = 0; c < nc; ++c)
    if (dmin[c] <= 1e-9)  // rfse.py:50-55
      return fail(FSE_ERR_CONFIG,
                  "support area is degenerate for pairwise selection (conjugate atoms nearly "
                  "parallel under the weight)");
  std::vector<float> inv(nc);
  for (int c = 0; c < nc; ++c) {
    if (w00[c] <= 1e-12 * (double)F * F)  // cfse.py:47-48
      return fail(FSE_ERR_CONFIG, "total support weight is numerically zero (empty support)");
    inv[c] = (float)(1.0 / w00[c]);
  }
  if (nc) CK(cudaMemcpyAsync(p->inv_w00, inv.data(), nc * sizeof(float), cudaMemcpyHostToDevice, st));

  if (p->fast) {
    // rounds of `slots` same-class blocks, grouped by class.  A batch too
    // small to fill every slot of every SM is spread: the fewest blocks per
    // round (the other slots idle) whose rounds still fit one wave of
    // persistent CTAs, so the blocks share SMs less and finish sooner
    // (config 2, 256 blocks: 165 -> 108 us; FSE_SPREAD=0 packs full rounds).
    const int Sl = p->cfg.slots;
    std::vector<std::vector<int32_t>> by(nc);
    for (int b = 0; b < n_blocks; ++b) by[bclass[b]].push_back(b);
    int use = Sl;
    const char *spread_env = getenv("FSE_SPREAD");
    if (!spread_env || atoi(spread_env) != 0) {
      const int ctas = std::max(1, p->cfg.grid);
      for (int u = 1; u < Sl; ++u) {
        long r = 0;
        for (int c = 0; c < nc; ++c) r += ((long)by[c].size() + u - 1) / u;
        if (r <= ctas) {
          use = u;
          break;
        }
      }
    }
    std::vector<int32_t> rounds, rcls;
    for (int c = 0; c < nc; ++c) {
      const auto &v = by[c];
      for (size_t i = 0; i < v.size(); i += use) {
        for (int s = 0; s < Sl; ++s) rounds.push_back(s < use && i + s < v.size() ? v[i + s] : -1);
        rcls.push_back(c);
      }
    }
    p->n_rounds = (int)rcls.size();
    CK(p->alloc(&p->rounds, rounds.size()));
    CK(p->alloc(&p->round_class, rcls.size()));
    if (!rounds.empty()) {
      CK(cudaMemcpyAsync(p->rounds, rounds.data(), rounds.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(p->round_class, rcls.data(), rcls.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    }
  } else {
    // generic per-window path (fp64, or sizes the fused kernel does not cover)
    p->chunk = std::max(1, std::min(n_blocks, F <= 64 ? 2048 : 296));
    const size_t C = p->chunk, It = std::max(iterations, 1);
    CK(p->alloc(&p->us, C * It));
    CK(p->alloc(&p->vs, C * It));
    CK(p->alloc(&p->cs, C * It * 2));
    CK(p->alloc(&p->es, C * It));
    CK(p->alloc(&p->status, C));
    if (algorithm == FSE_ALG_RFSE) {
      CK(p->alloc(&p->selfs, C * It));
      CK(p->alloc(&p->counts, C));
      CK(p->alloc(&p->tallies, C));
    }
    size_t ws = fse::generic_workspace_bytes((int)C, F, F, precision);
    if (ws) CK(p->alloc((char **)&p->gen_ws, ws));
  }
  CK(cudaStreamSynchronize(st));
  *out = p.release();
  return FSE_OK;
}

int fse_plan_get_info(const fse_plan *p, fse_plan_info *info) {
  if (!p || !info) return fail(FSE_ERR_VALUE, "null pointer");
  info->n_blocks = p->n_blocks;
  info->n_classes = p->n_classes;
  info->n_rounds = p->n_rounds;
  info->slots = p->fast ? p->cfg.slots : 1;
  info->threads = p->fast ? p->cfg.threads : 512;
  info->grid = p->fast ? std::min(p->cfg.grid, p->n_rounds) : p->chunk;
  info->smem_bytes = p->fast ? p->cfg.smem_bytes : 0;
  info->fast_path = p->fast ? 1 : 0;
  info->n_centred = p->n_sym;
  return FSE_OK;
}

int fse_plan_destroy(fse_plan *p) {
  delete p;
  return FSE_OK;
}

int fse_plan_run(const fse_plan *p, const void *frames, int dtype, long long pitch,
                 long long frame_stride, int n_frames, void *tiles, int tile_dtype,
                 int32_t *trace_uv, void *trace_c, void *trace_e, void *stream) {
  if (!p) return fail(FSE_ERR_VALUE, "null plan");
  if (dtype < 0 || dtype > 2 || tile_dtype < 0 || tile_dtype > 2)
    return fail(FSE_ERR_UNSUPPORTED, "dtype %d / tile dtype %d", dtype, tile_dtype);
  if (p->n_blocks == 0) return FSE_OK;
  if (!frames || !tiles) return fail(FSE_ERR_VALUE, "null frames / tiles");
  if (pitch < p->W) return fail(FSE_ERR_VALUE, "pitch %lld < width %d", pitch, p->W);
  if (p->max_frame >= n_frames)
    return fail(FSE_ERR_VALUE, "block frame index %d >= n_frames %d", p->max_frame, n_frames);
  if (n_frames > 1 && frame_stride < (long long)p->H * pitch)
    return fail(FSE_ERR_VALUE, "frame stride %lld < H x pitch %lld", frame_stride,
                (long long)p->H * pitch);
  cudaStream_t st = S(stream);
  if (p->iterations == 0) {  // basis_target = 0: transforms only, loss = Re{0} = 0
    size_t bytes = (size_t)p->n_blocks * p->B * p->B * (tile_dtype == 0 ? 1 : tile_dtype == 1 ? 4 : 8);
    CK(cudaMemsetAsync(tiles, 0, bytes, st));
    return FSE_OK;
  }
  if (p->fast) {
    if (trace_uv && (!trace_c || !trace_e)) return fail(FSE_ERR_VALUE, "partial trace buffers");
    fse::FastArgs a{};
    a.F = p->F; a.B = p->B; a.border = p->border; a.iterations = p->iterations;
    a.gamma = (float)p->gamma; a.n_rounds = p->n_rounds; a.rounds = p->rounds;
    a.n_blocks = p->n_blocks; a.n_classes = p->n_classes;
    a.round_class = p->round_class; a.blocks = p->blocks; a.wtab = p->wtab; a.table = p->table;
    a.table_bytes = p->cfg.table_bytes; a.inv_w00 = p->inv_w00; a.support_rect = p->rects;
    a.class_sym = p->class_sym;
    a.frames = frames; a.dtype = dtype; a.pitch = pitch; a.frame_stride = frame_stride;
    a.H = p->H; a.W = p->W; a.tiles = tiles; a.tile_dtype = tile_dtype;
    a.trace_uv = trace_uv; a.trace_c = (float *)trace_c; a.trace_e = (float *)trace_e;
    a.trace_scratch = p->trace_scratch;
    a.algorithm = p->algorithm;
    a.stop_tally = p->stop_tally;
    // TMA staging of each block's support window (u8 frames, default for
    // F=64; FSE_TMA=0/1 forces it off/on): one 3-D tile load per block with OOB zero
    // fill, prefetched during the slot's previous block, so the setup starts
    // from shared memory (+1.0 % on config 5).  A tile load whose start
    // column is not 16-byte aligned faults (illegal instruction), so plans
    // with such boxes (e.g. 8x8 blocks on an 8-pixel grid) load directly.
    CUtensorMap tmap;
    a.use_tma = 0;
    const int off = (p->F - p->B) / 2;
    a.box_off = std::max(0, off - p->border);
    a.box_h = std::min(p->F, off + p->B + p->border) - a.box_off;
    a.box_w = (a.box_h + 15) & ~15;
    EncodeTiledFn enc = encode_tiled();
    const char *tma_env = getenv("FSE_TMA");
    const bool tma_default = p->F == 64;  // measured: +1.0 % at F=64, -1.5 % at F=128
    if (dtype == FSE_U8 && enc && p->tma_aligned &&
        (tma_env ? atoi(tma_env) == 1 : tma_default) &&
        (size_t)a.box_w * a.box_h <= fse::fast_stage_bytes(p->F) && a.box_w <= 256 &&
        a.box_h <= 256 && ((uintptr_t)frames % 16) == 0 && (pitch % 16) == 0 &&
        (frame_stride % 16) == 0 && n_frames >= 1) {
      cuuint64_t dims[3] = {(cuuint64_t)p->W, (cuuint64_t)p->H, (cuuint64_t)n_frames};
      cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)frame_stride};
      cuuint32_t box[3] = {(cuuint32_t)a.box_w, (cuuint32_t)a.box_h, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)frames, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        a.use_tma = 1;
    }
    const CUtensorMap *tm = a.use_tma ? &tmap : nullptr;
    CK(p->variant == 2   ? fse::s16::launch_fast(a, p->cfg, tm, st)
       : p->variant == 1 ? fse::s32::launch_fast(a, p->cfg, tm, st)
                         : fse::launch_fast(a, p->cfg, tm, st));
    return FSE_OK;
  }
  if (trace_uv && (!trace_c || !trace_e)) return fail(FSE_ERR_VALUE, "partial trace buffers");
  const int F = p->F, B = p->B;
  for (int c0 = 0; c0 < p->n_blocks; c0 += p->chunk) {
    const int n = std::min(p->chunk, p->n_blocks - c0);
    fse::GenArgs a{};
    a.count = n; a.M = F; a.N = F; a.iterations = p->iterations; a.precision = p->precision;
    a.algorithm = p->algorithm; a.stop_tally = p->algorithm ? p->stop_tally : 0;
    a.selfs = p->selfs; a.counts = p->counts; a.tallies = p->tallies;
    a.rho = p->rho; a.gamma = p->gamma; a.signal = nullptr; a.labels = p->labels;
    a.labels_stride = (long long)F * F; a.label_index = p->block_class + c0;
    a.wtab = p->w64;  // the class weights (class_setup_kernel, same formula)
    a.recon = nullptr; a.model = nullptr; a.us = p->us; a.vs = p->vs; a.cs = p->cs; a.es = p->es;
    const size_t esz = tile_dtype == 0 ? 1 : tile_dtype == 1 ? 4 : 8;
    // image mode: windows cut from the frames and tiles written by the kernel
    a.frames = frames; a.dtype = dtype; a.pitch = pitch; a.frame_stride = frame_stride;
    a.H = p->H; a.W = p->W; a.B = B; a.blocks = p->blocks + (size_t)3 * c0;
    a.tiles = (char *)tiles + (size_t)c0 * B * B * esz; a.tile_dtype = tile_dtype;
    a.status = p->status;
    CK(fse::launch_generic_extrapolate(a, p->gen_ws, st));
    if (trace_uv) {  // trace: f64 entries for fp64 plans, f32 otherwise
      const size_t It = (size_t)p->iterations, tsz = p->precision == FSE_PREC_F64 ? 8 : 4;
      CK(fse::launch_pack_trace(p->us, p->vs, p->cs, p->es, p->algorithm ? p->counts : nullptr, n,
                                p->iterations, trace_uv + (size_t)c0 * It * 2,
                                (char *)trace_c + (size_t)c0 * It * 2 * tsz,
                                (char *)trace_e + (size_t)c0 * It * tsz,
                                p->precision == FSE_PREC_F64, st));
    }
  }
  return FSE_OK;
}

// ------------------------------------------------ spatial self-check

int fse_spatial_extrapolate(int count, int M, int N, const double *signal, const int8_t *labels,
                            long long labels_stride, double rho, double gamma, int iterations,
                            int pair_mode, int basis_target, double *recon, int64_t *us,
                            int64_t *vs, double *cs, double *es, double *es_direct,
                            int32_t *selfs, int32_t *counts, int32_t *tallies, int32_t *status,
                            void *stream) {
  if (int r = check_dims(M, N)) return r;
  if (int r = check_rho_gamma(rho, gamma)) return r;
  if (M > 32 || N > 32)
    return fail(FSE_ERR_UNSUPPORTED, "spatial brute force is O(I M^2 N^2): M, N <= 32 (got %dx%d)", M, N);
  if (iterations < 0) return fail(FSE_ERR_CONFIG, "iterations must be >= 0");
  if (count <= 0) return FSE_OK;
  if (!signal || !labels || !recon || !status || !us || !vs || !cs || !es || !es_direct)
    return fail(FSE_ERR_VALUE, "null pointer");
  fse::SpatialArgs a{};
  a.count = count; a.M = M; a.N = N; a.pair_mode = pair_mode ? 1 : 0;
  a.iterations = pair_mode && basis_target >= 0 ? basis_target : iterations;
  a.stop_tally = pair_mode && basis_target >= 0 ? basis_target : 2 * iterations + 1;
  a.rho = rho; a.gamma = gamma; a.signal = signal; a.labels = labels; a.labels_stride = labels_stride;
  a.recon = recon; a.us = us; a.vs = vs; a.cs = cs; a.es = es; a.es_direct = es_direct;
  a.selfs = selfs; a.counts = counts; a.tallies = tallies; a.status = status;
  CK(fse::launch_spatial(a, S(stream)));
  return FSE_OK;
}

// --------------------------------------------------- loss pattern (host)

static inline uint64_t splitmix64(uint64_t &x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int fse_loss_pattern(int H, int W, int B, int count, uint64_t seed, int32_t *top_left) {
  if (H < 1 || W < 1 || B < 1) return fail(FSE_ERR_CONFIG, "bad geometry");
  if (count < 0 || (count > 0 && !top_left)) return fail(FSE_ERR_VALUE, "bad output");
  const int gh = H / B, gw = W / B;
  const int n = gh * gw;
  std::vector<int32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  uint64_t s = seed;
  for (int i = n - 1; i > 0; --i) {  // Fisher-Yates
    int j = (int)(splitmix64(s) % (uint64_t)(i + 1));
    std::swap(perm[i], perm[j]);
  }
  std::vector<uint8_t> taken(n, 0);
  int k = 0;
  for (int t = 0; t < n && k < count; ++t) {
    const int c = perm[t], gy = c / gw, gx = c % gw;
    bool ok = true;
    for (int dy = -1; dy <= 1 && ok; ++dy)
      for (int dx = -1; dx <= 1 && ok; ++dx) {
        int y = gy + dy, x = gx + dx;
        if (y >= 0 && y < gh && x >= 0 && x < gw && taken[y * gw + x]) ok = false;
      }
    if (!ok) continue;
    taken[c] = 1;
    top_left[2 * k] = gy * B;
    top_left[2 * k + 1] = gx * B;
    ++k;
  }
  // deterministic row-major output order
  std::vector<std::pair<int, int>> v(k);
  for (int i = 0; i < k; ++i) v[i] = {top_left[2 * i], top_left[2 * i + 1]};
  std::sort(v.begin(), v.end());
  for (int i = 0; i < k; ++i) { top_left[2 * i] = v[i].first; top_left[2 * i + 1] = v[i].second; }
  return k;
}

}  // extern "C"

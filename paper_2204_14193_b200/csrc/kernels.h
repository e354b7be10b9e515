// kernels.h -- host-side launchers implemented in the .cu files and used by
// the C-ABI layer (api.cpp).  Internal; not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fse {

// ---------------------------------------------------------------- generic
struct GenArgs {
  int count, M, N, iterations, precision;  // precision: 0 f64, 1 f32
  double rho, gamma;
  const double *signal;
  const int8_t *labels;
  long long labels_stride;
  const int32_t *label_index;  // optional: window i uses labels + label_index[i]*labels_stride
  const double *wtab;          // optional (with label_index): per-class weights w, labels_stride apart
  // image mode (plans): frames != null -- window i is cut from the frames
  // around blocks[3 i..] (frame, top, left) instead of read from `signal`,
  // and the B x B loss tile goes straight to `tiles` (tile_dtype) instead of
  // `recon`
  const void *frames;
  int dtype, H, W, B, tile_dtype;
  long long pitch, frame_stride;
  const int32_t *blocks;
  void *tiles;
  double *recon, *model;
  int64_t *us, *vs;
  double *cs, *es;
  int32_t *status;
  // rFSE only (algorithm = 1): pair-selection trace and stopping rule
  int algorithm;        // 0 cfse, 1 rfse
  int stop_tally;       // rfse: stop when the basis-function tally reaches it
  int32_t *selfs;       // rfse: self-conjugate flag per iteration (count x iterations)
  int32_t *counts;      // rfse: executed iterations per window
  int32_t *tallies;     // rfse: basis-function tally per window
};
// Size of the global workspace the generic extrapolation needs for `count`
// windows (0 when everything fits in shared memory).
size_t generic_workspace_bytes(int count, int M, int N, int precision);
cudaError_t launch_generic_extrapolate(const GenArgs &a, void *workspace, cudaStream_t s);

cudaError_t launch_cfse_kernel_f64(int count, int M, int N, double *R, const double *W,
                                   long long w_stride, double gamma, const double *inv_w00,
                                   int iterations, const double *e0, double *G, int64_t *us,
                                   int64_t *vs, double *cs, double *es, cudaStream_t s);

cudaError_t launch_dft2_f64(int count, int M, int N, const double *in, double *out, int inverse,
                            double *tmp, cudaStream_t s);
cudaError_t launch_build_weight_f64(int count, int M, int N, const int8_t *labels, double rho,
                                    double *w, cudaStream_t s);
cudaError_t launch_select_basis_f64(int M, int N, const double *R, int64_t *uv, cudaStream_t s);
cudaError_t launch_update_residual_f64(int M, int N, double *R, const double *W, int u, int v,
                                       double cr, double ci, cudaStream_t s);

// ------------------------------------------------------------ class setup
// Per geometry class: w (fp64) from labels, W = DFT(w) in fp64, exact
// Hermitian symmetrisation, and the fast kernel's table layouts.
struct ClassSetupArgs {
  int n_classes, F;
  double rho;
  const int8_t *labels;   // n_classes x F x F
  double *W64;            // n_classes x F x F c128 (symmetrised spectrum)
  double *w64;            // n_classes x F x F (weights)
  float *wtab;            // n_classes x F x F (weights, fp32)
  void *fast_table;       // n_classes x fast_table_bytes(F) (may be null)
  size_t fast_table_bytes;
  double *w00;            // n_classes
  double *tmp;            // n_classes x F x F c128 scratch
  int rfse;               // also build the fused rFSE pair tables (F = 64)
  double *dmin;           // n_classes: min over pair bins of D / W00^2 (rfse only)
  const int32_t *sym;     // n_classes (may be null): 1 = mirror-symmetric weights, build the
                          // real centred table Q (fast.cu, "centred frame") instead of W'
};
cudaError_t launch_class_setup(const ClassSetupArgs &a, cudaStream_t s);

// ------------------------------------------------------------------ fast
// Fused register-resident fp32 kernel for F in {32, 64, 128}.
struct FastArgs {
  int F, B, border, iterations;
  float gamma;
  int n_rounds, n_blocks, n_classes;
  const int32_t *rounds;       // n_rounds x slots block ids (-1 = idle)
  const int32_t *round_class;  // n_rounds
  const int32_t *blocks;       // n_blocks x 3 (frame, top, left)
  const float *wtab;           // n_classes x F x F
  const void *table;           // n_classes x table_bytes
  size_t table_bytes;
  const float *inv_w00;        // n_classes
  const int32_t *support_rect; // n_classes x 4 (r0, c0, r1, c1) window coords
  const int32_t *class_sym;    // n_classes (may be null): 1 = the class table is the real centred Q
  const void *frames;
  int dtype;
  long long pitch, frame_stride;
  int H, W;
  void *tiles;
  int tile_dtype;
  int32_t *trace_uv;
  float *trace_c, *trace_e;
  float4 *trace_scratch;  // grid x slots x iterations, when the trace exceeds shared memory
  // TMA staging of the support window (u8 frames): box_w x box_h bytes at
  // window offset (box_off, box_off); 0 = direct loads
  int use_tma, box_w, box_h, box_off;
  int algorithm;   // 0 = cFSE, 1 = rFSE (F = 64)
  int stop_tally;  // rFSE: stop a block once its basis-function tally reaches this
};
struct FastConfig {
  int slots, threads, smem_bytes, grid;
  size_t table_bytes;
  bool global_trace;  // iteration trace kept in global scratch (large I)
};
// Returns false when F is not supported by the fused kernel.
bool fast_config(int F, int iterations, int sm_count, FastConfig *cfg, int algorithm = 0);
cudaError_t launch_fast(const FastArgs &a, const FastConfig &cfg, const CUtensorMap *tmap,
                        cudaStream_t s);
// staging capacity (bytes per slot) of the TMA window for window size F
size_t fast_stage_bytes(int F);
// latency builds of the fused kernel for small F = 64 cFSE plans
// (fast_small.cu: 16 bins per thread; fast_mid.cu: 32 bins per thread)
namespace s16 {
bool fast_config(int F, int iterations, int sm_count, FastConfig *cfg, int algorithm = 0);
cudaError_t launch_fast(const FastArgs &a, const FastConfig &cfg, const CUtensorMap *tmap, cudaStream_t s);
cudaError_t launch_class_setup(const ClassSetupArgs &a, cudaStream_t s);
}  // namespace s16
namespace s32 {
bool fast_config(int F, int iterations, int sm_count, FastConfig *cfg, int algorithm = 0);
cudaError_t launch_fast(const FastArgs &a, const FastConfig &cfg, const CUtensorMap *tmap, cudaStream_t s);
cudaError_t launch_class_setup(const ClassSetupArgs &a, cudaStream_t s);
}  // namespace s32

// ------------------------------------------------------------- image f64
// Pack the per-window trace (us, vs int64; cs re/im f64; es f64; `counts`
// executed iterations per window or null = all) into the plan trace layout:
// uv int32 (n, It, 2), c (n, It, 2) and e (n, It) as f64 (c64 != 0) or f32;
// iterations past a window's count get uv = -1, c = e = 0.
cudaError_t launch_pack_trace(const int64_t *us, const int64_t *vs, const double *cs,
                              const double *es, const int32_t *counts, int n, int It,
                              int32_t *uv, void *c, void *e, int c64, cudaStream_t s);

// ------------------------------------------------------------- spatial
// Spatial-domain brute-force matching pursuit (spatial.cu): the package's
// independent self-check.  M, N <= 32.
struct SpatialArgs {
  int count, M, N, iterations, pair_mode, stop_tally;
  double rho, gamma;
  const double *signal;   // count x M x N
  const int8_t *labels;   // labels_stride apart
  long long labels_stride;
  double *recon;          // count x M x N
  int64_t *us, *vs;       // count x iterations
  double *cs, *es, *es_direct;
  int32_t *selfs, *counts, *tallies, *status;  // selfs / counts / tallies optional
};
size_t spatial_smem_bytes(int M, int N);
cudaError_t launch_spatial(const SpatialArgs &a, cudaStream_t s);

}  // namespace fse

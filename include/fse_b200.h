/*
 * fse_b200.h -- C ABI of the B200-native cFSE library (libfse_b200.so).
 *
 * The reference (`fse`, /root/reference/pkg/src/fse) is a pure-Python
 * package whose only native boundary is the numba kernel `_cfse_kernel`
 * (cfse.py:55-56) plus numpy's pocketfft (spectral.py:46,56).  This ABI
 * replaces exactly those calls (and the spec'd-but-absent image harness)
 * with sm_100a CUDA.  Plain C types only: device pointers are `void*`-like
 * typed pointers allocated and owned by the caller (torch tensors or
 * cudaMalloc); `stream` is a cudaStream_t passed as void*.  No exception
 * crosses the ABI: every entry point returns FSE_OK (0) or a negative code
 * and records a message retrievable with fse_last_error().
 *
 * Error codes mirror the reference's exception convention (errors.py:4-10):
 *   FSE_ERR_CONFIG       -> ConfigError (range / geometry / empty support)
 *   FSE_ERR_VALUE        -> ValueError  (non-finite input, bad pointer)
 *   FSE_ERR_UNSUPPORTED  -> size/dtype outside what the kernels implement
 *   FSE_ERR_CUDA         -> CUDA runtime failure
 *
 * All entry points are reentrant; launches are asynchronous on `stream`
 * unless stated.  A plan owns device scratch (generic-path windows, the
 * fused path's global trace for large I), so one plan serves one run at a
 * time: runs of the same plan on different streams must be ordered by the
 * caller; distinct plans are independent.  Multi-GPU = one call per device (the caller sets the
 * current device), no collective is involved.
 */
#ifndef FSE_B200_H
#define FSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSE_OK 0
#define FSE_ERR_CONFIG (-1)
#define FSE_ERR_VALUE (-2)
#define FSE_ERR_UNSUPPORTED (-3)
#define FSE_ERR_CUDA (-4)

/* pixel / sample types */
#define FSE_U8 0
#define FSE_F32 1
#define FSE_F64 2

/* arithmetic precision of the extrapolation */
#define FSE_PREC_F64 0
#define FSE_PREC_F32 1

/* extrapolation variant of an image-level plan */
#define FSE_ALG_CFSE 0 /* complex-valued FSE, cfse.py */
#define FSE_ALG_RFSE 1 /* conjugate-pair (real-valued) FSE, rfse.py */

/* per-window status written by fse_extrapolate (device int32) */
#define FSE_STATUS_OK 0
#define FSE_STATUS_EMPTY_SUPPORT 1 /* w00 <= 1e-12*M*N, cfse.py:47-48 */
#define FSE_STATUS_DEGENERATE_PAIRS 2 /* rFSE pair Gram singular, rfse.py:50-54 */

/* Library version string and last error message (thread-local). */
const char *fse_version(void);
int fse_last_error(char *buf, size_t len);

/* ------------------------------------------------------------------ */
/* Spectral engine: replaces spectral.py:32-56 (np.fft.fft2 / ifft2).  */
/* Batched over `count` M x N grids; complex128 interleaved, device.    */
/* inverse=0: unnormalised forward (-j kernel); inverse=1: +j, 1/(MN).  */
/* Any M, N in [1, 4096].                                               */
int fse_dft2_f64(int count, int M, int N, const double *in, double *out, int inverse,
                 void *stream);

/* Weighting function: replaces weighting.py:130-145 (build_weight).
 * labels: int8 count x M x N (Area: 0 padding, 1 support, 2 loss);
 * w: float64 count x M x N.  rho in (0,1) is validated by the caller. */
int fse_build_weight_f64(int count, int M, int N, const int8_t *labels, double rho, double *w,
                         void *stream);

/* ------------------------------------------------------------------ */
/* Drop-in for the numba loop `_cfse_kernel(R_w, W, gamma, inv_w00,     */
/* iterations, e0)` (cfse.py:55-107), batched over `count` windows, fp64. */
/* R_w (c128 count x M x N) is mutated in place like the reference.     */
/* W: c128, window i uses W + i*w_stride*2 doubles (w_stride = 0 shares  */
/* one spectrum).  inv_w00, e0: device float64[count].  Outputs (device,  */
/* G nullable): G c128 count x M x N; us, vs int64 count x iterations;   */
/* cs c128 count x iterations; es f64 count x iterations.  The loop uses  */
/* the reference's unfused IEEE operation order, so identical inputs give */
/* bit-identical outputs.                                                 */
int fse_cfse_kernel_f64(int count, int M, int N, double *R_w, const double *W,
                        long long w_stride, double gamma, const double *inv_w00,
                        int iterations, const double *e0, double *G, int64_t *us, int64_t *vs,
                        double *cs, double *es, void *stream);

/* ------------------------------------------------------------------ */
/* Drop-in for `extrapolate_cfse(signal, mask, config)` (cfse.py:110-142) */
/* fused on device: weights -> two DFTs -> I iterations -> sparse        */
/* synthesis -> write-back, one CTA per window, batched over `count`.    */
/*   signal: f64 count x M x N (device); labels: int8, window i uses     */
/*           labels + i*labels_stride (0 = one shared mask)              */
/*   recon:  f64 count x M x N: input on support/padding (bit-identical), */
/*           Re{g} on loss (unclamped)                                    */
/*   model:  c128 count x M x N or NULL (g = idft2(G), cfse.py:126)      */
/*   us/vs/cs/es: trace, count x iterations (device, required)           */
/*   status: int32[count] (FSE_STATUS_*), device                          */
/* precision FSE_PREC_F64 reproduces the reference arithmetic; FSE_PREC_F32 */
/* runs the same algorithm in fp32 (inputs/outputs stay f64).             */
int fse_extrapolate(int count, int M, int N, int precision, const double *signal,
                    const int8_t *labels, long long labels_stride, double rho, double gamma,
                    int iterations, double *recon, double *model, int64_t *us, int64_t *vs,
                    double *cs, double *es, int32_t *status, void *stream);

/* Drop-in for `extrapolate_rfse(signal, mask, config)` (rfse.py:170-210),  */
/* the paper's real-valued conjugate-pair variant: per iteration the joint  */
/* projection of every bin onto {phi, conj(phi)} (per-bin 2x2 Gram solve,   */
/* self-conjugate bins as one real atom), canonical pair member, two-term   */
/* residual update.  max_iters / stop_tally follow rfse.py:182-187          */
/* (fixed count: max_iters = I, stop_tally = 2I+1; basis_target T: both T). */
/* Trace arrays hold max_iters entries; counts/tallies (int32[count]) give  */
/* the executed iterations and the basis-function tally; selfs marks        */
/* self-conjugate selections.  Same layout/ownership as fse_extrapolate.    */
int fse_extrapolate_rfse(int count, int M, int N, int precision, const double *signal,
                         const int8_t *labels, long long labels_stride, double rho, double gamma,
                         int max_iters, int stop_tally, double *recon, double *model, int64_t *us,
                         int64_t *vs, double *cs, double *es, int32_t *selfs, int32_t *counts,
                         int32_t *tallies, int32_t *status, void *stream);

/* Single-step ops of cfse.py:145-178 on device (SPEC test surface).       */
/* select_basis: argmax |R|^2, first max in row-major order -> uv[0..1].   */
int fse_select_basis_f64(int M, int N, const double *R, int64_t *uv, void *stream);
/* update_residual: R[k,l] -= c * W[(k-u) mod M, (l-v) mod N].             */
int fse_update_residual_f64(int M, int N, double *R, const double *W, int u, int v, double c_re,
                            double c_im, void *stream);

/* ------------------------------------------------------------------ */
/* Image-level concealment (the north-star entry "image + loss mask +    */
/* block size, border width, FFT size, iterations, rho, gamma"; semantics */
/* of the spec'd harness `conceal`): for every lost      */
/* B x B block (frame, top, left) an F x F window centred on it, support  */
/* ring `border` wide clipped to the image (valid_rect), I iterations,    */
/* Re{g} of the loss pixels written to a tile.                            */
/*                                                                        */
/* A plan holds the host-side schedule (geometry classes, rounds) and the */
/* per-class weight spectra on the device; it is reusable across frames   */
/* with the same loss pattern.                                            */
typedef struct fse_plan fse_plan;

typedef struct {
  int n_blocks;
  int n_classes;   /* distinct clipped-support geometries                */
  int n_rounds;    /* work items of `slots` same-class blocks            */
  int slots;       /* lost blocks resident per CTA                       */
  int threads;     /* threads per CTA                                    */
  int grid;        /* CTAs launched (persistent)                         */
  int smem_bytes;  /* dynamic shared memory per CTA                      */
  int fast_path;   /* 1 = fused register-resident fp32 kernel            */
  int n_centred;   /* classes iterated in the centred frame (mirror-      */
                   /* symmetric weights: one real table value per bin)    */
} fse_plan_info;

/* blocks: HOST int32 n x 3 (frame, top, left).  F in {32, 64, 128} for the
 * fused fp32 kernel (precision FSE_PREC_F32); any F with (F-B) even for
 * FSE_PREC_F64 (generic kernel).  Synchronous (builds tables on `stream`
 * and waits).  Errors: FSE_ERR_CONFIG for geometry (loss block outside the
 * image, empty support) or parameter range. */
int fse_plan_create(fse_plan **plan, const int32_t *blocks, int n_blocks, int H, int W, int B,
                    int border, int F, double rho, double gamma, int iterations, int precision,
                    void *stream);
/* As fse_plan_create, with the variant (FSE_ALG_CFSE / FSE_ALG_RFSE) and an
 * optional basis_target (>= 0; -1 = none): cFSE runs basis_target
 * iterations, rFSE stops each block once its basis-function tally (2 per
 * pair pick, 1 per self-conjugate pick) reaches it, with at most
 * basis_target iterations (types.py:55-60, rfse.py:184-189).  The fused fp32
 * kernel serves rFSE at F = 32, 64 and 128; other sizes and fp64 use the generic
 * kernel.
 * Errors additionally: FSE_ERR_CONFIG for a support degenerate for pairwise
 * selection (rfse.py:50-55). */
int fse_plan_create_ex(fse_plan **plan, const int32_t *blocks, int n_blocks, int H, int W, int B,
                       int border, int F, double rho, double gamma, int iterations, int precision,
                       int algorithm, int basis_target, void *stream);
int fse_plan_get_info(const fse_plan *plan, fse_plan_info *info);
int fse_plan_destroy(fse_plan *plan);

/* Run a plan.  frames: device, dtype FSE_U8/F32/F64, frame f row y starts
 * at frames + f*frame_stride + y*pitch (elements).  tiles: device memory or
 * page-locked host memory (unified addressing: the kernel stores each tile
 * straight into host memory), n_blocks x B x B of tile_dtype (FSE_U8:
 * clamp [0,255] + round-half-even;
 * FSE_F32 / FSE_F64: unclamped Re{g}).  trace_uv (int32 n x I x 2),
 * trace_c (float32/64 n x I x 2 per precision), trace_e (float32/64 n x I):
 * optional (NULL).  Asynchronous on `stream`. */
int fse_plan_run(const fse_plan *plan, const void *frames, int dtype, long long pitch,
                 long long frame_stride, int n_frames, void *tiles, int tile_dtype,
                 int32_t *trace_uv, void *trace_c, void *trace_e, void *stream);

/* Spatial-domain brute-force matching pursuit (no FFT): the independent
 * equivalence check of `fse selfcheck` (the spec's
 * `oracle` module, which the reference package does not ship).  Every
 * iteration projects the spatial residual onto every atom by direct
 * summation (Eq. 9), selects by Eq. (10) with the row-major first-max rule,
 * updates model and residual in the spatial domain (Eqs. 13, 14, 17).
 * pair_mode = 1: the rFSE pair rule (rfse.py:37-167), basis_target as in
 * fse_extrapolate_rfse.  M, N <= 32.  Device arrays: signal, labels (int8,
 * labels_stride apart), recon (count x M x N), us / vs / cs (c128) / es /
 * es_direct (the directly evaluated weighted residual energy) of count x
 * iterations (x basis_target in pair mode), selfs / counts / tallies
 * (int32, optional), status (int32: 0, 1 empty support, 2 degenerate pairs). */
int fse_spatial_extrapolate(int count, int M, int N, const double *signal, const int8_t *labels,
                            long long labels_stride, double rho, double gamma, int iterations,
                            int pair_mode, int basis_target, double *recon, int64_t *us,
                            int64_t *vs, double *cs, double *es, double *es_direct,
                            int32_t *selfs, int32_t *counts, int32_t *tallies, int32_t *status,
                            void *stream);

/* Seeded isolated-loss pattern: random-sequential
 * selection on the B x B block grid of an H x W frame, rejecting blocks
 * 8-adjacent to an already chosen one, until `count` blocks are chosen or
 * the grid is exhausted.  Host only.  Writes (top, left) pairs; returns the
 * number written (>= 0) or a negative error. */
int fse_loss_pattern(int H, int W, int B, int count, uint64_t seed, int32_t *top_left);

#ifdef __cplusplus
}
#endif
#endif /* FSE_B200_H */

/*
 * tensorsel_b200.h — C ABI of the B200-native execution path for the
 * convolution family of tensorsel (arXiv 2512.02371, "HardBoiled").
 *
 * The reference (/root/reference/pkg/src/tensorsel) is pure Python; every
 * entry point below replaces a Python function on its hot path.  The Python
 * package `paper_2512_02371_b200` binds these with ctypes (see INTEGRATION.md
 * for the binding a tensorsel maintainer would add).
 *
 * Conventions
 *   - Every call returns a ts_status; ts_last_error() returns a thread-local
 *     message for the last non-OK status on the calling thread.
 *   - Device pointers are caller-owned (torch tensors / cudaMalloc); all
 *     kernels are enqueued on the caller's stream (a cudaStream_t passed as
 *     void*, NULL = legacy default stream) and never synchronise it.
 *   - Images are planar with row / plane strides in elements that are
 *     multiples of 16 bytes (TMA).  Output rows are written in whole 16-byte
 *     units: the bytes from the last column to the next 16-byte boundary of
 *     a row may be overwritten (they belong to the row's stride); nothing
 *     beyond them is touched (tests/test_gpu_guards.py).
 *   - Status codes map 1:1 onto the reference exception classes:
 *       TS_ERR_OUT_OF_BOUNDS      -> interp.OutOfBounds / layout.OutOfBounds
 *       TS_ERR_PHASE_MISMATCH     -> layout.PhaseMismatch        (layout.py:24)
 *       TS_ERR_SHAPE_UNREGISTERED -> interp.ShapeUnregistered     (interp.py:50)
 *       TS_ERR_UNKNOWN_INTRINSIC  -> interp.UnknownIntrinsic      (interp.py:46)
 *       TS_ERR_INVALID            -> interp.EvalError             (interp.py:32)
 */
#ifndef TENSORSEL_B200_H
#define TENSORSEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 2

#if defined(__GNUC__)
#define TS_API __attribute__((visibility("default")))
#else
#define TS_API
#endif

typedef enum ts_status {
  TS_OK = 0,
  TS_ERR_INVALID = 1,
  TS_ERR_OUT_OF_BOUNDS = 2,
  TS_ERR_PHASE_MISMATCH = 3,
  TS_ERR_SHAPE_UNREGISTERED = 4,
  TS_ERR_UNKNOWN_INTRINSIC = 5,
  TS_ERR_UNSUPPORTED = 6, /* geometry the sm_100a kernels cannot tile        */
  TS_ERR_CUDA = 7,        /* CUDA runtime / driver error (message has detail) */
  TS_ERR_NO_DEVICE = 8    /* no sm_100 device visible                         */
} ts_status;

typedef enum ts_dtype { TS_BF16 = 1, TS_F32 = 2, TS_F16 = 3 } ts_dtype;

/* Axis-builder flags */
#define TS_AXIS_DC_EXACT 0x1 /* re-balance bf16-rounded taps so every output's taps keep their f32 sum */

/* Opaque handle: one axis of a separable linear transform, i.e. a banded
 * (n_out x n_in) resampling/filter matrix with clamp-to-edge folded in,
 * stored on the device as 16-output blocks: a window start per block and a
 * deduplicated set of bf16 B-operand tiles already in the tcgen05
 * shared-memory layout.  Built once per (scale, kernel, size) — the
 * analogue of the reference's hoisted ExprVar weight matrix
 * (selector.py:309-399, interp.py:214-219). */
typedef struct ts_axis ts_axis;

typedef struct ts_axis_info {
  int n_in, n_out;
  int taps;        /* max taps per output before folding                  */
  int window;      /* K: input window per 16-output block (multiple of 16) */
  int blocks;      /* number of 16-output blocks                           */
  int unique_tiles;/* distinct B tiles after dedup (incl. the zero tile)   */
  int row_span;    /* input rows one 128-output-row tile reads (pass 1)    */
  int col_blocks;  /* 16-output blocks per 128-input-column tile (pass 2)  */
  int col_span;    /* input columns those blocks read (<= 128)             */
} ts_axis_info;

TS_API const char* ts_last_error(void);
TS_API int ts_abi_version(void);
/* number of visible devices with compute capability 10.x; 0 if none */
TS_API int ts_device_count(void);

/* ---------------------------------------------------------------- builder */

/* General banded axis: output o reads inputs first[o] + t, t < taps, with
 * weights[o * taps + t]; indices outside [0, n_in) are clamped to the edge
 * (their weight is folded onto the edge sample).
 * Replaces layout.matrix_for (layout.py:72-84) + the clamp policy. */
TS_API ts_status ts_axis_create(int n_in, int n_out, int taps, const int32_t* first,
                         const float* weights, int flags, int device, ts_axis** out);

/* Axis from a reference ToeplitzSpec (layout.py:32-51): l taps per phase,
 * stride s (downsample) or p phases (upsample), first tap at input
 * offset + s*o (p == 1) or offset + o/p (p > 1).  kernel has kernel_len =
 * p*l entries; TS_ERR_PHASE_MISMATCH otherwise (layout.py:99-102).
 * Replaces layout.strided_toeplitz / polyphase_toeplitz (layout.py:87-103). */
TS_API ts_status ts_axis_from_toeplitz(int l, int s, int p, int offset, const float* kernel,
                                int kernel_len, int n_in, int n_out, int flags, int device,
                                ts_axis** out);

TS_API ts_status ts_axis_get_info(const ts_axis* a, ts_axis_info* info);

/* Dense (n_out x n_in, row-major, host f32) copy of the effective weights the
 * device uses (bf16-rounded, edge-folded).  For tests and diagnostics. */
TS_API ts_status ts_axis_dense(const ts_axis* a, float* out_host);

TS_API void ts_axis_destroy(ts_axis* a);

/* ----------------------------------------------------------- executors */

/* Output epilogue, applied inside the producing kernel to every f32 result
 * before its final cast (the "clamp / normalise" step of an image pipeline):
 *   y = min(max(x * scale + bias, lo), hi)      (NaN propagates)
 * The *_ep entry points take it; NULL (or the plain entry points) means none. */
typedef struct ts_epilogue {
  float scale, bias, lo, hi;
} ts_epilogue;

/* Fused separable transform  out[p] = R · in[p] · Cᵀ  for `planes` planes:
 * one sm_100a kernel (TMA-staged halo tiles -> tcgen05 vertical pass ->
 * TMEM -> smem -> tcgen05 horizontal pass -> TMEM -> cast -> TMA store).
 * in: bf16, out: bf16 or f32.  Strides are in elements; the row stride must
 * be a multiple of 8 (bf16) / 4 (f32) elements and the plane stride a
 * multiple of the row stride.  rows->n_in = input height,
 * cols->n_in = input width. */
TS_API ts_status ts_separable_run(const ts_axis* rows, const ts_axis* cols, int planes, const void* in,
                           int64_t in_row_stride, int64_t in_plane_stride, int in_dtype, void* out,
                           int64_t out_row_stride, int64_t out_plane_stride, int out_dtype,
                           void* stream);

/* ts_separable_run with an output epilogue (see ts_epilogue). */
TS_API ts_status ts_separable_run_ep(const ts_axis* rows, const ts_axis* cols, int planes,
                                     const void* in, int64_t in_row_stride,
                                     int64_t in_plane_stride, int in_dtype, void* out,
                                     int64_t out_row_stride, int64_t out_plane_stride,
                                     int out_dtype, const ts_epilogue* ep, void* stream);

/* One banded axis along rows (dim = 0: out is a->n_out x width) or columns
 * (dim = 1: out is height x a->n_out) of `planes` bf16 planes; out bf16 or
 * f32.  Any window up to 1024 inputs per 16 outputs (the K window streams
 * through a TMA ring).  ts_separable_run reports TS_ERR_UNSUPPORTED for
 * axes whose windows do not fit its fused tile (large downscale factors,
 * very wide filters); those run as two axis passes with a bf16
 * intermediate, the rounding point of the fused kernel's intermediate.
 * Replaces, for such geometries, the per-tile loop of interp.run_program
 * (interp.py:570-619) like ts_separable_run does. */
TS_API ts_status ts_axis_pass(const ts_axis* a, int dim, int planes, int height, int width,
                              const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                              void* out, int64_t out_row_stride, int64_t out_plane_stride,
                              int out_dtype, void* stream);

/* ts_axis_pass with an output epilogue (for the last pass of a pipeline). */
TS_API ts_status ts_axis_pass_ep(const ts_axis* a, int dim, int planes, int height, int width,
                                 const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                                 void* out, int64_t out_row_stride, int64_t out_plane_stride,
                                 int out_dtype, const ts_epilogue* ep, void* stream);

/* Launch geometry ts_separable_run would use for these axes:
 * out8 = {stages, V buffers, weights resident (0/1), smem bytes, staged rows
 * per tile, column blocks per tile, tiles, grid CTAs}. */
TS_API ts_status ts_separable_plan(const ts_axis* rows, const ts_axis* cols, int planes,
                                   int out_dtype, int* out8);

/* Fused DCT-16 transform-domain denoise: 16x16 tiles at
 * stride 8, sine window folded into the DCT-II matrices, coring of every
 * non-DC coefficient (soft = 0: |c| < threshold -> 0; soft = 1: shrink by
 * threshold), windowed inverse, overlap-add; clamp-to-edge outside the
 * image.  in: bf16 planes (height x width, both multiples of 8); out: bf16
 * or f32.  One sm_100a kernel (tcgen05, TMEM-resident coefficients). */
TS_API ts_status ts_denoise_dct16(const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                                  int in_dtype, void* out, int64_t out_row_stride,
                                  int64_t out_plane_stride, int out_dtype, int planes, int height,
                                  int width, float threshold, int soft, void* stream);

/* ts_denoise_dct16 with an output epilogue. */
TS_API ts_status ts_denoise_dct16_ep(const void* in, int64_t in_row_stride,
                                     int64_t in_plane_stride, int in_dtype, void* out,
                                     int64_t out_row_stride, int64_t out_plane_stride,
                                     int out_dtype, int planes, int height, int width,
                                     float threshold, int soft, const ts_epilogue* ep,
                                     void* stream);

/* One lowered convolution statement group of a tensorsel program, batched
 * over `instances` program instances (e.g. a difftest's seeds):
 *   acc = zero_init ? 0 : acc
 *   for v < iterations:
 *     acc = wmma_mma(wmma_load_a(src, a_base[v], a_stride, m, k),
 *                    wmma_load_b(B_v, 0, n, k, n), acc)
 *   B_v[kk][j] = b_off[kk*n + j] < 0 ? 0 : kern[k_base[v] + b_off[kk*n + j]]
 * evaluated with interp.py's exact semantics (interp.py:427-486): loaded
 * values re-rounded to their kind (0 f32, 1 f16, 2 bf16), f32 products,
 * k summed left to right, then acc + s — bit-identical to the reference.
 * Buffers are f32 carriers (device), instance t at base + t*stride.
 * *error (device) is set to 1 + index (src) or -(1 + index) (kern) on an
 * out-of-bounds read (interp.OutOfBounds). */
typedef struct ts_conv_group {
  int instances;
  const float* src;
  int64_t src_stride;
  int src_len, src_kind;
  const float* kern;
  int64_t kern_stride;
  int kern_len, kern_kind;
  float* acc;
  int64_t acc_stride;
  int zero_init;
  int m, k, n, a_stride;
  int iterations;
  const int32_t* a_base;
  const int32_t* k_base;
  const int32_t* b_off;
  /* Optional explicit gathers (source-form statements, interp.py:174-212):
   * when non-NULL, a_idx/b_idx ([iterations][m*n][k], device) give the src
   * and kern index of every (output, tap) product (b_idx -1 = zero) and
   * override a_base/a_stride/k_base/b_off. */
  const int32_t* a_idx;
  const int32_t* b_idx;
  /* device int32[3], zeroed by the caller: on an out-of-bounds read the
   * first failing thread writes {1 (src) | 2 (kern), index, iteration}. */
  int32_t* error;
  /* ABI 2, optional.  Compact explicit gathers: when a_shift is non-NULL,
   * a_idx / b_idx hold ONE [m*n][k] table shared by every iteration, and
   * iteration v reads src index a_idx[..] + a_shift[v]. */
  const int32_t* a_shift;
  /* ABI 2, optional.  Independent iterations (a For loop whose body is
   * zero-fill, one conv statement, then a copy or wmma_store of the result):
   * when out_base is non-NULL every iteration starts from 0 and stores its
   * m*n results at out[t*out_stride + out_base[v] + out_off[o]] (out_off NULL
   * = o); acc is not touched.  All iterations run in parallel. */
  const int32_t* out_base;
  const int32_t* out_off;
  float* out;
  int64_t out_stride;
} ts_conv_group;

/* Replaces the serial For/Store walk of interp.run_program (interp.py:570-619)
 * over a lowered conv group (interp.py:419-486, 488-534). */
TS_API ts_status ts_run_conv_group(const ts_conv_group* group, void* stream);

/* f32-input separable transform on the FMA pipe (config c1: an f32 image is
 * read once, no bf16 copy).  Replaces, for f32 images, the two 1-D
 * source-form conv passes of the reference (interp.py:162-167, 203-211;
 * oracle/pipelines_ref.py:78-97) in their exact evaluation order —
 * horizontal pass first, taps summed left to right, then + 0.  With
 * flags & TS_F32_EXACT every product and sum is rounded separately, as the
 * reference does, and f32 outputs are bit-identical to the reference's;
 * without it each tap is one fused multiply-add (faster; differs from the
 * reference by f32 rounding only, ~1e-7).  Uniform axes only: output o of an
 * axis reads inputs clamp(stride*o + base + t), t < taps, with the SAME taps
 * weights[t] for every o (device f32).  Instantiated (stride, taps, base & 3):
 * (2, 12, 3) = Lanczos-3 2x, (1, 9|15|21|31, -(taps-1)/2 & 3) = centred
 * filters; others return TS_ERR_UNSUPPORTED.  out: f32 or bf16 (strides in
 * elements); ep may be NULL. */
#define TS_F32_EXACT 0x1
TS_API ts_status ts_separable_f32_ep(int planes, const float* in, int in_h, int in_w,
                                     int64_t in_row_stride, int64_t in_plane_stride, int stride,
                                     int taps, int row_base, const float* row_weights, int out_h,
                                     int col_base, const float* col_weights, int out_w, void* out,
                                     int64_t out_row_stride, int64_t out_plane_stride,
                                     int out_dtype, int flags, const ts_epilogue* ep,
                                     void* stream);

/* Elementwise f32 -> bf16 (round to nearest even), n elements. */
TS_API ts_status ts_cast_f32_bf16(const float* in, void* out, int64_t n, void* stream);

/* Device-side dense Toeplitz family builder: writes the matrix_rows(spec) x k
 * row-major matrix of layout.matrix_for (layout.py:72-84) for kernel (device
 * f32, p*l entries) into out (device f32).  Replaces the Python double loop. */
TS_API ts_status ts_matrix_for(int l, int k, int s, int p, const float* kernel, float* out, void* stream);


#ifdef __cplusplus
}
#endif

#endif /* TENSORSEL_B200_H */

/*
 * tsb_diag.h — diagnostic entry points of libtsb200_diag.so (tools only).
 *
 * `make -C paper_2512_02371_b200/csrc diag` builds the product sources with
 * -DTSB_DIAG (per-tile clock64 trace stamps, TMEM dumps) plus the tcgen05 /
 * TMA / TMEM micro-probes of tools/diag/probe.cu into a separate library.
 * None of this is in the product library libtsb200.so or its header; the
 * tools under tools/ load it with paper_2512_02371_b200._lib.load_diag().
 */
#ifndef TSB_DIAG_H
#define TSB_DIAG_H

#include "../../include/tensorsel_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define TS_DIAG_API TS_API

/* Diagnostics: subsequent ts_denoise_dct16 launches also write every
 * forward coefficient (before coring, f32) into device_buffer, laid out like
 * oracle/pipelines_ref.dct_coefficients: (planes, H/8 + 1, W/8 + 1, 16, 16)
 * (tile row, tile column, row frequency, column frequency).  NULL turns it
 * off.  Measures the forward chain's error (tools/dct_coef_error.py). */
TS_DIAG_API ts_status ts_debug_dct16(float* device_buffer);

/* Diagnostics: make subsequent ts_separable_run launches record clock64()
 * stamps for the first `tiles` tiles of CTAs [0, ctas) into device_buffer
 * (u64[ctas][tiles][10]; events: 0 producer ready, 1 stage free, 2 input
 * landed, 3 pass-1 issued, 4 D_V ready, 5 V operand written, 6 pass-2 start,
 * 7 pass-2 issued, 8 D_H ready, 9 output stored).  NULL turns it off. */
TS_DIAG_API ts_status ts_debug_trace(void* device_buffer, int ctas, int tiles);

/* Diagnostics: one tcgen05 MMA  D(128 x n) = A(128 x k) · B(k x n)  with A
 * staged MN-major 128B-swizzled and B K-major interleaved exactly as the
 * separable kernel stages them.  a: row-major f32 (128 x k), b: row-major
 * f32 (k x n), d: row-major f32 (128 x n); all device pointers; k % 16 == 0,
 * n % 16 == 0, n <= 256, k <= 256. */
TS_DIAG_API ts_status ts_probe_umma(const float* a, const float* b, float* d, int k, int n, void* stream);

/* Diagnostics: tcgen05 operand-mode probe.  D(128 x n) = A(128 x k) · B(k x n),
 * the K loop issued `reps` times into one accumulator; *cycles (device
 * pointer, may be NULL) receives clock64 cycles from first issue to
 * completion.  amode 0: A smem MN-major SW128 bf16, 1: A smem K-major bf16,
 * 2: A in TMEM f32 (kind::tf32); bmode 0: B smem K-major (bf16, f32 for
 * amode 2), 1: B smem MN-major SW128 bf16.  nacc > 1 round-robins the
 * repetitions over nacc accumulators (columns [n*i, n*i + n)) to measure
 * independent-MMA throughput; d then holds accumulator 0. */
TS_DIAG_API ts_status ts_probe_mma(int amode, int bmode, const float* a, const float* b, float* d,
                              int k, int n, int reps, long long* cycles, int nacc, void* stream);

/* Diagnostics: tcgen05.mma issue-rate microbenchmark (64 warp-converged,
 * elect-issued M=128 K=16 MMAs; variant 0..5 = N/accumulators (16,1) (16,8)
 * (64,1) (64,4) (256,1) (256,2)); *cycles (device) = cycles to completion. */
TS_DIAG_API ts_status ts_probe_issue(int variant, long long* cycles, void* stream);
/* Same with A read from TMEM (TS mode); variant 0..3 = (N, kind) in
 * {(16, f16), (64, f16), (16, tf32), (64, tf32)}. */
TS_DIAG_API ts_status ts_probe_issue_ts(int variant, long long* cycles, void* stream);
/* Streaming-operand issue rate: `count` elected M=128, K=16 MMAs cycling over
 * 8 K-slices; amode 0 smem MN-major SW128 / 1 smem K-major / 2 TMEM,
 * bmode 0 smem K-major / 1 smem MN-major SW128; nacc accumulators. */
/* TMA streaming probe: grid CTAs stream a planes x H x W bf16 tensor in
 * chunks of rows x (64 * nbox) through an nr-slot ring (load path only). */
TS_DIAG_API ts_status ts_probe_tma(const void* src, int planes, int H, int W, int rows, int nbox, int nr,
                              int grid, void* stream);
/* TMEM load throughput probe: `warps` warps (multiple of 4) read `cols`
 * columns of their lane quarter `reps` times with tcgen05.ld.32x32b.x{x}. */
TS_DIAG_API ts_status ts_probe_tmem_ld(int x, int warps, int cols, int reps, long long* cycles,
                                  void* stream);
/* M = 64 accumulator layout probe: D (128 lanes x n, pre-filled with -1) after
 * one kind::f16 M=64 MMA (A 64 x 16, B 16 x n, row-major f32 in) issued at
 * TMEM lane lane_base; d receives all 128 lanes. */
TS_DIAG_API ts_status ts_probe_m64(const float* a, const float* b, float* d, int n, int lane_base,
                              void* stream);
TS_DIAG_API ts_status ts_probe_issue2(int amode, int bmode, int n, int count, int nacc,
                                 long long* cycles, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TSB_DIAG_H */

// separable.cu — fused separable linear transform on sm_100a:
//
//     out[p] = R · in[p] · Cᵀ        (R: rows axis, C: cols axis, both banded)
//
// This is the B200 execution of what the reference expresses as lowered
// `wmma_load_a(I, base, s·n, m, k)` / `wmma_load_b(Toeplitz)` / `wmma_mma`
// statements (rules.py:766-803, interp.py:427-486): an overlapped-window
// gather times a banded Toeplitz-family matrix, f32 accumulation.  One
// persistent kernel (one CTA per SM) does both passes of a separable
// resample / filter.  Work unit ("tile") = (plane p, 128 output rows,
// nb2·16 output columns).  Warp roles:
//
//  warp 0      TMA producer: the input halo tile (R1 rows x 128 cols bf16,
//              128B-swizzled, 4 boxes) into an nst-deep ring; B tiles are
//              either CTA-resident (copied once) or staged per tile.
//  warp 1      pass-1 MMA issuer (vertical), per super-block k of m1
//              16-output-row blocks (merge.cpp; m1 = 1 unless overlapping
//              windows make merging cheaper):
//                D_V[c, 16·m1·k..] = Σ_r X[r, c] · R_kᵀ[r, ·]   M=128 cols, N=16·m1
//                A = staged tile (MN-major SW128), B = R tile (K-major)
//  warp 10     pass-2 MMA issuer (horizontal), per super-block j of m2
//              16-output-column blocks (nb2 <= 16 blocks per tile):
//                D_H[i, 16·m2·j..] = Σ_c V[i, c] · C_jᵀ[c, ·]   M=128 rows, N=16·m2
//                A = V (bf16 MN-major SW128, written by warps 2-5)
//  warps 2-5   epilogue 1: D_V (TMEM) -> bf16 -> V operand (smem, x nmid)
//  warps 6-9   epilogue 2: D_H (TMEM) -> cast -> smem -> TMA store
//
// The issuing warps run converged and elect one lane per tcgen05 op; the
// per-block window starts / tile ids are read from the kernel-parameter
// (constant) bank so they land directly in uniform registers.
//
// TMEM (512 cols): D_V double-buffered at [0,128) and [128,256), D_H at
// [256, 256 + nb2·16).  Window starts are multiples of 8 rows/cols (the
// builder guarantees it) so every MMA operand starts on a 1024-byte atom.
// Waiting warps sleep in mbarrier.try_wait (sm100.cuh) rather than spin:
// under the sustained power cap that keeps ~70 MHz more SM clock.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.h"
#include "sm100.cuh"

namespace tsb {

const MergedAxis* axis_merged(const ts_axis* a, int m);
int choose_merge(const ts_axis* a, int blocks);

constexpr int kMaxStages = 4;
constexpr int kThreads = 352;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kMidBytes = 128 * 128 * 2;  // V tile: 128 rows x 128 cols bf16
constexpr uint32_t kSmemLimit = 232448;        // max dynamic smem per CTA on sm_100
constexpr int kParamTab = 3072;                // packed block entries carried in params

// Shared-memory plan, chosen on the host and passed to the kernel.
struct SepSmem {
  uint32_t nst;        // input stages
  uint32_t nmid;       // V-operand buffers (1 or 2)
  uint32_t resident;   // 1: all B tiles copied once; 0: staged with each tile
  uint32_t in_stage;   // bytes per input stage
  uint32_t w_stage;    // bytes per weight stage (staged mode)
  uint32_t w1_bytes;   // offset of the C tiles inside a weight stage / resident block
  uint32_t off_w, off_mid, off_out, off_bar, total;
};

struct SepParams {
  AxisDev r;  // rows axis (pass 1)
  AxisDev c;  // cols axis (pass 2)
  int nb2;    // column blocks per tile
  int m1, m2;    // merge factors: blocks per super-block (csrc/merge.cpp), rows / cols
  int sb1, sb2;  // super-blocks per tile: 8 / m1 (pass 1), nb2 / m2 (pass 2)
  int R1;     // staged input rows per tile (multiple of 16)
  int nrt, nct, planes, ntiles;
  // dynamic tile scheduling: CTAs claim tiles in order from *tile_next (and
  // the last CTA to finish resets both counters for the next launch on the
  // same stream); null = static round-robin
  int* tile_next;
  int* ctas_done;
  unsigned long long* trace;  // diagnostics: per-(CTA, tile, event) clock64 stamps or null
  int trace_ctas, trace_tiles;
  int ptab;      // 1: block tables below, 0: read r.tab / c.tab from global
  int ptab_c;    // offset of the cols table inside tab[]
  SepSmem L;
  int32_t tab[kParamTab];  // packed (ws << 16) | tid, rows then cols
  EpiK ep;                 // output epilogue (EPI kernels only)
};

__device__ __forceinline__ int32_t tab_r(const SepParams& P, int b) {
  return P.ptab ? P.tab[b] : P.r.tab[b];
}
__device__ __forceinline__ int32_t tab_c(const SepParams& P, int b) {
  return P.ptab ? P.tab[P.ptab_c + b] : P.c.tab[b];
}
__device__ __forceinline__ int tab_ws(int32_t e) { return e >> 16; }

// Diagnostics: stamp event `ev` of tile `it` (events 0..9, see ts_debug_trace).
__device__ __forceinline__ void trace_stamp(const SepParams& P, int it, int ev) {
#ifdef TSB_DIAG
  if (P.trace != nullptr && static_cast<int>(blockIdx.x) < P.trace_ctas && it < P.trace_tiles &&
      (threadIdx.x & 31) == 0)
    P.trace[(static_cast<size_t>(blockIdx.x) * P.trace_tiles + it) * 10 + ev] = clock64();
#endif
}
__device__ __forceinline__ int tab_tid(int32_t e) { return e & 0xFFFF; }

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// one 16-column block of an output row into the staging tile, with the
// output epilogue when EPI
template <typename OutT, bool EPI>
__device__ __forceinline__ void store_out_row(uint32_t dst, uint32_t (&r)[16], const EpiK& ep) {
  if constexpr (sizeof(OutT) == 2) {
    uint32_t p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      p[i] = EPI ? epi_bf16x2(ep, __uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]))
                 : pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    }
    st_shared_v4(dst, p[0], p[1], p[2], p[3]);
    st_shared_v4(dst + 16, p[4], p[5], p[6], p[7]);
  } else {
    if constexpr (EPI) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(epi_f32(ep, __uint_as_float(r[i])));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      st_shared_v4(dst + 16 * i, r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
  }
}

// Persistent tile walk t = blockIdx.x + it·gridDim.x with (p, rt, ct) kept
// incrementally (one division at start, none per tile).
// Tiles in flight, by claim order: the producer writes the claimed tile of
// iteration `it` ({t, plane, row tile, column tile}) to ring slot
// it % kTileRing before its stage's full barrier completes; every later role
// reads it after its own wait (t = -1: no more tiles).  Claims run at most
// ~nst + 5 iterations ahead of the last role.
constexpr int kTileRing = 16;

struct TileXY {
  int p, rt, ct;
};

__device__ __forceinline__ TileXY tile_xy(const SepParams& P, int t) {
  TileXY r;
  r.ct = t % P.nct;
  const int rest = t / P.nct;
  r.rt = rest % P.nrt;
  r.p = rest / P.nrt;
  return r;
}

template <typename OutT, int KQ1, int KQ2, bool EPI = false>
__global__ void __launch_bounds__(kThreads, 1)
    separable_kernel(const __grid_constant__ CUtensorMap tm_in,
                     const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ SepParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const SepSmem& L = P.L;

  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L.off_bar);
  uint64_t* full = bars;                      // [kMaxStages] input (+weights) landed
  uint64_t* empty = bars + kMaxStages;        // [kMaxStages] stage consumed
  uint64_t* dv_full = bars + 2 * kMaxStages;  // [2]
  uint64_t* dv_free = dv_full + 2;            // [2]
  uint64_t* mid_full = dv_full + 4;           // [2]
  uint64_t* mid_free = dv_full + 6;           // [2]
  uint64_t* dh_full = dv_full + 8;
  uint64_t* dh_free = dv_full + 9;
  uint64_t* wres = dv_full + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dv_full + 11);
  volatile int* tile_ring = reinterpret_cast<volatile int*>(dv_full + 12);  // [kTileRing][4]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dv_full[b], 1);
      mbar_init(&dv_free[b], 128);
      mbar_init(&mid_full[b], 128);
      mbar_init(&mid_free[b], 1);
    }
    mbar_init(dh_full, 1);
    mbar_init(dh_free, 128);
    mbar_init(wres, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_in);
    prefetch_tmap(&tm_out);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous kernel in the stream is complete

  const int nb2 = P.nb2;
  const int nst = static_cast<int>(L.nst);
  const int nmid = static_cast<int>(L.nmid);
  // N = 16 x merge factor (super-blocks of m 16-output blocks)
  const uint32_t idesc1 = make_idesc(kFmtBF16, 128, 16 * P.m1, /*a MN-major*/ 1, /*b K-major*/ 0);
  const uint32_t idesc2 = make_idesc(kFmtBF16, 128, 16 * P.m2, /*a MN-major*/ 1, /*b K-major*/ 0);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      if (L.resident) {
        const uint32_t rb = static_cast<uint32_t>(P.r.ntiles * P.r.tile_bytes);
        const uint32_t cb = static_cast<uint32_t>(P.c.ntiles * P.c.tile_bytes);
        mbar_arrive_expect_tx(wres, rb + cb);
        bulk_g2s(base + L.off_w, P.r.tiles, rb, wres);
        bulk_g2s(base + L.off_w + L.w1_bytes, P.c.tiles, cb, wres);
      }
      const int hr = P.R1 / 2;
      // claim tiles in order (dynamic) or round-robin (static); the claim for
      // the next iteration is issued one iteration early so the atomic's
      // round trip overlaps this tile's stage wait and TMA issue
      auto claim = [&](int it) {
        return P.tile_next ? atomicAdd(P.tile_next, 1)
                           : static_cast<int>(blockIdx.x) + it * static_cast<int>(gridDim.x);
      };
      int t_next = claim(0);
      for (int it = 0;; ++it) {
        const int s = it % nst;
        const uint32_t ph = (it / nst) & 1;
        int t = t_next;
        if (t >= P.ntiles) t = -1;
        if (t < 0) {  // no more tiles: complete a stage with no data
          mbar_wait(&empty[s], ph ^ 1);
          tile_ring[4 * (it % kTileRing)] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        t_next = claim(it + 1);
        // everything about the tile is computed before the stage wait, so
        // the TMA issue follows the wait immediately (the ring period sets
        // the kernel's pace)
        const TileXY tw = tile_xy(P, t);
        const int b1 = tw.rt * P.sb1, b2 = tw.ct * P.sb2;
        const int row0 = tab_ws(tab_r(P, b1)), col0 = tab_ws(tab_c(P, b2));
        uint32_t wbytes = 0;
        if (!L.resident) {
          for (int k = 0; k < P.sb1; ++k)
            if (k == 0 || tab_tid(tab_r(P, b1 + k)) != tab_tid(tab_r(P, b1 + k - 1)))
              wbytes += P.r.tile_bytes;
          for (int j = 0; j < P.sb2; ++j)
            if (j == 0 || tab_tid(tab_c(P, b2 + j)) != tab_tid(tab_c(P, b2 + j - 1)))
              wbytes += P.c.tile_bytes;
        }
        trace_stamp(P, it, 0);
        mbar_wait(&empty[s], ph ^ 1);
        trace_stamp(P, it, 1);
        volatile int* tslot = tile_ring + 4 * (it % kTileRing);
        tslot[0] = t;
        tslot[1] = tw.p;
        tslot[2] = tw.rt;
        tslot[3] = tw.ct;
        mbar_arrive_expect_tx(&full[s], L.in_stage + wbytes);
        uint8_t* dst = base + s * L.in_stage;
        tma_load_3d(dst, &tm_in, &full[s], col0, row0, tw.p);
        tma_load_3d(dst + hr * 128, &tm_in, &full[s], col0, row0 + hr, tw.p);
        tma_load_3d(dst + P.R1 * 128, &tm_in, &full[s], col0 + 64, row0, tw.p);
        tma_load_3d(dst + P.R1 * 128 + hr * 128, &tm_in, &full[s], col0 + 64, row0 + hr, tw.p);
        if (!L.resident) {
          uint8_t* wd = base + L.off_w + s * L.w_stage;
          for (int k = 0; k < P.sb1; ++k) {
            const int tid = tab_tid(tab_r(P, b1 + k));
            if (k == 0 || tid != tab_tid(tab_r(P, b1 + k - 1)))
              bulk_g2s(wd + k * P.r.tile_bytes,
                       P.r.tiles + static_cast<size_t>(tid) * P.r.tile_bytes, P.r.tile_bytes,
                       &full[s]);
          }
          for (int j = 0; j < P.sb2; ++j) {
            const int tid = tab_tid(tab_c(P, b2 + j));
            if (j == 0 || tid != tab_tid(tab_c(P, b2 + j - 1)))
              bulk_g2s(wd + L.w1_bytes + j * P.c.tile_bytes,
                       P.c.tiles + static_cast<size_t>(tid) * P.c.tile_bytes, P.c.tile_bytes,
                       &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ pass-1 issuer
    const uint32_t lbo_in = static_cast<uint32_t>(P.R1) * 128u;  // 64-col half stride
    const int kq1 = KQ1 > 0 ? KQ1 : P.r.K / 16;
    const uint32_t tb1 = P.r.tile_bytes;
    const uint32_t sbo1 = static_cast<uint32_t>(P.r.K) * 16u;
    if (L.resident) mbar_wait(wres, 0);
    for (int it = 0;; ++it) {
      const int s = it % nst;
      const int d = it & 1;
      const uint32_t a0 = base_s + s * L.in_stage;
      const uint32_t w0 = L.resident ? base_s + L.off_w : base_s + L.off_w + s * L.w_stage;
      mbar_wait(&full[s], (it / nst) & 1);
      trace_stamp(P, it, 2);
      const volatile int* tslot = tile_ring + 4 * (it % kTileRing);
      if (tslot[0] < 0) {  // pass the end on to epilogue 1
        // (only once epilogue 1 has drained D_V[d]: a barrier must never run
        // two phases ahead of its waiter, or the waiter's parity test reads
        // the older phase as still pending — the same wait before every
        // end-of-work signal below)
        mbar_wait(&dv_free[d], ((it >> 1) & 1) ^ 1);
        mma_commit_elect(&dv_full[d]);
        break;
      }
      const int b1 = tslot[2] * P.sb1;
      const int row0 = tab_ws(tab_r(P, b1));
      mbar_wait(&dv_free[d], ((it >> 1) & 1) ^ 1);
      __syncwarp();
      tc_fence_after();
      int slot = 0, prev = -1;
#pragma unroll
      for (int k = 0; k < kRowBlocksPerTile; ++k) {
        if (k >= P.sb1) break;
        const int32_t e = tab_r(P, b1 + k);
        const int tid = tab_tid(e);
        if (L.resident)
          slot = tid;
        else if (tid != prev)
          slot = k;
        prev = tid;
        const uint64_t ad = make_sdesc(a0 + static_cast<uint32_t>(tab_ws(e) - row0) * 128u, lbo_in,
                                       1024u, kSwizzle128B);
        const uint64_t bd = make_sdesc(w0 + slot * tb1, 128u, sbo1, kSwizzleNone);
        const uint32_t dcol = tmem + d * 128u + static_cast<uint32_t>(16 * P.m1 * k);
#pragma unroll
        for (int q = 0; q < (KQ1 > 0 ? KQ1 : 16); ++q) {
          if (KQ1 == 0 && q >= kq1) break;
          // +2048 B (16 rows of A) and +256 B (two k-chunks of B) per K step
          mma_f16_ss_elect(dcol, ad + 128u * q, bd + 16u * q, idesc1, q > 0 ? 1u : 0u);
        }
      }
      mma_commit_elect(&dv_full[d]);
      if (L.resident) mma_commit_elect(&empty[s]);
      trace_stamp(P, it, 3);
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ pass-2 issuer
    const int kq2 = KQ2 > 0 ? KQ2 : P.c.K / 16;
    const uint32_t tb2 = P.c.tile_bytes;
    const uint32_t sbo2 = static_cast<uint32_t>(P.c.K) * 16u;
    if (L.resident) mbar_wait(wres, 0);
    for (int it = 0;; ++it) {
      const int s = it % nst;
      const int m = it % nmid;
      const uint32_t w0 = L.resident ? base_s + L.off_w : base_s + L.off_w + s * L.w_stage;
      const uint32_t mid_s = base_s + L.off_mid + m * kMidBytes;
      mbar_wait(&mid_full[m], (it / nmid) & 1);
      trace_stamp(P, it, 6);
      const volatile int* tslot = tile_ring + 4 * (it % kTileRing);
      if (tslot[0] < 0) {  // pass the end on to epilogue 2 (once it drained D_H)
        mbar_wait(dh_free, (it & 1) ^ 1);
        mma_commit_elect(dh_full);
        break;
      }
      const int b2 = tslot[3] * P.sb2;
      const int col0 = tab_ws(tab_c(P, b2));
      mbar_wait(dh_free, (it & 1) ^ 1);
      __syncwarp();
      tc_fence_after();
      int slot = 0, prev = -1;
#pragma unroll 1
      for (int j = 0; j < P.sb2; ++j) {
        const int32_t e = tab_c(P, b2 + j);
        const int tid = tab_tid(e);
        if (L.resident)
          slot = tid;
        else if (tid != prev)
          slot = j;
        prev = tid;
        const uint64_t ad = make_sdesc(mid_s + static_cast<uint32_t>((tab_ws(e) - col0) / 8) * 1024u,
                                       16384u, 1024u, kSwizzle128B);
        const uint64_t bd = make_sdesc(w0 + L.w1_bytes + slot * tb2, 128u, sbo2, kSwizzleNone);
        const uint32_t dcol = tmem + 256u + static_cast<uint32_t>(16 * P.m2 * j);
#pragma unroll
        for (int q = 0; q < (KQ2 > 0 ? KQ2 : 16); ++q) {
          if (KQ2 == 0 && q >= kq2) break;
          mma_f16_ss_elect(dcol, ad + 128u * q, bd + 16u * q, idesc2, q > 0 ? 1u : 0u);
        }
      }
      mma_commit_elect(dh_full);
      mma_commit_elect(&mid_free[m]);
      if (!L.resident) mma_commit_elect(&empty[s]);
      trace_stamp(P, it, 7);
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue 1
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int c = quarter * 32 + lane;  // input column within the tile
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    for (int it = 0;; ++it) {
      const int d = it & 1;
      const int m = it % nmid;
      const uint32_t mid_row =
          base_s + L.off_mid + m * kMidBytes + (c / 8) * 1024u + (c % 8) * 128u;
      mbar_wait(&dv_full[d], (it >> 1) & 1);
      if (warp == 2) trace_stamp(P, it, 4);
      if (tile_ring[4 * (it % kTileRing)] < 0) {  // pass the end on to the pass-2 issuer
        mbar_wait(&mid_free[m], ((it / nmid) & 1) ^ 1);  // once it has read mid[m]
        mbar_arrive(&mid_full[m]);
        break;
      }
      mbar_wait(&mid_free[m], ((it / nmid) & 1) ^ 1);
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t r[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld16(t_lane + d * 128u + 64u * h + 16u * q, r[q]);
        tmem_wait_ld();
        if (h == 1) {
          tc_fence_before();
          mbar_arrive(&dv_free[d]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int i8 = h * 8 + q * 2 + g;  // 8-row group of output rows
            const uint32_t addr = mid_row + (i8 / 8) * 16384u + (((i8 % 8) ^ (c % 8)) * 16u);
            st_shared_v4(addr,
                         pack_bf16x2(__uint_as_float(r[q][8 * g + 0]), __uint_as_float(r[q][8 * g + 1])),
                         pack_bf16x2(__uint_as_float(r[q][8 * g + 2]), __uint_as_float(r[q][8 * g + 3])),
                         pack_bf16x2(__uint_as_float(r[q][8 * g + 4]), __uint_as_float(r[q][8 * g + 5])),
                         pack_bf16x2(__uint_as_float(r[q][8 * g + 6]), __uint_as_float(r[q][8 * g + 7])));
          }
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&mid_full[m]);
      if (warp == 2) trace_stamp(P, it, 5);
    }
  } else {
    // ------------------------------------------------------------ epilogue 2
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // output row within the tile
    const int et = threadIdx.x - 192;     // 0..127
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + 256u;
    const uint32_t out_row_bytes = static_cast<uint32_t>(nb2 * 16 * sizeof(OutT));
    const uint32_t orow = base_s + L.off_out + row * out_row_bytes;
    for (int it = 0;; ++it) {
      mbar_wait(dh_full, it & 1);
      if (warp == 6) trace_stamp(P, it, 8);
      const volatile int* tslot = tile_ring + 4 * (it % kTileRing);
      if (tslot[0] < 0) break;
      TileXY tw;
      tw.p = tslot[1];
      tw.rt = tslot[2];
      tw.ct = tslot[3];
      tc_fence_after();
      if (et == 0) bulk_wait_read0();  // previous TMA store finished reading staging
      named_bar_sync(2, 128);
      // up to 16 blocks, 8 per batch of TMEM loads (128 registers)
      for (int j0 = 0; j0 < nb2; j0 += 8) {
        uint32_t r[8][16];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < nb2) tmem_ld16(t_lane + 16u * (j0 + j), r[j]);
        tmem_wait_ld();
        if (j0 + 8 >= nb2) {
          tc_fence_before();
          mbar_arrive(dh_free);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < nb2)
            store_out_row<OutT, EPI>(orow + (j0 + j) * 16u * sizeof(OutT), r[j], P.ep);
      }
      fence_proxy_async_smem();
      named_bar_sync(2, 128);
      if (et == 0) {
        tma_store_3d(&tm_out, base + L.off_out, tw.ct * nb2 * 16, tw.rt * kRowBlocksPerTile * 16,
                     tw.p);
        bulk_commit();
      }
      if (warp == 6) trace_stamp(P, it, 9);
    }
    if (et == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  // the next kernel in the stream may launch only now: CTAs parked in
  // griddepcontrol.wait beside working ones slowed them (an early
  // trigger cost 30% on a 4K -> 540p two-pass resample)
  pdl_launch_dependents();
  // the last CTA out resets the claim counters for the next launch on this
  // stream (launches on one stream are ordered; streams get their own pair)
  if (threadIdx.x == 0 && P.tile_next != nullptr) {
    __threadfence();
    if (atomicAdd(P.ctas_done, 1) == static_cast<int>(gridDim.x) - 1) {
      atomicExch(P.tile_next, 0);
      atomicExch(P.ctas_done, 0);
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(TS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1),
                        static_cast<cuuint64_t>(d2)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(stride1_elems * esize),
                           static_cast<cuuint64_t>(stride2_elems * esize)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(TS_ERR_INVALID,
                     "cuTensorMapEncodeTiled failed (%d): dims %lld x %lld x %lld, strides %lld/%lld "
                     "elems, box %d x %d",
                     static_cast<int>(r), (long long)d0, (long long)d1, (long long)d2,
                     (long long)stride1_elems, (long long)stride2_elems, box0, box1);
  return TS_OK;
}

int sm_count_current() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cache[dev] > 0) return cache[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  n = n > 0 ? n : 148;
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

// Pick stages / V buffers / weight residency to fit the shared-memory budget,
// preferring (in order) two V buffers, resident weights, then more stages.
static bool plan_smem(SepParams& P, int oes) {
  const uint32_t in_stage = 2u * static_cast<uint32_t>(P.R1) * 128u;
  const uint32_t tb1 = P.r.tile_bytes, tb2 = P.c.tile_bytes;
  const uint32_t res_w1 = align_up(static_cast<uint32_t>(P.r.ntiles) * tb1, 128);
  const uint32_t res_bytes = align_up(res_w1 + static_cast<uint32_t>(P.c.ntiles) * tb2, 1024);
  const uint32_t st_w1 = static_cast<uint32_t>(P.sb1) * tb1;
  const uint32_t st_bytes = align_up(st_w1 + static_cast<uint32_t>(P.sb2) * tb2, 1024);
  const uint32_t out_bytes = align_up(128u * P.nb2 * 16u * oes, 1024);
  const uint32_t fixed = out_bytes + 512 + 1024;  // barriers + tile ring + alignment slack
  // (a single input stage was measured slower than two axis passes: 2048^2 ->
  // 921^2 at 48 planes 0.280 vs 0.248 ms, so plans need >= 2 stages)
  for (uint32_t nmid = 2; nmid >= 1; --nmid) {
    for (int resident = 1; resident >= 0; --resident) {
      for (uint32_t nst = kMaxStages; nst >= 2; --nst) {
        const uint32_t wb = resident ? res_bytes : nst * st_bytes;
        const uint32_t total = nst * in_stage + wb + nmid * kMidBytes + fixed;
        if (total > kSmemLimit) continue;
        SepSmem& L = P.L;
        L.nst = nst;
        L.nmid = nmid;
        L.resident = static_cast<uint32_t>(resident);
        L.in_stage = in_stage;
        L.w_stage = st_bytes;
        L.w1_bytes = resident ? res_w1 : st_w1;
        L.off_w = nst * in_stage;
        L.off_mid = L.off_w + wb;
        L.off_out = L.off_mid + nmid * kMidBytes;
        L.off_bar = L.off_out + out_bytes;
        L.total = L.off_bar + 512 + 1024;
        return true;
      }
    }
  }
  return false;
}

template <typename OutT, int KQ1, int KQ2, bool EPI = false>
static ts_status launch_sep_k(const SepParams& P, const CUtensorMap& tin, const CUtensorMap& tout,
                              cudaStream_t stream) {
  auto kern = separable_kernel<OutT, KQ1, KQ2, EPI>;
  // the smem ceiling is set once per device (to the maximum any plan uses)
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaSuccess;
  if (dev < 0 || dev >= 64 || !attr_done[dev]) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemLimit));
    if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(separable smem)");
    if (dev >= 0 && dev < 64) attr_done[dev] = true;
  }
  const int sms = sm_count_current();
  const int grid = P.ntiles < sms ? P.ntiles : sms;
  e = launch_pdl(kern, grid, kThreads, P.L.total, stream, tin, tout, P);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_error(e, "separable_kernel launch");
  return TS_OK;
}

// Compile-time K-step counts for the common windows (32, 48, 64 inputs per
// 16-output block); anything else runs the runtime-count variant.
template <typename OutT, int KQ1, bool EPI>
static ts_status launch_sep_k2(const SepParams& P, const CUtensorMap& tin,
                               const CUtensorMap& tout, cudaStream_t stream) {
  switch (P.c.K / 16) {
    case 2: return launch_sep_k<OutT, KQ1, 2, EPI>(P, tin, tout, stream);
    case 3: return launch_sep_k<OutT, KQ1, 3, EPI>(P, tin, tout, stream);
    case 4: return launch_sep_k<OutT, KQ1, 4, EPI>(P, tin, tout, stream);
    case 5: return launch_sep_k<OutT, KQ1, 5, EPI>(P, tin, tout, stream);
    default: return launch_sep_k<OutT, KQ1, 0, EPI>(P, tin, tout, stream);
  }
}

template <typename OutT, bool EPI>
static ts_status launch_sep_e(const SepParams& P, const CUtensorMap& tin, const CUtensorMap& tout,
                              cudaStream_t stream) {
  switch (P.r.K / 16) {
    case 2: return launch_sep_k2<OutT, 2, EPI>(P, tin, tout, stream);
    case 3: return launch_sep_k2<OutT, 3, EPI>(P, tin, tout, stream);
    case 4: return launch_sep_k2<OutT, 4, EPI>(P, tin, tout, stream);
    case 5: return launch_sep_k2<OutT, 5, EPI>(P, tin, tout, stream);
    case 6: return launch_sep_k2<OutT, 6, EPI>(P, tin, tout, stream);
    default: return launch_sep_k2<OutT, 0, EPI>(P, tin, tout, stream);
  }
}

// with an output epilogue the EPI twins of the same kernels run (the plain
// kernels carry no epilogue code)
template <typename OutT>
static ts_status launch_sep(const SepParams& P, const CUtensorMap& tin, const CUtensorMap& tout,
                            cudaStream_t stream, bool epi) {
  return epi ? launch_sep_e<OutT, true>(P, tin, tout, stream)
             : launch_sep_e<OutT, false>(P, tin, tout, stream);
}

// Tile-claim counters, one pair per (device, stream): launches on one stream
// run in order, so a kernel's last CTA can reset its pair for the next one;
// concurrent streams must not share a pair.
static bool claim_counters(int device, cudaStream_t stream, int** next, int** done) {
  constexpr int kSlots = 256;
  struct Dev {
    int* d = nullptr;
    std::vector<cudaStream_t> streams;
  };
  static Dev devs[64];
  static std::mutex mu;
  if (device < 0 || device >= 64) return false;
  std::lock_guard<std::mutex> lock(mu);
  Dev& D = devs[device];
  if (!D.d) {
    if (cudaMalloc(&D.d, 2 * kSlots * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      D.d = nullptr;
      return false;
    }
    if (cudaMemset(D.d, 0, 2 * kSlots * sizeof(int)) != cudaSuccess) return false;
  }
  size_t slot = 0;
  while (slot < D.streams.size() && D.streams[slot] != stream) ++slot;
  if (slot == D.streams.size()) {
    if (slot >= static_cast<size_t>(kSlots)) return false;
    D.streams.push_back(stream);
  }
  *next = D.d + 2 * slot;
  *done = D.d + 2 * slot + 1;
  return true;
}

static unsigned long long* g_trace = nullptr;
static int g_trace_ctas = 0, g_trace_tiles = 0;

void get_trace(unsigned long long** buf, int* ctas, int* tiles) {
  *buf = g_trace;
  *ctas = g_trace_ctas;
  *tiles = g_trace_tiles;
}

#ifdef TSB_DIAG
void set_trace(void* buf, int ctas, int tiles) {
  g_trace = static_cast<unsigned long long*>(buf);
  g_trace_ctas = buf ? ctas : 0;
  g_trace_tiles = buf ? tiles : 0;
}
#endif  // TSB_DIAG

static ts_status make_params(const ts_axis* ra, const ts_axis* ca, int planes, int oes,
                             SepParams& P) {
  P.trace = g_trace;
  P.trace_ctas = g_trace_ctas;
  P.trace_tiles = g_trace_tiles;
  if (!ra->tab_ok || !ca->tab_ok)
    return set_error(TS_ERR_UNSUPPORTED,
                     "separable: axis longer than the fused kernel's packed block tables (32K)");
  if (ra->K > 256 || ca->K > 256)
    return set_error(TS_ERR_UNSUPPORTED,
                     "separable: windows %d / %d exceed the fused kernel's 256 (use axis passes)",
                     ra->K, ca->K);
  if (ra->row_span > kMaxRowSpan || ra->row_span % 16)
    return set_error(TS_ERR_UNSUPPORTED, "rows axis: row tile span %d > %d", ra->row_span,
                     kMaxRowSpan);
  if (ca->col_nbt < 1)
    return set_error(TS_ERR_UNSUPPORTED, "cols axis: window %d does not fit a 128-column tile",
                     ca->K);
  auto dev_of = [](const ts_axis* a, int m) {
    if (m <= 1) return a->dev();
    const MergedAxis* M = axis_merged(a, m);
    return AxisDev{nullptr, nullptr, M->d_tab, M->d_tiles, M->K, M->ng, M->tile_bytes, M->ntiles};
  };
  auto tab_of = [](const ts_axis* a, int m) -> const std::vector<int32_t>& {
    return m <= 1 ? a->tab : axis_merged(a, m)->tab;
  };
  // operand rows / columns one tile's MMAs read: every (super-)block's K
  // window measured from the tile's first window start.  A merged window
  // spans the largest K_m of the axis, so a tile's last super-block can
  // reach past the unmerged span — the stage and the V tile must cover it
  // (else those MMA rows read neighbouring shared memory, times zero
  // weights: NaN if that memory holds a NaN pattern)
  auto tile_span = [](const ts_axis* a, int m, int per_tile, int ntiles) {
    const std::vector<int32_t>& ws = m <= 1 ? a->ws : axis_merged(a, m)->ws;
    const int K = m <= 1 ? a->K : axis_merged(a, m)->K;
    const int n = static_cast<int>(ws.size());
    int need = 0;
    for (int t = 0; t < ntiles && t * per_tile < n; ++t)
      for (int k = 0; k < per_tile && t * per_tile + k < n; ++k)
        need = std::max(need, ws[t * per_tile + k] + K - ws[t * per_tile]);
    return need;
  };
  P.nrt = (ra->nb + kRowBlocksPerTile - 1) / kRowBlocksPerTile;
  auto row_span_of = [&](int m) {
    return (tile_span(ra, m, kRowBlocksPerTile / m, P.nrt) + 15) / 16 * 16;
  };
  P.m1 = choose_merge(ra, kRowBlocksPerTile);
  if (P.m1 > 1 && row_span_of(P.m1) > kMaxRowSpan) P.m1 = 1;
  P.sb1 = kRowBlocksPerTile / P.m1;
  P.r = dev_of(ra, P.m1);
  P.R1 = row_span_of(P.m1);
  P.planes = planes;
  // widest column tile (most output blocks per staged V tile) that fits
  // smem; at each width try the chosen super-block merges first, then
  // unmerged axes (merged tiles are larger and may not fit resident)
  const int m1_best = P.m1;
  for (int nb2 = ca->col_nbt; nb2 >= 1; --nb2) {
    const int m2_best = choose_merge(ca, nb2);
    for (int variant = 0; variant < 3; ++variant) {
      const int m1 = variant == 2 ? 1 : m1_best;
      const int m2 = variant >= 1 ? 1 : m2_best;
      if (variant > 0 && m1 == m1_best && m2 == m2_best) continue;
      if (variant == 2 && m1_best == 1) continue;
      P.m1 = m1;
      P.sb1 = kRowBlocksPerTile / m1;
      P.r = dev_of(ra, m1);
      P.R1 = row_span_of(m1);
      P.nb2 = nb2;
      P.m2 = m2;
      P.sb2 = nb2 / m2;
      P.c = dev_of(ca, m2);
      P.nct = (ca->nb + nb2 - 1) / nb2;
      if (tile_span(ca, m2, P.sb2, P.nct) > kColTile) continue;  // windows past the V tile
      const std::vector<int32_t>& tr = tab_of(ra, m1);
      const std::vector<int32_t>& tc = tab_of(ca, m2);
      const int ntr = static_cast<int>(tr.size()), ntc = static_cast<int>(tc.size());
      P.ptab = (ntr + ntc <= kParamTab) ? 1 : 0;
      P.ptab_c = ntr;
      if (P.ptab) {
        for (int i = 0; i < ntr; ++i) P.tab[i] = tr[i];
        for (int i = 0; i < ntc; ++i) P.tab[ntr + i] = tc[i];
      }
      P.ntiles = planes * P.nrt * P.nct;
      if (plan_smem(P, oes)) {
        if (std::getenv("TSB_PLAN_VERBOSE"))  // the chosen plan, for debugging
          fprintf(stderr,
                  "separable plan: m1 %d sb1 %d K1 %d R1 %d | nb2 %d m2 %d sb2 %d K2 %d | ntiles r %d "
                  "c %d tb %d %d | nst %u nmid %u res %u off_w %u off_mid %u off_out %u off_bar %u "
                  "total %u\n",
                  P.m1, P.sb1, P.r.K, P.R1, P.nb2, P.m2, P.sb2, P.c.K, P.r.ntiles, P.c.ntiles,
                  P.r.tile_bytes, P.c.tile_bytes, P.L.nst, P.L.nmid, P.L.resident, P.L.off_w,
                  P.L.off_mid, P.L.off_out, P.L.off_bar, P.L.total);
        return TS_OK;
      }
    }
  }
  return set_error(TS_ERR_UNSUPPORTED, "separable: tile (R1=%d) does not fit smem", P.R1);
}

ts_status separable_run(const ts_axis* ra, const ts_axis* ca, int planes, const void* in,
                        int64_t in_rs, int64_t in_ps, int in_dtype, void* out, int64_t out_rs,
                        int64_t out_ps, int out_dtype, const ts_epilogue* ep, cudaStream_t stream) {
  if (!ra || !ca || !in || !out) return set_error(TS_ERR_INVALID, "separable: null argument");
  if (planes < 1) return set_error(TS_ERR_INVALID, "separable: planes must be >= 1");
  if (in_dtype != TS_BF16)
    return set_error(TS_ERR_UNSUPPORTED, "separable: input must be bf16 (cast f32 first)");
  if (out_dtype != TS_BF16 && out_dtype != TS_F32)
    return set_error(TS_ERR_UNSUPPORTED, "separable: output must be bf16 or f32");
  const int oes = out_dtype == TS_BF16 ? 2 : 4;
  if (in_rs < ca->n_in || (in_rs * 2) % 16 || in_ps < in_rs * ra->n_in || (in_ps * 2) % 16)
    return set_error(TS_ERR_INVALID, "separable: input strides (%lld, %lld) invalid for %d x %d",
                     (long long)in_rs, (long long)in_ps, ra->n_in, ca->n_in);
  if (out_rs < ca->n_out || (out_rs * oes) % 16 || out_ps < out_rs * ra->n_out ||
      (out_ps * oes) % 16)
    return set_error(TS_ERR_INVALID, "separable: output strides (%lld, %lld) invalid for %d x %d",
                     (long long)out_rs, (long long)out_ps, ra->n_out, ca->n_out);
  if (ra->device != ca->device)
    return set_error(TS_ERR_INVALID, "separable: axes live on devices %d and %d", ra->device,
                     ca->device);
  DeviceGuard guard(ra->device);
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");

  // launch parameters (block tables, smem plan) are cached per (axes, planes,
  // output size): rebuilding them costs more host time than a 1-frame launch
  struct Cached {
    uint64_t ru = 0, cu = 0;
    int planes = 0, oes = 0;
    SepParams P;
  };
  static thread_local Cached cache[4];
  static thread_local int cache_next = 0;
  Cached* hit = nullptr;
  for (auto& c : cache)
    if (c.ru == ra->uid && c.cu == ca->uid && c.planes == planes && c.oes == oes) hit = &c;
  if (!hit) {
    Cached& c = cache[cache_next];
    cache_next = (cache_next + 1) % 4;
    c.ru = 0;
    ts_status st = make_params(ra, ca, planes, oes, c.P);
    if (st != TS_OK) return st;
    c.ru = ra->uid;
    c.cu = ca->uid;
    c.planes = planes;
    c.oes = oes;
    hit = &c;
  }
  SepParams& P = hit->P;
  P.ep = make_epik(ep);
  // Tile order.  Static round-robin (CTA b takes tiles b, b + grid, ...)
  // keeps the ~grid tiles in flight contiguous, so neighbouring tiles share
  // their halo rows / columns in L2 — until the CTAs drift apart: beyond
  // ~128 tiles per CTA the in-flight set spreads, halos are evicted and DRAM
  // reads grow (48 frames of c2 in one launch: 1.68x algorithmic).  Long
  // launches therefore claim tiles in order from a counter (DRAM 1.00x at
  // any length); short ones keep the counter-free static order, which is a
  // few per cent faster there (c2, 16 frames: 0.848 vs 0.82 of HBM).
  // TSB_STATIC_TILES=1 / TSB_DYNAMIC_TILES=1 force either.
  static const bool force_static = std::getenv("TSB_STATIC_TILES") != nullptr;
  static const bool force_dynamic = std::getenv("TSB_DYNAMIC_TILES") != nullptr;
  const bool dynamic = !force_static &&
                       (force_dynamic || P.ntiles > 128 * sm_count_current());
  if (!dynamic || !claim_counters(ra->device, stream, &P.tile_next, &P.ctas_done)) {
    P.tile_next = nullptr;  // static round-robin tiles
    P.ctas_done = nullptr;
  }
  P.trace = g_trace;
  P.trace_ctas = g_trace_ctas;
  P.trace_tiles = g_trace_tiles;
  ts_status st;
  CUtensorMap tin, tout;
  st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, ca->n_in, ra->n_in, planes,
                      in_rs, in_ps, 64, P.R1 / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  st = encode_tmap_3d(&tout,
                      out_dtype == TS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                      oes, out, ca->n_out, ra->n_out, planes, out_rs, out_ps, P.nb2 * 16, 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TS_OK) return st;
  if (out_dtype == TS_BF16) return launch_sep<__nv_bfloat16>(P, tin, tout, stream, ep != nullptr);
  return launch_sep<float>(P, tin, tout, stream, ep != nullptr);
}

// The launch geometry a run would use (ts_separable_plan).
ts_status separable_plan(const ts_axis* ra, const ts_axis* ca, int planes, int out_dtype,
                         int* out8) {
  if (!ra || !ca || !out8) return set_error(TS_ERR_INVALID, "separable_plan: null argument");
  SepParams P;
  ts_status st = make_params(ra, ca, planes < 1 ? 1 : planes, out_dtype == TS_BF16 ? 2 : 4, P);
  if (st != TS_OK) return st;
  out8[0] = static_cast<int>(P.L.nst);
  out8[1] = static_cast<int>(P.L.nmid);
  out8[2] = static_cast<int>(P.L.resident);
  out8[3] = static_cast<int>(P.L.total);
  out8[4] = P.R1;
  out8[5] = P.nb2;
  out8[6] = P.ntiles;
  out8[7] = P.ntiles < sm_count_current() ? P.ntiles : sm_count_current();
  return TS_OK;
}

}  // namespace tsb

// dct16.cu — fused DCT-16 transform-domain denoise on sm_100a.
//
// Tiles of 16x16 at stride 8 (4 tiles cover every pixel), sine window folded
// into the transform matrix Dw = D·diag(w) (w[m]² + w[m+8]² = 1, so the
// windowed synthesis overlap-adds to the identity), coring in the transform
// domain (hard or soft threshold; DC kept), clamp-to-edge outside the image.
//
// One persistent CTA per SM; work unit = a 128x128 input band at image
// offset (Y-8, X-8) producing the 112x112 output block (Y.., X..).  The 16x16
// tiles of the band split into row phases p (tile rows at band row 8p+16i)
// and column phases q (8q+16j); for each p the kernel runs four tcgen05
// steps (M=128, N=16), choosing operand majors so no explicit transposes are
// needed:
//   S1 (SS, bf16)  D1[c][16i+k]   = Σ_r X[16i+8p+r][c] Dw[k][r]    A = band, MN-major
//   E1             D1 -> S_Y (bf16 hi + lo pair, MN-major: M = freq-row m, K = col)
//   S3 (SS, bf16)  D2[m][16(8q+j)+l] = Σ_c (Y_hi + Y_lo)[m][16j+8q+c] Dw[l][c]
//   E2             coring of D2 in TMEM (in place)
//   S5 (TS, tf32)  D3[m][16j+8q+c] += Σ_l C'[m][..+l] Dw[l][c]     A = D2 from TMEM
//   E3             D3 -> S_R (bf16 hi + lo, MN-major: M = col, K = freq-row)
//   S7 (SS, bf16)  D4[c][16i+8p+r] += Σ_k (R_hi + R_lo)[16i+k][c] Dw[k][r]  (both p accumulate)
// (kind::tf32 does not accept an MN-major A from shared memory on sm_100a —
// it silently yields zeros, see ts_probe_mma amode 3 — so f32 intermediates
// travel as bf16 hi/lo pairs, two MMAs per K step, ~16 mantissa bits.)
// and finally E4: D4 (lane = column, columns = band rows) -> bf16/f32 -> TMA
// store of the 112x112 block.  Steps run in sequence within a CTA (MMA warp
// and epilogue warpgroup hand off through mbarriers); the next band's TMA
// load overlaps the current band.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "common.h"
#include "sm100.cuh"

namespace tsb {

ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz);
int sm_count_current();

namespace dct {

constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kBand = 128;
constexpr int kOut = 112;
constexpr uint32_t kBandBytes = kBand * kBand * 2;  // bf16 band, two 64-col SW128 halves
constexpr uint32_t kOpBytes = 128 * 128 * 4;        // bf16 hi + lo operand (S_Y / S_R alias)
constexpr uint32_t kOpLo = 128 * 128 * 2;           // offset of the lo half

// smem layout (bytes from the 1024-aligned base)
constexpr uint32_t kOffX = 0;                           // 2 band buffers
constexpr uint32_t kOffOp = kOffX + 2 * kBandBytes;     // S_Y / S_R
constexpr uint32_t kOffOut = kOffOp + kOpBytes;         // 112 x 112 staging (f32 worst case)
constexpr uint32_t kOutBytes = kOut * kOut * 4;
constexpr uint32_t kOffB = kOffOut + ((kOutBytes + 1023) / 1024) * 1024;
// constant B tiles: bf16 Dwᵀ hi + lo (S1, S3: the steps whose rounding decides
// which coefficients are cored) in three edge variants each — 0 interior,
// 1 "low cut" (samples 0..7 lie outside the image: their weight is folded
// onto sample 8, clamp-to-edge), 2 "high cut" (8..15 outside, folded onto
// 7); TMA zero-fills the outside samples — then f32 Dw (S5), bf16 Dw (S7)
constexpr uint32_t kOffB1 = kOffB, kOffB1L = kOffB + 1536, kOffB5 = kOffB + 3072,
                   kOffB7 = kOffB + 4096;
constexpr uint32_t kConstBytes = 4608;
constexpr uint32_t kOffBar = kOffB + kConstBytes;
constexpr uint32_t kSmem = kOffBar + 256 + 1024;

struct Params {
  int planes, H, W, nry, nrx, nregions;
  float threshold;
  int soft;                 // 0 hard, 1 soft coring
  const uint8_t* consts;    // kConstBytes: the three B tiles in smem layout
  float* dbg;               // diagnostics: [4 stages][2 phases][128 lanes][256] for CTA 0, band 0
};

// Diagnostics: copy `ncols` TMEM columns of this thread's lane to dbg.
__device__ __forceinline__ void dbg_dump(const Params& P, int it, int stage, int p, uint32_t taddr,
                                         int row, int ncols) {
  if (P.dbg == nullptr || blockIdx.x != 0 || it != 0) return;
  float* dst = P.dbg + ((static_cast<size_t>(stage) * 2 + p) * 128 + row) * 256;
  for (int c0 = 0; c0 < ncols; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(taddr + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) dst[c0 + i] = __uint_as_float(r[i]);
  }
}

__device__ __forceinline__ void mma_tf32_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t b,
                                                  uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// bf16 MN-major 128B-swizzled operand: M = 128 (2 atoms of 64 at 16 KB),
// K = 128 (16 groups of 8 rows at 1 KB).  Address of the 16-byte chunk
// holding m = 8*m8 .. 8*m8+7 at K row k.
__device__ __forceinline__ uint32_t opbf_chunk(uint32_t base, int m8, int k) {
  return base + (m8 / 8) * 16384u + (k / 8) * 1024u + (k % 8) * 128u +
         ((((m8 % 8) ^ (k % 8))) * 16u);
}

// Write 16 consecutive-M f32 values of K row k as bf16 hi/lo pairs.
__device__ __forceinline__ void put_hilo16(uint32_t op_s, int m8_first, int k,
                                           const uint32_t (&r)[16]) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float a = __uint_as_float(r[8 * g + 2 * e]), b = __uint_as_float(r[8 * g + 2 * e + 1]);
      const __nv_bfloat16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
      hi[e] = pack_bf16x2(a, b);
      lo[e] = pack_bf16x2(a - __bfloat162float(ah), b - __bfloat162float(bh));
    }
    const uint32_t addr = opbf_chunk(op_s, m8_first + g, k);
    st_shared_v4(addr, hi[0], hi[1], hi[2], hi[3]);
    st_shared_v4(addr + kOpLo, lo[0], lo[1], lo[2], lo[3]);
  }
}

// Edge variant of a 16-sample tile starting at image coordinate x0 (multiple
// of 8) on an axis of length n (multiple of 8).
__device__ __forceinline__ uint32_t edge_variant(int x0, int n) {
  if (x0 < 0 && x0 + 16 > 0) return 1u;
  if (x0 < n && x0 + 16 > n) return 2u;
  return 0u;
}

struct Region {
  int p, ry, rx;
};

__device__ __forceinline__ Region region_of(const Params& P, int t) {
  Region r;
  r.rx = t % P.nrx;
  const int rest = t / P.nrx;
  r.ry = rest % P.nry;
  r.p = rest / P.nry;
  return r;
}

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    dct16_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                 const Params P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kOffBar);
  uint64_t* xfull = bars;        // [2]
  uint64_t* xempty = bars + 2;   // [2]
  uint64_t* b_s1 = bars + 4;
  uint64_t* b_s3 = bars + 5;
  uint64_t* b_s5 = bars + 6;
  uint64_t* b_s7 = bars + 7;
  uint64_t* e1 = bars + 8;
  uint64_t* e2 = bars + 9;
  uint64_t* e3 = bars + 10;
  uint64_t* e4 = bars + 11;
  uint64_t* cbar = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    mbar_init(b_s1, 1);
    mbar_init(b_s3, 1);
    mbar_init(b_s5, 1);
    mbar_init(b_s7, 1);
    mbar_init(e1, 128);
    mbar_init(e2, 128);
    mbar_init(e3, 128);
    mbar_init(e4, 128);
    mbar_init(cbar, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_in);
    prefetch_tmap(&tm_out);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: [0,256) D1 / D2, [256,384) D3, [384,512) D4
  const uint32_t tD1 = tmem, tD2 = tmem, tD3 = tmem + 256u, tD4 = tmem + 384u;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(cbar, kConstBytes);
      bulk_g2s(base + kOffB, P.consts, kConstBytes, cbar);
      int it = 0;
      for (int t = blockIdx.x; t < P.nregions; t += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&xempty[s], ((it >> 1) & 1) ^ 1);
        const Region R = region_of(P, t);
        const int Y = R.ry * kOut, X = R.rx * kOut;
        mbar_arrive_expect_tx(&xfull[s], kBandBytes);
        uint8_t* dst = base + kOffX + s * kBandBytes;
        tma_load_3d(dst, &tm_in, &xfull[s], X - 8, Y - 8, R.p);
        tma_load_3d(dst + kBand * 128, &tm_in, &xfull[s], X - 8 + 64, Y - 8, R.p);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id_bf = make_idesc(kFmtBF16, 128, 16, /*A MN*/ 1, 0);
    const uint32_t id_tf_k = make_idesc(kFmtTF32, 128, 16, 0, 0);
    // B descriptors (K-major, no swizzle): bf16 16x16 (LBO 128, SBO 256);
    // f32 16x16 (core matrices 8 n x 4 k: LBO 128, SBO 512)
    const uint64_t bd1 = make_sdesc(base_s + kOffB1, 128u, 256u, kSwizzleNone);
    const uint64_t bd1l = make_sdesc(base_s + kOffB1L, 128u, 256u, kSwizzleNone);
    const uint64_t bd5 = make_sdesc(base_s + kOffB5, 128u, 512u, kSwizzleNone);
    const uint64_t bd7 = make_sdesc(base_s + kOffB7, 128u, 256u, kSwizzleNone);
    const uint32_t op_s = base_s + kOffOp;
    mbar_wait(cbar, 0);
    int it = 0;
    uint32_t ph_e = 0;  // phase of e1/e2/e3 (each completes twice per region)
    for (int t = blockIdx.x; t < P.nregions; t += gridDim.x, ++it) {
      const int s = it & 1;
      const Region R = region_of(P, t);
      const int Y = R.ry * kOut, X = R.rx * kOut;
      mbar_wait(&xfull[s], (it >> 1) & 1);
      const uint32_t band_s = base_s + kOffX + s * kBandBytes;
      for (int p = 0; p < 2; ++p) {
        const int ni = p == 0 ? 8 : 7;
        // ---- S1: column forward (A = band MN-major: M = cols, K = rows)
        if (p == 1) mbar_wait(b_s7, 0 ^ (static_cast<uint32_t>(it * 2) & 1));  // S7_0 done: S_R free
        tc_fence_after();
        for (int i = 0; i < ni; ++i) {
          const uint64_t ad =
              make_sdesc(band_s + (16u * i + 8u * p) * 128u, kBand * 128u, 1024u, kSwizzle128B);
          const uint32_t v = edge_variant(Y - 8 + 16 * i + 8 * p, P.H);
          mma_f16_ss_elect(tD1 + 16u * i, ad, bd1 + 32u * v, id_bf, 0u);
          mma_f16_ss_elect(tD1 + 16u * i, ad, bd1l + 32u * v, id_bf, 1u);
        }
        mma_commit_elect(b_s1);
        if (p == 1) mma_commit_elect(&xempty[s]);
        // ---- S3: row forward (A = S_Y hi/lo MN-major: M = freq-row, K = col)
        mbar_wait(e1, ph_e);
        tc_fence_after();
        for (int q = 0; q < 2; ++q) {
          const int nj = q == 0 ? 8 : 7;
          for (int j = 0; j < nj; ++j) {
            const uint32_t kc = 16u * j + 8u * q;  // first column of the tile
            const uint64_t ad = make_sdesc(op_s + (kc / 8u) * 1024u, 16384u, 1024u, kSwizzle128B);
            const uint64_t adl =
                make_sdesc(op_s + kOpLo + (kc / 8u) * 1024u, 16384u, 1024u, kSwizzle128B);
            const uint32_t v = edge_variant(X - 8 + static_cast<int>(kc), P.W);
            mma_f16_ss_elect(tD2 + 16u * (8 * q + j), ad, bd1 + 32u * v, id_bf, 0u);
            mma_f16_ss_elect(tD2 + 16u * (8 * q + j), adl, bd1 + 32u * v, id_bf, 1u);
            mma_f16_ss_elect(tD2 + 16u * (8 * q + j), ad, bd1l + 32u * v, id_bf, 1u);
          }
        }
        mma_commit_elect(b_s3);
        // ---- S5: row inverse (A = cored D2 from TMEM, K = freq l)
        mbar_wait(e2, ph_e);
        tc_fence_after();
        for (int q = 0; q < 2; ++q) {
          const int nj = q == 0 ? 8 : 7;
          for (int j = 0; j < nj; ++j) {
            const uint32_t c0 = 16u * j + 8u * q;
            for (int h = 0; h < 2; ++h)
              mma_tf32_ts_elect(tD3 + c0, tD2 + 16u * (8 * q + j) + 8u * h, bd5 + 16u * h,
                                id_tf_k, (q > 0 || h > 0) ? 1u : 0u);
          }
        }
        mma_commit_elect(b_s5);
        // ---- S7: column inverse (A = S_R hi/lo MN-major: M = col, K = freq-row)
        mbar_wait(e3, ph_e);
        if (p == 0 && it > 0) mbar_wait(e4, (it - 1) & 1);  // previous E4 read D4
        tc_fence_after();
        for (int i = 0; i < ni; ++i) {
          const uint64_t ad = make_sdesc(op_s + (2u * i) * 1024u, 16384u, 1024u, kSwizzle128B);
          const uint64_t adl =
              make_sdesc(op_s + kOpLo + (2u * i) * 1024u, 16384u, 1024u, kSwizzle128B);
          mma_f16_ss_elect(tD4 + 16u * i + 8u * p, ad, bd7, id_bf, p > 0 ? 1u : 0u);
          mma_f16_ss_elect(tD4 + 16u * i + 8u * p, adl, bd7, id_bf, 1u);
        }
        mma_commit_elect(b_s7);
        ph_e ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2-5)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t op_s = base_s + kOffOp;
    const int et = threadIdx.x - 64;
    int it = 0;
    uint32_t ph = 0;  // phase of b_s1/b_s3/b_s5/b_s7 (each completes twice per region)
    for (int t = blockIdx.x; t < P.nregions; t += gridDim.x, ++it) {
      const Region R = region_of(P, t);
      const int Y = R.ry * kOut, X = R.rx * kOut;
      for (int p = 0; p < 2; ++p) {
        // ---- E1: D1 (lane = col c) -> S_Y[m][c] f32 MN-major (M = m, K = c)
        mbar_wait(b_s1, ph);
        tc_fence_after();
        dbg_dump(P, it, 0, p, tD1 + lane_off, row, 128);
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t r[16];
          tmem_ld16(tD1 + lane_off + 16u * ch, r);
          tmem_wait_ld();
          put_hilo16(op_s, 2 * ch, row, r);  // M = freq-row 16ch.., K = this column
        }
        tc_fence_before();
        fence_proxy_async_smem();
        mbar_arrive(e1);
        // ---- E2: coring of D2 (lane = freq-row m, cols = 16*(8q+j) + l) in place
        mbar_wait(b_s3, ph);
        tc_fence_after();
        dbg_dump(P, it, 1, p, tD2 + lane_off, row, 240);
        for (int ch = 0; ch < 15; ++ch) {
          uint32_t r[16];
          tmem_ld16(tD2 + lane_off + 16u * ch, r);
          tmem_wait_ld();
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            float v = __uint_as_float(r[l]);
            const bool dc = (row % 16 == 0) && (l == 0);
            if (!dc) {
              if (P.soft)
                v = copysignf(fmaxf(fabsf(v) - P.threshold, 0.0f), v);
              else if (fabsf(v) < P.threshold)
                v = 0.0f;
            }
            r[l] = __float_as_uint(v);
          }
          tmem_st16(tD2 + lane_off + 16u * ch, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(e2);
        // ---- E3: D3 (lane = m, cols = band col c) -> S_R[c][m] f32 MN-major (M = c, K = m)
        mbar_wait(b_s5, ph);
        tc_fence_after();
        dbg_dump(P, it, 2, p, tD3 + lane_off, row, 128);
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t r[16];
          tmem_ld16(tD3 + lane_off + 16u * ch, r);
          tmem_wait_ld();
          put_hilo16(op_s, 2 * ch, row, r);  // M = band col 16ch.., K = this freq-row
        }
        tc_fence_before();
        fence_proxy_async_smem();
        mbar_arrive(e3);
        // next phase's E1 overwrites S_Y = S_R: wait for S7 of this phase
        mbar_wait(b_s7, ph);
        ph ^= 1;
      }
      // ---- E4: D4 (lane = band col c, cols = band row) -> output block
      tc_fence_after();
      dbg_dump(P, it, 3, 0, tD4 + lane_off, row, 128);
      if (et == 0) bulk_wait_read0();
      named_bar_sync(1, 128);
      OutT* stg = reinterpret_cast<OutT*>(base + kOffOut);
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t r[16];
        tmem_ld16(tD4 + lane_off + 16u * ch, r);
        tmem_wait_ld();
        if (row >= 8 && row < 8 + kOut) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int br = ch * 16 + e;
            if (br >= 8 && br < 8 + kOut) {
              const float v = __uint_as_float(r[e]);
              if constexpr (sizeof(OutT) == 2)
                stg[(br - 8) * kOut + (row - 8)] = __float2bfloat16_rn(v);
              else
                stg[(br - 8) * kOut + (row - 8)] = v;
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(e4);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (et == 0) {
        tma_store_3d(&tm_out, stg, X, Y, R.p);
        bulk_commit();
      }
    }
    if (et == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace dct

static float* g_dct_dbg = nullptr;
void dct_set_debug(float* p) { g_dct_dbg = p; }

// Host: the constant B tiles in their smem byte layout.
static void build_consts(uint8_t* out) {
  double D[16][16], w[16];
  for (int m = 0; m < 16; ++m) w[m] = std::sin(3.14159265358979323846 * (m + 0.5) / 16.0);
  for (int k = 0; k < 16; ++k)
    for (int m = 0; m < 16; ++m)
      D[k][m] = std::cos(3.14159265358979323846 * (2 * m + 1) * k / 32.0) *
                std::sqrt((k == 0 ? 1.0 : 2.0) / 16.0) * w[m];
  auto bf16_bits = [](double v) {
    const float f = static_cast<float>(v);
    uint32_t b;
    std::memcpy(&b, &f, 4);
    return static_cast<uint16_t>((static_cast<uint64_t>(b) + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
  };
  auto bf16_val = [](uint16_t h) {
    const uint32_t b = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return static_cast<double>(f);
  };
  // lo = 0: bf16(v); lo = 1: bf16(v - bf16(v))
  auto put16 = [&](uint8_t* dst, int kk, int n, double v, int lo) {
    uint16_t h = bf16_bits(v);
    if (lo) h = bf16_bits(v - bf16_val(h));
    std::memcpy(dst + (n / 8) * 256 + (kk / 8) * 128 + (n % 8) * 16 + (kk % 8) * 2, &h, 2);
  };
  // f32 K-major core matrices (8 n x 4 k): (n/8)*512 + (k/4)*128 + (n%8)*16 + (k%4)*4
  auto put32 = [&](uint8_t* dst, int kk, int n, double v) {
    const float f = static_cast<float>(v);
    std::memcpy(dst + (n / 8) * 512 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4, &f, 4);
  };
  for (int v = 0; v < 3; ++v) {
    // B1[K = sample][N = freq] = Dw[freq][sample], edge-folded (variant v)
    double F[16][16];
    for (int n = 0; n < 16; ++n)
      for (int kk = 0; kk < 16; ++kk) F[n][kk] = D[n][kk];
    for (int n = 0; n < 16; ++n) {
      if (v == 1) {
        for (int kk = 0; kk < 8; ++kk) { F[n][8] += F[n][kk]; F[n][kk] = 0; }
      } else if (v == 2) {
        for (int kk = 8; kk < 16; ++kk) { F[n][7] += F[n][kk]; F[n][kk] = 0; }
      }
    }
    for (int kk = 0; kk < 16; ++kk)
      for (int n = 0; n < 16; ++n) {
        put16(out + 512 * v, kk, n, F[n][kk], 0);         // hi
        put16(out + 1536 + 512 * v, kk, n, F[n][kk], 1);  // lo
      }
  }
  for (int kk = 0; kk < 16; ++kk)
    for (int n = 0; n < 16; ++n) {
      put32(out + 3072, kk, n, D[kk][n]);    // B5[K=l][N=c] = Dw[l][c] (S5, f32)
      put16(out + 4096, kk, n, D[kk][n], 0); // B7[K=k][N=r] = Dw[k][r] (S7)
    }
}

ts_status dct16_run(const void* in, int64_t in_rs, int64_t in_ps, int in_dtype, void* out,
                    int64_t out_rs, int64_t out_ps, int out_dtype, int planes, int H, int W,
                    float threshold, int soft, cudaStream_t stream) {
  if (!in || !out || planes < 1 || H < 8 || W < 8)
    return set_error(TS_ERR_INVALID, "dct16: bad arguments");
  if (H % 8 || W % 8) return set_error(TS_ERR_UNSUPPORTED, "dct16: H and W must be multiples of 8");
  if (in_dtype != TS_BF16) return set_error(TS_ERR_UNSUPPORTED, "dct16: input must be bf16");
  if (out_dtype != TS_BF16 && out_dtype != TS_F32)
    return set_error(TS_ERR_UNSUPPORTED, "dct16: output must be bf16 or f32");
  const int oes = out_dtype == TS_BF16 ? 2 : 4;
  if (in_rs < W || (in_rs * 2) % 16 || in_ps < in_rs * H || (in_ps * 2) % 16 || out_rs < W ||
      (out_rs * oes) % 16 || out_ps < out_rs * H || (out_ps * oes) % 16)
    return set_error(TS_ERR_INVALID, "dct16: strides");
  static uint8_t* d_consts[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(TS_ERR_INVALID, "dct16: device index");
  if (!d_consts[dev]) {
    uint8_t h[dct::kConstBytes] = {0};
    build_consts(h);
    cudaError_t e = cudaMalloc(&d_consts[dev], dct::kConstBytes);
    if (e != cudaSuccess) return cuda_error(e, "dct16 consts");
    e = cudaMemcpy(d_consts[dev], h, dct::kConstBytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_error(e, "dct16 consts copy");
  }
  dct::Params P;
  P.planes = planes;
  P.H = H;
  P.W = W;
  P.nry = (H + dct::kOut - 1) / dct::kOut;
  P.nrx = (W + dct::kOut - 1) / dct::kOut;
  P.nregions = planes * P.nry * P.nrx;
  P.threshold = threshold;
  P.soft = soft;
  P.consts = d_consts[dev];
  P.dbg = g_dct_dbg;
  CUtensorMap tin, tout;
  ts_status st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, W, H, planes, in_rs,
                                in_ps, 64, dct::kBand, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  st = encode_tmap_3d(&tout,
                      out_dtype == TS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                      oes, out, W, H, planes, out_rs, out_ps, dct::kOut, dct::kOut,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TS_OK) return st;
  const int sms = sm_count_current();
  const int grid = P.nregions < sms ? P.nregions : sms;
  cudaError_t e;
  if (out_dtype == TS_BF16) {
    e = cudaFuncSetAttribute(dct::dct16_kernel<__nv_bfloat16>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, dct::kSmem);
    if (e == cudaSuccess)
      dct::dct16_kernel<__nv_bfloat16><<<grid, dct::kThreads, dct::kSmem, stream>>>(tin, tout, P);
  } else {
    e = cudaFuncSetAttribute(dct::dct16_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dct::kSmem);
    if (e == cudaSuccess)
      dct::dct16_kernel<float><<<grid, dct::kThreads, dct::kSmem, stream>>>(tin, tout, P);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "dct16 launch");
}

}  // namespace tsb

extern "C" ts_status ts_debug_dct16(float* device_buffer) {
  tsb::dct_set_debug(device_buffer);
  return TS_OK;
}

extern "C" ts_status ts_denoise_dct16(const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                                      int in_dtype, void* out, int64_t out_row_stride,
                                      int64_t out_plane_stride, int out_dtype, int planes, int height,
                                      int width, float threshold, int soft, void* stream) {
  return tsb::dct16_run(in, in_row_stride, in_plane_stride, in_dtype, out, out_row_stride,
                        out_plane_stride, out_dtype, planes, height, width, threshold, soft,
                        static_cast<cudaStream_t>(stream));
}

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
//   E1             D1 -> S_Y (f32, MN-major: M = freq-row m, K = col)
//   S3 (SS, tf32)  D2[m][16(8q+j)+l] = Σ_c Y[m][16j+8q+c] Dw[l][c]
//   E2             coring of D2 in TMEM (in place)
//   S5 (TS, tf32)  D3[m][16j+8q+c] += Σ_l C'[m][..+l] Dw[l][c]     A = D2 from TMEM
//   E3             D3 -> S_R (f32, MN-major: M = col, K = freq-row)
//   S7 (SS, tf32)  D4[c][16i+8p+r] += Σ_k R[16i+k][c] Dw[k][r]     (both p accumulate)
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
constexpr uint32_t kOpBytes = 128 * 128 * 4;        // f32 operand (S_Y / S_R alias)

// smem layout (bytes from the 1024-aligned base)
constexpr uint32_t kOffX = 0;                           // 2 band buffers
constexpr uint32_t kOffOp = kOffX + 2 * kBandBytes;     // S_Y / S_R
constexpr uint32_t kOffOut = kOffOp + kOpBytes;         // 112 x 112 staging (f32 worst case)
constexpr uint32_t kOutBytes = kOut * kOut * 4;
constexpr uint32_t kOffB = kOffOut + ((kOutBytes + 1023) / 1024) * 1024;
// constant B tiles: [0] bf16 Dwᵀ (512 B), [1] f32 Dwᵀ (1 KB), [2] f32 Dw (1 KB)
constexpr uint32_t kOffB1 = kOffB, kOffB3 = kOffB + 512, kOffB5 = kOffB + 1536;
constexpr uint32_t kOffBar = kOffB + 2560;
constexpr uint32_t kSmem = kOffBar + 256 + 1024;

struct Params {
  int planes, H, W, nry, nrx, nregions;
  float threshold;
  int soft;                 // 0 hard, 1 soft coring
  const uint8_t* consts;    // 2560 bytes: the three B tiles in smem layout
};

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

// f32 MN-major 128B-swizzled operand: M = 128 (4 atoms of 32), K = 128 (16
// groups of 8 at 1 KB); element (m, k)
__device__ __forceinline__ uint32_t opf32_chunk(uint32_t base, int m4, int k) {
  // address of the 16-byte chunk holding m = 4*m4 .. 4*m4+3 at row k
  return base + (m4 / 8) * 16384u + (k / 8) * 1024u + (k % 8) * 128u +
         ((((m4 % 8) ^ (k % 8))) * 16u);
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

// Replicate the image edge into the out-of-image rows/cols of a band
// (TMA zero-filled them).  band row b <-> image row Y-8+b, col c <-> X-8+c.
__device__ void fixup_band(uint8_t* band, int Y, int X, int H, int W, int lane) {
  auto at = [&](int r, int c) -> __nv_bfloat16* {
    const int half = c / 64, cc = c % 64;
    const uint32_t off = half * (kBand * 128u) + r * 128u + ((((cc / 8) ^ (r % 8))) * 16u) +
                         (cc % 8) * 2u;
    return reinterpret_cast<__nv_bfloat16*>(band + off);
  };
  const int r_lo = max(0, 8 - Y);                        // first band row inside the image
  const int r_hi = min(kBand, H - (Y - 8));              // one past the last
  const int c_lo = max(0, 8 - X);
  const int c_hi = min(kBand, W - (X - 8));
  if (r_lo == 0 && r_hi == kBand && c_lo == 0 && c_hi == kBand) return;
  // columns first (rows inside the image), then full rows from the nearest valid row
  for (int e = lane; e < kBand * kBand; e += 32) {
    const int r = e / kBand, c = e % kBand;
    if (r < r_lo || r >= r_hi) continue;
    if (c < c_lo) *at(r, c) = *at(r, c_lo);
    else if (c >= c_hi) *at(r, c) = *at(r, c_hi - 1);
  }
  __syncwarp();
  for (int e = lane; e < kBand * kBand; e += 32) {
    const int r = e / kBand, c = e % kBand;
    if (r < r_lo) *at(r, c) = *at(r_lo, c);
    else if (r >= r_hi) *at(r, c) = *at(r_hi - 1, c);
  }
  __syncwarp();
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
      mbar_arrive_expect_tx(cbar, 2560);
      bulk_g2s(base + kOffB, P.consts, 2560, cbar);
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
    const uint32_t id_tf_mn = make_idesc(kFmtTF32, 128, 16, 1, 0);
    const uint32_t id_tf_k = make_idesc(kFmtTF32, 128, 16, 0, 0);
    // B descriptors (K-major, no swizzle): bf16 16x16 (LBO 128, SBO 256);
    // f32 16x16 (core matrices 8 n x 4 k: LBO 128, SBO 512)
    const uint64_t bd1 = make_sdesc(base_s + kOffB1, 128u, 256u, kSwizzleNone);
    const uint64_t bd3 = make_sdesc(base_s + kOffB3, 128u, 512u, kSwizzleNone);
    const uint64_t bd5 = make_sdesc(base_s + kOffB5, 128u, 512u, kSwizzleNone);
    const uint32_t op_s = base_s + kOffOp;
    mbar_wait(cbar, 0);
    int it = 0;
    uint32_t ph_e = 0;  // phase of e1/e2/e3 (each completes twice per region)
    for (int t = blockIdx.x; t < P.nregions; t += gridDim.x, ++it) {
      const int s = it & 1;
      const Region R = region_of(P, t);
      const int Y = R.ry * kOut, X = R.rx * kOut;
      mbar_wait(&xfull[s], (it >> 1) & 1);
      uint8_t* band = base + kOffX + s * kBandBytes;
      fixup_band(band, Y, X, P.H, P.W, lane);
      fence_proxy_async_smem();
      __syncwarp();
      const uint32_t band_s = base_s + kOffX + s * kBandBytes;
      for (int p = 0; p < 2; ++p) {
        const int ni = p == 0 ? 8 : 7;
        // ---- S1: column forward (A = band MN-major: M = cols, K = rows)
        if (p == 1) mbar_wait(b_s7, 0 ^ (static_cast<uint32_t>(it * 2) & 1));  // S7_0 done: S_R free
        tc_fence_after();
        for (int i = 0; i < ni; ++i) {
          const uint64_t ad =
              make_sdesc(band_s + (16u * i + 8u * p) * 128u, kBand * 128u, 1024u, kSwizzle128B);
          mma_f16_ss_elect(tD1 + 16u * i, ad, bd1, id_bf, 0u);
        }
        mma_commit_elect(b_s1);
        if (p == 1) mma_commit_elect(&xempty[s]);
        // ---- S3: row forward (A = S_Y f32 MN-major: M = freq-row, K = col)
        mbar_wait(e1, ph_e);
        tc_fence_after();
        for (int q = 0; q < 2; ++q) {
          const int nj = q == 0 ? 8 : 7;
          for (int j = 0; j < nj; ++j) {
            const uint32_t kc = 16u * j + 8u * q;  // first column of the tile
            for (int h = 0; h < 2; ++h) {
              const uint64_t ad =
                  make_sdesc(op_s + ((kc / 8u) + h) * 1024u, 16384u, 1024u, kSwizzle128B);
              mma_tf32_ss_elect(tD2 + 16u * (8 * q + j), ad, bd3 + 16u * h, id_tf_mn,
                                h ? 1u : 0u);
            }
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
        // ---- S7: column inverse (A = S_R f32 MN-major: M = col, K = freq-row)
        mbar_wait(e3, ph_e);
        if (p == 0 && it > 0) mbar_wait(e4, (it - 1) & 1);  // previous E4 read D4
        tc_fence_after();
        for (int i = 0; i < ni; ++i) {
          for (int h = 0; h < 2; ++h) {
            const uint64_t ad =
                make_sdesc(op_s + (2u * i + h) * 1024u, 16384u, 1024u, kSwizzle128B);
            mma_tf32_ss_elect(tD4 + 16u * i + 8u * p, ad, bd5 + 16u * h, id_tf_mn,
                              (p > 0 || h > 0) ? 1u : 0u);
          }
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
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t r[16];
          tmem_ld16(tD1 + lane_off + 16u * ch, r);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g)
            st_shared_v4(opf32_chunk(op_s, ch * 4 + g, row), r[4 * g], r[4 * g + 1], r[4 * g + 2],
                         r[4 * g + 3]);
        }
        tc_fence_before();
        fence_proxy_async_smem();
        mbar_arrive(e1);
        // ---- E2: coring of D2 (lane = freq-row m, cols = 16*(8q+j) + l) in place
        mbar_wait(b_s3, ph);
        tc_fence_after();
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
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t r[16];
          tmem_ld16(tD3 + lane_off + 16u * ch, r);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 4; ++g)
            st_shared_v4(opf32_chunk(op_s, ch * 4 + g, row), r[4 * g], r[4 * g + 1], r[4 * g + 2],
                         r[4 * g + 3]);
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

// Host: the constant B tiles in their smem byte layout.
static void build_consts(uint8_t* out) {
  double D[16][16], w[16];
  for (int m = 0; m < 16; ++m) w[m] = std::sin(3.14159265358979323846 * (m + 0.5) / 16.0);
  for (int k = 0; k < 16; ++k)
    for (int m = 0; m < 16; ++m)
      D[k][m] = std::cos(3.14159265358979323846 * (2 * m + 1) * k / 32.0) *
                std::sqrt((k == 0 ? 1.0 : 2.0) / 16.0) * w[m];
  // [0,512): bf16 B1[K=r][N=k] = Dw[k][r], K-major core matrices (8 n x 8 k)
  for (int kk = 0; kk < 16; ++kk)
    for (int n = 0; n < 16; ++n) {
      const float v = static_cast<float>(D[n][kk]);
      uint32_t b;
      std::memcpy(&b, &v, 4);
      const uint16_t h = static_cast<uint16_t>((static_cast<uint64_t>(b) + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
      const int off = (n / 8) * 256 + (kk / 8) * 128 + (n % 8) * 16 + (kk % 8) * 2;
      std::memcpy(out + off, &h, 2);
    }
  // f32 K-major core matrices (8 n x 4 k): (n/8)*512 + (k/4)*128 + (n%8)*16 + (k%4)*4
  auto put32 = [&](uint8_t* dst, int kk, int n, double v) {
    const float f = static_cast<float>(v);
    std::memcpy(dst + (n / 8) * 512 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4, &f, 4);
  };
  for (int kk = 0; kk < 16; ++kk)
    for (int n = 0; n < 16; ++n) {
      put32(out + 512, kk, n, D[n][kk]);   // B3[K=c][N=l] = Dw[l][c]
      put32(out + 1536, kk, n, D[kk][n]);  // B5[K=l][N=c] = Dw[l][c]
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
    uint8_t h[2560] = {0};
    build_consts(h);
    cudaError_t e = cudaMalloc(&d_consts[dev], 2560);
    if (e != cudaSuccess) return cuda_error(e, "dct16 consts");
    e = cudaMemcpy(d_consts[dev], h, 2560, cudaMemcpyHostToDevice);
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

extern "C" ts_status ts_denoise_dct16(const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                                      int in_dtype, void* out, int64_t out_row_stride,
                                      int64_t out_plane_stride, int out_dtype, int planes, int height,
                                      int width, float threshold, int soft, void* stream) {
  return tsb::dct16_run(in, in_row_stride, in_plane_stride, in_dtype, out, out_row_stride,
                        out_plane_stride, out_dtype, planes, height, width, threshold, soft,
                        static_cast<cudaStream_t>(stream));
}

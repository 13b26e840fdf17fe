// axis_pass.cu — one banded axis applied along rows or columns of planar
// images, for geometries the fused separable kernel cannot tile (windows of
// more than ~128-512 inputs per 16 outputs: large downscale factors, very
// wide filters).  A resample then runs as two passes with a
// bf16 intermediate in HBM (the same rounding point as the fused kernel's V):
//
//   vertical   mid[p][o][c] = Σ_k R[o][k] in[p][k][c]
//              A = 16 input rows x 128 columns per K-step (TMA, MN-major,
//              128B swizzle), B = the block's K x 16 weight tile,
//              D (TMEM) lane = column, 16 outputs
//   horizontal out[p][r][j] = Σ_k mid[p][r][k] C[j][k]
//              A = 128 rows x 16 columns per K-step (TMA, K-major core
//              matrices), B = the block's weight tile, D lane = row
//
// One CTA per (plane, group of up to 8 16-output blocks, 128-wide strip);
// each block's K window streams through an 8-slot TMA ring with no upper
// bound on its length (windows up to 1024 inputs, i.e. ~45x downscale), the
// blocks accumulate into adjacent 16-column TMEM slices and leave in one TMA
// store.  Several CTAs share an SM (the ring depth, group size and TMEM
// columns are sized per pass so that loads from many CTAs overlap).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "common.h"
#include "sm100.cuh"

namespace tsb {

ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz);

namespace apass {

constexpr int kThreads = 128;
// ring slot: vertical = one K-step (16 rows x 128 columns, two 64-column
// boxes); horizontal = four K-steps (128 rows x 64 columns, one 128B-swizzled
// K-major box: 128-byte rows keep the TMA efficient)
template <bool VERT>
struct Ring {
  static constexpr int kSlots = VERT ? 6 : 4;
  static constexpr uint32_t kSlot = VERT ? 4096u : 16384u;
  static constexpr int kSteps = VERT ? 1 : 4;  // K-steps per slot
};

struct Params {
  AxisDev ax;
  int planes, nb, nstrip;  // blocks along the axis, 128-wide strips across it
  int nbg, ngroups;        // blocks per CTA (<= 8) and block groups
  int nunits;
  uint32_t tmem_cols;  // accumulator columns: 16 per block, power of two >= 32
  int nring;  // ring slots in use (<= Ring::kSlots): a group never needs more than it loads
  uint32_t off_b, off_out, off_bar;
  EpiK ep;  // output epilogue (EPI kernels only)
};

template <bool VERT, typename OutT, bool EPI>
__global__ void __launch_bounds__(kThreads)
    axis_pass_kernel(const __grid_constant__ CUtensorMap tm_in,
                     const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ Params P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const uint32_t tile_bytes = static_cast<uint32_t>(P.ax.tile_bytes);
  // [ring][B tiles of the group][staging][barriers]
  using RG = Ring<VERT>;
  constexpr int kRing = RG::kSlots;  // barrier array size
  const int nring = P.nring;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kRing;
  uint64_t* wbar = bars + 2 * kRing;
  uint64_t* done = wbar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int u = blockIdx.x;
  const int strip = u % P.nstrip;
  const int g = (u / P.nstrip) % P.ngroups;
  const int p = u / (P.nstrip * P.ngroups);
  const int b0 = g * P.nbg;
  const int nblk = min(P.nbg, P.nb - b0);
  const int nq = P.ax.K / 16;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(wbar, 1);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_n(tmem_slot, P.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(wbar, tile_bytes * nblk);
      for (int j = 0; j < nblk; ++j) {
        const int tid = __ldg(P.ax.tid + b0 + j);
        bulk_g2s(base + P.off_b + j * tile_bytes, P.ax.tiles + static_cast<size_t>(tid) * tile_bytes,
                 tile_bytes, wbar);
      }
      int s = 0;
      uint32_t ph = 0;
      const int nslot = (nq + RG::kSteps - 1) / RG::kSteps;
      for (int j = 0; j < nblk; ++j) {
        const int ws = __ldg(P.ax.ws + b0 + j);  // window start (may be negative)
        for (int q = 0; q < nslot; ++q) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], RG::kSlot);
          uint8_t* dst = base + s * RG::kSlot;
          if (VERT) {  // rows ws+16q.., columns 128*strip.. as two 64-column boxes
            tma_load_3d(dst, &tm_in, &full[s], 128 * strip, ws + 16 * q, p);
            tma_load_3d(dst + 2048, &tm_in, &full[s], 128 * strip + 64, ws + 16 * q, p);
          } else {     // rows 128*strip.., columns ws+64q.. as one 64-column box
            tma_load_3d(dst, &tm_in, &full[s], ws + 64 * q, 128 * strip, p);
          }
          if (++s == nring) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, 16, VERT ? 1u : 0u, 0u);
    const uint64_t bd0 = make_sdesc(base_s + P.off_b, 128u, static_cast<uint32_t>(P.ax.K) * 16u,
                                    kSwizzleNone);
    // vertical: MN-major SW128 (64-column atoms 2 KB apart, 8-row groups at
    // 1 KB); horizontal: K-major SW128 (8-row groups at 1 KB, K-steps are
    // 32-byte advances inside the swizzle atom)
    const uint64_t ad0 = VERT ? make_sdesc(base_s, 2048u, 1024u, kSwizzle128B)
                              : make_sdesc(base_s, 16u, 1024u, kSwizzle128B);
    mbar_wait(wbar, 0);
    int s = 0;
    uint32_t ph = 0;
    for (int j = 0; j < nblk; ++j) {
      const uint64_t bdj = bd0 + static_cast<uint64_t>(j * (tile_bytes >> 4));
      for (int q0 = 0; q0 < nq; q0 += RG::kSteps) {
        mbar_wait(&full[s], ph);
        __syncwarp();
        tc_fence_after();
        const uint64_t ads = ad0 + static_cast<uint64_t>(s * (RG::kSlot >> 4));
#pragma unroll
        for (int u = 0; u < RG::kSteps; ++u) {
          const int q = q0 + u;
          if (q < nq)
            mma_f16_ss_elect(tmem + 16u * j, ads + static_cast<uint64_t>(u * 2), bdj + 16u * q,
                             idesc, q > 0 ? 1u : 0u);
        }
        mma_commit_elect(&empty[s]);
        if (++s == nring) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    mma_commit_elect(done);
  }
  // epilogue: all four warps (lane = TMEM row)
  mbar_wait(done, 0);
  __syncwarp();  // reconverge warp 0 (lane 0 ran the producer loop)
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  OutT* stg = reinterpret_cast<OutT*>(base + P.off_out);
#pragma unroll 1
  for (int j = 0; j < nblk; ++j) {
    uint32_t r[16];
    tmem_ld16(tl + 16u * j, r);
    tmem_wait_ld();
    if constexpr (EPI) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(epi_f32(P.ep, __uint_as_float(r[i])));
    }
    if (VERT) {  // lane = column c, values = 16 output rows: staging [nout][128]
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float v = __uint_as_float(r[i]);
        if constexpr (sizeof(OutT) == 2)
          stg[(16 * j + i) * 128 + row] = __float2bfloat16_rn(v);
        else
          stg[(16 * j + i) * 128 + row] = v;
      }
    } else {     // lane = row r, values = 16 output columns: staging [128][nout]
      OutT* d = stg + row * (16 * P.nbg) + 16 * j;  // box row pitch: nbg blocks
      if constexpr (sizeof(OutT) == 2) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
        uint4* d4 = reinterpret_cast<uint4*>(d);
        d4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      } else {
        uint4* d4 = reinterpret_cast<uint4*>(d);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
      }
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    // the box covers nbg blocks; a short last group is clipped by the axis end
    if (VERT)
      tma_store_3d(&tm_out, stg, 128 * strip, 16 * b0, p);
    else
      tma_store_3d(&tm_out, stg, 16 * b0, 128 * strip, p);
    bulk_commit();
    bulk_wait_read0();  // smem may be released once read; the write completes on its own
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_n(tmem, P.tmem_cols);
  }
}

template <bool VERT, typename OutT>
static cudaError_t launch(const Params& P, const CUtensorMap& tin, const CUtensorMap& tout,
                          uint32_t smem, cudaStream_t stream, bool epi) {
  if (epi) {
    auto k = axis_pass_kernel<VERT, OutT, true>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) k<<<P.nunits, kThreads, smem, stream>>>(tin, tout, P);
    return e;
  }
  auto k = axis_pass_kernel<VERT, OutT, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) k<<<P.nunits, kThreads, smem, stream>>>(tin, tout, P);
  return e;
}

}  // namespace apass

// Apply axis `a` along dimension `dim` (0: rows, 1: columns) of `planes`
// planes: in (planes x H x W, bf16) -> out (rows: a->n_out x W; columns:
// H x a->n_out), bf16 or f32.
ts_status axis_pass_run(const ts_axis* a, int dim, int planes, int H, int W, const void* in,
                        int64_t in_rs, int64_t in_ps, void* out, int64_t out_rs, int64_t out_ps,
                        int out_dtype, const ts_epilogue* ep, cudaStream_t stream) {
  if (!a || !in || !out || planes < 1 || H < 1 || W < 1 || (dim != 0 && dim != 1))
    return set_error(TS_ERR_INVALID, "axis_pass: bad arguments");
  if (out_dtype != TS_BF16 && out_dtype != TS_F32)
    return set_error(TS_ERR_UNSUPPORTED, "axis_pass: output must be bf16 or f32");
  const int n_in = dim == 0 ? H : W;
  if (a->n_in != n_in)
    return set_error(TS_ERR_INVALID, "axis_pass: axis expects %d inputs, image has %d", a->n_in,
                     n_in);
  const int oes = out_dtype == TS_BF16 ? 2 : 4;
  const int OH = dim == 0 ? a->n_out : H, OW = dim == 0 ? W : a->n_out;
  if (in_rs < W || (in_rs * 2) % 16 || in_ps < in_rs * H || (in_ps * 2) % 16 || out_rs < OW ||
      (out_rs * oes) % 16 || out_ps < out_rs * OH || (out_ps * oes) % 16)
    return set_error(TS_ERR_INVALID, "axis_pass: strides");
  DeviceGuard guard(a->device);
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");
  apass::Params P;
  P.ep = make_epik(ep);
  P.ax = a->dev();
  P.planes = planes;
  P.nb = a->nb;
  P.nstrip = ((dim == 0 ? W : H) + 127) / 128;
  // blocks per CTA: more blocks amortise the per-CTA setup, fewer keep more
  // CTAs (and so more 2 KB TMA boxes) in flight per SM, which is what the
  // load path needs — group only when there are plenty of units
  const uint32_t tb = static_cast<uint32_t>(a->tile_bytes);
  const int64_t base_units = static_cast<int64_t>(planes) * a->nb * P.nstrip;
  P.nbg = 1;
  // (measured on B200, tools/sweep_apass.sh: 4K->540p and 2048^2->{143,450,921}^2)
  if (dim == 0) {
    const int64_t want = 148 * 64;
    if (base_units / 2 >= want && 2u * tb <= 32768u) P.nbg = 2;
  } else if (base_units >= 148 * 32 && 2u * tb <= 32768u) {
    P.nbg = 2;  // horizontal: small CTAs, many per SM
  }
  if (const char* f = std::getenv("TSB_APASS_NBG")) P.nbg = std::atoi(f) > 0 ? std::atoi(f) : 1;
  if (P.nbg > P.nb) P.nbg = P.nb;
  P.ngroups = (P.nb + P.nbg - 1) / P.nbg;
  P.tmem_cols = 32;
  while (P.tmem_cols < 16u * P.nbg) P.tmem_cols *= 2;
  const int64_t units = static_cast<int64_t>(planes) * P.ngroups * P.nstrip;
  if (units > 0x7FFFFFFF) return set_error(TS_ERR_UNSUPPORTED, "axis_pass: too many blocks");
  P.nunits = static_cast<int>(units);
  {
    const int kslots = dim == 0 ? apass::Ring<true>::kSlots : apass::Ring<false>::kSlots;
    const int ksteps = dim == 0 ? apass::Ring<true>::kSteps : apass::Ring<false>::kSteps;
    const int per_block = (a->K / 16 + ksteps - 1) / ksteps;
    // vertical: 4 of the 6 slots; horizontal: one 64-column slot (the
    // short-lived CTAs then fit ~7 per SM, which keeps more loads in flight
    // than a deeper ring per CTA)
    P.nring = dim == 0 ? 4 : 1;
    if (const char* f = std::getenv("TSB_APASS_RING")) P.nring = std::atoi(f);
    if (P.nring > P.nbg * per_block) P.nring = P.nbg * per_block;
    if (P.nring < 1) P.nring = 1;
    if (P.nring > kslots) P.nring = kslots;
  }
  P.off_b = P.nring * (dim == 0 ? apass::Ring<true>::kSlot : apass::Ring<false>::kSlot);
  P.off_out = P.off_b + ((static_cast<uint32_t>(P.nbg) * tb + 1023u) & ~1023u);
  P.off_bar = P.off_out + ((128u * 16u * P.nbg * oes + 1023u) & ~1023u);
  const uint32_t smem = P.off_bar + 256u + 1024u;
  CUtensorMap tin, tout;
  ts_status st;
  if (dim == 0)
    st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, W, H, planes, in_rs, in_ps,
                        64, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  else
    st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, W, H, planes, in_rs, in_ps,
                        64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  const CUtensorMapDataType odt =
      out_dtype == TS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  st = encode_tmap_3d(&tout, odt, oes, out, OW, OH, planes, out_rs, out_ps,
                      dim == 0 ? 128 : 16 * P.nbg, dim == 0 ? 16 * P.nbg : 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TS_OK) return st;
  cudaError_t e;
  if (dim == 0)
    e = out_dtype == TS_BF16
            ? apass::launch<true, __nv_bfloat16>(P, tin, tout, smem, stream, ep != nullptr)
            : apass::launch<true, float>(P, tin, tout, smem, stream, ep != nullptr);
  else
    e = out_dtype == TS_BF16
            ? apass::launch<false, __nv_bfloat16>(P, tin, tout, smem, stream, ep != nullptr)
            : apass::launch<false, float>(P, tin, tout, smem, stream, ep != nullptr);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "axis_pass launch");
}

}  // namespace tsb

// axis_pass.cu — one banded axis applied along rows ("vertical") or columns
// ("horizontal") of planar images, for geometries the fused separable kernel
// cannot tile (windows of more than ~128-512 inputs per 16 outputs: large
// downscale factors, very wide filters).  A resample then
// runs as two passes with a bf16 intermediate in HBM (the same rounding
// point as the fused kernel's V):
//
//   vertical   mid[p][o][c] = Σ_k R[o][k] in[p][k][c]
//              A = 64 input rows x 128 columns per ring slot (two 64-column
//              TMA boxes, MN-major, 128B swizzle) = 4 K-steps of 16 rows,
//              B = the block's K x 16 weight tile, D (TMEM) lane = column
//   horizontal out[p][r][j] = Σ_k mid[p][r][k] C[j][k]
//              A = 128 rows x 64 columns per ring slot (one K-major 128B
//              swizzled box) = 4 K-steps of 16 columns, D lane = row
//
// A unit = (plane, group of nbg 16-output blocks, 128-wide strip); each
// block's K window (up to 1024 inputs, ~45x downscale) streams through the
// ring, the group's blocks accumulate into adjacent 16-column TMEM slices
// and leave in one TMA store.
//
// Persistent CTAs: a kernel that contains tcgen05 (TMEM) instructions starts
// CTAs ~4x slower than a plain kernel (tools/probes/launch_rate.cu on B200:
// ~250 vs ~1000 CTAs/us for the whole GPU), so one short-lived CTA per unit
// made these passes launch-rate bound (22k CTAs >= 89 us of the vertical
// pass's 131 us at 2048^2 -> 921^2, 48 planes).  Each CTA here keeps its
// barriers and TMEM and takes units strided over the grid:
//
//   warp 0     producer: the unit's weight tiles (bulk copy) into one of two
//              weight buffers, then every block's K window through the ring
//   warp 1     MMA issuer: N = 16 per block into one of two TMEM
//              accumulators, so unit k+1 accumulates while unit k drains
//   warps 2-5  epilogue: TMEM -> registers -> staging -> one TMA store
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.h"
#include "sm100.cuh"

namespace tsb {

int sm_count_current();
ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz);

namespace apass {

constexpr int kThreads = 192;
constexpr uint32_t kSlot = 16384;  // 4 K-steps of A
constexpr int kMaxRing = 4;

// a decoded unit, handed from the producer to the MMA and epilogue warps
struct Unit {
  int live;  // 0 = end of work
  int p, b0, nblk, strip;
};

struct Params {
  AxisDev ax;
  int nb, nstrip, nbg, ngroups;
  int nq;      // K-steps per block (K / 16)
  int nchunk;  // ring slots per block
  int nunits;
  int nring;        // ring slots in use
  uint32_t tcols;   // TMEM columns per accumulator buffer
  uint32_t wbytes;  // bytes per weight buffer
  uint32_t off_w, off_out, off_bar;
  EpiK ep;  // output epilogue (EPI kernels only)
};

__device__ __forceinline__ void write_unit(Unit* dst, const Unit& u) {
  volatile int* d = reinterpret_cast<volatile int*>(dst);
  d[0] = u.live, d[1] = u.p, d[2] = u.b0, d[3] = u.nblk, d[4] = u.strip;
}

__device__ __forceinline__ Unit read_unit(const Unit* src) {
  const volatile int* s = reinterpret_cast<const volatile int*>(src);
  Unit u;
  u.live = s[0], u.p = s[1], u.b0 = s[2], u.nblk = s[3], u.strip = s[4];
  return u;
}

// (at most 4 CTAs per SM fit the shared-memory layouts: 85 registers each)
template <bool VERT, typename OutT, bool EPI>
__global__ void __launch_bounds__(kThreads, 4)
    axis_pass_kernel(const __grid_constant__ CUtensorMap tm_in,
                     const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ Params P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxRing;
  uint64_t* wfull = bars + 2 * kMaxRing;  // [2] weights + unit info landed
  uint64_t* ufree = wfull + 2;            // [2] epilogue done with buffer b (4 arrivals)
  uint64_t* afull = ufree + 2;            // [2] accumulator b complete
  Unit* units = reinterpret_cast<Unit*>(afull + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(units + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tb = static_cast<uint32_t>(P.ax.tile_bytes);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxRing; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&wfull[b], 1);
      mbar_init(&ufree[b], 4);
      mbar_init(&afull[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_n(tmem_slot, 2 * P.tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the previous kernel in the stream (e.g. the other pass) is complete

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int k = 0;; ++k) {
        const int u = blockIdx.x + k * gridDim.x;
        const int b = k & 1;
        // buffer b (unit info, weights) was last used by unit k - 2
        if (k >= 2) mbar_wait(&ufree[b], ((k >> 1) - 1) & 1);
        Unit U{};
        if (u >= P.nunits) {
          write_unit(&units[b], U);
          mbar_arrive(&wfull[b]);
          break;
        }
        const int local = u % (P.nstrip * P.ngroups);
        U.live = 1;
        U.p = u / (P.nstrip * P.ngroups);
        U.strip = local % P.nstrip;
        U.b0 = (local / P.nstrip) * P.nbg;
        U.nblk = min(P.nbg, P.nb - U.b0);
        write_unit(&units[b], U);
        mbar_arrive_expect_tx(&wfull[b], tb * U.nblk);
        uint8_t* wb = base + P.off_w + b * P.wbytes;
        for (int j = 0; j < U.nblk; ++j) {
          const int tid = __ldg(P.ax.tid + U.b0 + j);
          bulk_g2s(wb + j * tb, P.ax.tiles + static_cast<size_t>(tid) * tb, tb, &wfull[b]);
        }
        for (int j = 0; j < U.nblk; ++j) {
          const int ws = __ldg(P.ax.ws + U.b0 + j);  // window start (may be negative)
          for (int c = 0; c < P.nchunk; ++c) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], kSlot);
            uint8_t* dst = base + s * kSlot;
            if (VERT) {  // rows ws+64c.., columns 128*strip.. as two 64-column boxes
              tma_load_3d(dst, &tm_in, &full[s], 128 * U.strip, ws + 64 * c, U.p);
              tma_load_3d(dst + kSlot / 2, &tm_in, &full[s], 128 * U.strip + 64, ws + 64 * c, U.p);
            } else {  // rows 128*strip.., columns ws+64c..
              tma_load_3d(dst, &tm_in, &full[s], ws + 64 * c, 128 * U.strip, U.p);
            }
            if (++s == P.nring) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, 16, VERT ? 1u : 0u, 0u);
    int s = 0;
    uint32_t ph = 0;
    for (int k = 0;; ++k) {
      const int b = k & 1;
      const uint32_t n = static_cast<uint32_t>(k >> 1);
      mbar_wait(&wfull[b], n & 1);
      const Unit U = read_unit(&units[b]);
      if (!U.live) break;
      if (k >= 2) mbar_wait(&ufree[b], (n - 1) & 1);  // accumulator b drained
      tc_fence_after();
      const uint64_t bd0 = make_sdesc(base_s + P.off_w + b * P.wbytes, 128u,
                                      static_cast<uint32_t>(P.ax.K) * 16u, kSwizzleNone);
      const uint32_t acc = tmem + b * P.tcols;
      for (int j = 0; j < U.nblk; ++j) {
        const uint64_t bdj = bd0 + static_cast<uint64_t>(j * (tb >> 4));
        for (int c = 0; c < P.nchunk; ++c) {
          mbar_wait(&full[s], ph);
          __syncwarp();
          tc_fence_after();
          const uint32_t sa = base_s + s * kSlot;
          // vertical: MN-major SW128, the two 64-column halves 8 KB apart,
          // K-steps of 16 rows 2 KB apart; horizontal: K-major SW128, K-steps
          // 32 bytes apart inside the swizzle atom
          const uint64_t ad = VERT ? make_sdesc(sa, kSlot / 2, 1024u, kSwizzle128B)
                                   : make_sdesc(sa, 16u, 1024u, kSwizzle128B);
          constexpr uint32_t adv = VERT ? 2048u >> 4 : 32u >> 4;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = 4 * c + i;
            if (q < P.nq)
              mma_f16_ss_elect(acc + 16u * j, ad + static_cast<uint64_t>(i * adv), bdj + 16u * q,
                               idesc, q > 0 ? 1u : 0u);
          }
          mma_commit_elect(&empty[s]);
          if (++s == P.nring) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      mma_commit_elect(&afull[b]);
    }
  } else {
    // epilogue warps 2-5: TMEM lane quadrant = warp % 4
    const int et = threadIdx.x - 64;
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    for (int k = 0;; ++k) {
      const int b = k & 1;
      const uint32_t n = static_cast<uint32_t>(k >> 1);
      mbar_wait(&wfull[b], n & 1);
      const Unit U = read_unit(&units[b]);
      if (!U.live) break;
      mbar_wait(&afull[b], n & 1);
      tc_fence_after();
      named_bar_sync(1, 128);  // staging free: the previous store has read it
      const uint32_t tl = tmem + (static_cast<uint32_t>(qd * 32) << 16) + b * P.tcols;
      OutT* stg = reinterpret_cast<OutT*>(base + P.off_out);
      for (int j = 0; j < U.nblk; ++j) {
        uint32_t r[16];
        tmem_ld16(tl + 16u * j, r);
        tmem_wait_ld();
        if constexpr (EPI) {
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(epi_f32(P.ep, __uint_as_float(r[i])));
        }
        if (VERT) {  // lane = column, values = 16 output rows: staging [16 nbg][128]
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float v = __uint_as_float(r[i]);
            if constexpr (sizeof(OutT) == 2)
              stg[(16 * j + i) * 128 + row] = __float2bfloat16_rn(v);
            else
              stg[(16 * j + i) * 128 + row] = v;
          }
        } else {  // lane = row, values = 16 output columns: staging [128][16 nbg]
          OutT* d = stg + row * (16 * P.nbg) + 16 * j;
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ufree[b]);  // accumulator, weights and unit info free
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (et == 0) {
        // the box covers nbg blocks; a short last group is clipped by the axis end
        if (VERT)
          tma_store_3d(&tm_out, stg, 128 * U.strip, 16 * U.b0, U.p);
        else
          tma_store_3d(&tm_out, stg, 16 * U.b0, 128 * U.strip, U.p);
        bulk_commit();
        bulk_wait_read0();  // staging may be rewritten once read; the write completes on its own
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_n(tmem, 2 * P.tcols);
  }
  // the next kernel in the stream may launch only now: CTAs parked in
  // griddepcontrol.wait beside working ones slowed them (an early
  // trigger cost 30% on a 4K -> 540p two-pass resample)
  pdl_launch_dependents();
}

template <bool VERT, typename OutT, bool EPI>
static cudaError_t launch(const Params& P, const CUtensorMap& tin, const CUtensorMap& tout,
                          int grid, uint32_t smem, cudaStream_t stream) {
  auto k = axis_pass_kernel<VERT, OutT, EPI>;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_done[dev] = true;
  }
  const cudaError_t e = launch_pdl(k, grid, kThreads, smem, stream, tin, tout, P);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool VERT, bool EPI>
static cudaError_t launch_t(int out_dtype, const Params& P, const CUtensorMap& tin,
                            const CUtensorMap& tout, int grid, uint32_t smem,
                            cudaStream_t stream) {
  return out_dtype == TS_BF16 ? launch<VERT, __nv_bfloat16, EPI>(P, tin, tout, grid, smem, stream)
                              : launch<VERT, float, EPI>(P, tin, tout, grid, smem, stream);
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

  apass::Params P{};
  P.ep = make_epik(ep);
  P.ax = a->dev();
  P.nb = a->nb;
  P.nstrip = ((dim == 0 ? W : H) + 127) / 128;
  P.nq = a->K / 16;
  P.nchunk = (P.nq + 3) / 4;
  // wide windows (K >= 128: each block already streams >= 2 slots) run one
  // block per unit through a 3-slot ring; narrower ones two blocks per unit
  // (the weight copy and the store amortised) through 2 slots — measured on
  // B200 over nbg 1/2/4 x ring 1-4, 2048^2 -> {921, 450, 245, 143}^2 and
  // 4K -> 540p, 48 planes (K4)
  const bool wide = a->K >= 128;
  P.nbg = wide ? 1 : 2;
  // (a vertical pass with K >= 96 streams two slots per block: a third slot
  // keeps its loads going — 2048^2 -> 450^2 and 4K -> 540p vertical passes
  // 1% faster; the horizontal passes gain nothing from it)
  P.nring = wide || (dim == 0 && a->K >= 96) ? 3 : 2;
  if (const char* f = std::getenv("TSB_APASS_NBG")) P.nbg = std::max(1, std::atoi(f));
  if (const char* f = std::getenv("TSB_APASS_RING")) P.nring = std::atoi(f);
  P.nbg = std::min(std::min(P.nbg, 8), P.nb);
  P.nring = std::max(1, std::min(P.nring, apass::kMaxRing));
  const uint32_t tb = static_cast<uint32_t>(a->tile_bytes);
  uint32_t smem = 0;
  for (;;) {  // shrink a (knob-requested) group, then the ring, until the layout fits
    P.tcols = 32;
    while (P.tcols < 16u * P.nbg) P.tcols *= 2;
    P.wbytes = (P.nbg * tb + 127u) & ~127u;
    P.off_w = P.nring * apass::kSlot;
    P.off_out = (P.off_w + 2 * P.wbytes + 1023u) & ~1023u;
    P.off_bar = P.off_out + ((128u * 16u * P.nbg * oes + 1023u) & ~1023u);
    smem = P.off_bar + 256u + 1024u;
    if (smem <= 232448u) break;
    if (P.nbg > 1)
      --P.nbg;
    else if (P.nring > 1)
      --P.nring;
    else
      return set_error(TS_ERR_UNSUPPORTED, "axis_pass: window %d too large", a->K);
  }
  P.ngroups = (P.nb + P.nbg - 1) / P.nbg;
  const int64_t units = static_cast<int64_t>(planes) * P.ngroups * P.nstrip;
  if (units > 0x7FFFFFFF) return set_error(TS_ERR_UNSUPPORTED, "axis_pass: too many blocks");
  P.nunits = static_cast<int>(units);
  // CTAs per SM from shared memory, TMEM (two accumulators each) and threads
  int per_sm = static_cast<int>((228u * 1024u) / (smem + 1024u));
  per_sm = std::min(per_sm, static_cast<int>(512u / (2u * P.tcols)));
  per_sm = std::max(1, std::min(per_sm, 2048 / apass::kThreads));
  const int grid = static_cast<int>(std::min<int64_t>(units, per_sm * sm_count_current()));

  CUtensorMap tin, tout;
  ts_status st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, W, H, planes, in_rs,
                                in_ps, 64, dim == 0 ? 64 : 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  const CUtensorMapDataType odt =
      out_dtype == TS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  st = encode_tmap_3d(&tout, odt, oes, out, OW, OH, planes, out_rs, out_ps,
                      dim == 0 ? 128 : 16 * P.nbg, dim == 0 ? 16 * P.nbg : 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TS_OK) return st;
  const bool epi = ep != nullptr;
  cudaError_t e;
  if (dim == 0)
    e = epi ? apass::launch_t<true, true>(out_dtype, P, tin, tout, grid, smem, stream)
            : apass::launch_t<true, false>(out_dtype, P, tin, tout, grid, smem, stream);
  else
    e = epi ? apass::launch_t<false, true>(out_dtype, P, tin, tout, grid, smem, stream)
            : apass::launch_t<false, false>(out_dtype, P, tin, tout, grid, smem, stream);
  return e == cudaSuccess ? TS_OK : cuda_error(e, "axis_pass launch");
}

}  // namespace tsb

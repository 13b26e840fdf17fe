// separable.cu — fused separable linear transform on sm_100a:
//
//     out[p] = R · in[p] · Cᵀ        (R: rows axis, C: cols axis, both banded)
//
// This is the B200 execution of what the reference expresses as lowered
// `wmma_load_a(I, base, s·n, m, k)` / `wmma_load_b(Toeplitz)` / `wmma_mma`
// statements (rules.py:766-803, interp.py:427-486): an overlapped-window
// gather times a banded Toeplitz-family matrix, f32 accumulation.  One
// persistent kernel does both passes of a separable resample / filter:
//
//  tile = (plane p, 128 output rows, nb2*16 output columns)
//  warp 0      TMA producer: input halo tile (R1 rows x 128 cols, bf16,
//              128B-swizzled) + the block's B tiles (bulk copies) into a
//              2-stage ring.
//  warp 1      MMA issuer (one thread):
//                pass 1 (vertical): for each 16-output-row block k
//                  D_V[c, 16k..] = Σ_r X[r, c] · R_kᵀ[r, ·]      (M=128 cols, N=16, K=R.K)
//                  A = staged tile, MN-major SW128; B = R block tile, K-major
//                pass 2 (horizontal): for each 16-output-column block j
//                  D_H[i, 16j..] = Σ_c V[i, c] · C_jᵀ[c, ·]      (M=128 rows, N=16, K=C.K)
//                  A = V (bf16, MN-major SW128, written by the epilogue)
//  warps 2..5  epilogue: TMEM -> regs -> bf16 -> smem (V operand),
//              then TMEM -> regs -> cast -> smem -> TMA store.
//
// Window starts are multiples of 8 rows/cols (the builder guarantees it) so
// every MMA operand starts on a 1024-byte swizzle atom.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "sm100.cuh"

namespace tsb {

constexpr int kStages = 2;
constexpr int kThreads = 192;  // warp0 TMA, warp1 MMA, warps 2-5 epilogue
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kMidBytes = 128 * 128 * 2;  // V tile: 128 rows x 128 cols bf16

struct SepParams {
  AxisDev r;  // rows axis (pass 1)
  AxisDev c;  // cols axis (pass 2)
  int nb2;    // column blocks per tile
  int R1;     // staged input rows per tile (multiple of 16)
  int nrt, nct, planes, ntiles;
};

struct SepSmem {
  uint32_t in_stage, w_stage, w1_bytes, out_bytes;
  uint32_t off_w, off_mid, off_out, off_bar, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline SepSmem sep_smem_layout(const SepParams& P, int out_bytes_per_elem) {
  SepSmem L;
  L.in_stage = 2u * static_cast<uint32_t>(P.R1) * 128u;
  L.w1_bytes = static_cast<uint32_t>(kRowBlocksPerTile * P.r.tile_bytes);
  L.w_stage = align_up(L.w1_bytes + static_cast<uint32_t>(P.nb2 * P.c.tile_bytes), 1024);
  L.out_bytes = align_up(128u * P.nb2 * 16u * out_bytes_per_elem, 1024);
  L.off_w = kStages * L.in_stage;
  L.off_mid = L.off_w + kStages * L.w_stage;
  L.off_out = L.off_mid + kMidBytes;
  L.off_bar = L.off_out + L.out_bytes;
  L.total = L.off_bar + 256 + 1024;  // barriers + alignment slack
  return L;
}

template <typename OutT>
__device__ __forceinline__ void store_out_row(uint32_t dst, const uint32_t (&r)[16]);

template <>
__device__ __forceinline__ void store_out_row<__nv_bfloat16>(uint32_t dst, const uint32_t (&r)[16]) {
  uint32_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
  st_shared_v4(dst, p[0], p[1], p[2], p[3]);
  st_shared_v4(dst + 16, p[4], p[5], p[6], p[7]);
}

template <>
__device__ __forceinline__ void store_out_row<float>(uint32_t dst, const uint32_t (&r)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) st_shared_v4(dst + 16 * i, r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
}

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    separable_kernel(const __grid_constant__ CUtensorMap tm_in,
                     const __grid_constant__ CUtensorMap tm_out, const SepParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const SepSmem L = sep_smem_layout(P, sizeof(OutT));

  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L.off_bar);
  uint64_t* full = bars;                // [kStages] TMA + bulk bytes landed
  uint64_t* empty = bars + kStages;     // [kStages] tile consumed by both passes
  uint64_t* dv_full = bars + 2 * kStages;
  uint64_t* dv_free = dv_full + 1;
  uint64_t* mid_full = dv_full + 2;
  uint64_t* dh_full = dv_full + 3;
  uint64_t* dh_free = dv_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dv_full + 5);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(dv_full, 1);
    mbar_init(dv_free, 128);
    mbar_init(mid_full, 128);
    mbar_init(dh_full, 1);
    mbar_init(dh_free, 128);
    fence_barrier_init();
    prefetch_tmap(&tm_in);
    prefetch_tmap(&tm_out);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int K1 = P.r.K, K2 = P.c.K;
  const int nb2 = P.nb2;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const int hr = P.R1 / 2;
      int it = 0;
      for (int t = blockIdx.x; t < P.ntiles; t += gridDim.x, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int ct = t % P.nct;
        const int rest = t / P.nct;
        const int rt = rest % P.nrt;
        const int p = rest / P.nrt;
        const int b1 = rt * kRowBlocksPerTile, b2 = ct * nb2;
        const int row0 = P.r.ws[b1], col0 = P.c.ws[b2];
        uint32_t wbytes = 0;
        for (int k = 0; k < kRowBlocksPerTile; ++k)
          if (k == 0 || P.r.tid[b1 + k] != P.r.tid[b1 + k - 1]) wbytes += P.r.tile_bytes;
        for (int j = 0; j < nb2; ++j)
          if (j == 0 || P.c.tid[b2 + j] != P.c.tid[b2 + j - 1]) wbytes += P.c.tile_bytes;
        mbar_arrive_expect_tx(&full[s], L.in_stage + wbytes);
        uint8_t* dst = base + s * L.in_stage;
        tma_load_3d(dst, &tm_in, &full[s], col0, row0, p);
        tma_load_3d(dst + hr * 128, &tm_in, &full[s], col0, row0 + hr, p);
        tma_load_3d(dst + P.R1 * 128, &tm_in, &full[s], col0 + 64, row0, p);
        tma_load_3d(dst + P.R1 * 128 + hr * 128, &tm_in, &full[s], col0 + 64, row0 + hr, p);
        uint8_t* wd = base + L.off_w + s * L.w_stage;
        for (int k = 0; k < kRowBlocksPerTile; ++k)
          if (k == 0 || P.r.tid[b1 + k] != P.r.tid[b1 + k - 1])
            bulk_g2s(wd + k * P.r.tile_bytes,
                     P.r.tiles + static_cast<size_t>(P.r.tid[b1 + k]) * P.r.tile_bytes,
                     P.r.tile_bytes, &full[s]);
        for (int j = 0; j < nb2; ++j)
          if (j == 0 || P.c.tid[b2 + j] != P.c.tid[b2 + j - 1])
            bulk_g2s(wd + L.w1_bytes + j * P.c.tile_bytes,
                     P.c.tiles + static_cast<size_t>(P.c.tid[b2 + j]) * P.c.tile_bytes,
                     P.c.tile_bytes, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc(kFmtBF16, 128, 16, /*a MN-major*/ 1, /*b K-major*/ 0);
      const uint32_t lbo_in = static_cast<uint32_t>(P.R1) * 128u;  // 64-col half stride
      const uint32_t mid_s = base_s + L.off_mid;
      int it = 0;
      for (int t = blockIdx.x; t < P.ntiles; t += gridDim.x, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        const int ct = t % P.nct;
        const int rt = (t / P.nct) % P.nrt;
        const int b1 = rt * kRowBlocksPerTile, b2 = ct * nb2;
        const int row0 = P.r.ws[b1], col0 = P.c.ws[b2];
        const uint32_t a0 = base_s + s * L.in_stage;
        const uint32_t w0 = base_s + L.off_w + s * L.w_stage;

        mbar_wait(&full[s], ph);
        mbar_wait(dv_free, (it & 1) ^ 1);
        tc_fence_after();
        int slot = 0;
        for (int k = 0; k < kRowBlocksPerTile; ++k) {
          if (k == 0 || P.r.tid[b1 + k] != P.r.tid[b1 + k - 1]) slot = k;
          const uint32_t aoff = static_cast<uint32_t>(P.r.ws[b1 + k] - row0) * 128u;
          for (int q = 0; q < K1 / 16; ++q) {
            const uint64_t ad = make_sdesc(a0 + aoff + q * 2048u, lbo_in, 1024u, kSwizzle128B);
            const uint64_t bd =
                make_sdesc(w0 + slot * P.r.tile_bytes + q * 256u, 128u, K1 * 16u, kSwizzleNone);
            mma_f16_ss(tmem + 16u * k, ad, bd, idesc, q > 0 ? 1u : 0u);
          }
        }
        mma_commit(dv_full);

        mbar_wait(mid_full, it & 1);
        mbar_wait(dh_free, (it & 1) ^ 1);
        tc_fence_after();
        int slot2 = 0;
        for (int j = 0; j < nb2; ++j) {
          if (j == 0 || P.c.tid[b2 + j] != P.c.tid[b2 + j - 1]) slot2 = j;
          const uint32_t aoff = static_cast<uint32_t>((P.c.ws[b2 + j] - col0) / 8) * 1024u;
          for (int q = 0; q < K2 / 16; ++q) {
            const uint64_t ad = make_sdesc(mid_s + aoff + q * 2048u, 16384u, 1024u, kSwizzle128B);
            const uint64_t bd = make_sdesc(w0 + L.w1_bytes + slot2 * P.c.tile_bytes + q * 256u,
                                           128u, K2 * 16u, kSwizzleNone);
            mma_f16_ss(tmem + 128u + 16u * j, ad, bd, idesc, q > 0 ? 1u : 0u);
          }
        }
        mma_commit(dh_full);
        mma_commit(&empty[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t mid_s = base_s + L.off_mid;
    const uint32_t out_s = base_s + L.off_out;
    const uint32_t out_row_bytes = static_cast<uint32_t>(nb2 * 16 * sizeof(OutT));
    // V operand address pieces for input column c = row
    const uint32_t mid_row = mid_s + (row / 8) * 1024u + (row % 8) * 128u;
    int it = 0;
    for (int t = blockIdx.x; t < P.ntiles; t += gridDim.x, ++it) {
      const int ct = t % P.nct;
      const int rest = t / P.nct;
      const int rt = rest % P.nrt;
      const int p = rest / P.nrt;

      // pass-1 accumulator: lane = input column c, column = output row i
      mbar_wait(dv_full, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t r[16];
        tmem_ld16(t_lane + 16u * ch, r);
        tmem_wait_ld();
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int i8 = ch * 2 + g;  // 8-row group of output rows
          const uint32_t addr = mid_row + (i8 / 8) * 16384u + (((i8 % 8) ^ (row % 8)) * 16u);
          st_shared_v4(addr,
                       pack_bf16x2(__uint_as_float(r[8 * g + 0]), __uint_as_float(r[8 * g + 1])),
                       pack_bf16x2(__uint_as_float(r[8 * g + 2]), __uint_as_float(r[8 * g + 3])),
                       pack_bf16x2(__uint_as_float(r[8 * g + 4]), __uint_as_float(r[8 * g + 5])),
                       pack_bf16x2(__uint_as_float(r[8 * g + 6]), __uint_as_float(r[8 * g + 7])));
        }
      }
      tc_fence_before();
      mbar_arrive(dv_free);
      fence_proxy_async_smem();
      mbar_arrive(mid_full);

      // pass-2 accumulator: lane = output row i, column = output column j
      mbar_wait(dh_full, it & 1);
      tc_fence_after();
      if (et == 0) bulk_wait_read0();  // previous TMA store finished reading staging
      named_bar_sync(1, 128);
      const uint32_t orow = out_s + row * out_row_bytes;
#pragma unroll 1
      for (int j = 0; j < nb2; ++j) {
        uint32_t r[16];
        tmem_ld16(t_lane + 128u + 16u * j, r);
        tmem_wait_ld();
        store_out_row<OutT>(orow + j * 16u * sizeof(OutT), r);
      }
      tc_fence_before();
      mbar_arrive(dh_free);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (et == 0) {
        tma_store_3d(&tm_out, base + L.off_out, ct * nb2 * 16, rt * kRowBlocksPerTile * 16, p);
        bulk_commit();
      }
    }
    if (et == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
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
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <typename OutT>
static ts_status launch_sep(const SepParams& P, const CUtensorMap& tin, const CUtensorMap& tout,
                            cudaStream_t stream) {
  const SepSmem L = sep_smem_layout(P, sizeof(OutT));
  // per-device attribute; cheap, so set it on every launch
  cudaError_t e = cudaFuncSetAttribute(separable_kernel<OutT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(L.total));
  if (e != cudaSuccess) return cuda_error(e, "cudaFuncSetAttribute(separable smem)");
  const int grid = P.ntiles < sm_count_current() ? P.ntiles : sm_count_current();
  separable_kernel<OutT><<<grid, kThreads, L.total, stream>>>(tin, tout, P);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_error(e, "separable_kernel launch");
  return TS_OK;
}

ts_status separable_run(const ts_axis* ra, const ts_axis* ca, int planes, const void* in,
                        int64_t in_rs, int64_t in_ps, int in_dtype, void* out, int64_t out_rs,
                        int64_t out_ps, int out_dtype, cudaStream_t stream) {
  if (!ra || !ca || !in || !out) return set_error(TS_ERR_INVALID, "separable: null argument");
  if (planes < 1) return set_error(TS_ERR_INVALID, "separable: planes must be >= 1");
  if (in_dtype != TS_BF16)
    return set_error(TS_ERR_UNSUPPORTED, "separable: input must be bf16 (cast f32 first)");
  if (out_dtype != TS_BF16 && out_dtype != TS_F32)
    return set_error(TS_ERR_UNSUPPORTED, "separable: output must be bf16 or f32");
  const int oes = out_dtype == TS_BF16 ? 2 : 4;
  if (ra->row_span > kMaxRowSpan || ra->row_span % 16)
    return set_error(TS_ERR_UNSUPPORTED, "rows axis: row tile span %d > %d", ra->row_span,
                     kMaxRowSpan);
  if (ca->col_nbt < 1)
    return set_error(TS_ERR_UNSUPPORTED, "cols axis: window %d does not fit a 128-column tile",
                     ca->K);
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
  cudaError_t de = cudaSetDevice(ra->device);
  if (de != cudaSuccess) return cuda_error(de, "cudaSetDevice");

  SepParams P;
  P.r = ra->dev();
  P.c = ca->dev();
  P.nb2 = ca->col_nbt;
  P.R1 = ra->row_span;
  P.nrt = (ra->nb + kRowBlocksPerTile - 1) / kRowBlocksPerTile;
  P.nct = (ca->nb + P.nb2 - 1) / P.nb2;
  P.planes = planes;
  P.ntiles = planes * P.nrt * P.nct;

  CUtensorMap tin, tout;
  ts_status st = encode_tmap_3d(&tin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, in, ca->n_in, ra->n_in,
                                planes, in_rs, in_ps, 64, P.R1 / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  st = encode_tmap_3d(&tout,
                      out_dtype == TS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                      oes, out, ca->n_out, ra->n_out, planes, out_rs, out_ps, P.nb2 * 16, 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TS_OK) return st;
  const SepSmem L = sep_smem_layout(P, oes);
  if (L.total > 232448u)
    return set_error(TS_ERR_UNSUPPORTED, "separable: %u bytes of shared memory needed", L.total);
  if (out_dtype == TS_BF16) return launch_sep<__nv_bfloat16>(P, tin, tout, stream);
  return launch_sep<float>(P, tin, tout, stream);
}

}  // namespace tsb

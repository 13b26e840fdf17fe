// separable_f32.cu — f32-input separable transform on the FMA pipe.
//
// Config c1 (a 1080p f32 image, Lanczos-3 2x) is HBM-bound at ~9 multiply-adds
// per input pixel (2 FLOP per HBM byte, far below the FP32 pipe's ridge), so
// the tensor-core path's separate f32 -> bf16 cast (4 B read + 2 B write +
// 2 B re-read per pixel) costs more than the arithmetic it feeds.  This kernel
// reads the f32 image once, keeps every intermediate in f32 and follows the
// order of the reference's source-form conv statement (one 1-D pass per
// axis, horizontal first, taps summed left to right, then `+ acc` with
// acc = 0 — interp.py:162-167, 203-211; restated in
// oracle/pipelines_ref.py:78-97); in TS_F32_EXACT mode its f32 output is
// bit-identical to the oracle's.
//
// Uniform axes only (first[o] = S*o + base and the same T taps for every
// output: the exact-2x Lanczos-3 axis and the centred filters).  Persistent
// CTAs walk 32 x 64 output tiles; a tile's (S*31+T) x (S*63+T) input window
// arrives as ONE TMA box (pitch 4 mod 32 floats, zero-filled outside the
// image; border tiles then replicate the edge rows / columns — the
// reference's clamp-to-edge), the horizontal pass runs into a shared f32
// buffer, and while the vertical pass writes this tile straight to global
// the next tile's window is already in flight.  Taps live in
// registers; each thread computes 4 consecutive outputs from one register
// window (float4 shared loads of S*3+T inputs instead of 4*T scalar ones);
// the vertical pass takes column pairs through packed f32x2 FMAs (FFMA2).
// With TS_F32_EXACT the taps are multiplied and added separately (the
// reference's rounding, bit-exact); without it they are fused multiply-adds
// (one rounding per tap fewer, ~half the FP32 instructions).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "sm100.cuh"

namespace tsb {
ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz);
int sm_count_current();

namespace {

constexpr int kTR = 32, kTC = 64, kThreads = 256, kR = 4, kRH = 8;

// Window geometry of one tile for (stride S, taps T, column misalignment OFF):
// the staged window starts at the 16-byte-aligned column c0 - OFF.
template <int S, int T, int OFF>
struct Geo {
  static constexpr int SR = S * (kTR - 1) + T;             // window rows
  static constexpr int SCA = (OFF + S * (kTC - 1) + T + 3) & ~3;  // aligned window columns
  static constexpr int WP = ((SCA + 27) & ~31) + 4;        // pitch = 4 mod 32 floats: the
                                                           // float4 row walks of 8 lanes
                                                           // cover all 32 banks
  static constexpr int HP = kTC + 4;                       // 4 mod 32: float4 stores of 8
                                                           // lanes on consecutive rows and
                                                           // float2 column-pair loads are
                                                           // conflict-free
  static constexpr int NV = S * (kR - 1) + T;              // taps of kR outputs
  static constexpr int NVH = S * (kRH - 1) + T;            // taps of kRH horizontal outputs
  static constexpr int NVA = (OFF + NVH + 3) & ~3;         // as whole float4s
  static constexpr int smem = 4 * (SR * WP + SR * HP);
  static_assert(WP <= 256 && SR <= 256, "one TMA box per window");
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // FFMA2
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// (column block, row block, plane) of a tile, advanced by the grid stride
// with carries instead of a runtime division per tile
struct TileIdx {
  int tx, ty, p;
};

template <int S, int T, int OFF, bool BF16, bool EXACT, bool EPI>
__global__ void __launch_bounds__(kThreads, T > 16 ? 2 : 3) separable_f32_kernel(
    const __grid_constant__ CUtensorMap tm_in, int H, int W, int ntx, int nty, int planes,
    void* __restrict__ out, int OH, int OW, int64_t ors, int64_t ops, int vec2, int rbase,
    int cbase, const float* __restrict__ rw, const float* __restrict__ cw, EpiK ek) {
  using G = Geo<S, T, OFF>;
  extern __shared__ __align__(128) float sm[];
  float* win = sm;                  // SR x WP  input window (f32, one TMA box)
  float* hb = win + G::SR * G::WP;  // SR x HP  horizontal pass
  __shared__ __align__(8) uint64_t full;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  (void)lane;
  (void)warp;

  auto decompose = [&](int t) {
    TileIdx c;
    c.tx = t % ntx;
    const int rest = t / ntx;
    c.ty = rest % nty;
    c.p = rest / nty;
    return c;
  };
  const TileIdx step = decompose(gridDim.x);
  auto advance = [&](TileIdx c) {
    c.tx += step.tx;
    if (c.tx >= ntx) c.tx -= ntx, ++c.ty;
    c.ty += step.ty;
    if (c.ty >= nty) c.ty -= nty, ++c.p;
    c.p += step.p;
    return c;
  };
  // the whole (SR x WP) window as one TMA box at (column S*oc0 + cbase - OFF,
  // row S*or0 + rbase); samples outside the image arrive as zeros
  auto issue = [&](const TileIdx& c) {
    fence_proxy_async_smem();  // this CTA's generic writes (edge fix-up) before the async overwrite
    mbar_arrive_expect_tx(&full, G::SR * G::WP * 4);
    tma_load_3d(win, &tm_in, &full, S * kTC * c.tx + cbase - OFF, S * kTR * c.ty + rbase, c.p);
  };
  TileIdx cur = decompose(blockIdx.x);
  pdl_wait();  // the previous kernel in the stream is complete
  if (tid == 0) {
    mbar_init(&full, 1);
    fence_barrier_init();
    prefetch_tmap(&tm_in);
    if (cur.p < planes) issue(cur);
  }
  __syncthreads();

  // every output of a uniform axis has the same taps: hold them in registers
  float wc[T];
  float2 wr2[T];  // row taps duplicated for the packed column-pair FMAs
  float2 wcp[T / 2];  // column taps (OFF & 1) + 2i, + 2i + 1 as register pairs (S == 2)
#pragma unroll
  for (int t = 0; t < T; ++t) {
    wc[t] = __ldg(cw + t);
    const float w = __ldg(rw + t);
    wr2[t] = make_float2(w, w);
  }
#pragma unroll
  for (int i = 0; i < T / 2; ++i)
    wcp[i] = make_float2(wc[min((OFF & 1) + 2 * i, T - 1)], wc[min((OFF & 1) + 2 * i + 1, T - 1)]);

  int it = 0;
  for (; cur.p < planes; cur = advance(cur), ++it) {
  const int p = cur.p, or0 = kTR * cur.ty, oc0 = kTC * cur.tx;
  const int r0 = S * or0 + rbase, c0a = S * oc0 + cbase - OFF;
  // horizontal pass: task = (group g of kRH output columns, window row r); the
  // lanes of a warp walk consecutive rows
  auto hpass = [&]() {
  for (int task = tid; task < G::SR * (kTC / kRH); task += kThreads) {
    const int g = task / G::SR, r = task - g * G::SR;
    const float4* x = reinterpret_cast<const float4*>(win + r * G::WP + S * kRH * g);
    float v[G::NVA];
#pragma unroll
    for (int i = 0; i < G::NVA / 4; ++i) {
      const float4 f = x[i];
      v[4 * i] = f.x, v[4 * i + 1] = f.y, v[4 * i + 2] = f.z, v[4 * i + 3] = f.w;
    }
    float o[kRH];
    if constexpr (!EXACT && S == 2) {
      // even stride: input OFF + 2k + t sits at an even register index for
      // every output k exactly when t = OFF (mod 2), so taps (t, t+1) from
      // there on are one aligned register pair -> one FFMA2 per two taps
      // (even- and odd-tap partial sums, added at the end)
      constexpr int T0 = OFF & 1, NP = (T - T0) / 2;
#pragma unroll
      for (int k = 0; k < kRH; ++k) {
        const int e = OFF + S * k + T0;
        float2 acc2 = make_float2(__fmul_rn(v[e], wcp[0].x), __fmul_rn(v[e + 1], wcp[0].y));
#pragma unroll
        for (int i = 1; i < NP; ++i) acc2 = ffma2(make_float2(v[e + 2 * i], v[e + 2 * i + 1]), wcp[i], acc2);
#pragma unroll
        for (int t = 0; t < T0; ++t) acc2.x = fmaf(v[OFF + S * k + t], wc[t], acc2.x);
#pragma unroll
        for (int t = T0 + 2 * NP; t < T; ++t) acc2.y = fmaf(v[OFF + S * k + t], wc[t], acc2.y);
        o[k] = acc2.x + acc2.y;
      }
    } else {
#pragma unroll
    for (int k = 0; k < kRH; ++k) {
      float acc = __fmul_rn(v[OFF + S * k], wc[0]);
#pragma unroll
      for (int t = 1; t < T; ++t)
        acc = EXACT ? __fadd_rn(acc, __fmul_rn(v[OFF + S * k + t], wc[t]))
                    : fmaf(v[OFF + S * k + t], wc[t], acc);
      o[k] = __fadd_rn(acc, 0.0f);
    }
    }
    #pragma unroll
    for (int i = 0; i < kRH / 4; ++i)
      *reinterpret_cast<float4*>(hb + r * G::HP + kRH * g + 4 * i) =
          make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
  }
  };
  mbar_wait(&full, it & 1);
  if (r0 < 0 || r0 + G::SR > H || c0a < 0 || c0a + G::SCA > W) {
    // clamp-to-edge (the reference's boundary policy): replicate the edge
    // rows, then the edge columns, over the zero-filled samples
    const int top = min(max(-r0, 0), G::SR);          // window rows above the image
    const int bot = max(min(H - r0, G::SR), top);     // first window row below it
    const int nr = top + (G::SR - bot);
    for (int idx = tid; idx < nr * G::SCA; idx += kThreads) {
      const int i = idx / G::SCA, q = idx - i * G::SCA;
      const int r = i < top ? i : bot + (i - top);
      win[r * G::WP + q] = win[(i < top ? -r0 : H - 1 - r0) * G::WP + q];
    }
    __syncthreads();
    const int nl = min(max(-c0a, 0), G::SCA);            // columns left of the image
    const int rb0 = max(min(W - c0a, G::SCA), nl);       // first column right of it
    const int nb = nl + (G::SCA - rb0);
    for (int idx = tid; idx < G::SR * nb; idx += kThreads) {
      const int r = idx / nb, j = idx - r * nb;
      const int q = j < nl ? j : rb0 + (j - nl);
      win[r * G::WP + q] = win[r * G::WP + (min(max(c0a + q, 0), W - 1) - c0a)];
    }
    __syncthreads();
  }
  hpass();
  __syncthreads();  // window consumed: stage the next tile while the vertical pass runs
  if (tid == 0) {
    const TileIdx nxt = advance(cur);
    if (nxt.p < planes) issue(nxt);
  }

  // vertical pass: task = (group g of kR output rows, column pair j, j+1);
  // the lanes walk consecutive column pairs (one float2 per window row), and
  // the fast mode runs both columns through one packed FFMA2 per tap
  for (int task = tid; task < (kTR / kR) * (kTC / 2); task += kThreads) {
    const int g = task / (kTC / 2), j = 2 * (task - g * (kTC / 2));
    const int oc = oc0 + j;
    const float2* x = reinterpret_cast<const float2*>(hb + S * kR * g * G::HP + j);
    float2 v[G::NV];
#pragma unroll
    for (int i = 0; i < G::NV; ++i) v[i] = x[i * (G::HP / 2)];
#pragma unroll
    for (int k = 0; k < kR; ++k) {
      float2 acc = make_float2(__fmul_rn(v[S * k].x, wr2[0].x), __fmul_rn(v[S * k].y, wr2[0].x));
#pragma unroll
      for (int t = 1; t < T; ++t) {
        if constexpr (EXACT) {
          acc.x = __fadd_rn(acc.x, __fmul_rn(v[S * k + t].x, wr2[t].x));
          acc.y = __fadd_rn(acc.y, __fmul_rn(v[S * k + t].y, wr2[t].x));
        } else {
          acc = ffma2(v[S * k + t], wr2[t], acc);
        }
      }
      const int orow = or0 + kR * g + k;
      if (orow < OH) {
        float y0 = __fadd_rn(acc.x, 0.0f), y1 = __fadd_rn(acc.y, 0.0f);
        if constexpr (EPI) {
          y0 = epi_f32(ek, y0);
          y1 = epi_f32(ek, y1);
        }
        const int64_t o = p * ops + orow * ors + oc;
        if constexpr (BF16) {
          __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(out) + o;
          if (vec2 && oc + 1 < OW) {
            *reinterpret_cast<uint32_t*>(ob) = pack_bf16x2(y0, y1);
          } else {
            if (oc < OW) ob[0] = __float2bfloat16_rn(y0);
            if (oc + 1 < OW) ob[1] = __float2bfloat16_rn(y1);
          }
        } else {
          float* of = static_cast<float*>(out) + o;
          if (vec2 && oc + 1 < OW) {
            *reinterpret_cast<float2*>(of) = make_float2(y0, y1);
          } else {
            if (oc < OW) of[0] = y0;
            if (oc + 1 < OW) of[1] = y1;
          }
        }
      }
    }
  }
  __syncthreads();  // hb consumed before the next tile's horizontal pass
  }
  // the next kernel may start only now: CTAs waiting in pdl_wait() on an SM
  // take issue slots from this FMA-pipe-bound kernel (an early trigger
  // halved c1's throughput)
  pdl_launch_dependents();
}

template <int S, int T, int OFF, bool BF16, bool EXACT, bool EPI>
ts_status launch_f32(int planes, const float* in, int H, int W, int64_t irs, int64_t ips, int rb,
                     const float* rw, int OH, int cb, const float* cw, int OW, void* out,
                     int64_t ors, int64_t ops, const EpiK& ek, cudaStream_t st) {
  constexpr int smem = Geo<S, T, OFF>::smem;
  auto fn = separable_f32_kernel<S, T, OFF, BF16, EXACT, EPI>;
  static std::atomic<bool> attr_done[64] = {};  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(TS_ERR_INVALID, "separable_f32: device index");
  if (!attr_done[dev].load()) {
    cudaError_t attr = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) return cuda_error(attr, "separable_f32: smem attribute");
    attr_done[dev].store(true);
  }
  if (reinterpret_cast<uintptr_t>(in) % 16 || irs % 4 || ips % 4)
    return set_error(TS_ERR_UNSUPPORTED,
                     "separable_f32: TMA needs a 16-byte aligned image with row and plane "
                     "strides that are multiples of 4 floats");
  CUtensorMap tm;
  ts_status ts = encode_tmap_3d(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, in, W, H, planes, irs, ips,
                                Geo<S, T, OFF>::WP, Geo<S, T, OFF>::SR,
                                CU_TENSOR_MAP_SWIZZLE_NONE);
  if (ts != TS_OK) return ts;
  const int ntx = (OW + kTC - 1) / kTC, nty = (OH + kTR - 1) / kTR;
  const int64_t ntiles64 = static_cast<int64_t>(ntx) * nty * planes;
  if (ntiles64 > (1 << 30)) return set_error(TS_ERR_UNSUPPORTED, "separable_f32: too many tiles");
  const int ntiles = static_cast<int>(ntiles64);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem);
  // persistent CTAs: each stages its next tile while it runs this one's vertical pass
  const int slots = (per_sm > 0 ? per_sm : 1) * sm_count_current();
  const int grid = ntiles < slots ? ntiles : slots;
  // paired stores need 2-element aligned rows (4 B bf16 pairs / 8 B f32 pairs)
  const int vec2 = ors % 2 == 0 && ops % 2 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % (BF16 ? 4 : 8) == 0;
  cudaError_t e = launch_pdl(fn, grid, kThreads, smem, st, tm, H, W, ntx, nty, planes, out, OH,
                             OW, ors, ops, vec2, rb, cb, rw, cw, ek);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "separable_f32 launch");
}

template <int S, int T, int OFF, bool EPI>
ts_status launch_f32_epi(bool bf, bool exact, int planes, const float* in, int H, int W,
                         int64_t irs, int64_t ips, int rb, const float* rw, int OH, int cb,
                         const float* cw, int OW, void* out, int64_t ors, int64_t ops,
                         const EpiK& ek, cudaStream_t st) {
#define TS_F32_ARGS planes, in, H, W, irs, ips, rb, rw, OH, cb, cw, OW, out, ors, ops, ek, st
  if (bf) return exact ? launch_f32<S, T, OFF, true, true, EPI>(TS_F32_ARGS)
                       : launch_f32<S, T, OFF, true, false, EPI>(TS_F32_ARGS);
  return exact ? launch_f32<S, T, OFF, false, true, EPI>(TS_F32_ARGS)
               : launch_f32<S, T, OFF, false, false, EPI>(TS_F32_ARGS);
#undef TS_F32_ARGS
}

template <int S, int T, int OFF>
ts_status launch_f32_any(bool epi, bool bf, bool exact, int planes, const float* in, int H, int W,
                         int64_t irs, int64_t ips, int rb, const float* rw, int OH, int cb,
                         const float* cw, int OW, void* out, int64_t ors, int64_t ops,
                         const EpiK& ek, cudaStream_t st) {
  return epi ? launch_f32_epi<S, T, OFF, true>(bf, exact, planes, in, H, W, irs, ips, rb, rw, OH,
                                               cb, cw, OW, out, ors, ops, ek, st)
             : launch_f32_epi<S, T, OFF, false>(bf, exact, planes, in, H, W, irs, ips, rb, rw, OH,
                                                cb, cw, OW, out, ors, ops, ek, st);
}

}  // namespace
}  // namespace tsb

using namespace tsb;

extern "C" ts_status ts_separable_f32_ep(int planes, const float* in, int in_h, int in_w,
                                         int64_t in_row_stride, int64_t in_plane_stride,
                                         int stride, int taps, int row_base,
                                         const float* row_weights, int out_h, int col_base,
                                         const float* col_weights, int out_w, void* out,
                                         int64_t out_row_stride, int64_t out_plane_stride,
                                         int out_dtype, int flags, const ts_epilogue* ep,
                                         void* stream) {
  if (planes < 0 || in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1)
    return set_error(TS_ERR_INVALID, "separable_f32: bad sizes");
  if (planes == 0) return TS_OK;
  if (!in || !out || !row_weights || !col_weights)
    return set_error(TS_ERR_INVALID, "separable_f32: null pointer");
  if (out_dtype != TS_F32 && out_dtype != TS_BF16)
    return set_error(TS_ERR_INVALID, "separable_f32: out dtype must be f32 or bf16");
  if (in_row_stride < in_w || in_plane_stride < in_row_stride * in_h ||
      out_row_stride < out_w || out_plane_stride < out_row_stride * out_h)
    return set_error(TS_ERR_INVALID, "separable_f32: strides smaller than the image");
  if (ep && ep->lo > ep->hi) return set_error(TS_ERR_INVALID, "epilogue: lo > hi");
  DeviceGuard guard(device_of(in));
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");
  const EpiK ek = make_epik(ep);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool bf = out_dtype == TS_BF16, exact = flags & TS_F32_EXACT;
  const int off = col_base & 3;  // misalignment of every tile's first column
#define TS_F32_CASE(S_, T_, OFF_)                                                                \
  if (stride == S_ && taps == T_ && off == OFF_)                                                 \
    return launch_f32_any<S_, T_, OFF_>(ep != nullptr, bf, exact, planes, in, in_h, in_w, in_row_stride,        \
                                        in_plane_stride, row_base, row_weights, out_h, col_base, \
                                        col_weights, out_w, out, out_row_stride,                 \
                                        out_plane_stride, ek, st);
  TS_F32_CASE(2, 12, 3)  // Lanczos-3 2x: first tap 2o - 5
  TS_F32_CASE(1, 9, 0)   // centred filters: first tap o - (T-1)/2
  TS_F32_CASE(1, 15, 1)
  TS_F32_CASE(1, 21, 2)
  TS_F32_CASE(1, 31, 1)
#undef TS_F32_CASE
  return set_error(TS_ERR_UNSUPPORTED,
                   "separable_f32: (stride %d, taps %d, column base %d) not instantiated", stride,
                   taps, col_base);
}

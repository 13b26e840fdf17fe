// probe.cu — tcgen05 operand-mode probe (diagnostics, used by tests and for
// kernel design): one CTA stages A (128 x k) and B (k x n) in a chosen
// layout, issues the K loop `reps` times into one TMEM accumulator and
// reports D plus the clock64 cycles from first issue to completion.
//
//   amode 0: A in smem, MN-major, 128B swizzle (bf16)
//   amode 1: A in smem, K-major, no swizzle core matrices (bf16)
//   amode 2: A in TMEM, f32 read as tf32 (kind::tf32), lane = row, column = k
//   bmode 0: B in smem, K-major, no swizzle (bf16; f32 for amode 2)
//   bmode 1: B in smem, MN-major, 128B swizzle (bf16)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "sm100.cuh"
#include "tsb_diag.h"

namespace tsb {

// ------------------------------------------------------------ UMMA probe
__global__ void __launch_bounds__(128, 1)
    probe_umma_kernel(const float* __restrict__ a, const float* __restrict__ b,
                      float* __restrict__ d, int k, int n) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const uint32_t a_bytes = 128u * k * 2u;                   // two 64-wide m-atoms
  const uint32_t b_bytes = static_cast<uint32_t>(k) * n * 2u;
  uint8_t* sa = base;
  uint8_t* sb = base + a_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + a_bytes + ((b_bytes + 1023u) & ~1023u));
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const uint32_t lbo_a = static_cast<uint32_t>(k / 8) * 1024u;

  // A (128 x k): MN-major, 128B swizzle — exactly the pass-1 staging layout
  for (int e = threadIdx.x; e < 128 * k; e += blockDim.x) {
    const int m = e / k, kk = e % k;
    const uint32_t off = (m / 64) * lbo_a + (kk / 8) * 1024u + (kk % 8) * 128u +
                         ((((m % 64) / 8) ^ (kk % 8)) * 16u) + (m % 8) * 2u;
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16_rn(a[e]);
  }
  // B (k x n): K-major, no swizzle, 8x8 core matrices
  for (int e = threadIdx.x; e < k * n; e += blockDim.x) {
    const int kk = e / n, nn = e % n;
    const uint32_t off = (nn / 8) * (k * 16u) + (kk / 8) * 128u + (nn % 8) * 16u + (kk % 8) * 2u;
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16_rn(b[e]);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<256>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, n, 1, 0);
    for (int q = 0; q < k / 16; ++q) {
      const uint64_t ad = make_sdesc(base_s + q * 2048u, lbo_a, 1024u, kSwizzle128B);
      const uint64_t bd = make_sdesc(base_s + a_bytes + q * 256u, 128u, k * 16u, kSwizzleNone);
      mma_f16_ss(tmem, ad, bd, idesc, q > 0 ? 1u : 0u);
    }
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < n; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) d[row * n + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}


__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
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

__global__ void __launch_bounds__(128, 1)
    probe_mma_kernel(int amode, int bmode, const float* __restrict__ a, const float* __restrict__ b,
                     float* __restrict__ d, int k, int n, int reps, long long* cycles, int nacc) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const bool tf32 = amode >= 2 && amode <= 4;
  const bool a_tmem = amode == 2 || amode == 5;
  const int es = tf32 ? 4 : 2;
  const uint32_t a_bytes = a_tmem ? 0u : 128u * k * (tf32 ? 4u : 2u);
  const uint32_t b_bytes = static_cast<uint32_t>(k) * n * es;
  uint8_t* sa = base;
  uint8_t* sb = base + a_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + a_bytes + ((b_bytes + 1023u) & ~1023u));
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- stage A
  const uint32_t lbo_a_mn = static_cast<uint32_t>(k / 8) * 1024u;  // m-atom stride (amode 0)
  const uint32_t sbo_a_k = static_cast<uint32_t>(k / 8) * 128u;    // 8-row group stride (amode 1)
  if (amode == 3 || amode == 4) {
    for (int e = threadIdx.x; e < 128 * k; e += blockDim.x) {
      const int m = e / k, kk = e % k;
      uint32_t off;
      if (amode == 3)  // MN-major SW128: 32 f32 per atom row, k rows at 128 B
        off = (m / 32) * (static_cast<uint32_t>(k / 8) * 1024u) + (kk / 8) * 1024u +
              (kk % 8) * 128u + ((((m % 32) / 4) ^ (kk % 8)) * 16u) + (m % 4) * 4u;
      else  // K-major no swizzle: core matrices 8 m x 4 k
        off = (m / 8) * (static_cast<uint32_t>(k / 4) * 128u) + (kk / 4) * 128u + (m % 8) * 16u +
              (kk % 4) * 4u;
      *reinterpret_cast<float*>(sa + off) = a[e];
    }
  }
  if (!tf32 && !a_tmem) {
    for (int e = threadIdx.x; e < 128 * k; e += blockDim.x) {
      const int m = e / k, kk = e % k;
      uint32_t off;
      if (amode == 0)
        off = (m / 64) * lbo_a_mn + (kk / 8) * 1024u + (kk % 8) * 128u +
              ((((m % 64) / 8) ^ (kk % 8)) * 16u) + (m % 8) * 2u;
      else
        off = (m / 8) * sbo_a_k + (kk / 8) * 128u + (m % 8) * 16u + (kk % 8) * 2u;
      *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16_rn(a[e]);
    }
  }
  // ---- stage B
  const uint32_t lbo_b_mn = static_cast<uint32_t>(k / 8) * 1024u;  // n-atom stride (bmode 1)
  for (int e = threadIdx.x; e < k * n; e += blockDim.x) {
    const int kk = e / n, nn = e % n;
    if (tf32) {
      const uint32_t off = (nn / 8) * (static_cast<uint32_t>(k / 4) * 128u) + (kk / 4) * 128u +
                           (nn % 8) * 16u + (kk % 4) * 4u;
      *reinterpret_cast<float*>(sb + off) = b[e];
    } else {
      uint32_t off;
      if (bmode == 0)
        off = (nn / 8) * (k * 16u) + (kk / 8) * 128u + (nn % 8) * 16u + (kk % 8) * 2u;
      else
        off = (nn / 64) * lbo_b_mn + (kk / 8) * 1024u + (kk % 8) * 128u +
              ((((nn % 64) / 8) ^ (kk % 8)) * 16u) + (nn % 8) * 2u;
      *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16_rn(b[e]);
    }
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);

  if (a_tmem && amode == 5) {
    // A row m = lane m; packed bf16 pairs: column c holds (k = 2c, 2c + 1)
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < k / 2; c0 += 16) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i)
        r[i] = (c0 + i) * 2 < k ? pack_bf16x2(a[m * k + 2 * (c0 + i)], a[m * k + 2 * (c0 + i) + 1])
                                : 0u;
      tmem_st16(lane_base + 256u + c0, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  } else if (a_tmem) {
    // A row m = this thread's TMEM lane, columns [256, 256 + k)
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < k; c0 += 16) {
      uint32_t r[16];
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(a[m * k + c0 + i]);
      tmem_st16(lane_base + 256u + c0, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc =
        make_idesc(tf32 ? kFmtTF32 : kFmtBF16, 128, n, (amode == 0 || amode == 3) ? 1u : 0u,
                   bmode == 1 ? 1u : 0u);
    const int kstep = tf32 ? 8 : 16;  // amode 5 (f16 TS) uses K = 16
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      // nacc > 1: round-robin the repetitions over nacc accumulators (columns
      // n*i .. n*i+n-1) so consecutive K loops are independent
      const uint32_t dcol = static_cast<uint32_t>((r % nacc) * n);
      for (int q = 0; q < k / kstep; ++q) {
        const uint32_t acc = (r >= nacc || q > 0) ? 1u : 0u;
        if (amode == 5) {
          const uint64_t bd = make_sdesc(base_s + a_bytes + q * 256u, 128u, k * 16u, kSwizzleNone);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + dcol),
              "r"(tmem + 256u + q * 8u), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        } else if (tf32) {
          const uint64_t bd = make_sdesc(base_s + a_bytes + q * 256u, 128u,
                                         static_cast<uint32_t>(k / 4) * 128u, kSwizzleNone);
          if (amode == 2) {
            mma_tf32_ts(tmem + dcol, tmem + 256u + q * 8u, bd, idesc, acc);
          } else {
            const uint64_t ad =
                amode == 3
                    ? make_sdesc(base_s + q * 1024u, static_cast<uint32_t>(k / 8) * 1024u, 1024u,
                                 kSwizzle128B)
                    : make_sdesc(base_s + q * 256u, 128u, static_cast<uint32_t>(k / 4) * 128u,
                                 kSwizzleNone);
            mma_tf32_ss(tmem + dcol, ad, bd, idesc, acc);
          }
        } else {
          const uint64_t ad =
              amode == 0 ? make_sdesc(base_s + q * 2048u, lbo_a_mn, 1024u, kSwizzle128B)
                         : make_sdesc(base_s + q * 256u, 128u, sbo_a_k, kSwizzleNone);
          const uint64_t bd =
              bmode == 0 ? make_sdesc(base_s + a_bytes + q * 256u, 128u, k * 16u, kSwizzleNone)
                         : make_sdesc(base_s + a_bytes + q * 2048u, lbo_b_mn, 1024u, kSwizzle128B);
          mma_f16_ss(tmem + dcol, ad, bd, idesc, acc);
        }
      }
    }
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  if (threadIdx.x == 0) {
    t1 = clock64();
    if (cycles) *cycles = t1 - t0;
  }
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < n; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(lane_base + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) d[row * n + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace tsb

using namespace tsb;

extern "C" ts_status ts_probe_mma(int amode, int bmode, const float* a, const float* b, float* d,
                                  int k, int n, int reps, long long* cycles, int nacc,
                                  void* stream) {
  const int kstep = (amode >= 2 && amode <= 4) ? 8 : 16;
  if (amode < 0 || amode > 5 || bmode < 0 || bmode > 1 || (amode >= 2 && bmode != 0) || !a ||
      !b || !d || k < kstep || k > 256 || k % 16 || n < 16 || n > 256 || n % 16 || reps < 1 ||
      nacc < 1 || nacc * n > ((amode == 2 || amode == 5) ? 256 : 512) ||
      (amode >= 3 && amode <= 4 && k > 128))
    return set_error(TS_ERR_INVALID, "probe_mma: bad arguments");
  const int es = (amode >= 2 && amode <= 4) ? 4 : 2;
  const uint32_t a_bytes = (amode == 2 || amode == 5) ? 0u : 128u * k * (amode >= 3 ? 4u : 2u);
  const uint32_t b_bytes = static_cast<uint32_t>(k) * n * es;
  const uint32_t smem = 1024 + a_bytes + ((b_bytes + 1023u) & ~1023u) + 64;
  cudaError_t e =
      cudaFuncSetAttribute(probe_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_error(e, "probe_mma smem attribute");
  probe_mma_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(amode, bmode, a, b, d, k,
                                                                        n, reps, cycles, nacc);
  e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_mma launch");
}

// ---------------------------------------------------------------------------
// Issue-rate microbenchmark: one warp (converged) issues COUNT tcgen05.mma
// (M=128, K=16, N) with precomputed descriptors, fully unrolled, round-robin
// over NACC accumulators; returns clock64 cycles from first issue to the
// commit's completion.  Operands are uninitialised smem (values unused).
namespace tsb {
template <int N, int NACC, int COUNT, int ASRC>
__global__ void __launch_bounds__(128, 1) probe_issue_kernel(long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + (base_s - raw_s) + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, N, ASRC == 0 ? 1u : 0u, 0u);
    const uint64_t ad = make_sdesc(base_s, 4096u, 1024u, kSwizzle128B);
    const uint64_t bd = make_sdesc(base_s + 32768u, 128u, 256u, kSwizzleNone);
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < COUNT; ++i)
      mma_f16_ss_elect(tmem + (i % NACC) * N, ad, bd, idesc, i >= NACC ? 1u : 0u);
    mma_commit_elect(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N, int NACC>
static cudaError_t launch_issue(long long* cycles, cudaStream_t s) {
  auto k = probe_issue_kernel<N, NACC, 64, 0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  if (e != cudaSuccess) return e;
  k<<<1, 128, 70000, s>>>(cycles);
  return cudaGetLastError();
}
}  // namespace tsb

// variant: 0..5 = (N, NACC) in {(16,1), (16,8), (64,1), (64,4), (256,1), (256,2)}
extern "C" ts_status ts_probe_issue(int variant, long long* cycles, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (variant) {
    case 0: e = launch_issue<16, 1>(cycles, s); break;
    case 1: e = launch_issue<16, 8>(cycles, s); break;
    case 2: e = launch_issue<64, 1>(cycles, s); break;
    case 3: e = launch_issue<64, 4>(cycles, s); break;
    case 4: e = launch_issue<256, 1>(cycles, s); break;
    case 5: e = launch_issue<256, 2>(cycles, s); break;
    default: return set_error(TS_ERR_INVALID, "probe_issue: variant 0..5");
  }
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_issue launch");
}

// TS-mode issue rate: A from TMEM (kind::tf32 or kind::f16), B in smem.
namespace tsb {
__device__ __forceinline__ void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t acc, bool tf32) {
  if (tf32)
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

template <int N, int TF32>
__global__ void __launch_bounds__(128, 1) probe_issue_ts_kernel(long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + (base_s - raw_s) + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc(TF32 ? kFmtTF32 : kFmtBF16, 128, N, 0u, 0u);
    const uint64_t bd = make_sdesc(base_s, 128u, 256u, kSwizzleNone);
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i)
      mma_ts_elect(tmem + (i % 4) * N, tmem + 256u + (i % 8) * 8u, bd, idesc, i >= 4 ? 1u : 0u,
                   TF32 != 0);
    mma_commit_elect(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N, int TF32>
static cudaError_t launch_issue_ts(long long* cycles, cudaStream_t s) {
  auto k = probe_issue_ts_kernel<N, TF32>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  if (e != cudaSuccess) return e;
  k<<<1, 128, 40000, s>>>(cycles);
  return cudaGetLastError();
}
}  // namespace tsb

// variant: 0..3 = (N, kind) in {(16, f16), (64, f16), (16, tf32), (64, tf32)}
extern "C" ts_status ts_probe_issue_ts(int variant, long long* cycles, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (variant) {
    case 0: e = launch_issue_ts<16, 0>(cycles, s); break;
    case 1: e = launch_issue_ts<64, 0>(cycles, s); break;
    case 2: e = launch_issue_ts<16, 1>(cycles, s); break;
    case 3: e = launch_issue_ts<64, 1>(cycles, s); break;
    default: return set_error(TS_ERR_INVALID, "probe_issue_ts: variant 0..3");
  }
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_issue_ts launch");
}

// Issue-rate probe with streaming operands: `count` elected MMAs, M = 128,
// K = 16, cycling over 8 distinct K-slices of A and B (as a real K loop does).
//   amode 0: A smem MN-major SW128   1: A smem K-major no swizzle   2: A TMEM (bf16 pairs)
//   bmode 0: B smem K-major no swizzle   1: B smem MN-major SW128 (64-col atoms at 2048 B)
namespace tsb {
__global__ void __launch_bounds__(128, 1)
    probe_issue2_kernel(int amode, int bmode, int n, int count, int nacc, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 131072);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc(kFmtBF16, 128, n, amode == 0 ? 1u : 0u, bmode == 1 ? 1u : 0u);
    const uint32_t b0 = base_s + 65536u;
    const uint32_t bstep = bmode == 0 ? static_cast<uint32_t>(n) * 32u : ((n + 63) / 64) * 2048u;
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const int q = i & 7;
      const uint32_t d = tmem + static_cast<uint32_t>((i % nacc) * n);
      const uint32_t acc = i >= nacc ? 1u : 0u;
      const uint64_t bd = bmode == 0 ? make_sdesc(b0 + q * bstep, 128u, 256u, kSwizzleNone)
                                     : make_sdesc(b0 + q * bstep, 2048u, 1024u, kSwizzle128B);
      if (amode == 2) {
        asm volatile(
            "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(tmem + 384u + q * 8u), "l"(bd), "r"(idesc), "r"(acc)
            : "memory");
      } else {
        const uint64_t ad = amode == 0 ? make_sdesc(base_s + q * 2048u, 16384u, 1024u, kSwizzle128B)
                                       : make_sdesc(base_s + q * 4096u, 128u, 256u, kSwizzleNone);
        mma_f16_ss_elect(d, ad, bd, idesc, acc);
      }
    }
    mma_commit_elect(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}
}  // namespace tsb

extern "C" ts_status ts_probe_issue2(int amode, int bmode, int n, int count, int nacc,
                                     long long* cycles, void* stream) {
  if (amode < 0 || amode > 2 || bmode < 0 || bmode > 1 || n < 16 || n > 256 || n % 16 ||
      nacc < 1 || n * nacc > (amode == 2 ? 384 : 512) || count < 1)
    return set_error(TS_ERR_INVALID, "probe_issue2: bad arguments");
  auto k = probe_issue2_kernel;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  if (e == cudaSuccess) {
    k<<<1, 128, 140000, static_cast<cudaStream_t>(stream)>>>(amode, bmode, n, count, nacc, cycles);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_issue2 launch");
}

// TMA streaming probe: every CTA walks column strips of a (planes x H x W)
// bf16 tensor top to bottom in chunks of `rows` rows x (64 * nbox) columns
// through an `nr`-slot ring; the consumer releases each chunk as soon as it
// lands.  Measures the load path alone (boxes of 64 x rows, 128B swizzle).
namespace tsb {
ts_status encode_tmap_3d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* ptr,
                         int64_t d0, int64_t d1, int64_t d2, int64_t stride1_elems,
                         int64_t stride2_elems, int box0, int box1, CUtensorMapSwizzle swz);

__global__ void __launch_bounds__(64, 1)
    probe_tma_kernel(const __grid_constant__ CUtensorMap tm, int planes, int H, int W, int rows,
                     int nbox, int nr) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  const uint32_t chunk = static_cast<uint32_t>(rows) * 128u * nbox;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + nr * chunk);
  uint64_t* empty = full + 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nr; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int strips = (W + 64 * nbox - 1) / (64 * nbox);
  const int chunks = (H + rows - 1) / rows;
  const int units = planes * strips;
  if (threadIdx.x == 0) {
    int slot = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int p = u / strips, st = u % strips;
      for (int c = 0; c < chunks; ++c) {
        mbar_wait(&empty[slot], ph ^ 1);
        mbar_arrive_expect_tx(&full[slot], chunk);
        for (int h = 0; h < nbox; ++h)
          tma_load_3d(base + slot * chunk + h * rows * 128, &tm, &full[slot], (st * nbox + h) * 64,
                      c * rows, p);
        if (++slot == nr) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  } else if (threadIdx.x == 32) {
    int slot = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x)
      for (int c = 0; c < chunks; ++c) {
        mbar_wait(&full[slot], ph);
        mbar_arrive(&empty[slot]);
        if (++slot == nr) {
          slot = 0;
          ph ^= 1;
        }
      }
  }
}
}  // namespace tsb

extern "C" ts_status ts_probe_tma(const void* src, int planes, int H, int W, int rows, int nbox,
                                  int nr, int grid, void* stream) {
  using namespace tsb;
  if (!src || rows < 1 || rows > 256 || nbox < 1 || nr < 1 || nr > 32 || W % 64)
    return set_error(TS_ERR_INVALID, "probe_tma: bad arguments");
  const uint32_t smem = static_cast<uint32_t>(nr) * rows * 128u * nbox + 1024u + 1024u;
  if (smem > 232448) return set_error(TS_ERR_INVALID, "probe_tma: ring too large");
  CUtensorMap tm;
  ts_status st = encode_tmap_3d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, W, H, planes, W,
                                static_cast<int64_t>(W) * H, 64, rows, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TS_OK) return st;
  cudaError_t e =
      cudaFuncSetAttribute(probe_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) {
    probe_tma_kernel<<<grid, 64, smem, static_cast<cudaStream_t>(stream)>>>(tm, planes, H, W, rows,
                                                                            nbox, nr);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_tma launch");
}

// TMEM load throughput probe: `warps` warps (4 per lane quarter group) each
// read `cols` columns of their lane quarter with tcgen05.ld.32x32b.x{16,32,64}
// `reps` times; reports cycles for the whole CTA.
namespace tsb {
template <int X>
__device__ __forceinline__ void tmem_ldx(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tmem_ldx<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ldx<32>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

template <int X>
__global__ void __launch_bounds__(512, 1) probe_tmem_ld_kernel(int cols, int reps, long long* cycles,
                                                               unsigned* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int nw = blockDim.x / 32;
  const int per_quarter = nw / 4;        // warps sharing a lane quarter
  const int sub = (warp >> 2);           // which of them
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const int my_cols = cols / per_quarter;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < my_cols; c += X) {
      uint32_t v[X];
      tmem_ldx<X>(tmem + lane_off + static_cast<uint32_t>(sub * my_cols + c), v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= v[i];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cycles = t1 - t0;
  if (acc == 0x12345678u) *sink = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}
}  // namespace tsb

extern "C" ts_status ts_probe_tmem_ld(int x, int warps, int cols, int reps, long long* cycles,
                                      void* stream) {
  using namespace tsb;
  if ((x != 16 && x != 32) || warps < 4 || warps > 16 || warps % 4 || cols < 16 || cols > 512 ||
      reps < 1 || !cycles)
    return set_error(TS_ERR_INVALID, "probe_tmem_ld: bad arguments");
  static unsigned* sink = nullptr;
  if (!sink && cudaMalloc(&sink, 4) != cudaSuccess) return set_error(TS_ERR_CUDA, "probe sink");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (x == 16)
    probe_tmem_ld_kernel<16><<<1, warps * 32, 0, s>>>(cols, reps, cycles, sink);
  else
    probe_tmem_ld_kernel<32><<<1, warps * 32, 0, s>>>(cols, reps, cycles, sink);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_tmem_ld launch");
}

// M = 64 layout probe: D (TMEM, pre-filled with -1) = A (64 x 16, K-major core
// matrices) x B (16 x n, K-major), kind::f16, issued at TMEM lane `lane_base`
// (0 or 64).  Dumps all 128 lanes x n columns so the caller sees where an
// M = 64 accumulator lands.
namespace tsb {
__global__ void __launch_bounds__(128, 1)
    probe_m64_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ d,
                     int n, int lane_base) {
  __shared__ __align__(1024) uint8_t sm[64 * 32 + 256 * 32 + 64];
  uint8_t* sa = sm;
  uint8_t* sb = sm + 64 * 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 64 * 32 + 256 * 32);
  __shared__ uint32_t slot;
  for (int e = threadIdx.x; e < 64 * 16; e += blockDim.x) {
    const int m = e / 16, kk = e % 16;
    *reinterpret_cast<__nv_bfloat16*>(sa + (m / 8) * 256 + (kk / 8) * 128 + (m % 8) * 16 + (kk % 8) * 2) =
        __float2bfloat16_rn(a[e]);
  }
  for (int e = threadIdx.x; e < 16 * n; e += blockDim.x) {
    const int kk = e / n, nn = e % n;
    *reinterpret_cast<__nv_bfloat16*>(sb + (nn / 8) * 256 + (kk / 8) * 128 + (nn % 8) * 16 + (kk % 8) * 2) =
        __float2bfloat16_rn(b[e]);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(-1.0f);
    for (int c = 0; c < n; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tl + c),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
          "r"(r[15])
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(kFmtBF16, 64, n, 0, 0);
    const uint64_t ad = make_sdesc(smem_u32(sa), 128u, 256u, kSwizzleNone);
    const uint64_t bd = make_sdesc(smem_u32(sb), 128u, 256u, kSwizzleNone);
    mma_f16_ss(tmem + (static_cast<uint32_t>(lane_base) << 16), ad, bd, idesc, 0u);
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c = 0; c < n; c += 16) {
    uint32_t r[16];
    tmem_ld16(tl + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) d[row * n + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}
}  // namespace tsb

extern "C" ts_status ts_probe_m64(const float* a, const float* b, float* d, int n, int lane_base,
                                  void* stream) {
  using namespace tsb;
  if (!a || !b || !d || n < 16 || n > 256 || n % 16 || (lane_base != 0 && lane_base != 64 &&
                                                         lane_base != 32 && lane_base != 96))
    return set_error(TS_ERR_INVALID, "probe_m64: bad arguments");
  probe_m64_kernel<<<1, 128, 0, static_cast<cudaStream_t>(stream)>>>(a, b, d, n, lane_base);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe_m64 launch");
}

extern "C" TS_DIAG_API ts_status ts_probe_umma(const float* a, const float* b, float* d, int k, int n, void* stream) {
  if (!a || !b || !d || k < 16 || k > 256 || k % 16 || n < 16 || n > 256 || n % 16)
    return set_error(TS_ERR_INVALID, "probe: need k, n multiples of 16 in [16, 256]");
  const uint32_t a_bytes = 128u * k * 2u;
  const uint32_t b_bytes = static_cast<uint32_t>(k) * n * 2u;
  const uint32_t smem = 1024 + a_bytes + ((b_bytes + 1023u) & ~1023u) + 64;
  cudaError_t e = cudaFuncSetAttribute(probe_umma_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_error(e, "probe smem attribute");
  probe_umma_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(a, b, d, k, n);
  e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "probe launch");
}


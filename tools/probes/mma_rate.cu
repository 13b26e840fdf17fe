// Tensor-pipe cost of the DCT-16 kernel's MMA shapes on sm_100a, with
// descriptors precomputed (an unrolled issue stream, as in the kernel):
// 64 MMAs, one commit, cycles / MMA.  One CTA.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2512_02371_b200/csrc/sm100.cuh"

using namespace tsb;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// mode 0: SS, A K-major no-swizzle (strip), B MN-major SW128, N = n
// mode 1: TS, A TMEM, B K-major no-swizzle, N = n
// mode 2: SS, A MN-major SW128 (M-major, 128 x 16), B K-major no-swizzle, N = n
// mode 3: SS, A K-major no-swizzle, B K-major no-swizzle, N = n
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = smem_u32(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_s - raw_s);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 196608);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
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
    const uint32_t idesc = make_idesc(kFmtBF16, 128, N, MODE == 2 ? 1u : 0u, MODE == 0 ? 1u : 0u);
    (void)0;
    const uint64_t a0 = MODE == 2 ? make_sdesc(base_s, 16384u, 1024u, kSwizzle128B)
                                  : make_sdesc(base_s, 128u, 256u, kSwizzleNone);
    const uint64_t b0 = MODE == 0 ? make_sdesc(base_s + 65536u, 16384u, 1024u, kSwizzle128B)
                                  : make_sdesc(base_s + 65536u, 128u, 256u, kSwizzleNone);
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const uint32_t q = i & 7;
      const uint32_t d = tmem + (MODE == 1 ? 256u : 0u) + (N <= 128 ? (i & 1) * N : 0u);
      if (MODE == 1)
        mma_ts(d, tmem + 8u * q, b0 + q * 32u, idesc, i > 1 ? 1u : 0u);
      else if (MODE == 4) {  // S5 pattern: 8 tiles at 16j (overwrite), 7 at 16j + 8 (accumulate)
        const int r = i % 16;
        const uint32_t dd = r < 8 ? 256u + 16u * r : 256u + 16u * (r - 8) + 8u;
        if (r < 15) mma_ts(tmem + dd, tmem + 8u * q, b0 + q * 32u, idesc, r >= 8 ? 1u : 0u);
      } else if (MODE == 5) {  // same accumulator every MMA
        mma_ts(tmem + 256u, tmem + 8u * q, b0 + q * 32u, idesc, i > 0 ? 1u : 0u);
      }
      else if (MODE != 4 && MODE != 5)
        mma_f16_ss_elect(d, a0 + q * (MODE == 2 ? 128u : 256u), b0 + q * (MODE == 0 ? 128u : 32u), idesc,
                         i > 1 ? 1u : 0u);
    }
    mma_commit_elect(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE, int N>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  auto f = k<MODE, N>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  long long c = 0;
  for (int r = 0; r < 3; ++r) {
    f<<<1, 128, 200000>>>(d);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  }
  cudaError_t e = cudaGetLastError();
  printf("%-44s N=%3d  %.1f cycles/MMA  %s\n", name, N, c / 64.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 128>("SS A Kmaj-noswz, B MNmaj-SW128 (S1, S7)");
  run<0, 64>("SS A Kmaj-noswz, B MNmaj-SW128");
  run<1, 16>("TS A tmem, B Kmaj-noswz (S3, S5)");
  run<1, 32>("TS A tmem, B Kmaj-noswz");
  run<1, 64>("TS A tmem, B Kmaj-noswz");
  run<1, 128>("TS A tmem, B Kmaj-noswz");
  run<2, 16>("SS A MNmaj-SW128, B Kmaj-noswz (S7 transposed)");
  run<2, 32>("SS A MNmaj-SW128, B Kmaj-noswz");
  run<3, 16>("SS A Kmaj-noswz, B Kmaj-noswz");
  run<3, 128>("SS A Kmaj-noswz, B Kmaj-noswz");
  run<4, 16>("TS S5 pattern (x60/64 issued)");
  run<5, 16>("TS one accumulator chain");
  return 0;
}

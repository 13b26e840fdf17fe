// Block-launch throughput probe (128-thread CTAs, 33408 per launch): empty
// CTAs with varying dynamic shared memory / parameter size, and CTAs whose
// code merely contains tcgen05 (TMEM) instructions, allocates 32 TMEM
// columns, or initialises an mbarrier.  Prints CTAs per microsecond.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Big { char b[1024]; };
struct Small { char b[64]; };

template <typename PT>
__global__ void empty_kernel(const __grid_constant__ PT p, int* sink) {
  extern __shared__ char sm[];
  if (p.b[threadIdx.x & 63] == 123 && sink) sink[0] = sm[0];
}

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mode 0: tcgen05 code present but skipped; 1: alloc + dealloc 32 columns;
// 2: mode 1 without relinquish; 3: mbarrier init only
__global__ void tmem_kernel(int mode, int* sink) {
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  if (mode == 3) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    return;
  }
  if (mode == 0 && sink == nullptr) return;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)) : "memory");
    if (mode != 2) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot) : "memory");
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / 20;
}

int main() {
  const int blocks = 33408;
  for (int smem : {0, 30000}) {
    auto k = empty_kernel<Big>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float us = timeit([&] { k<<<blocks, 128, smem>>>(Big{}, nullptr); });
    printf("empty, 1 KB params, smem %5d: %6.1f us  %5.0f CTA/us\n", smem, us, blocks / us);
  }
  const char* names[] = {"tcgen05 code skipped", "TMEM alloc+dealloc", "alloc, no relinquish",
                         "mbarrier init"};
  for (int mode = 0; mode < 4; ++mode) {
    float us = timeit([&] { tmem_kernel<<<blocks, 128>>>(mode, nullptr); });
    printf("%-22s: %6.1f us  %5.0f CTA/us\n", names[mode], us, blocks / us);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

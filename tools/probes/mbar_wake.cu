// mbarrier wake-up latency on sm_100a: warp 1 arrives at clock t0, warp 0
// (already waiting) sees the phase flip at t1; try_wait with and without a
// suspend-time hint, and a satisfied wait (barrier completed long before).
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2512_02371_b200/csrc/sm100.cuh"

using namespace tsb;

template <int MODE>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
  if (MODE == 0) {
    while (!mbar_try_wait(bar, par)) {
    }
  } else {
    while (!mbar_try_wait_sleep(bar, par)) {
    }
  }
}

template <int MODE>
__global__ void k(long long* out, int reps) {
  __shared__ uint64_t bar[2];
  __shared__ long long tarr;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  long long sum = 0, sat = 0;
  for (int r = 0; r < reps; ++r) {
    const uint32_t par = r & 1;
    if (threadIdx.x < 32) {
      wait<MODE>(&bar[0], par);
      const long long t1 = clock64();
      sum += t1 - *(volatile long long*)&tarr;
      const long long t2 = clock64();
      wait<MODE>(&bar[0], par);  // satisfied
      sat += clock64() - t2;
      if (threadIdx.x == 0) mbar_arrive(&bar[1]);
    } else if (threadIdx.x == 32) {
      const long long t = clock64();
      while (clock64() - t < 2000) {
      }
      *(volatile long long*)&tarr = clock64();
      __threadfence_block();
      mbar_arrive(&bar[0]);
      wait<0>(&bar[1], par);
    }
  }
  if (threadIdx.x == 0) {
    out[0] = sum / reps;
    out[1] = sat / reps;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  k<0><<<1, 64>>>(d, 64);
  k<0><<<1, 64>>>(d, 256);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("try_wait spin      : wake %lld cycles, satisfied wait %lld cycles\n", h[0], h[1]);
  k<1><<<1, 64>>>(d, 64);
  k<1><<<1, 64>>>(d, 256);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("try_wait + suspend : wake %lld cycles, satisfied wait %lld cycles\n", h[0], h[1]);
  return 0;
}

// Test helper: fill every SM's shared memory with a bit pattern, so a later
// kernel that reads shared memory it never wrote gives pattern-dependent
// (with 0xFFFFFFFF: NaN) results instead of silently multiplying stale data
// by zero weights.  Compiled by tests/test_gpu_smem_poison.py on the GPU box.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void poison_kernel(uint32_t words, uint32_t pattern) {
  extern __shared__ uint32_t sm[];
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sm[i] = pattern;
  __syncthreads();
}

extern "C" int smem_poison(unsigned pattern, void* stream) {
  const int bytes = 232448;  // the sm_100 per-CTA maximum: one CTA covers an SM's carve-out
  cudaFuncSetAttribute(poison_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  poison_kernel<<<sms * 4, 1024, bytes, static_cast<cudaStream_t>(stream)>>>(bytes / 4, pattern);
  return static_cast<int>(cudaGetLastError());
}

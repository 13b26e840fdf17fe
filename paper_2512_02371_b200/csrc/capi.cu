// capi.cu — extern "C" entry points (include/tensorsel_b200.h) plus the small
// device kernels that sit beside the fused executors: the f32->bf16 cast and
// the device-side dense Toeplitz builder (layout.matrix_for).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "sm100.cuh"

namespace tsb {
ts_status separable_run(const ts_axis* ra, const ts_axis* ca, int planes, const void* in,
                        int64_t in_rs, int64_t in_ps, int in_dtype, void* out, int64_t out_rs,
                        int64_t out_ps, int out_dtype, const ts_epilogue* ep, cudaStream_t stream);
ts_status separable_plan(const ts_axis* ra, const ts_axis* ca, int planes, int out_dtype,
                         int* out8);
#ifdef TSB_DIAG
void set_trace(void* buf, int ctas, int tiles);
#endif
ts_status axis_pass_run(const ts_axis* a, int dim, int planes, int H, int W, const void* in,
                        int64_t in_rs, int64_t in_ps, void* out, int64_t out_rs, int64_t out_ps,
                        int out_dtype, const ts_epilogue* ep, cudaStream_t stream);

// ------------------------------------------------------------------ cast
__global__ void cast_f32_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                     int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 8;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i < n;
       i += stride) {
    if (i + 8 <= n && ((reinterpret_cast<uintptr_t>(in + i) & 15) == 0) &&
        ((reinterpret_cast<uintptr_t>(out + i) & 15) == 0)) {
      float4 a = *reinterpret_cast<const float4*>(in + i);
      float4 b = *reinterpret_cast<const float4*>(in + i + 4);
      uint4 o;
      o.x = pack_bf16x2(a.x, a.y);
      o.y = pack_bf16x2(a.z, a.w);
      o.z = pack_bf16x2(b.x, b.y);
      o.w = pack_bf16x2(b.z, b.w);
      *reinterpret_cast<uint4*>(out + i) = o;
    } else {
      for (int64_t j = i; j < n && j < i + 8; ++j) out[j] = __float2bfloat16_rn(in[j]);
    }
  }
}

// ------------------------------------------------------------ matrix_for
// out[y][x] = K[tap(y, x)] or 0, tap per layout.kernel_taps (layout.py:60-69)
__global__ void matrix_for_kernel(int l, int k, int s, int p, int rows,
                                  const float* __restrict__ kern, float* __restrict__ out) {
  const int64_t n = static_cast<int64_t>(rows) * k;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(e / k), x = static_cast<int>(e % k);
    int tap = -1;
    if (p > 1) {
      const int u = y - x / p;
      if (u >= 0 && u < l) tap = p * u + x % p;
    } else {
      const int t = y - s * x;
      if (t >= 0 && t < l) tap = t;
    }
    out[e] = tap >= 0 ? kern[tap] : 0.0f;
  }
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int ts_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int good = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major == 10) ++good;
  }
  return good;
}

ts_status ts_separable_run(const ts_axis* rows, const ts_axis* cols, int planes, const void* in,
                           int64_t in_row_stride, int64_t in_plane_stride, int in_dtype, void* out,
                           int64_t out_row_stride, int64_t out_plane_stride, int out_dtype,
                           void* stream) {
  return separable_run(rows, cols, planes, in, in_row_stride, in_plane_stride, in_dtype, out,
                       out_row_stride, out_plane_stride, out_dtype, nullptr,
                       static_cast<cudaStream_t>(stream));
}

ts_status ts_separable_run_ep(const ts_axis* rows, const ts_axis* cols, int planes, const void* in,
                              int64_t in_row_stride, int64_t in_plane_stride, int in_dtype,
                              void* out, int64_t out_row_stride, int64_t out_plane_stride,
                              int out_dtype, const ts_epilogue* ep, void* stream) {
  return separable_run(rows, cols, planes, in, in_row_stride, in_plane_stride, in_dtype, out,
                       out_row_stride, out_plane_stride, out_dtype, ep,
                       static_cast<cudaStream_t>(stream));
}

ts_status ts_separable_plan(const ts_axis* rows, const ts_axis* cols, int planes, int out_dtype,
                            int* out8) {
  return separable_plan(rows, cols, planes, out_dtype, out8);
}

ts_status ts_axis_pass(const ts_axis* a, int dim, int planes, int height, int width, const void* in,
                       int64_t in_row_stride, int64_t in_plane_stride, void* out,
                       int64_t out_row_stride, int64_t out_plane_stride, int out_dtype,
                       void* stream) {
  return axis_pass_run(a, dim, planes, height, width, in, in_row_stride, in_plane_stride, out,
                       out_row_stride, out_plane_stride, out_dtype, nullptr,
                       static_cast<cudaStream_t>(stream));
}

ts_status ts_axis_pass_ep(const ts_axis* a, int dim, int planes, int height, int width,
                          const void* in, int64_t in_row_stride, int64_t in_plane_stride,
                          void* out, int64_t out_row_stride, int64_t out_plane_stride,
                          int out_dtype, const ts_epilogue* ep, void* stream) {
  return axis_pass_run(a, dim, planes, height, width, in, in_row_stride, in_plane_stride, out,
                       out_row_stride, out_plane_stride, out_dtype, ep,
                       static_cast<cudaStream_t>(stream));
}

#ifdef TSB_DIAG
TS_API ts_status ts_debug_trace(void* device_buffer, int ctas, int tiles) {
  if (device_buffer && (ctas < 1 || tiles < 1))
    return set_error(TS_ERR_INVALID, "trace: ctas and tiles must be >= 1");
  set_trace(device_buffer, ctas, tiles);
  return TS_OK;
}
#endif  // TSB_DIAG

ts_status ts_cast_f32_bf16(const float* in, void* out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!in || !out))) return set_error(TS_ERR_INVALID, "cast: bad arguments");
  if (n == 0) return TS_OK;
  DeviceGuard guard(device_of(in));
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");
  int64_t blocks = (n / 8 + 255) / 256 + 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cast_f32_bf16_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      in, static_cast<__nv_bfloat16*>(out), n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "cast kernel launch");
}

ts_status ts_matrix_for(int l, int k, int s, int p, const float* kernel, float* out,
                        void* stream) {
  if (l < 1 || k < 1 || s < 1 || p < 1)
    return set_error(TS_ERR_INVALID, "ToeplitzSpec needs l, k, s, p >= 1");
  if (s != 1 && p != 1) return set_error(TS_ERR_INVALID, "stride and phases are exclusive");
  if (!kernel || !out) return set_error(TS_ERR_INVALID, "matrix_for: null pointer");
  DeviceGuard guard(device_of(out));
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");
  const int rows = p > 1 ? k / p + l : s * k + l;  // layout.matrix_rows (layout.py:54-57)
  const int64_t n = static_cast<int64_t>(rows) * k;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  matrix_for_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(l, k, s, p, rows, kernel,
                                                                          out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "matrix_for kernel launch");
}

}  // extern "C"

// executor.cu — GPU execution of lowered convolution statement groups, the
// backend of interp.run_program for the conv family.
//
// A lowered group (rules.py:766-803, 887-902 produce it) is
//     acc = wmma_zero | acc
//     for v in iterations:
//         tmp = ConvolutionShuffle | PolyphaseShuffle | Shuffle(load K[kbase_v ..])
//         acc = wmma_mma(wmma_load_a(I, abase_v, a_stride, m, k),
//                        wmma_load_b(tmp, 0, n, k, n), acc)
// evaluated by interp.py:419-486 as: tiles re-rounded to their buffer kind,
// products in f32, k summed left to right from k = 0, then C + s.  This
// kernel evaluates every output (instance t, row i, column j) with exactly
// that operation order (no FMA contraction), so results are bit-identical to
// the reference; it batches all instances of a program (a difftest's seeds,
// or the tiles of an image) into one launch.
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"

namespace tsb {

__device__ __forceinline__ float round_kind(float x, int kind) {
  if (kind == 1) return __half2float(__float2half_rn(x));
  if (kind == 2) return __bfloat162float(__float2bfloat16_rn(x));
  return x;
}

// First out-of-bounds read wins: error[0] = 1 (src) | 2 (kern), error[1] =
// the offending index, error[2] = the iteration (statement instance).
__device__ __forceinline__ void report_oob(int32_t* error, int which, int index, int iteration) {
  if (atomicCAS(error, 0, which) == 0) {
    error[1] = index;
    error[2] = iteration;
    __threadfence();
  }
}

// One iteration's sum for output o (row i, column j) of instance t, in
// interp's order: f32 products, k left to right, the first product as the
// start value.  Returns false (after recording the error) on an
// out-of-bounds read.
__device__ __forceinline__ bool iteration_sum(const ts_conv_group& g, int t, int v, int o,
                                              float* out) {
  const int64_t outs = static_cast<int64_t>(g.m) * g.n;
  const int i = o / g.n, j = o % g.n;
  const float* I = g.src + static_cast<int64_t>(t) * g.src_stride;
  const float* K = g.kern + static_cast<int64_t>(t) * g.kern_stride;
  const bool expl = g.a_idx != nullptr;
  const int ab = expl ? 0 : g.a_base[v] + i * g.a_stride;
  const int kb = expl ? 0 : g.k_base[v];
  const int shift = g.a_shift ? g.a_shift[v] : 0;
  // explicit-gather row: per iteration, or one table shared by all (a_shift)
  const int64_t xo = ((g.a_shift ? 0 : static_cast<int64_t>(v) * outs) + o) * g.k;
  float s = 0.0f;
  for (int kk = 0; kk < g.k; ++kk) {
    const int ai = expl ? g.a_idx[xo + kk] + shift : ab + kk;
    if (ai < 0 || ai >= g.src_len) {
      report_oob(g.error, 1, ai, v);  // OutOfBounds on the A buffer
      return false;
    }
    const float a = round_kind(I[ai], g.src_kind);
    const int off = expl ? g.b_idx[xo + kk] : g.b_off[kk * g.n + j];
    float b = 0.0f;
    if (off >= 0) {
      const int ki = kb + off;
      if (ki < 0 || ki >= g.kern_len) {
        report_oob(g.error, 2, ki, v);  // OutOfBounds on the kernel buffer
        return false;
      }
      b = round_kind(K[ki], g.kern_kind);
    }
    const float p = __fmul_rn(a, b);
    s = kk == 0 ? p : __fadd_rn(s, p);
  }
  *out = s;
  return true;
}

// Accumulating mode: one thread per (instance, output), iterations in order
// into acc (interp.py:485: out = c + s per statement).
__global__ void conv_group_kernel(ts_conv_group g) {
  const int64_t outs = static_cast<int64_t>(g.m) * g.n;
  const int64_t total = static_cast<int64_t>(g.instances) * outs;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(e / outs);
    const int o = static_cast<int>(e % outs);
    float* acc = g.acc + static_cast<int64_t>(t) * g.acc_stride;
    float c = g.zero_init ? 0.0f : acc[o];
    for (int v = 0; v < g.iterations; ++v) {
      float s;
      if (!iteration_sum(g, t, v, o, &s)) return;
      c = __fadd_rn(c, s);
    }
    acc[o] = c;
  }
}

// Independent-iteration mode (out_base): one thread per (instance,
// iteration, output); each iteration is 0 + s, stored to its own slot.
__global__ void conv_scatter_kernel(ts_conv_group g) {
  const int64_t outs = static_cast<int64_t>(g.m) * g.n;
  const int64_t per = outs * g.iterations;
  const int64_t total = static_cast<int64_t>(g.instances) * per;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(e / per);
    const int64_t r = e % per;
    const int v = static_cast<int>(r / outs), o = static_cast<int>(r % outs);
    float s;
    if (!iteration_sum(g, t, v, o, &s)) return;
    g.out[static_cast<int64_t>(t) * g.out_stride + g.out_base[v] + (g.out_off ? g.out_off[o] : o)] =
        __fadd_rn(0.0f, s);
  }
}

}  // namespace tsb

using namespace tsb;

extern "C" ts_status ts_run_conv_group(const ts_conv_group* g, void* stream) {
  if (!g || !g->src || !g->kern || !g->acc || !g->error ||
      (!g->a_idx && (!g->a_base || !g->k_base || !g->b_off)) || (!g->a_idx != !g->b_idx))
    return set_error(TS_ERR_INVALID, "conv group: null pointer");
  if (g->instances < 0 || g->m < 1 || g->n < 1 || g->k < 1 || g->iterations < 0)
    return set_error(TS_ERR_INVALID, "conv group: bad shape");
  if (g->out_base && !g->out) return set_error(TS_ERR_INVALID, "conv group: out_base without out");
  const int64_t total = static_cast<int64_t>(g->instances) * g->m * g->n *
                        (g->out_base ? g->iterations : 1);
  if (total == 0) return TS_OK;
  DeviceGuard guard(device_of(g->acc));
  if (guard.err != cudaSuccess) return cuda_error(guard.err, "cudaSetDevice");
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (g->out_base)
    conv_scatter_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(*g);
  else
    conv_group_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(*g);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_error(e, "conv group launch");
}

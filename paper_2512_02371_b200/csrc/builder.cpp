// builder.cpp — the weight-matrix builder.
//
// Reference: layout.py:54-103 builds a dense (rows x k) Toeplitz-family matrix
// per (spec, kernel) with a Python double loop, and selector.lower_exprvars
// (selector.py:309-399) hoists it so it is built once per distinct operand.
// Here one *axis* of a separable transform is built once per
// (kernel, scale, size) into what the sm_100a kernels consume directly:
//
//   * the banded n_out x n_in matrix, clamp-to-edge folded in (an index that
//     falls off the image puts its weight on the edge sample);
//   * cut into 16-output blocks; block b reads the input window
//     [ws[b], ws[b] + K) with ws[b] a multiple of 8 so every window start is
//     a whole number of 128B-swizzle atoms / core matrices;
//   * each block's K x 16 slice rounded to bf16 (optionally re-balanced so
//     every output keeps its f32 tap sum — TS_AXIS_DC_EXACT) and laid out in
//     the tcgen05 K-major no-swizzle smem layout, so the kernel copies it
//     into shared memory with one bulk copy and points a descriptor at it;
//   * identical slices deduplicated (interior blocks of a Toeplitz axis all
//     share one tile; only the edge blocks differ).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.h"

namespace tsb {

namespace {
thread_local std::string g_last_error;

uint16_t f32_to_bf16_bits(float f) {
  uint32_t b;
  std::memcpy(&b, &f, 4);
  if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) return 0x7FC0;  // NaN
  // round to nearest even (same rule as interp.round_bf16, interp.py:62-69)
  uint64_t r = (static_cast<uint64_t>(b) + 0x7FFFu + ((b >> 16) & 1u)) >> 16;
  return static_cast<uint16_t>(r);
}

float bf16_bits_to_f32(uint16_t h) {
  uint32_t b = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }
int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Nudge bf16-rounded taps by single ulps (largest taps first, each at most
// one ulp away from its round-to-nearest value) so that an output's taps sum
// as close as possible to their f32 sum: a flat image stays flat.
void dc_rebalance(std::vector<uint16_t>& col_bits, const std::vector<double>& col_w) {
  double target = 0, got = 0;
  std::vector<int> order;
  for (size_t i = 0; i < col_w.size(); ++i) {
    target += col_w[i];
    got += bf16_bits_to_f32(col_bits[i]);
    if (col_w[i] != 0.0) order.push_back(static_cast<int>(i));
  }
  if (order.empty() || got == target) return;
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return std::fabs(col_w[a]) > std::fabs(col_w[b]); });
  // Greedy: each round take the single one-ulp step (on any tap, at most two
  // ulps from its rounded value) that most reduces the sum error; ties go to
  // the larger tap.  Stops when no step helps.
  std::vector<int> moved(col_bits.size(), 0);
  for (int round = 0; round < 64 && got != target; ++round) {
    double best_err = std::fabs(got - target);
    int best_i = -1, best_d = 0;
    uint16_t best_bits = 0;
    for (int i : order) {
      for (int d = -1; d <= 1; d += 2) {
        if (std::abs(moved[i] + d) > 2) continue;
        const uint16_t b = col_bits[i];
        const int mag = static_cast<int>(b & 0x7FFF) + d;
        if (mag <= 0 || mag >= 0x7F80) continue;  // never flip sign or reach inf
        const uint16_t cand = static_cast<uint16_t>((b & 0x8000) | mag);
        const double err =
            std::fabs(got - bf16_bits_to_f32(b) + bf16_bits_to_f32(cand) - target);
        if (err < best_err) {
          best_err = err;
          best_i = i;
          best_d = d;
          best_bits = cand;
        }
      }
    }
    if (best_i < 0) break;
    got += static_cast<double>(bf16_bits_to_f32(best_bits)) - bf16_bits_to_f32(col_bits[best_i]);
    col_bits[best_i] = best_bits;
    moved[best_i] += best_d;
  }
}
}  // namespace

ts_status set_error(ts_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

ts_status cuda_error(int err, const char* what) {
  return set_error(TS_ERR_CUDA, "%s: %s (%d)", what,
                   cudaGetErrorString(static_cast<cudaError_t>(err)), err);
}

const char* last_error_cstr() { return g_last_error.c_str(); }

// Build the host side of an axis.  `first`/`weights` describe output o as
// taps at first[o] + t, t < taps (unclamped input indices).
static ts_status build_axis_host(int n_in, int n_out, int taps, const int32_t* first,
                                 const float* weights, int flags, ts_axis* a) {
  if (n_in <= 0 || n_out <= 0 || taps <= 0)
    return set_error(TS_ERR_INVALID, "axis needs n_in, n_out, taps >= 1 (got %d, %d, %d)", n_in,
                     n_out, taps);
  if (!first || !weights) return set_error(TS_ERR_INVALID, "axis: null first/weights");
  a->n_in = n_in;
  a->n_out = n_out;
  a->taps = taps;
  const int nb = (n_out + kBlockN - 1) / kBlockN;
  a->nb = nb;

  // window start per block and the window length K
  std::vector<int32_t> ws(nb);
  int need = 1;
  for (int b = 0; b < nb; ++b) {
    int lo = INT32_MAX, hi = INT32_MIN;
    for (int n = 0; n < kBlockN; ++n) {
      int o = b * kBlockN + n;
      if (o >= n_out) break;
      lo = std::min(lo, static_cast<int>(first[o]));
      hi = std::max(hi, static_cast<int>(first[o]) + taps - 1);
    }
    ws[b] = floor_div(lo, 8) * 8;
    need = std::max(need, hi - ws[b] + 1);
  }
  const int K = round_up(need, 16);
  if (K > kMaxWindow)
    return set_error(TS_ERR_UNSUPPORTED,
                     "axis window %d exceeds %d inputs per 16 outputs (scale too large)", K,
                     kMaxWindow);
  a->K = K;
  a->tile_bytes = K * kBlockN * 2;

  // folded dense tiles, rounded, deduplicated
  std::map<std::string, int> ids;
  std::vector<uint16_t> tiles;
  const size_t tile_elems = static_cast<size_t>(K) * kBlockN;
  {
    std::vector<uint16_t> zero(tile_elems, 0);
    ids[std::string(reinterpret_cast<const char*>(zero.data()), tile_elems * 2)] = 0;
    tiles.insert(tiles.end(), zero.begin(), zero.end());
  }
  std::vector<int32_t> tid(nb);
  std::vector<double> colw(K);
  std::vector<uint16_t> colb(K);
  std::vector<uint16_t> tile(tile_elems);
  for (int b = 0; b < nb; ++b) {
    std::fill(tile.begin(), tile.end(), 0);
    for (int n = 0; n < kBlockN; ++n) {
      int o = b * kBlockN + n;
      if (o >= n_out) break;
      std::fill(colw.begin(), colw.end(), 0.0);
      for (int t = 0; t < taps; ++t) {
        int idx = first[o] + t;
        idx = std::min(std::max(idx, 0), n_in - 1);  // clamp-to-edge
        int k = idx - ws[b];
        if (k < 0 || k >= K)
          return set_error(TS_ERR_INVALID, "internal: folded tap outside window (o=%d)", o);
        colw[k] += static_cast<double>(weights[static_cast<size_t>(o) * taps + t]);
      }
      for (int k = 0; k < K; ++k) colb[k] = f32_to_bf16_bits(static_cast<float>(colw[k]));
      if (flags & TS_AXIS_DC_EXACT) dc_rebalance(colb, colw);
      for (int k = 0; k < K; ++k) tile[btile_offset(K, k, n) / 2] = colb[k];
    }
    std::string key(reinterpret_cast<const char*>(tile.data()), tile_elems * 2);
    auto it = ids.find(key);
    if (it == ids.end()) {
      int id = static_cast<int>(ids.size());
      ids.emplace(std::move(key), id);
      tiles.insert(tiles.end(), tile.begin(), tile.end());
      tid[b] = id;
    } else {
      tid[b] = it->second;
    }
  }
  a->ntiles = static_cast<int>(ids.size());
  a->tiles = std::move(tiles);

  // padded block tables
  a->ws.assign(nb + kBlockPad, ws[nb - 1]);
  a->tid.assign(nb + kBlockPad, 0);
  for (int b = 0; b < nb; ++b) {
    a->ws[b] = ws[b];
    a->tid[b] = tid[b];
  }
  // packed (ws << 16 | tid) tables for the fused kernel's uniform reads; axes
  // beyond +-32K inputs or 64K distinct tiles run as axis passes, which read
  // the plain ws / tid arrays
  a->tab_ok = a->ws[0] >= -32768 && a->ws[nb - 1] <= 32767 && a->ntiles <= 65535;
  a->tab.assign(a->ws.size(), 0);
  if (a->tab_ok)
    for (size_t b = 0; b < a->ws.size(); ++b)
      a->tab[b] = static_cast<int32_t>(static_cast<uint32_t>(a->ws[b]) << 16) |
                  static_cast<int32_t>(a->tid[b] & 0xFFFF);

  // pass-1 (rows) geometry: 8 blocks per tile
  int rspan = 0;
  for (int b0 = 0; b0 < nb; b0 += kRowBlocksPerTile) {
    int b1 = b0 + kRowBlocksPerTile - 1;
    rspan = std::max(rspan, a->ws[b1] + K - a->ws[b0]);
  }
  a->row_span = round_up(rspan, 16);

  // pass-2 (cols) geometry: as many blocks as fit a 128-column tile
  a->col_nbt = 0;
  a->col_span = 0;
  for (int n = kMaxColBlocks; n >= 1; --n) {
    int span = 0;
    for (int b0 = 0; b0 < nb; b0 += n) span = std::max(span, a->ws[b0 + n - 1] + K - a->ws[b0]);
    if (span <= kColTile) {
      a->col_nbt = n;
      a->col_span = span;
      break;
    }
  }
  return TS_OK;
}

static ts_status upload_axis(ts_axis* a, int device) {
  int prev = 0;
  cudaError_t e = cudaGetDevice(&prev);
  if (e != cudaSuccess) return cuda_error(e, "cudaGetDevice");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  a->device = device;
  const size_t nbp = a->ws.size();
  ts_status st = TS_OK;
  if ((e = cudaMalloc(&a->d_ws, nbp * 4)) != cudaSuccess ||
      (e = cudaMalloc(&a->d_tid, nbp * 4)) != cudaSuccess ||
      (e = cudaMalloc(&a->d_tab, nbp * 4)) != cudaSuccess ||
      (e = cudaMalloc(&a->d_tiles, a->tiles.size() * 2)) != cudaSuccess) {
    st = cuda_error(e, "cudaMalloc(axis)");
  } else if ((e = cudaMemcpy(a->d_ws, a->ws.data(), nbp * 4, cudaMemcpyHostToDevice)) !=
                 cudaSuccess ||
             (e = cudaMemcpy(a->d_tid, a->tid.data(), nbp * 4, cudaMemcpyHostToDevice)) !=
                 cudaSuccess ||
             (e = cudaMemcpy(a->d_tab, a->tab.data(), nbp * 4, cudaMemcpyHostToDevice)) !=
                 cudaSuccess ||
             (e = cudaMemcpy(a->d_tiles, a->tiles.data(), a->tiles.size() * 2,
                             cudaMemcpyHostToDevice)) != cudaSuccess) {
    st = cuda_error(e, "cudaMemcpy(axis)");
  }
  cudaSetDevice(prev);
  return st;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

const char* ts_last_error(void) { return tsb::last_error_cstr(); }

int ts_abi_version(void) { return TS_ABI_VERSION; }

void ts_axis_destroy(ts_axis* a) {
  if (!a) return;
  if (a->d_ws) cudaFree(a->d_ws);
  if (a->d_tid) cudaFree(a->d_tid);
  if (a->d_tab) cudaFree(a->d_tab);
  for (auto* m : a->merged) {
    if (!m) continue;
    if (m->d_tab) cudaFree(m->d_tab);
    if (m->d_tiles) cudaFree(m->d_tiles);
    delete m;
  }
  if (a->d_tiles) cudaFree(a->d_tiles);
  delete a;
}

ts_status ts_axis_create(int n_in, int n_out, int taps, const int32_t* first,
                         const float* weights, int flags, int device, ts_axis** out) {
  if (!out) return set_error(TS_ERR_INVALID, "ts_axis_create: null out");
  *out = nullptr;
  ts_axis* a = new ts_axis();
  ts_status st = build_axis_host(n_in, n_out, taps, first, weights, flags, a);
  if (st == TS_OK && device >= 0) st = upload_axis(a, device);
  if (st != TS_OK) {
    ts_axis_destroy(a);
    return st;
  }
  *out = a;
  return TS_OK;
}

ts_status ts_axis_from_toeplitz(int l, int s, int p, int offset, const float* kernel,
                                int kernel_len, int n_in, int n_out, int flags, int device,
                                ts_axis** out) {
  if (out) *out = nullptr;
  if (l < 1 || s < 1 || p < 1)
    return set_error(TS_ERR_INVALID, "ToeplitzSpec needs l, s, p >= 1 (got %d, %d, %d)", l, s, p);
  if (s != 1 && p != 1)
    return set_error(TS_ERR_INVALID, "stride and phases are exclusive (s=%d, p=%d)", s, p);
  if (kernel_len != p * l)
    return set_error(TS_ERR_PHASE_MISMATCH, "kernel has %d taps, spec needs %d", kernel_len,
                     p * l);
  if (!kernel) return set_error(TS_ERR_INVALID, "null kernel");
  if (n_out <= 0) return set_error(TS_ERR_INVALID, "n_out must be >= 1");
  std::vector<int32_t> first(n_out);
  std::vector<float> w(static_cast<size_t>(n_out) * l);
  for (int o = 0; o < n_out; ++o) {
    if (p == 1) {
      // A[y][x] = K[y - s*x]  =>  out[x] = sum_t in[s*x + t] * K[t]   (layout.py:60-69)
      first[o] = offset + s * o;
      for (int t = 0; t < l; ++t) w[static_cast<size_t>(o) * l + t] = kernel[t];
    } else {
      // A[y][x] = K[p*(y - x//p) + x%p]  =>  out[x] = sum_u in[x//p + u] * K[p*u + x%p]
      first[o] = offset + o / p;
      for (int u = 0; u < l; ++u) w[static_cast<size_t>(o) * l + u] = kernel[p * u + o % p];
    }
  }
  return ts_axis_create(n_in, n_out, l, first.data(), w.data(), flags, device, out);
}

ts_status ts_axis_get_info(const ts_axis* a, ts_axis_info* info) {
  if (!a || !info) return set_error(TS_ERR_INVALID, "ts_axis_get_info: null argument");
  info->n_in = a->n_in;
  info->n_out = a->n_out;
  info->taps = a->taps;
  info->window = a->K;
  info->blocks = a->nb;
  info->unique_tiles = a->ntiles;
  info->row_span = a->row_span;
  info->col_blocks = a->col_nbt;
  info->col_span = a->col_span;
  return TS_OK;
}

ts_status ts_axis_dense(const ts_axis* a, float* out_host) {
  if (!a || !out_host) return set_error(TS_ERR_INVALID, "ts_axis_dense: null argument");
  std::fill(out_host, out_host + static_cast<size_t>(a->n_out) * a->n_in, 0.0f);
  const size_t tile_elems = static_cast<size_t>(a->K) * kBlockN;
  for (int b = 0; b < a->nb; ++b) {
    const uint16_t* t = a->tiles.data() + static_cast<size_t>(a->tid[b]) * tile_elems;
    for (int n = 0; n < kBlockN; ++n) {
      int o = b * kBlockN + n;
      if (o >= a->n_out) break;
      for (int k = 0; k < a->K; ++k) {
        int i = a->ws[b] + k;
        float v = bf16_bits_to_f32(t[btile_offset(a->K, k, n) / 2]);
        if (v == 0.0f) continue;
        if (i < 0 || i >= a->n_in)
          return set_error(TS_ERR_INVALID, "internal: nonzero weight outside the image");
        out_host[static_cast<size_t>(o) * a->n_in + i] = v;
      }
    }
  }
  return TS_OK;
}

}  // extern "C"

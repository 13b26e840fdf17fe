// merge.cpp — super-block form of an axis for the fused separable kernel.
//
// m consecutive 16-output blocks become one N = 16·m block whose window
// starts at the first block's window and spans all m windows; its B tile
// (K_m x 16m, same K-major core-matrix layout) holds block j's weights in
// columns 16j..16j+15, shifted down by that block's window offset.  One
// M = 128, N = 16m MMA then replaces m MMAs that re-read overlapping rows
// of the same A operand: for a 31-tap Gaussian (windows of 48 inputs every
// 16) four blocks cost 6 K-steps instead of 4 x 3, i.e. 33% fewer
// shared-memory operand bytes and half the MMAs.  Values are copied from
// the axis' bf16 block tiles, so results are identical up to f32
// summation order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "common.h"

namespace tsb {

namespace {
std::mutex g_merge_mu;
}

const MergedAxis* axis_merged(const ts_axis* a, int m) {
  if (m <= 1 || m > kMaxMerge) return nullptr;
  std::lock_guard<std::mutex> lock(g_merge_mu);
  if (a->merged[m]) return a->merged[m];
  MergedAxis* M = new MergedAxis();
  a->merged[m] = M;
  M->m = m;
  const int nbp = static_cast<int>(a->ws.size());  // real blocks + padding
  const int ng = (nbp + m - 1) / m;
  // window of each super-block
  int need = 0;
  for (int g = 0; g < ng; ++g)
    for (int j = 0; j < m && g * m + j < nbp; ++j)
      need = std::max(need, a->ws[g * m + j] - a->ws[g * m] + a->K);
  M->K = (need + 15) / 16 * 16;
  M->tile_bytes = M->K * 16 * m * 2;
  M->ng = ng;
  const size_t elems = static_cast<size_t>(M->K) * 16 * m;
  std::map<std::string, int> ids;
  std::vector<uint16_t> tile(elems);
  M->ws.resize(ng);
  M->tid.resize(ng);
  {
    std::vector<uint16_t> zero(elems, 0);
    ids[std::string(reinterpret_cast<const char*>(zero.data()), elems * 2)] = 0;
    M->tiles.insert(M->tiles.end(), zero.begin(), zero.end());
  }
  for (int g = 0; g < ng; ++g) {
    std::fill(tile.begin(), tile.end(), 0);
    const int ws0 = a->ws[g * m];
    for (int j = 0; j < m && g * m + j < nbp; ++j) {
      const int b = g * m + j;
      const int sh = a->ws[b] - ws0;
      const uint16_t* src = a->tiles.data() + static_cast<size_t>(a->tid[b]) * a->K * kBlockN;
      for (int n = 0; n < kBlockN; ++n)
        for (int k = 0; k < a->K; ++k)
          tile[btile_offset(M->K, k + sh, 16 * j + n) / 2] = src[btile_offset(a->K, k, n) / 2];
    }
    std::string key(reinterpret_cast<const char*>(tile.data()), elems * 2);
    auto it = ids.find(key);
    int id;
    if (it == ids.end()) {
      id = static_cast<int>(ids.size());
      ids.emplace(std::move(key), id);
      M->tiles.insert(M->tiles.end(), tile.begin(), tile.end());
    } else {
      id = it->second;
    }
    M->ws[g] = ws0;
    M->tid[g] = id;
  }
  M->ntiles = static_cast<int>(ids.size());
  M->tab.resize(ng);
  for (int g = 0; g < ng; ++g)
    M->tab[g] = static_cast<int32_t>(static_cast<uint32_t>(M->ws[g]) << 16) |
                static_cast<int32_t>(M->tid[g] & 0xFFFF);
  M->ok = a->tab_ok && M->ntiles <= 65535;
  if (!M->ok) return M;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(a->device) != cudaSuccess ||
      cudaMalloc(&M->d_tab, M->tab.size() * 4) != cudaSuccess ||
      cudaMalloc(&M->d_tiles, M->tiles.size() * 2) != cudaSuccess ||
      cudaMemcpy(M->d_tab, M->tab.data(), M->tab.size() * 4, cudaMemcpyHostToDevice) !=
          cudaSuccess ||
      cudaMemcpy(M->d_tiles, M->tiles.data(), M->tiles.size() * 2, cudaMemcpyHostToDevice) !=
          cudaSuccess)
    M->ok = false;
  cudaSetDevice(prev);
  return M;
}

// Shared-memory operand bytes one tile's MMAs read for `blocks` blocks at
// merge factor m (A: 4 KB per K-step, B: the K_m x 16m tile).
static double operand_bytes(int K, int blocks, int m) {
  return static_cast<double>(blocks / m) * ((K / 16) * 4096.0 + K * 16.0 * m * 2.0);
}

int choose_merge(const ts_axis* a, int blocks) {
  if (std::getenv("TSB_NO_MERGE")) return 1;
  const char* th = std::getenv("TSB_MERGE_GAIN");  // required saving (default 0.05)
  const double keep = 1.0 - (th ? std::atof(th) : 0.05);
  int best = 1;
  double best_cost = operand_bytes(a->K, blocks, 1);
  for (int m = 2; m <= kMaxMerge && m <= blocks; ++m) {
    if (blocks % m) continue;
    const MergedAxis* M = axis_merged(a, m);
    if (!M || !M->ok || M->K > 256) continue;
    const double c = operand_bytes(M->K, blocks, m);
    if (c < keep * best_cost) {  // only merge for a clear saving
      best = m;
      best_cost = c;
    }
  }
  return best;
}

}  // namespace tsb

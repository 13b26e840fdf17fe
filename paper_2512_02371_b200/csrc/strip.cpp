// strip.cpp — builds the shift-invariant strip form of an axis for the v5
// separable kernel (separable_strip.cu).
//
// For a Toeplitz-like axis (16-output blocks whose windows advance by a
// constant S inputs), the operand slice a tile needs for K-step q (16
// consecutive inputs) is the same banded pattern shifted by 256/S outputs:
//     slice_q[o][kk] = W(o0 + o, in0 + 16q + kk) = strip[o - shift*q][kk]
// so one strip (plus a handful of edge slices where clamp-to-edge folding
// or the image border breaks the pattern) replaces the per-block B tiles.
// Values are read from the same bf16 block tiles the v4 kernel uses, so both
// kernels compute with identical weights.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "common.h"

namespace tsb {

namespace {
std::mutex g_strip_mu;

float bf16f(uint16_t h) {
  uint32_t b = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

// Effective weight (bf16 bits) of output o on input i (0 if outside the band).
uint16_t weight_bits(const ts_axis* a, int o, int i) {
  if (o < 0 || o >= a->n_out) return 0;
  const int b = o / kBlockN, n = o % kBlockN;
  const int k = i - a->ws[b];
  if (k < 0 || k >= a->K) return 0;
  const uint16_t* t = a->tiles.data() + static_cast<size_t>(a->tid[b]) * a->K * kBlockN;
  return t[btile_offset(a->K, k, n) / 2];
}

inline int slot_off(int row, int kk) {  // K-major core matrices, 16 K per slice
  return (row / 8) * 128 + (kk / 8) * 64 + (row % 8) * 8 + (kk % 8);  // in elements
}
}  // namespace

// Build (once) the strip plan of axis `a` for `role` (0 rows, 1 cols).
StripPlan* strip_plan(const ts_axis* a, int role) {
  std::lock_guard<std::mutex> lock(g_strip_mu);
  if (a->strip[role]) return a->strip[role];
  StripPlan* P = new StripPlan();
  a->strip[role] = P;
  P->role = role;
  const int nb = a->nb;
  if (nb < 3) {
    P->why = "axis too short";
    return P;
  }
  const int S = a->ws[1] - a->ws[0];
  for (int b = 1; b + 1 < nb; ++b)
    if (a->ws[b + 1] - a->ws[b] != S) {
      P->why = "non-uniform block spacing";
      return P;
    }
  if (S <= 0 || 256 % S || ((256 / S) % 8)) {
    P->why = "block spacing must be 8, 16 or 32 inputs";
    return P;
  }
  P->S = S;
  P->shift = 256 / S;  // outputs per 16 inputs
  int nblk;            // 16-output blocks per tile
  if (role == 0) {
    nblk = kRowBlocksPerTile;
    const int span = (nblk - 1) * S + a->K;
    P->Q = (span + 15) / 16;
    P->staged = 0;
  } else {
    // as many blocks as fit 256 staged input columns, N <= 256
    nblk = 0;
    for (int n = 16; n >= 1; --n) {
      if ((n - 1) * S + a->K <= 256) {
        nblk = n;
        break;
      }
    }
    if (nblk < 1) {
      P->why = "window too wide for a 256-column strip";
      return P;
    }
    const int span = (nblk - 1) * S + a->K;
    P->Q = (span + 15) / 16;
    P->staged = (span + 63) / 64 * 64;
  }
  P->nout = nblk * kBlockN;
  P->ntiles = (nb + nblk - 1) / nblk;
  P->G = (P->shift * (P->Q - 1) + 7) / 8;
  if (P->shift * (P->Q - 1) % 8) {
    P->why = "shift not a multiple of 8";
    return P;
  }
  const int rows = P->nout + 8 * P->G;
  // reference tile: the middle one (interior, no clamp folding)
  const int tref = P->ntiles / 2;
  const int o_ref = tref * P->nout;
  const int in_ref = a->ws[tref * nblk];
  P->strip.assign(static_cast<size_t>(rows) * 16, 0);
  for (int r = 0; r < rows; ++r)
    for (int kk = 0; kk < 16; ++kk)
      P->strip[slot_off(r, kk)] = weight_bits(a, o_ref + r - 8 * P->G, in_ref + kk);
  // per tile and K-step: strip shift or a special slice
  P->first_in.resize(P->ntiles);
  P->map.assign(static_cast<size_t>(P->ntiles) * P->Q, -1);
  std::map<std::string, int> dedup;
  const size_t slice = static_cast<size_t>(P->nout) * 16;
  std::vector<uint16_t> buf(slice);
  for (int t = 0; t < P->ntiles; ++t) {
    const int o0 = t * P->nout;
    const int i0 = a->ws[t * nblk];
    P->first_in[t] = i0;
    for (int q = 0; q < P->Q; ++q) {
      bool same = true;
      for (int o = 0; o < P->nout; ++o) {
        const bool valid = o0 + o < a->n_out;
        for (int kk = 0; kk < 16; ++kk) {
          const uint16_t w = weight_bits(a, o0 + o, i0 + 16 * q + kk);
          const int srow = o - P->shift * q + 8 * P->G;
          const uint16_t sw = (srow >= 0 && srow < rows) ? P->strip[slot_off(srow, kk)] : 0;
          buf[slot_off(o, kk)] = valid ? w : sw;  // invalid outputs: anything (clipped)
          if (valid && w != sw) same = false;
        }
      }
      if (same) continue;
      std::string key(reinterpret_cast<const char*>(buf.data()), slice * 2);
      auto it = dedup.find(key);
      int id;
      if (it == dedup.end()) {
        id = static_cast<int>(dedup.size());
        if (id >= 127) {
          P->why = "too many edge slices";
          return P;
        }
        dedup.emplace(std::move(key), id);
        P->specials.insert(P->specials.end(), buf.begin(), buf.end());
      } else {
        id = it->second;
      }
      P->map[static_cast<size_t>(t) * P->Q + q] = static_cast<int8_t>(id);
    }
  }
  P->nspec = static_cast<int>(dedup.size());
  // device copies
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(a->device) != cudaSuccess ||
      cudaMalloc(&P->d_strip, P->strip.size() * 2) != cudaSuccess ||
      cudaMemcpy(P->d_strip, P->strip.data(), P->strip.size() * 2, cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaSetDevice(prev);
    P->why = "device upload failed";
    return P;
  }
  if (P->nspec) {
    if (cudaMalloc(&P->d_specials, P->specials.size() * 2) != cudaSuccess ||
        cudaMemcpy(P->d_specials, P->specials.data(), P->specials.size() * 2,
                   cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaSetDevice(prev);
      P->why = "device upload failed";
      return P;
    }
  }
  cudaSetDevice(prev);
  P->ok = true;
  return P;
}

}  // namespace tsb

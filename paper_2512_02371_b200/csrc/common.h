// common.h — internal types shared by the builder, the C ABI glue and the kernels.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <string>
#include <atomic>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/tensorsel_b200.h"

namespace tsb {

// One 16-output block per MMA N-tile.
constexpr int kBlockN = 16;
// Extra (ws, tid) entries past the last real block so tiles whose block range
// overhangs the axis read a harmless zero block (window = last window).
constexpr int kBlockPad = 64;
// pass-1 (rows) tile = 8 blocks = 128 output rows = the M of pass 2
constexpr int kRowBlocksPerTile = 8;
// pass-1 MMA M = 128 input columns staged per tile
constexpr int kColTile = 128;
// TMA boxes are at most 256 rows; a row tile is staged as two boxes
constexpr int kMaxRowSpan = 512;
constexpr int kMaxColBlocks = 16;  // pass-2 output blocks per tile (D_H: 256 TMEM columns)
constexpr int kMaxWindow = 1024;  // inputs per 16-output block (axis_pass streams K)

// Device-facing view of an axis (passed by value into kernels).
struct AxisDev {
  const int32_t* ws;      // window start (input index, multiple of 8) per block
  const int32_t* tid;     // B-tile id per block (0 = the all-zero tile)
  const int32_t* tab;     // packed per block: (ws << 16) | tid
  const uint8_t* tiles;   // ntiles * tile_bytes, tcgen05 K-major no-swizzle layout
  int K;                  // window length, multiple of 16
  int nb;                 // real block count
  int tile_bytes;         // K * 16 * 2
  int ntiles;             // distinct tiles (tile 0 is all zeros)
};

}  // namespace tsb

namespace tsb {
constexpr int kMaxMerge = 8;  // 16-output blocks per super-block (merge.cpp)

// Super-block form of an axis (csrc/merge.cpp): m blocks -> one N = 16m block.
struct MergedAxis {
  bool ok = false;
  int m = 1, K = 0, tile_bytes = 0, ng = 0, ntiles = 0;
  std::vector<int32_t> ws, tid, tab;  // per super-block (padding included)
  std::vector<uint16_t> tiles;        // ntiles x (K x 16m) bf16, K-major core matrices
  int32_t* d_tab = nullptr;
  uint8_t* d_tiles = nullptr;
};

}  // namespace tsb

namespace tsb {
// process-unique axis id (launch-parameter caches key on it, never on the
// pointer, which the allocator may reuse)
inline uint64_t next_axis_uid() {
  static std::atomic<uint64_t> n{1};
  return n.fetch_add(1);
}
// Launch with programmatic stream serialization (PDL): the kernel's CTAs may
// be scheduled while the previous kernel in the stream finishes, running
// their prologue (barrier init, TMEM allocation) until pdl_wait().  Every
// image kernel calls pdl_wait() before touching global memory and
// pdl_launch_dependents() right after.  TSB_PDL=0 launches plainly.
template <typename... Exp, typename... Act>
inline cudaError_t launch_pdl(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Act&&... args) {
  static const bool on = [] {
    const char* e = std::getenv("TSB_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

}  // namespace tsb

struct ts_axis {
  uint64_t uid = tsb::next_axis_uid();
  int n_in = 0, n_out = 0, taps = 0;
  int K = 0, nb = 0, ntiles = 0, tile_bytes = 0;
  int row_span = 0;            // rows staged per pass-1 tile (multiple of 16)
  int col_nbt = 0, col_span = 0;
  std::vector<int32_t> ws, tid;     // nb + kBlockPad entries
  std::vector<uint16_t> tiles;      // host copy of the bf16 tiles
  int device = 0;
  int32_t* d_ws = nullptr;
  int32_t* d_tid = nullptr;
  int32_t* d_tab = nullptr;
  uint8_t* d_tiles = nullptr;
  std::vector<int32_t> tab;         // packed (ws << 16) | tid, nb + kBlockPad entries
  bool tab_ok = true;               // packing fits (|ws| < 32K, < 64K tiles)
  mutable tsb::MergedAxis* merged[tsb::kMaxMerge + 1] = {};  // lazily built per factor

  tsb::AxisDev dev() const {
    return tsb::AxisDev{d_ws, d_tid, d_tab, d_tiles, K, nb, tile_bytes, ntiles};
  }
};

namespace tsb {
ts_status set_error(ts_status st, const char* fmt, ...);
ts_status cuda_error(int err, const char* what);

// Scoped current-device switch: an entry point runs on the device its
// operands live on and leaves the caller's current device as it found it.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Device that owns a device pointer (-1 if the runtime does not know it).
inline int device_of(const void* p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ? a.device : -1;
}
// Byte offset of element (k, n) inside a K x 16 B tile (K-major, no swizzle:
// 8x8 core matrices of 128 contiguous bytes; LBO = 128 B between k-chunks,
// SBO = K*16 B between the two 8-column groups).
inline int btile_offset(int K, int k, int n) {
  return (n / 8) * (K * 16) + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
}
}  // namespace tsb

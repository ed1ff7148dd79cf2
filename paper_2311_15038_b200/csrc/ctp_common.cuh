// Shared helpers for the ctprev B200 kernels: error plumbing for the C ABI,
// launch accounting, level addressing (volume / slicemap atlas layouts).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/ctprev_b200.h"

namespace ctp {

constexpr int kNumSMs = 148;  // B200; re-queried at runtime for grid sizing

// ---- error plumbing: thread-local message, status codes, never throw ----
void set_error(const char* fmt, ...);
int64_t& launch_counter();
int num_sms();

#define CTP_REQUIRE(cond, code, ...)            \
  do {                                          \
    if (!(cond)) {                              \
      ::ctp::set_error(__VA_ARGS__);            \
      return (code);                            \
    }                                           \
  } while (0)

#define CTP_CUDA_CHECK_LAUNCH(name)                                        \
  do {                                                                     \
    cudaError_t e_ = cudaGetLastError();                                   \
    if (e_ != cudaSuccess) {                                               \
      ::ctp::set_error("%s: %s", (name), cudaGetErrorString(e_));          \
      return CTP_E_CUDA;                                                   \
    }                                                                      \
    ++::ctp::launch_counter();                                             \
  } while (0)

#define CTP_CUDA_CALL(expr)                                                \
  do {                                                                     \
    cudaError_t e_ = (expr);                                               \
    if (e_ != cudaSuccess) {                                               \
      ::ctp::set_error("%s: %s", #expr, cudaGetErrorString(e_));           \
      return CTP_E_CUDA;                                                   \
    }                                                                      \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- level destination addressing ---------------------------------------
// Device-side copy of ctp_level_out plus the level's dense dims.
struct LevelDst {
  uint8_t* out;
  int32_t layout;
  int32_t s, grid, atlas_dim;
  int32_t gshift;          // log2(grid) when grid is a power of two, else -1 (dense: 0)
  int32_t z_off;           // added to the slab-local z: global slice index for atlases, 0 for dense
  int64_t nx, ny;          // level dims (x, y) for the dense layout
  int64_t map_bytes;       // atlas_dim^2 (dense: bytes per slice)
  int32_t row;             // bytes between rows (atlas_dim, or nx for dense)
  int32_t cell_row;        // s * atlas_dim (dense: 0)
  int32_t cell_col;        // s (dense: 0)
  int32_t gmask;           // grid - 1 (dense: 0)
};

// Byte offset of level voxel (z, y, x), z slab-local (z_off makes it the
// global slice index for atlases).  Atlas: slicemap.py:79-85 (slice_cell) and the mosaic of
// slicemap.py:139-140: atlas[m][cy*s + y, cx*s + x] = cube[m*g^2 + cy*g + cx, y, x].
// POW2: power-of-two grid -- branch-free shifts/masks; a dense level is the
// degenerate 1x1-grid atlas whose "maps" are its slices.
template <bool POW2 = false>
__device__ __forceinline__ int64_t level_offset(const LevelDst& d, int z, int y, int x) {
  z += d.z_off;
  if (POW2) {
    return (int64_t)(z >> (2 * d.gshift)) * d.map_bytes +
           (int64_t)(((z >> d.gshift) & d.gmask) * d.cell_row + (z & d.gmask) * d.cell_col + y * d.row + x);
  }
  if (d.layout == CTP_LAYOUT_ATLAS) {
    int m, cy, cx;
    if (d.gshift >= 0) {
      const int w = z & ((1 << (2 * d.gshift)) - 1);
      m = z >> (2 * d.gshift);
      cy = w >> d.gshift;
      cx = w & (d.grid - 1);
    } else {
      const int per = d.grid * d.grid;
      m = z / per;
      const int w = z - m * per;
      cy = w / d.grid;
      cx = w - cy * d.grid;
    }
    return (int64_t)m * d.map_bytes + (int64_t)(cy * d.s + y) * d.atlas_dim + (cx * d.s + x);
  }
  return ((int64_t)z * d.ny + y) * d.nx + x;
}

// Store 8 consecutive level bytes (x .. x+7 on one row): one 8-byte store
// when aligned, else bytewise.  Rows of one level never straddle cells
// because a cell row is s >= 8 contiguous bytes when s % 8 == 0.
__device__ __forceinline__ void store8(uint8_t* p, uint32_t lo, uint32_t hi) {
  if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
    *reinterpret_cast<uint2*>(p) = make_uint2(lo, hi);
  } else {
#pragma unroll
    for (int i = 0; i < 4; i++) p[i] = (uint8_t)(lo >> (8 * i));
#pragma unroll
    for (int i = 0; i < 4; i++) p[4 + i] = (uint8_t)(hi >> (8 * i));
  }
}

inline LevelDst make_dst(const ctp_level_out& lo, int64_t nx, int64_t ny, int64_t z_off_atlas = 0) {
  LevelDst d;
  d.out = lo.out;
  d.layout = lo.layout;
  d.s = lo.s;
  d.grid = lo.grid;
  d.atlas_dim = lo.atlas_dim;
  d.nx = nx;
  d.ny = ny;
  if (lo.layout == CTP_LAYOUT_ATLAS) {
    d.z_off = (int32_t)z_off_atlas;
    d.gshift = -1;
    if (lo.grid > 0 && (lo.grid & (lo.grid - 1)) == 0) {
      d.gshift = 0;
      while ((1 << d.gshift) < lo.grid) d.gshift++;
    }
    d.map_bytes = (int64_t)lo.atlas_dim * lo.atlas_dim;
    d.row = lo.atlas_dim;
    d.cell_row = lo.s * lo.atlas_dim;
    d.cell_col = lo.s;
    d.gmask = lo.grid - 1;
  } else {  // dense level == 1x1-grid atlas of slices
    d.z_off = 0;
    d.gshift = 0;
    d.map_bytes = nx * ny;
    d.row = (int32_t)nx;
    d.cell_row = 0;
    d.cell_col = 0;
    d.gmask = 0;
  }
  return d;
}

inline bool dst_is_pow2(const LevelDst& d) { return d.out == nullptr || d.gshift >= 0; }

// Host-side validation of an atlas descriptor (slicemap.py:52-61) against
// the level dims it will receive (_pad_to_cube: every dim <= s).
int check_level_desc(const ctp_level_out& lo, int64_t lnx, int64_t lny, int64_t lnz_global, int level);

}  // namespace ctp

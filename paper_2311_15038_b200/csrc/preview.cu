// The fused preview pass: histogram (kernel 1) + LUT filter / 16->8 rescale
// (kernel 2) + exact multi-level 2x2x2 mean pyramid (kernel 3) + slicemap
// atlas writes (kernel 4) in ONE read of the volume.
//
// Reference semantics reproduced (paths under /root/reference/pkg/src/ctprev):
//   hist     = volume_histogram(v)                      volume.py:252-262
//   f        = lut[v]                                   mask.py:246 (LUT: mask.py:241-245)
//   level l  = downscale_volume(f, (nx>>l, ny>>l, nz>>l)) volume.py:277-309
//              -- every level straight from full resolution (pipeline.py:275):
//              exact integer block sums carried up the levels, rounded half up
//              once per level as (sum + 2^(3l-1)) >> 3l  ==  (2acc+cnt)//(2cnt).
//   atlases  = encode_slicemaps(level, scheme) packing  slicemap.py:120-142
//              (+ _pad_to_cube, pipeline.py:226-237, for levels smaller than s)
//
// Work decomposition (B200: 148 SMs, persistent CTAs of 256 threads):
//   * a TILE is 2^L z-slices x (ky*2^L) rows x (TXu*UXW) columns, <= 1024 UNITS,
//     tiles walked in memory order;
//   * a UNIT is UXW x-voxels (one 16-byte vector: 16 u8 or 8 u16) on 2 rows x
//     2 slices (L >= 1) -- exactly the 2x2x2 cells of level 1 along one vector.
//     Each thread owns the same 4 unit slots in every tile (coordinates computed
//     once), loaded as 16-byte vectors, 4 or 8 in flight per thread;
//   * histogram + LUT in ONE shared-memory atomic per voxel: the counter word
//     holds lut[v] in bits 0..7 and the count in bits 12..31; atom.add(+4096)
//     returns the old word whose low byte is f = lut[v].  Summing the 8 old
//     words of a level-1 cell and masking 12 bits gives sum(f) exactly (<= 2040).
//     Per voxel the hot loop is PRMT (byte) + LEA (address) + ATOMS + 1/2 IADD3.
//     u8 tables: per-lane columns [bin][lane] (bank == lane: conflict-free for
//     any data) or warp-private [warp][bin] (same-address lanes merge: faster on
//     concentrated histograms); u16: one 4096-word table per CTA;
//   * level-1 sums go to shared memory; levels 2..L are reduced from there
//     (u16 / u32 sums) and written as coalesced row segments.
#include <stdlib.h>
#include "ctp_common.cuh"

namespace ctp {

constexpr int kPvThreads = 256;
constexpr int kMaxUnits = 1024;                 // per tile
constexpr int kUnitsPerThread = kMaxUnits / kPvThreads;
constexpr uint32_t kOne = 1u << 12;             // count increment
constexpr uint32_t kCountCap = (1u << 20) - 1;  // 20-bit count field
constexpr int kCellSlots = 4;                   // level-2 cells per thread per tile (<= 1024 / 256)

enum { kLaneCols = 0, kWarpPriv = 1 };

template <typename T> struct Vox;
template <> struct Vox<uint8_t> {
  static constexpr int UXW = 16, NBINS = 256;
};
template <> struct Vox<uint16_t> {
  static constexpr int UXW = 8, NBINS = 4096;
};

template <typename T, int LAYOUT>
struct Table {
  static constexpr int WORDS = sizeof(T) == 2 ? 4096 : (LAYOUT == kLaneCols ? 256 * 32 : 256 * (kPvThreads / 32));
};

struct PvGeom {
  int64_t nx, ny, nz, z_base;
  int32_t txu;          // units per tile along x
  int32_t ty;           // rows per tile (multiple of 2^L)
  int32_t tiles_x, tiles_y, n_tiles;
  int32_t flush_tiles;  // flush the smem counters every this many tiles
};

struct PvArgs {
  const void* vol;
  const uint8_t* lut;
  unsigned long long* hist;
  LevelDst lv[CTP_MAX_LEVELS];
  PvGeom g;
};

__device__ __forceinline__ uint32_t atom_add_shared(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}

template <typename T, int LAYOUT>
__device__ void flush_counts(uint32_t* hs, unsigned long long* hist) {
  __syncthreads();
  if constexpr (sizeof(T) == 1) {
    const int bin = threadIdx.x;  // 256 threads == 256 bins
    uint32_t s = 0;
    constexpr int COPIES = LAYOUT == kLaneCols ? 32 : kPvThreads / 32;
#pragma unroll 8
    for (int k = 0; k < COPIES; k++) {
      const int idx = LAYOUT == kLaneCols ? bin * 32 + ((k + bin) & 31) : k * 256 + bin;
      const uint32_t wv = hs[idx];
      s += wv >> 12;
      hs[idx] = wv & 0xFFFu;
    }
    if (s && hist) atomicAdd(hist + bin, (unsigned long long)s);
  } else {
    for (int b = threadIdx.x; b < 4096; b += kPvThreads) {
      const uint32_t wv = hs[b];
      if ((wv >> 12) && hist) atomicAdd(hist + b, (unsigned long long)(wv >> 12));
      hs[b] = wv & 0xFFFu;
    }
  }
  __syncthreads();
}

// One 16-byte row vector of a unit: UXW atomics; returns the old counter words.
template <typename T, int LAYOUT>
__device__ __forceinline__ void row_atomics(const uint4& q, uint32_t lb, uint32_t* o) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  if constexpr (sizeof(T) == 1) {
    constexpr int SH = LAYOUT == kLaneCols ? 7 : 2;  // bytes per bin row: 32 lanes x 4 B, or 4 B
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const uint32_t v = __byte_perm(w[k], 0u, 0x4440u | (uint32_t)b);
        o[4 * k + b] = atom_add_shared(lb + (v << SH), kOne);
      }
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      o[2 * k] = atom_add_shared(lb + (min(w[k] & 0xFFFFu, 4095u) << 2), kOne);
      o[2 * k + 1] = atom_add_shared(lb + (min(w[k] >> 16, 4095u) << 2), kOne);
    }
  }
}

template <typename T, int L, int MINB, int kBatch, int LAYOUT>
__global__ void __launch_bounds__(kPvThreads, MINB) preview_kernel(const PvArgs a) {
  constexpr int UXW = Vox<T>::UXW;
  constexpr int HW = Table<T, LAYOUT>::WORDS;
  constexpr int UZ = (L == 0) ? 1 : 2;
  constexpr int ROWS = UZ * UZ;
  constexpr int TZ = 1 << L;
  constexpr int L1PU = UXW / 2;  // level-1 sums per unit

  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* hs = smem;                                          // HW counter words
  uint16_t* s1 = reinterpret_cast<uint16_t*>(smem + HW);        // level-1 sums
  uint32_t* s2 = reinterpret_cast<uint32_t*>(s1 + kMaxUnits * L1PU);  // level-2 sums
  uint32_t* s3 = s2 + kMaxUnits * L1PU / 8;                     // level-3 sums

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const PvGeom& g = a.g;

  // counter words: LUT value in the low byte, count 0
  for (int i = threadIdx.x; i < HW; i += kPvThreads) {
    int bin;
    if constexpr (sizeof(T) == 2) bin = i;
    else bin = (LAYOUT == kLaneCols) ? (i >> 5) : (i & 255);
    hs[i] = a.lut ? (uint32_t)a.lut[bin] : (uint32_t)min(bin, 255);
  }
  // this thread's table base in the shared window
  const uint32_t tbl = (uint32_t)__cvta_generic_to_shared(hs);
  uint32_t lb;
  if constexpr (sizeof(T) == 2) lb = tbl;
  else lb = (LAYOUT == kLaneCols) ? tbl + 4u * (uint32_t)lane : tbl + 1024u * (uint32_t)warp;
  __syncthreads();

  const int rows_u = g.ty / UZ;               // unit rows along y in a tile
  const int units = (TZ / UZ) * rows_u * g.txu;
  const int xw = g.txu * UXW;                 // tile width in voxels
  const int64_t sy = g.nx, sz = g.nx * g.ny;
  const T* __restrict__ vol = reinterpret_cast<const T*>(a.vol);

  // unit slots of this thread: identical in every tile
  int uxu[kUnitsPerThread], uyr[kUnitsPerThread], uzr[kUnitsPerThread];
  int64_t uoff[kUnitsPerThread];
#pragma unroll
  for (int i = 0; i < kUnitsPerThread; i++) {
    const int u = threadIdx.x + kPvThreads * i;
    uxu[i] = u % g.txu;
    const int r = u / g.txu;
    uyr[i] = r % rows_u;
    uzr[i] = u < units ? r / rows_u : TZ;   // TZ marks "slot unused"
    uoff[i] = (int64_t)(uzr[i] * UZ) * sz + (int64_t)(uyr[i] * UZ) * sy + uxu[i] * UXW;
  }

  // level-2..L cell slots of this thread (packed xq | yq << 12 | zq << 24; -1 = none),
  // kept in shared memory [slot][thread] to spare registers
  int* cslot = reinterpret_cast<int*>(s3 + kMaxUnits * L1PU / 64 + 4);
  if constexpr (L >= 2) {
#pragma unroll
    for (int sl = 0; sl < kCellSlots + 2; sl++) {
      const int l = sl < kCellSlots ? 2 : sl - kCellSlots + 3;
      const int k = sl < kCellSlots ? sl : 0;
      int code = -1;
      if (l <= L) {
        const int nzc = TZ >> l, nyc = g.ty >> l, nxc = xw >> l;
        const int c = threadIdx.x + kPvThreads * k;
        if (c < nzc * nyc * nxc) {
          const int xq = c % nxc, yq = (c / nxc) % nyc, zq = c / (nxc * nyc);
          code = xq | (yq << 12) | (zq << 24);
        }
      }
      cslot[sl * kPvThreads + threadIdx.x] = code;
    }
  }

  int since_flush = 0;
  for (int tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
    const int tx_i = tile % g.tiles_x;
    const int rest = tile / g.tiles_x;
    const int ty_i = rest % g.tiles_y;
    const int tz_i = rest / g.tiles_y;
    const int x0 = tx_i * xw, y0 = ty_i * g.ty, z0 = tz_i * TZ;
    const T* tile_base = vol + (int64_t)z0 * sz + (int64_t)y0 * sy + x0;

#pragma unroll
    for (int bt = 0; bt < kUnitsPerThread; bt += kBatch) {
      uint4 q[kBatch][ROWS];
      bool ok[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; i++) {
        const int s = bt + i;
        ok[i] = (uzr[s] < TZ / UZ) && (x0 + uxu[s] * UXW < g.nx) && (y0 + uyr[s] * UZ < g.ny);
        if (ok[i]) {
          const T* p = tile_base + uoff[s];
#pragma unroll
          for (int r2 = 0; r2 < ROWS; r2++)
            q[i][r2] = __ldcs(reinterpret_cast<const uint4*>(p + (r2 / UZ) * sz + (r2 % UZ) * sy));
        }
      }

#pragma unroll
      for (int i = 0; i < kBatch; i++) {
        if (!ok[i]) continue;
        const int s = bt + i;
        const int xu = uxu[s], yr = uyr[s], zr = uzr[s];
        const int x = x0 + xu * UXW, y = y0 + yr * UZ, z = z0 + zr * UZ;
        uint32_t acc[L1PU];
#pragma unroll
        for (int j = 0; j < L1PU; j++) acc[j] = 0;
#pragma unroll
        for (int r2 = 0; r2 < ROWS; r2++) {
          uint32_t o[UXW];
          row_atomics<T, LAYOUT>(q[i][r2], lb, o);
          if (a.lv[0].out) {  // level 0: the filtered voxels themselves
            uint8_t* dst = a.lv[0].out + level_offset(a.lv[0], z + r2 / UZ, y + r2 % UZ, x);
            uint32_t pk[UXW / 4];
#pragma unroll
            for (int k = 0; k < UXW / 4; k++)
              pk[k] = __byte_perm(__byte_perm(o[4 * k], o[4 * k + 1], 0x0040),
                                  __byte_perm(o[4 * k + 2], o[4 * k + 3], 0x0040), 0x5410);
            if constexpr (UXW == 16) {
              if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)
                *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              else {
                store8(dst, pk[0], pk[1]);
                store8(dst + 8, pk[2], pk[3]);
              }
            } else {
              store8(dst, pk[0], pk[1]);
            }
          }
          if constexpr (L >= 1) {
#pragma unroll
            for (int j = 0; j < L1PU; j++) acc[j] += o[2 * j] + o[2 * j + 1];
          }
        }
        if constexpr (L >= 1) {
          uint32_t sum[L1PU];
#pragma unroll
          for (int j = 0; j < L1PU; j++) sum[j] = acc[j] & 0xFFFu;  // sum of f over the 2x2x2 cell (<= 2040)
          if (a.lv[1].out) {
            uint32_t pk[L1PU / 4];
#pragma unroll
            for (int k = 0; k < L1PU / 4; k++)
              pk[k] = ((sum[4 * k] + 4) >> 3) | (((sum[4 * k + 1] + 4) >> 3) << 8) |
                      (((sum[4 * k + 2] + 4) >> 3) << 16) | (((sum[4 * k + 3] + 4) >> 3) << 24);
            uint8_t* dst = a.lv[1].out + level_offset(a.lv[1], z >> 1, y >> 1, x >> 1);
            if constexpr (L1PU == 8) {
              store8(dst, pk[0], pk[1]);
            } else {
              if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) *reinterpret_cast<uint32_t*>(dst) = pk[0];
              else for (int b = 0; b < 4; b++) dst[b] = (uint8_t)(pk[0] >> (8 * b));
            }
          }
          if constexpr (L >= 2) {
            // s1 layout [zr][yr][x1], x1 = xu*L1PU + j
            uint16_t* d = s1 + ((zr * rows_u + yr) * g.txu + xu) * L1PU;
            if constexpr (L1PU == 8)
              *reinterpret_cast<uint4*>(d) = make_uint4(sum[0] | (sum[1] << 16), sum[2] | (sum[3] << 16),
                                                        sum[4] | (sum[5] << 16), sum[6] | (sum[7] << 16));
            else
              *reinterpret_cast<uint2*>(d) = make_uint2(sum[0] | (sum[1] << 16), sum[2] | (sum[3] << 16));
          }
        }
      }
    }  // batch loop

    // ---- levels 2..L from shared memory ----------------------------------------
    if constexpr (L >= 2) {
      __syncthreads();
#pragma unroll
      for (int l = 2; l <= L; l++) {
        const int cy = g.ty >> (l - 1), cx = xw >> (l - 1);  // child dims (y, x)
        const int lnx = (int)(g.nx >> l), lny = (int)(g.ny >> l);
        const int shift = 3 * l;
        uint32_t* dsts = (l == 2) ? s2 : s3;
        const uint32_t* srcs = (l == 3) ? s2 : s3;
        const bool want = a.lv[l].out != nullptr;
#pragma unroll
        for (int k = 0; k < kCellSlots; k++) {
          if (l > 2 && k > 0) break;
          const int code = cslot[(l == 2 ? k : kCellSlots + l - 3) * kPvThreads + threadIdx.x];
          if (code < 0) continue;
          const int xq = code & 0xFFF, yq = (code >> 12) & 0xFFF, zq = code >> 24;
          const int gx = (x0 >> l) + xq, gy = (y0 >> l) + yq;
          if (gx >= lnx || gy >= lny) continue;
          uint32_t sum = 0;
#pragma unroll
          for (int dz = 0; dz < 2; dz++)
#pragma unroll
            for (int dy = 0; dy < 2; dy++) {
              const int base = ((2 * zq + dz) * cy + (2 * yq + dy)) * cx + 2 * xq;
              if (l == 2) {
                const uint32_t pair = *reinterpret_cast<const uint32_t*>(s1 + base);
                sum += (pair & 0xFFFFu) + (pair >> 16);
              } else {
                sum += srcs[base] + srcs[base + 1];
              }
            }
          if (l < L) dsts[threadIdx.x + kPvThreads * k] = sum;
          if (want)
            a.lv[l].out[level_offset(a.lv[l], (z0 >> l) + zq, gy, gx)] =
                (uint8_t)((sum + (1u << (shift - 1))) >> shift);
        }
        __syncthreads();
      }
    }

    if (++since_flush == g.flush_tiles) {
      since_flush = 0;
      flush_counts<T, LAYOUT>(hs, a.hist);
    }
  }
  flush_counts<T, LAYOUT>(hs, a.hist);
}

template <typename T, int LAYOUT>
static size_t smem_bytes(int L) {
  size_t b = (size_t)Table<T, LAYOUT>::WORDS * 4;
  if (L >= 2) {
    const size_t l1 = (size_t)kMaxUnits * (Vox<T>::UXW / 2);
    b += l1 * 2 + (l1 / 8) * 4 + (l1 / 64) * 4 + 16 + (kCellSlots + 2) * kPvThreads * 4;
  }
  return b;
}

template <typename T, int L, int MINB, int BATCH, int LAYOUT>
static int launch_v(PvArgs a, cudaStream_t st) {
  const size_t sm = smem_bytes<T, LAYOUT>(L);
  auto kern = preview_kernel<T, L, MINB, BATCH, LAYOUT>;
  CTP_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  // a counter word gains at most this many counts per tile
  constexpr int UZ = L == 0 ? 1 : 2;
  const int64_t vox_per_unit = (int64_t)Vox<T>::UXW * UZ * UZ;
  int64_t per_tile;
  if (sizeof(T) == 2) per_tile = (int64_t)kMaxUnits * vox_per_unit;                // whole CTA
  else if (LAYOUT == kLaneCols) per_tile = 8LL * kUnitsPerThread * vox_per_unit;    // one lane of 8 warps
  else per_tile = 32LL * kUnitsPerThread * vox_per_unit;                            // one warp
  a.g.flush_tiles = (int)(kCountCap / per_tile);
  if (a.g.flush_tiles < 1) a.g.flush_tiles = 1;
  int grid = num_sms() * MINB;
  if (a.g.n_tiles < grid) grid = a.g.n_tiles;
  kern<<<grid, kPvThreads, sm, st>>>(a);
  CTP_CUDA_CHECK_LAUNCH("preview_kernel");
  return CTP_OK;
}

// Launch-shape variants, selectable with CTP_PREVIEW_VARIANT for tuning
// (tools/prof_preview.py); the default was the fastest measured on B200.
static int preview_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CTP_PREVIEW_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <typename T, int L>
static int launch_l(const PvArgs& a, cudaStream_t st) {
  if constexpr (sizeof(T) == 1) {
    switch (preview_variant()) {
      case 1: return launch_v<T, L, 3, 1, kLaneCols>(a, st);
      case 2: return launch_v<T, L, 2, 2, kWarpPriv>(a, st);
      case 3: return launch_v<T, L, 3, 1, kWarpPriv>(a, st);
      case 4: return launch_v<T, L, 4, 1, kLaneCols>(a, st);
      default: return launch_v<T, L, 2, 2, kLaneCols>(a, st);
    }
  } else {
    return launch_v<T, L, 2, 2, kLaneCols>(a, st);
  }
}

template <typename T>
static int preview_impl(const T* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut,
                        int nlev, const ctp_level_out* levels, uint64_t* hist, void* stream) {
  constexpr int UXW = Vox<T>::UXW;
  CTP_REQUIRE(vol != nullptr && levels != nullptr, CTP_E_INVALID, "preview: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "preview: degenerate shape");
  CTP_REQUIRE(nx < (1LL << 30) && ny < (1LL << 30) && nz < (1LL << 30), CTP_E_INVALID, "preview: shape too large");
  CTP_REQUIRE(nlev >= 0 && nlev <= 4, CTP_E_INVALID, "preview: nlev %d outside [0, 4]", nlev);
  CTP_REQUIRE((reinterpret_cast<uintptr_t>(vol) & 15) == 0, CTP_E_ALIGN, "preview: volume not 16-byte aligned");
  CTP_REQUIRE(nx % UXW == 0, CTP_E_ALIGN, "preview: nx=%lld not a multiple of %d", (long long)nx, UXW);
  const int64_t blk = 1LL << nlev;
  CTP_REQUIRE(nx % blk == 0 && ny % blk == 0 && nz % blk == 0 && z_base % blk == 0, CTP_E_INVALID,
              "preview: dims (%lld,%lld,%lld) / z_base %lld not divisible by 2^%d", (long long)nx, (long long)ny,
              (long long)nz, (long long)z_base, nlev);
  for (int l = 0; l <= nlev; l++) {
    const int64_t lnz_global = ((z_base + nz) >> l);
    int rc = check_level_desc(levels[l], nx >> l, ny >> l, lnz_global, l);
    if (rc != CTP_OK) return rc;
  }
  for (int l = nlev + 1; l < CTP_MAX_LEVELS; l++)
    CTP_REQUIRE(levels[l].out == nullptr, CTP_E_INVALID, "preview: level %d requested above nlev %d", l, nlev);

  PvArgs a;
  a.vol = vol;
  a.lut = lut;
  a.hist = reinterpret_cast<unsigned long long*>(hist);
  for (int l = 0; l < CTP_MAX_LEVELS; l++) {
    a.lv[l] = make_dst(levels[l], nx >> l, ny >> l, z_base >> l);
    if (l > nlev) a.lv[l].out = nullptr;
  }
  // tile geometry: <= kMaxUnits units
  const int uz = nlev == 0 ? 1 : 2;
  const int tz = 1 << nlev;
  const int64_t xu_total = nx / UXW;
  const int64_t urows_per_block = (int64_t)(tz / uz) * (blk / uz);  // unit rows in a 2^L x 2^L block
  PvGeom& g = a.g;
  g.nx = nx; g.ny = ny; g.nz = nz; g.z_base = z_base;
  if (xu_total * urows_per_block <= kMaxUnits) {
    g.txu = (int)xu_total;
    int64_t ky = kMaxUnits / (xu_total * urows_per_block);
    const int64_t ky_max = (ny + blk - 1) / blk;
    if (ky > ky_max) ky = ky_max;
    if (ky < 1) ky = 1;
    g.ty = (int)(ky * blk);
  } else {
    g.txu = (int)(kMaxUnits / urows_per_block);
    g.ty = (int)blk;
  }
  const int64_t tiles_x = (xu_total + g.txu - 1) / g.txu;
  const int64_t tiles_y = (ny + g.ty - 1) / g.ty;
  const int64_t n_tiles = tiles_x * tiles_y * (nz / tz);
  CTP_REQUIRE(n_tiles < (1LL << 31), CTP_E_INVALID, "preview: too many tiles");
  g.tiles_x = (int)tiles_x;
  g.tiles_y = (int)tiles_y;
  g.n_tiles = (int)n_tiles;
  g.flush_tiles = 1;

  cudaStream_t st = as_stream(stream);
  switch (nlev) {
    case 0: return launch_l<T, 0>(a, st);
    case 1: return launch_l<T, 1>(a, st);
    case 2: return launch_l<T, 2>(a, st);
    case 3: return launch_l<T, 3>(a, st);
    default: return launch_l<T, 4>(a, st);
  }
}

}  // namespace ctp

extern "C" {

int ctp_preview_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut,
                   int32_t nlev, const ctp_level_out* levels, uint64_t* hist, void* stream) {
  return ctp::preview_impl<uint8_t>(vol, nz, ny, nx, z_base, lut, nlev, levels, hist, stream);
}

int ctp_preview_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut4096,
                    int32_t nlev, const ctp_level_out* levels, uint64_t* hist4096, void* stream) {
  CTP_REQUIRE(lut4096 != nullptr, CTP_E_INVALID, "ctp_preview_u16: a 4096-entry LUT is required");
  return ctp::preview_impl<uint16_t>(vol, nz, ny, nx, z_base, lut4096, nlev, levels, hist4096, stream);
}

}  // extern "C"

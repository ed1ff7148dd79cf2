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
// Work decomposition (B200: 148 SMs, 2 resident 256-thread CTAs per SM):
//   * a TILE is 2^L z-slices x (ky*2^L) rows x (TXu*UXW) columns, <= 1024 UNITS;
//     CTAs are persistent and walk tiles in memory order.
//   * a UNIT is UXW x-voxels (one 16-byte vector: 16 u8 or 8 u16) on 2 rows x
//     2 slices (L >= 1) -- exactly the 2x2x2 cells of level 1 along one vector.
//     Each thread owns 4 units per tile: 16 independent 16-byte loads in flight.
//   * histogram + LUT in ONE shared-memory atomic per voxel: the counter word
//     holds lut[v] in bits 0..7 and the count in bits 12..31; atomicAdd(+4096)
//     returns the old word whose low byte is f = lut[v].  Summing the 8 old
//     words of a level-1 cell and masking 12 bits gives sum(f) exactly (<= 2040).
//     u8: per-lane columns [bin][lane] (bank == lane, conflict-free);
//     u16: one 4096-word table per CTA.
//   * level-1 sums go to shared memory; levels 2..L are reduced from there
//     (u16 / u32 sums) and written, byte per thread, as coalesced row segments.
#include "ctp_common.cuh"

namespace ctp {

constexpr int kPvThreads = 256;
constexpr int kMaxUnits = 1024;                 // per tile
constexpr int kUnitsPerThread = kMaxUnits / kPvThreads;
constexpr int kBatch = 2;  // units loaded together (8 x 16 B in flight per thread)
constexpr uint32_t kOne = 1u << 12;             // count increment
constexpr uint32_t kCountCap = (1u << 20) - 1;  // 20-bit count field

template <typename T> struct Vox;
template <> struct Vox<uint8_t> {
  static constexpr int UXW = 16, NBINS = 256, HWORDS = 256 * 32;
};
template <> struct Vox<uint16_t> {
  static constexpr int UXW = 8, NBINS = 4096, HWORDS = 4096;
};

struct PvGeom {
  int64_t nx, ny, nz, z_base;
  int32_t txu;      // units per tile along x
  int32_t ty;       // rows per tile (multiple of 2^L)
  int64_t tiles_x, tiles_y, n_tiles;
  int32_t flush_tiles;  // flush the smem counters every this many tiles
};

struct PvArgs {
  const void* vol;
  const uint8_t* lut;
  unsigned long long* hist;
  LevelDst lv[CTP_MAX_LEVELS];
  PvGeom g;
};

template <typename T>
__device__ __forceinline__ uint32_t hist_word(uint32_t v, int lane) {
  if constexpr (sizeof(T) == 1) return (v << 5) | (uint32_t)lane;
  else return min(v, 4095u);
}

// Process one 32-bit word of voxels: 4 u8 or 2 u16.  Returns old counter words.
template <typename T>
__device__ __forceinline__ void atom_word(uint32_t* hs, uint32_t w, int lane, uint32_t* o) {
  if constexpr (sizeof(T) == 1) {
#pragma unroll
    for (int b = 0; b < 4; b++) o[b] = atomicAdd(&hs[hist_word<T>((w >> (8 * b)) & 255u, lane)], kOne);
  } else {
    o[0] = atomicAdd(&hs[hist_word<T>(w & 0xFFFFu, lane)], kOne);
    o[1] = atomicAdd(&hs[hist_word<T>(w >> 16, lane)], kOne);
  }
}

template <typename T>
__device__ void flush_counts(uint32_t* hs, unsigned long long* hist) {
  constexpr int NB = Vox<T>::NBINS;
  __syncthreads();
  if constexpr (sizeof(T) == 1) {
    const int bin = threadIdx.x;  // 256 threads == 256 bins
    uint32_t s = 0;
#pragma unroll 8
    for (int k = 0; k < 32; k++) {
      const int idx = bin * 32 + ((k + bin) & 31);
      const uint32_t wv = hs[idx];
      s += wv >> 12;
      hs[idx] = wv & 0xFFFu;
    }
    if (s && hist) atomicAdd(hist + bin, (unsigned long long)s);
  } else {
    for (int b = threadIdx.x; b < NB; b += kPvThreads) {
      const uint32_t wv = hs[b];
      if ((wv >> 12) && hist) atomicAdd(hist + b, (unsigned long long)(wv >> 12));
      hs[b] = wv & 0xFFFu;
    }
  }
  __syncthreads();
}

template <typename T, int L>
__global__ void __launch_bounds__(kPvThreads, 2) preview_kernel(const PvArgs a) {
  constexpr int UXW = Vox<T>::UXW;
  constexpr int HW = Vox<T>::HWORDS;
  constexpr int UZ = (L == 0) ? 1 : 2;
  constexpr int ROWS = UZ * UZ;
  constexpr int TZ = 1 << L;
  constexpr int L1PU = UXW / 2;  // level-1 sums per unit

  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* hs = smem;                                          // HW counter words
  uint16_t* s1 = reinterpret_cast<uint16_t*>(smem + HW);        // level-1 sums
  uint32_t* s2 = reinterpret_cast<uint32_t*>(s1 + kMaxUnits * L1PU);  // level-2 sums
  uint32_t* s3 = s2 + kMaxUnits * L1PU / 8;                     // level-3 sums
  uint32_t* sl[5] = {nullptr, nullptr, s2, s3, nullptr};

  const int lane = threadIdx.x & 31;
  const PvGeom& g = a.g;

  // counter words: LUT value in the low byte, count 0
  for (int i = threadIdx.x; i < HW; i += kPvThreads) {
    const int bin = (sizeof(T) == 1) ? (i >> 5) : i;
    hs[i] = a.lut ? (uint32_t)a.lut[bin] : (uint32_t)min(bin, 255);
  }
  __syncthreads();

  const int rows_u = g.ty / UZ;               // unit rows along y in a tile
  const int units = (TZ / UZ) * rows_u * g.txu;
  const int xw = g.txu * UXW;                 // tile width in voxels
  const T* __restrict__ vol = reinterpret_cast<const T*>(a.vol);
  int since_flush = 0;

  for (int64_t tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
    const int64_t tx_i = tile % g.tiles_x;
    const int64_t rest = tile / g.tiles_x;
    const int64_t ty_i = rest % g.tiles_y;
    const int64_t tz_i = rest / g.tiles_y;
    const int64_t x0 = tx_i * xw, y0 = ty_i * g.ty, z0 = tz_i * TZ;

    // ---- load + process in batches of kBatch units (16-byte vectors) ----------
#pragma unroll 1
    for (int bt = 0; bt < kUnitsPerThread; bt += kBatch) {
    uint4 q[kBatch][ROWS];
    bool ok[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; i++) {
      const int u = threadIdx.x + kPvThreads * (bt + i);
      const int xu = u % g.txu;
      const int r = u / g.txu;
      const int yr = r % rows_u;
      const int zr = r / rows_u;
      const int64_t x = x0 + (int64_t)xu * UXW, y = y0 + (int64_t)yr * UZ, z = z0 + (int64_t)zr * UZ;
      ok[i] = (u < units) && (x < g.nx) && (y < g.ny);
      if (ok[i]) {
#pragma unroll
        for (int r2 = 0; r2 < ROWS; r2++) {
          const int dz = r2 / UZ, dy = r2 % UZ;
          q[i][r2] = __ldcs(reinterpret_cast<const uint4*>(vol + ((z + dz) * g.ny + (y + dy)) * g.nx + x));
        }
      }
    }

    // ---- histogram + LUT + level 0/1 -----------------------------------------
#pragma unroll
    for (int i = 0; i < kBatch; i++) {
      if (!ok[i]) continue;
      const int u = threadIdx.x + kPvThreads * (bt + i);
      const int xu = u % g.txu;
      const int r = u / g.txu;
      const int yr = r % rows_u;
      const int zr = r / rows_u;
      const int64_t x = x0 + (int64_t)xu * UXW, y = y0 + (int64_t)yr * UZ, z = z0 + (int64_t)zr * UZ;

      // per row: UXW atomics (hist + LUT), optional level-0 store, and the
      // running level-1 pair sums (low 12 bits of the summed old words)
      uint32_t acc[L1PU];
#pragma unroll
      for (int j = 0; j < L1PU; j++) acc[j] = 0;
#pragma unroll
      for (int r2 = 0; r2 < ROWS; r2++) {
        uint32_t o[UXW];
        const uint32_t w[4] = {q[i][r2].x, q[i][r2].y, q[i][r2].z, q[i][r2].w};
#pragma unroll
        for (int k = 0; k < 4; k++) atom_word<T>(hs, w[k], lane, &o[k * (UXW / 4)]);
        if (a.lv[0].out) {  // level 0: the filtered voxels themselves
          const int dz = r2 / UZ, dy = r2 % UZ;
          uint8_t* dst = a.lv[0].out + level_offset(a.lv[0], z + dz, y + dy, x);
          uint32_t pk[UXW / 4];
#pragma unroll
          for (int k = 0; k < UXW / 4; k++)
            pk[k] = __byte_perm(__byte_perm(o[4 * k], o[4 * k + 1], 0x0040),
                                __byte_perm(o[4 * k + 2], o[4 * k + 3], 0x0040), 0x5410);
          if constexpr (UXW == 16) {
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            else { store8(dst, pk[0], pk[1]); store8(dst + 8, pk[2], pk[3]); }
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
          for (int k = 0; k < L1PU / 4; k++) {
            pk[k] = ((sum[4 * k] + 4) >> 3) | (((sum[4 * k + 1] + 4) >> 3) << 8) |
                    (((sum[4 * k + 2] + 4) >> 3) << 16) | (((sum[4 * k + 3] + 4) >> 3) << 24);
          }
          uint8_t* dst = a.lv[1].out + level_offset(a.lv[1], z >> 1, y >> 1, x >> 1);
          if constexpr (L1PU == 8) store8(dst, pk[0], pk[1]);
          else {
            if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) *reinterpret_cast<uint32_t*>(dst) = pk[0];
            else for (int b = 0; b < 4; b++) dst[b] = (uint8_t)(pk[0] >> (8 * b));
          }
        }
        if constexpr (L >= 2) {
          // s1 layout [zr][yr][x1], x1 = xu*L1PU + j
          uint16_t* d = s1 + ((size_t)(zr * rows_u + yr) * g.txu + xu) * L1PU;
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
        const int cz = TZ >> (l - 1), cy = g.ty >> (l - 1), cx = xw >> (l - 1);  // child dims
        const int nzc = cz >> 1, nyc = cy >> 1, nxc = cx >> 1;
        const int cells = nzc * nyc * nxc;
        const int64_t lnx = g.nx >> l, lny = g.ny >> l;
        const int shift = 3 * l;
        for (int c = threadIdx.x; c < cells; c += kPvThreads) {
          const int xq = c % nxc;
          const int rr = c / nxc;
          const int yq = rr % nyc;
          const int zq = rr / nyc;
          const int64_t gx = (x0 >> l) + xq, gy = (y0 >> l) + yq;
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
                const uint32_t* src = sl[l - 1];
                sum += src[base] + src[base + 1];
              }
            }
          if (l < L) sl[l][c] = sum;
          if (a.lv[l].out) {
            const int64_t gz = (z0 >> l) + zq;
            a.lv[l].out[level_offset(a.lv[l], gz, gy, gx)] = (uint8_t)((sum + (1u << (shift - 1))) >> shift);
          }
        }
        __syncthreads();
      }
    }

    if (++since_flush == g.flush_tiles) {
      since_flush = 0;
      flush_counts<T>(hs, a.hist);
    }
  }
  flush_counts<T>(hs, a.hist);
}

template <typename T>
static size_t smem_bytes(int L) {
  size_t b = (size_t)Vox<T>::HWORDS * 4;
  if (L >= 2) {
    const size_t l1 = (size_t)kMaxUnits * (Vox<T>::UXW / 2);
    b += l1 * 2 + (l1 / 8) * 4 + (l1 / 64) * 4 + 16;
  }
  return b;
}

template <typename T, int L>
static int launch_l(const PvArgs& a, int grid, cudaStream_t st) {
  const size_t sm = smem_bytes<T>(L);
  CTP_CUDA_CALL(cudaFuncSetAttribute(preview_kernel<T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  preview_kernel<T, L><<<grid, kPvThreads, sm, st>>>(a);
  CTP_CUDA_CHECK_LAUNCH("preview_kernel");
  return CTP_OK;
}

template <typename T>
static int preview_impl(const T* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut,
                        int nlev, const ctp_level_out* levels, uint64_t* hist, void* stream) {
  constexpr int UXW = Vox<T>::UXW;
  CTP_REQUIRE(vol != nullptr && levels != nullptr, CTP_E_INVALID, "preview: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "preview: degenerate shape");
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
  g.tiles_x = (xu_total + g.txu - 1) / g.txu;
  g.tiles_y = (ny + g.ty - 1) / g.ty;
  g.n_tiles = g.tiles_x * g.tiles_y * (nz / tz);
  // a counter word gains at most (units per thread) * (voxels per unit) per warp per tile,
  // from 8 warps (u8 lane columns) or from every thread (u16 shared table)
  const int64_t vox_per_unit = (int64_t)UXW * uz * uz;
  const int64_t per_tile = (sizeof(T) == 1) ? 8LL * kUnitsPerThread * vox_per_unit
                                            : (int64_t)kMaxUnits * vox_per_unit;
  g.flush_tiles = (int)(kCountCap / per_tile);
  if (g.flush_tiles < 1) g.flush_tiles = 1;

  int grid = num_sms() * 2;
  if (g.n_tiles < grid) grid = (int)g.n_tiles;
  cudaStream_t st = as_stream(stream);
  switch (nlev) {
    case 0: return launch_l<T, 0>(a, grid, st);
    case 1: return launch_l<T, 1>(a, grid, st);
    case 2: return launch_l<T, 2>(a, grid, st);
    case 3: return launch_l<T, 3>(a, grid, st);
    default: return launch_l<T, 4>(a, grid, st);
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

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
// B200 mapping (148 SMs, one persistent CTA per SM):
//   * a TILE is 2^L z-slices x (ky*2^L) rows x (TXu*UXW) columns, <= MAXU units.
//     Tiles stream from HBM into a ring of NST shared-memory stages with TMA
//     (cp.async.bulk.tensor.3d, boxes of <= 256 x ty x 2^L elements, completion
//     on an mbarrier): while the CTA reduces tile k, tiles k+1..k+NST-1 are in
//     flight, and no register is spent on in-flight data.
//   * a UNIT is UXW x-voxels (one 16-byte vector: 16 u8 or 8 u16) on 2 rows x
//     2 slices (L >= 1) -- exactly the 2x2x2 cells of level 1 along one vector;
//     every thread owns the same unit slots in every tile (offsets computed once).
//   * histogram + LUT in ONE shared-memory atomic per voxel: the counter word
//     holds lut[v] in bits 0..7 and the count in bits 12..31; atom.add(+4096)
//     returns the old word whose low byte is f = lut[v].  Summing the 8 old
//     words of a level-1 cell and masking 12 bits gives sum(f) exactly (<= 2040).
//     Per voxel the hot loop is PRMT (byte) + IMAD (address) + ATOMS + 1/2 add.
//     u8: per-lane columns [bin][lane] -- bank == lane, so a warp-wide ATOMS is
//     conflict-free for any data (tools/microbench/hist_bench.cu); u16: one
//     4096-word table per CTA.
//   * level-1 sums go to shared memory; levels 2..L are reduced from there
//     (u16 / u32 sums) and written as coalesced row segments.
#include <stdlib.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <atomic>
#include <mutex>
#include <cooperative_groups.h>
#include "ctp_common.cuh"

namespace ctp {

constexpr uint32_t kOne = 1u << 12;             // count increment
constexpr uint32_t kCountCap = (1u << 20) - 1;  // 20-bit count field
constexpr int kBoxX = 256;                      // TMA box limit per dimension (elements)

template <typename T> struct Vox;
// u8: [bin][lane] counter words in 256-byte bin rows (lanes in words 0..31,
// words 32..63 unused) so that a voxel's table offset (v << 8) | (lane << 2) is
// ONE byte permute of the voxel word with the lane byte, and the table base a
// warp-uniform operand of the atomic ([R+UR]): PRMT + ATOMS per voxel.
template <> struct Vox<uint8_t> {
  static constexpr int UXW = 16, NBINS = 256, ROWW = 64, HWORDS = 256 * ROWW;
};
// u16 (4096 bins): a random-bin warp-wide ATOMS on one shared table costs ~3.4
// wavefronts (bank conflicts), which bounded round 1's pass (4 interleaved
// columns [bin][lane % 4]: 58% of HBM).  Now a HOT WINDOW of HOT consecutive
// bins, chosen per CTA from its first tile (the densest HOT/64 of 64 coarse
// buckets), lives in per-lane columns [slot][lane] (bank == lane: conflict-free,
// like u8); the other bins go to one shared 4096-word table.  A voxel costs ONE
// ATOMS either way (the counter word still carries the LUT byte) and the warp
// pays an extra wavefront only for its out-of-window lanes.  CTP_U16_HOT=0
// restores round 1's COLS-column table.
#ifndef CTP_U16_COLS
#define CTP_U16_COLS 4
#endif
#ifndef CTP_U16_HOT
#define CTP_U16_HOT 512
#endif
template <> struct Vox<uint16_t> {
  static constexpr int UXW = 8, NBINS = 4096, COLS = CTP_U16_COLS, HOT = CTP_U16_HOT;
  static_assert(HOT % 64 == 0 && HOT <= 4096, "the hot window is whole 64-bin buckets");
  static constexpr int HWORDS = HOT > 0 ? HOT * 32 + 4096 : 4096 * COLS;
};

struct PvGeom {
  int32_t nx, ny, nz;
  int32_t txu;          // units per tile along x
  int32_t ty;           // rows per tile (multiple of 2^L)
  int32_t tiles_x, tiles_y, n_tiles;
  int32_t flush_tiles;  // flush the smem counters every this many tiles
  int32_t box_x;        // TMA box width (elements); a tile is nboxes boxes side by side
  int32_t nboxes;
  uint32_t box_bytes;   // box_x * ty * 2^L * sizeof(T)
};

struct PvArgs {
  const uint8_t* lut;
  unsigned long long* hist;
  LevelDst lv[CTP_MAX_LEVELS];
  PvGeom g;
  // in-kernel artifact LUT (the whole step in ONE cooperative launch) when top != nullptr
  const void* top;                 // the top n_top slices (mask.py:227), 16-byte aligned
  int64_t top_n;                   // elements in the top slab
  unsigned long long cutoff_floor; // floor(frac * top.size), mask.py:229-230
  int32_t vmax;                    // 0: identity LUT (u8); > 0: filter o 16->8 rescale
  uint8_t* lut_out;                // optional copies for the host
  uint8_t* flags_out;
  unsigned long long* ws;          // uint64[4097], zero on entry, left zero
  int32_t fence_sys;               // a level destination is a peer GPU's memory (CTP_OUT_PEER)
};

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
#ifndef CTP_TMA_NO_HINT  // the volume is read once: evict-first in L2 (keeps room for the atlas writes; -0.5%)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], "
      "[%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
#endif
}

template <typename T>
__device__ void flush_counts(uint32_t* hs, unsigned long long* hist, int threads, int hot_base) {
  __syncthreads();
  if constexpr (sizeof(T) == 1) {
    for (int bin = threadIdx.x; bin < 256; bin += threads) {
      uint32_t s = 0;
#pragma unroll 8
      for (int k = 0; k < 32; k++) {
        const int idx = bin * Vox<uint8_t>::ROWW + ((k + bin) & 31);  // rotated: conflict-free
        const uint32_t wv = hs[idx];
        s += wv >> 12;
        hs[idx] = wv & 0xFFFu;
      }
      if (s && hist) atomicAdd(hist + bin, (unsigned long long)s);
    }
  } else if constexpr (Vox<uint16_t>::HOT > 0) {
    constexpr int H = Vox<uint16_t>::HOT;
    for (int sl = threadIdx.x; sl < H; sl += threads) {  // hot window: [slot][lane], rotated (conflict-free)
      uint32_t s = 0;
#pragma unroll 8
      for (int k = 0; k < 32; k++) {
        const int idx = sl * 32 + ((k + sl) & 31);
        const uint32_t wv = hs[idx];
        s += wv >> 12;
        hs[idx] = wv & 0xFFFu;
      }
      if (s && hist) atomicAdd(hist + hot_base + sl, (unsigned long long)s);
    }
    uint32_t* cold = hs + H * 32;
    for (int b = threadIdx.x; b < 4096; b += threads) {
      const uint32_t wv = cold[b];
      cold[b] = wv & 0xFFFu;
      if ((wv >> 12) && hist) atomicAdd(hist + b, (unsigned long long)(wv >> 12));
    }
  } else {
    constexpr int C = Vox<uint16_t>::COLS;
    for (int b = threadIdx.x; b < 4096; b += threads) {
      uint32_t s = 0;
#pragma unroll
      for (int c = 0; c < C; c++) {
        const uint32_t wv = hs[b * C + c];
        s += wv >> 12;
        hs[b * C + c] = wv & 0xFFFu;
      }
      if (s && hist) atomicAdd(hist + b, (unsigned long long)s);
    }
  }
  __syncthreads();
}

// One 16-byte row vector of a unit: UXW atomics; returns the old counter words.
// u8: tbl = table base (uniform), lb = 4 * lane.  u16 with a hot window: tbl =
// the shared (cold) table, lb = hot table + 4 * lane - (hot_base << 7), hb =
// hot_base.  u16 without: lb = table base + column.
template <typename T>
__device__ __forceinline__ void row_atomics(const uint4& q, uint32_t tbl, uint32_t lb, uint32_t hb, uint32_t* o) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  if constexpr (sizeof(T) == 1) {
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int b = 0; b < 4; b++) {
        // [0, 0, v, 4*lane] = (v << 8) | (lane << 2): the voxel's counter word
        const uint32_t off = __byte_perm(w[k], lb, 0x7604u | ((uint32_t)b << 4));
        o[4 * k + b] = atom_add_shared(tbl + off, kOne);
      }
  } else if constexpr (Vox<uint16_t>::HOT > 0) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t wc = __vminu2(w[k], 0x0FFF0FFFu);  // both voxels saturated to 4095 (VIMNMX.U16x2)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t v = __byte_perm(wc, 0u, h ? 0x4432u : 0x4410u);  // one PRMT per voxel
#ifdef CTP_U16_REL_ADDR
        // (measured, not the default: 3.903 vs 3.895 ms on config 3 -- one instruction fewer per voxel
        // buys nothing, the pass is not issue-bound; profiles/r02_u16_rel_addr_ab.txt)
        // offsets from the table base (hot window first, cold table right behind it): rel =
        // (v - hot_base) * 128 + 4 * lane wraps far above the window for every bin outside
        // it, so ONE multiply-add and ONE compare find the hot slot, a predicated
        // multiply-add (immediate operands) the cold word, and the base rides on the
        // atomic's uniform operand: PRMT + IMAD + ISETP + @IMAD + ATOMS per voxel (the
        // absolute-address form below needs one more subtract)
        constexpr uint32_t kHotBytes = (uint32_t)Vox<uint16_t>::HOT * 128u;
        const uint32_t rel = v * 128u + lb;  // lb = 4 * lane - hot_base * 128 (mod 2^32)
        const uint32_t off = rel < kHotBytes ? rel : v * 4u + kHotBytes;
        o[2 * k + h] = atom_add_shared(tbl + off, kOne);
#else
        const uint32_t addr = (v - hb < (uint32_t)Vox<uint16_t>::HOT) ? lb + (v << 7) : tbl + (v << 2);
        o[2 * k + h] = atom_add_shared(addr, kOne);
#endif
      }
    }
  } else {
    constexpr uint32_t SH = 2 + (Vox<uint16_t>::COLS == 1 ? 0 : Vox<uint16_t>::COLS == 2 ? 1 : Vox<uint16_t>::COLS == 4 ? 2 : 3);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      o[2 * k] = atom_add_shared(lb + (min(w[k] & 0xFFFFu, 4095u) << SH), kOne);
      o[2 * k + 1] = atom_add_shared(lb + (min(w[k] >> 16, 4095u) << SH), kOne);
    }
  }
}

template <typename T, int L, int MAXU>
struct PvLayout {
  static constexpr int UXW = Vox<T>::UXW;
  static constexpr int UZ = (L == 0) ? 1 : 2;
  static constexpr int ROWS = UZ * UZ;
  static constexpr int L1PU = UXW / 2;
  static constexpr int STAGE_BYTES = MAXU * ROWS * 16;
  static constexpr int HIST_BYTES = Vox<T>::HWORDS * 4;
  static constexpr int S1_BYTES = L >= 2 ? MAXU * L1PU * 2 : 0;
};

// (sum + 4) >> 3 of two packed 12-bit level-1 sums, as two bytes in 16-bit lanes
__device__ __forceinline__ uint32_t round_l1_pair(uint32_t p) { return ((p + 0x00040004u) >> 3) & 0x00FF00FFu; }

template <typename T, int L, int THREADS, int NST, int MAXU, bool WANT0, bool POW2>
__global__ void __launch_bounds__(THREADS, 1)
    preview_kernel(const __grid_constant__ CUtensorMap tmap, const PvArgs a) {
  using LY = PvLayout<T, L, MAXU>;
  constexpr int UXW = LY::UXW, UZ = LY::UZ, ROWS = LY::ROWS, L1PU = LY::L1PU;
  constexpr int TZ = 1 << L;
  constexpr int UPT = MAXU / THREADS;  // unit slots per thread
  static_assert(MAXU % THREADS == 0 && UPT >= 1, "a tile is a whole number of unit slots per thread");
  constexpr int HW = Vox<T>::HWORDS;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* hs = reinterpret_cast<uint32_t*>(smem + NST * LY::STAGE_BYTES);
  uint16_t* s1 = reinterpret_cast<uint16_t*>(smem + NST * LY::STAGE_BYTES + LY::HIST_BYTES);
  // level-1 sums are double-buffered so tile k+1's unit phase may overwrite
  // nothing that tile k's level phase still reads (one barrier per tile)
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(s1) + 2 * LY::S1_BYTES);

  const int lane = threadIdx.x & 31;
  const PvGeom& g = a.g;
  const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(stages);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
  const uint32_t s1a = (uint32_t)__cvta_generic_to_shared(s1);
  const int xw = g.txu * UXW;  // tile width (elements)
  const int rows_u = g.ty / UZ;
  const int units = (TZ / UZ) * rows_u * g.txu;
  const int s1_row = g.txu * L1PU;  // level-1 sums per (z1, y1) row of the tile
  // Bank swizzle of the level-1 sums: the 4 lanes of a level-3 group read rows
  // (z1, y1) that are whole 1-KB rows apart (same banks); XOR-ing x1 with a
  // per-row 16-element (32-byte) offset taken from bit 1 of y1 and of z1 puts
  // them in 4 different bank quarters.  Needs rows of whole 64-element blocks.
  const int swz_mask = (s1_row & 63) == 0 ? 0x30 : 0;
  auto s1_swz = [&](int z1, int y1) -> int { return ((((y1 >> 1) & 1) | (((z1 >> 1) & 1) << 1)) << 4) & swz_mask; };

  // this CTA's contiguous range of tiles (coordinates advance incrementally)
  const int per = g.n_tiles / gridDim.x, extra = g.n_tiles % gridDim.x;
  const int t_begin = blockIdx.x * per + min((int)blockIdx.x, extra);
  const int t_end = t_begin + per + ((int)blockIdx.x < extra ? 1 : 0);

  auto issue = [&](int tile, int stage) {
    const int tx_i = tile % g.tiles_x;
    const int rest = tile / g.tiles_x;
    const int ty_i = rest % g.tiles_y;
    const int tz_i = rest / g.tiles_y;
    const uint32_t bar = bar0 + 8u * stage;
    mbar_expect_tx(bar, g.box_bytes * (uint32_t)g.nboxes);
    for (int b = 0; b < g.nboxes; b++)
      tma_load_3d(stage0 + (uint32_t)stage * LY::STAGE_BYTES + (uint32_t)b * g.box_bytes, &tmap,
                  tx_i * xw + b * g.box_x, ty_i * g.ty, tz_i * TZ, bar);
  };

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    for (int s = 0; s < NST; s++) mbar_init(bar0 + 8u * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NST; s++)
      if (t_begin + s < t_end) issue(t_begin + s, s);

  // the LUT of the in-kernel artifact step, until it is copied into the counter words:
  // u16 (L >= 2) keeps it in the level-1 sum buffers (free until the first tile), so the
  // 4 KB do not come out of the hot window's budget
  uint8_t* slut;
  if constexpr (sizeof(T) == 2 && L >= 2) {
    static_assert(2 * LY::S1_BYTES >= Vox<T>::NBINS, "the LUT fits the level-1 sum buffers");
    slut = reinterpret_cast<uint8_t*>(s1);
  } else {
    __shared__ uint8_t slut_s[Vox<T>::NBINS];
    slut = slut_s;
  }
  if (a.top != nullptr) {
    // ---- the artifact-LUT step inside this launch (mask.py:215-231, 241-245):
    // the first tiles are already streaming in while every CTA histograms its
    // share of the top slab; one grid barrier; every CTA derives the LUT.
    constexpr int NB = Vox<T>::NBINS;
    for (int i = threadIdx.x; i < NB; i += THREADS) hs[i] = 0;
    __syncthreads();
    const int64_t nvec = a.top_n / UXW;  // 16-byte vectors (rows are 16-byte aligned)
    const int64_t per_cta = (nvec + gridDim.x - 1) / gridDim.x;
    const int64_t v0 = blockIdx.x * per_cta, v1 = min(nvec, v0 + per_cta);
    const uint4* tp = reinterpret_cast<const uint4*>(a.top);
    for (int64_t i = v0 + threadIdx.x; i < v1; i += THREADS) {
      const uint4 q = __ldcs(tp + i);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if constexpr (sizeof(T) == 1) {
#pragma unroll
          for (int b = 0; b < 4; b++) atomicAdd(&hs[(w[k] >> (8 * b)) & 255u], 1u);
        } else {
          atomicAdd(&hs[min(w[k] & 0xFFFFu, 4095u)], 1u);
          atomicAdd(&hs[min(w[k] >> 16, 4095u)], 1u);
        }
      }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NB; b += THREADS)
      if (hs[b]) atomicAdd(a.ws + b, (unsigned long long)hs[b]);
    if (blockIdx.x == 0 && a.hist)
      for (int b = threadIdx.x; b < NB; b += THREADS) a.hist[b] = 0;  // before any CTA can flush into it
    __threadfence();
    cooperative_groups::this_grid().sync();
    for (int b = threadIdx.x; b < NB; b += THREADS) {
      const unsigned long long c = __ldcg(a.ws + b);
      const bool flagged = (b == 0) || (c > a.cutoff_floor);  // mask.py:230-231
      uint32_t val = (uint32_t)b;
      if (a.vmax > 0) {
        const uint32_t v = min((uint32_t)b, (uint32_t)a.vmax);
        val = (uint32_t)((2ull * 255ull * v + (uint64_t)a.vmax) / (2ull * (uint64_t)a.vmax));
      }
      slut[b] = flagged ? 0 : (uint8_t)val;
      if (blockIdx.x == 0) {
        if (a.lut_out) a.lut_out[b] = slut[b];
        if (a.flags_out) a.flags_out[b] = flagged ? 1 : 0;
      }
    }
    __shared__ bool last_reader;
    __syncthreads();
    if (threadIdx.x == 0) last_reader = atomicAdd(a.ws + 4096, 1ull) == gridDim.x - 1;
    __syncthreads();
    if (last_reader) {  // every CTA has read ws: reset it for the next call
      for (int b = threadIdx.x; b < NB; b += THREADS) a.ws[b] = 0;
      if (threadIdx.x == 0) a.ws[4096] = 0;
    }
  }
  // unit slots of this thread (same in every tile): coordinates + stage offset
  int uxu[UPT], uyr[UPT], uzr[UPT];
  uint32_t uso[UPT];
#pragma unroll
  for (int i = 0; i < UPT; i++) {
    const int u = threadIdx.x + THREADS * i;
    uxu[i] = u % g.txu;
    const int r = u / g.txu;
    uyr[i] = r % rows_u;
    uzr[i] = u < units ? r / rows_u : TZ;  // TZ marks "slot unused"
    const int x = uxu[i] * UXW;
    const int b = x / g.box_x, xi = x - b * g.box_x;
    uso[i] = (uint32_t)b * g.box_bytes + (uint32_t)(((uzr[i] * UZ) * g.ty + uyr[i] * UZ) * g.box_x + xi) * sizeof(T);
  }
  const uint32_t row_dy = (uint32_t)g.box_x * sizeof(T);
  const uint32_t row_dz = (uint32_t)g.box_x * g.ty * sizeof(T);

  // u16 hot window: the densest HOT/64 consecutive 64-bin buckets of a sample of
  // this CTA's first tile (one row vector per thread) -- any choice is exact, it
  // only decides which voxels take the conflict-free per-lane columns
  __shared__ int s_hot_base;
  int hot_base = 0;
  if constexpr (sizeof(T) == 2 && Vox<uint16_t>::HOT > 0) {
    constexpr int WB = Vox<uint16_t>::HOT / 64;
    for (int i = threadIdx.x; i < 64; i += THREADS) hs[i] = 0;
    __syncthreads();
    if (t_begin < t_end && uzr[0] < TZ / UZ) {
      mbar_wait(bar0, 0u);  // the first tile (stage 0) has landed
      const uint4 q = lds128(stage0 + uso[0]);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        atomicAdd(&hs[min(w[k] & 0xFFFFu, 4095u) >> 6], 1u);
        atomicAdd(&hs[min(w[k] >> 16, 4095u) >> 6], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t best = 0;
      int best_s = 0;
      for (int st = lane; st <= 64 - WB; st += 32) {
        uint32_t m = 0;
        for (int j = 0; j < WB; j++) m += hs[st + j];
        if (m > best) { best = m; best_s = st; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {  // max mass, smallest start on ties
        const uint32_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        const int os = __shfl_xor_sync(0xFFFFFFFFu, best_s, off);
        if (ob > best || (ob == best && os < best_s)) { best = ob; best_s = os; }
      }
      if (lane == 0) s_hot_base = best_s * 64;
    }
    __syncthreads();
    hot_base = s_hot_base;
  }

  // counter words: LUT value in the low byte, count 0
  for (int i = threadIdx.x; i < HW; i += THREADS) {
    int bin;
    if constexpr (sizeof(T) == 1) bin = i >> 6;
    else if constexpr (Vox<uint16_t>::HOT > 0) bin = i < Vox<uint16_t>::HOT * 32 ? hot_base + (i >> 5) : i - Vox<uint16_t>::HOT * 32;
    else bin = i / Vox<uint16_t>::COLS;
    hs[i] = a.top ? (uint32_t)slut[bin] : (a.lut ? (uint32_t)a.lut[bin] : (uint32_t)min(bin, 255));
  }
  const uint32_t hs_a = (uint32_t)__cvta_generic_to_shared(hs);
  uint32_t tbl, lb;
  if constexpr (sizeof(T) == 1) {
    tbl = hs_a;
    lb = 4u * (uint32_t)lane;
  } else if constexpr (Vox<uint16_t>::HOT > 0) {
#ifdef CTP_U16_REL_ADDR
    tbl = hs_a;                                                          // hot window, then the cold table
    lb = 4u * (uint32_t)lane - ((uint32_t)hot_base << 7);                // rel = v * 128 + lb
#else
    // (an opaque copy: keeps the cold-table base in one register, a cold address is one IMAD/LEA)
    asm volatile("mov.u32 %0, %1;" : "=r"(tbl) : "r"(hs_a + 4u * Vox<uint16_t>::HOT * 32));  // cold table
    lb = hs_a + 4u * (uint32_t)lane - ((uint32_t)hot_base << 7);         // hot [slot][lane], slot = v - hot_base
#endif
  } else {
    tbl = hs_a;
    lb = hs_a + 4u * (uint32_t)(lane % Vox<uint16_t>::COLS);
  }

  // Level >= 3 reduction slot (tile-invariant): a lane owns one (z2, y2) row run
  // of four x-adjacent level-2 cells (x-quad q: level-1 x-cells 8q .. 8q+7, one
  // aligned 16-byte run of an s1 row); the 4 lanes of a group are (dz, dy) of one
  // level-3 row (z3, y3) and reduce its two level-3 cells (x3 = 2q, 2q+1) by
  // shuffles; for L = 4 the 4 groups (z3, y3 parity) of one level-4 cell are 16
  // consecutive lanes.
  int c_q = -1, c_y2 = 0, c_z2 = 0;
  uint32_t c_s1 = 0;
  if constexpr (L >= 3) {
    const int nq = xw >> 4;  // x-quads of level-2 cells per row (= level-4 cells per row for L = 4)
    const int grp = threadIdx.x >> 2, ql = threadIdx.x & 3;
    int q = -1, y3 = 0, z3 = 0;
    if constexpr (L == 3) {
      if (grp < nq * (g.ty >> 3)) {  // TZ == 8: a single level-3 slice per tile
        q = grp % nq;
        y3 = grp / nq;
      }
    } else {
      const int cell = grp >> 2, sub = grp & 3;  // TZ == 16: a single level-4 slice per tile
      if (cell < nq * (g.ty >> 4)) {
        q = cell % nq;
        z3 = sub >> 1;
        y3 = 2 * (cell / nq) + (sub & 1);
      }
    }
    if (q >= 0) {
      c_q = q;
      c_z2 = 2 * z3 + (ql >> 1);
      c_y2 = 2 * y3 + (ql & 1);
      // first level-1 row of the run (z1 = 2 z2, y1 = 2 y2); the swizzle (bit 1 of y1, z1) is
      // the same for all four rows the lane reads
      c_s1 = s1a + 2u * (uint32_t)(((2 * c_z2) * rows_u + 2 * c_y2) * s1_row + ((8 * q) ^ s1_swz(2 * c_z2, 2 * c_y2)));
    }
  }
  const bool lvl_warp = __any_sync(0xFFFFFFFFu, c_q >= 0);  // warp-uniform: this warp has level work
  __syncthreads();

  constexpr bool want0 = WANT0;
  const bool want1 = a.lv[1].out != nullptr;
  int since_flush = 0;
  int tx_i = 0, ty_i = 0, tz_i = 0;
  {
    const int rest = t_begin / g.tiles_x;
    tx_i = t_begin - rest * g.tiles_x;
    ty_i = rest % g.tiles_y;
    tz_i = rest / g.tiles_y;
  }
  int k = 0;
#ifdef CTP_PHASE_TIMING  // per-phase cycle counts (tools/build_variant.py ... -DCTP_PHASE_TIMING)
  long long t_data = 0, t_units = 0, t_bar = 0, t_lvl = 0;
  const long long t_start = clock64();
#endif
  for (int tile = t_begin; tile < t_end; tile++, k++) {
    const int stage = k % NST;
    const uint32_t sbase = stage0 + (uint32_t)stage * LY::STAGE_BYTES;
    const int x0 = tx_i * xw, y0 = ty_i * g.ty, z0 = tz_i * TZ;
#ifdef CTP_PHASE_TIMING
    const long long ph0 = clock64();
#endif
    mbar_wait(bar0 + 8u * stage, (uint32_t)((k / NST) & 1));
#ifdef CTP_PHASE_TIMING
    const long long ph1 = clock64();
#endif
    uint16_t* s1k = s1 + (k & 1) * (LY::S1_BYTES / 2);
    const uint32_t s1off = (uint32_t)(k & 1) * LY::S1_BYTES;

#pragma unroll
    for (int i = 0; i < UPT; i++) {
      const int xu = uxu[i], yr = uyr[i], zr = uzr[i];
      const int x = x0 + xu * UXW, y = y0 + yr * UZ, z = z0 + zr * UZ;
      if (zr >= TZ / UZ || x >= g.nx || y >= g.ny) continue;
      uint32_t acc[L1PU];
#pragma unroll
      for (int j = 0; j < L1PU; j++) acc[j] = 0;
#pragma unroll
      for (int r2 = 0; r2 < ROWS; r2 += (L >= 1 ? 2 : 1)) {
        // two rows at a time: acc += o_r[2j] + o_r[2j+1] + o_r'[2j] + o_r'[2j+1] as 3-input adds
        uint32_t o[2][UXW];
#pragma unroll
        for (int h = 0; h < (L >= 1 ? 2 : 1); h++) {
          const int rr = r2 + h;
          const uint4 q = lds128(sbase + uso[i] + (rr / UZ) * row_dz + (rr % UZ) * row_dy);
          row_atomics<T>(q, tbl, lb, (uint32_t)hot_base, o[h]);
          if (want0) {  // level 0: the filtered voxels themselves
            uint8_t* dst = a.lv[0].out + level_offset<POW2>(a.lv[0], z + rr / UZ, y + rr % UZ, x);
            uint32_t pk[UXW / 4];
#pragma unroll
            for (int kk = 0; kk < UXW / 4; kk++)
              pk[kk] = __byte_perm(__byte_perm(o[h][4 * kk], o[h][4 * kk + 1], 0x0040),
                                   __byte_perm(o[h][4 * kk + 2], o[h][4 * kk + 3], 0x0040), 0x5410);
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
        }
        if constexpr (L >= 1) {
#pragma unroll
          for (int j = 0; j < L1PU; j++) acc[j] = acc[j] + (o[0][2 * j] + o[0][2 * j + 1]) + (o[1][2 * j] + o[1][2 * j + 1]);
        }
      }
      if constexpr (L >= 1) {
        // pack the 12-bit sums of f (<= 2040) two per word: the s1 layout
        uint32_t pr[L1PU / 2];
#pragma unroll
        for (int j = 0; j < L1PU / 2; j++) pr[j] = __byte_perm(acc[2 * j], acc[2 * j + 1], 0x5410) & 0x0FFF0FFFu;
        if (want1) {
          uint32_t pk[L1PU / 4];
#pragma unroll
          for (int kk = 0; kk < L1PU / 4; kk++)
            pk[kk] = __byte_perm(round_l1_pair(pr[2 * kk]), round_l1_pair(pr[2 * kk + 1]), 0x6420);
          uint8_t* dst = a.lv[1].out + level_offset<POW2>(a.lv[1], z >> 1, y >> 1, x >> 1);
          if constexpr (L1PU == 8) {
            store8(dst, pk[0], pk[1]);
          } else {
            if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) *reinterpret_cast<uint32_t*>(dst) = pk[0];
            else for (int b = 0; b < 4; b++) dst[b] = (uint8_t)(pk[0] >> (8 * b));
          }
        }
        if constexpr (L >= 2) {
          // s1 layout [zr][yr][x1], x1 = xu*L1PU + j
          uint16_t* d = s1k + (zr * rows_u + yr) * s1_row + ((xu * L1PU) ^ s1_swz(zr, yr));
          if constexpr (L1PU == 8) *reinterpret_cast<uint4*>(d) = make_uint4(pr[0], pr[1], pr[2], pr[3]);
          else *reinterpret_cast<uint2*>(d) = make_uint2(pr[0], pr[1]);
        }
      }
    }

    // every thread is done with this stage (and s1 is complete): refill it
#ifdef CTP_PHASE_TIMING
    const long long ph2 = clock64();
#endif
    __syncthreads();
#ifdef CTP_PHASE_TIMING
    const long long ph3 = clock64();
#endif
    if (threadIdx.x == 0 && tile + NST < t_end) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
      issue(tile + NST, stage);
    }

    // ---- levels 2..L from the level-1 sums -------------------------------------------
    if constexpr (L == 2) {
      // four x-adjacent level-2 cells per thread: their 8 level-1 x-cells are one
      // aligned 16-byte run of an s1 row (the swizzle moves 32-byte blocks), one
      // 4-byte store of the level row
      const int nq = xw >> 4, ny2 = g.ty >> 2;  // quads of level-2 cells per row, rows
      const bool want2 = a.lv[2].out != nullptr;
      for (int c = threadIdx.x; c < ny2 * nq; c += THREADS) {
        const int q = c % nq, y2 = c / nq;
        const int gx = (x0 >> 2) + 4 * q, gy = (y0 >> 2) + y2;
        if (gx >= (g.nx >> 2) || gy >= (g.ny >> 2)) continue;
        uint32_t sum[4] = {0, 0, 0, 0};
#pragma unroll
        for (int ez = 0; ez < 2; ez++)
#pragma unroll
          for (int ey = 0; ey < 2; ey++) {
            const uint4 w = lds128(s1a + s1off +
                                   2u * (uint32_t)((ez * rows_u + 2 * y2 + ey) * s1_row + ((8 * q) ^ s1_swz(ez, 2 * y2 + ey))));
            sum[0] += (w.x & 0xFFFFu) + (w.x >> 16);
            sum[1] += (w.y & 0xFFFFu) + (w.y >> 16);
            sum[2] += (w.z & 0xFFFFu) + (w.z >> 16);
            sum[3] += (w.w & 0xFFFFu) + (w.w >> 16);
          }
        if (want2) {
          uint8_t* dst = a.lv[2].out + level_offset<POW2>(a.lv[2], z0 >> 2, gy, gx);
          const uint32_t v = ((sum[0] + 32) >> 6) | (((sum[1] + 32) >> 6) << 8) | (((sum[2] + 32) >> 6) << 16) |
                             (((sum[3] + 32) >> 6) << 24);
          if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) *reinterpret_cast<uint32_t*>(dst) = v;
          else for (int b = 0; b < 4; b++) dst[b] = (uint8_t)(v >> (8 * b));
        }
      }
    } else if constexpr (L >= 3) {
      if (lvl_warp) {
        uint32_t l2[4] = {0, 0, 0, 0};  // four x-adjacent level-2 sums of this lane's (z2, y2) row
        if (c_q >= 0) {
#pragma unroll
          for (int ez = 0; ez < 2; ez++)
#pragma unroll
            for (int ey = 0; ey < 2; ey++) {
              const uint4 w = lds128(c_s1 + s1off + 2u * (uint32_t)((ez * rows_u + ey) * s1_row));
              l2[0] += (w.x & 0xFFFFu) + (w.x >> 16);
              l2[1] += (w.y & 0xFFFFu) + (w.y >> 16);
              l2[2] += (w.z & 0xFFFFu) + (w.z >> 16);
              l2[3] += (w.w & 0xFFFFu) + (w.w >> 16);
            }
          const int gx = (x0 >> 2) + 4 * c_q, gy = (y0 >> 2) + c_y2;
          if (a.lv[2].out != nullptr && gx < (g.nx >> 2) && gy < (g.ny >> 2)) {
            uint8_t* dst = a.lv[2].out + level_offset<POW2>(a.lv[2], (z0 >> 2) + c_z2, gy, gx);
            const uint32_t v = ((l2[0] + 32) >> 6) | (((l2[1] + 32) >> 6) << 8) | (((l2[2] + 32) >> 6) << 16) |
                               (((l2[3] + 32) >> 6) << 24);
            if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) *reinterpret_cast<uint32_t*>(dst) = v;
            else for (int b = 0; b < 4; b++) dst[b] = (uint8_t)(v >> (8 * b));
          }
        }
        uint32_t s3a = l2[0] + l2[1], s3b = l2[2] + l2[3];  // level-3 cells x3 = 2q, 2q + 1 (partial)
        s3a += __shfl_xor_sync(0xFFFFFFFFu, s3a, 1);
        s3b += __shfl_xor_sync(0xFFFFFFFFu, s3b, 1);
        s3a += __shfl_xor_sync(0xFFFFFFFFu, s3a, 2);
        s3b += __shfl_xor_sync(0xFFFFFFFFu, s3b, 2);
        if (c_q >= 0 && (lane & 3) == 0) {
          const int gx = (x0 >> 3) + 2 * c_q, gy = (y0 >> 3) + (c_y2 >> 1);
          if (a.lv[3].out != nullptr && gx < (g.nx >> 3) && gy < (g.ny >> 3)) {
            uint8_t* dst = a.lv[3].out + level_offset<POW2>(a.lv[3], (z0 >> 3) + (c_z2 >> 1), gy, gx);
            const uint32_t v = ((s3a + 256) >> 9) | (((s3b + 256) >> 9) << 8);
            if ((reinterpret_cast<uintptr_t>(dst) & 1) == 0) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)v;
            else { dst[0] = (uint8_t)v; dst[1] = (uint8_t)(v >> 8); }
          }
        }
        if constexpr (L == 4) {
          uint32_t s4v = s3a + s3b;
          s4v += __shfl_xor_sync(0xFFFFFFFFu, s4v, 4);
          s4v += __shfl_xor_sync(0xFFFFFFFFu, s4v, 8);
          if (c_q >= 0 && (lane & 15) == 0) {
            const int gx = (x0 >> 4) + c_q, gy = (y0 >> 4) + (c_y2 >> 2);
            if (a.lv[4].out != nullptr && gx < (g.nx >> 4) && gy < (g.ny >> 4))
              a.lv[4].out[level_offset<POW2>(a.lv[4], (z0 >> 4), gy, gx)] = (uint8_t)((s4v + 2048) >> 12);
          }
        }
      }
    }

#ifdef CTP_PHASE_TIMING
    const long long ph4 = clock64();
    t_data += ph1 - ph0; t_units += ph2 - ph1; t_bar += ph3 - ph2; t_lvl += ph4 - ph3;
#endif
    if (++since_flush == g.flush_tiles) {
      since_flush = 0;
      flush_counts<T>(hs, a.hist, THREADS, hot_base);
    }
    // next tile (row-major: x fastest)
    if (++tx_i == g.tiles_x) {
      tx_i = 0;
      if (++ty_i == g.tiles_y) { ty_i = 0; ++tz_i; }
    }
  }
  flush_counts<T>(hs, a.hist, THREADS, hot_base);
  // atlas rows stored into a peer's atlases (the fused gather of a sharded step):
  // system-scope fence, so they are visible to the peer before the collective that
  // follows this kernel on the stream completes the step
  if (a.fence_sys) __threadfence_system();
#ifdef CTP_PHASE_TIMING
  if ((blockIdx.x == 0 || blockIdx.x == gridDim.x / 2) && (threadIdx.x & 31) == 0 && (threadIdx.x >> 5) % 8 == 0)
    printf("PHASE cta %d warp %2d tiles %d total %lld  data-wait %lld  units %lld  barrier %lld  levels+refill %lld\n",
           (int)blockIdx.x, (int)(threadIdx.x >> 5), k, clock64() - t_start, t_data, t_units, t_bar, t_lvl);
#endif
}

template <typename T, int L, int NST, int MAXU, int THREADS>
static constexpr size_t smem_bytes() {
  using LY = PvLayout<T, L, MAXU>;
  static_assert(L < 3 || MAXU * LY::L1PU <= 16 * THREADS, "level-3 lane groups must fit in the CTA");
  return (size_t)NST * LY::STAGE_BYTES + LY::HIST_BYTES + 2 * LY::S1_BYTES + NST * 8;
}

// ---- TMA descriptor ---------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  });
  return fn;
}

template <typename T>
static int make_tmap(CUtensorMap* map, const T* vol, const PvGeom& g, int tz) {
  PFN_cuTensorMapEncodeTiled fn = encode_fn();
  CTP_REQUIRE(fn != nullptr, CTP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)g.nx * sizeof(T), (cuuint64_t)g.nx * g.ny * sizeof(T)};
  const cuuint32_t box[3] = {(cuuint32_t)g.box_x, (cuuint32_t)g.ty, (cuuint32_t)tz};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                  const_cast<T*>(vol), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CTP_REQUIRE(r == CUDA_SUCCESS, CTP_E_CUDA, "cuTensorMapEncodeTiled failed (%d): box (%d,%d,%d)", (int)r, g.box_x,
              g.ty, tz);
  return CTP_OK;
}

// tile geometry for at most `maxu` units per tile; boxes of <= 256 x-elements.
// Rows are staged whole when a 2^L x 2^L block row of the full width fits the
// tile (one box if the row fits in one, else whole boxes, the last one partly
// out of bounds and zero-filled): then the tile takes as many block rows as fit,
// so every level count keeps tiles of ~maxu units (2^L-row tiles of a wide
// volume would be 16-64x smaller for L <= 2).  Otherwise tiles are 2^L rows of
// whole boxes.
template <typename T>
static void plan_tiles(PvGeom& g, int nlev, int maxu) {
  constexpr int UXW = Vox<T>::UXW;
  const int uz = nlev == 0 ? 1 : 2;
  const int tz = 1 << nlev;
  const int64_t blk = 1LL << nlev;
  const int64_t xu_total = g.nx / UXW;
  const int64_t urows_per_block = (int64_t)(tz / uz) * (blk / uz);  // unit rows in a 2^L x 2^L block
  const int64_t box_u = kBoxX / UXW;
  const int64_t xu_stage = xu_total <= box_u ? xu_total : ((xu_total + box_u - 1) / box_u) * box_u;
  if (xu_stage * urows_per_block <= maxu) {
    g.txu = (int)xu_total;
    int64_t ky = maxu / (xu_stage * urows_per_block);
    const int64_t ky_max = (g.ny + blk - 1) / blk;
    if (ky > ky_max) ky = ky_max;
    if (ky * blk > 256) ky = 256 / blk;  // TMA box rows <= 256
    if (ky < 1) ky = 1;
    g.ty = (int)(ky * blk);
  } else {
    int64_t txu = maxu / urows_per_block;
    if (txu > xu_total) txu = xu_total;
    if (txu > box_u) txu = (txu / box_u) * box_u;  // a tile wider than one box is whole boxes
    g.txu = (int)txu;
    g.ty = (int)blk;
  }
  const int xw = g.txu * UXW;
  g.box_x = xw <= kBoxX ? xw : kBoxX;
  g.nboxes = (xw + g.box_x - 1) / g.box_x;
  g.box_bytes = (uint32_t)g.box_x * g.ty * tz * sizeof(T);
  g.tiles_x = (int)((xu_total + g.txu - 1) / g.txu);
  g.tiles_y = (g.ny + g.ty - 1) / g.ty;
}

template <typename T, int L, int THREADS, int NST, int MAXU, bool WANT0, bool POW2>
static int launch_k(const PvArgs& a, const CUtensorMap& map, int grid, cudaStream_t st) {
  constexpr size_t sm = smem_bytes<T, L, NST, MAXU, THREADS>();
  if constexpr (sm > 227 * 1024 - 1024) {  // a variant that does not fit (static smem: < 1 KB)
    set_error("preview: launch shape needs %zu bytes of shared memory", sm);
    return CTP_E_UNSUPPORTED;
  } else {
  auto kern = preview_kernel<T, L, THREADS, NST, MAXU, WANT0, POW2>;
  // once per kernel variant and device (function attributes are per context): the dynamic
  // shared-memory limit and the resident CTAs per SM -- two driver round trips off every
  // later launch's host path (config 1's step is 16 us on the device)
  static std::atomic<int> per_sm_of[64];
  int dev = 0;
  CTP_CUDA_CALL(cudaGetDevice(&dev));
  int per_sm = (dev >= 0 && dev < 64) ? per_sm_of[dev].load(std::memory_order_acquire) : 0;
  if (per_sm == 0) {
    CTP_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CTP_CUDA_CALL(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, sm));
    CTP_REQUIRE(per_sm >= 1, CTP_E_CUDA, "preview: kernel does not fit on an SM");
    if (dev >= 0 && dev < 64) per_sm_of[dev].store(per_sm, std::memory_order_release);
  }
  if (a.top != nullptr) {
    // the in-kernel LUT step has one grid barrier: a cooperative launch
    // guarantees every CTA is resident (one per SM here)
    if (grid > per_sm * num_sms()) grid = per_sm * num_sms();
    CUtensorMap map_copy = map;
    PvArgs a_copy = a;
    void* params[] = {&map_copy, &a_copy};
    CTP_CUDA_CALL(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(THREADS), params,
                                              sm, st));
    ++launch_counter();
    return CTP_OK;
  }
  kern<<<grid, THREADS, sm, st>>>(map, a);
  CTP_CUDA_CHECK_LAUNCH("preview_kernel");
  return CTP_OK;
  }
}

template <typename T, int L, int THREADS, int NST, int MAXU>
static int launch_v(PvArgs a, const T* vol, cudaStream_t st) {
  plan_tiles<T>(a.g, L, MAXU);
  constexpr int64_t kStage = PvLayout<T, L, MAXU>::STAGE_BYTES;
  CTP_REQUIRE((int64_t)a.g.box_bytes * a.g.nboxes <= kStage, CTP_E_UNSUPPORTED,
              "preview: tile of %d boxes x %u bytes exceeds the stage", a.g.nboxes, a.g.box_bytes);
  const int64_t n_tiles = (int64_t)a.g.tiles_x * a.g.tiles_y * (a.g.nz >> L);
  CTP_REQUIRE(n_tiles < (1LL << 31), CTP_E_INVALID, "preview: too many tiles");
  a.g.n_tiles = (int)n_tiles;
  // a counter word gains at most this many counts per tile
  constexpr int UZ = L == 0 ? 1 : 2;
  const int64_t vox_per_unit = (int64_t)Vox<T>::UXW * UZ * UZ;
  const int64_t per_tile = sizeof(T) == 2 ? (int64_t)MAXU * vox_per_unit                    // whole CTA
                                          : (int64_t)(THREADS / 32) * (MAXU / THREADS) * vox_per_unit;  // a lane column
  a.g.flush_tiles = (int)(kCountCap / per_tile);
  if (a.g.flush_tiles < 1) a.g.flush_tiles = 1;
  CUtensorMap map;
  int rc = make_tmap<T>(&map, vol, a.g, 1 << L);
  if (rc != CTP_OK) return rc;
  int grid = num_sms();
  if (a.g.n_tiles < grid) grid = a.g.n_tiles;
  bool pow2 = true;
  for (int l = 0; l <= L; l++) pow2 = pow2 && dst_is_pow2(a.lv[l]);
  const bool want0 = a.lv[0].out != nullptr;
  if (pow2) {
    if (want0) return launch_k<T, L, THREADS, NST, MAXU, true, true>(a, map, grid, st);
    return launch_k<T, L, THREADS, NST, MAXU, false, true>(a, map, grid, st);
  }
  if (want0) return launch_k<T, L, THREADS, NST, MAXU, true, false>(a, map, grid, st);
  return launch_k<T, L, THREADS, NST, MAXU, false, false>(a, map, grid, st);
}

// Launch-shape variants, selectable with CTP_PREVIEW_VARIANT for tuning
// (tools/prof_preview.py); the default is the fastest measured on B200.
static int preview_variant() {
  static const int v = [] {  // read once, thread-safe initialisation
    const char* e = getenv("CTP_PREVIEW_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <typename T, int L>
static int launch_l(const PvArgs& a, const T* vol, cudaStream_t st) {
  // defaults measured on B200 (tools/prof_preview.py): u8 is bound by the
  // shared-memory atomic pipe and gains from 32 warps/SM; u16 prefers 16
  switch (preview_variant()) {
    case 1: return launch_v<T, L, 512, 2, 1024>(a, vol, st);
    case 2: return launch_v<T, L, 512, 3, 512>(a, vol, st);
    case 3: return launch_v<T, L, 1024, 2, 1024>(a, vol, st);
    case 4: return launch_v<T, L, 512, 2, 512>(a, vol, st);
    case 5: return launch_v<T, L, 512, 4, 512>(a, vol, st);
    case 6:  // L = 0: 4 one-row units per thread, 64 KB tiles
      if constexpr (L == 0) return launch_v<T, L, 1024, 2, 4096>(a, vol, st);
      return launch_v<T, L, 1024, 2, 1024>(a, vol, st);
    default: {
      const bool small = (int64_t)a.g.nx * a.g.ny * a.g.nz < (int64_t(1) << 26);
      // L = 0: a unit is ONE 16-byte row vector, so 4 units per thread keep the tile
      // at 64 KB (1024-unit tiles were 16 KB: c2 with a level-0 atlas 0.513 -> 0.370 ms)
      if constexpr (L == 0) {
        if (!small) return launch_v<T, L, 1024, 2, 4096>(a, vol, st);
      }
      if constexpr (sizeof(T) == 1) {
        // small volumes (config 1: 16 MiB) are latency-bound: 16 warps/SM finish the
        // handful of tiles per CTA sooner (16.4 vs 18.1 us per graph-replayed step)
        if (small) return launch_v<T, L, 512, 2, 1024>(a, vol, st);
        return launch_v<T, L, 1024, 2, 1024>(a, vol, st);
      } else {
        return launch_v<T, L, 512, 2, 1024>(a, vol, st);
      }
    }
  }
}

struct AutoLut {  // the artifact-LUT step fused into the launch (ctp_preview_step_*)
  int n_top;
  uint64_t cutoff_floor;
  uint8_t* lut_out;
  uint8_t* flags_out;
  uint64_t* workspace;
};

template <typename T>
static int preview_impl(const T* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut,
                        int nlev, const ctp_level_out* levels, uint64_t* hist, void* stream,
                        const AutoLut* autolut = nullptr) {
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
  a.lut = lut;
  a.hist = reinterpret_cast<unsigned long long*>(hist);
  for (int l = 0; l < CTP_MAX_LEVELS; l++) {
    a.lv[l] = make_dst(levels[l], nx >> l, ny >> l, z_base >> l);
    if (l > nlev) a.lv[l].out = nullptr;
  }
  a.g.nx = (int)nx;
  a.g.ny = (int)ny;
  a.g.nz = (int)nz;
  a.top = nullptr;
  a.top_n = 0;
  a.cutoff_floor = 0;
  a.vmax = 0;
  a.lut_out = a.flags_out = nullptr;
  a.ws = nullptr;
  a.fence_sys = 0;
  for (int l = 0; l <= nlev; l++)
    if (levels[l].out != nullptr && (levels[l].flags & CTP_OUT_PEER)) a.fence_sys = 1;
  if (autolut != nullptr) {
    CTP_REQUIRE(1 <= autolut->n_top && autolut->n_top <= nz, CTP_E_INVALID, "n_top %d outside [1, %lld]",
                autolut->n_top, (long long)nz);  // mask.py:223-224
    CTP_REQUIRE(autolut->workspace != nullptr, CTP_E_INVALID, "preview step: workspace required");
    a.top = vol + (nz - autolut->n_top) * ny * nx;
    a.top_n = (int64_t)autolut->n_top * ny * nx;
    a.cutoff_floor = (unsigned long long)autolut->cutoff_floor;
    a.vmax = sizeof(T) == 2 ? 4095 : 0;
    a.lut_out = autolut->lut_out;
    a.flags_out = autolut->flags_out;
    a.ws = reinterpret_cast<unsigned long long*>(autolut->workspace);
    a.lut = nullptr;
  }

  cudaStream_t st = as_stream(stream);
  switch (nlev) {
    case 0: return launch_l<T, 0>(a, vol, st);
    case 1: return launch_l<T, 1>(a, vol, st);
    case 2: return launch_l<T, 2>(a, vol, st);
    case 3: return launch_l<T, 3>(a, vol, st);
    default: return launch_l<T, 4>(a, vol, st);
  }
}

}  // namespace ctp

extern "C" {

int ctp_preview_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut,
                   int32_t nlev, const ctp_level_out* levels, uint64_t* hist, void* stream) {
  return ctp::preview_impl<uint8_t>(vol, nz, ny, nx, z_base, lut, nlev, levels, hist, stream);
}

int ctp_preview_step_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int32_t n_top, uint64_t cutoff_floor,
                        int32_t nlev, const ctp_level_out* levels, uint64_t* hist, uint8_t* lut_out, uint8_t* flags_out,
                        uint64_t* workspace, void* stream) {
  const ctp::AutoLut al{n_top, cutoff_floor, lut_out, flags_out, workspace};
  return ctp::preview_impl<uint8_t>(vol, nz, ny, nx, 0, nullptr, nlev, levels, hist, stream, &al);
}

int ctp_preview_step_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int32_t n_top,
                         uint64_t cutoff_floor, int32_t nlev, const ctp_level_out* levels, uint64_t* hist4096,
                         uint8_t* lut_out, uint8_t* flags_out, uint64_t* workspace, void* stream) {
  const ctp::AutoLut al{n_top, cutoff_floor, lut_out, flags_out, workspace};
  return ctp::preview_impl<uint16_t>(vol, nz, ny, nx, 0, nullptr, nlev, levels, hist4096, stream, &al);
}

int ctp_preview_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base, const uint8_t* lut4096,
                    int32_t nlev, const ctp_level_out* levels, uint64_t* hist4096, void* stream) {
  CTP_REQUIRE(lut4096 != nullptr, CTP_E_INVALID, "ctp_preview_u16: a 4096-entry LUT is required");
  return ctp::preview_impl<uint16_t>(vol, nz, ny, nx, z_base, lut4096, nlev, levels, hist4096, stream);
}

}  // extern "C"

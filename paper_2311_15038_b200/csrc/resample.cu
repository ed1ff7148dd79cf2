// General-ratio box downscale and slicemap atlas packing (device side).
//
//   ctp_downscale_u8     <- volume.py:277-309 downscale_volume (+ _cell_starts, volume.py:265-274)
//   ctp_encode_atlas_u8  <- slicemap.py:120-142 packing + pipeline.py:226-237 _pad_to_cube
//   ctp_decode_atlas_u8  <- slicemap.py:145-155 decode_slicemaps
//
// The fused power-of-two pyramid lives in preview.cu; this file covers the
// non-integer ratios (e.g. the 160 -> 128 level of demo-scan-01 or 768 -> 512
// of config 5), which assign each source voxel to the cell containing its
// centre, so cells hold floor(n/t) or ceil(n/t) voxels per axis.
#include "ctp_common.cuh"

namespace ctp {

// start[j] = ceil((2 j n - t) / (2 t)), start[0] = 0, start[t] = n (volume.py:265-274);
// 32-bit arithmetic (the host keeps n, t < 2^15 so that 2 j n < 2^31)
__device__ __forceinline__ uint32_t cell_start(uint32_t j, uint32_t n, uint32_t t) {
  if (j == 0) return 0;
  if (j >= t) return n;
  return (2u * j * n - t + 2u * t - 1u) / (2u * t);
}

// One CTA per output row (jz, jy): the row's z and y cell bounds once, each
// thread sums the cells of its outputs along x (contiguous source segments).
__global__ void __launch_bounds__(256) downscale_u8_kernel(const uint8_t* __restrict__ in, int nz, int ny, int nx,
                                                           int tz, int ty, int tx, uint8_t* __restrict__ out) {
  const int64_t row = blockIdx.x;  // jz * ty + jy
  const uint32_t jz = (uint32_t)(row / ty), jy = (uint32_t)(row - (int64_t)jz * ty);
  const uint32_t ya = cell_start(jy, ny, ty), yb = cell_start(jy + 1, ny, ty);
  const uint32_t za = cell_start(jz, nz, tz), zb = cell_start(jz + 1, nz, tz);
  const uint32_t cyz = (yb - ya) * (zb - za);
  for (uint32_t jx = threadIdx.x; jx < (uint32_t)tx; jx += blockDim.x) {
    const uint32_t xa = cell_start(jx, nx, tx), xb = cell_start(jx + 1, nx, tx);
    uint64_t acc = 0;
    for (uint32_t z = za; z < zb; z++)
      for (uint32_t y = ya; y < yb; y++) {
        const uint8_t* r = in + ((int64_t)z * ny + y) * nx;
        uint32_t rs = 0;
        for (uint32_t x = xa; x < xb; x++) rs += __ldg(r + x);
        acc += rs;
      }
    const uint64_t cnt = (uint64_t)(xb - xa) * cyz;
    out[row * tx + jx] = (uint8_t)((2 * acc + cnt) / (2 * cnt));  // volume.py:306-308 round half up
  }
}

// Vector path of the same (16-byte rows, cells of <= 257 source rows, nx <= 16384):
// each thread owns 16 source columns, sums them over the output row's (z, y)
// cell rows in packed 16-bit lanes (even / odd bytes of each word), spills the
// column sums to shared memory, and the outputs of the row then sum their
// x-cells from there.  Every source byte is read once, with 16-byte loads.
__global__ void __launch_bounds__(256) downscale_u8_vec_kernel(const uint8_t* __restrict__ in, int nz, int ny, int nx,
                                                               int tz, int ty, int tx, int tpr,
                                                               uint8_t* __restrict__ out) {
  extern __shared__ uint32_t colsum_all[];  // (256 / tpr) rows x (nx + 16), then the tx + 1 x-cell starts
  // tpr threads per output row, 256 / tpr output rows at a time per CTA (grid-stride)
  const int rpc = blockDim.x / tpr;
  uint32_t* xs = colsum_all + (int64_t)rpc * (nx + 16);  // the x partition is the same for every row
  for (int j = threadIdx.x; j <= tx; j += blockDim.x) xs[j] = cell_start(j, nx, tx);
  __syncthreads();
  const int g = threadIdx.x / tpr, t = threadIdx.x - g * tpr;
  const int nc = nx / 16;  // 16-byte column chunks
  // column x lives at (x % 16) * (nc + 1) + x / 16: the 16 stores of a thread and
  // the x-cell reads of neighbouring outputs both spread over the banks
  uint32_t* colsum = colsum_all + (int64_t)g * (nx + 16);
  const int64_t rows = (int64_t)ty * tz;
  for (int64_t base = (int64_t)blockIdx.x * rpc; base < rows; base += (int64_t)gridDim.x * rpc) {
    const int64_t row = base + g;  // jz * ty + jy
    const bool live = row < rows;
    uint32_t ya = 0, yb = 0, za = 0, zb = 0;
    if (live) {
      const uint32_t jz = (uint32_t)(row / ty), jy = (uint32_t)(row - (int64_t)jz * ty);
      ya = cell_start(jy, ny, ty);
      yb = cell_start(jy + 1, ny, ty);
      za = cell_start(jz, nz, tz);
      zb = cell_start(jz + 1, nz, tz);
      for (int c = t; c < nc; c += tpr) {
        uint32_t ev[4] = {0, 0, 0, 0}, od[4] = {0, 0, 0, 0};
        for (uint32_t z = za; z < zb; z++)
          for (uint32_t y = ya; y < yb; y++) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + ((int64_t)z * ny + y) * nx + 16 * c));
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int i = 0; i < 4; i++) {
              ev[i] += w[i] & 0x00FF00FFu;
              od[i] += (w[i] >> 8) & 0x00FF00FFu;
            }
          }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          colsum[(4 * i + 0) * (nc + 1) + c] = ev[i] & 0xFFFFu;
          colsum[(4 * i + 1) * (nc + 1) + c] = od[i] & 0xFFFFu;
          colsum[(4 * i + 2) * (nc + 1) + c] = ev[i] >> 16;
          colsum[(4 * i + 3) * (nc + 1) + c] = od[i] >> 16;
        }
      }
    }
    __syncthreads();
    if (live) {
      const uint32_t cyz = (yb - ya) * (zb - za);
      for (uint32_t jx = t; jx < (uint32_t)tx; jx += tpr) {
        const uint32_t xa = xs[jx], xb = xs[jx + 1];
        uint32_t acc = 0;
        for (uint32_t x = xa; x < xb; x++) acc += colsum[(x & 15) * (nc + 1) + (x >> 4)];
        // floor((2 acc + cnt) / (2 cnt)) (volume.py:306-308, round half up), <= 255: a float
        // estimate corrected to the exact integer quotient (cnt <= 257 * 16384: 32-bit safe)
        const uint32_t cnt = (xb - xa) * cyz, num = 2u * acc + cnt, den = 2u * cnt;
        uint32_t q = (uint32_t)__fmul_rz((float)num, __frcp_rn((float)den));
        if ((q + 1) * den <= num) q++;
        if (q * den > num) q--;
        out[row * tx + jx] = (uint8_t)q;
      }
    }
    __syncthreads();  // colsum is rewritten by the next rows
  }
}

// Warp-per-output-row path (16-byte rows, cells of <= 257 source rows, x cells of
// <= WMAX columns, the cell tables and one column-sum row per warp in shared
// memory).  Cell starts (volume.py:265-274) are tabulated once per CTA -- the x
// table packed as (column-sum index of the cell's first column, width) -- so a
// row costs no division but jz = row / ty.  Per output row (jz, jy) a warp
//   1. sums its cell's source rows column-wise: each lane owns 16-byte column
//      chunks, every source byte read once with a 16-byte load (four in flight),
//      sums in packed 16-bit lanes (even / odd bytes);
//   2. writes the 16 column sums of each chunk with four 16-byte stores to a
//      column-sum row laid out as idx(x) = x + 4 * (x >> 5) -- chunk c starts at
//      word 16c + 4(c >> 1), so the 8 lanes of a 16-byte-store phase hit 8
//      distinct 4-bank groups (conflict-free);
//   3. sums each output's x cell from there (WMAX predicated reads) and rounds
//      half up, floor((2 acc + cnt) / (2 cnt)) (volume.py:306-308), with a
//      per-row magic multiplier per cell width (exact while 2 cnt < 4099), one
//      byte per lane and output (coalesced stores).
// No CTA barrier inside the loop: a warp only ever reads its own row.
constexpr int kDsWarps = 8;

__host__ __device__ __forceinline__ uint32_t ds_idx(uint32_t x) { return x + ((x >> 5) << 2); }

template <int WMAX>
__global__ void __launch_bounds__(32 * kDsWarps) downscale_u8_warp_kernel(const uint8_t* __restrict__ in, int nz,
                                                                          int ny, int nx, int tz, int ty, int tx,
                                                                          uint8_t* __restrict__ out) {
  extern __shared__ __align__(16) uint32_t dsm[];
  const int row_words = (int)ds_idx((uint32_t)nx) + 4;  // one column-sum row (16-byte multiple)
  // per output x (WMAX <= 2): idx(xa) | idx(second column, or of the warp row's zero
  // word) << 15 | (w - 1) << 30;  (WMAX > 2): idx(xa) | width << 20 | b << 26, b =
  // columns before the next 32-column boundary (where idx skips its 4 pad words)
  uint32_t* xt = dsm + kDsWarps * row_words;
  uint32_t* ys = xt + tx;
  uint32_t* zs = ys + ty + 1;
  for (int j = threadIdx.x; j < tx; j += blockDim.x) {
    const uint32_t xa = cell_start(j, nx, tx), xb = cell_start(j + 1, nx, tx);
    if constexpr (WMAX <= 2)
      xt[j] = ds_idx(xa) | ((xb - xa == 2 ? ds_idx(xa + 1) : ds_idx((uint32_t)nx)) << 15) | ((xb - xa - 1) << 30);
    else
      xt[j] = ds_idx(xa) | ((xb - xa) << 20) | ((32u - (xa & 31u)) << 26);
  }
  for (int w = threadIdx.x; w < kDsWarps; w += blockDim.x) dsm[w * row_words + ds_idx((uint32_t)nx)] = 0u;  // zero words
  for (int j = threadIdx.x; j <= ty; j += blockDim.x) ys[j] = cell_start(j, ny, ty);
  for (int j = threadIdx.x; j <= tz; j += blockDim.x) zs[j] = cell_start(j, nz, tz);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* colsum = dsm + warp * row_words;
  const uint32_t cs_base = (uint32_t)__cvta_generic_to_shared(colsum);
  const int nc = nx >> 4;
  const uint32_t rows = (uint32_t)ty * (uint32_t)tz;
  const uint32_t stride = gridDim.x * kDsWarps;
  const int64_t slice = (int64_t)ny * nx;
  for (uint32_t row = blockIdx.x * kDsWarps + warp; row < rows; row += stride) {
    const uint32_t jz = row / (uint32_t)ty, jy = row - jz * (uint32_t)ty;
    const uint32_t ya = ys[jy], yb = ys[jy + 1], za = zs[jz], zb = zs[jz + 1];
    const uint32_t cy = yb - ya, ncell = cy * (zb - za);
    const uint8_t* row0 = in + (int64_t)za * slice + (int64_t)ya * nx;  // source row (za, ya)
    for (int c = lane; c < nc; c += 32) {
      uint32_t ev[4] = {0, 0, 0, 0}, od[4] = {0, 0, 0, 0};
      uint32_t y = 0, z = 0;  // next cell row (row-major over (z, y))
      for (uint32_t r = 0; r < ncell; r += 4) {
        // the next four cell rows' offsets first (no memory dependence), then four loads in flight
        int64_t off[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          off[u] = (int64_t)z * slice + (int64_t)y * nx;
          if (++y == cy) {
            y = 0;
            ++z;
          }
        }
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
          q[u] = (r + u < ncell) ? __ldg(reinterpret_cast<const uint4*>(row0 + off[u] + 16 * c)) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
          for (int i = 0; i < 4; i++) {
            ev[i] += w[i] & 0x00FF00FFu;
            od[i] += (w[i] >> 8) & 0x00FF00FFu;
          }
        }
      }
      // columns 4i..4i+3 = (ev lo, od lo, ev hi, od hi)
      const uint32_t dst = cs_base + 4u * ds_idx(16u * (uint32_t)c);
#pragma unroll
      for (int i = 0; i < 4; i++)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * i), "r"(ev[i] & 0xFFFFu),
                     "r"(od[i] & 0xFFFFu), "r"(ev[i] >> 16), "r"(od[i] >> 16)
                     : "memory");
    }
    __syncwarp();
    uint8_t* orow = out + (int64_t)row * tx;
    auto lds = [&](uint32_t idx) -> uint32_t {
      uint32_t v;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(cs_base + 4u * idx));
      return v;
    };
    if (2u * (uint32_t)WMAX * ncell < 4099u) {
      // q = floor((2 acc + cnt) / (2 cnt)) by a magic multiplier of den = 2 w ncell: exact
      // while den < 4099 (num <= 255.5 den, num * (M - 2^32 / den) < 2^32 / den)
      if constexpr (WMAX <= 2) {
        uint32_t m1 = 0xFFFFFFFFu / (2u * ncell) + 1u, m2 = 0xFFFFFFFFu / (4u * ncell) + 1u;
        // opaque: otherwise the compiler folds the select into a division per output
        asm volatile("mov.u32 %0, %0;" : "+r"(m1));
        asm volatile("mov.u32 %0, %0;" : "+r"(m2));
        auto one = [&](uint32_t e) -> uint32_t {
          const uint32_t acc = lds(e & 0x7FFFu) + lds((e >> 15) & 0x7FFFu);
          const bool two = (e >> 30) != 0u;
          return __umulhi(2u * acc + (two ? 2u : 1u) * ncell, two ? m2 : m1);
        };
        if (((tx & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 3) == 0)) {
          // 4 consecutive outputs per lane: one 16-byte table load, one 4-byte store
          for (int j4 = lane; 4 * j4 < tx; j4 += 32) {
            const uint4 e = *reinterpret_cast<const uint4*>(xt + 4 * j4);
            *reinterpret_cast<uint32_t*>(orow + 4 * j4) =
                one(e.x) | (one(e.y) << 8) | (one(e.z) << 16) | (one(e.w) << 24);
          }
        } else {
          for (int jx = lane; jx < tx; jx += 32) orow[jx] = (uint8_t)one(xt[jx]);
        }
      } else {
        uint32_t mg = (lane >= 1 && lane <= WMAX) ? 0xFFFFFFFFu / (2u * (uint32_t)lane * ncell) + 1u : 0u;
        asm volatile("mov.u32 %0, %0;" : "+r"(mg));
        for (int j0 = 0; j0 < tx; j0 += 32) {  // warp-uniform trip count: every lane takes the shuffle
          const int jx = j0 + lane;
          const bool live = jx < tx;
          const uint32_t e = live ? xt[jx] : (1u << 20);
          const uint32_t i0 = e & 0xFFFFFu, w = (e >> 20) & 63u, b = e >> 26;
          uint32_t acc = 0;
#pragma unroll
          for (int k = 0; k < WMAX; k++)
            if ((uint32_t)k < w) acc += lds(i0 + k + ((uint32_t)k >= b ? 4u : 0u));
          const uint32_t m = __shfl_sync(0xFFFFFFFFu, mg, (int)w);
          if (live) orow[jx] = (uint8_t)__umulhi(2u * acc + w * ncell, m);
        }
      }
    } else {  // large cells: a float estimate corrected to the exact integer quotient
      for (int jx = lane; jx < tx; jx += 32) {
        const uint32_t e = xt[jx];
        uint32_t acc = 0, w;
        if constexpr (WMAX <= 2) {
          w = (e >> 30) + 1u;
          acc = lds(e & 0x7FFFu) + lds((e >> 15) & 0x7FFFu);
        } else {
          const uint32_t i0 = e & 0xFFFFFu, b = e >> 26;
          w = (e >> 20) & 63u;
          for (uint32_t k = 0; k < w; k++) acc += lds(i0 + k + (k >= b ? 4u : 0u));
        }
        const uint32_t cnt = w * ncell, num = 2u * acc + cnt, den = 2u * cnt;
        uint32_t q = (uint32_t)__fmul_rz((float)num, __frcp_rn((float)den));
        if ((q + 1) * den <= num) q++;
        if (q * den > num) q--;
        orow[jx] = (uint8_t)q;
      }
    }
    __syncwarp();  // the next row rewrites colsum
  }
}

// One CTA per atlas row (map m, row R of the atlas): every 16-byte chunk of the
// row is one slice row segment (slice k = m*grid^2 + (R / s)*grid + C / s, row
// R % s, columns C % s ..) copied with one 16-byte load and store -- or zero
// where the level is smaller than the cell (_pad_to_cube, pipeline.py:226-237).
// Byte path when s or the slice rows are not 16-byte granular.
__global__ void __launch_bounds__(256) encode_atlas_kernel(const uint8_t* __restrict__ cube, int64_t nz, int64_t ny,
                                                           int64_t nx, int s, int grid, int atlas_dim,
                                                           uint8_t* __restrict__ atlases) {
  const int64_t row = blockIdx.x;  // m * atlas_dim + R
  const int64_t m = row / atlas_dim;
  const int R = (int)(row - m * atlas_dim);
  const int cy = R / s, y = R - cy * s;
  const int64_t k0 = m * (int64_t)grid * grid + (int64_t)cy * grid;  // slice of cell (cy, 0)
  uint8_t* dst = atlases + row * atlas_dim;
  const bool vec = (s % 16 == 0) && (nx % 16 == 0) && (atlas_dim % 16 == 0);
  if (vec) {
    for (int C = threadIdx.x * 16; C < atlas_dim; C += blockDim.x * 16) {
      const int cx = C / s, x = C - cx * s;
      const int64_t k = k0 + cx;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (k < nz && y < ny && x < nx) v = __ldg(reinterpret_cast<const uint4*>(cube + (k * ny + y) * nx + x));
      *reinterpret_cast<uint4*>(dst + C) = v;
    }
  } else {
    for (int C = threadIdx.x; C < atlas_dim; C += blockDim.x) {
      const int cx = C / s, x = C - cx * s;
      const int64_t k = k0 + cx;
      dst[C] = (k < nz && y < ny && x < nx) ? __ldg(cube + (k * ny + y) * nx + x) : (uint8_t)0;
    }
  }
}

// One CTA per ATLAS row (map m, row R), the inverse of encode_atlas_kernel: every
// 16-byte chunk of the atlas row is one slice row segment (slice k = m*grid^2 +
// (R / s)*grid + C / s, row R % s, columns C % s ..) copied with one 16-byte load
// and store; cells past the last slice (k >= s) are skipped.  (A CTA per cube row
// left 7/8 of its threads idle for s = 512: 12% of HBM.)  Byte path when s or the
// atlas rows are not 16-byte granular.
__global__ void __launch_bounds__(256) decode_atlas_kernel(const uint8_t* __restrict__ atlases, int s, int grid,
                                                           int atlas_dim, uint8_t* __restrict__ cube) {
  const int64_t row = blockIdx.x;  // m * atlas_dim + R
  const int64_t m = row / atlas_dim;
  const int R = (int)(row - m * atlas_dim);
  const int cy = R / s, y = R - cy * s;
  const int64_t k0 = m * (int64_t)grid * grid + (int64_t)cy * grid;  // slice of cell (cy, 0)
  const uint8_t* src = atlases + row * atlas_dim;
  if (s % 16 == 0 && atlas_dim % 16 == 0) {
    for (int C = threadIdx.x * 16; C < atlas_dim; C += blockDim.x * 16) {
      const int cx = C / s, x = C - cx * s;
      const int64_t k = k0 + cx;
      if (k < s)
        *reinterpret_cast<uint4*>(cube + (k * s + y) * s + x) = __ldg(reinterpret_cast<const uint4*>(src + C));
    }
  } else {
    for (int C = threadIdx.x; C < atlas_dim; C += blockDim.x) {
      const int cx = C / s, x = C - cx * s;
      const int64_t k = k0 + cx;
      if (k < s) cube[(k * s + y) * s + x] = __ldg(src + C);
    }
  }
}

// mask.py:208-211 apply_circle_mask: keep (x, y) iff (x - cx)^2 + (y - cy)^2 <= r_eff^2,
// evaluated in fp64 with explicit round-to-nearest products/sums (no FMA
// contraction), i.e. exactly numpy's (ix - cx)**2 + (iy - cy)**2 <= r_eff**2.
__device__ __forceinline__ bool in_circle(int64_t x, int64_t y, double cx, double cy, double r2) {
  const double dx = __dsub_rn((double)x, cx), dy = __dsub_rn((double)y, cy);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r2;
}

// The kept set of row y is an interval [xa, xb] of x: the fp64 predicate is
// monotone in |fl(x - cx)| (every rounding step is monotone), so it holds on
// the integers around the one nearest cx and fails beyond two boundaries,
// found by binary search with the exact predicate (row_span_kernel, one thread
// per row y); every slice then applies the same spans with 16-byte copies.

__global__ void circle_span_kernel(int64_t ny, int64_t nx, double cx, double cy, double r2, int2* __restrict__ span) {
  const int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (y >= ny) return;
  int64_t xc = (int64_t)floor(cx + 0.5);
  if (xc > nx - 1) xc = nx - 1;
  if (xc < 0) xc = 0;
  if (xc + 1 <= nx - 1 && !in_circle(xc, y, cx, cy, r2) && in_circle(xc + 1, y, cx, cy, r2)) xc++;
  if (!in_circle(xc, y, cx, cy, r2)) {
    span[y] = make_int2(1, 0);  // empty
    return;
  }
  int64_t lo = 0, hi = xc;  // smallest x in [0, xc] inside
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (in_circle(mid, y, cx, cy, r2)) hi = mid; else lo = mid + 1;
  }
  const int64_t xa = lo;
  lo = xc;
  hi = nx - 1;  // largest x in [xc, nx - 1] inside
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (in_circle(mid, y, cx, cy, r2)) lo = mid; else hi = mid - 1;
  }
  span[y] = make_int2((int)xa, (int)lo);
}

// keep [xa, xb] of every row, zero the rest: one 16-byte chunk per thread
// (grid-stride) when rows are 16-byte granular, else one CTA per row, bytewise
__global__ void __launch_bounds__(256) circle_apply_vec_kernel(const uint8_t* __restrict__ in, uint32_t ny,
                                                               uint32_t nc, uint32_t total, const int2* __restrict__ span,
                                                               uint8_t* __restrict__ out) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
    const uint32_t row = c / nc, x = (c - row * nc) * 16;
    const int2 sp = span[row % ny];
    uint4 v = make_uint4(0, 0, 0, 0);
    if ((int)x >= sp.x && (int)x + 15 <= sp.y) {
      v = __ldg(reinterpret_cast<const uint4*>(in) + c);
    } else if ((int)x + 15 >= sp.x && (int)x <= sp.y) {  // a boundary chunk
      uint8_t b[16];
      *reinterpret_cast<uint4*>(b) = __ldg(reinterpret_cast<const uint4*>(in) + c);
#pragma unroll
      for (int q = 0; q < 16; q++)
        if ((int)x + q < sp.x || (int)x + q > sp.y) b[q] = 0;
      v = *reinterpret_cast<uint4*>(b);
    }
    reinterpret_cast<uint4*>(out)[c] = v;
  }
}

__global__ void __launch_bounds__(256) circle_apply_kernel(const uint8_t* __restrict__ in, int64_t ny, int64_t nx,
                                                           const int2* __restrict__ span, uint8_t* __restrict__ out) {
  const int64_t row = blockIdx.x;  // z * ny + y
  const int2 sp = span[row % ny];
  const uint8_t* src = in + row * nx;
  uint8_t* dst = out + row * nx;
  for (int64_t x = threadIdx.x; x < nx; x += blockDim.x) dst[x] = (x >= sp.x && x <= sp.y) ? __ldg(src + x) : 0;
}

static int grid1d(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_downscale_u8(const uint8_t* in, int64_t nz, int64_t ny, int64_t nx, int64_t tz, int64_t ty, int64_t tx,
                     uint8_t* out, void* stream) {
  CTP_REQUIRE(in && out, CTP_E_INVALID, "ctp_downscale_u8: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "ctp_downscale_u8: degenerate shape");
  // volume.py:287-289
  CTP_REQUIRE(1 <= tx && tx <= nx, CTP_E_INVALID, "target x=%lld outside [1, %lld]", (long long)tx, (long long)nx);
  CTP_REQUIRE(1 <= ty && ty <= ny, CTP_E_INVALID, "target y=%lld outside [1, %lld]", (long long)ty, (long long)ny);
  CTP_REQUIRE(1 <= tz && tz <= nz, CTP_E_INVALID, "target z=%lld outside [1, %lld]", (long long)tz, (long long)nz);
  cudaStream_t st = as_stream(stream);
  if (tx == nx && ty == ny && tz == nz) {  // volume.py:290-291
    CTP_CUDA_CALL(cudaMemcpyAsync(out, in, (size_t)(nx * ny * nz), cudaMemcpyDeviceToDevice, st));
    return CTP_OK;
  }
  CTP_REQUIRE(nx < 32768 && ny < 32768 && nz < 32768, CTP_E_UNSUPPORTED,
              "ctp_downscale_u8: axes of 32768 or more voxels are not supported (32-bit cell bounds)");
  // the vector path needs 16-byte rows, <= 257 source rows per cell (packed 16-bit
  // column sums) and the column sums of one row in shared memory
  const int64_t cell_rows = ((ny + ty - 1) / ty + 1) * ((nz + tz - 1) / tz + 1);
  const bool vec_ok = nx % 16 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 && nx <= 16384 && cell_rows <= 257;
  {
    // warp-per-row path: kDsWarps column-sum rows + the three cell tables in shared memory
    const size_t sm = ((size_t)kDsWarps * (ds_idx((uint32_t)nx) + 4) + (size_t)(tx + ty + tz + 2)) * sizeof(uint32_t);
    static const bool force_old = [] { const char* e = getenv("CTP_DOWNSCALE_OLD"); return e && e[0] == '1'; }();
    int64_t wx = 0;  // widest x cell (volume.py:265-274 starts, the kernel's 32-bit formula)
    for (int64_t j = 0, prev = 0; j < tx; j++) {
      const int64_t nxt = (j + 1 >= tx) ? nx : (2 * (j + 1) * nx - tx + 2 * tx - 1) / (2 * tx);
      if (nxt - prev > wx) wx = nxt - prev;
      prev = nxt;
    }
    if (vec_ok && sm <= 200 * 1024 && wx <= 16 && !force_old) {
      const int64_t rows = ty * tz;
      auto go = [&](auto kern) -> int {
        if (sm > 48 * 1024)
          CTP_CUDA_CALL(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int per_sm = 0;
        CTP_CUDA_CALL(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kDsWarps, sm));
        if (per_sm < 1) per_sm = 1;
        int64_t blocks = (rows + kDsWarps - 1) / kDsWarps;
        if (blocks > (int64_t)per_sm * num_sms()) blocks = (int64_t)per_sm * num_sms();
        kern<<<(unsigned)blocks, 32 * kDsWarps, sm, st>>>(in, (int)nz, (int)ny, (int)nx, (int)tz, (int)ty, (int)tx,
                                                           out);
        CTP_CUDA_CHECK_LAUNCH("downscale_u8_warp_kernel");
        return CTP_OK;
      };
      if (wx <= 2) return go(downscale_u8_warp_kernel<2>);
      if (wx <= 4) return go(downscale_u8_warp_kernel<4>);
      if (wx <= 8) return go(downscale_u8_warp_kernel<8>);
      return go(downscale_u8_warp_kernel<16>);
    }
  }
  if (vec_ok) {
    int tpr = 32;  // threads per output row: one 16-byte column chunk each, <= 256
    while (tpr < 256 && tpr * 16 < nx) tpr *= 2;
    const int rpc = 256 / tpr;
    const size_t sm = ((size_t)rpc * (nx + 16) + (size_t)tx + 1) * sizeof(uint32_t);
    if (sm > 48 * 1024)
      CTP_CUDA_CALL(cudaFuncSetAttribute(downscale_u8_vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t rows = ty * tz;
    int64_t blocks = (rows + rpc - 1) / rpc;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    downscale_u8_vec_kernel<<<(unsigned)blocks, 256, sm, st>>>(in, (int)nz, (int)ny, (int)nx, (int)tz, (int)ty,
                                                               (int)tx, tpr, out);
    CTP_CUDA_CHECK_LAUNCH("downscale_u8_vec_kernel");
    return CTP_OK;
  }
  downscale_u8_kernel<<<(unsigned)(ty * tz), 256, 0, st>>>(in, (int)nz, (int)ny, (int)nx, (int)tz, (int)ty, (int)tx,
                                                          out);
  CTP_CUDA_CHECK_LAUNCH("downscale_u8_kernel");
  return CTP_OK;
}

int ctp_encode_atlas_u8(const uint8_t* cube, int64_t nz, int64_t ny, int64_t nx, int32_t s, int32_t grid,
                        int32_t atlas_dim, int32_t map_count, uint8_t* atlases, void* stream) {
  CTP_REQUIRE(cube && atlases, CTP_E_INVALID, "ctp_encode_atlas_u8: null pointer");
  ctp_level_out lo{atlases, CTP_LAYOUT_ATLAS, s, grid, atlas_dim, map_count, 0};
  int rc = check_level_desc(lo, nx, ny, nz, 0);
  if (rc != CTP_OK) return rc;
  const int64_t rows = (int64_t)atlas_dim * map_count;
  CTP_REQUIRE(rows < (1LL << 31), CTP_E_INVALID, "ctp_encode_atlas_u8: too many atlas rows");
  encode_atlas_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(cube, nz, ny, nx, s, grid, atlas_dim, atlases);
  CTP_CUDA_CHECK_LAUNCH("encode_atlas_kernel");
  return CTP_OK;
}

int ctp_circle_mask_u8(const uint8_t* in, int64_t nz, int64_t ny, int64_t nx, double cx, double cy, double r_eff_sq,
                       uint8_t* out, void* stream) {
  CTP_REQUIRE(in && out, CTP_E_INVALID, "ctp_circle_mask_u8: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "ctp_circle_mask_u8: degenerate shape");
  // mask.py:202-205 (the radius / margin checks stay with the caller, which holds the Circle)
  CTP_REQUIRE(0.0 <= cx && cx < (double)nx && 0.0 <= cy && cy < (double)ny, CTP_E_INVALID,
              "center (%.1f, %.1f) outside %lldx%lld slice", cx, cy, (long long)nx, (long long)ny);
  CTP_REQUIRE(nx < (1LL << 31) && ny * nz < (1LL << 31), CTP_E_INVALID, "ctp_circle_mask_u8: shape too large");
  cudaStream_t st = as_stream(stream);
  int2* span = nullptr;
  CTP_CUDA_CALL(cudaMallocAsync(&span, (size_t)ny * sizeof(int2), st));
  circle_span_kernel<<<(unsigned)((ny + 127) / 128), 128, 0, st>>>(ny, nx, cx, cy, r_eff_sq, span);
  CTP_CUDA_CHECK_LAUNCH("circle_span_kernel");
  const int64_t chunks = nx / 16 * ny * nz;
  if ((nx & 15) == 0 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
      chunks < (1LL << 32)) {
    circle_apply_vec_kernel<<<grid1d(chunks, 256), 256, 0, st>>>(in, (uint32_t)ny, (uint32_t)(nx / 16),
                                                                  (uint32_t)chunks, span, out);
    CTP_CUDA_CHECK_LAUNCH("circle_apply_vec_kernel");
  } else {
    circle_apply_kernel<<<(unsigned)(ny * nz), 256, 0, st>>>(in, ny, nx, span, out);
    CTP_CUDA_CHECK_LAUNCH("circle_apply_kernel");
  }
  CTP_CUDA_CALL(cudaFreeAsync(span, st));
  return CTP_OK;
}

int ctp_decode_atlas_u8(const uint8_t* atlases, int32_t s, int32_t grid, int32_t atlas_dim, int32_t map_count,
                        uint8_t* cube, void* stream) {
  CTP_REQUIRE(cube && atlases, CTP_E_INVALID, "ctp_decode_atlas_u8: null pointer");
  ctp_level_out lo{const_cast<uint8_t*>(atlases), CTP_LAYOUT_ATLAS, s, grid, atlas_dim, map_count, 0};
  int rc = check_level_desc(lo, s, s, s, 0);
  if (rc != CTP_OK) return rc;
  const int64_t rows = (int64_t)atlas_dim * map_count;
  CTP_REQUIRE(rows < (1LL << 31), CTP_E_INVALID, "ctp_decode_atlas_u8: too many atlas rows");
  decode_atlas_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(atlases, s, grid, atlas_dim, cube);
  CTP_CUDA_CHECK_LAUNCH("decode_atlas_kernel");
  return CTP_OK;
}

}  // extern "C"

// Kernels 1 and 2: volume histograms, the artifact-bin LUT, and the stand-alone
// LUT filter.
//
//   ctp_hist_u8       <- volume.py:252-262 volume_histogram / volume.py:117-122 Histogram256.of
//   ctp_hist_u16      <- extension (4096-bin, 12-bit data)
//   ctp_lut_build     <- mask.py:215-231 artifact_bins (cutoff test) + mask.py:241-245 (LUT)
//   ctp_lut_apply_u8  <- mask.py:246 lut[volume.voxels]  (+ optional raw histogram)
//   ctp_lut_apply_u16 <- extension: filter o 16->8 rescale for any row length (+ 4096-bin histogram)
//
// Privatisation (measured in tools/microbench/hist_bench.cu on B200): per-lane
// columns [bin][lane] of u32 in shared memory, shared by the block's warps.
// Every lane of a warp hits its own bank (bank == lane) so a warp-wide ATOMS is
// conflict-free for ANY data distribution (warp-private [warp][bin] bins lose 2x
// on uniform data to bank conflicts).  Loads are 16-byte vectors, 4 in flight
// per thread.
#include "ctp_common.cuh"

namespace ctp {

constexpr int kHistThreads = 256;

// ---------------------------------------------------------------------------
// u8 histogram of a contiguous byte range
__global__ void __launch_bounds__(kHistThreads) hist_u8_kernel(const uint8_t* __restrict__ p, int64_t n,
                                                               unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[256 * 32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += kHistThreads) hs[i] = 0;
  __syncthreads();

  // split into head (unaligned), body (uint4), tail
  const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
  int64_t head = (int64_t)((16 - (addr & 15)) & 15);
  if (head > n) head = n;
  const int64_t nbody = (n - head) >> 4;
  const uint4* body = reinterpret_cast<const uint4*>(p + head);
  const int64_t tail0 = head + (nbody << 4);

  if (blockIdx.x == 0) {
    for (int64_t i = threadIdx.x; i < head; i += kHistThreads) atomicAdd(&hs[(uint32_t)p[i] * 32 + lane], 1u);
    for (int64_t i = tail0 + threadIdx.x; i < n; i += kHistThreads) atomicAdd(&hs[(uint32_t)p[i] * 32 + lane], 1u);
  }

  const int64_t stride = (int64_t)gridDim.x * kHistThreads * 4;
  int64_t i = (int64_t)blockIdx.x * kHistThreads * 4 + threadIdx.x;
  for (; i + 3 * kHistThreads < nbody; i += stride) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) q[u] = __ldcs(body + i + u * kHistThreads);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; k++)
#pragma unroll
        for (int b = 0; b < 4; b++) atomicAdd(&hs[((w[k] >> (8 * b)) & 255u) * 32 + lane], 1u);
    }
  }
  for (; i < nbody; i += kHistThreads) {  // remainder of this block's last stride
    uint4 q = __ldcs(body + i);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
      for (int b = 0; b < 4; b++) atomicAdd(&hs[((w[k] >> (8 * b)) & 255u) * 32 + lane], 1u);
  }
  __syncthreads();
  // bin = threadIdx.x: sum the 32 lane columns (rotated start -> conflict-free)
  const int bin = threadIdx.x;
  uint32_t s = 0;
#pragma unroll 8
  for (int k = 0; k < 32; k++) s += hs[bin * 32 + ((k + bin) & 31)];
  if (s) atomicAdd(hist + bin, (unsigned long long)s);
}

// ---------------------------------------------------------------------------
// u16 histogram (nbins <= 4096, saturating), block-shared bins
__global__ void __launch_bounds__(kHistThreads) hist_u16_kernel(const uint16_t* __restrict__ p, int64_t n,
                                                                int nbins, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[4096];
  for (int i = threadIdx.x; i < nbins; i += kHistThreads) hs[i] = 0;
  __syncthreads();
  const uint32_t top = (uint32_t)nbins - 1;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
  int64_t head = (int64_t)(((16 - (addr & 15)) & 15) >> 1);
  if (head > n) head = n;
  const int64_t nbody = (n - head) >> 3;
  const uint4* body = reinterpret_cast<const uint4*>(p + head);
  const int64_t tail0 = head + (nbody << 3);
  if (blockIdx.x == 0) {
    for (int64_t i = threadIdx.x; i < head; i += kHistThreads) atomicAdd(&hs[min((uint32_t)p[i], top)], 1u);
    for (int64_t i = tail0 + threadIdx.x; i < n; i += kHistThreads) atomicAdd(&hs[min((uint32_t)p[i], top)], 1u);
  }
  const int64_t stride = (int64_t)gridDim.x * kHistThreads * 4;
  int64_t i = (int64_t)blockIdx.x * kHistThreads * 4 + threadIdx.x;
  for (; i + 3 * kHistThreads < nbody; i += stride) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) q[u] = __ldcs(body + i + u * kHistThreads);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        atomicAdd(&hs[min(w[k] & 0xFFFFu, top)], 1u);
        atomicAdd(&hs[min(w[k] >> 16, top)], 1u);
      }
    }
  }
  for (; i < nbody; i += kHistThreads) {
    uint4 q = __ldcs(body + i);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      atomicAdd(&hs[min(w[k] & 0xFFFFu, top)], 1u);
      atomicAdd(&hs[min(w[k] >> 16, top)], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += kHistThreads)
    if (hs[b]) atomicAdd(hist + b, (unsigned long long)hs[b]);
}

// ---------------------------------------------------------------------------
// LUT from the top-slab histogram: mask.py:229-231 + mask.py:241-245
__global__ void lut_build_kernel(const unsigned long long* __restrict__ top_hist, int nbins,
                                 unsigned long long cutoff_floor, int vmax, uint8_t* __restrict__ lut,
                                 uint8_t* __restrict__ flags) {
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    const bool flagged = (b == 0) || (top_hist[b] > cutoff_floor);  // mask.py:230-231 ({0} | flagged)
    uint32_t val;
    if (vmax > 0) {
      const uint32_t v = min((uint32_t)b, (uint32_t)vmax);
      val = (uint32_t)((2ull * 255ull * v + (uint64_t)vmax) / (2ull * (uint64_t)vmax));  // frozen 16->8 rule
    } else {
      val = (uint32_t)b;
    }
    lut[b] = flagged ? 0 : (uint8_t)val;
    if (flags) flags[b] = flagged ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// out = lut[in] (+ raw histogram): per-lane columns whose low byte holds the
// LUT value, so ONE ATOMS both counts the voxel and returns lut[v]
// (count lives in bits 12..31, see preview.cu for the overflow bound).
constexpr uint32_t kCountOne = 1u << 12;

__global__ void __launch_bounds__(kHistThreads) lut_apply_u8_kernel(const uint8_t* __restrict__ in,
                                                                    uint8_t* __restrict__ out, int64_t n16,
                                                                    const uint8_t* __restrict__ lut,
                                                                    unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[256 * 32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += kHistThreads) hs[i] = lut ? lut[i >> 5] : (uint32_t)(i >> 5);
  __syncthreads();
  const uint4* src = reinterpret_cast<const uint4*>(in);
  uint4* dst = reinterpret_cast<uint4*>(out);
  // count field is 20 bits: a lane column gains <= 8 warps x 16 voxels per
  // iteration, and the host keeps iterations per block < 8000 (< 2^20 / 128).
  for (int64_t i = (int64_t)blockIdx.x * kHistThreads + threadIdx.x; i < n16; i += (int64_t)gridDim.x * kHistThreads) {
    uint4 q = __ldcs(src + i);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      uint32_t o[4];
#pragma unroll
      for (int b = 0; b < 4; b++) o[b] = atomicAdd(&hs[((w[k] >> (8 * b)) & 255u) * 32 + lane], kCountOne);
      r[k] = __byte_perm(__byte_perm(o[0], o[1], 0x0040), __byte_perm(o[2], o[3], 0x0040), 0x5410);
    }
    __stcs(dst + i, make_uint4(r[0], r[1], r[2], r[3]));
  }
  __syncthreads();
  if (hist) {
    const int bin = threadIdx.x;
    uint32_t s = 0;
#pragma unroll 8
    for (int k = 0; k < 32; k++) s += hs[bin * 32 + ((k + bin) & 31)] >> 12;
    if (s) atomicAdd(hist + bin, (unsigned long long)s);
  }
}

__global__ void lut_apply_tail_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n,
                                      const uint8_t* __restrict__ lut, unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t v = in[i];
    out[i] = lut ? lut[v] : v;
    if (hist) atomicAdd(hist + v, 1ull);
  }
}


// u16 (12-bit) filter o rescale for any length / alignment (the extension of
// mask.py:246 the fused pass uses, for rows that are not whole 16-byte
// vectors): out[i] = lut4096[min(in[i], 4095)], raw 4096-bin histogram in the
// same pass.  Per-block table of 4096 (lut | count << 12) words: the atomic's
// old word carries the LUT byte, as in the fused kernel; 20-bit count fields
// are flushed by the host keeping a block's share below 2^20 elements.
__global__ void __launch_bounds__(kHistThreads) lut_apply_u16_kernel(const uint16_t* __restrict__ in,
                                                                     uint8_t* __restrict__ out, int64_t n,
                                                                     const uint8_t* __restrict__ lut,
                                                                     unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[4096];
  for (int i = threadIdx.x; i < 4096; i += kHistThreads) hs[i] = lut[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kHistThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kHistThreads) {
    const uint32_t v = min((uint32_t)__ldcs(in + i), 4095u);
    out[i] = (uint8_t)atomicAdd(&hs[v], kCountOne);
  }
  __syncthreads();
  if (hist)
    for (int b = threadIdx.x; b < 4096; b += kHistThreads) {
      const uint32_t c = hs[b] >> 12;
      if (c) atomicAdd(hist + b, (unsigned long long)c);
    }
}

// The same over 16-byte vectors (8 voxels: one 16-byte load, one 8-byte store per
// thread and vector) for the aligned bulk of the array; the scalar kernel above
// takes the tail.
__global__ void __launch_bounds__(kHistThreads) lut_apply_u16_vec_kernel(const uint4* __restrict__ in,
                                                                         uint2* __restrict__ out, int64_t nv,
                                                                         const uint8_t* __restrict__ lut,
                                                                         unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[4096];
  for (int i = threadIdx.x; i < 4096; i += kHistThreads) hs[i] = lut[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kHistThreads + threadIdx.x; i < nv; i += (int64_t)gridDim.x * kHistThreads) {
    const uint4 q = __ldcs(in + i);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      o[2 * k] = atomicAdd(&hs[min(w[k] & 0xFFFFu, 4095u)], kCountOne);
      o[2 * k + 1] = atomicAdd(&hs[min(w[k] >> 16, 4095u)], kCountOne);
    }
    out[i] = make_uint2(__byte_perm(__byte_perm(o[0], o[1], 0x0040), __byte_perm(o[2], o[3], 0x0040), 0x5410),
                        __byte_perm(__byte_perm(o[4], o[5], 0x0040), __byte_perm(o[6], o[7], 0x0040), 0x5410));
  }
  __syncthreads();
  if (hist)
    for (int b = threadIdx.x; b < 4096; b += kHistThreads) {
      const uint32_t c = hs[b] >> 12;
      if (c) atomicAdd(hist + b, (unsigned long long)c);
    }
}

// ---------------------------------------------------------------------------
// One launch for the whole artifact-LUT step (mask.py:215-231 + 241-245):
// every CTA histograms a share of the top slab in shared memory and adds it to
// a global workspace; the LAST CTA to finish (grid-wide counter) builds the
// LUT and flags, zeroes the caller's main histogram for the coming fused pass,
// and resets the workspace, which therefore stays zero between calls.
template <typename T>
__global__ void __launch_bounds__(256) artifact_lut_kernel(const T* __restrict__ p, int64_t n, int nbins,
                                                           unsigned long long cutoff_floor, int vmax,
                                                           uint8_t* __restrict__ lut, uint8_t* __restrict__ flags,
                                                           unsigned long long* __restrict__ zero_hist,
                                                           unsigned long long* __restrict__ ws) {
  __shared__ uint32_t hs[4096];  // u8: 8 warp-private copies of 256 bins (merged below)
  __shared__ bool last;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  const uint32_t top = (uint32_t)nbins - 1;
  constexpr int PER = 16 / sizeof(T);  // elements per 16-byte vector
  const int64_t nv = (reinterpret_cast<uintptr_t>(p) & 15) == 0 ? n / PER : 0;  // scalar if unaligned
  const uint4* pv = reinterpret_cast<const uint4*>(p);
  uint32_t* wh = hs + (sizeof(T) == 1 ? (threadIdx.x >> 5) * 256 : 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 q = __ldg(pv + i);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if constexpr (sizeof(T) == 1) {
#pragma unroll
        for (int b = 0; b < 4; b++) atomicAdd(&wh[(w[k] >> (8 * b)) & 255u], 1u);
      } else {
        atomicAdd(&wh[min(w[k] & 0xFFFFu, top)], 1u);
        atomicAdd(&wh[min(w[k] >> 16, top)], 1u);
      }
    }
  }
  for (int64_t i = nv * PER + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&wh[min((uint32_t)__ldg(p + i), top)], 1u);
  __syncthreads();
  if constexpr (sizeof(T) == 1) {  // merge the warp copies into copy 0
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
      uint32_t t = 0;
      for (int c = 0; c < (int)(blockDim.x >> 5); c++) t += hs[c * 256 + b];
      hs[b] = t;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (hs[b]) atomicAdd(ws + b, (unsigned long long)hs[b]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ws + 4096, 1ull) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    const unsigned long long c = atomicExch(ws + b, 0ull);  // read + reset
    const bool flagged = (b == 0) || (c > cutoff_floor);     // mask.py:230-231
    uint32_t val = (uint32_t)b;
    if (vmax > 0) {
      const uint32_t v = min((uint32_t)b, (uint32_t)vmax);
      val = (uint32_t)((2ull * 255ull * v + (uint64_t)vmax) / (2ull * (uint64_t)vmax));
    }
    lut[b] = flagged ? 0 : (uint8_t)val;
    if (flags) flags[b] = flagged ? 1 : 0;
  }
  if (zero_hist)
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) zero_hist[b] = 0;
  if (threadIdx.x == 0) ws[4096] = 0;
}

static int grid_for(int64_t work_items, int per_block, int blocks_per_sm) {
  int64_t g = (work_items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)num_sms() * blocks_per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_hist_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z0, int64_t z1, uint64_t* hist,
                void* stream) {
  CTP_REQUIRE(vol && hist, CTP_E_INVALID, "ctp_hist_u8: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "ctp_hist_u8: degenerate shape");
  // volume.py:260-261
  CTP_REQUIRE(0 <= z0 && z0 < z1 && z1 <= nz, CTP_E_INVALID, "z_range (%lld, %lld) outside [0, %lld]",
              (long long)z0, (long long)z1, (long long)nz);
  const int64_t slice = ny * nx;
  const int64_t n = (z1 - z0) * slice;
  const int grid = grid_for(n / 16, kHistThreads * 4 * 4, 8);
  hist_u8_kernel<<<grid, kHistThreads, 0, as_stream(stream)>>>(vol + z0 * slice, n,
                                                               reinterpret_cast<unsigned long long*>(hist));
  CTP_CUDA_CHECK_LAUNCH("hist_u8_kernel");
  return CTP_OK;
}

int ctp_hist_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z0, int64_t z1, int32_t nbins,
                 uint64_t* hist, void* stream) {
  CTP_REQUIRE(vol && hist, CTP_E_INVALID, "ctp_hist_u16: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "ctp_hist_u16: degenerate shape");
  CTP_REQUIRE(nbins >= 2 && nbins <= 4096, CTP_E_INVALID, "nbins %d outside [2, 4096]", nbins);
  CTP_REQUIRE(0 <= z0 && z0 < z1 && z1 <= nz, CTP_E_INVALID, "z_range (%lld, %lld) outside [0, %lld]",
              (long long)z0, (long long)z1, (long long)nz);
  const int64_t slice = ny * nx;
  const int64_t n = (z1 - z0) * slice;
  const int grid = grid_for(n / 8, kHistThreads * 4 * 4, 8);
  hist_u16_kernel<<<grid, kHistThreads, 0, as_stream(stream)>>>(vol + z0 * slice, n, nbins,
                                                                reinterpret_cast<unsigned long long*>(hist));
  CTP_CUDA_CHECK_LAUNCH("hist_u16_kernel");
  return CTP_OK;
}

int ctp_lut_build(const uint64_t* top_hist, int32_t nbins, uint64_t cutoff_floor, int32_t rescale_vmax, uint8_t* lut,
                  uint8_t* flags, void* stream) {
  CTP_REQUIRE(top_hist && lut, CTP_E_INVALID, "ctp_lut_build: null pointer");
  CTP_REQUIRE(nbins >= 2 && nbins <= 4096, CTP_E_INVALID, "nbins %d outside [2, 4096]", nbins);
  CTP_REQUIRE(rescale_vmax >= 0, CTP_E_INVALID, "rescale_vmax %d < 0", rescale_vmax);
  CTP_REQUIRE(rescale_vmax > 0 || nbins <= 256, CTP_E_INVALID, "identity LUT needs nbins <= 256");
  lut_build_kernel<<<1, 1024, 0, as_stream(stream)>>>(reinterpret_cast<const unsigned long long*>(top_hist), nbins,
                                                      (unsigned long long)cutoff_floor, rescale_vmax, lut, flags);
  CTP_CUDA_CHECK_LAUNCH("lut_build_kernel");
  return CTP_OK;
}

int ctp_artifact_lut(const void* vol, int32_t elem_bytes, int64_t nz, int64_t ny, int64_t nx, int32_t n_top,
                     uint64_t cutoff_floor, int32_t rescale_vmax, uint8_t* lut, uint8_t* flags, uint64_t* zero_hist,
                     uint64_t* workspace, void* stream) {
  CTP_REQUIRE(vol && lut && workspace, CTP_E_INVALID, "ctp_artifact_lut: null pointer");
  CTP_REQUIRE(elem_bytes == 1 || elem_bytes == 2, CTP_E_UNSUPPORTED, "elem_bytes must be 1 or 2");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1, CTP_E_INVALID, "ctp_artifact_lut: degenerate shape");
  CTP_REQUIRE(1 <= n_top && n_top <= nz, CTP_E_INVALID, "n_top %d outside [1, %lld]", n_top, (long long)nz);  // mask.py:223-224
  CTP_REQUIRE(rescale_vmax >= 0 && (elem_bytes == 2) == (rescale_vmax > 0), CTP_E_INVALID,
              "u8 takes the identity LUT (vmax 0), u16 the 16->8 rescale (vmax > 0)");
  const int nbins = elem_bytes == 1 ? 256 : 4096;
  const int64_t slice = ny * nx;
  const int64_t n = (int64_t)n_top * slice;
  const int grid = grid_for(n / (16 / elem_bytes), 256 * 4, 2);
  auto* h = reinterpret_cast<unsigned long long*>(zero_hist);
  auto* w = reinterpret_cast<unsigned long long*>(workspace);
  if (elem_bytes == 1)
    artifact_lut_kernel<uint8_t><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const uint8_t*>(vol) + (nz - n_top) * slice, n, nbins, (unsigned long long)cutoff_floor, 0, lut,
        flags, h, w);
  else
    artifact_lut_kernel<uint16_t><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const uint16_t*>(vol) + (nz - n_top) * slice, n, nbins, (unsigned long long)cutoff_floor,
        rescale_vmax, lut, flags, h, w);
  CTP_CUDA_CHECK_LAUNCH("artifact_lut_kernel");
  return CTP_OK;
}

int ctp_lut_apply_u16(const uint16_t* in, uint8_t* out, int64_t n, const uint8_t* lut4096, uint64_t* hist4096,
                      void* stream) {
  CTP_REQUIRE(in && out && lut4096, CTP_E_INVALID, "ctp_lut_apply_u16: null pointer");
  CTP_REQUIRE(n >= 0, CTP_E_INVALID, "negative length");
  if (n == 0) return CTP_OK;
  auto* h = reinterpret_cast<unsigned long long*>(hist4096);
  int64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(in) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0 && n >= 8) {
    const int64_t nv = n / 8;
    int grid = grid_for(nv, kHistThreads, 8);
    while ((nv * 8 + (int64_t)grid - 1) / grid >= (1LL << 20) - 1) grid *= 2;  // a block's share fits the count field
    lut_apply_u16_vec_kernel<<<grid, kHistThreads, 0, as_stream(stream)>>>(reinterpret_cast<const uint4*>(in),
                                                                          reinterpret_cast<uint2*>(out), nv, lut4096, h);
    CTP_CUDA_CHECK_LAUNCH("lut_apply_u16_vec_kernel");
    done = nv * 8;
  }
  if (done == n) return CTP_OK;
  const int64_t rest = n - done;
  int grid = grid_for(rest, kHistThreads, 8);
  while ((rest + (int64_t)grid - 1) / grid >= (1LL << 20) - 1) grid *= 2;  // a block's share fits the count field
  lut_apply_u16_kernel<<<grid, kHistThreads, 0, as_stream(stream)>>>(in + done, out + done, rest, lut4096, h);
  CTP_CUDA_CHECK_LAUNCH("lut_apply_u16_kernel");
  return CTP_OK;
}

int ctp_lut_apply_u8(const uint8_t* in, uint8_t* out, int64_t n, const uint8_t* lut, uint64_t* hist, void* stream) {
  CTP_REQUIRE(in && out, CTP_E_INVALID, "ctp_lut_apply_u8: null pointer");
  CTP_REQUIRE(n >= 0, CTP_E_INVALID, "negative length");
  if (n == 0) return CTP_OK;
  auto* h = reinterpret_cast<unsigned long long*>(hist);
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  int64_t done = 0;
  if (aligned && n >= 16) {
    const int64_t n16 = n / 16;
    // per-block iteration count must stay below the 20-bit count field: a lane
    // column gains <= 8 warps * 16 voxels per iteration -> < 8192 iterations
    int grid = grid_for(n16, kHistThreads, 8);
    while ((n16 + (int64_t)grid * kHistThreads - 1) / ((int64_t)grid * kHistThreads) >= 8000) grid *= 2;
    lut_apply_u8_kernel<<<grid, kHistThreads, 0, as_stream(stream)>>>(in, out, n16, lut, h);
    CTP_CUDA_CHECK_LAUNCH("lut_apply_u8_kernel");
    done = n16 * 16;
  }
  if (done < n) {
    lut_apply_tail_kernel<<<grid_for(n - done, 256, 4), 256, 0, as_stream(stream)>>>(in + done, out + done, n - done,
                                                                                      lut, h);
    CTP_CUDA_CHECK_LAUNCH("lut_apply_tail_kernel");
  }
  return CTP_OK;
}

}  // extern "C"

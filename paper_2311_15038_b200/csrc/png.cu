// PNG scanline filtering of 8-bit grayscale atlases on the device (SURVEY.md
// s8(f) row 2: writing the atlases as PNG, slicemap.py:158-166, dominates the
// bundle time once the reduction runs in a millisecond).
//
// For every image row the kernel evaluates the five PNG filters (None, Sub,
// Up, Average, Paeth; bpp = 1), picks the one with the smallest sum of
// |signed residual| (the classic adaptive heuristic; ties -> lowest type) and
// writes the filter byte + the filtered row: the exact byte stream that the
// PNG IDAT zlib stream compresses.  The host deflates row blocks in parallel
// (paper_2311_15038_b200/png.py).  One CTA per row, HBM-bound: W bytes read
// twice (this row and the one above, L2-resident), W + 1 written.
#include "ctp_common.cuh"

namespace ctp {

constexpr int kPngThreads = 256;

__device__ __forceinline__ int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = abs(p - a), pb = abs(p - b), pc = abs(p - c);
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

__device__ __forceinline__ uint8_t residual(int f, int x, int a, int b, int c) {
  switch (f) {
    case 0: return (uint8_t)x;
    case 1: return (uint8_t)(x - a);
    case 2: return (uint8_t)(x - b);
    case 3: return (uint8_t)(x - ((a + b) >> 1));
    default: return (uint8_t)(x - paeth(a, b, c));
  }
}

__device__ __forceinline__ uint32_t cost(uint8_t r) { return (uint32_t)abs((int)(int8_t)r); }

// rows = n_images * height; row r of image i = r % height
__global__ void __launch_bounds__(kPngThreads) png_filter_kernel(const uint8_t* __restrict__ in, int64_t height,
                                                                 int width, uint8_t* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const bool first = (row % height) == 0;
  const uint8_t* cur = in + row * width;
  const uint8_t* up = first ? nullptr : cur - width;
  uint32_t s[5] = {0, 0, 0, 0, 0};
  for (int x = threadIdx.x; x < width; x += kPngThreads) {
    const int v = __ldg(cur + x);
    const int a = x > 0 ? __ldg(cur + x - 1) : 0;
    const int b = up ? __ldg(up + x) : 0;
    const int c = (up && x > 0) ? __ldg(up + x - 1) : 0;
#pragma unroll
    for (int f = 0; f < 5; f++) s[f] += cost(residual(f, v, a, b, c));
  }
  __shared__ uint32_t red[5][kPngThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < 5; f++) {
    uint32_t t = s[f];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if (lane == 0) red[f][warp] = t;
  }
  __syncthreads();
  __shared__ int best_f;
  if (threadIdx.x == 0) {
    uint64_t best = ~0ull;
    int bf = 0;
    for (int f = 0; f < 5; f++) {
      uint64_t t = 0;
      for (int w = 0; w < kPngThreads / 32; w++) t += red[f][w];
      if (t < best) { best = t; bf = f; }
    }
    best_f = bf;
  }
  __syncthreads();
  const int f = best_f;
  uint8_t* dst = out + row * (int64_t)(width + 1);
  if (threadIdx.x == 0) dst[0] = (uint8_t)f;
  for (int x = threadIdx.x; x < width; x += kPngThreads) {
    const int v = __ldg(cur + x);
    const int a = x > 0 ? __ldg(cur + x - 1) : 0;
    const int b = up ? __ldg(up + x) : 0;
    const int c = (up && x > 0) ? __ldg(up + x - 1) : 0;
    dst[1 + x] = residual(f, v, a, b, c);
  }
}

}  // namespace ctp

using namespace ctp;

extern "C" int ctp_png_filter_u8(const uint8_t* images, int32_t n_images, int64_t height, int64_t width, uint8_t* out,
                                 void* stream) {
  CTP_REQUIRE(images && out, CTP_E_INVALID, "ctp_png_filter_u8: null pointer");
  CTP_REQUIRE(n_images >= 1 && height >= 1 && width >= 1 && width < (1 << 30), CTP_E_INVALID,
              "ctp_png_filter_u8: bad shape (%d, %lld, %lld)", n_images, (long long)height, (long long)width);
  const int64_t rows = (int64_t)n_images * height;
  CTP_REQUIRE(rows < (1LL << 31), CTP_E_INVALID, "ctp_png_filter_u8: too many rows");
  png_filter_kernel<<<(unsigned)rows, kPngThreads, 0, as_stream(stream)>>>(images, height, (int)width, out);
  CTP_CUDA_CHECK_LAUNCH("png_filter_kernel");
  return CTP_OK;
}

// PNG scanline filtering of 8-bit grayscale atlases on the device (SURVEY.md
// s8(f) row 2: writing the atlases as PNG, slicemap.py:158-166, dominates the
// bundle time once the reduction runs in a millisecond).
//
// For every image row the kernel evaluates the five PNG filters (None, Sub,
// Up, Average, Paeth; bpp = 1), picks the one whose residual bytes have the
// lowest order-0 entropy (or a fixed one) and writes the filter byte + the
// filtered row: the exact byte stream that the PNG IDAT zlib stream
// compresses.  The host deflates row blocks in parallel
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


// rows = n_images * height; row r of image i = r % height
__global__ void __launch_bounds__(kPngThreads) png_filter_kernel(const uint8_t* __restrict__ in, int64_t height,
                                                                 int width, int fixed, uint8_t* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const bool first = (row % height) == 0;
  const uint8_t* cur = in + row * width;
  const uint8_t* up = first ? nullptr : cur - width;
  // adaptive choice: the filter whose residual bytes have the lowest order-0
  // entropy in this row (sum_b h_b log2(W / h_b) bits) -- a Huffman coder's
  // view; the classic min-sum-|residual| rule prefers smoothing filters that
  // lose on noisy slices (c2 atlases: 44.2 MB vs 32.6 MB with entropy)
  __shared__ uint32_t hist[5][256];
  __shared__ float red[5][kPngThreads / 32];
  __shared__ int best_f;
  if (fixed < 0) {
    for (int i = threadIdx.x; i < 5 * 256; i += kPngThreads) (&hist[0][0])[i] = 0;
    __syncthreads();
    for (int x = threadIdx.x; x < width; x += kPngThreads) {
      const int v = __ldg(cur + x);
      const int a = x > 0 ? __ldg(cur + x - 1) : 0;
      const int b = up ? __ldg(up + x) : 0;
      const int c = (up && x > 0) ? __ldg(up + x - 1) : 0;
#pragma unroll
      for (int f = 0; f < 5; f++) atomicAdd(&hist[f][residual(f, v, a, b, c)], 1u);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float e[5];
#pragma unroll
    for (int f = 0; f < 5; f++) {
      const uint32_t h = hist[f][threadIdx.x];  // kPngThreads == 256 bins
      float t = h ? (float)h * __log2f((float)h) : 0.f;  // sum h log2 h: larger = lower entropy
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
      e[f] = t;
      if (lane == 0) red[f][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float best = -1.f;
      int bf = 0;
      for (int f = 0; f < 5; f++) {
        float t = 0.f;
        for (int w = 0; w < kPngThreads / 32; w++) t += red[f][w];
        if (t > best) { best = t; bf = f; }
      }
      best_f = bf;
    }
    (void)e;
  } else if (threadIdx.x == 0) {
    best_f = fixed;
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

extern "C" int ctp_png_filter_u8(const uint8_t* images, int32_t n_images, int64_t height, int64_t width, int32_t filter,
                                 uint8_t* out, void* stream) {
  CTP_REQUIRE(images && out, CTP_E_INVALID, "ctp_png_filter_u8: null pointer");
  CTP_REQUIRE(n_images >= 1 && height >= 1 && width >= 1 && width < (1 << 30), CTP_E_INVALID,
              "ctp_png_filter_u8: bad shape (%d, %lld, %lld)", n_images, (long long)height, (long long)width);
  const int64_t rows = (int64_t)n_images * height;
  CTP_REQUIRE(rows < (1LL << 31), CTP_E_INVALID, "ctp_png_filter_u8: too many rows");
  CTP_REQUIRE(filter >= -1 && filter <= 4, CTP_E_INVALID, "ctp_png_filter_u8: filter %d outside [-1, 4]", filter);
  png_filter_kernel<<<(unsigned)rows, kPngThreads, 0, as_stream(stream)>>>(images, height, (int)width, filter, out);
  CTP_CUDA_CHECK_LAUNCH("png_filter_kernel");
  return CTP_OK;
}

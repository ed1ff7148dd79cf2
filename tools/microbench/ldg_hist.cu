// Microbenchmark: is the fused u8 pass bound by shared-memory bandwidth (TMA fill +
// LDS read + one ATOMS per voxel)?  Histogram + LUT (one PRMT + ATOMS per voxel,
// 256-byte bin rows as in preview.cu) over a 1 GiB volume in HBM, the voxels
// brought in by:
//   G: ld.global.nc.L1::no_allocate.v4 straight into registers, the next
//      iteration's 64 bytes per thread prefetched (no shared-memory staging)
//   R: G without the atomics (pure streaming read: the HBM ceiling of this access)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldg_hist ldg_hist.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void gen(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t w = 0;
    for (int b = 0; b < 4; b++) {
      const uint32_t hb = mix32((uint32_t)i * 4 + b);
      const int s = (hb & 255) + ((hb >> 8) & 255) + ((hb >> 16) & 255) + (hb >> 24);
      int v = 20 + (s - 510) * 6 / 148;
      v = v < 0 ? 0 : (v > 255 ? 255 : v);
      w |= (uint32_t)v << (8 * b);
    }
    p[i] = w;
  }
}
__device__ __forceinline__ uint4 ldg_na(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int MODE, int THR, int VPT>  // VPT: 16-byte vectors per thread per iteration
__global__ void __launch_bounds__(THR, 1) k(const uint4* __restrict__ vol, size_t nvec, unsigned long long* sink) {
  extern __shared__ __align__(16) uint32_t tb[];  // 256 rows x 64 words
  for (int i = threadIdx.x; i < 256 * 64; i += THR) tb[i] = (uint32_t)(i >> 6);
  __syncthreads();
  const uint32_t tbl = (uint32_t)__cvta_generic_to_shared(tb);
  const uint32_t lane4 = 4u * (threadIdx.x & 31);
  const size_t per_iter = (size_t)gridDim.x * THR * VPT;
  size_t base = ((size_t)blockIdx.x * THR + threadIdx.x);
  uint4 cur[VPT], nxt[VPT];
#pragma unroll
  for (int j = 0; j < VPT; j++) cur[j] = ldg_na(vol + (base + (size_t)j * gridDim.x * THR) % nvec);
  uint32_t acc = 0;
  for (size_t it = 0; it * per_iter < nvec; it++) {
    const size_t nb = base + per_iter;
#pragma unroll
    for (int j = 0; j < VPT; j++) nxt[j] = ldg_na(vol + (nb + (size_t)j * gridDim.x * THR) % nvec);
#pragma unroll
    for (int j = 0; j < VPT; j++) {
      const uint32_t w[4] = {cur[j].x, cur[j].y, cur[j].z, cur[j].w};
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (MODE == 0) {
#pragma unroll
          for (int b = 0; b < 4; b++) {
            uint32_t old;
            const uint32_t off = __byte_perm(w[q], lane4, 0x7604u | ((uint32_t)b << 4));
            asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(tbl + off), "r"(4096u));
            acc += old;
          }
        } else {
          acc += w[q];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < VPT; j++) cur[j] = nxt[j];
    base = nb;
  }
  atomicAdd(sink, (unsigned long long)(acc & 0xFFF));
}

template <int MODE, int THR, int VPT>
int run(const uint4* d, size_t nvec, unsigned long long* sink, int sms, const char* name) {
  const int smem = 256 * 64 * 4;
  CK(cudaFuncSetAttribute(k<MODE, THR, VPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<MODE, THR, VPT><<<sms, THR, smem>>>(d, nvec, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 10;
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) k<MODE, THR, VPT><<<sms, THR, smem>>>(d, nvec, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double vox = (double)nvec * 16;
  printf("  %-44s THR=%4d VPT=%d  %.4f ms  %.1f GB/s  %.2f vox/clk/SM (1.965 GHz)\n", name, THR, VPT, ms, vox / ms / 1e6,
         vox / (ms * 1e-3) / (sms * 1.965e9));
  return 0;
}

int main() {
  const size_t n = (size_t)1 << 30;  // 1 GiB of u8 voxels
  uint32_t* d;
  unsigned long long* sink;
  CK(cudaMalloc(&d, n));
  CK(cudaMalloc(&sink, 8));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  gen<<<sms * 8, 256>>>(d, n / 4);
  CK(cudaDeviceSynchronize());
  const uint4* v = reinterpret_cast<const uint4*>(d);
  const size_t nvec = n / 16;
  printf("1 GiB u8 volume, N(20,6)-like bytes, %d CTAs\n", sms);
  if (run<1, 1024, 4>(v, nvec, sink, sms, "R streaming read only") || run<1, 512, 8>(v, nvec, sink, sms, "R streaming read only") ||
      run<0, 1024, 2>(v, nvec, sink, sms, "G ldg + PRMT/ATOMS") || run<0, 1024, 4>(v, nvec, sink, sms, "G ldg + PRMT/ATOMS") ||
      run<0, 512, 4>(v, nvec, sink, sms, "G ldg + PRMT/ATOMS") || run<0, 512, 8>(v, nvec, sink, sms, "G ldg + PRMT/ATOMS"))
    return 1;
  return 0;
}

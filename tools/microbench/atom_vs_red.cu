// Microbenchmark: per-voxel shared-memory cost of the u8 histogram + LUT, data
// staged in shared memory (as the fused kernel's TMA tiles are):
//   A: one atom.shared.add with return on [bin][lane] counter words whose low
//      byte is the LUT (the fused kernel's scheme)
//   B: red.shared.add (no return) on [bin][lane] counters + ld.shared of the LUT
//      from a separate [bin][lane] word table
//   C: red.shared.add only (histogram without the LUT: the lower bound)
//   D: A with [bin][64-word] rows (256 B per bin, lanes in words 0..31): the
//      address offset (v << 8) | (lane << 2) is ONE PRMT merging the voxel byte
//      with the lane byte, the table base is a uniform register ([R+UR])
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atom_vs_red atom_vs_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kStage = 65536;
constexpr int kReps = 1024;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(unsigned long long* sink) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint4* st = reinterpret_cast<uint4*>(sm);
  uint32_t* cnt = sm + kStage / 4;         // 256 x 32 words (D: 256 x 64)
  uint32_t* lut = cnt + 256 * 64;          // 256 x 32 words
  for (int i = threadIdx.x; i < kStage / 4; i += 1024) {
    const uint32_t h = mix32(i * 2654435761u + blockIdx.x);
    uint32_t w = 0;
    for (int b = 0; b < 4; b++) {  // ~N(20, 6)-like bytes
      const uint32_t hb = mix32(h + b);
      const int s = (hb & 255) + ((hb >> 8) & 255) + ((hb >> 16) & 255) + (hb >> 24);
      int v = 20 + (s - 510) * 6 / 148;
      v = v < 0 ? 0 : (v > 255 ? 255 : v);
      w |= (uint32_t)v << (8 * b);
    }
    sm[i] = w;
  }
  for (int i = threadIdx.x; i < 256 * 64; i += 1024) cnt[i] = (uint32_t)(i >> (MODE == 3 ? 6 : 5));
  for (int i = threadIdx.x; i < 256 * 32; i += 1024) lut[i] = (uint32_t)(i >> 5);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t cb = (uint32_t)__cvta_generic_to_shared(cnt) + 4u * lane;
  const uint32_t lb = (uint32_t)__cvta_generic_to_shared(lut) + 4u * lane;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(st);
  const uint32_t cb0 = (uint32_t)__cvta_generic_to_shared(cnt);
  const uint32_t lane4 = 4u * lane;
  uint32_t acc = 0;
  for (int r = 0; r < kReps; r++) {
    for (int i = threadIdx.x; i < kStage / 16; i += 1024) {
      uint4 q;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(sb + 16u * i));
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int kk = 0; kk < 4; kk++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
          const uint32_t v = __byte_perm(w[kk], 0u, 0x4440u | (uint32_t)b);
          if (MODE == 3) {
            uint32_t old;
            const uint32_t off = __byte_perm(w[kk], lane4, 0x7604u | ((uint32_t)b << 4));  // [b3 b2 v 4*lane]
            asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(cb0 + off), "r"(4096u));
            acc += old;
          } else if (MODE == 0) {
            uint32_t old;
            asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(cb + (v << 7)), "r"(4096u));
            acc += old;
          } else if (MODE == 1) {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cb + (v << 7)), "r"(4096u));
            uint32_t f;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(f) : "r"(lb + (v << 7)));
            acc += f;
          } else {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cb + (v << 7)), "r"(4096u));
          }
        }
    }
  }
  atomicAdd(sink, (unsigned long long)(acc & 0xFFF));
}

template <int MODE>
int run(int sms, unsigned long long* sink, const char* name) {
  const int smem = kStage + 3 * 256 * 32 * 4;
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<MODE><<<sms, 1024, smem>>>(sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 5; i++) k<MODE><<<sms, 1024, smem>>>(sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double vox = (double)sms * kReps * kStage;
  printf("  %-34s %.3f ms  %.1f Gvox/s  %.2f vox/clk/SM (1.9 GHz)\n", name, ms, vox / ms / 1e6, vox / (ms * 1e-3) / (sms * 1.9e9));
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  printf("u8 histogram + LUT, data in shared memory, 1024 thr x %d CTAs\n", sms);
  if (run<0>(sms, sink, "A atom-with-return (LUT in word)") || run<1>(sms, sink, "B red + ld LUT") ||
      run<2>(sms, sink, "C red only (no LUT)") || run<3>(sms, sink, "D atom, one-PRMT address") ||
      run<0>(sms, sink, "A atom-with-return (LUT in word)") || run<3>(sms, sink, "D atom, one-PRMT address"))
    return 1;
  return 0;
}

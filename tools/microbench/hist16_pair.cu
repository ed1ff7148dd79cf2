// Microbenchmark: candidate shared-memory schemes for the u16 fused pass's
// "histogram + filter o rescale" step (one atomic per voxel, old word -> f):
//   V0  [bin][lane%4] 32-bit words, LUT byte in bits 0..7, count in 12..31
//       (the round-1 kernel: 64 KB, ~3.3 wavefronts per warp ATOMS)
//   V3  the same with 8 columns (128 KB, ~3.0 wavefronts)
//   V1  [bin>>1][lane%16] words holding TWO adjacent bins as 16-bit halves,
//       bit 0 of a half = "keep" (bin not flagged), count in bits 1..15; the
//       increment and the keep bit are selected by rotating by 16*(bin&1);
//       f = keep * ((v*4081 + 32768) >> 16)  (== (2*255*v + 4095) // 8190 for
//       v in 0..4095); 128 KB, ~2.0 wavefronts
//   V4  V1 hand-scheduled; V5 V4 with the keep bit at bit 15 of a half (PRMT mask)
//   V2  [bin][lane%8] words, the 16-bit half chosen by lane bit 3 (constant
//       increment and keep-bit position per lane); 128 KB, ~3.0 wavefronts
// Data: config-3-like 12-bit values staged once in shared memory (the fused
// kernel's tiles arrive by TMA), histogrammed kReps times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o hist16_pair hist16_pair.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void gen(uint16_t* p, size_t n, int uniform) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = mix32((uint32_t)i * 2654435761U + (uint32_t)(i >> 32));
    uint32_t h2 = mix32(h ^ 0x9e3779b9U);
    int s = (h & 255) + ((h >> 8) & 255) + ((h >> 16) & 255) + (h >> 24);
    int v;
    const int sel = h2 & 1023;
    if (sel < 10) v = (h2 >> 10) & 4095;
    else if (sel < 92) v = 2800 + (s - 510) * 300 / 148;
    else v = 400 + (s - 510) * 120 / 148;
    if (uniform) v = h2 & 4095;
    v = v < 0 ? 0 : (v > 4095 ? 4095 : v);
    p[i] = (uint16_t)v;
  }
}

__device__ __forceinline__ uint32_t atom_ret(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}
__device__ __forceinline__ uint32_t rotl(uint32_t x, uint32_t s) { return __funnelshift_l(x, x, s); }
__device__ __forceinline__ uint32_t rotr(uint32_t x, uint32_t s) { return __funnelshift_r(x, x, s); }
__device__ __forceinline__ uint32_t min_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

constexpr int kStage = 32768;
constexpr int kReps = 1024;

template <int V>
struct Cfg;
template <> struct Cfg<0> { static constexpr int WORDS = 4096 * 4; };
template <> struct Cfg<3> { static constexpr int WORDS = 4096 * 8; };
template <> struct Cfg<1> { static constexpr int WORDS = 2048 * 16; };
template <> struct Cfg<2> { static constexpr int WORDS = 4096 * 8; };
template <> struct Cfg<4> { static constexpr int WORDS = 2048 * 16; };
template <> struct Cfg<5> { static constexpr int WORDS = 2048 * 16; };

template <int V, int THR>
__global__ void __launch_bounds__(THR, 1) k(const uint4* __restrict__ in, size_t n16, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint32_t sm[];
  uint32_t* tb = sm;                                   // table first (offset 0 of dynamic smem)
  uint4* st = reinterpret_cast<uint4*>(sm + Cfg<V>::WORDS);
  for (int i = threadIdx.x; i < Cfg<V>::WORDS; i += THR) {
    if (V == 0) tb[i] = (uint32_t)((i / 4) * 255 / 4095) & ((i / 4 >= 300 && i / 4 < 500) ? 0 : 0xFF);
    else if (V == 3) tb[i] = (uint32_t)((i / 8) * 255 / 4095) & ((i / 8 >= 300 && i / 8 < 500) ? 0 : 0xFF);
    else if (V == 1 || V == 4) {
      const int b0 = 2 * (i / 16), b1 = b0 + 1;
      tb[i] = ((b0 >= 300 && b0 < 500) ? 0u : 1u) | ((b1 >= 300 && b1 < 500) ? 0u : 0x10000u);
    } else if (V == 5) {  // keep bit = bit 15 of a half, count in bits 0..14
      const int b0 = 2 * (i / 16), b1 = b0 + 1;
      tb[i] = ((b0 >= 300 && b0 < 500) ? 0u : 0x8000u) | ((b1 >= 300 && b1 < 500) ? 0u : 0x80000000u);
    } else {
      const int b = i / 8;
      tb[i] = (b >= 300 && b < 500) ? 0u : 0x10001u;
    }
  }
  const size_t off = (size_t)blockIdx.x * (kStage / 16);
  for (int i = threadIdx.x; i < kStage / 16; i += THR) st[i] = in[(off + i) % n16];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t t0 = (uint32_t)__cvta_generic_to_shared(tb);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(st);
  uint32_t base;
  if (V == 0) base = t0 + 4u * (lane & 3);
  else if (V == 3) base = t0 + 4u * (lane & 7);
  else if (V == 1 || V == 4 || V == 5) base = t0 + 4u * (lane & 15);
  else base = t0 + 4u * (lane & 7);
  const uint32_t hs = (V == 2) ? 16u * ((lane >> 3) & 1) : 0u;  // V2: this lane's half
  const uint32_t inc2 = (V == 2) ? (2u << hs) : 0u;
  uint32_t acc = 0;
  for (int r = 0; r < kReps; r++) {
    for (int i = threadIdx.x; i < kStage / 16; i += THR) {
      uint4 q;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                   : "r"(sbase + 16u * (uint32_t)i));
      const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int kk = 0; kk < 4; kk++) {
        if (V == 0 || V == 3) {
          constexpr uint32_t SH = V == 0 ? 4 : 5;
          const uint32_t o0 = atom_ret(base + (min(w4[kk] & 0xFFFFu, 4095u) << SH), 1u << 12);
          const uint32_t o1 = atom_ret(base + (min(w4[kk] >> 16, 4095u) << SH), 1u << 12);
          acc += o0 + o1;  // the fused kernel masks 12 bits of the cell sum
        } else if (V == 4) {
          // hand-scheduled V1: addresses by LOP3 (the table sits at shared offset 0),
          // rotation amounts straight from the packed word, f masked at bits 16..23
          const uint32_t w = min_u16x2(w4[kk], 0x0FFF0FFFu);
          const uint32_t sl = w << 4, sh = w >> 12;  // mod 32: 16*(v_lo&1), 16*(v_hi&1)
          const uint32_t ol = atom_ret(((w << 5) & 0x1FFC0u) | base, rotl(2u, sl));
          const uint32_t oh = atom_ret(((w >> 11) & 0x1FFC0u) | base, rotl(2u, sh));
          const uint32_t tl = ((w & 0xFFFFu) * 4081u + 32768u) & 0xFF0000u;
          const uint32_t th = ((w >> 16) * 4081u + 32768u) & 0xFF0000u;
          acc += (rotr(ol, sl) & 1u) * tl;
          acc += (rotr(oh, sh) & 1u) * th;
          (void)0;
        } else if (V == 5) {
          // V4 with the keep bit at bit 15 of a half: rotate my half down, then one
          // PRMT replicates bit 15 into a 0 / ~0 mask, one LOP3 applies it to f << 16
          const uint32_t w = min_u16x2(w4[kk], 0x0FFF0FFFu);
          const uint32_t sl = w << 4, sh = w >> 12;
          const uint32_t ol = atom_ret(((w << 5) & 0x1FFC0u) | base, rotl(1u, sl));
          const uint32_t oh = atom_ret(((w >> 11) & 0x1FFC0u) | base, rotl(1u, sh));
          const uint32_t tl = (w & 0xFFFFu) * 4081u + 32768u;
          const uint32_t th = (w >> 16) * 4081u + 32768u;
          acc += tl & 0xFF0000u & __byte_perm(rotr(ol, sl), 0u, 0x9999);
          acc += th & 0xFF0000u & __byte_perm(rotr(oh, sh), 0u, 0x9999);
        } else {
          const uint32_t w = min_u16x2(w4[kk], 0x0FFF0FFFu);
          const uint32_t v[2] = {w & 0xFFFFu, w >> 16};
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const uint32_t f = (v[h] * 4081u + 32768u) >> 16;
            if (V == 1) {
              const uint32_t sh = v[h] << 4;  // rotations use sh mod 32 = 16*(v&1)
              const uint32_t old = atom_ret(base + ((v[h] >> 1) << 6), rotl(2u, sh));
              acc += (rotr(old, sh) & 1u) * f;
            } else {
              const uint32_t old = atom_ret(base + (v[h] << 5), inc2);
              acc += ((old >> hs) & 1u) * f;
            }
          }
        }
      }
    }
  }
  atomicAdd(sink, (unsigned long long)(acc & 0xFFFu));
}

template <int V, int THR>
int run(const uint4* d, size_t n16, unsigned long long* sink, int sms, const char* name) {
  const int smem = Cfg<V>::WORDS * 4 + kStage;
  CK(cudaFuncSetAttribute(k<V, THR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<V, THR><<<sms, THR, smem>>>(d, n16, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 5;
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) k<V, THR><<<sms, THR, smem>>>(d, n16, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double vox = (double)sms * kReps * (kStage / 2);
  printf("  %-40s THR=%4d  %.3f ms  %.1f Gvox/s  %.2f vox/clk/SM (1.965 GHz)\n", name, THR, ms, vox / ms / 1e6,
         vox / (ms * 1e-3) / (sms * 1.965e9));
  return 0;
}

int main() {
  const size_t n = (size_t)1 << 28;
  uint16_t* d;
  unsigned long long* sink;
  CK(cudaMalloc(&d, n * 2));
  CK(cudaMalloc(&sink, 8));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int uni = 0; uni < 2; uni++) {
    gen<<<sms * 8, 256>>>(d, n, uni);
    CK(cudaDeviceSynchronize());
    printf("u16 hist + filter o rescale, data %s\n", uni ? "uniform 12-bit" : "config-3-like");
    const uint4* v = reinterpret_cast<const uint4*>(d);
    const size_t m = n / 8;
    if (run<0, 512>(v, m, sink, sms, "V0 lut-in-word, 4 cols (round 1)") ||
        run<0, 1024>(v, m, sink, sms, "V0 lut-in-word, 4 cols (round 1)") ||
        run<3, 512>(v, m, sink, sms, "V3 lut-in-word, 8 cols") ||
        run<1, 512>(v, m, sink, sms, "V1 pair halves by bin parity, 16 cols") ||
        run<1, 1024>(v, m, sink, sms, "V1 pair halves by bin parity, 16 cols") ||
        run<4, 512>(v, m, sink, sms, "V4 = V1 hand-scheduled") ||
        run<4, 1024>(v, m, sink, sms, "V4 = V1 hand-scheduled") ||
        run<5, 512>(v, m, sink, sms, "V5 = V4 + PRMT keep mask") ||
        run<5, 1024>(v, m, sink, sms, "V5 = V4 + PRMT keep mask") ||
        run<2, 512>(v, m, sink, sms, "V2 halves by lane, 8 word cols") ||
        run<2, 1024>(v, m, sink, sms, "V2 halves by lane, 8 word cols"))
      return 1;
  }
  return 0;
}

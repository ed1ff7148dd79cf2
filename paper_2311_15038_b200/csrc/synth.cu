// Seeded synthetic micro-CT volumes for the BASELINE configs (the NOVA scans
// of PAPER.md:374-389 are not available): a Gaussian background, random
// ellipsoidal shells with Gaussian intensity and uniform speckle, generated
// on the device with a counter-based hash RNG keyed by (seed, global voxel
// index), so every z-slab of a volume can be produced independently (sharded
// runs) and the CPU oracle checks the same bytes copied back.
#include "ctp_common.cuh"

namespace ctp {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float u01(uint32_t h) { return ((float)(h >> 8) + 0.5f) * (1.0f / 16777216.0f); }

__device__ __forceinline__ float gauss(uint64_t h) {
  const float a = u01((uint32_t)h), b = u01((uint32_t)(h >> 32));
  return sqrtf(-2.0f * logf(a)) * cospif(2.0f * b);
}

struct SynthArgs {
  void* vol;
  int elem;
  int64_t nz, ny, nx, z_base;
  uint64_t seed;
  float bg_mean, bg_sd, speckle_p, speckle_lambda;
  int vmax;
  const ctp_shell* shells;
  int n_shells;
};

__global__ void synth_kernel(const SynthArgs a) {
  __shared__ ctp_shell sh[64];
  for (int s = threadIdx.x; s < a.n_shells; s += blockDim.x) sh[s] = a.shells[s];
  __syncthreads();
  const int64_t total = a.nz * a.ny * a.nx;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = o % a.nx;
    const int64_t r = o / a.nx;
    const int64_t y = r % a.ny;
    const int64_t z = r / a.ny + a.z_base;
    const uint64_t gi = (uint64_t)(z * a.ny + y) * (uint64_t)a.nx + (uint64_t)x;
    const uint64_t h0 = splitmix64(a.seed * 0x2545F4914F6CDD1Dull ^ gi);
    float v = a.bg_mean + a.bg_sd * gauss(h0);
    const float fx = (float)x + 0.5f, fy = (float)y + 0.5f, fz = (float)z + 0.5f;
    for (int s = 0; s < a.n_shells; s++) {
      const ctp_shell& S = sh[s];
      const float dx = fx - S.cx, dy = fy - S.cy, dz = fz - S.cz;
      const float qo = (dx * dx) / (S.ax * S.ax) + (dy * dy) / (S.ay * S.ay) + (dz * dz) / (S.az * S.az);
      if (qo > 1.0f) continue;
      const float ix = fmaxf(S.ax - S.thickness, 0.5f), iy = fmaxf(S.ay - S.thickness, 0.5f),
                  iz = fmaxf(S.az - S.thickness, 0.5f);
      const float qi = (dx * dx) / (ix * ix) + (dy * dy) / (iy * iy) + (dz * dz) / (iz * iz);
      if (qi < 1.0f) continue;
      v = S.mean + S.sd * gauss(splitmix64(h0 ^ (0xD1B54A32D192ED03ull * (uint64_t)(s + 1))));
    }
    const uint64_t h2 = splitmix64(h0 ^ 0xA0761D6478BD642Full);
    if (u01((uint32_t)h2) < a.speckle_p) {
      if (a.speckle_lambda > 0.0f)  // Poisson-like count: N(lambda, lambda)
        v = a.speckle_lambda + sqrtf(a.speckle_lambda) * gauss(splitmix64(h2));
      else
        v = u01((uint32_t)(h2 >> 32)) * (float)(a.vmax + 1) - 0.5f;
    }
    float c = rintf(v);
    c = fminf(fmaxf(c, 0.0f), (float)a.vmax);
    if (a.elem == 1) reinterpret_cast<uint8_t*>(a.vol)[o] = (uint8_t)c;
    else reinterpret_cast<uint16_t*>(a.vol)[o] = (uint16_t)c;
  }
}

}  // namespace ctp

using namespace ctp;

extern "C" int ctp_synth_volume(void* vol, int32_t elem_bytes, int64_t nz, int64_t ny, int64_t nx, int64_t z_base,
                                int64_t full_nz, uint64_t seed, float bg_mean, float bg_sd, int32_t vmax,
                                const ctp_shell* shells, int32_t n_shells, float speckle_p, float speckle_lambda,
                                void* stream) {
  CTP_REQUIRE(vol != nullptr, CTP_E_INVALID, "ctp_synth_volume: null volume");
  CTP_REQUIRE(elem_bytes == 1 || elem_bytes == 2, CTP_E_UNSUPPORTED, "elem_bytes must be 1 or 2");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1 && z_base >= 0 && z_base + nz <= full_nz, CTP_E_INVALID,
              "ctp_synth_volume: bad slab");
  CTP_REQUIRE(n_shells >= 0 && n_shells <= 64, CTP_E_INVALID, "n_shells %d outside [0, 64]", n_shells);
  CTP_REQUIRE(vmax >= 1 && vmax <= (elem_bytes == 1 ? 255 : 65535), CTP_E_INVALID, "bad vmax %d", vmax);
  cudaStream_t st = as_stream(stream);
  ctp_shell* dsh = nullptr;
  if (n_shells > 0) {
    CTP_CUDA_CALL(cudaMallocAsync(reinterpret_cast<void**>(&dsh), sizeof(ctp_shell) * n_shells, st));
    CTP_CUDA_CALL(cudaMemcpyAsync(dsh, shells, sizeof(ctp_shell) * n_shells, cudaMemcpyHostToDevice, st));
  }
  CTP_REQUIRE(speckle_lambda >= 0.0f, CTP_E_INVALID, "speckle_lambda must be >= 0");
  SynthArgs a{vol, elem_bytes, nz, ny, nx, z_base, seed, bg_mean, bg_sd, speckle_p, speckle_lambda, vmax, dsh, n_shells};
  synth_kernel<<<num_sms() * 8, 256, 0, st>>>(a);
  cudaError_t le = cudaGetLastError();
  if (dsh) cudaFreeAsync(dsh, st);
  CTP_REQUIRE(le == cudaSuccess, CTP_E_CUDA, "synth_kernel: %s", cudaGetErrorString(le));
  ++launch_counter();
  return CTP_OK;
}

// Kernel 5: server-side orthographic ray casting (render.py:125-236) plus the
// MIP and front-to-back alpha-TF extensions, and per-image histograms for
// image_entropy (render.py:248-262).
//
// Geometry (render.py:212-223, 128-140): the camera orbits z at elevation 0;
// pixel (i, j) starts at (rx*wx, ry*wx, wy) and marches t_k = -R + (k+1/2) dt,
// so every image row lives at ONE z -- a ray only ever touches the two slices
// bracketing its row.  Sampling is render.py:68-122 (clamped trilinear,
// outside the half-voxel-padded box -> skipped).
//
// Arithmetic: the fp64 path performs the reference's operations in the
// reference's order with NO contraction (this file is compiled with
// --fmad=false), so surface/additive images are bit-identical to numba's
// fastmath-free output.  Samples that are provably outside the volume are
// skipped via a conservative analytic [k_lo, k_hi] window (+-1 step margin),
// which does not change any result: outside samples contribute nothing in any
// mode (v = -1: not > 0, not >= threshold, not > max, not composited).
#include "ctp_common.cuh"
#include <math.h>

namespace ctp {

struct RenderGeom {
  double big_r, inv_vx, dx, dy, rx, ry, px_size, dt;
};

struct ViewDev {
  RenderGeom g;
  int32_t steps, mode, threshold, channels;
  double gain;
  float tf[4][5];
  float early_stop;
};

template <typename R>
__device__ __forceinline__ R sample_tri(const uint8_t* __restrict__ vox, R ux, R uy, R uz, int nx, int ny, int nz) {
  // render.py:68-111
  const R fx0 = floor(ux), fy0 = floor(uy), fz0 = floor(uz);
  int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
  const R fx = ux - (R)x0, fy = uy - (R)y0, fz = uz - (R)z0;
  int x1 = x0 + 1, y1 = y0 + 1, z1 = z0 + 1;
  x0 = min(max(x0, 0), nx - 1); y0 = min(max(y0, 0), ny - 1); z0 = min(max(z0, 0), nz - 1);
  x1 = min(max(x1, 0), nx - 1); y1 = min(max(y1, 0), ny - 1); z1 = min(max(z1, 0), nz - 1);
  const int64_t sy = nx, sz = (int64_t)nx * ny;
  const uint8_t* p00 = vox + z0 * sz + y0 * sy;
  const uint8_t* p10 = vox + z0 * sz + y1 * sy;
  const uint8_t* p01 = vox + z1 * sz + y0 * sy;
  const uint8_t* p11 = vox + z1 * sz + y1 * sy;
  const R ofx = (R)1 - fx, ofy = (R)1 - fy, ofz = (R)1 - fz;
  const R c00 = (R)__ldg(p00 + x0) * ofx + (R)__ldg(p00 + x1) * fx;
  const R c10 = (R)__ldg(p10 + x0) * ofx + (R)__ldg(p10 + x1) * fx;
  const R c01 = (R)__ldg(p01 + x0) * ofx + (R)__ldg(p01 + x1) * fx;
  const R c11 = (R)__ldg(p11 + x0) * ofx + (R)__ldg(p11 + x1) * fx;
  const R c0 = c00 * ofy + c10 * fy;
  const R c1 = c01 * ofy + c11 * fy;
  return c0 * ofz + c1 * fz;
}

template <typename R>
__device__ __forceinline__ R sample_world(const uint8_t* __restrict__ vox, R px, R py, R pz, R inv_vx, int nx, int ny,
                                          int nz) {
  // render.py:114-122
  const R ux = px * inv_vx + (R)(nx - 1) * (R)0.5;
  const R uy = py * inv_vx + (R)(ny - 1) * (R)0.5;
  const R uz = pz * inv_vx + (R)(nz - 1) * (R)0.5;
  if (ux < (R)-0.5 || ux > (R)nx - (R)0.5 || uy < (R)-0.5 || uy > (R)ny - (R)0.5 || uz < (R)-0.5 ||
      uz > (R)nz - (R)0.5)
    return (R)-1;
  return sample_tri<R>(vox, ux, uy, uz, nx, ny, nz);
}

// Conservative range of k whose sample may lie inside |p_axis| <= half (+ margin).
__device__ __forceinline__ void clip_axis(double o, double d, double half, double big_r, double dt, int steps, int& klo,
                                          int& khi) {
  if (fabs(d) < 1e-9) {
    if (fabs(o) > half * (1.0 + 1e-9) + 1e-9) { klo = steps; khi = -1; }
    return;
  }
  double ta = (-half - o) / d, tb = (half - o) / d;
  if (ta > tb) { const double t = ta; ta = tb; tb = t; }
  const double ka = (ta + big_r) / dt - 0.5, kb = (tb + big_r) / dt - 0.5;
  const double lo = floor(ka) - 1.0, hi = ceil(kb) + 1.0;
  if (lo > klo) klo = lo < (double)steps ? (int)lo : steps;
  if (hi < khi) khi = hi > -1.0 ? (int)hi : -1;
}

// piecewise-linear RGBA transfer function (frozen in oracle/ctp_oracle.py tf_eval)
template <typename R>
__device__ __forceinline__ void tf_eval(const float (*tf)[5], R x, R* c) {
  if (x <= (R)tf[0][0]) {
    for (int q = 0; q < 4; q++) c[q] = (R)tf[0][q + 1];
    return;
  }
  if (x >= (R)tf[3][0]) {
    for (int q = 0; q < 4; q++) c[q] = (R)tf[3][q + 1];
    return;
  }
  int j = (x < (R)tf[1][0]) ? 0 : ((x < (R)tf[2][0]) ? 1 : 2);
  const R x0 = (R)tf[j][0], x1 = (R)tf[j + 1][0];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const R c0 = (R)tf[j][q + 1], c1 = (R)tf[j + 1][q + 1];
    c[q] = c0 + (x - x0) * ((c1 - c0) / (x1 - x0));
  }
}

template <typename R>
__device__ __forceinline__ uint8_t to_u8_unit(R v) {  // floor(min(v, 1) * 255 + 0.5), v >= 0
  if (v > (R)1) v = (R)1;
  if (v < (R)0) v = (R)0;
  return (uint8_t)(int)floor(v * (R)255 + (R)0.5);
}

template <typename R>
__global__ void __launch_bounds__(128) render_kernel(const uint8_t* __restrict__ vox, int nx, int ny, int nz,
                                                     const ViewDev* __restrict__ views, int dim, int row0, int row1,
                                                     uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = row0 + blockIdx.y;
  const int view = blockIdx.z;
  if (i >= dim || j >= row1) return;
  const ViewDev& V = views[view];
  const RenderGeom& G = V.g;
  const int ch = V.channels;
  uint8_t* dst = out + (((int64_t)view * (row1 - row0) + (j - row0)) * dim + i) * ch;

  // render.py:131-137 (fp64, reference order)
  const double wy = G.big_r - ((double)j + 0.5) * G.px_size;
  const double wx = -G.big_r + ((double)i + 0.5) * G.px_size;
  const double ox = G.rx * wx, oy = G.ry * wx, oz = wy;
  const int steps = V.steps;

  // conservative inside window in k
  int klo = 0, khi = steps - 1;
  {
    const double n_max = G.inv_vx;
    clip_axis(ox, G.dx, (double)nx / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
    clip_axis(oy, G.dy, (double)ny / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
    if (fabs(oz) > (double)nz / (2.0 * n_max) * (1.0 + 1e-9) + 1e-9) { klo = steps; khi = -1; }
    if (klo < 0) klo = 0;
    if (khi > steps - 1) khi = steps - 1;
  }

  const R inv_vx = (R)G.inv_vx, dx = (R)G.dx, dy = (R)G.dy;
  const R rox = (R)ox, roy = (R)oy, roz = (R)oz;
  const R big_r = (R)G.big_r, dt = (R)G.dt;

  if (V.mode == CTP_MODE_ADDITIVE) {  // render.py:125-146
    R acc = 0;
    for (int k = klo; k <= khi; k++) {
      const R t = -big_r + ((R)k + (R)0.5) * dt;
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz);
      if (v > (R)0) acc += v;
    }
    R val = (R)V.gain * acc / (R)steps;
    if (val > (R)255) val = (R)255;
    const uint8_t o = (uint8_t)(int)floor(val + (R)0.5);
    for (int c = 0; c < ch; c++) dst[c] = (c == 3) ? 255 : o;
  } else if (V.mode == CTP_MODE_SURFACE) {  // render.py:149-202
    const R thr = (R)V.threshold;
    R shade = 0;
    for (int k = klo; k <= khi; k++) {
      const R t = -big_r + ((R)k + (R)0.5) * dt;
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz);
      if (v >= thr) {
        R t_lo = t - dt, t_hi = t;
        for (int b = 0; b < 4; b++) {
          const R tm = (R)0.5 * (t_lo + t_hi);
          const R vm = sample_world<R>(vox, rox + dx * tm, roy + dy * tm, roz, inv_vx, nx, ny, nz);
          if (vm >= thr) t_hi = tm;
          else t_lo = tm;
        }
        const R th = t_hi;
        const R hx = rox + dx * th, hy = roy + dy * th, hz = roz;
        const R ux = hx * inv_vx + (R)(nx - 1) * (R)0.5;
        const R uy = hy * inv_vx + (R)(ny - 1) * (R)0.5;
        const R uz = hz * inv_vx + (R)(nz - 1) * (R)0.5;
        const R gx = sample_tri<R>(vox, ux + (R)1, uy, uz, nx, ny, nz) - sample_tri<R>(vox, ux - (R)1, uy, uz, nx, ny, nz);
        const R gy = sample_tri<R>(vox, ux, uy + (R)1, uz, nx, ny, nz) - sample_tri<R>(vox, ux, uy - (R)1, uz, nx, ny, nz);
        const R gz = sample_tri<R>(vox, ux, uy, uz + (R)1, nx, ny, nz) - sample_tri<R>(vox, ux, uy, uz - (R)1, nx, ny, nz);
        const R gn = sqrt(gx * gx + gy * gy + gz * gz);
        if (gn < (R)1e-12) {
          shade = 1;
        } else {
          const R lam = (gx * dx + gy * dy) / gn;
          shade = lam > (R)0 ? lam : (R)0;
        }
        break;
      }
    }
    const uint8_t o = (uint8_t)(int)floor((R)255 * shade + (R)0.5);
    for (int c = 0; c < ch; c++) dst[c] = (c == 3) ? 255 : o;
  } else if (V.mode == CTP_MODE_MIP) {
    R m = 0;
    for (int k = klo; k <= khi; k++) {
      const R t = -big_r + ((R)k + (R)0.5) * dt;
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz);
      m = v > m ? v : m;
    }
    if (m > (R)255) m = (R)255;
    const uint8_t o = (uint8_t)(int)floor(m + (R)0.5);
    for (int c = 0; c < ch; c++) dst[c] = (c == 3) ? 255 : o;
  } else {  // CTP_MODE_ALPHA: front-to-back, premultiplied
    R C[3] = {0, 0, 0}, A = 0;
    const R stop = (R)V.early_stop;
    for (int k = klo; k <= khi; k++) {
      const R t = -big_r + ((R)k + (R)0.5) * dt;
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz);
      if (v < (R)0) continue;
      R c[4];
      tf_eval<R>(V.tf, v, c);
      const R w = ((R)1 - A) * c[3];
      C[0] += w * c[0];
      C[1] += w * c[1];
      C[2] += w * c[2];
      A += w;
      if (A >= stop) break;
    }
    if (ch == 4) {
      dst[0] = to_u8_unit<R>(C[0]);
      dst[1] = to_u8_unit<R>(C[1]);
      dst[2] = to_u8_unit<R>(C[2]);
      dst[3] = to_u8_unit<R>(A);
    } else {
      dst[0] = to_u8_unit<R>(A);
    }
  }
}

__global__ void image_hist_kernel(const uint8_t* __restrict__ imgs, int64_t pixels, unsigned long long* __restrict__ hist) {
  __shared__ uint32_t hs[256];
  const int img = blockIdx.y;
  for (int b = threadIdx.x; b < 256; b += blockDim.x) hs[b] = 0;
  __syncthreads();
  const uint8_t* p = imgs + (int64_t)img * pixels;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < pixels; q += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hs[p[q]], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (hs[b]) atomicAdd(hist + (int64_t)img * 256 + b, (unsigned long long)hs[b]);
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_render_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, const ctp_view* views, int32_t n_views,
                  int64_t row0, int64_t row1, uint8_t* out, void* stream) {
  CTP_REQUIRE(vol && views && out, CTP_E_INVALID, "ctp_render_u8: null pointer");
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1 && nx < (1LL << 31) && ny < (1LL << 31) && nz < (1LL << 31),
              CTP_E_INVALID, "ctp_render_u8: bad shape");
  CTP_REQUIRE(n_views >= 1 && n_views <= 65535, CTP_E_INVALID, "n_views %d outside [1, 65535]", n_views);
  const ctp_view& v0 = views[0];
  const int dim = v0.image_dim;
  // render.py:56-65 (ViewParams validation)
  CTP_REQUIRE(dim >= 16, CTP_E_INVALID, "image_dim %d below minimum 16", dim);
  CTP_REQUIRE(0 <= row0 && row0 < row1 && row1 <= dim, CTP_E_INVALID, "rows [%lld, %lld) outside [0, %d]",
              (long long)row0, (long long)row1, dim);
  ViewDev hv[64];
  CTP_REQUIRE(n_views <= 64, CTP_E_INVALID, "at most 64 views per call (got %d)", n_views);
  const int64_t n_max = nx > ny ? (nx > nz ? nx : nz) : (ny > nz ? ny : nz);
  for (int q = 0; q < n_views; q++) {
    const ctp_view& v = views[q];
    CTP_REQUIRE(v.image_dim == dim && v.mode == v0.mode && v.channels == v0.channels && v.fp32 == v0.fp32,
                CTP_E_INVALID, "views must share image_dim/mode/channels/fp32");
    CTP_REQUIRE(v.steps >= 32, CTP_E_INVALID, "steps %d below minimum 32", v.steps);
    CTP_REQUIRE(v.mode >= 0 && v.mode <= 3, CTP_E_INVALID, "mode %d unknown", v.mode);
    CTP_REQUIRE(0 <= v.threshold && v.threshold <= 255, CTP_E_INVALID, "threshold %d outside [0, 255]", v.threshold);
    CTP_REQUIRE(v.gain > 0, CTP_E_INVALID, "gain must be positive");
    CTP_REQUIRE(v.channels == 1 || v.channels == 4, CTP_E_INVALID, "channels must be 1 or 4");
    // render.py:212-223
    const double hx = (double)nx / (2.0 * (double)n_max), hy = (double)ny / (2.0 * (double)n_max),
                 hz = (double)nz / (2.0 * (double)n_max);
    RenderGeom& G = hv[q].g;
    G.big_r = sqrt(hx * hx + hy * hy + hz * hz);
    G.inv_vx = (double)n_max;
    const double theta = v.azimuth_deg * (M_PI / 180.0);  // math.radians
    G.dx = -cos(theta);
    G.dy = -sin(theta);
    G.rx = -sin(theta);
    G.ry = cos(theta);
    G.px_size = 2.0 * G.big_r / dim;
    G.dt = 2.0 * G.big_r / v.steps;
    hv[q].steps = v.steps;
    hv[q].mode = v.mode;
    hv[q].threshold = v.threshold;
    hv[q].channels = v.channels;
    hv[q].gain = v.gain;
    for (int a = 0; a < 4; a++)
      for (int b = 0; b < 5; b++) hv[q].tf[a][b] = v.tf[a][b];
    hv[q].early_stop = v.early_stop;
  }
  cudaStream_t st = as_stream(stream);
  ViewDev* dv = nullptr;
  CTP_CUDA_CALL(cudaMallocAsync(reinterpret_cast<void**>(&dv), sizeof(ViewDev) * n_views, st));
  CTP_CUDA_CALL(cudaMemcpyAsync(dv, hv, sizeof(ViewDev) * n_views, cudaMemcpyHostToDevice, st));
  dim3 grid((dim + 127) / 128, (unsigned)(row1 - row0), (unsigned)n_views);
  if (v0.fp32)
    render_kernel<float><<<grid, 128, 0, st>>>(vol, (int)nx, (int)ny, (int)nz, dv, dim, (int)row0, (int)row1, out);
  else
    render_kernel<double><<<grid, 128, 0, st>>>(vol, (int)nx, (int)ny, (int)nz, dv, dim, (int)row0, (int)row1, out);
  cudaError_t le = cudaGetLastError();
  cudaFreeAsync(dv, st);
  CTP_REQUIRE(le == cudaSuccess, CTP_E_CUDA, "render_kernel: %s", cudaGetErrorString(le));
  ++launch_counter();
  return CTP_OK;
}

int ctp_image_hist_u8(const uint8_t* imgs, int32_t n_images, int64_t pixels, uint64_t* hist, void* stream) {
  CTP_REQUIRE(imgs && hist, CTP_E_INVALID, "ctp_image_hist_u8: null pointer");
  CTP_REQUIRE(n_images >= 1 && n_images <= 65535 && pixels >= 1, CTP_E_INVALID, "bad image batch");
  int bx = (int)((pixels + 256 * 16 - 1) / (256 * 16));
  if (bx > 64) bx = 64;
  dim3 grid(bx, n_images);
  image_hist_kernel<<<grid, 256, 0, as_stream(stream)>>>(imgs, pixels, reinterpret_cast<unsigned long long*>(hist));
  CTP_CUDA_CHECK_LAUNCH("image_hist_kernel");
  return CTP_OK;
}

}  // extern "C"

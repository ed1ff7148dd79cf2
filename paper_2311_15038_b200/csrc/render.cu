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
#include <stdlib.h>

#include <memory>
#include <mutex>

namespace ctp {

struct RenderGeom {
  double big_r, inv_vx, dx, dy, rx, ry, px_size, dt;
};

struct ViewDev {
  RenderGeom g;
  int32_t steps, mode, threshold, channels;
  double gain;
  float tf[4][5];
  double slope[3][4];  // (c_{j+1} - c_j) / (x_{j+1} - x_j) per segment and channel
  float early_stop;
  float skip_lvl;  // alpha: 8.8 level at or below which the transfer function's alpha is 0 (-1: none)
};

constexpr int kMaxViews = 64;
struct ViewBatch {  // passed by value (kernel parameter space), <= 64 views per launch
  ViewDev v[kMaxViews];
  int64_t vstride;  // bytes between consecutive views' first rows in `out`
  int32_t peer;     // `out` is a peer GPU's memory: system-scope fence after the stores
  // fp32 MIP on the row planes: grid.z walks the PRIMARY views prim[0..]; mirror[z] >= 0 names the
  // view at azimuth + 180 degrees, whose image is the primary's mirrored left-right (see
  // pair_opposite_views) and is stored by the same thread.  Identity / -1 everywhere else.
  int8_t prim[kMaxViews];
  int8_t mirror[kMaxViews];
};

// 2x2 footprint of one slice of a layered u8 texture (clamp addressing): the
// exact voxel values at (x0, y0) .w, (x0+1, y0) .z, (x0, y0+1) .x, (x0+1, y0+1) .y
__device__ __forceinline__ uint4 tld4_a2d(cudaTextureObject_t tex, int layer, float x, float y) {
  uint4 r;
  asm volatile("tld4.r.a2d.v4.u32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %7}];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(tex), "r"(layer), "f"(x), "f"(y));
  return r;
}

// tex != 0: the volume slices [zb, ...) as a layered u8 texture; the eight voxel
// VALUES then come from two gathers instead of eight byte loads (the texture's
// clamp addressing is render.py's index clamping), and the arithmetic below is
// unchanged -- bit-identical results.
template <typename R>
__device__ __forceinline__ R sample_tri(const uint8_t* __restrict__ vox, R ux, R uy, R uz, int nx, int ny, int nz,
                                        int zb, cudaTextureObject_t tex = 0) {
  // render.py:68-111
  const R fx0 = floor(ux), fy0 = floor(uy), fz0 = floor(uz);
  int x0 = (int)fx0, y0 = (int)fy0, z0 = (int)fz0;
  const R fx = ux - (R)x0, fy = uy - (R)y0, fz = uz - (R)z0;
  if (tex) {
    const int za = min(max(z0, 0), nz - 1) - zb, zc = min(max(z0 + 1, 0), nz - 1) - zb;
    const float gxc = (float)x0 + 1.0f, gyc = (float)y0 + 1.0f;
    const uint4 g0 = tld4_a2d(tex, za, gxc, gyc), g1 = tld4_a2d(tex, zc, gxc, gyc);
    const R ofx = (R)1 - fx, ofy = (R)1 - fy, ofz = (R)1 - fz;
    const R c00 = (R)g0.w * ofx + (R)g0.z * fx;
    const R c10 = (R)g0.x * ofx + (R)g0.y * fx;
    const R c01 = (R)g1.w * ofx + (R)g1.z * fx;
    const R c11 = (R)g1.x * ofx + (R)g1.y * fx;
    const R c0 = c00 * ofy + c10 * fy;
    const R c1 = c01 * ofy + c11 * fy;
    return c0 * ofz + c1 * fz;
  }
  int x1 = x0 + 1, y1 = y0 + 1, z1 = z0 + 1;
  x0 = min(max(x0, 0), nx - 1); y0 = min(max(y0, 0), ny - 1); z0 = min(max(z0, 0), nz - 1);
  x1 = min(max(x1, 0), nx - 1); y1 = min(max(y1, 0), ny - 1); z1 = min(max(z1, 0), nz - 1);
  // vox holds slices [zb, ...) (a z-slab with its halo; zb = 0 for a whole volume)
  const int64_t sy = nx, sz = (int64_t)nx * ny;
  const uint8_t* p00 = vox + (z0 - zb) * sz + y0 * sy;
  const uint8_t* p10 = vox + (z0 - zb) * sz + y1 * sy;
  const uint8_t* p01 = vox + (z1 - zb) * sz + y0 * sy;
  const uint8_t* p11 = vox + (z1 - zb) * sz + y1 * sy;
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
                                          int nz, int zb, cudaTextureObject_t tex = 0) {
  // render.py:114-122
  const R ux = px * inv_vx + (R)(nx - 1) * (R)0.5;
  const R uy = py * inv_vx + (R)(ny - 1) * (R)0.5;
  const R uz = pz * inv_vx + (R)(nz - 1) * (R)0.5;
  if (ux < (R)-0.5 || ux > (R)nx - (R)0.5 || uy < (R)-0.5 || uy > (R)ny - (R)0.5 || uz < (R)-0.5 ||
      uz > (R)nz - (R)0.5)
    return (R)-1;
  return sample_tri<R>(vox, ux, uy, uz, nx, ny, nz, zb, tex);
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
__device__ __forceinline__ void tf_eval(const float (*tf)[5], const double (*slope)[4], R x, R* c) {
  if (x <= (R)tf[0][0]) {
    for (int q = 0; q < 4; q++) c[q] = (R)tf[0][q + 1];
    return;
  }
  if (x >= (R)tf[3][0]) {
    for (int q = 0; q < 4; q++) c[q] = (R)tf[3][q + 1];
    return;
  }
  int j = (x < (R)tf[1][0]) ? 0 : ((x < (R)tf[2][0]) ? 1 : 2);
  const R x0 = (R)tf[j][0];
#pragma unroll
  for (int q = 0; q < 4; q++) c[q] = (R)tf[j][q + 1] + (x - x0) * (R)slope[j][q];
}

template <typename R>
__device__ __forceinline__ uint8_t to_u8_unit(R v) {  // floor(min(v, 1) * 255 + 0.5), v >= 0
  if (v > (R)1) v = (R)1;
  if (v < (R)0) v = (R)0;
  return (uint8_t)(int)floor(v * (R)255 + (R)0.5);
}

#ifndef CTP_RENDER_MINB
#define CTP_RENDER_MINB 10  // 10 CTAs of 128 per SM (<= 48 registers): the fp64 walk is latency-bound at 64 registers
#endif
template <typename R>
__global__ void __launch_bounds__(128, CTP_RENDER_MINB) render_kernel(const uint8_t* __restrict__ vox, int zb, int nx, int ny,
                                                     int nz, const __grid_constant__ ViewBatch views, int dim,
                                                     int row0, int row1, uint8_t* __restrict__ out,
                                                     cudaTextureObject_t tex) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = row0 + blockIdx.y;
  const int view = blockIdx.z;
  if (i >= dim || j >= row1) return;
  const ViewDev& V = views.v[view];
  const RenderGeom& G = V.g;
  const int ch = V.channels;
  uint8_t* dst = out + (int64_t)view * views.vstride + ((int64_t)(j - row0) * dim + i) * ch;

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

  // kUnroll samples are computed independently (their loads in flight together)
  // and then consumed strictly in k order: every accumulation, comparison and
  // break happens in the reference's sequence, so results are unchanged.
  auto sample_at = [&](int k) -> R {
    const R t = -big_r + ((R)k + (R)0.5) * dt;
    return sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz, zb, tex);
  };
  constexpr int kUnroll = 4;
  if (V.mode == CTP_MODE_ADDITIVE) {  // render.py:125-146
    R acc = 0;
    int k = klo;
    for (; k + kUnroll - 1 <= khi; k += kUnroll) {
      R v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) v[u] = sample_at(k + u);
#pragma unroll
      for (int u = 0; u < kUnroll; u++)
        if (v[u] > (R)0) acc += v[u];
    }
    for (; k <= khi; k++) {
      const R v = sample_at(k);
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
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz, zb, tex);
      if (v >= thr) {
        R t_lo = t - dt, t_hi = t;
        for (int b = 0; b < 4; b++) {
          const R tm = (R)0.5 * (t_lo + t_hi);
          const R vm = sample_world<R>(vox, rox + dx * tm, roy + dy * tm, roz, inv_vx, nx, ny, nz, zb, tex);
          if (vm >= thr) t_hi = tm;
          else t_lo = tm;
        }
        const R th = t_hi;
        const R hx = rox + dx * th, hy = roy + dy * th, hz = roz;
        const R ux = hx * inv_vx + (R)(nx - 1) * (R)0.5;
        const R uy = hy * inv_vx + (R)(ny - 1) * (R)0.5;
        const R uz = hz * inv_vx + (R)(nz - 1) * (R)0.5;
        const R gx = sample_tri<R>(vox, ux + (R)1, uy, uz, nx, ny, nz, zb, tex) - sample_tri<R>(vox, ux - (R)1, uy, uz, nx, ny, nz, zb, tex);
        const R gy = sample_tri<R>(vox, ux, uy + (R)1, uz, nx, ny, nz, zb, tex) - sample_tri<R>(vox, ux, uy - (R)1, uz, nx, ny, nz, zb, tex);
        const R gz = sample_tri<R>(vox, ux, uy, uz + (R)1, nx, ny, nz, zb, tex) - sample_tri<R>(vox, ux, uy, uz - (R)1, nx, ny, nz, zb, tex);
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
    int k = klo;
    for (; k + kUnroll - 1 <= khi; k += kUnroll) {
      R v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) v[u] = sample_at(k + u);
#pragma unroll
      for (int u = 0; u < kUnroll; u++) m = v[u] > m ? v[u] : m;
    }
    for (; k <= khi; k++) {
      const R v = sample_at(k);
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
      const R v = sample_world<R>(vox, rox + dx * t, roy + dy * t, roz, inv_vx, nx, ny, nz, zb, tex);
      if (v < (R)0) continue;
      R c[4];
      tf_eval<R>(V.tf, V.slope, v, c);
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
  if (views.peer) __threadfence_system();  // stores into a peer's images: visible before the completing collective
}


// ---------------------------------------------------------------------------
// fp32 fast path for the extension modes (MIP, alpha): the volume is bound to a
// layered 2D texture (one layer per z-slice, block-linear, clamp addressing)
// and every trilinear sample is TWO gathers (tld4: the 2x2 footprint of slice
// z0 and of slice z1) instead of eight byte loads.  The geometry, sample
// positions, clamping and skip rule are those of render.py:68-140; the
// interpolation weights are computed in fp32 (tolerance 1/255).

template <int MODE>
__global__ void __launch_bounds__(128) render_tex_kernel(cudaTextureObject_t tex, int zb, int nx, int ny, int nz,
                                                         const __grid_constant__ ViewBatch views, int dim, int row0,
                                                         int row1, uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = row0 + blockIdx.y;
  const int view = views.prim[blockIdx.z];
  if (i >= dim || j >= row1) return;
  const ViewDev& V = views.v[view];
  const RenderGeom& G = V.g;
  const int ch = V.channels;
  uint8_t* dst = out + (int64_t)view * views.vstride + ((int64_t)(j - row0) * dim + i) * ch;
  const double wy = G.big_r - ((double)j + 0.5) * G.px_size;
  const double wx = -G.big_r + ((double)i + 0.5) * G.px_size;
  const double ox = G.rx * wx, oy = G.ry * wx, oz = wy;
  const int steps = V.steps;
  int klo = 0, khi = steps - 1;
  const double n_max = G.inv_vx;
  clip_axis(ox, G.dx, (double)nx / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
  clip_axis(oy, G.dy, (double)ny / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
  const double uzd = oz * G.inv_vx + (double)(nz - 1) * 0.5;
  if (uzd < -0.5 || uzd > (double)nz - 0.5) { klo = steps; khi = -1; }
  if (klo < 0) klo = 0;
  if (khi > steps - 1) khi = steps - 1;
  // per-row constants: the row's two slices and z weight (render.py:72-79, 105-111)
  const int zf = (int)floor(uzd);
  const float fz = (float)(uzd - (double)zf);
  const int l0 = min(max(zf, 0), nz - 1) - zb, l1 = min(max(zf + 1, 0), nz - 1) - zb;  // texture layers = slab slices
  // u(k) = a + k * b exactly as an FMA per step (no drift): u = (o + d*t)*n + (n-1)/2, t = -R + (k+1/2)dt
  const double bx = G.dx * G.dt * G.inv_vx, by = G.dy * G.dt * G.inv_vx;
  const double ax = (ox + G.dx * (-G.big_r + 0.5 * G.dt)) * G.inv_vx + (double)(nx - 1) * 0.5;
  const double ay = (oy + G.dy * (-G.big_r + 0.5 * G.dt)) * G.inv_vx + (double)(ny - 1) * 0.5;
  const float fax = (float)ax, fbx = (float)bx, fay = (float)ay, fby = (float)by;
  const float xlo = -0.5f, xhi = (float)nx - 0.5f, ylo = -0.5f, yhi = (float)ny - 0.5f;
  float m = 0.f;
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
  const float stop = V.early_stop;
  for (int k = klo; k <= khi; k++) {
    const float ux = fmaf((float)k, fbx, fax), uy = fmaf((float)k, fby, fay);
    if (ux < xlo || ux > xhi || uy < ylo || uy > yhi) continue;
    const float x0 = floorf(ux), y0 = floorf(uy);
    const float fx = ux - x0, fy = uy - y0;
    // tld4 footprint at (x0 + 1, y0 + 1): .w = (x0, y0), .z = (x0+1, y0), .x = (x0, y0+1), .y = (x0+1, y0+1)
    const uint4 g0 = tld4_a2d(tex, l0, x0 + 1.0f, y0 + 1.0f);
    const uint4 g1 = tld4_a2d(tex, l1, x0 + 1.0f, y0 + 1.0f);
    const float a00 = fmaf(fx, (float)g0.z - (float)g0.w, (float)g0.w);
    const float a10 = fmaf(fx, (float)g0.y - (float)g0.x, (float)g0.x);
    const float b00 = fmaf(fx, (float)g1.z - (float)g1.w, (float)g1.w);
    const float b10 = fmaf(fx, (float)g1.y - (float)g1.x, (float)g1.x);
    const float c0 = fmaf(fy, a10 - a00, a00), c1 = fmaf(fy, b10 - b00, b00);
    const float v = fmaf(fz, c1 - c0, c0);
    if (MODE == CTP_MODE_MIP) {
      m = fmaxf(m, v);
    } else {
      float c[4];
      tf_eval<float>(V.tf, V.slope, v, c);
      const float w = (1.f - A) * c[3];
      C0 = fmaf(w, c[0], C0);
      C1 = fmaf(w, c[1], C1);
      C2 = fmaf(w, c[2], C2);
      A += w;
      if (A >= stop) break;
    }
  }
  if (MODE == CTP_MODE_MIP) {
    const uint8_t o = (uint8_t)(int)floorf(fminf(m, 255.f) + 0.5f);
    if (ch == 4) *reinterpret_cast<uchar4*>(dst) = make_uchar4(o, o, o, 255);
    else dst[0] = o;
    const int mv = views.mirror[blockIdx.z];
    if (mv >= 0) {  // the opposite azimuth sees this ray's sample set from the other end: pixel dim-1-i
      uint8_t* d2 = out + (int64_t)mv * views.vstride + ((int64_t)(j - row0) * dim + (dim - 1 - i)) * ch;
      if (ch == 4) *reinterpret_cast<uchar4*>(d2) = make_uchar4(o, o, o, 255);
      else d2[0] = o;
    }
  } else {
    if (ch == 4) *reinterpret_cast<uchar4*>(dst) = make_uchar4(to_u8_unit<float>(C0), to_u8_unit<float>(C1),
                                                              to_u8_unit<float>(C2), to_u8_unit<float>(A));
    else dst[0] = to_u8_unit<float>(A);
  }
  if (views.peer) __threadfence_system();
}

// Row planes: every image row j of the turntable lives at one z (render.py:140),
// so its two slices can be blended ONCE per volume into a plane
//   P_j(x, y) = (1 - fz_j) V[z0_j](x, y) + fz_j V[z0_j + 1](x, y)
// stored as 8.8 fixed point (u16, 2 B/voxel/row) and shared by all azimuths;
// a trilinear sample is then ONE gather (tld4) + a bilinear blend.
// Mathematically the reference's trilinear (z applied first instead of last
// only changes rounding, tolerance 1/255).  Measured and not kept: fp32 planes
// (4 B/voxel, slower), the texture unit's own bilinear filter (1-3% faster,
// 8-bit weights), empty-space skipping for MIP (a noisy background rarely
// drops below the running max: the lookups cost more than they save), reusing
// the previous gather while (x0, y0) is unchanged (~half the samples; the
// predicated gathers made it 5-10% slower).
//
// Empty-space skipping (alpha on the row planes): the planes are cut into
// kSkip x kSkip texel blocks and each block stores the max 8.8 value over its
// texels DILATED by one texel on the high side -- every bilinear footprint whose
// lower-left texel lies in the block is covered -- so a run of samples inside a
// block whose bound is <= the transfer function's zero-alpha level contributes
// w = (1 - A) * 0 exactly and is stepped over analytically.
constexpr int kSkip = 8;
constexpr int kBlendThreads = 256, kBlendVec = 4, kBlendCols = kBlendThreads * kBlendVec;

// one CTA = kBlendCols columns x one kSkip-row band of one row plane: blends the
// two slices into the plane (8.8 fixed point, |error| <= 1/512 of a gray level)
// and writes the band's block maxima.
__global__ void __launch_bounds__(kBlendThreads) blend_rows_kernel(const uint8_t* __restrict__ vol, int zb, int nx,
                                                                   int ny, int nz, double big_r, double px_size,
                                                                   double inv_vx, int row0, cudaSurfaceObject_t surf,
                                                                   uint16_t* __restrict__ bmax, int nbx, int nby) {
  __shared__ uint16_t colmax[kBlendCols + 1];
  const int x = blockIdx.x * kBlendCols + threadIdx.x * kBlendVec;
  const int by = blockIdx.y;
  const int layer = blockIdx.z;
  const int j = row0 + layer;
  const double wy = big_r - ((double)j + 0.5) * px_size;
  const double uz = wy * inv_vx + (double)(nz - 1) * 0.5;
  const bool inside = !(uz < -0.5 || uz > (double)nz - 0.5);
  int z0 = 0, z1 = 0;
  float fz = 0.f;
  if (inside) {
    const int zf = (int)floor(uz);
    fz = (float)(uz - (double)zf);
    z0 = min(max(zf, 0), nz - 1);
    z1 = min(max(zf + 1, 0), nz - 1);
  }
  const uint8_t* s0 = vol + (int64_t)(inside ? z0 - zb : 0) * ny * nx;  // vol holds slices [zb, ...)
  const uint8_t* s1 = vol + (int64_t)(inside ? z1 - zb : 0) * ny * nx;
  const int ya = by * kSkip, yw = min(ya + kSkip, ny), yd = min(ya + kSkip, ny - 1);
  auto blend = [&](uint32_t a, uint32_t b) -> uint32_t {
    return __float2uint_rn(fmaf(fz, (float)b - (float)a, (float)a) * 256.0f);
  };
  auto texel = [&](int xx, int yy) -> uint32_t {
    if (!inside) return 0u;
    return blend(__ldg(s0 + (int64_t)yy * nx + xx), __ldg(s1 + (int64_t)yy * nx + xx));
  };
  // 4 consecutive texels per thread: one 4-byte load per slice, one 8-byte surface store
  const bool vec = ((nx & 3) == 0) && (x + kBlendVec <= nx);
  uint32_t cm[kBlendVec] = {0, 0, 0, 0};
  if (x < nx) {
    for (int y = ya; y <= yd; y++) {
      uint32_t t[kBlendVec] = {0, 0, 0, 0};
      if (vec) {
        if (inside) {
          const uint32_t a4 = __ldg(reinterpret_cast<const uint32_t*>(s0 + (int64_t)y * nx + x));
          const uint32_t b4 = __ldg(reinterpret_cast<const uint32_t*>(s1 + (int64_t)y * nx + x));
#pragma unroll
          for (int q = 0; q < kBlendVec; q++) t[q] = blend((a4 >> (8 * q)) & 0xFFu, (b4 >> (8 * q)) & 0xFFu);
        }
        if (y < yw)
          surf2DLayeredwrite(make_ushort4((unsigned short)t[0], (unsigned short)t[1], (unsigned short)t[2],
                                          (unsigned short)t[3]),
                             surf, x * (int)sizeof(unsigned short), y, layer);
      } else {
#pragma unroll
        for (int q = 0; q < kBlendVec; q++)
          if (x + q < nx) {
            t[q] = texel(x + q, y);
            if (y < yw) surf2DLayeredwrite((unsigned short)t[q], surf, (x + q) * (int)sizeof(unsigned short), y, layer);
          }
      }
#pragma unroll
      for (int q = 0; q < kBlendVec; q++) cm[q] = max(cm[q], t[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < kBlendVec; q++) colmax[threadIdx.x * kBlendVec + q] = (uint16_t)cm[q];
  if (threadIdx.x == 0) {  // the dilation column of the CTA's last block
    const int xe = blockIdx.x * kBlendCols + kBlendCols;
    uint32_t ce = 0;
    if (xe < nx)
      for (int y = ya; y <= yd; y++) ce = max(ce, texel(xe, y));
    colmax[kBlendCols] = (uint16_t)ce;
  }
  __syncthreads();
  const int bx = blockIdx.x * (kBlendCols / kSkip) + threadIdx.x;
  if (threadIdx.x < kBlendCols / kSkip && bx < nbx) {
    uint32_t b = 0;
#pragma unroll
    for (int q = 0; q <= kSkip; q++) b = max(b, (uint32_t)colmax[threadIdx.x * kSkip + q]);
    bmax[((int64_t)layer * nby + by) * nbx + bx] = (uint16_t)b;
  }
}

// first step index at which floor(u(k)) leaves [lo, lo + kSkip) along one axis
// (u(k) = a + k b); conservative by construction of the caller (it re-checks one
// step early).  Returns INT_MAX when the axis never leaves (b == 0 or open edge).
__device__ __forceinline__ int block_exit(float a, float b, int blk, int nblk) {
  float t;
  if (b > 0.f) {
    if (blk >= nblk - 1) return INT_MAX;
    t = ((float)((blk + 1) * kSkip) - a) / b;
  } else if (b < 0.f) {
    if (blk <= 0) return INT_MAX;
    t = ((float)(blk * kSkip) - a) / b;
  } else {
    return INT_MAX;
  }
  return t < 1.0e9f ? (int)ceilf(t) : INT_MAX;
}

template <int MODE>
__global__ void __launch_bounds__(128) render_rows_kernel(cudaTextureObject_t tex, int nx, int ny, int nz,
                                                          const __grid_constant__ ViewBatch views, int dim, int row0,
                                                          int row1, uint8_t* __restrict__ out,
                                                          const uint16_t* __restrict__ bmax, int nbx, int nby, int skip) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = row0 + blockIdx.y;
  const int view = views.prim[blockIdx.z];
  if (i >= dim || j >= row1) return;
  const ViewDev& V = views.v[view];
  const RenderGeom& G = V.g;
  const int ch = V.channels;
  uint8_t* dst = out + (int64_t)view * views.vstride + ((int64_t)(j - row0) * dim + i) * ch;
  const double wy = G.big_r - ((double)j + 0.5) * G.px_size;
  const double wx = -G.big_r + ((double)i + 0.5) * G.px_size;
  const double ox = G.rx * wx, oy = G.ry * wx, oz = wy;
  const int steps = V.steps;
  int klo = 0, khi = steps - 1;
  const double n_max = G.inv_vx;
  clip_axis(ox, G.dx, (double)nx / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
  clip_axis(oy, G.dy, (double)ny / (2.0 * n_max), G.big_r, G.dt, steps, klo, khi);
  const double uzd = oz * G.inv_vx + (double)(nz - 1) * 0.5;
  if (uzd < -0.5 || uzd > (double)nz - 0.5) { klo = steps; khi = -1; }
  if (klo < 0) klo = 0;
  if (khi > steps - 1) khi = steps - 1;
  const int layer = j - row0;
  const double bx = G.dx * G.dt * G.inv_vx, by = G.dy * G.dt * G.inv_vx;
  const double ax = (ox + G.dx * (-G.big_r + 0.5 * G.dt)) * G.inv_vx + (double)(nx - 1) * 0.5;
  const double ay = (oy + G.dy * (-G.big_r + 0.5 * G.dt)) * G.inv_vx + (double)(ny - 1) * 0.5;
  const float fax = (float)ax, fbx = (float)bx, fay = (float)ay, fby = (float)by;
  const float xlo = -0.5f, xhi = (float)nx - 0.5f, ylo = -0.5f, yhi = (float)ny - 0.5f;
  float m = 0.f;  // MIP: running max in 8.8 units (the final * 1/256 is exact)
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
  if (MODE == CTP_MODE_MIP) {
    // MIP: every sample (a noisy background leaves no block below the running
    // max often enough to pay for the lookups -- measured)
#pragma unroll 4
    for (int k = klo; k <= khi; k++) {
      const float ux = fmaf((float)k, fbx, fax), uy = fmaf((float)k, fby, fay);
      if (ux < xlo || ux > xhi || uy < ylo || uy > yhi) continue;
      const float x0 = floorf(ux), y0 = floorf(uy);
      const float fx = ux - x0, fy = uy - y0;
      const uint4 gi = tld4_a2d(tex, layer, x0 + 1.0f, y0 + 1.0f);  // .w (x0,y0) .z (x1,y0) .x (x0,y1) .y (x1,y1)
      const float4 g = make_float4((float)gi.x, (float)gi.y, (float)gi.z, (float)gi.w);
      const float a0 = fmaf(fx, g.z - g.w, g.w), a1 = fmaf(fx, g.y - g.x, g.x);
      m = fmaxf(m, fmaf(fy, a1 - a0, a0));
    }
  } else {
    // alpha: samples in blocks whose bound is at or below the transfer function's
    // zero-alpha level contribute w = (1 - A) * 0 exactly and are stepped over
    const uint16_t* bm = bmax + (int64_t)layer * nby * nbx;
    const float stop = V.early_stop;
    const float zero_lvl = skip ? V.skip_lvl : -1.f;
    int cur = -1;  // block of the last bound lookup
    float bound = 0.f;
    int k = klo;
    while (k <= khi) {
      const float ux = fmaf((float)k, fbx, fax), uy = fmaf((float)k, fby, fay);
      if (ux < xlo || ux > xhi || uy < ylo || uy > yhi) { k++; continue; }
      const float x0 = floorf(ux), y0 = floorf(uy);
      const int bxi = min(max((int)x0, 0) / kSkip, nbx - 1), byi = min(max((int)y0, 0) / kSkip, nby - 1);
      const int blk = byi * nbx + bxi;
      if (blk != cur) { cur = blk; bound = (float)__ldg(bm + blk); }
      if (bound <= zero_lvl) {
        // resume one step before the ray leaves the block (the re-check absorbs fp rounding)
        const int kn = min(block_exit(fax, fbx, bxi, nbx), block_exit(fay, fby, byi, nby));
        k = (kn == INT_MAX) ? khi + 1 : max(k + 1, kn - 1);
        continue;
      }
      const float fx = ux - x0, fy = uy - y0;
      const uint4 gi = tld4_a2d(tex, layer, x0 + 1.0f, y0 + 1.0f);
      const float4 g = make_float4((float)gi.x, (float)gi.y, (float)gi.z, (float)gi.w);
      const float a0 = fmaf(fx, g.z - g.w, g.w), a1 = fmaf(fx, g.y - g.x, g.x);
      float c[4];
      tf_eval<float>(V.tf, V.slope, fmaf(fy, a1 - a0, a0) * (1.0f / 256.0f), c);
      const float w = (1.f - A) * c[3];
      C0 = fmaf(w, c[0], C0);
      C1 = fmaf(w, c[1], C1);
      C2 = fmaf(w, c[2], C2);
      A += w;
      k++;
      if (A >= stop) break;
    }
  }
  m *= (1.0f / 256.0f);
  if (MODE == CTP_MODE_MIP) {
    const uint8_t o = (uint8_t)(int)floorf(fminf(m, 255.f) + 0.5f);
    if (ch == 4) *reinterpret_cast<uchar4*>(dst) = make_uchar4(o, o, o, 255);
    else dst[0] = o;
    const int mv = views.mirror[blockIdx.z];
    if (mv >= 0) {  // the opposite azimuth sees this ray's sample set from the other end: pixel dim-1-i
      uint8_t* d2 = out + (int64_t)mv * views.vstride + ((int64_t)(j - row0) * dim + (dim - 1 - i)) * ch;
      if (ch == 4) *reinterpret_cast<uchar4*>(d2) = make_uchar4(o, o, o, 255);
      else d2[0] = o;
    }
  } else {
    if (ch == 4) *reinterpret_cast<uchar4*>(dst) = make_uchar4(to_u8_unit<float>(C0), to_u8_unit<float>(C1),
                                                              to_u8_unit<float>(C2), to_u8_unit<float>(A));
    else dst[0] = to_u8_unit<float>(A);
  }
  if (views.peer) __threadfence_system();
}

struct RowPlanes {
  cudaArray_t arr = nullptr;
  cudaTextureObject_t tex = 0;
  cudaSurfaceObject_t surf = 0;
  uint16_t* bmax = nullptr;  // (rows, nby, nbx) block maxima
  int64_t rows = 0, ny = 0, nx = 0;
  ~RowPlanes() {
    if (bmax) cudaFree(bmax);
    if (tex) cudaDestroyTextureObject(tex);
    if (surf) cudaDestroySurfaceObject(surf);
    if (arr) cudaFreeArray(arr);
  }
};

// Row planes stay allocated between calls (per device, reused while the plane
// shape is unchanged): allocating and freeing a 2 GiB layered array costs
// milliseconds, a 36-view batch renders in ~40 ms.  ctp_render_release() frees them.
constexpr int kMaxDevices = 64;
static std::mutex g_planes_mu;
static std::unique_ptr<RowPlanes> g_planes[kMaxDevices];

static int get_planes(RowPlanes** out, int64_t rows, int64_t ny, int64_t nx) {
  int d = 0;
  CTP_CUDA_CALL(cudaGetDevice(&d));
  CTP_REQUIRE(d >= 0 && d < kMaxDevices, CTP_E_INVALID, "device %d out of range", d);
  std::unique_ptr<RowPlanes>& slot = g_planes[d];
  if (slot && slot->rows == rows && slot->ny == ny && slot->nx == nx) {
    *out = slot.get();
    return CTP_OK;
  }
  slot.reset();  // free the old shape before allocating the new one
  std::unique_ptr<RowPlanes> rp(new RowPlanes());
  cudaChannelFormatDesc fd = cudaCreateChannelDesc<unsigned short>();
  CTP_CUDA_CALL(cudaMalloc3DArray(&rp->arr, &fd, make_cudaExtent((size_t)nx, (size_t)ny, (size_t)rows),
                                  cudaArrayLayered | cudaArraySurfaceLoadStore));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = rp->arr;
  CTP_CUDA_CALL(cudaCreateSurfaceObject(&rp->surf, &rd));
  cudaTextureDesc td = {};
  td.addressMode[0] = cudaAddressModeClamp;
  td.addressMode[1] = cudaAddressModeClamp;
  td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  CTP_CUDA_CALL(cudaCreateTextureObject(&rp->tex, &rd, &td, nullptr));
  const int64_t nbx = (nx + kSkip - 1) / kSkip, nby = (ny + kSkip - 1) / kSkip;
  CTP_CUDA_CALL(cudaMalloc(&rp->bmax, (size_t)rows * nbx * nby * sizeof(uint16_t)));
  rp->rows = rows;
  rp->ny = ny;
  rp->nx = nx;
  slot = std::move(rp);
  *out = slot.get();
  return CTP_OK;
}

struct TexVolume {
  cudaArray_t arr = nullptr;
  cudaTextureObject_t tex = 0;
  ~TexVolume() {
    if (tex) cudaDestroyTextureObject(tex);
    if (arr) cudaFreeArray(arr);
  }
};

static int make_tex_volume(TexVolume& tv, const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, cudaStream_t st) {
  cudaChannelFormatDesc fd = cudaCreateChannelDesc<unsigned char>();
  CTP_CUDA_CALL(cudaMalloc3DArray(&tv.arr, &fd, make_cudaExtent((size_t)nx, (size_t)ny, (size_t)nz), cudaArrayLayered));
  cudaMemcpy3DParms p = {};
  p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(vol), (size_t)nx, (size_t)nx, (size_t)ny);
  p.dstArray = tv.arr;
  p.extent = make_cudaExtent((size_t)nx, (size_t)ny, (size_t)nz);
  p.kind = cudaMemcpyDeviceToDevice;
  CTP_CUDA_CALL(cudaMemcpy3DAsync(&p, st));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = tv.arr;
  cudaTextureDesc td = {};
  td.addressMode[0] = cudaAddressModeClamp;
  td.addressMode[1] = cudaAddressModeClamp;
  td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  CTP_CUDA_CALL(cudaCreateTextureObject(&tv.tex, &rd, &td, nullptr));
  return CTP_OK;
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

// Opposite azimuths of an orthographic MIP are mirror images: for theta' = theta + 180 degrees the
// march direction and the image's right vector both change sign (render.py:212-216), so pixel
// i' = dim-1-i of row j starts on the SAME line (o' = r' wx' = r wx = o) and, because steps * dt =
// 2R exactly (render.py:222), its sample k' = steps-1-k sits at t' = -R + (k'+1/2) dt = -t_k on the
// reversed direction: the same point.  Both rays take the maximum over the same sample set, so a
// turntable renders each opposite pair once and stores it twice.  (Only for the order-independent
// maximum on the fp32 path, whose contract is max-abs 1/255 -- positions agree to fp rounding;
// the fp64 paths keep the reference's per-view operation order bit for bit.)  n_prim primaries
// come out in vb.prim, each with its mirror or -1.
static int pair_opposite_views(const ViewDev* hv, int n_views, ViewBatch& vb, bool enable) {
  bool used[kMaxViews] = {false};
  int n_prim = 0;
  for (int q = 0; q < n_views; q++) {
    if (used[q]) continue;
    used[q] = true;
    int m = -1;
    for (int p = q + 1; enable && p < n_views && m < 0; p++) {
      if (used[p] || hv[p].steps != hv[q].steps || hv[p].channels != hv[q].channels) continue;
      const RenderGeom &A = hv[q].g, &B = hv[p].g;
      const double e = 1e-12;
      if (fabs(A.dx + B.dx) < e && fabs(A.dy + B.dy) < e && fabs(A.rx + B.rx) < e && fabs(A.ry + B.ry) < e) m = p;
    }
    if (m >= 0) used[m] = true;
    vb.prim[n_prim] = (int8_t)q;
    vb.mirror[n_prim] = (int8_t)m;
    n_prim++;
  }
  return n_prim;
}

// Slices a row band reads, for any mode and either precision: the trilinear
// pair around uz(j) (render.py:105-111) plus the surface gradient's +-1 and a
// one-slice margin for the fp32 floor (render.py:185-192).
static void row_slices(int64_t j, double big_r, double px_size, double n_max, int64_t nz, int64_t* lo, int64_t* hi) {
  const double uz = (big_r - ((double)j + 0.5) * px_size) * n_max + (double)(nz - 1) * 0.5;
  if (uz < -0.51 || uz > (double)nz - 0.49) { *lo = 1; *hi = 0; return; }  // row outside the volume: no slices
  const int64_t zf = (int64_t)floor(uz);
  *lo = zf - 2 < 0 ? 0 : zf - 2;
  *hi = zf + 3 > nz - 1 ? nz - 1 : zf + 3;
}

static int render_impl(const uint8_t* vol, int64_t zb, int64_t snz, int64_t nz, int64_t ny, int64_t nx,
                       const ctp_view* views, int32_t n_views, int64_t row0, int64_t row1, uint8_t* out,
                       int64_t vstride, int32_t out_flags, void* stream) {
  CTP_REQUIRE(vol && views && out, CTP_E_INVALID, "ctp_render_u8: null pointer");
  CTP_REQUIRE((out_flags & ~CTP_OUT_PEER) == 0, CTP_E_INVALID, "unknown out_flags %d", out_flags);
  CTP_REQUIRE(nz >= 1 && ny >= 1 && nx >= 1 && nx < (1LL << 31) && ny < (1LL << 31) && nz < (1LL << 31),
              CTP_E_INVALID, "ctp_render_u8: bad shape");
  CTP_REQUIRE(0 <= zb && snz >= 1 && zb + snz <= nz, CTP_E_INVALID, "slab [%lld, %lld) outside [0, %lld)",
              (long long)zb, (long long)(zb + snz), (long long)nz);
  CTP_REQUIRE(n_views >= 1 && n_views <= 65535, CTP_E_INVALID, "n_views %d outside [1, 65535]", n_views);
  const ctp_view& v0 = views[0];
  const int dim = v0.image_dim;
  // render.py:56-65 (ViewParams validation)
  CTP_REQUIRE(dim >= 16, CTP_E_INVALID, "image_dim %d below minimum 16", dim);
  CTP_REQUIRE(0 <= row0 && row0 < row1 && row1 <= dim, CTP_E_INVALID, "rows [%lld, %lld) outside [0, %d]",
              (long long)row0, (long long)row1, dim);
  ViewDev hv[kMaxViews];
  CTP_REQUIRE(n_views <= kMaxViews, CTP_E_INVALID, "at most %d views per call (got %d)", kMaxViews, n_views);
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
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 4; b++) {
        const double c0 = v.tf[a][b + 1], c1 = v.tf[a + 1][b + 1], x0 = v.tf[a][0], x1 = v.tf[a + 1][0];
        // fp64 views: the slope in double (as the oracle); fp32 views: in float, as it would be per sample
        hv[q].slope[a][b] = v.fp32 ? (double)(((float)c1 - (float)c0) / ((float)x1 - (float)x0)) : (c1 - c0) / (x1 - x0);
      }
    hv[q].early_stop = v.early_stop;
    // alpha is exactly 0 up to the last leading control point with alpha 0
    // (flat segments between them have slope 0; tf_eval clamps below tf[0])
    float zl = -1.f;
    for (int a = 0; a < 4 && v.tf[a][4] == 0.f; a++) zl = v.tf[a][0] * 256.0f;
    if (v.mode != CTP_MODE_ALPHA) zl = -1.f;
    hv[q].skip_lvl = zl;
  }
  if (zb != 0 || snz != nz) {  // a z-slab: every requested row must read only held slices
    for (int64_t j = row0; j < row1; j++) {
      int64_t lo, hi;
      row_slices(j, hv[0].g.big_r, hv[0].g.px_size, hv[0].g.inv_vx, nz, &lo, &hi);
      CTP_REQUIRE(lo > hi || (lo >= zb && hi < zb + snz), CTP_E_INVALID,
                  "row %lld reads slices [%lld, %lld], slab holds [%lld, %lld)", (long long)j, (long long)lo,
                  (long long)hi, (long long)zb, (long long)(zb + snz));
    }
  }
  cudaStream_t st = as_stream(stream);
  ViewBatch vb;
  for (int q = 0; q < n_views; q++) vb.v[q] = hv[q];
  const int64_t band = (row1 - row0) * (int64_t)dim * v0.channels;
  CTP_REQUIRE(vstride == 0 || vstride >= band, CTP_E_INVALID, "out_view_stride %lld below one band (%lld bytes)",
              (long long)vstride, (long long)band);
  vb.vstride = vstride ? vstride : band;
  vb.peer = (out_flags & CTP_OUT_PEER) ? 1 : 0;
  for (int q = 0; q < kMaxViews; q++) {
    vb.prim[q] = (int8_t)q;
    vb.mirror[q] = -1;
  }
  dim3 grid((dim + 127) / 128, (unsigned)(row1 - row0), (unsigned)n_views);
  const bool tex_path = v0.fp32 && (v0.mode == CTP_MODE_MIP || v0.mode == CTP_MODE_ALPHA) && snz <= 2048 &&
                        nx <= 32768 && ny <= 32768;
  if (tex_path) {
    // row planes when they fit comfortably (4 B per voxel per image row)
    std::unique_lock<std::mutex> lock(g_planes_mu);  // held until the planes' last reader finished
    int dev_id = 0;
    cudaGetDevice(&dev_id);
    const bool in_range = dev_id >= 0 && dev_id < kMaxDevices;
    const size_t plane_bytes = (size_t)(row1 - row0) * (size_t)nx * (size_t)ny * 2;
    // planes of this shape are already allocated: no free-memory query (cudaMemGetInfo is a
    // driver round trip that was seen to block for tens of milliseconds while the driver was
    // still working through gigabytes freed earlier by the process -- the occasional 45-135 ms
    // batch of profiles/r02_mip_hiccups.txt)
    bool fits = in_range && g_planes[dev_id] && g_planes[dev_id]->rows == row1 - row0 && g_planes[dev_id]->ny == ny &&
                g_planes[dev_id]->nx == nx;
    if (!fits) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      if (in_range && g_planes[dev_id])  // cached planes count as free
        free_b += (size_t)g_planes[dev_id]->rows * g_planes[dev_id]->ny * g_planes[dev_id]->nx * 2;
      fits = plane_bytes < free_b / 2;
    }
    const char* rp_env = getenv("CTP_RENDER_ROWPLANES");  // "0" forces the two-gather path
    if (!(rp_env && rp_env[0] == '0') && row1 - row0 <= 2048 && fits) {
      RowPlanes* rpp = nullptr;
      int rc = get_planes(&rpp, row1 - row0, ny, nx);
      if (rc != CTP_OK) return rc;
      RowPlanes& rp = *rpp;
      const RenderGeom& G0 = hv[0].g;
      const char* sk_env = getenv("CTP_RENDER_SKIP");  // "0" disables empty-space skipping
      const int skip = (sk_env && sk_env[0] == '0') ? 0 : 1;
      const int nbx = (int)((nx + kSkip - 1) / kSkip), nby = (int)((ny + kSkip - 1) / kSkip);
      dim3 bg((unsigned)((nx + kBlendCols - 1) / kBlendCols), (unsigned)nby, (unsigned)(row1 - row0));
      blend_rows_kernel<<<bg, kBlendThreads, 0, st>>>(vol, (int)zb, (int)nx, (int)ny, (int)nz, G0.big_r, G0.px_size, G0.inv_vx,
                                                   (int)row0, rp.surf, rp.bmax, nbx, nby);
      CTP_CUDA_CHECK_LAUNCH("blend_rows_kernel");
      if (v0.mode == CTP_MODE_MIP) {
        const char* mi_env = getenv("CTP_RENDER_MIRROR");  // "0": every view on its own
        dim3 pgrid = grid;
        pgrid.z = (unsigned)pair_opposite_views(hv, n_views, vb, !(mi_env && mi_env[0] == '0'));
        render_rows_kernel<CTP_MODE_MIP><<<pgrid, 128, 0, st>>>(rp.tex, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0,
                                                                (int)row1, out, rp.bmax, nbx, nby, skip);
      } else
        render_rows_kernel<CTP_MODE_ALPHA><<<grid, 128, 0, st>>>(rp.tex, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0,
                                                                 (int)row1, out, rp.bmax, nbx, nby, skip);
      CTP_CUDA_CHECK_LAUNCH("render_rows_kernel");
      CTP_CUDA_CALL(cudaStreamSynchronize(st));  // planes must outlive the kernel
      return CTP_OK;
    }
    lock.unlock();
    TexVolume tv;
    int rc = make_tex_volume(tv, vol, snz, ny, nx, st);
    if (rc != CTP_OK) return rc;
    if (v0.mode == CTP_MODE_MIP)
      render_tex_kernel<CTP_MODE_MIP><<<grid, 128, 0, st>>>(tv.tex, (int)zb, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0,
                                                            (int)row1, out);
    else
      render_tex_kernel<CTP_MODE_ALPHA><<<grid, 128, 0, st>>>(tv.tex, (int)zb, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0,
                                                              (int)row1, out);
    CTP_CUDA_CHECK_LAUNCH("render_tex_kernel");
    // the array / texture object must outlive the kernel
    CTP_CUDA_CALL(cudaStreamSynchronize(st));
    return CTP_OK;
  }
  // fp64 (the reference's modes, bit-exact): the voxel values through two texture
  // gathers per sample instead of eight scattered byte loads, which saturated L1
  // (ncu: L1/TEX 99%, issue 12%); the arithmetic is unchanged.  The texture is a
  // copy of the slab made per call (one read + one write per voxel), so it is used
  // where every ray walks its whole window (additive / MIP / alpha) and the batch
  // takes at least ~2 samples per voxel; surface rays stop at the first hit and
  // keep the byte loads.
  const double walk = (double)n_views * (double)(row1 - row0) * dim * v0.steps;
  const char* fe = getenv("CTP_RENDER_FP64_TEX");  // "0": never, "1": always (tests), else the rule above
  const bool fp64_tex = (fe && fe[0] == '1') ? true
                        : (fe && fe[0] == '0') ? false
                                               : (v0.mode != CTP_MODE_SURFACE && walk >= 2.0 * (double)snz * ny * nx);
  if (!v0.fp32 && fp64_tex && snz <= 2048 && nx <= 32768 && ny <= 32768) {
    {
      TexVolume tv;
      int rc = make_tex_volume(tv, vol, snz, ny, nx, st);
      if (rc != CTP_OK) return rc;
      render_kernel<double><<<grid, 128, 0, st>>>(vol, (int)zb, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0,
                                                  (int)row1, out, tv.tex);
      CTP_CUDA_CHECK_LAUNCH("render_kernel");
      CTP_CUDA_CALL(cudaStreamSynchronize(st));  // the array / texture object must outlive the kernel
      return CTP_OK;
    }
  }
  if (v0.fp32)
    render_kernel<float><<<grid, 128, 0, st>>>(vol, (int)zb, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0, (int)row1,
                                               out, 0);
  else
    render_kernel<double><<<grid, 128, 0, st>>>(vol, (int)zb, (int)nx, (int)ny, (int)nz, vb, dim, (int)row0, (int)row1,
                                                out, 0);
  CTP_CUDA_CHECK_LAUNCH("render_kernel");
  return CTP_OK;
}

}  // namespace ctp

using namespace ctp;

extern "C" {

int ctp_render_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, const ctp_view* views, int32_t n_views,
                  int64_t row0, int64_t row1, uint8_t* out, void* stream) {
  return render_impl(vol, 0, nz, nz, ny, nx, views, n_views, row0, row1, out, 0, 0, stream);
}

int ctp_render_slab_u8(const uint8_t* slab, int64_t z_base, int64_t slab_nz, int64_t nz, int64_t ny, int64_t nx,
                       const ctp_view* views, int32_t n_views, int64_t row0, int64_t row1, uint8_t* out,
                       int64_t out_view_stride, int32_t out_flags, void* stream) {
  return render_impl(slab, z_base, slab_nz, nz, ny, nx, views, n_views, row0, row1, out, out_view_stride, out_flags,
                     stream);
}

int ctp_render_release(void) {
  std::lock_guard<std::mutex> lock(g_planes_mu);
  for (int d = 0; d < kMaxDevices; d++) g_planes[d].reset();
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

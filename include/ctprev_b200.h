/*
 * ctprev_b200.h -- C ABI of the B200-native preview data-reduction path.
 *
 * Drop-in boundary for the ctprev reference (arXiv 2311.15038), whose hot
 * path is the Python functions re-exported by ctprev/__init__.py:29-88.
 * The reference has no FFI of its own (pure Python + numpy + numba), so
 * every entry point below names the reference function it replaces; the
 * Python mirror in paper_2311_15038_b200/ binds these through ctypes exactly
 * as a maintainer would bind them from ctprev.
 *
 * Conventions
 *   - Data pointers are DEVICE pointers (view/level descriptor arrays are host).
 *   - Volumes are C-contiguous (nz, ny, nx), x fastest (volume.py:38-62).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Calls are asynchronous on that stream; nothing here synchronises
 *     except the fp32 MIP / alpha render paths, which wait for their kernels
 *     (the texture objects they bind must outlive them).
 *   - Return value: CTP_OK (0) or a negative CTP_E* code; the message of the
 *     last failure on the calling thread is ctp_last_error().  Nothing
 *     throws across the ABI.  Functions are re-entrant ("pure and
 *     re-entrant"); the one piece of state kept between calls is the fp32
 *     render path's per-device row-plane cache (mutex-guarded,
 *     ctp_render_release() frees it).
 */
#ifndef CTPREV_B200_H
#define CTPREV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTP_ABI_VERSION 1

enum ctp_status {
  CTP_OK = 0,
  CTP_E_INVALID = -1,     /* argument outside its valid range (maps to RangeOutOfBounds / InvalidTarget) */
  CTP_E_UNSUPPORTED = -2, /* layout / dtype not supported (UnsupportedPixelFormat / UnsupportedScheme) */
  CTP_E_CUDA = -3,        /* CUDA runtime error */
  CTP_E_ALIGN = -4        /* pointer / row alignment precondition violated */
};

enum ctp_layout {
  CTP_LAYOUT_XYZ = 0,   /* dense (nz, ny, nx) level volume (volume.py Volume layout) */
  CTP_LAYOUT_ATLAS = 1  /* slicemap atlases, slicemap.py:120-142 */
};

/* One output product of a pyramid level.  For CTP_LAYOUT_ATLAS the level is
 * written straight into the packed slicemap layout of scheme (s, grid,
 * atlas_dim, map_count) -- slicemap.py:43-61 validation must already hold --
 * with slice k (global z index at this level) in map k / grid^2, cell
 * (w % grid, w / grid), w = k % grid^2 (slicemap.py:79-85).  A level smaller
 * than s on some axis is the origin-anchored _pad_to_cube case
 * (pipeline.py:226-237); the caller pre-zeroes the padding. */
typedef struct ctp_level_out {
  uint8_t* out;        /* NULL = level not materialised */
  int32_t layout;      /* enum ctp_layout */
  int32_t s;           /* atlas: scheme edge length */
  int32_t grid;        /* atlas: cells per atlas row */
  int32_t atlas_dim;   /* atlas: grid * s */
  int32_t map_count;   /* atlas: number of maps */
  int32_t flags;       /* CTP_OUT_PEER: `out` is another GPU's memory (ctp_ipc_import) */
} ctp_level_out;

/* Output flag: the destination is a peer GPU's buffer mapped through CUDA IPC.
 * Kernels writing there end with a system-scope fence (__threadfence_system),
 * so their stores are visible to the peer before any later signal issued on
 * the same stream (the collective that completes a sharded step). */
#define CTP_OUT_PEER 1

#define CTP_MAX_LEVELS 5  /* level 0 (full res) .. level 4 (16:1) */

/* ---------------- histogram (kernel 1) ---------------------------------- */

/* Replaces volume.py:252-262 volume_histogram (and Histogram256.of,
 * volume.py:117-122): hist[b] += #voxels == b over z-slab [z0, z1).
 * hist is uint64[256] and is ACCUMULATED into (zero it first), so z-slab
 * shards can be summed before an all-reduce. */
int ctp_hist_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx,
                int64_t z0, int64_t z1, uint64_t* hist, void* stream);

/* Extension (no reference): 4096-bin histogram of 12-bit uint16 voxels;
 * values >= nbins saturate into bin nbins-1.  nbins in [2, 4096]. */
int ctp_hist_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx,
                 int64_t z0, int64_t z1, int32_t nbins, uint64_t* hist, void* stream);

/* ---------------- filter LUT (kernel 2) --------------------------------- */

/* Replaces mask.py:215-231 artifact_bins + mask.py:241-245 LUT build, on
 * device: lut[b] = 0 if b == 0 or top_hist[b] > cutoff_floor, else
 * rescale(b).  cutoff_floor = floor(frac * top.size) computed by the host in
 * float64 exactly as mask.py:229 (count > cutoff <=> count > floor(cutoff)).
 * rescale_vmax = 0: identity (the u8 reference LUT); > 0: the frozen 16->8
 * rule (2*255*b + vmax) // (2*vmax) (extension).  flags (optional, uint8[nbins])
 * receives 1 for every flagged bin so the host can return the frozenset. */
int ctp_lut_build(const uint64_t* top_hist, int32_t nbins, uint64_t cutoff_floor,
                  int32_t rescale_vmax, uint8_t* lut, uint8_t* flags, void* stream);

/* The whole artifact-LUT step in ONE launch (mask.py:215-231 + 241-245): the
 * histogram of the top n_top slices of vol (elem_bytes 1: 256 bins, identity
 * LUT, rescale_vmax 0; elem_bytes 2: 4096 bins, filter o rescale), the LUT and
 * flags as ctp_lut_build, and -- if zero_hist != NULL -- zeroing of the
 * nbins-entry histogram the following fused pass accumulates into.
 * workspace: uint64[4097] that is ZERO on entry and left zero on return (the
 * last CTA resets it), so one zero-initialised buffer serves every call on
 * one stream. */
int ctp_artifact_lut(const void* vol, int32_t elem_bytes, int64_t nz, int64_t ny, int64_t nx, int32_t n_top,
                     uint64_t cutoff_floor, int32_t rescale_vmax, uint8_t* lut, uint8_t* flags, uint64_t* zero_hist,
                     uint64_t* workspace, void* stream);

/* Replaces mask.py:246 lut[volume.voxels] (filter_histogram_bins), for any
 * layout/size: out[i] = lut[in[i]] over n bytes.  If hist != NULL the raw
 * input histogram (256 bins) is accumulated in the same pass. */
int ctp_lut_apply_u8(const uint8_t* in, uint8_t* out, int64_t n, const uint8_t* lut,
                     uint64_t* hist, void* stream);

/* Extension (uint16, 12-bit; the any-size companion of ctp_preview_u16 for rows
 * that are not whole 16-byte vectors): out[i] = lut4096[min(in[i], 4095)] over
 * n elements (the filter o 16->8 rescale LUT of ctp_lut_build(vmax = 4095)).
 * If hist4096 != NULL the raw 4096-bin histogram is accumulated in the same pass. */
int ctp_lut_apply_u16(const uint16_t* in, uint8_t* out, int64_t n, const uint8_t* lut4096,
                      uint64_t* hist4096, void* stream);

/* ---------------- fused preview pass (kernels 1+2+3+4) ------------------ */

/* One HBM pass over a (z-slab of a) uint8 volume:
 *   hist (raw voxels, volume.py:252-262)          += ...      (if hist != NULL)
 *   f = lut[v]                                   (mask.py:246)
 *   level l (1 <= l <= nlev) = round_half_up(mean of 2^l x 2^l x 2^l block of f)
 *     == downscale_volume(f, (nx>>l, ny>>l, nz>>l)) (volume.py:277-309, exact
 *     integer block sums, rounded once per level -- never cascaded)
 *   levels[l].out (if non-NULL) receives level l (level 0 = f itself) in its layout.
 * Preconditions: nx % 16 == 0, nx,ny,nz divisible by 2^nlev, 0 <= nlev <= 4,
 * vol 16-byte aligned.  z_base = global z of this slab's first slice (a multiple
 * of 2^nlev), used for slab-sharded runs so atlas slice indices are global.
 * levels[] has CTP_MAX_LEVELS entries. */
int ctp_preview_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base,
                   const uint8_t* lut, int32_t nlev, const ctp_level_out* levels,
                   uint64_t* hist, void* stream);

/* Extension: the same pass over 12-bit uint16 voxels with a 4096-entry LUT
 * (filter o 16->8 rescale) and a 4096-bin histogram. nx % 8 == 0. */
int ctp_preview_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int64_t z_base,
                    const uint8_t* lut4096, int32_t nlev, const ctp_level_out* levels,
                    uint64_t* hist4096, void* stream);

/* The whole preview step of a full volume in ONE cooperative launch: the
 * artifact-LUT step of ctp_artifact_lut (top n_top slices of this volume,
 * cutoff_floor, the identity LUT for u8 / filter o rescale for u16) runs inside
 * the fused pass while its first tiles are already streaming in (one grid
 * barrier), then the pass of ctp_preview_u8 / _u16 with that LUT.  hist is
 * zeroed by the launch; lut_out / flags_out (optional) receive the LUT and the
 * artifact-bin flags; workspace: uint64[4097], zero on entry, left zero. */
int ctp_preview_step_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx, int32_t n_top,
                        uint64_t cutoff_floor, int32_t nlev, const ctp_level_out* levels, uint64_t* hist,
                        uint8_t* lut_out, uint8_t* flags_out, uint64_t* workspace, void* stream);
int ctp_preview_step_u16(const uint16_t* vol, int64_t nz, int64_t ny, int64_t nx, int32_t n_top,
                         uint64_t cutoff_floor, int32_t nlev, const ctp_level_out* levels, uint64_t* hist4096,
                         uint8_t* lut_out, uint8_t* flags_out, uint64_t* workspace, void* stream);

/* ---------------- general resampling / atlas packing -------------------- */

/* Replaces volume.py:277-309 downscale_volume for ANY target (half-open
 * cells from _cell_starts, volume.py:265-274, round half up).  Identity
 * targets copy.  Returns CTP_E_INVALID unless 1 <= t <= n on every axis. */
int ctp_downscale_u8(const uint8_t* in, int64_t nz, int64_t ny, int64_t nx,
                     int64_t tz, int64_t ty, int64_t tx, uint8_t* out, void* stream);

/* Replaces the packing half of slicemap.py:120-142 (encode_slicemaps after its
 * downscale) fused with pipeline.py:226-237 (_pad_to_cube): cube (nz,ny,nx)
 * with every dim <= s is written into map_count atlases of atlas_dim^2 bytes
 * (contiguous), cells beyond the data zero-filled. */
int ctp_encode_atlas_u8(const uint8_t* cube, int64_t nz, int64_t ny, int64_t nx,
                        int32_t s, int32_t grid, int32_t atlas_dim, int32_t map_count,
                        uint8_t* atlases, void* stream);

/* Replaces mask.py:194-212 apply_circle_mask: out = in where (x - cx)^2 +
 * (y - cy)^2 <= r_eff_sq (fp64, no FMA contraction: numpy's exact predicate),
 * else 0, on every slice.  r_eff_sq = (r * (1 - margin))**2 from the host. */
int ctp_circle_mask_u8(const uint8_t* in, int64_t nz, int64_t ny, int64_t nx, double cx, double cy,
                       double r_eff_sq, uint8_t* out, void* stream);

/* Inverse (slicemap.py:145-155 decode_slicemaps): atlases -> s^3 cube. */
int ctp_decode_atlas_u8(const uint8_t* atlases, int32_t s, int32_t grid, int32_t atlas_dim,
                        int32_t map_count, uint8_t* cube, void* stream);

/* ---------------- server-side ray casting (kernel 5) -------------------- */

enum ctp_render_mode {
  CTP_MODE_SURFACE = 0,   /* render.py:149-202 */
  CTP_MODE_ADDITIVE = 1,  /* render.py:125-146 */
  CTP_MODE_MIP = 2,       /* extension */
  CTP_MODE_ALPHA = 3      /* extension: front-to-back, 1D RGBA TF */
};

/* One view: ViewParams (render.py:39-65) + the extension knobs. */
typedef struct ctp_view {
  double azimuth_deg;      /* already normalised to [0, 360) (render.py:55) */
  int32_t image_dim;
  int32_t steps;
  int32_t mode;            /* enum ctp_render_mode */
  int32_t threshold;       /* surface */
  double gain;             /* additive */
  float tf[4][5];          /* alpha: 4 control points (value, r, g, b, a), ascending value */
  float early_stop;        /* alpha: stop when accumulated alpha >= this (0.99) */
  int32_t channels;        /* 1 = gray u8, 4 = RGBA8 */
  int32_t fp32;            /* 0 = fp64 arithmetic (bit-exact to render.py), 1 = fp32 */
} ctp_view;

/* Replaces render.py:205-236 render_view, batched: n_views images of
 * image_dim^2 * channels bytes each, rows [row0, row1) only (image-tile
 * split across GPUs; pass 0, image_dim for whole frames).  All views must
 * share image_dim, mode, channels and fp32. */
int ctp_render_u8(const uint8_t* vol, int64_t nz, int64_t ny, int64_t nx,
                  const ctp_view* views, int32_t n_views, int64_t row0, int64_t row1,
                  uint8_t* out, void* stream);

/* The same over a z-slab (sort-last at the reference's elevation-0 camera,
 * render.py:131-140: image row j samples only the slices around one uz(j), so
 * per-slab images are disjoint row bands).  `slab` holds slices
 * [z_base, z_base + slab_nz) of an nz-deep volume; the geometry is the full
 * volume's.  Every row in [row0, row1) must read only held slices (the
 * trilinear pair, the surface gradient's +-1 and one slice of margin:
 * [floor(uz)-2, floor(uz)+3]), else CTP_E_INVALID.  View q's band is written
 * at out + q * out_view_stride (0 = packed bands); with `out` pointing at row
 * row0 of a full-image buffer (stride = image bytes) -- e.g. rank 0's images
 * mapped through ctp_ipc_import, out_flags = CTP_OUT_PEER) -- the sort-last
 * composite is the render. */
int ctp_render_slab_u8(const uint8_t* slab, int64_t z_base, int64_t slab_nz,
                       int64_t nz, int64_t ny, int64_t nx,
                       const ctp_view* views, int32_t n_views, int64_t row0, int64_t row1,
                       uint8_t* out, int64_t out_view_stride, int32_t out_flags, void* stream);

/* The fp32 MIP/alpha path keeps its per-row planes (2 B per voxel per image
 * row) allocated between calls while the shape is unchanged; this frees them. */
int ctp_render_release(void);

/* Per-image 256-bin histograms for image_entropy (render.py:248-262):
 * hist[i*256 + b] = #pixels of image i equal to b (accumulated). */
int ctp_image_hist_u8(const uint8_t* imgs, int32_t n_images, int64_t pixels,
                      uint64_t* hist, void* stream);

/* ---------------- atlas PNG encoding --------------- */

/* PNG scanline filtering for save_slicemaps (slicemap.py:158-166, which
 * writes every atlas with Pillow): for each row of n_images grayscale
 * images (height x width, u8) applies PNG filter `filter` (0..4: None/Sub/
 * Up/Average/Paeth, bpp 1) or, with filter = -1, the one whose residual
 * bytes have the lowest order-0 entropy in the row, and writes [filter byte,
 * residuals] -- out is n_images x height x (width + 1) bytes, the raw stream
 * a PNG IDAT deflates. */
int ctp_png_filter_u8(const uint8_t* images, int32_t n_images, int64_t height, int64_t width,
                      int32_t filter, uint8_t* out, void* stream);

/* DEFLATE (RFC 1951) of n_streams byte streams of stream_len bytes each (the
 * PNG-filtered scanlines of ctp_png_filter_u8): every stream is cut into
 * chunks (ctp_deflate_geometry: chunk_bytes in, at most chunk_out_bytes out),
 * each one dynamic-Huffman (or stored) block, non-final chunks ending with a
 * sync flush, so the chunks of a stream concatenate into one raw deflate
 * stream.  Chunk c (= stream * chunks_per_stream + k) is written at
 * out + c * chunk_out_bytes, its size to out_bytes[c], and its Adler-32
 * partials (sum d_i, sum (n - i) d_i) to adler[2c], adler[2c + 1].  row_len
 * adds the image row (and two rows) to the match distances.  scratch holds
 * grid * chunk_bytes uint32 tokens; grid CTAs loop over all chunks. */
int ctp_deflate_geometry(int32_t* chunk_bytes, int32_t* chunk_out_bytes);
int ctp_deflate_u8(const uint8_t* data, int64_t n_streams, int64_t stream_len, int32_t row_len,
                   uint8_t* out, int32_t* out_bytes, uint64_t* adler, uint32_t* scratch,
                   int32_t grid, void* stream);
/* Gather the chunks into one buffer: chunk c's out_bytes[c] bytes to dst + offsets[c]. */
int ctp_deflate_compact(const uint8_t* out, const int32_t* out_bytes, const int64_t* offsets,
                        int64_t total_chunks, uint8_t* dst, void* stream);

/* ---------------- peer memory between the ranks of a node (s8(e)) ------- */

#define CTP_IPC_HANDLE_BYTES 64

/* Export a device buffer to the other processes of the node: the CUDA IPC
 * handle of the allocation holding `ptr` and ptr's offset in it.  With the
 * imported pointer as a level's destination, a rank's fused pass
 * (ctp_preview_u8/u16) stores its slab's atlas rows straight into rank 0's
 * atlases over NVLink -- the atlas gather of the z-slab sharding
 * fused into the pass. */
int ctp_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset);
int ctp_ipc_import(const uint8_t* handle, int64_t offset, void** ptr);
int ctp_ipc_close(void* ptr, int64_t offset);

/* ---------------- synthetic inputs (BASELINE configs) ------------------- */

/* One ellipsoidal shell of the synthetic generators. */
typedef struct ctp_shell {
  float cx, cy, cz;        /* centre, voxels */
  float ax, ay, az;        /* semi-axes, voxels */
  float thickness;         /* voxels */
  float mean, sd;          /* intensity N(mean, sd) */
  float _pad;
} ctp_shell;

/* Fill a (z-slab of a) volume: background N(bg_mean, bg_sd) clipped, shells,
 * speckle with probability speckle_p -- uniform in [0, vmax] (speckle_lambda
 * = 0, config 2) or a Poisson-like count of mean speckle_lambda (the normal
 * approximation N(lambda, lambda), config 3/5); counter-based hash RNG keyed
 * by (seed, global voxel index), so any slab of the same volume is
 * reproducible.  elem_bytes = 1 (uint8, vmax 255) or 2 (uint16, vmax). */
int ctp_synth_volume(void* vol, int32_t elem_bytes, int64_t nz, int64_t ny, int64_t nx,
                     int64_t z_base, int64_t full_nz, uint64_t seed, float bg_mean, float bg_sd,
                     int32_t vmax, const ctp_shell* shells, int32_t n_shells,
                     float speckle_p, float speckle_lambda, void* stream);

/* ---------------- misc --------------------------------------------------- */

const char* ctp_last_error(void);
int ctp_abi_version(void);
/* Number of kernels this library launched on the calling thread since the
 * last reset (for bench.py's gpu_launches). */
int64_t ctp_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* CTPREV_B200_H */

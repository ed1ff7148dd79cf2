"""B200-native preview data-reduction path of arXiv 2311.15038 (reference: ``ctprev``).

The public surface mirrors the reference's hot-path API
(ctprev/__init__.py:29-88) so it is a drop-in for that path:

    volume_histogram, Histogram256.of, artifact_bins, filter_histogram_bins,
    downscale_volume, encode_slicemaps, decode_slicemaps, plan_scheme,
    slice_cell, render_view, image_entropy, optimal_snapshot, apply_circle_mask,
    build_data_preview, build_interactive_preview, build_list_preview, save_slicemaps

plus the fused one-pass ``preview_pipeline`` and batched ``render_views``
(MIP / front-to-back alpha extensions).  All arithmetic runs in the sm_100a
kernels of ``csrc/`` behind the C ABI of ``include/ctprev_b200.h``; there is
no CPU fallback.  ``install()`` rebinds these functions inside an imported
``ctprev`` package.
"""
from .errors import *  # noqa: F401,F403
from .types import (ADDITIVE, ALPHA, MIP, SURFACE, EntropyResult, Histogram256, SlicemapScheme, SlicemapSet,
                    SnapshotResult, ViewParams, Volume, plan_scheme, slice_cell)
from .ops import (PreviewResult, apply_circle_mask, artifact_bins, build_data_preview, build_interactive_preview,
                  build_list_preview,
                  decode_slicemaps, downscale_volume, encode_slicemaps, save_slicemaps,
                  filter_histogram_bins, image_entropy, load_slice_stack, load_volume, optimal_snapshot, preview_pipeline,
                  render_view, render_views, volume_histogram)
from .install import install, uninstall

__version__ = "0.1.0"

__all__ = [
    "Volume", "Histogram256", "SlicemapScheme", "SlicemapSet", "ViewParams", "EntropyResult",
    "SnapshotResult", "SURFACE", "ADDITIVE", "MIP", "ALPHA", "plan_scheme", "slice_cell",
    "volume_histogram", "artifact_bins", "filter_histogram_bins", "downscale_volume", "encode_slicemaps",
    "decode_slicemaps", "render_view", "render_views", "image_entropy", "optimal_snapshot",
    "preview_pipeline", "PreviewResult", "build_data_preview", "build_interactive_preview", "build_list_preview",
    "apply_circle_mask",
    "save_slicemaps", "load_slice_stack", "load_volume", "install", "uninstall",
]

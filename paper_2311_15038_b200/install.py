"""Drop-in installation into the reference package ``ctprev``.

The reference has no plugin mechanism: its modules bind the hot-path names at
import time (pipeline.py:36-59, slicemap.py:26, cli.py:20-24, and the package
namespace __init__.py:29-88), so replacing the path means rebinding the
attribute at every site.  ``install()`` does exactly that and points result
construction at the reference's own classes; ``uninstall()`` restores the
originals.
"""
from __future__ import annotations

import importlib

from . import ops
from .types import FACTORY

# function name -> modules (under ctprev) that bind it
BINDINGS = {
    "volume_histogram": ["volume", "pipeline", "cli", ""],
    "downscale_volume": ["volume", "slicemap", "pipeline", "cli", ""],
    "artifact_bins": ["mask", "pipeline", "cli", ""],
    "filter_histogram_bins": ["mask", "pipeline", "cli", ""],
    "encode_slicemaps": ["slicemap", "pipeline", "cli", ""],
    "decode_slicemaps": ["slicemap", "pipeline", "cli", ""],
    "render_view": ["render", "cli", ""],
    "image_entropy": ["render", "cli", ""],
    "optimal_snapshot": ["render", "pipeline", "cli", ""],
    "build_data_preview": ["pipeline", ""],
    "apply_circle_mask": ["mask", "pipeline", "cli", ""],
    "build_interactive_preview": ["pipeline", ""],
    "build_list_preview": ["pipeline", ""],
    "save_slicemaps": ["slicemap", "pipeline", ""],
    "load_slice_stack": ["volume", "pipeline", ""],
    "load_volume": ["volume", "pipeline", "cli", ""],
}

_saved: dict = {}


def install(package: str = "ctprev", exclude=()) -> list[str]:
    """Rebind the reference's hot-path functions to the B200 implementation.
    Returns the list of patched 'module.name' sites.  ``exclude``: names to leave
    bound to the reference (e.g. ``("save_slicemaps",)`` keeps Pillow's PNG writer,
    whose bytes the reference's recorded bundle checksums pin)."""
    root = importlib.import_module(package)
    vol = importlib.import_module(f"{package}.volume")
    sm = importlib.import_module(f"{package}.slicemap")
    rd = importlib.import_module(f"{package}.render")
    FACTORY.Volume = vol.Volume
    FACTORY.Histogram256 = vol.Histogram256
    FACTORY.SlicemapScheme = sm.SlicemapScheme
    FACTORY.SlicemapSet = sm.SlicemapSet
    FACTORY.EntropyResult = rd.EntropyResult
    FACTORY.SnapshotResult = rd.SnapshotResult
    pl = importlib.import_module(f"{package}.pipeline")
    FACTORY.DataPreview = pl.DataPreview
    FACTORY.InteractivePreview = pl.InteractivePreview
    FACTORY.ListPreview = pl.ListPreview
    FACTORY.Circle = importlib.import_module(f"{package}.mask").Circle
    # the error classes must BE the reference's (its callers catch them, pipeline.py:176-191,
    # cli.py:211; our builders catch NoCircleFound / DegenerateHistogram raised by the
    # reference's host helpers): rebind them when ctprev was imported after this package
    from . import errors as _errors
    _errors.bind(importlib.import_module(f"{package}.errors"))
    patched = []
    for name, mods in BINDINGS.items():
        if name in exclude:
            continue
        new = getattr(ops, name)
        for m in mods:
            modname = f"{package}.{m}" if m else package
            try:
                mod = importlib.import_module(modname) if m else root
            except Exception:
                continue
            if hasattr(mod, name):
                _saved.setdefault((modname, name), getattr(mod, name))
                setattr(mod, name, new)
                patched.append(f"{modname}.{name}")
    return patched


def uninstall() -> None:
    for (modname, name), fn in _saved.items():
        setattr(importlib.import_module(modname), name, fn)
    _saved.clear()
    FACTORY.reset()

"""ctypes binding of the C ABI declared in ``include/ctprev_b200.h``.

The shared library is built in-tree (``_lib/libctprev_b200.so``) by
``_build.py``.  There is no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises ``NativeUnavailable`` loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libctprev_b200.so"

CTP_OK = 0
CTP_E_INVALID = -1
CTP_E_UNSUPPORTED = -2
CTP_E_CUDA = -3
CTP_E_ALIGN = -4

LAYOUT_XYZ = 0
LAYOUT_ATLAS = 1
OUT_PEER = 1  # ctp_level_out.flags / out_flags: destination mapped from a peer GPU
MAX_LEVELS = 5

MODE_SURFACE, MODE_ADDITIVE, MODE_MIP, MODE_ALPHA = 0, 1, 2, 3


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or no CUDA device is visible."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code
        self.msg = msg


class LevelOut(C.Structure):
    _fields_ = [
        ("out", C.c_void_p),
        ("layout", C.c_int32),
        ("s", C.c_int32),
        ("grid", C.c_int32),
        ("atlas_dim", C.c_int32),
        ("map_count", C.c_int32),
        ("flags", C.c_int32),   # OUT_PEER: a peer GPU's memory (ctp_ipc_import)
    ]


class View(C.Structure):
    _fields_ = [
        ("azimuth_deg", C.c_double),
        ("image_dim", C.c_int32),
        ("steps", C.c_int32),
        ("mode", C.c_int32),
        ("threshold", C.c_int32),
        ("gain", C.c_double),
        ("tf", (C.c_float * 5) * 4),
        ("early_stop", C.c_float),
        ("channels", C.c_int32),
        ("fp32", C.c_int32),
    ]


class Shell(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("cx", "cy", "cz", "ax", "ay", "az", "thickness", "mean", "sd", "_pad")]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

# name -> (argtypes); every function returns int status unless listed in _RESTYPE
SIGNATURES = {
    "ctp_hist_u8": [_P, _I64, _I64, _I64, _I64, _I64, _P, _P],
    "ctp_hist_u16": [_P, _I64, _I64, _I64, _I64, _I64, _I32, _P, _P],
    "ctp_lut_build": [_P, _I32, C.c_uint64, _I32, _P, _P, _P],
    "ctp_lut_apply_u8": [_P, _P, _I64, _P, _P, _P],
    "ctp_lut_apply_u16": [_P, _P, _I64, _P, _P, _P],
    "ctp_artifact_lut": [_P, _I32, _I64, _I64, _I64, _I32, C.c_uint64, _I32, _P, _P, _P, _P, _P],
    "ctp_preview_u8": [_P, _I64, _I64, _I64, _I64, _P, _I32, C.POINTER(LevelOut), _P, _P],
    "ctp_preview_u16": [_P, _I64, _I64, _I64, _I64, _P, _I32, C.POINTER(LevelOut), _P, _P],
    "ctp_preview_step_u8": [_P, _I64, _I64, _I64, _I32, C.c_uint64, _I32, C.POINTER(LevelOut), _P, _P, _P, _P, _P],
    "ctp_preview_step_u16": [_P, _I64, _I64, _I64, _I32, C.c_uint64, _I32, C.POINTER(LevelOut), _P, _P, _P, _P, _P],
    "ctp_downscale_u8": [_P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P],
    "ctp_encode_atlas_u8": [_P, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P],
    "ctp_decode_atlas_u8": [_P, _I32, _I32, _I32, _I32, _P, _P],
    "ctp_circle_mask_u8": [_P, _I64, _I64, _I64, C.c_double, C.c_double, C.c_double, _P, _P],
    "ctp_render_u8": [_P, _I64, _I64, _I64, C.POINTER(View), _I32, _I64, _I64, _P, _P],
    "ctp_render_slab_u8": [_P, _I64, _I64, _I64, _I64, _I64, C.POINTER(View), _I32, _I64, _I64, _P, _I64, _I32, _P],
    "ctp_render_release": [],
    "ctp_png_filter_u8": [_P, _I32, _I64, _I64, _I32, _P, _P],
    "ctp_deflate_geometry": [C.POINTER(_I32), C.POINTER(_I32)],
    "ctp_deflate_u8": [_P, _I64, _I64, _I32, _P, _P, _P, _P, _I32, _P],
    "ctp_deflate_compact": [_P, _P, _P, _I64, _P, _P],
    "ctp_ipc_export": [_P, _P, C.POINTER(C.c_int64)],
    "ctp_ipc_import": [_P, _I64, C.POINTER(C.c_void_p)],
    "ctp_ipc_close": [_P, _I64],
    "ctp_image_hist_u8": [_P, _I32, _I64, _P, _P],
    "ctp_synth_volume": [_P, _I32, _I64, _I64, _I64, _I64, _I64, C.c_uint64, C.c_float, C.c_float, _I32,
                         C.POINTER(Shell), _I32, C.c_float, C.c_float, _P],
    "ctp_last_error": [],
    "ctp_abi_version": [],
    "ctp_launch_count": [_I32],
}
_RESTYPE = {"ctp_last_error": C.c_char_p, "ctp_abi_version": C.c_int, "ctp_launch_count": C.c_int64}

_lib = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the shared library.  Raises NativeUnavailable."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -m paper_2311_15038_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, C.c_int)
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise NativeError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != CTP_OK:
        msg = lib.ctp_last_error().decode(errors="replace")
        raise NativeError(name, rc, msg)


def launch_count(reset: bool = False) -> int:
    return int(load().ctp_launch_count(1 if reset else 0))


def levels_array(levels: list[LevelOut | None]):
    arr = (LevelOut * MAX_LEVELS)()
    for i, lv in enumerate(levels[:MAX_LEVELS]):
        if lv is not None:
            arr[i] = lv
    return arr

"""The C-ABI library loads, exports every symbol include/ctprev_b200.h declares,
and validates arguments before touching the GPU (CPU only: no compute calls)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2311_15038_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "ctprev_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ctp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2311_15038_b200 import _build
        _build.build(verbose=False)
    return _lib.load()


def test_header_declares_the_api():
    names = declared_functions()
    for must in ("ctp_hist_u8", "ctp_lut_build", "ctp_lut_apply_u8", "ctp_preview_u8", "ctp_preview_u16",
                 "ctp_downscale_u8", "ctp_encode_atlas_u8", "ctp_render_u8", "ctp_image_hist_u8",
                 "ctp_last_error"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"


def test_abi_version(lib):
    assert lib.ctp_abi_version() == 1


def test_struct_layouts_match_header():
    # ctp_level_out: pointer + 6 x int32 -> 32 bytes; ctp_view: see header
    assert C.sizeof(_lib.LevelOut) == 32
    assert C.sizeof(_lib.View) == 8 + 4 * 4 + 8 + 80 + 4 + 4 + 4 + 4  # + tail padding
    assert C.sizeof(_lib.Shell) == 40


def _err(lib) -> str:
    return lib.ctp_last_error().decode()


def test_validation_errors_without_gpu(lib):
    # z_range checks mirror volume.py:260-261 and fire before any launch
    rc = lib.ctp_hist_u8(C.c_void_p(16), 4, 4, 4, 3, 3, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "z_range" in _err(lib)
    rc = lib.ctp_hist_u8(None, 4, 4, 4, 0, 4, None, None)
    assert rc == _lib.CTP_E_INVALID
    # downscale target checks mirror volume.py:287-289
    rc = lib.ctp_downscale_u8(C.c_void_p(16), 4, 4, 4, 4, 4, 8, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "target x=8" in _err(lib)
    rc = lib.ctp_downscale_u8(C.c_void_p(16), 4, 4, 4, 0, 4, 4, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "target z=0" in _err(lib)
    # scheme checks mirror slicemap.py:52-61
    rc = lib.ctp_encode_atlas_u8(C.c_void_p(16), 128, 128, 128, 128, 8, 1000, 2, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_UNSUPPORTED and "atlas 1000" in _err(lib)
    rc = lib.ctp_encode_atlas_u8(C.c_void_p(16), 128, 128, 128, 128, 8, 1024, 3, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_UNSUPPORTED and "3 maps" in _err(lib)
    # fused pass preconditions
    lv = _lib.levels_array([None] * 5)
    rc = lib.ctp_preview_u8(C.c_void_p(16), 8, 8, 24, 0, None, 1, lv, None, None)
    assert rc == _lib.CTP_E_ALIGN
    rc = lib.ctp_preview_u8(C.c_void_p(16), 7, 8, 32, 0, None, 1, lv, None, None)
    assert rc == _lib.CTP_E_INVALID
    rc = lib.ctp_preview_u8(C.c_void_p(16), 8, 8, 32, 0, None, 5, lv, None, None)
    assert rc == _lib.CTP_E_INVALID
    # render: ViewParams bounds (render.py:56-65)
    v = _lib.View()
    v.image_dim, v.steps, v.mode, v.threshold, v.gain, v.channels = 15, 64, 0, 1, 4.0, 1
    rc = lib.ctp_render_u8(C.c_void_p(16), 8, 8, 8, C.byref(v), 1, 0, 15, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "image_dim" in _err(lib)
    v.image_dim, v.steps = 16, 31
    rc = lib.ctp_render_u8(C.c_void_p(16), 8, 8, 8, C.byref(v), 1, 0, 16, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "steps" in _err(lib)
    # LUT build
    rc = lib.ctp_lut_build(C.c_void_p(16), 4097, 0, 4095, C.c_void_p(16), None, None)
    assert rc == _lib.CTP_E_INVALID


def test_launch_counter_starts_at_zero(lib):
    lib.ctp_launch_count(1)
    assert lib.ctp_launch_count(0) == 0


def test_validation_errors_without_gpu_newer_entry_points(lib):
    # slab rendering: the slab must lie inside the volume
    view = _lib.View()
    rc = lib.ctp_render_slab_u8(C.c_void_p(16), 90, 20, 100, 8, 8, C.byref(view), 1, 0, 16, C.c_void_p(16), 0, 0, None)
    assert rc == _lib.CTP_E_INVALID and "slab" in _err(lib)
    rc = lib.ctp_render_slab_u8(None, 0, 8, 8, 8, 8, C.byref(view), 1, 0, 16, C.c_void_p(16), 0, 0, None)
    assert rc == _lib.CTP_E_INVALID
    # PNG filtering and IPC argument checks
    rc = lib.ctp_png_filter_u8(None, 1, 4, 4, -1, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID
    rc = lib.ctp_png_filter_u8(C.c_void_p(16), 0, 4, 4, -1, C.c_void_p(16), None)
    assert rc == _lib.CTP_E_INVALID and "bad shape" in _err(lib)
    rc = lib.ctp_ipc_import(None, 0, C.byref(C.c_void_p()))
    assert rc == _lib.CTP_E_INVALID
    rc = lib.ctp_ipc_close(None, 0)
    assert rc == _lib.CTP_E_INVALID
    rc = lib.ctp_ipc_export(None, C.create_string_buffer(64), C.byref(C.c_int64()))
    assert rc == _lib.CTP_E_INVALID

"""NVTX ranges around the stages of the path (visible in nsys / ncu timelines;
no-ops without a profiler attached).

    with trace.range("preview.fused_pass"):
        ...
"""
from __future__ import annotations

import contextlib

import torch


@contextlib.contextmanager
def range(name: str):  # noqa: A001 - mirrors nvtx's own name
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()

"""Build the library with extra nvcc flags into another path (A/B timing of
kernel variants with tools/prof_preview.py --lib PATH).

usage: python tools/build_variant.py OUT.so -DFLAG [...]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
out, flags = sys.argv[1], sys.argv[2:]
os.environ["CTP_NVCC_EXTRA"] = " ".join(flags)
from paper_2311_15038_b200 import _build  # noqa: E402

_build.COMMON += flags
_build.LIB = Path(out).resolve()
_build.build(verbose=False, force=True)
print("built", _build.LIB, flags)

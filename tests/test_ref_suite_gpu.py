"""The REFERENCE's own test suite on the GPU, with its hot path rebound by ``install()``
("a drop-in for that path"): ctprev's WHOLE suite -- volume / mask / slicemap /
render / pipeline / threshold / phantom / cli / service plus its ten acceptance criteria
(/root/reference/pkg/tests: 287 pass, 15 skip, as for the unmodified reference) -- runs UNMODIFIED in a subprocess whose pytest loads
tools/ref_suite_plugin.py: ``install()`` is called before any test module is imported, so
every ``from ctprev.volume import ...`` binds the B200 drop-ins, and the session ends with
the number of kernels launched through libctprev_b200.so.

The reference's tests are not part of this repository and are never copied into its history:
they are read from the mounted reference, or from ``baseline/_ref_tests`` if someone placed
them next to the installed reference for a GPU run (``tools/r2_ref_suite.sh`` does, into that
git-ignored directory, and removes nothing else); where neither exists -- the GPU box of a
plain checkout -- the test is skipped, and the log of the round's run is
``profiles/r02_ref_suite_under_install.txt`` (287 passed, 15 skipped, 49 binding sites, 665 launches)."""
from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
FILES: list = []  # none named: the reference's whole suite (volume, mask, slicemap, render, pipeline,
                  # acceptance, threshold, phantom, cli, service)


@pytest.mark.gpu
def test_reference_test_suite_passes_with_the_b200_path_installed(cuda, tmp_path):
    ref = ROOT / "baseline" / "_ref"
    tests = next((d for d in (ROOT / "baseline" / "_ref_tests", Path("/root/reference/pkg/tests"))
                  if (d / "test_volume.py").is_file()), None)
    if tests is None or not (ref / "ctprev").is_dir():
        pytest.skip("the reference's tests (baseline/_ref_tests) or its install (baseline/_ref) are not present")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tools"), str(ROOT), str(ref)])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/ctp_ref_numba_cache")
    r = subprocess.run([sys.executable, "-m", "pytest", *FILES, "-q", "-p", "ref_suite_plugin", "-p", "no:cacheprovider",
                        "--basetemp", str(tmp_path / "ref")], cwd=tests, env=env, capture_output=True, text=True,
                       timeout=1800)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail + r.stderr[-2000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 280 and "failed" not in r.stdout, tail
    for k in range(1, 11):  # the ten acceptance criteria of the reference (tests/conftest.py summary)
        assert re.search(rf"criterion\s+{k}: PASS", r.stdout), tail
    lm = re.search(r"(\d+) binding sites rebound, (\d+) kernel launches", r.stdout)
    assert lm and int(lm.group(1)) > 0 and int(lm.group(2)) > 100, tail  # the device path ran

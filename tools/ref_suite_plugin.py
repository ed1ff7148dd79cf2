"""pytest plugin: run the REFERENCE's own test suite with its hot path rebound to the
B200 drop-ins (``-p ref_suite_plugin`` with tools/ on PYTHONPATH).

``install()`` runs in pytest_configure, i.e. before any test module is imported, so the
tests' ``from ctprev.volume import volume_histogram`` (and every other binding site) see
the device implementations.  See tests/test_ref_suite_gpu.py and tools/r2_ref_suite.sh.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
_patched = []


def pytest_configure(config):
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    import ctprev  # noqa: F401  (the reference, from baseline/_ref on PYTHONPATH)
    import paper_2311_15038_b200 as b200
    _patched.extend(b200.install())


def pytest_report_header(config):
    return f"ctprev hot path rebound to paper_2311_15038_b200: {len(_patched)} binding sites"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    # evidence that the device path ran: kernels launched through the C ABI during the session
    from paper_2311_15038_b200 import _lib
    n = _lib.launch_count()
    terminalreporter.write_line(f"B200 drop-in: {len(_patched)} binding sites rebound, {n} kernel launches "
                                f"through libctprev_b200.so during this session")

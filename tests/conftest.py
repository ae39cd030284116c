import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle", ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


def pytest_sessionfinish(session, exitstatus):
    """With FDSWEEP_REDZONE set (tests/test_gpu_redzone.py runs the GPU suites that way in a child
    process), the session fails unless every guard zone around the library's device allocations is
    intact; the summary line is what the parent test reads."""
    import os

    if not os.environ.get("FDSWEEP_REDZONE"):
        return
    import paper_1511_04355_b200.api as api

    if api._lib is None:  # no GPU test ran
        return
    r = api.redzone_check()
    print(f"\nredzone: enabled={int(r['enabled'])} overwritten_bytes={r['overwritten_bytes']} "
          f"checks={r['checks']} live={r['live']}")
    if not r["enabled"] or r["overwritten_bytes"] != 0:
        session.exitstatus = 1

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# the multi-view chunk lists switch on only for large launches (n x views >= 2^26); the GPU tests force them for
# every multi-view launch (ADOP_MV_LISTS bit 3) so the small parity cases exercise them too
# (test_multi_view_list_orders runs the default and the flat lists in subprocesses)
os.environ.setdefault("ADOP_MV_LISTS", "13")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_sessionfinish(session, exitstatus):
    """Write the parity error report of the GPU comparisons (tests/parity.py REPORT), if any ran."""
    parity = sys.modules.get("tests.parity")
    if parity is None or not parity.REPORT:
        return
    import json
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_report.json"), "w") as f:
        json.dump(parity.REPORT, f, indent=1)

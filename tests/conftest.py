import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


# ---- the oracle's full cfg4 PageRank vector, computed in the background -------------------------
# tests/test_zz_cfg4_full_gpu.py compares all 67,108,864 cfg4 PageRank values with the oracle.
# The oracle needs ~12 min of one host core there, so it starts as soon as collection finds that
# test (on a machine with a GPU) and runs while the other GPU tests do; the test waits for it.
from tests._bg import CFG4_FULL  # noqa: E402


def _gpu_present():
    import glob
    return bool(glob.glob("/dev/nvidia[0-9]*"))


def pytest_collection_finish(session):
    import subprocess
    import tempfile
    import time
    if os.environ.get("IPREGEL_CFG4_FULL", "1") == "0" or not _gpu_present():
        return
    if not any("test_zz_cfg4_full_gpu" in item.nodeid for item in session.items):
        return
    d = tempfile.mkdtemp(prefix="ipregel_cfg4_")
    out = os.path.join(d, "pagerank")
    log = open(os.path.join(d, "oracle.log"), "w")
    CFG4_FULL["proc"] = subprocess.Popen(
        [sys.executable, os.path.join(ROOT, "tests", "golden", "cfg4_pagerank_full.py"),
         "--out", out], stdout=log, stderr=subprocess.STDOUT, cwd=ROOT)
    CFG4_FULL.update(out=out, log=log.name, t0=time.time())


def pytest_sessionfinish(session, exitstatus):
    p = CFG4_FULL["proc"]
    if p is not None and p.poll() is None:
        p.kill()   # the exact process this session started
        p.wait()

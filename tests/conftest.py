import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _ensure_built():
    so = os.path.join(REPO, "paper_2507_06608_b200", "libnexus_b200.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "paper_2507_06608_b200"), "-j8"],
                       check=True)
    ref = os.path.join(REPO, "oracle", "_ref", "libnexussim_ref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle"), "-j8"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def nx():
    import paper_2507_06608_b200 as m
    return m


@pytest.fixture(scope="session")
def ref():
    from oracle import reference as r
    if not r.available():
        pytest.skip("reference oracle library not built (needs /root/reference here)")
    return r


def has_gpu() -> bool:
    try:
        import ctypes
        cudart = ctypes.CDLL("libcuda.so.1")
        return cudart is not None
    except OSError:
        return False

"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libfvb.so; they fail (never skip into a fallback) when either is missing."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# Every lowered kernel the tests use is compiled fresh: the on-disk image
# cache points at a directory private to this session.
if "FVB_CACHE_DIR" not in os.environ:
    import tempfile
    os.environ["FVB_CACHE_DIR"] = tempfile.mkdtemp(prefix="fvb-test-cache-")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    # A fresh checkout has no built artefacts (they are git-ignored): build
    # them once (__graft_entry__.build: libfvb.so for sm_100a, the C oracle,
    # and -- where /root/reference exists -- the reference build and the
    # native harnesses) instead of failing on the first library load.
    built = [os.path.join(ROOT, "paper_1809_09851_b200", "lib", "libfvb.so"),
             os.path.join(ROOT, "oracle", "build", "libfvb_oracle.so")]
    if not all(os.path.exists(p) for p in built):
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.reference()
    if r is None:
        pytest.skip("reference build oracle/_ref/libfvref.so not present")
    return r


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "gpu-marked test run without a CUDA device"
    import paper_1809_09851_b200 as fvb
    fvb.lib()  # raises if libfvb.so is missing: no fallback path exists
    return torch.device("cuda:0")

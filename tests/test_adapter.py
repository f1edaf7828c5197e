"""The drop-in through the reference's own C++ API: tests/native/
device_acceptance (the reference compiled as fvref + the product adapter
paper_1809_09851_b200/host/fusevec_device.cpp + libfvb.so)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "native", "build", "device_acceptance")


def run(mode):
    if not os.path.exists(BIN):
        pytest.skip("tests/native/build/device_acceptance not built (needs /root/reference "
                    "headers at build time; build() makes it)")
    p = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "[FAIL]" not in p.stdout
    return p.stdout


def test_reference_trees_resolve_to_fused_kernels():
    out = run("keys")
    assert out.count("[PASS]") == 10 and "11 trees" in out


@pytest.mark.gpu
def test_reference_api_on_device(cuda):
    out = run("gpu")
    assert out.count("[PASS]") == 12

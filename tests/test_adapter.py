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
    assert out.count("[PASS]") == 25


@pytest.mark.gpu
def test_reference_api_on_device_all_lowered(cuda, monkeypatch):
    # The same acceptance checks with every tree -- flux, conversions,
    # Jacobians -- run through the general NVRTC lowering instead of the
    # hand-written kernels: still bitwise against the reference engine.
    monkeypatch.setenv("FVB_FORCE_LOWER", "1")
    out = run("gpu")
    assert out.count("[PASS]") == 25


def test_adapter_compiles_in_the_references_own_namespace():
    # A maintainer compiles the adapter into fusevec itself,
    # i.e. without the test build's -Dfusevec=fvref rename.
    inc = "/root/reference/proj/include"
    if not os.path.isdir(inc):
        pytest.skip("reference headers not mounted")
    src = os.path.join(ROOT, "paper_1809_09851_b200", "host", "fusevec_device.cpp")
    p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", f"-I{inc}",
                        f"-I{ROOT}/include", f"-I{ROOT}/paper_1809_09851_b200/host",
                        "-I/usr/local/cuda/include", src], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr

"""The reference's own property suites (verify.cpp:81-400) grading the GPU
kernel through the reference's plugin hook, VerifyOptions::int_flash
(verify.hpp:15-24), via the C++ shim include/ifa_b200.hpp.

oracle/_ref/verify_gpu is built here by `make ref` (it needs the reference
headers) and travels to the GPU box with the snapshot; see
tests/cpp/verify_gpu.cpp for what it checks.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "verify_gpu")


@pytest.mark.gpu
def test_reference_verify_suites_accept_the_gpu_kernel():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/verify_gpu not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "verify_gpu: all passed" in r.stdout
    assert "mutant kernel rejected" in r.stdout


def test_verify_driver_links_the_product_library():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/verify_gpu not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libifa_b200.so" in out

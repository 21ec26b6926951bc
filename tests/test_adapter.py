"""The reference's own C++ API vs the drop-in adapter include/paro_b200.hpp
(tests/cpp/adapter_test.cpp, built by __graft_entry__.build() where the
reference headers exist; the binary travels to the GPU box)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "adapter_test")


def run(mode):
    if not os.path.exists(BIN):
        pytest.skip("adapter_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_adapter_host_stages():
    run("host")


@pytest.mark.gpu
def test_cpp_adapter_device_stages():
    run("gpu")

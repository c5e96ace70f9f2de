"""Runs the C++ drop-in parity binary (tests/cpp/test_shim.cpp) on the GPU box:
seqfm::b200::rank_forward_batch / dedup_segments vs the unmodified reference
linked into the same process."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "build", "test_shim")


@pytest.mark.gpu
def test_cpp_shim_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/test_shim not built (needs /root/reference headers: make -C tests/cpp)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout

"""The host thread pool used by the multi-GPU host path and the C++ shim (csrc/host_pool.hpp):
compiled with g++ and run on the CPU (no GPU involved)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_host_pool(tmp_path):
    exe = tmp_path / "test_pool"
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-o", str(exe), os.path.join(HERE, "cpp", "test_pool.cpp")],
                   check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout

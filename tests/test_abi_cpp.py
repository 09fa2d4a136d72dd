"""The reference's C++ KvShard interface over the ABI (include/sd_b200.hpp):
tests/abi_cpp/kvshard_test.cpp restates proj/tests/test_attention.cpp against
it — the same cases, inputs, bars and exception types — compiled with g++
as a C++ host of the reference would build it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2403_11421_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("abi_cpp") / "kvshard_test")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "abi_cpp", "kvshard_test.cpp"), "-L", PKG, "-lsd_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_cpp_interface_host_cases(exe):
    r = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_interface_reference_attention_cases(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout

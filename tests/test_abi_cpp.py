"""The reference's C++ interfaces over the ABI (include/sd_b200.hpp):
tests/abi_cpp/kvshard_test.cpp restates proj/tests/test_attention.cpp and
tests/abi_cpp/dense_test.cpp proj/tests/test_dense.cpp against it — the same
cases, inputs, bars and exception types — compiled with g++ as a C++ host of
the reference would build it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2403_11421_b200")


def _build(tmp_path_factory, name):
    out = str(tmp_path_factory.mktemp("abi_cpp") / name)
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "abi_cpp", name + ".cpp"), "-L", PKG, "-lsd_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    return _build(tmp_path_factory, "kvshard_test")


@pytest.fixture(scope="module")
def dense_exe(tmp_path_factory):
    return _build(tmp_path_factory, "dense_test")


def test_cpp_interface_host_cases(exe):
    r = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_interface_reference_attention_cases(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_interface_reference_dense_cases(dense_exe):
    """test_dense.cpp through the C++ interface: a projected row is bitwise
    batch-independent, argmax rescaling, batch-of-one decode equals the
    batched decode bitwise, and drive_schedule reproduces the golden
    transcript byte for byte."""
    golden = os.path.join(ROOT, "tests", "golden", "golden_transcript_2x64_3seq_20.csv")
    r = subprocess.run([dense_exe, golden], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.fixture(scope="module")
def dist_exe(tmp_path_factory):
    return _build(tmp_path_factory, "dist_test")


@pytest.mark.gpu
def test_cpp_interface_reference_distributed_cases(dist_exe):
    """test_workers.cpp:280-332 through the C++ interface: forked ranks on
    one device (by sequence with one or two S-ranks, by head, four-rank
    hybrid, two interleaved mini-batches, the stabilized schedule with
    retirement) produce the monolithic transcript row for row, and every
    shard is empty afterwards."""
    r = subprocess.run([dist_exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.fixture(scope="module")
def worker_exe(tmp_path_factory):
    return _build(tmp_path_factory, "worker_test")


@pytest.mark.gpu
def test_cpp_interface_attention_worker_session(worker_exe):
    """AttentionWorkerSession over SDWP through the C++ interface: HELLO,
    CONFIG, a first-token QKV_BATCH returning O == V bitwise (also fed one
    byte at a time), DROP_SEQ, SHUTDOWN stats, fatal bad magic."""
    r = subprocess.run([worker_exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout

"""The drop-in boundary from C: tests/abi_c/sd_abi_test.c, compiled with gcc
against include/sd_abi.h and linked with libsd_b200.so, as a non-Python
host would bind it. Host-only entry points run here; the GPU leg drives the
toy model through sd_drive and matches the golden transcript."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2403_11421_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("abi_c") / "sd_abi_test")
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "abi_c", "sd_abi_test.c"), "-L", PKG, "-lsd_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_c_host_entry_points(exe):
    r = subprocess.run([exe, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "sd_abi_test ok" in r.stdout


@pytest.mark.gpu
def test_c_end_to_end_golden_transcript(exe):
    golden = os.path.join(ROOT, "tests", "golden", "golden_transcript_2x64_3seq_20.csv")
    r = subprocess.run([exe, "gpu", golden], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr

"""H1: csrc/glibc_math.cuh restates glibc's __log_fma / __cos_fma
bit for bit on the RngStream::normal domain.  Host-side check against the
live libm (the device runs the same source; tests/test_gpu_mutate.py checks
device normals against the oracle)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_glibc_log_cos_normal_bit_exact(tmp_path):
    inc = os.path.join(ROOT, "paper_2504_08339_b200", "csrc", "libm_tables.inc")
    if not os.path.exists(inc):
        subprocess.run(["python", os.path.join(ROOT, "paper_2504_08339_b200", "gen_libm_tables.py")], check=True)
    exe = str(tmp_path / "tgm")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-mfma", "-I",
                    os.path.join(ROOT, "paper_2504_08339_b200", "csrc"), "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "test_glibc_math.cpp"), "-lm"], check=True)
    r = subprocess.run([exe, "2000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "log mismatches 0  cos mismatches 0  normal mismatches 0" in r.stdout

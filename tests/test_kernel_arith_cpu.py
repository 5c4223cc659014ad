"""Host builds of two pieces of the CUDA path's arithmetic, checked against their plain
definitions (no GPU needed):

* qf::quant_fast (csrc/qflash_quant_elem.cuh), the fast element quantizer of Eq. 2:
  wherever it does not defer to the exact path, sat8(result) == sat8(roundf(x / s))
  (readings R1, R2), over every float near each rounding boundary for 400 scales
  (tools/quant_fast_check.cpp, compiled with g++ and fmaf for __fmaf_rn);
* qf::udiv_small (csrc/qflash_params.cuh), the division behind the magic constants:
  equal to 64-bit '/' and '%' for every divisor 1..2^25 (tools/udiv_check.cu, host half;
  the device half runs in the GPU session).
"""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd, cwd=ROOT, timeout=300):
    return subprocess.run(cmd, cwd=cwd, capture_output=True, text=True, timeout=timeout)


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_quant_fast_matches_exact_definition(tmp_path):
    exe = str(tmp_path / "qfc")
    b = _run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "tools/quant_fast_check.cpp", "-o", exe])
    assert b.returncode == 0, b.stderr
    r = _run([exe])
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_udiv_small_exhaustive_host(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "udiv")
    b = _run([nvcc, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "tools/udiv_check.cu", "-o", exe])
    assert b.returncode == 0, b.stderr
    r = _run([exe])
    assert "host:   D in [1, 2^25], 9 numerators each: 0 mismatches" in r.stdout, r.stdout

"""The per-matrix C++ drop-in (include/kog2/kogsvd2_gpu.hpp) against the
reference library in one process: oracle/_ref/kog2_shim_test (built by
oracle/Makefile from tests/cpp/shim_test.cpp against the unmodified reference
headers, linked with libkog2.so) compares kogsvd2::gpu::{svd2, hypot_cr,
svd2_ext, metrics, generate, run_batch_any, csv_row} with kogsvd2::{...} on
2^20 config-1 matrices, targeted and any-finite matrices under every Options
value, and SURVEY.md Appendix B's run_batch rows (svd2.hpp:603-604,
kogsvd2.hpp:1-10, harness.hpp:226-321)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "kog2_shim_test")
APPENDIX_B_FIRST = ("double,gen,circ,0,1048576,0000000000c0ffee,kog,5.262556799095865e-16,4.469753940626907e-16,"
                    "5.475477442600766e-16,4.740088882553483e-16,4.726642799363624e-16,14512464.951216837")


def test_shim_header_is_self_contained_c_abi():
    """The shim only uses the C-ABI (no CUDA headers): it compiles here."""
    src = open(os.path.join(ROOT, "include", "kog2", "kogsvd2_gpu.hpp")).read()
    assert "cuda_runtime" not in src and '#include "../kog2.h"' in src


@pytest.mark.gpu
def test_cpp_shim_matches_reference(cuda):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/kog2_shim_test not built (needs the reference headers at build time)")
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=1800)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    assert "0 mismatches" in res.stdout
    assert APPENDIX_B_FIRST in res.stdout.splitlines()

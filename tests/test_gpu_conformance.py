"""GPU: the reference's OWN unit tests for the hot path
(/root/reference/proj/tests/test_projector.cpp and test_subspace_opt.cpp),
compiled unmodified against the B200 drop-in headers (include/lsp/*.hpp ->
include/lsp_b200/lsp.hpp) and liblsp_b200_cxx.so by oracle/Makefile
(`conformance` target, built where /root/reference exists; the binaries travel
in oracle/_ref/).  Every projector product, adam_step, fit and reproject_state
they exercise runs on the GPU in fp64 through the C-ABI."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINS = ["conformance_projector", "conformance_subspace_opt"]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", BINS)
def test_reference_unit_tests_pass_on_b200(cuda, name):
    path = os.path.join(ROOT, "oracle", "_ref", name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    res = subprocess.run([path], capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    summary = re.search(r"\[==========\] (\d+) tests, (\d+) failed", out)
    assert summary, out[-3000:]
    total, failed = int(summary.group(1)), int(summary.group(2))
    assert total >= 10
    assert res.returncode == 0 and failed == 0, out[-6000:]

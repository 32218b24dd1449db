import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


@pytest.hookimpl(tryfirst=True)  # before pytest-timeout reads its settings
def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblsp_b200.so")
    # a kernel that deadlocks (e.g. an mbarrier expecting bytes that never
    # arrive) must fail its test, not hang the whole run: per-test time limit
    # via pytest-timeout when no --timeout was given on the command line
    if config.pluginmanager.hasplugin("timeout") and not config.getoption("timeout", None):
        config.option.timeout = 600


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        meta = json.load(f)
    return data, meta


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def reference():
    import oracle

    if not oracle.available("reference"):
        pytest.skip("oracle/_ref/liblsp_ref.so not built")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2406_10181_b200 as lsp

    lsp.lib.load()  # fail loudly if the native library is missing
    return torch.device("cuda:0")

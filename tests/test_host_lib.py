"""CPU: the C-ABI library loads, exports every symbol include/lsp_b200.h declares,
and its host-side pieces (index generation, text I/O, argument validation) match
the reference.  No device compute here."""
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200._lib import EXPORTED

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINIT = 0x1A171


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lsp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(lsp_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    cdll = lsp.lib.raw
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(cdll, s), s
    # the Python binding covers the whole header
    assert syms == set(EXPORTED)


def test_version_and_device_count():
    assert lsp.lib.raw.lsp_version() == 1
    import ctypes as C

    c = C.c_int(-1)
    lsp.lib.device_count(C.byref(c))
    assert c.value >= 0


def test_init_sparse_bit_exact_vs_golden(golden):
    data, meta = golden
    i = 0
    while f"init{i}" in meta:
        c = meta[f"init{i}"]
        pos, val = lsp.init_sparse(c["n_rows"], c["d"], c["r"], c["seed"])
        assert sha(pos) == c["pos_sha"] and sha(val) == c["val_sha"], f"init{i}"
        i += 1


def test_derive_seed(golden):
    _, meta = golden
    for s, t, i, want in meta["derive_seed"]:
        assert lsp.derive_seed(s, t, i) == want


def test_init_sparse_rejects_bad_args():
    with pytest.raises(lsp.InvalidArgument):
        lsp.init_sparse(4, 3, 4, 0)
    with pytest.raises(lsp.InvalidArgument):
        lsp.init_sparse(4, 3, 0, 0)


def test_identity_pattern():
    pos, val = lsp.identity_pattern(5)
    np.testing.assert_array_equal(pos, np.arange(5))
    np.testing.assert_array_equal(val, np.ones(5))


def test_save_projector_matches_reference_text(golden):
    _, meta = golden
    pos, val = lsp.init_sparse(5, 7, 3, 113)
    assert lsp.save_projector(5, 7, 3, pos, val) == meta["save_projector"]


def test_load_projector_round_trip_and_errors():
    pos, val = lsp.init_sparse(7, 9, 3, 113)
    text = lsp.save_projector(7, 9, 3, pos, val)
    nr, d, r, p2, v2 = lsp.load_projector(text)
    assert (nr, d, r) == (7, 9, 3)
    np.testing.assert_array_equal(p2, pos)
    np.testing.assert_array_equal(v2, val)  # shortest round-trip: exact
    for bad in ("3 2", "2 4 2\n0 9 1 1\n0 1 1 1\n", "2 4 2\n1 0 1 1\n0 1 1 1\n",
                "2 4 2\n0 1 nan 1\n0 1 1 1\n"):
        with pytest.raises(lsp.IoError):
            lsp.load_projector(bad)


def test_subsample_size(golden):
    _, meta = golden
    for g_, b_, m_, n_, t_, dl, want in meta["subsample_size"]:
        assert lsp.subsample_size(g_, b_, m_, n_, t_, dl) == want
    with pytest.raises(lsp.InvalidArgument):
        lsp.subsample_size(0.0, 0.5, 4, 4, 10, 0.1)


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    pos, val = lsp.init_sparse(8, 4, 2, 1)
    with pytest.raises(lsp.CudaError):
        lsp.DeviceProjector(8, 4, 2, pos, val)


def test_schedule_rejects_bad_args():
    """lsp_schedule_create validates its arguments before touching the device
    (InvalidArgument, like the reference's std::invalid_argument)."""
    import ctypes as C

    h = C.c_void_p()
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.schedule_create(0, None, None, C.byref(h))
    arr = (C.c_void_p * 2)(None, None)
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.schedule_create(2, arr, None, C.byref(h))
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.schedule_step(None, 1e-3, None)
    lsp.lib.schedule_destroy(None)  # a null handle is a no-op


def test_schedule_set_pipeline_rejects_bad_args():
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.schedule_set_pipeline(None, 1)


def test_schedule_set_partition_rejects_bad_args():
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.schedule_set_partition(None, 64, None, None)


def test_layer_fused_entries_reject_null_layer():
    """lsp_layer_compress_adam / _compress_finish_adam (stage 2 with Adam fused)
    check their handle before touching the device."""
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.layer_compress_adam(None, None)
    with pytest.raises(lsp.InvalidArgument):
        lsp.lib.layer_compress_finish_adam(None, None)

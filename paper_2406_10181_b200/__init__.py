"""B200-native LSP-Offload (d,r)-sparse projector path.

Python mirror of the reference's hot-path API (lspkit `lsp_core`,
/root/reference/proj/include/lsp/{projector,subspace_opt}.hpp) over the C-ABI
library ``liblsp_b200.so`` (include/lsp_b200.h).  Device memory, streams and
torch.distributed come from PyTorch; every computation on the path is one of
our sm_100a kernels.  There is no CPU fallback: importing works without a GPU
(host-side index generation and text I/O only), but every device call raises
when the CUDA library or the device is missing.

Naming follows the reference: ``d`` = subspace width, ``r`` = nonzeros per
projector row (BASELINE.json swaps the letters).
"""
from __future__ import annotations

from ._lib import (  # noqa: F401
    CudaError,
    InvalidArgument,
    IoError,
    LspError,
    NcclError,
    NumericError,
    Layout,
    lib,
    library_path,
    launch_count,
    set_sm_budget,
)
from .projector import (  # noqa: F401
    AdamState,
    Comm,
    DevicePair,
    DeviceProjector,
    FitConfig,
    FitReport,
    Layer,
    Schedule,
    derive_seed,
    identity_pattern,
    init_sparse,
    load_projector,
    nccl_version,
    projector_gram,
    maybe_update,
    reproject_state,
    save_projector,
    step,
    subsample_size,
    update,
)

__all__ = [
    "AdamState", "Comm", "nccl_version", "NcclError", "DevicePair", "Layer", "Schedule", "DeviceProjector", "FitConfig", "FitReport", "derive_seed",
    "identity_pattern", "init_sparse", "load_projector", "projector_gram", "reproject_state", "maybe_update",
    "save_projector", "step", "subsample_size", "update", "LspError", "InvalidArgument",
    "NumericError", "IoError", "CudaError", "Layout", "lib", "library_path", "launch_count", "set_sm_budget",
]

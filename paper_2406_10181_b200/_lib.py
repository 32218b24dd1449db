"""ctypes binding of include/lsp_b200.h (the C-ABI of liblsp_b200.so)."""
from __future__ import annotations

import ctypes as C
import enum
import os

HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(HERE, "liblsp_b200.so")


class LspError(RuntimeError):
    """Base error; ``code`` is the lsp_status."""

    code = -1


class InvalidArgument(LspError, ValueError):
    """std::invalid_argument in the reference (LSP_EINVAL)."""

    code = 1


class NumericError(LspError):
    """lsp::NumericError (LSP_ENUMERIC)."""

    code = 2


class IoError(LspError):
    """lsp::IoError (LSP_EIO)."""

    code = 3


class CudaError(LspError):
    """CUDA runtime failure, incl. missing device (LSP_ECUDA / LSP_ENOMEM)."""

    code = 4


class NcclError(LspError):
    """NCCL missing or failed (LSP_ENCCL)."""

    code = 6


_ERRORS = {1: InvalidArgument, 2: NumericError, 3: IoError, 4: CudaError, 5: CudaError,
           6: NcclError}


class DType(enum.IntEnum):
    F64 = 0
    F32 = 1
    BF16 = 2


class Layout(enum.IntEnum):
    ROW = 0  # reference layout S[a][b] at a*d + b
    T = 1    # transposed, the fused device path's internal layout


class FitConfigC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("reg_beta", C.c_double), ("step_size", C.c_double),
                ("max_steps", C.c_int), ("timeout_steps", C.c_int), ("seed", C.c_uint64),
                ("reg_kind", C.c_int)]


class FitReportC(C.Structure):
    _fields_ = [("final_rel_bias", C.c_double), ("success", C.c_int), ("timed_out", C.c_int),
                ("stalled", C.c_int), ("steps", C.c_int), ("n_loss", C.c_int)]


_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_d = C.c_double
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)

_SIGS = {
    "lsp_last_error": (C.c_char_p, []),
    "lsp_version": (_i, []),
    "lsp_device_count": (_i, [_ip]),
    "lsp_launch_count": (C.c_uint64, []),
    "lsp_set_sm_budget": (_i, [_i, _i]),
    "lsp_fit_config_default": (FitConfigC, []),
    "lsp_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "lsp_init_sparse": (_i, [_i, _i, _i, C.c_uint64, _i32p, _dp]),
    "lsp_identity_pattern": (_i, [_i, _i32p, _dp]),
    "lsp_save_projector": (_i, [_i, _i, _i, _i32p, _dp, C.c_char_p, _i64, C.POINTER(_i64)]),
    "lsp_load_projector": (_i, [C.c_char_p, _i64, _ip, _ip, _ip, _i32p, _dp]),
    "lsp_subsample_size": (_i, [_d, _d, _i, _i, _i, _d, C.POINTER(_i64)]),
    "lsp_projector_create": (_i, [_i, _i, _i, _i32p, _dp, _i, C.POINTER(_vp)]),
    "lsp_projector_set_values": (_i, [_vp, _dp]),
    "lsp_projector_get": (_i, [_vp, _i32p, _dp]),
    "lsp_projector_shape": (_i, [_vp, _ip, _ip, _ip]),
    "lsp_projector_destroy": (_i, [_vp]),
    "lsp_projector_mul": (_i, [_vp, _i, _i, _vp, _i64, _vp, _i64, _vp]),
    "lsp_pair_create": (_i, [_vp, _vp, C.POINTER(_vp)]),
    "lsp_pair_destroy": (_i, [_vp]),
    "lsp_compress": (_i, [_vp, _vp, _i64, _i, _vp, _i, _vp]),
    "lsp_decompress": (_i, [_vp, _vp, _i, _vp, _i64, _i, _vp]),
    "lsp_decompress_apply": (_i, [_vp, _vp, _i, _d, _vp, _i64, _i, _vp]),
    "lsp_estimation_bias": (_i, [_vp, _vp, _i64, _i, _vp, _i64, _vp]),
    "lsp_relative_bias": (_i, [_vp, _vp, _i64, _i, _dp, _vp]),
    "lsp_adam_create": (_i, [_i, _i, _d, _d, _d, _i, _i, C.POINTER(_vp)]),
    "lsp_adam_destroy": (_i, [_vp]),
    "lsp_adam_step": (_i, [_vp, _vp, _vp, _vp]),
    "lsp_adam_check": (_i, [_vp, _vp]),
    "lsp_adam_get": (_i, [_vp, _dp, _dp, C.POINTER(_i64), _i]),
    "lsp_adam_set": (_i, [_vp, _dp, _dp, _i64, _i]),
    "lsp_adam_info": (_i, [_vp, _ip, _ip, _dp, _dp, _dp]),
    "lsp_step": (_i, [_vp, _vp, _vp, _i64, _i, _vp, _i64, _i, _d, _vp, _vp]),
    "lsp_update": (_i, [_vp, _vp, _vp, _vp, _i64, _i, _d, _vp]),
    "lsp_layer_create": (_i, [_i, C.POINTER(_vp), _d, _d, _d, C.POINTER(_vp)]),
    "lsp_layer_destroy": (_i, [_vp]),
    "lsp_layer_bind": (_i, [_vp, _i, _vp, _i64, _i, _vp, _i64, _i]),
    "lsp_layer_s_buffer": (_i, [_vp, C.POINTER(_vp), C.POINTER(_i64)]),
    "lsp_layer_compress": (_i, [_vp, _vp]),
    "lsp_layer_compress_prepare": (_i, [_vp, _vp]),
    "lsp_layer_compress_finish": (_i, [_vp, _vp]),
    "lsp_layer_compress_adam": (_i, [_vp, _vp]),
    "lsp_layer_compress_finish_adam": (_i, [_vp, _vp]),
    "lsp_layer_update": (_i, [_vp, _d, _i, _vp]),
    "lsp_layer_adam": (_i, [_vp, _i, _vp]),
    "lsp_maybe_update": (_i, [_vp, _vp, _vp, C.c_int64, _i, _vp, _i, _i, _d, _vp, _i,
                              C.c_uint64, _vp, _vp, _vp, _vp, _vp]),
    "lsp_layer_apply": (_i, [_vp, _d, _vp]),
    "lsp_layer_apply_prepare": (_i, [_vp, _vp]),
    "lsp_layer_apply_finish": (_i, [_vp, _d, _vp]),
    "lsp_layer_step": (_i, [_vp, _d, _vp]),
    "lsp_layer_check": (_i, [_vp, _vp]),
    "lsp_layer_adam_get": (_i, [_vp, _i, _dp, _dp, C.POINTER(_i64), _i]),
    "lsp_fit_loss": (_i, [_vp, C.POINTER(_vp), _i, _i64, _i, C.POINTER(FitConfigC), _dp, _vp]),
    "lsp_fit_gradient": (_i, [_vp, C.POINTER(_vp), _i, _i64, _i, C.POINTER(FitConfigC), _dp,
                              _dp, _vp]),
    "lsp_fit": (_i, [_vp, C.POINTER(_vp), _i, _i64, _i, C.POINTER(FitConfigC),
                     C.POINTER(FitReportC), _dp, _i, _vp]),
    "lsp_projector_gram": (_i, [_vp, _vp, _vp, _vp]),
    "lsp_comm_unique_id": (_i, [_vp]),
    "lsp_comm_init": (_i, [_vp, _i, _i, C.POINTER(_vp)]),
    "lsp_comm_destroy": (_i, [_vp]),
    "lsp_comm_size": (_i, [_vp, _ip, _ip]),
    "lsp_nccl_version": (_i, [_ip]),
    "lsp_allreduce_mean": (_i, [_vp, _vp, _i64, _i, _vp]),
    "lsp_layer_allreduce": (_i, [_vp, _vp, _vp]),
    "lsp_reproject_state": (_i, [_vp, _vp, _vp, _i, _vp]),
    "lsp_schedule_create": (_i, [_i, C.POINTER(_vp), _vp, C.POINTER(_vp)]),
    "lsp_schedule_set_backward": (_i, [_vp, _vp, _vp]),
    "lsp_schedule_set_pipeline": (_i, [_vp, _i]),
    "lsp_schedule_set_partition": (_i, [_vp, _i, C.POINTER(_i), C.POINTER(_i)]),
    "lsp_schedule_step": (_i, [_vp, _d, _vp]),
    "lsp_schedule_destroy": (_i, [_vp]),
}

EXPORTED = tuple(_SIGS)


class _Lib:
    """Lazily loaded library; attribute access returns checked callables."""

    def __init__(self):
        self._cdll = None

    def load(self) -> C.CDLL:
        if self._cdll is None:
            if not os.path.exists(library_path):
                raise ImportError(
                    f"{library_path} is not built; run `python -c \"import __graft_entry__ as g; "
                    "g.build()\"` (nvcc, sm_100a)")
            cdll = C.CDLL(library_path, mode=C.RTLD_LOCAL)
            for name, (res, args) in _SIGS.items():
                fn = getattr(cdll, name)
                fn.restype = res
                fn.argtypes = args
            self._cdll = cdll
        return self._cdll

    @property
    def raw(self) -> C.CDLL:
        return self.load()

    def __getattr__(self, name):
        cdll = self.load()
        fn = getattr(cdll, "lsp_" + name)
        if fn.restype is not _i:
            return fn

        def call(*args):
            rc = fn(*args)
            if rc != 0:
                msg = cdll.lsp_last_error().decode(errors="replace")
                raise _ERRORS.get(rc, LspError)(msg)
            return rc

        call.__name__ = name
        return call


lib = _Lib()


def set_sm_budget(compress_sms: int = 0, update_sms: int = 0) -> None:
    """Cap the SMs the persistent compress / update grids size for (0 = all);
    see lsp_set_sm_budget in include/lsp_b200.h."""
    lib.set_sm_budget(int(compress_sms), int(update_sms))


def launch_count() -> int:
    """Kernels launched by liblsp_b200 in this process."""
    return int(lib.raw.lsp_launch_count())

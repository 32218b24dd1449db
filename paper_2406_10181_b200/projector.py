"""Reference-shaped Python API over the C-ABI (device tensors are torch CUDA tensors).

Each function/class names the reference interface it mirrors:
  init_sparse / identity_pattern / save_projector / load_projector
                                  proj/include/lsp/projector.hpp:62-97
  DevicePair.compress / decompress / estimation_bias / relative_bias / fit*
                                  proj/include/lsp/projector.hpp:76-94
  AdamState                       proj/include/lsp/subspace_opt.hpp:17-37
  projector_gram / reproject_state
                                  proj/include/lsp/subspace_opt.hpp:47-53
  step / update                   the per-layer loop body, proj/src/trainer.cpp:187-190
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import DType, FitConfigC, FitReportC, InvalidArgument, Layout, lib

_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)


def _np_i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _np_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------------------
# torch interop (lazy import: host-only helpers do not need torch)
# ---------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _dtype_of(t) -> DType:
    torch = _torch()
    m = {torch.float64: DType.F64, torch.float32: DType.F32, torch.bfloat16: DType.BF16}
    if t.dtype not in m:
        raise InvalidArgument(f"unsupported dtype {t.dtype}")
    return m[t.dtype]


def _torch_dtype(dt: DType):
    torch = _torch()
    return {DType.F64: torch.float64, DType.F32: torch.float32, DType.BF16: torch.bfloat16}[dt]


def _check_dev(t, name: str, rows: Optional[int] = None, cols: Optional[int] = None):
    if not t.is_cuda:
        raise InvalidArgument(f"{name}: expected a CUDA tensor")
    if t.dim() != 2 or t.stride(1) != 1:
        raise InvalidArgument(f"{name}: expected a 2-D row-major tensor")
    if rows is not None and t.shape[0] != rows or cols is not None and t.shape[1] != cols:
        raise InvalidArgument(f"{name}: dims do not match pair ({tuple(t.shape)})")
    return t.data_ptr(), t.stride(0)


def _stream(stream):
    if stream is None:
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _compute(c) -> DType:
    if isinstance(c, DType):
        return c
    return {"f32": DType.F32, "f64": DType.F64, "float32": DType.F32,
            "float64": DType.F64}[str(c)]


# ---------------------------------------------------------------------------
# host side
# ---------------------------------------------------------------------------
def derive_seed(master: int, tag: int, index: int = 0) -> int:
    """proj/include/lsp/common.hpp:42-45"""
    return int(lib.raw.lsp_derive_seed(master, tag, index))


def init_sparse(n_rows: int, d: int, r: int, seed: int):
    """proj/src/projector.cpp:66-85 (bit-exact).  Returns (positions int32, values f64)."""
    n = max(n_rows * r, 1) if n_rows > 0 and r > 0 else 1
    pos = np.zeros(n, np.int32)
    val = np.zeros(n, np.float64)
    lib.init_sparse(n_rows, d, r, seed, _ip(pos), _dptr(val))
    return pos, val


def identity_pattern(n_rows: int):
    """proj/src/projector.cpp:87-96: d = n_rows, r = 1, value 1."""
    pos = np.zeros(max(n_rows, 1), np.int32)
    val = np.zeros(max(n_rows, 1), np.float64)
    lib.identity_pattern(n_rows, _ip(pos), _dptr(val))
    return pos, val


def save_projector(n_rows: int, d: int, r: int, pos, val) -> str:
    """proj/src/projector.cpp:317-327"""
    pos, val = _np_i32(pos), _np_f64(val)
    need = C.c_int64()
    lib.save_projector(n_rows, d, r, _ip(pos), _dptr(val), None, 0, C.byref(need))
    buf = C.create_string_buffer(int(need.value))
    lib.save_projector(n_rows, d, r, _ip(pos), _dptr(val), buf, need.value, C.byref(need))
    return buf.value.decode()


def load_projector(text: str):
    """proj/src/projector.cpp:329-354 -> (n_rows, d, r, positions, values); IoError if malformed."""
    b = text.encode()
    nr, d, r = C.c_int(), C.c_int(), C.c_int()
    lib.load_projector(b, len(b), C.byref(nr), C.byref(d), C.byref(r), None, None)
    pos = np.zeros(nr.value * r.value, np.int32)
    val = np.zeros(nr.value * r.value, np.float64)
    lib.load_projector(b, len(b), C.byref(nr), C.byref(d), C.byref(r), _ip(pos), _dptr(val))
    return nr.value, d.value, r.value, pos, val


def subsample_size(gamma_bound, chernoff_beta, m, n, total_steps, delta) -> int:
    """proj/src/trainer.cpp:60-72"""
    out = C.c_int64()
    lib.subsample_size(gamma_bound, chernoff_beta, m, n, total_steps, delta, C.byref(out))
    return out.value


# ---------------------------------------------------------------------------
# device projector / pair
# ---------------------------------------------------------------------------
class DeviceProjector:
    """Device-resident SparseProjector (CSR + CSC), projector.hpp:18-30."""

    def __init__(self, n_rows: int, d: int, r: int, pos, val, compute="f32"):
        self.n_rows, self.d, self.r = n_rows, d, r
        self.compute = _compute(compute)
        pos, val = _np_i32(pos), _np_f64(val)
        if pos.size < n_rows * r or val.size < n_rows * r:
            raise InvalidArgument("projector: arrays shorter than n_rows * r")
        h = C.c_void_p()
        lib.projector_create(n_rows, d, r, _ip(pos), _dptr(val), int(self.compute), C.byref(h))
        self._h = h

    @classmethod
    def _adopt(cls, handle, compute):
        """Wrap a projector handle created by the library (takes ownership)."""
        obj = cls.__new__(cls)
        n_rows, d, r = C.c_int(), C.c_int(), C.c_int()
        lib.projector_shape(handle, C.byref(n_rows), C.byref(d), C.byref(r))
        obj.n_rows, obj.d, obj.r = n_rows.value, d.value, r.value
        obj.compute = compute
        obj._h = handle
        return obj

    @classmethod
    def random(cls, n_rows: int, d: int, r: int, seed: int, compute="f32"):
        pos, val = init_sparse(n_rows, d, r, seed)
        return cls(n_rows, d, r, pos, val, compute)

    @property
    def handle(self):
        return self._h

    def get(self):
        pos = np.zeros(self.n_rows * self.r, np.int32)
        val = np.zeros(self.n_rows * self.r, np.float64)
        lib.projector_get(self._h, _ip(pos), _dptr(val))
        return pos, val

    def set_values(self, val):
        val = _np_f64(val)
        if val.size < self.n_rows * self.r:
            raise InvalidArgument("projector set_values: array shorter than n_rows * r")
        lib.projector_set_values(self._h, _dptr(val))

    def close(self):
        if getattr(self, "_h", None):
            lib.projector_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class FitConfig:
    """proj/include/lsp/projector.hpp:43-51"""

    alpha: float = 0.1
    reg_beta: float = 0.0
    step_size: float = 1e-2
    max_steps: int = 500
    timeout_steps: int = 500
    seed: int = 0
    reg_kind: int = 0  # 0 squared, 1 unsquared

    def c(self) -> FitConfigC:
        return FitConfigC(self.alpha, self.reg_beta, self.step_size, self.max_steps,
                          self.timeout_steps, self.seed, self.reg_kind)


@dataclass
class FitReport:
    """proj/include/lsp/projector.hpp:53-60"""

    loss_curve: list = field(default_factory=list)
    final_rel_bias: float = 0.0
    success: bool = False
    timed_out: bool = False
    stalled: bool = False
    steps: int = 0


class DevicePair:
    """ProjectorPair (projector.hpp:32-36) with its device workspace."""

    def __init__(self, p: DeviceProjector, q: DeviceProjector, handle=None):
        h = handle
        if h is None:
            h = C.c_void_p()
            lib.pair_create(p.handle, q.handle, C.byref(h))
        self._h, self.p, self.q = h, p, q
        self.m, self.n, self.d = p.n_rows, q.n_rows, p.d
        self.compute = p.compute

    @property
    def handle(self):
        return self._h

    def _sd(self):
        return _torch_dtype(self.compute)

    def compress(self, g, out=None, layout=Layout.ROW, stream=None):
        """S = P^T G Q (projector.cpp:163-168)."""
        torch = _torch()
        gp, ldg = _check_dev(g, "compress: g", self.m, self.n)
        if out is None:
            out = torch.empty(self.d, self.d, dtype=self._sd(), device=g.device)
        else:
            _check_dev(out, "compress: out", self.d, self.d)
            if out.dtype != self._sd() or not out.is_contiguous():
                raise InvalidArgument("compress: out must be a contiguous d x d tensor of the "
                                      "pair's compute dtype")
        lib.compress(self._h, C.c_void_p(gp), ldg, int(_dtype_of(g)), C.c_void_p(out.data_ptr()),
                     int(layout), _stream(stream))
        return out

    def decompress(self, s, out=None, dtype=None, layout=Layout.ROW, stream=None):
        """P S Q^T (projector.cpp:170-175)."""
        torch = _torch()
        _check_dev(s, "decompress: s", self.d, self.d)
        if out is None:
            out = torch.empty(self.m, self.n, dtype=dtype or self._sd(), device=s.device)
        op, ldo = _check_dev(out, "decompress: out", self.m, self.n)
        lib.decompress(self._h, C.c_void_p(s.data_ptr()), int(layout), C.c_void_p(op), ldo,
                       int(_dtype_of(out)), _stream(stream))
        return out

    def decompress_apply(self, delta, lr: float, w, layout=Layout.ROW, stream=None):
        """w -= lr * P delta Q^T in one pass (trainer.cpp:190)."""
        _check_dev(delta, "decompress_apply: delta", self.d, self.d)
        wp, ldw = _check_dev(w, "decompress_apply: w", self.m, self.n)
        lib.decompress_apply(self._h, C.c_void_p(delta.data_ptr()), int(layout), float(lr),
                             C.c_void_p(wp), ldw, int(_dtype_of(w)), _stream(stream))
        return w

    def estimation_bias(self, sigma, out=None, stream=None):
        """P P^T sigma Q Q^T - sigma (projector.cpp:177-181)."""
        torch = _torch()
        sp, lds = _check_dev(sigma, "estimation_bias: sigma", self.m, self.n)
        if out is None:
            out = torch.empty_like(sigma)
        op, ldo = _check_dev(out, "estimation_bias: out", self.m, self.n)
        if out.dtype != sigma.dtype:
            raise InvalidArgument("estimation_bias: out dtype must match sigma")
        lib.estimation_bias(self._h, C.c_void_p(sp), lds, int(_dtype_of(sigma)), C.c_void_p(op),
                            ldo, _stream(stream))
        return out

    def relative_bias(self, sigma, stream=None) -> float:
        """|b(sigma)|_F / |sigma|_F (projector.cpp:183-187); synchronous."""
        sp, lds = _check_dev(sigma, "relative_bias: sigma", self.m, self.n)
        out = C.c_double()
        lib.relative_bias(self._h, C.c_void_p(sp), lds, int(_dtype_of(sigma)), C.byref(out),
                          _stream(stream))
        return out.value

    def _targets(self, targets: Sequence):
        if len(targets) == 0:
            return (C.c_void_p * 1)(), 0, self.n, DType.F64
        dt = _dtype_of(targets[0])
        ld = None
        for t in targets:
            _, l = _check_dev(t, "fit: target", self.m, self.n)
            if _dtype_of(t) != dt or (ld is not None and l != ld):
                raise InvalidArgument("fit: targets must share dtype and leading dimension")
            ld = l
        arr = (C.c_void_p * len(targets))(*[t.data_ptr() for t in targets])
        return arr, len(targets), ld, dt

    def fit_loss(self, targets, cfg: Optional[FitConfig] = None, stream=None) -> float:
        arr, t, ld, dt = self._targets(targets)
        out = C.c_double()
        c = (cfg or FitConfig()).c()
        lib.fit_loss(self._h, arr, t, ld, int(dt), C.byref(c), C.byref(out), _stream(stream))
        return out.value

    def fit_gradient(self, targets, cfg: Optional[FitConfig] = None, stream=None):
        arr, t, ld, dt = self._targets(targets)
        gp = np.zeros(self.m * self.p.r)
        gq = np.zeros(self.n * self.q.r)
        c = (cfg or FitConfig()).c()
        lib.fit_gradient(self._h, arr, t, ld, int(dt), C.byref(c), _dptr(gp), _dptr(gq),
                         _stream(stream))
        return gp, gq

    def fit(self, targets, cfg: Optional[FitConfig] = None, max_curve: int = 4096,
            stream=None) -> FitReport:
        """projector.cpp:253-315; updates this pair's projector values in place."""
        arr, t, ld, dt = self._targets(targets)
        rep = FitReportC()
        curve = np.zeros(max_curve)
        c = (cfg or FitConfig()).c()
        lib.fit(self._h, arr, t, ld, int(dt), C.byref(c), C.byref(rep), _dptr(curve), max_curve,
                _stream(stream))
        return FitReport(loss_curve=list(curve[: min(rep.n_loss, max_curve)]),
                         final_rel_bias=rep.final_rel_bias, success=bool(rep.success),
                         timed_out=bool(rep.timed_out), stalled=bool(rep.stalled),
                         steps=rep.steps)

    def close(self):
        if getattr(self, "_h", None):
            lib.pair_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AdamState:
    """SubspaceOptState + adam_step (subspace_opt.hpp:17-37), device resident."""

    def __init__(self, rows: int, cols: Optional[int] = None, beta1=0.9, beta2=0.999, eps=1e-8,
                 compute="f32", layout=Layout.T):
        cols = rows if cols is None else cols
        self.rows, self.cols = rows, cols
        self.compute = _compute(compute)
        self.layout = Layout(layout)
        h = C.c_void_p()
        lib.adam_create(rows, cols, beta1, beta2, eps, int(self.compute), int(self.layout),
                        C.byref(h))
        self._h = h

    @property
    def handle(self):
        return self._h

    def step(self, grad, delta=None, stream=None):
        """adam_step: moments updated in place; returns delta (no lr)."""
        torch = _torch()
        _check_dev(grad, "adam_step: grad", self.rows, self.cols)
        if delta is None:
            delta = torch.empty_like(grad)
        lib.adam_step(self._h, C.c_void_p(grad.data_ptr()), C.c_void_p(delta.data_ptr()),
                      _stream(stream))
        return delta

    def check(self, stream=None):
        """Raises NumericError if a non-finite gradient was seen (synchronous)."""
        lib.adam_check(self._h, _stream(stream))

    def get(self, layout=Layout.ROW):
        m = np.zeros(self.rows * self.cols)
        v = np.zeros(self.rows * self.cols)
        st = C.c_int64()
        lib.adam_get(self._h, _dptr(m), _dptr(v), C.byref(st), int(layout))
        shape = (self.rows, self.cols) if layout == Layout.ROW else (self.cols, self.rows)
        return m.reshape(shape), v.reshape(shape), st.value

    def set(self, m, v, step: int, layout=Layout.ROW):
        m, v = _np_f64(m).ravel(), _np_f64(v).ravel()
        lib.adam_set(self._h, _dptr(m), _dptr(v), int(step), int(layout))

    def close(self):
        if getattr(self, "_h", None):
            lib.adam_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Layer:
    """Per-layer schedule unit: the matrices of one block stepped together with one
    grouped launch per stage (the body of proj/src/trainer.cpp:186-198).

    The layer owns contiguous S^T / delta^T buffers and all Adam moments, so a
    data-parallel caller all-reduces ``s_buffer()`` once between ``compress()``
    and ``update()``.
    """

    def __init__(self, pairs: Sequence[DevicePair], beta1=0.9, beta2=0.999, eps=1e-8):
        self.pairs = list(pairs)
        arr = (C.c_void_p * len(self.pairs))(*[p.handle for p in self.pairs])
        h = C.c_void_p()
        lib.layer_create(len(self.pairs), arr, beta1, beta2, eps, C.byref(h))
        self._h = h
        self.d = self.pairs[0].d
        self._bound = [None] * len(self.pairs)
        self._s_view = None

    @property
    def handle(self):
        return self._h

    def bind(self, idx: int, g, w):
        pr = self.pairs[idx]
        gp, ldg = _check_dev(g, "layer_bind: g", pr.m, pr.n)
        wp, ldw = _check_dev(w, "layer_bind: w", pr.m, pr.n)
        lib.layer_bind(self._h, idx, C.c_void_p(gp), ldg, int(_dtype_of(g)), C.c_void_p(wp),
                       ldw, int(_dtype_of(w)))
        self._bound[idx] = (g, w)  # keep the tensors alive

    def allreduce(self, comm, stream=None):
        """Mean of the layer's S^T buffer over the ranks of ``comm`` (NCCL, on
        ``stream``), then a finiteness re-check so every rank latches the flag
        together (lsp_layer_allreduce)."""
        lib.layer_allreduce(self._h, comm.handle, _stream(stream))

    def s_buffer(self):
        """torch view of the layer's S^T buffer [count, d, d] (device memory owned by the layer)."""
        if self._s_view is None:
            torch = _torch()
            ptr = C.c_void_p()
            cnt = C.c_int64()
            lib.layer_s_buffer(self._h, C.byref(ptr), C.byref(cnt))
            dt = _torch_dtype(self.pairs[0].compute)
            self._s_view = _device_view(ptr.value, int(cnt.value), dt).view(
                len(self.pairs), self.d, self.d)
        return self._s_view

    def compress(self, stream=None):
        lib.layer_compress(self._h, _stream(stream))

    def compress_prepare(self, stream=None):
        """First half of compress(): stage 1 (Z^T = G^T P, the pass over G)."""
        lib.layer_compress_prepare(self._h, _stream(stream))

    def compress_finish(self, stream=None):
        """Second half of compress(): stage 2 (S^T = Q^T Z^T) and the non-finite latch."""
        lib.layer_compress_finish(self._h, _stream(stream))

    def compress_adam(self, stream=None):
        """compress() + adam() for a single rank (no S exchange in between): Adam
        runs in the stage-2 epilogue (lsp_layer_compress_adam), bitwise the
        unfused pair."""
        lib.layer_compress_adam(self._h, _stream(stream))

    def compress_finish_adam(self, stream=None):
        """compress_finish() + adam() in one launch (lsp_layer_compress_finish_adam)."""
        lib.layer_compress_finish_adam(self._h, _stream(stream))

    def update(self, lr: float, check_finite: bool = False, stream=None):
        lib.layer_update(self._h, float(lr), int(bool(check_finite)), _stream(stream))

    def adam(self, check_finite: bool = False, stream=None):
        lib.layer_adam(self._h, int(bool(check_finite)), _stream(stream))

    def apply(self, lr: float, stream=None):
        lib.layer_apply(self._h, float(lr), _stream(stream))

    def apply_prepare(self, stream=None):
        """First half of apply(): enqueue the Y = delta Q^T build (no-op for groups
        the Y path does not cover)."""
        lib.layer_apply_prepare(self._h, _stream(stream))

    def apply_finish(self, lr: float, stream=None):
        """Second half of apply(): the streaming W update (the whole apply if
        apply_prepare enqueued nothing)."""
        lib.layer_apply_finish(self._h, float(lr), _stream(stream))

    def step(self, lr: float, stream=None):
        lib.layer_step(self._h, float(lr), _stream(stream))

    def check(self, stream=None):
        lib.layer_check(self._h, _stream(stream))

    def adam_get(self, idx: int, layout=Layout.ROW):
        d = self.d
        m = np.zeros(d * d)
        v = np.zeros(d * d)
        st = C.c_int64()
        lib.layer_adam_get(self._h, idx, _dptr(m), _dptr(v), C.byref(st), int(layout))
        return m.reshape(d, d), v.reshape(d, d), st.value

    def close(self):
        if getattr(self, "_h", None):
            lib.layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr: int, numel: int, dtype):
    """A torch tensor aliasing library-owned device memory (no copy, no ownership)."""
    torch = _torch()
    if dtype not in (torch.float32, torch.float64):
        raise InvalidArgument("only fp32/fp64 compute buffers are exposed")

    class _Holder:
        pass

    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (numel,),
                                  "typestr": "<f4" if dtype == torch.float32 else "<f8",
                                  "data": (ptr, False), "version": 3}
    return torch.as_tensor(h, device="cuda")


def step(pair: DevicePair, adam: AdamState, g, w, lr: float, s_out=None, stream=None):
    """compress -> Adam -> decompress-and-apply for one matrix (trainer.cpp:187-190)."""
    gp, ldg = _check_dev(g, "step: g", pair.m, pair.n)
    wp, ldw = _check_dev(w, "step: w", pair.m, pair.n)
    sp = C.c_void_p(s_out.data_ptr()) if s_out is not None else None
    lib.step(pair.handle, adam.handle, C.c_void_p(gp), ldg, int(_dtype_of(g)), C.c_void_p(wp),
             ldw, int(_dtype_of(w)), float(lr), sp, _stream(stream))
    return w


def update(pair: DevicePair, adam: AdamState, s_t, w, lr: float, stream=None):
    """Adam + decompress-and-apply from an (all-reduced) S^T."""
    _check_dev(s_t, "update: s_t", pair.d, pair.d)
    wp, ldw = _check_dev(w, "update: w", pair.m, pair.n)
    lib.update(pair.handle, adam.handle, C.c_void_p(s_t.data_ptr()), C.c_void_p(wp), ldw,
               int(_dtype_of(w)), float(lr), _stream(stream))
    return w


def projector_gram(a: DeviceProjector, b: DeviceProjector, stream=None):
    """A^T B as a (a.d x b.d) float64 CUDA tensor (subspace_opt.cpp:59-70)."""
    torch = _torch()
    out = torch.empty(a.d, b.d, dtype=torch.float64, device="cuda")
    lib.projector_gram(a.handle, b.handle, C.c_void_p(out.data_ptr()), _stream(stream))
    return out


class MaybeUpdateResultC(C.Structure):
    _fields_ = [("refreshed", C.c_int), ("fit_timed_out", C.c_int),
                ("skipped_zero_grad", C.c_int), ("fit_steps", C.c_int),
                ("bias_before", C.c_double), ("bias_after", C.c_double)]


def maybe_update(pair: DevicePair, adam: AdamState, grad_sub, extra_targets=(), r: int = 4,
                 alpha: float = 0.5, fit: Optional[FitConfig] = None, transfer: int = 0,
                 reinit_seed: int = 0, stream=None):
    """Bias-gated projector refresh (trainer.cpp:74-112): returns (pair, result)
    where pair is the SAME pair when the relative bias on grad_sub is within
    alpha, else a new fitted DevicePair; adam is reprojected in place."""
    targets = [grad_sub] + list(extra_targets)
    arr, _, ld, dt = pair._targets(targets)
    extra = (C.c_void_p * max(1, len(extra_targets)))(*arr[1:]) if extra_targets else None
    c = (fit or FitConfig()).c()
    np_h, nq_h, npair = C.c_void_p(), C.c_void_p(), C.c_void_p()
    res = MaybeUpdateResultC()
    lib.maybe_update(pair.handle, adam.handle, C.c_void_p(arr[0]), ld, int(dt), extra,
                     len(extra_targets), int(r), float(alpha), C.byref(c), int(transfer),
                     C.c_uint64(reinit_seed), C.byref(np_h), C.byref(nq_h), C.byref(npair),
                     C.byref(res), _stream(stream))
    out = dict(refreshed=bool(res.refreshed), fit_timed_out=bool(res.fit_timed_out),
               skipped_zero_grad=bool(res.skipped_zero_grad), fit_steps=res.fit_steps,
               bias_before=res.bias_before, bias_after=res.bias_after)
    if not res.refreshed:
        return pair, out
    p = DeviceProjector._adopt(np_h, pair.compute)
    q = DeviceProjector._adopt(nq_h, pair.compute)
    return DevicePair(p, q, handle=npair), out


def reproject_state(adam: AdamState, old_pair: DevicePair, new_pair: DevicePair, kind: int = 0,
                    stream=None):
    """In-place moment transfer into a refitted subspace (subspace_opt.cpp:72-101)."""
    lib.reproject_state(adam.handle, old_pair.handle, new_pair.handle, int(kind),
                        _stream(stream))


class Comm:
    """The library's NCCL communicator (include/lsp_b200.h lsp_comm_*): the data
    plane of the data-parallel step (SURVEY 8(b) ``lsp_allreduce_S``).  The
    ncclUniqueId is created by rank 0 and shipped over a torch.distributed
    group (any backend: gloo is enough for the bootstrap)."""

    ID_BYTES = 128

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        if len(unique_id) != self.ID_BYTES:
            raise InvalidArgument("comm: unique id must be 128 bytes")
        buf = C.create_string_buffer(unique_id, self.ID_BYTES)
        h = C.c_void_p()
        lib.comm_init(buf, int(nranks), int(rank), C.byref(h))
        self._h = h
        self.nranks, self.rank = int(nranks), int(rank)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(Comm.ID_BYTES)
        lib.comm_unique_id(buf)
        return buf.raw

    @classmethod
    def from_group(cls, group=None):
        """Collective over ``group`` (torch.distributed): rank 0's id to everyone."""
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        return cls(world, rank, obj[0])

    @property
    def handle(self):
        return self._h

    def allreduce_mean(self, t, stream=None):
        """In-place mean over ranks of a contiguous CUDA tensor (f64 / f32 / bf16)."""
        if not t.is_cuda or not t.is_contiguous():
            raise InvalidArgument("allreduce_mean: expected a contiguous CUDA tensor")
        lib.allreduce_mean(self._h, C.c_void_p(t.data_ptr()), t.numel(), int(_dtype_of(t)),
                           _stream(stream))
        return t

    def close(self):
        if getattr(self, "_h", None):
            lib.comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# void (*)(int layer, cudaStream_t stream, void* user)
_BACKWARD_FN = C.CFUNCTYPE(None, C.c_int, C.c_void_p, C.c_void_p)


class Schedule:
    """Native multi-layer step schedule (include/lsp_b200.h lsp_schedule_*): the
    same pipeline as ``schedule.LayerSchedule`` -- layers in backward order,
    compress(l) -> all-reduce(S_l) on a comm stream -> Adam + apply of layer l+1,
    optionally gated per layer by a backward producer -- enqueued by the
    library in C++ (csrc/schedule.cpp).  Capturable in a CUDA graph.

    backward(layer, stream): optional; called on the host in backward order to
    enqueue the backward of ``layer`` on ``stream`` (a torch.cuda.ExternalStream).
    pipeline: 1 / 2 -- stage 2 + Adam of layer l on a side stream beside the Y
    build (and apply, 2) of layer l+1 (``LayerSchedule(pipeline=...)``).
    partition: SMs of a green-context partition that runs stage 1 of every layer
    back to back while the rest of the SMs run each layer's stage 2, Adam, Y
    build and apply (``set_partition``); 0: no partition.
    """

    def __init__(self, layers: Sequence[Layer], comm: Optional[Comm] = None, backward=None,
                 pipeline: int = 0, partition: int = 0):
        self.layers = list(layers)
        self.comm = comm
        arr = (C.c_void_p * len(self.layers))(*[l.handle for l in self.layers])
        h = C.c_void_p()
        lib.schedule_create(len(self.layers), arr, comm.handle if comm is not None else None,
                            C.byref(h))
        self._h = h
        self._cb = None
        if backward is not None:
            self.set_backward(backward)
        if pipeline:
            lib.schedule_set_pipeline(self._h, int(pipeline))
        self.partition = (0, 0)
        if partition:
            self.set_partition(partition)

    def set_partition(self, compress_sms: int):
        """Split the SMs into a stage-1 partition of ``compress_sms`` (rounded up
        by the driver) and an update partition (lsp_schedule_set_partition);
        returns the provisioned (compress, update) SM counts."""
        c, u = C.c_int(), C.c_int()
        lib.schedule_set_partition(self._h, int(compress_sms), C.byref(c), C.byref(u))
        self.partition = (c.value, u.value)
        return self.partition

    def set_backward(self, backward):
        torch = _torch()

        def tramp(layer, stream_ptr, _user):
            # NULL (ctypes None) is the legacy default stream
            with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr or 0)):
                backward(int(layer), torch.cuda.current_stream())

        self._cb = _BACKWARD_FN(tramp) if backward is not None else None
        lib.schedule_set_backward(self._h, self._cb, None)

    def step(self, lr: float, stream=None):
        lib.schedule_step(self._h, float(lr), _stream(stream))

    def close(self):
        if getattr(self, "_h", None):
            lib.schedule_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_version() -> int:
    v = C.c_int()
    lib.nccl_version(C.byref(v))
    return int(v.value)

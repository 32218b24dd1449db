"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the LSP projector hot path.

Two interchangeable CPU implementations with the same numpy-level API:

* ``Oracle("port")``      -- oracle/liblsp_oracle.so, our plain-C restatement of the
                             reference algorithm (oracle/lsp_oracle.c).
* ``Oracle("reference")`` -- oracle/_ref/liblsp_ref.so, the UNMODIFIED reference
                             sources (/root/reference/proj/src) compiled by
                             oracle/Makefile behind an extern "C" shim.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this package, and only as the checker / the timed CPU baseline.  The
product path (paper_2406_10181_b200) never touches it.

Argument naming follows the reference: ``d`` = subspace width (BASELINE.json's
"r"), ``r`` = nonzeros per projector row (BASELINE.json's "d"); see SURVEY.md 0.2.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS = {
    "port": os.path.join(HERE, "liblsp_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "liblsp_ref.so"),
}

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    """Raised with the reference exception kind: invalid_argument / numeric / io."""

    KINDS = {1: "invalid_argument", 2: "numeric", 3: "io", 4: "other"}

    def __init__(self, code: int, msg: str):
        super().__init__(f"{self.KINDS.get(code, code)}: {msg}")
        self.code = code
        self.kind = self.KINDS.get(code, str(code))


def available(kind: str) -> bool:
    return os.path.exists(_LIBS[kind])


@dataclass
class Projector:
    """Host (d,r)-sparse projector, same layout as lsp::SparseProjector
    (proj/include/lsp/projector.hpp:18-30): row-major positions/values, r per row."""

    n_rows: int
    d: int
    r: int
    pos: np.ndarray  # int32 [n_rows*r]
    val: np.ndarray  # float64 [n_rows*r]

    def dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.d))
        rows = np.repeat(np.arange(self.n_rows), self.r)
        out[rows, self.pos] = self.val
        return out

    def copy(self) -> "Projector":
        return Projector(self.n_rows, self.d, self.r, self.pos.copy(), self.val.copy())


class Oracle:
    def __init__(self, kind: str = "port"):
        path = _LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        p = "ref_" if kind == "reference" else "orc_"
        self._p = p
        L = self.lib
        f = lambda name: getattr(L, p + name)  # noqa: E731
        f("last_error").restype = C.c_char_p
        f("derive_seed").restype = C.c_uint64
        f("derive_seed").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        f("init_sparse").argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _i32p, _f64p]
        pair = [C.c_int, C.c_int, C.c_int, C.c_int, _i32p, _f64p, _i32p, _f64p]
        f("compress").argtypes = pair + [_f64p, _f64p]
        f("decompress").argtypes = pair + [_f64p, _f64p]
        f("decompress_apply").argtypes = pair + [_f64p, C.c_double, _f64p]
        f("estimation_bias").argtypes = pair + [_f64p, _f64p]
        f("relative_bias").argtypes = pair + [_f64p, C.POINTER(C.c_double)]
        f("adam_step").argtypes = [C.c_int, C.c_int, C.c_int64, C.c_double, C.c_double,
                                   C.c_double, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p,
                                   C.POINTER(C.c_int64)]
        f("fit_loss").argtypes = pair + [C.c_int, _f64p, C.c_double, C.c_int,
                                         C.POINTER(C.c_double)]
        f("fit_gradient").argtypes = pair + [C.c_int, _f64p, C.c_double, C.c_int, _f64p, _f64p]
        f("fit").argtypes = pair + [C.c_int, _f64p, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.c_int, C.c_int, _f64p, _f64p, C.c_int]
        f("projector_gram").argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _f64p, C.c_int,
                                        C.c_int, _i32p, _f64p, _f64p]
        f("reproject_state").argtypes = [C.c_int] * 4 + [_i32p, _f64p] * 4 + [
            _f64p, _f64p, C.c_int, _f64p, _f64p]
        f("subsample_size").argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.POINTER(C.c_int64)]
        if kind == "reference":
            L.ref_save_projector.restype = C.c_int64
            L.ref_save_projector.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _f64p,
                                             C.c_char_p, C.c_int64]
            L.ref_time_step.argtypes = pair + [_f64p, _f64p, C.c_double, C.c_int, C.c_int,
                                               C.POINTER(C.c_double)]
            if hasattr(L, "ref_schedule_eval"):
                L.ref_schedule_eval.argtypes = [C.c_int, _f64p, C.c_double, C.c_double, C.c_int,
                                                C.c_double, C.c_int, C.c_int, _f64p]
                L.ref_schedule_file.argtypes = [C.c_char_p, C.c_int, _f64p]
            L.ref_maybe_update.argtypes = pair + [_f64p, _f64p, C.c_int64, _f64p, C.c_int, _f64p,
                                                  C.c_int, C.c_double, C.c_double, C.c_double,
                                                  C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                                  C.c_uint64,
                                                  _i32p, _f64p, _i32p, _f64p, _f64p, _f64p, _f64p]

    # -- plumbing ---------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self._p + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    @staticmethod
    def _f64(a) -> np.ndarray:
        return np.ascontiguousarray(a, dtype=np.float64)

    def _pair_args(self, P: Projector, Q: Projector):
        if P.d != Q.d or P.r != Q.r:
            raise ValueError("oracle pair helpers need matching d and r")
        return (P.n_rows, Q.n_rows, P.d, P.r, P.pos, P.val, Q.pos, Q.val)

    # -- API (names follow proj/include/lsp/projector.hpp, subspace_opt.hpp) --
    def derive_seed(self, master: int, tag: int, index: int = 0) -> int:
        return int(self._fn("derive_seed")(master, tag, index))

    def init_sparse(self, n_rows: int, d: int, r: int, seed: int) -> Projector:
        pos = np.zeros(max(n_rows * r, 1), np.int32)
        val = np.zeros(max(n_rows * r, 1), np.float64)
        self._check(self._fn("init_sparse")(n_rows, d, r, seed, pos, val))
        return Projector(n_rows, d, r, pos, val)

    def compress(self, P, Q, g) -> np.ndarray:
        g = self._f64(g)
        out = np.zeros((P.d, Q.d))
        self._check(self._fn("compress")(*self._pair_args(P, Q), g, out))
        return out

    def decompress(self, P, Q, s) -> np.ndarray:
        out = np.zeros((P.n_rows, Q.n_rows))
        self._check(self._fn("decompress")(*self._pair_args(P, Q), self._f64(s), out))
        return out

    def decompress_apply(self, P, Q, delta, lr: float, w) -> np.ndarray:
        w = self._f64(w).copy()
        self._check(self._fn("decompress_apply")(*self._pair_args(P, Q), self._f64(delta), lr, w))
        return w

    def estimation_bias(self, P, Q, sigma) -> np.ndarray:
        out = np.zeros((P.n_rows, Q.n_rows))
        self._check(self._fn("estimation_bias")(*self._pair_args(P, Q), self._f64(sigma), out))
        return out

    def relative_bias(self, P, Q, sigma) -> float:
        out = C.c_double()
        self._check(self._fn("relative_bias")(*self._pair_args(P, Q), self._f64(sigma),
                                              C.byref(out)))
        return out.value

    def adam_step(self, m, v, grad, step: int, beta1=0.9, beta2=0.999, eps=1e-8):
        grad = self._f64(grad)
        rows, cols = grad.shape
        mo, vo, de = np.zeros_like(grad), np.zeros_like(grad), np.zeros_like(grad)
        st = C.c_int64()
        self._check(self._fn("adam_step")(rows, cols, step, beta1, beta2, eps, self._f64(m),
                                          self._f64(v), grad, mo, vo, de, C.byref(st)))
        return mo, vo, de, st.value

    def fit_loss(self, P, Q, targets, reg_beta=0.0, reg_kind=0) -> float:
        t = self._f64(np.stack(targets)) if len(targets) else np.zeros(1)
        out = C.c_double()
        self._check(self._fn("fit_loss")(*self._pair_args(P, Q), len(targets), t, reg_beta,
                                         reg_kind, C.byref(out)))
        return out.value

    def fit_gradient(self, P, Q, targets, reg_beta=0.0, reg_kind=0):
        t = self._f64(np.stack(targets)) if len(targets) else np.zeros(1)
        gp = np.zeros(P.n_rows * P.r)
        gq = np.zeros(Q.n_rows * Q.r)
        self._check(self._fn("fit_gradient")(*self._pair_args(P, Q), len(targets), t, reg_beta,
                                             reg_kind, gp, gq))
        return gp, gq

    def fit(self, P, Q, targets, alpha=0.1, reg_beta=0.0, step_size=1e-2, max_steps=500,
            timeout_steps=500, reg_kind=0, max_curve=4096):
        P, Q = P.copy(), Q.copy()
        t = self._f64(np.stack(targets)) if len(targets) else np.zeros(1)
        rep = np.zeros(6)
        curve = np.zeros(max_curve)
        self._check(self._fn("fit")(P.n_rows, Q.n_rows, P.d, P.r, P.pos, P.val, Q.pos, Q.val,
                                    len(targets), t, alpha, reg_beta, step_size, max_steps,
                                    timeout_steps, reg_kind, rep, curve, max_curve))
        report = dict(final_rel_bias=rep[0], success=bool(rep[1]), timed_out=bool(rep[2]),
                      stalled=bool(rep[3]), steps=int(rep[4]),
                      loss_curve=curve[: min(int(rep[5]), max_curve)].copy())
        return P, Q, report

    def projector_gram(self, A: Projector, B: Projector) -> np.ndarray:
        out = np.zeros((A.d, B.d))
        self._check(self._fn("projector_gram")(A.n_rows, A.d, A.r, A.pos, A.val, B.d, B.r,
                                               B.pos, B.val, out))
        return out

    def reproject_state(self, oldP, oldQ, newP, newQ, m, v, kind=0):
        d = oldP.d
        mo, vo = np.zeros((d, d)), np.zeros((d, d))
        self._check(self._fn("reproject_state")(
            oldP.n_rows, oldQ.n_rows, d, oldP.r, oldP.pos, oldP.val, oldQ.pos, oldQ.val,
            newP.pos, newP.val, newQ.pos, newQ.val, self._f64(m), self._f64(v), kind, mo, vo))
        return mo, vo

    def subsample_size(self, gamma, beta, m, n, total_steps, delta) -> int:
        out = C.c_int64()
        self._check(self._fn("subsample_size")(gamma, beta, m, n, total_steps, delta,
                                               C.byref(out)))
        return out.value

    # reference-only helpers
    def has_schedule(self) -> bool:
        return self.kind == "reference" and hasattr(self.lib, "ref_schedule_eval")

    def schedule_eval(self, prof, d: int, iters: int = 5) -> dict:
        """proj/src/schedule_sim.cpp on a calibrate.TimingProfile (ref_capi.cpp)."""
        out = np.zeros(5)
        vecs = self._f64(prof.vecs())
        self._check(self.lib.ref_schedule_eval(prof.n_layers, vecs, prof.bandwidth_d2h,
                                               prof.bandwidth_h2d, int(prof.duplex),
                                               prof.bytes_per_element, d, iters, out))
        return {"transition_layer": out[0], "closed_form_lsp": out[1],
                "closed_form_zero": out[2], "iter_lsp_layerwise": out[3], "iter_zero": out[4]}

    def schedule_file(self, path: str, iters: int = 5) -> dict:
        """load_profile + simulate(lsp_layerwise) on a profile JSON file."""
        out = np.zeros(3)
        self._check(self.lib.ref_schedule_file(path.encode(), iters, out))
        return {"n_layers": int(out[0]), "transition_layer": out[1], "iter_lsp_layerwise": out[2]}

    def save_projector(self, P: Projector) -> str:
        need = self.lib.ref_save_projector(P.n_rows, P.d, P.r, P.pos, P.val, None, 0)
        buf = C.create_string_buffer(int(need))
        self.lib.ref_save_projector(P.n_rows, P.d, P.r, P.pos, P.val, buf, need)
        return buf.value.decode()

    def maybe_update(self, P, Q, m, v, step, grad, extras, r, alpha, fit_alpha=0.1,
                     reg_beta=0.0, step_size=1e-2, max_steps=500, timeout_steps=500,
                     reg_kind=0, transfer=0, reinit_seed=0):
        """Reference maybe_update (trainer.cpp:74-112).  Returns (newP, newQ, m, v,
        result dict); newP/newQ equal P/Q when not refreshed."""
        d = P.d
        mm, nn = P.n_rows, Q.n_rows
        npos, nval = np.zeros(mm * r, np.int32), np.zeros(mm * r)
        qpos, qval = np.zeros(nn * r, np.int32), np.zeros(nn * r)
        mo, vo = np.zeros((d, d)), np.zeros((d, d))
        res = np.zeros(6)
        ex = self._f64(np.stack(extras)) if extras else np.zeros(1)
        self._check(self.lib.ref_maybe_update(
            *self._pair_args(P, Q), self._f64(m), self._f64(v), step, self._f64(grad),
            len(extras), ex, r, alpha, fit_alpha, reg_beta, step_size, max_steps, timeout_steps,
            reg_kind,
            transfer, reinit_seed, npos, nval, qpos, qval, mo, vo, res))
        out = dict(refreshed=bool(res[0]), fit_timed_out=bool(res[1]),
                   skipped_zero_grad=bool(res[2]), bias_before=res[3], bias_after=res[4],
                   fit_steps=int(res[5]))
        if not out["refreshed"]:
            return P, Q, mo, vo, out
        return (Projector(mm, d, r, npos, nval), Projector(nn, d, r, qpos, qval), mo, vo, out)

    def time_step(self, P, Q, g, w0, lr, count, threads) -> float:
        secs = C.c_double()
        self._check(self.lib.ref_time_step(*self._pair_args(P, Q), self._f64(g), self._f64(w0),
                                           lr, count, threads, C.byref(secs)))
        return secs.value

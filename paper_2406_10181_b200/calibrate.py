"""Schedule-model calibration with measured B200 layer times.

The reference models the paper's layer-wise pipeline in a discrete-event
simulator over a ``TimingProfile`` (proj/include/lsp/schedule_sim.hpp:38-54,
proj/src/schedule_sim.cpp): per layer fwd/bwd on the GPU, the gradient
offload on a d2h link, the host update on the CPU, the delta upload on an h2d
link and the apply on the GPU.  On B200 the LSP step never leaves the device,
and the only communication is the data-parallel all-reduce of each layer's S.
``b200_profile`` maps one measured step onto the reference's profile schema:

  reference resource        B200 data-parallel LSP step
  ------------------        ---------------------------
  bwd_gpu (layer l)         model backward of l (caller-supplied, default 0)
                            + compress(l) (measured)
  d2h link, grad_bytes      NCCL all-reduce of S_l over NVLink: ring bytes
                            2(N-1)/N * |S_l| at the bus bandwidth
  upd_cpu                   0 (Adam runs on the device, inside upd_gpu)
  h2d link, delta_bytes     0 (every rank applies its own replica)
  upd_gpu (apply task)      Adam + Y build + streaming apply of l (measured)

so ``json.dumps(profile.to_json())`` is a file the reference's own
``load_profile``/``simulate`` (lspkit simulate) accepts, and the closed forms
below restate the reference's (transition_layer, closed_form_zero,
closed_form_lsp, lsp_rescale) for the same profile.  Host-side arithmetic only;
tests/test_calibrate.py pins every function to the reference's on random
profiles and feeds a generated profile to the reference simulator.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field, asdict
from typing import Dict, List, Optional, Sequence

_VEC_FIELDS = ("fwd_gpu", "bwd_gpu", "upd_gpu", "fwd_cpu", "bwd_cpu", "upd_cpu",
               "grad_bytes", "delta_bytes")


@dataclass
class TimingProfile:
    """Same fields and units as lsp::TimingProfile (schedule_sim.hpp:38-54):
    seconds, bytes, bytes/second."""

    n_layers: int
    fwd_gpu: List[float]
    bwd_gpu: List[float]
    upd_gpu: List[float]
    fwd_cpu: List[float]
    bwd_cpu: List[float]
    upd_cpu: List[float]
    grad_bytes: List[float]
    delta_bytes: List[float]
    bandwidth_d2h: float
    bandwidth_h2d: float
    duplex: bool = False
    mem_total: float = 0.0
    mem_gpu: float = 0.0
    bytes_per_element: float = 8.0

    def validate(self) -> None:
        """validate_profile (schedule_sim.cpp:313-334); raises ValueError."""
        if self.n_layers < 1:
            raise ValueError("profile needs at least one layer")
        for name in _VEC_FIELDS:
            v = getattr(self, name)
            if len(v) != self.n_layers:
                raise ValueError(f"{name} must have one entry per layer")
            for x in v:
                if not (x >= 0.0) or x == float("inf"):
                    raise ValueError(f"{name} entries must be finite and non-negative")
        for bw in (self.bandwidth_d2h, self.bandwidth_h2d):
            if not (0.0 < bw < float("inf")):
                raise ValueError("bandwidths must be positive")
        if not (0.0 <= self.mem_gpu <= self.mem_total < float("inf")):
            raise ValueError("memory sizes must satisfy 0 <= mem_gpu <= mem_total")
        if not (0.0 < self.bytes_per_element < float("inf")):
            raise ValueError("bytes_per_element must be positive")

    def to_json(self) -> Dict:
        """The load_profile document (schedule_sim.cpp:456-505): exactly these keys."""
        self.validate()
        return asdict(self)

    def vecs(self) -> List[float]:
        out: List[float] = []
        for name in _VEC_FIELDS:
            out.extend(float(x) for x in getattr(self, name))
        return out


def _offload(p: TimingProfile, l: int) -> float:  # schedule_sim.cpp:149-151
    return p.grad_bytes[l] / p.bandwidth_d2h


def _upload(p: TimingProfile, l: int) -> float:  # schedule_sim.cpp:153-155
    return p.delta_bytes[l] / p.bandwidth_h2d


def _sum(v: Sequence[float]) -> float:
    # std::accumulate order (left to right), so results match the reference bitwise
    t = 0.0
    for x in v:
        t += x
    return t


def lsp_rescale(p: TimingProfile, d: int) -> TimingProfile:
    """schedule_sim.cpp:354-371: payload 2*d^2*bytes_per_element per layer and
    direction; host update scaled by d^2 / gradient elements."""
    p.validate()
    if d < 1:
        raise ValueError("subspace dimension must be at least 1")
    payload = 2.0 * float(d) * float(d) * p.bytes_per_element
    out = TimingProfile(**{k: (list(v) if isinstance(v, list) else v) for k, v in asdict(p).items()})
    for l in range(p.n_layers):
        out.grad_bytes[l] = payload
        out.delta_bytes[l] = payload
        elems = p.grad_bytes[l] / p.bytes_per_element
        if elems > 0.0:
            out.upd_cpu[l] = p.upd_cpu[l] * (float(d) * float(d)) / elems
    return out


def transition_layer(p: TimingProfile) -> float:
    """schedule_sim.cpp:373-395: deepest layer whose round trip can block the next
    forward; layers below L - result are scheduled LCFS."""
    p.validate()
    L = p.n_layers
    t_bwd = _sum(p.bwd_gpu)
    t_off = 0.0
    t_up = 0.0
    for l in range(L):
        t_off += _offload(p, l)
        t_up += _upload(p, l)
    t_off /= L
    t_up /= L
    t_upd = _sum(p.upd_cpu) / L
    denom = max(t_off, t_up, t_upd)
    if denom == 0.0:
        return 0.0 if t_bwd > 0.0 else float(L)
    raw = float(L) - (t_bwd - (t_off + t_up + t_upd)) / denom
    return min(max(raw, 0.0), float(L))


def closed_form_zero(p: TimingProfile) -> float:
    """schedule_sim.cpp:397-405."""
    p.validate()
    t_d2h = _sum(p.grad_bytes) / p.bandwidth_d2h
    t_h2d = _sum(p.delta_bytes) / p.bandwidth_h2d
    return _sum(p.fwd_gpu) + max(_sum(p.bwd_gpu), t_d2h) + max(_sum(p.upd_cpu), t_h2d)


def _pipelined(p: TimingProfile) -> float:
    L = p.n_layers
    t_fwd = _sum(p.fwd_gpu)
    t_bwd = _sum(p.bwd_gpu)
    t_upd = _sum(p.upd_cpu)
    t_d2h = _sum(p.grad_bytes) / p.bandwidth_d2h
    t_h2d = _sum(p.delta_bytes) / p.bandwidth_h2d
    layer_comm = t_d2h / L + t_h2d / L
    layer_upd = t_upd / L
    pipelined = t_fwd + t_bwd + layer_comm + layer_upd
    if p.duplex:
        return max(pipelined, t_d2h, t_h2d, t_upd)
    return max(pipelined, t_d2h + t_h2d, t_upd)


def closed_form_lsp(p: TimingProfile, d: int) -> float:
    """schedule_sim.cpp:407-422 (on the d-rescaled profile)."""
    return _pipelined(lsp_rescale(p, d))


def closed_form_b200(p: TimingProfile) -> float:
    """The same bound on a profile whose payloads are already the compressed S
    (b200_profile), i.e. closed_form_lsp without the rescale.  Note it leaves
    out the apply task (upd_gpu), as the reference's does; ``step_estimate``
    adds it."""
    p.validate()
    return _pipelined(p)


def step_estimate(p: TimingProfile) -> Dict[str, float]:
    """Per-iteration estimate of the B200 data-parallel LSP step: the device
    chain (fwd + bwd/compress + Adam/apply of every layer, one GPU resource)
    against the all-reduce link, with one layer of all-reduce exposed at the
    end of the backward pass (the last layer's S is reduced after its compress
    and before its update)."""
    p.validate()
    L = p.n_layers
    gpu = _sum(p.fwd_gpu) + _sum(p.bwd_gpu) + _sum(p.upd_gpu)
    link = _sum(p.grad_bytes) / p.bandwidth_d2h
    tail = _offload(p, 0)  # layer 0 is reduced last (backward order)
    return {"device_s": gpu, "allreduce_s": link, "allreduce_per_layer_s": link / L,
            "estimate_s": max(gpu + tail, link),
            "exposed_allreduce_frac": (max(gpu + tail, link) - gpu) / max(gpu, 1e-30)}


def b200_profile(compress_s: Sequence[float], update_s: Sequence[float], s_bytes: Sequence[float],
                 world: int, busbw: float, fwd_s: Optional[Sequence[float]] = None,
                 bwd_s: Optional[Sequence[float]] = None, d: Optional[int] = None) -> TimingProfile:
    """Profile of a measured B200 step (module docstring for the mapping).
    compress_s / update_s: per-layer seconds in FORWARD layer order (update =
    Adam + Y build + apply); s_bytes: bytes of each layer's S buffer; busbw:
    all-reduce bus bandwidth in bytes/s (NCCL's busbw convention, so the ring
    volume 2(N-1)/N * |S| divided by it is the all-reduce time).

    With ``d`` (and world > 1, equal S sizes per layer) the profile is also
    invariant under the reference's ``lsp_rescale(profile, d)``, which the
    ``lspkit sim --policy lsp_layerwise --d`` path applies first: the element
    width is set so that 2*d^2*bytes_per_element equals the layer's ring bytes,
    and the upload link is made free (there is no upload on B200)."""
    L = len(compress_s)
    if len(update_s) != L or len(s_bytes) != L:
        raise ValueError("per-layer lists must have equal length")
    if world < 1:
        raise ValueError("world must be >= 1")
    fwd = list(fwd_s) if fwd_s is not None else [0.0] * L
    bwd = list(bwd_s) if bwd_s is not None else [0.0] * L
    ring = 2.0 * (world - 1) / world
    bytes_per_element, bw_up = 4.0, float(busbw)
    if d is not None and world > 1:
        if len(set(float(b) for b in s_bytes)) != 1:
            raise ValueError("rescale-invariant profile needs equal S bytes per layer")
        bytes_per_element = ring * float(s_bytes[0]) / (2.0 * float(d) * float(d))
        bw_up = 1e18
    prof = TimingProfile(
        n_layers=L,
        fwd_gpu=[float(x) for x in fwd],
        bwd_gpu=[float(b) + float(c) for b, c in zip(bwd, compress_s)],
        upd_gpu=[float(x) for x in update_s],
        fwd_cpu=[0.0] * L, bwd_cpu=[0.0] * L, upd_cpu=[0.0] * L,
        grad_bytes=[ring * float(b) for b in s_bytes],
        delta_bytes=[0.0] * L,
        bandwidth_d2h=float(busbw), bandwidth_h2d=bw_up, duplex=True,
        mem_total=0.0, mem_gpu=0.0, bytes_per_element=float(bytes_per_element))
    prof.validate()
    return prof


def save_profile(p: TimingProfile, path: str) -> None:
    with open(path, "w") as f:
        json.dump(p.to_json(), f, indent=1)

"""Per-layer schedule for a data-parallel step (north-star subsystem 5).

The reference runs its per-layer loop only after the whole backward pass
(proj/src/trainer.cpp:186-198) and *models* the paper's layer-wise pipeline in a
simulator (build_lsp_layerwise, proj/src/schedule_sim.cpp:255-283: per layer
bwd -> offload -> update -> upload -> apply, deeper layers first).  On B200 the
offload/upload legs become an NCCL all-reduce of the layer's S over NVLink, and
the pipeline is real:

    for layer l in backward order (last layer first):
        compress(l)                          # S_l = P^T G_l Q, one grouped launch
        all_reduce(S_l, mean)  async         # rides on NCCL's stream
        finish(l+1): wait(S_{l+1}) -> Adam -> W -= lr P dS Q^T

so the all-reduce of layer l overlaps the compress of layer l-1 and the apply of
layer l+1.  Anything that exposes ``compress()``, ``s_buffer()``, ``adam(check)``
and ``apply(lr)`` can be scheduled: ``paper_2406_10181_b200.Layer`` on the GPU,
or a CPU stand-in (tests/test_dist_cpu.py runs this exact class over gloo).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence


class LayerSchedule:
    def __init__(self, layers: Sequence, lr: float, group=None,
                 record: Optional[Callable[[str, int, str], None]] = None):
        """layers: in forward order; group: a torch.distributed process group or
        None for a single rank; record(phase, layer, "begin"|"end") is called
        around every stage (bench.py hangs CUDA events on it)."""
        self.layers = list(layers)
        self.lr = lr
        self.group = group
        self.record = record
        self.world = 1
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)

    def _rec(self, phase, li, when):
        if self.record is not None:
            self.record(phase, li, when)

    def _allreduce(self, li):
        if self.world == 1:
            return None
        import torch.distributed as dist

        buf = self.layers[li].s_buffer()
        if dist.get_backend(self.group) == "nccl":
            return dist.all_reduce(buf, op=dist.ReduceOp.AVG, group=self.group, async_op=True)
        # gloo has no AVG: sum, then scale when the result is consumed
        return _SumThenScale(dist.all_reduce(buf, group=self.group, async_op=True), buf,
                             1.0 / self.world)

    def _finish(self, li, work):
        if work is not None:
            work.wait()
        self._rec("adam", li, "begin")
        self.layers[li].adam(self.world > 1)  # re-check finiteness after the reduction
        self._rec("adam", li, "end")
        lay = self.layers[li]
        if hasattr(lay, "apply_prepare"):
            self._rec("build", li, "begin")
            lay.apply_prepare()
            self._rec("build", li, "end")
            self._rec("apply", li, "begin")
            lay.apply_finish(self.lr)
            self._rec("apply", li, "end")
        else:
            self._rec("apply", li, "begin")
            lay.apply(self.lr)
            self._rec("apply", li, "end")

    def order(self):
        return list(reversed(range(len(self.layers))))

    def step(self):
        pending = None
        for li in self.order():
            self._rec("compress", li, "begin")
            self.layers[li].compress()
            self._rec("compress", li, "end")
            work = self._allreduce(li)
            if pending is not None:
                self._finish(*pending)
            pending = (li, work)
        if pending is not None:
            self._finish(*pending)


class _SumThenScale:
    def __init__(self, work, buf, scale):
        self.work, self.buf, self.scale = work, buf, scale

    def wait(self):
        self.work.wait()
        self.buf.mul_(self.scale)

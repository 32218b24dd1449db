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
layer l+1.  With ``streams=(compress_stream, update_stream)`` (concurrent mode)
the compress chain and the update chain (Adam -> Y build -> W stream) also run
on two CUDA streams, joined by one event per layer: the compress of layer l-1
(an L2-gather-latency-bound kernel) overlaps the HBM-bound W update of layer
l+1 on the device.  ``lsp_set_sm_budget`` sizes the two persistent grids so
neither starves the other.  Anything that exposes ``compress()``, ``s_buffer()``, ``adam(check)``
and ``apply(lr)`` can be scheduled: ``paper_2406_10181_b200.Layer`` on the GPU,
or a CPU stand-in (tests/test_dist_cpu.py runs this exact class over gloo).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence


class LayerSchedule:
    def __init__(self, layers: Sequence, lr: float, group=None,
                 record: Optional[Callable[[str, int, str], None]] = None, streams=None):
        """layers: in forward order; group: a torch.distributed process group or
        None for a single rank; record(phase, layer, "begin"|"end") is called
        around every stage (bench.py hangs CUDA events on it)."""
        self.layers = list(layers)
        self.lr = lr
        self.group = group
        self.record = record
        self.streams = streams  # None or (compress stream, update stream), torch.cuda.Stream
        self._events = None
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
        if self.streams is not None:
            return self._step_concurrent()
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


    def _step_concurrent(self):
        import torch

        sc, su = self.streams
        if self._events is None:
            self._events = [torch.cuda.Event() for _ in self.layers]
        main = torch.cuda.current_stream()
        sc.wait_stream(main)
        su.wait_stream(main)
        pending = None
        for li in self.order():
            with torch.cuda.stream(sc):
                self._rec("compress", li, "begin")
                self.layers[li].compress()
                self._rec("compress", li, "end")
                work = self._allreduce(li)
                ev = None
                if work is None:
                    ev = self._events[li]
                    ev.record(sc)
            if pending is not None:
                self._finish_on(su, *pending)
            pending = (li, work, ev)
        if pending is not None:
            self._finish_on(su, *pending)
        main.wait_stream(sc)
        main.wait_stream(su)

    def _finish_on(self, su, li, work, ev):
        import torch

        with torch.cuda.stream(su):
            if ev is not None:
                su.wait_event(ev)
            self._finish(li, work)


class _SumThenScale:
    def __init__(self, work, buf, scale):
        self.work, self.buf, self.scale = work, buf, scale

    def wait(self):
        self.work.wait()
        self.buf.mul_(self.scale)

"""Per-layer schedule for a data-parallel step (north-star subsystem 5).

The reference runs its per-layer loop only after the whole backward pass
(proj/src/trainer.cpp:186-198) and *models* the paper's layer-wise pipeline in a
simulator (build_lsp_layerwise, proj/src/schedule_sim.cpp:255-283: per layer
bwd -> offload -> update -> upload -> apply, deeper layers first, and the next
forward of layer l waits on apply(l), :266).  On B200 the offload/upload legs
become an NCCL all-reduce of the layer's S over NVLink, and the pipeline is real:

    for layer l in backward order (last layer first):
        [bwd(l) on the compute stream -> G_l]            (backward=...)
        compress(l)            S_l = P^T G_l Q, one grouped launch (waits on G_l)
        all_reduce(S_l, mean)  on the comm stream                 (world > 1)
        finish(l+1): wait(S_{l+1}) -> Adam -> Y build -> W -= lr P dS Q^T

so the all-reduce of layer l overlaps the compress of layer l-1 and the apply of
layer l+1, and -- with a ``backward`` producer -- the compress of layer l (an
L2-latency-bound kernel) runs on a side stream while the compute stream already
executes the backward GEMMs of layer l-1.  The next step's work on the compute
stream waits on every apply (the forward of layer l needs W_l updated).

Data plane: ``comm`` (paper_2406_10181_b200.Comm, the library's own NCCL
communicator, lsp_layer_allreduce) or ``group`` (torch.distributed: NCCL AVG,
or gloo sum-then-scale for the CPU stand-in tests).

Anything that exposes ``compress()``, ``s_buffer()``, ``adam(check)`` and
``apply(lr)`` can be scheduled: ``paper_2406_10181_b200.Layer`` on the GPU, or a
CPU stand-in (tests/test_dist_cpu.py runs this exact class over gloo).

Single rank (no ``comm``/``group``): there is no exchange between stage 2 and
Adam, so layers that offer ``compress_adam`` run Adam in the stage-2 epilogue
(one launch fewer per layer, bitwise the same results; ``fuse_adam=False``
keeps the separate Adam launch).

``pipeline=1|2`` moves stage 2 (``compress_finish``), the all-reduce and Adam of
layer l onto a side stream beside the Y build (and, 2, the apply) of layer l+1
(faster for bf16 W).  The library's native twin of this class is
``paper_2406_10181_b200.Schedule`` (csrc/schedule.cpp, lsp_schedule_*), which
bench.py times; the two enqueue the same kernels in the same order (bitwise
equal results, tests/test_gpu_comm_overlap.py), this one adds the per-stage
``record`` hooks used for the phase split.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence


class LayerSchedule:
    def __init__(self, layers: Sequence, lr: float, group=None,
                 record: Optional[Callable[[str, int, str], None]] = None, streams=None,
                 comm=None, backward: Optional[Callable[[int], None]] = None,
                 lsp_stream=None, comm_stream=None, pipeline: int = 0,
                 fuse_adam: bool = True):
        """layers: in forward order.
        group: a torch.distributed process group or None (single rank).
        comm: a paper_2406_10181_b200.Comm (the library's NCCL communicator);
            takes precedence over ``group`` for the S all-reduce.
        record(phase, layer, "begin"|"end"): called around every stage on the
            stream the stage runs on (bench.py hangs CUDA events on it).
        streams: None or (compress stream, update stream) -- concurrent mode.
        backward(li): enqueue the backward of layer li (producing its bound
            gradients) on the current (compute) stream; the LSP chain then runs
            on ``lsp_stream`` gated by one event per layer.
        """
        self.layers = list(layers)
        self.lr = lr
        self.group = group
        self.comm = comm
        self.record = record
        self.streams = streams
        self.backward = backward
        self.lsp_stream = lsp_stream
        self.comm_stream = comm_stream
        self.pipeline = pipeline
        self.fuse_adam = fuse_adam
        self._side = None
        self._events = None
        self.world = 1
        if comm is not None:
            self.world = comm.nranks
        elif group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)

    def _fused(self, li):
        """Adam of layer li runs inside its stage 2 (single rank, native layer)."""
        return (self.fuse_adam and self.world == 1 and self.comm is None
                and hasattr(self.layers[li], "compress_adam"))

    def _compress(self, li):
        lay = self.layers[li]
        lay.compress_adam() if self._fused(li) else lay.compress()

    def _rec(self, phase, li, when):
        if self.record is not None:
            self.record(phase, li, when)

    # ---- the all-reduce of one layer's S ---------------------------------
    def _allreduce(self, li):
        if self.comm is not None:  # also at nranks == 1 (an identity exchange)
            return self._allreduce_comm(li)
        if self.world == 1:
            return None
        import torch.distributed as dist

        buf = self.layers[li].s_buffer()
        if dist.get_backend(self.group) == "nccl":
            return dist.all_reduce(buf, op=dist.ReduceOp.AVG, group=self.group, async_op=True)
        # gloo has no AVG: sum, then scale when the result is consumed
        return _SumThenScale(dist.all_reduce(buf, group=self.group, async_op=True), buf,
                             1.0 / self.world)

    def _allreduce_comm(self, li):
        """lsp_layer_allreduce on the comm stream, ordered after compress(li)."""
        import torch

        ev = self._ev()
        src = torch.cuda.current_stream()
        cs = self.comm_stream
        if cs is None:
            cs = self.comm_stream = torch.cuda.Stream()
        ev["compressed"][li].record(src)
        with torch.cuda.stream(cs):
            cs.wait_event(ev["compressed"][li])
            self._rec("allreduce", li, "begin")
            self.layers[li].allreduce(self.comm)
            self._rec("allreduce", li, "end")
            ev["reduced"][li].record(cs)
        return _EventWork(ev["reduced"][li])

    def _ev(self):
        import torch

        if self._events is None:
            n = len(self.layers)
            self._events = {k: [torch.cuda.Event() for _ in range(n)]
                            for k in ("compressed", "reduced", "grad", "update")}
        return self._events

    # ---- Adam + apply of one layer ---------------------------------------
    def _finish(self, li, work):
        if work is not None:
            work.wait()
        self._rec("adam", li, "begin")
        if not self._fused(li):
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
        if self.pipeline:
            return self._step_pipeline()
        if self.backward is not None:
            return self._step_backward()
        if self.streams is not None:
            return self._step_concurrent()
        pending = None
        for li in self.order():
            self._rec("compress", li, "begin")
            self._compress(li)
            self._rec("compress", li, "end")
            work = self._allreduce(li)
            if pending is not None:
                self._finish(*pending)
            pending = (li, work)
        if pending is not None:
            self._finish(*pending)

    def _step_backward(self):
        """Backward producer on the compute (current) stream; compress, Adam and
        apply on the LSP stream, each compress(l) gated by the event that
        follows bwd(l); the all-reduce on the comm stream.  The compute stream
        waits on the LSP stream at the end (the next forward needs W)."""
        import torch

        main = torch.cuda.current_stream()
        ls = self.lsp_stream
        if ls is None:
            ls = self.lsp_stream = torch.cuda.Stream()
        ev = self._ev()
        ls.wait_stream(main)  # previous work on the compute stream (e.g. the forward)
        pending = None
        for li in self.order():
            self._rec("backward", li, "begin")
            self.backward(li)
            self._rec("backward", li, "end")
            ev["grad"][li].record(main)
            with torch.cuda.stream(ls):
                ls.wait_event(ev["grad"][li])
                self._rec("compress", li, "begin")
                self._compress(li)
                self._rec("compress", li, "end")
                work = self._allreduce(li)
                if pending is not None:
                    self._finish(*pending)
                pending = (li, work)
        with torch.cuda.stream(ls):
            if pending is not None:
                self._finish(*pending)
        main.wait_stream(ls)

    def _step_pipeline(self):
        """Stage 2, the all-reduce and Adam of layer l on a side stream beside the
        Y build (and, with pipeline=2, the apply) of layer l+1 on the caller's
        stream: the light, latency-bound kernels share SMs with the Y build
        (L1-bound) instead of running alone between the heavy ones.  Same
        kernels on the same data, so bitwise the serial schedule's results."""
        import torch

        main = torch.cuda.current_stream()
        side = self._side
        if side is None:
            side = self._side = torch.cuda.Stream()
        ev = self._ev()
        side.wait_stream(main)  # fork (also what graph capture needs)
        prev = None
        for li in self.order():
            lay = self.layers[li]
            self._rec("compress", li, "begin")
            lay.compress_prepare()
            ev["compressed"][li].record(main)
            with torch.cuda.stream(side):
                side.wait_event(ev["compressed"][li])
                fused = self._fused(li)
                lay.compress_finish_adam() if fused else lay.compress_finish()
                self._rec("compress", li, "end")
                if self.comm is not None:
                    lay.allreduce(self.comm)
                self._rec("adam", li, "begin")
                if not fused:
                    lay.adam(self.world > 1)
                self._rec("adam", li, "end")
                ev["update"][li].record(side)
            if prev is not None:
                self._finish_pipelined(prev, li, main)
            prev = li
        self._finish_pipelined(prev, None, main)

    def _finish_pipelined(self, li, nxt, main):
        ev = self._ev()
        lay = self.layers[li]
        main.wait_event(ev["update"][li])
        self._rec("build", li, "begin")
        lay.apply_prepare()
        self._rec("build", li, "end")
        if nxt is not None and self.pipeline == 1:
            main.wait_event(ev["update"][nxt])  # the apply runs alone (full-SM persistent kernel)
        self._rec("apply", li, "begin")
        lay.apply_finish(self.lr)
        self._rec("apply", li, "end")

    def _step_concurrent(self):
        import torch

        sc, su = self.streams
        ev = self._ev()
        main = torch.cuda.current_stream()
        sc.wait_stream(main)
        su.wait_stream(main)
        pending = None
        for li in self.order():
            with torch.cuda.stream(sc):
                self._rec("compress", li, "begin")
                self._compress(li)
                self._rec("compress", li, "end")
                work = self._allreduce(li)
                e = None
                if work is None:
                    e = ev["compressed"][li]
                    e.record(sc)
            if pending is not None:
                self._finish_on(su, *pending)
            pending = (li, work, e)
        if pending is not None:
            self._finish_on(su, *pending)
        main.wait_stream(sc)
        main.wait_stream(su)

    def _finish_on(self, su, li, work, e):
        import torch

        with torch.cuda.stream(su):
            if e is not None:
                su.wait_event(e)
            self._finish(li, work)


class _SumThenScale:
    def __init__(self, work, buf, scale):
        self.work, self.buf, self.scale = work, buf, scale

    def wait(self):
        self.work.wait()
        self.buf.mul_(self.scale)


class _EventWork:
    """Completion of an all-reduce enqueued on the comm stream: the consumer's
    current stream waits on its event (no host blocking)."""

    def __init__(self, event):
        self.event = event

    def wait(self):
        import torch

        torch.cuda.current_stream().wait_event(self.event)

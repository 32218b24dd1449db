"""CPU, world_size 2 over gloo: the data-parallel per-layer schedule
(paper_2406_10181_b200/schedule.py, the code bench.py runs on NCCL) with CPU
stand-in layers built on the oracle.  Checks the DP semantics the reference's
linearity tests pin (proj/tests/test_projector.cpp:208-235): after each step
every rank holds identical weights, equal to a single-process run on the mean
gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(24, 20), (24, 36), (36, 24)]
D, R, LR = 8, 3, 1e-2


class OracleLayer:
    """CPU stand-in exposing the Layer interface (S kept transposed like the device)."""

    def __init__(self, port, mats):
        self.port, self.mats = port, mats  # [(P, Q, G, W)]
        self.S = torch.zeros(len(mats), D, D, dtype=torch.float64)
        self.m = [np.zeros((D, D)) for _ in mats]
        self.v = [np.zeros((D, D)) for _ in mats]
        self.t = 0
        self.delta = [None] * len(mats)

    def compress(self):
        for i, (P, Q, G, _) in enumerate(self.mats):
            self.S[i] = torch.from_numpy(self.port.compress(P, Q, G).T.copy())

    def s_buffer(self):
        return self.S

    def adam(self, check_finite):
        if check_finite:
            assert torch.isfinite(self.S).all()
        t = self.t
        for i in range(len(self.mats)):
            s = self.S[i].numpy().T
            self.m[i], self.v[i], self.delta[i], st = self.port.adam_step(self.m[i], self.v[i], s, t)
        self.t = st

    def apply(self, lr):
        for i, (P, Q, G, W) in enumerate(self.mats):
            self.mats[i] = (P, Q, G, self.port.decompress_apply(P, Q, self.delta[i], lr, W))


def build(port, rank, scale=1.0, grads=None):
    layers = []
    k = 0
    for li in range(2):
        mats = []
        for (m, n) in SHAPES:
            P = port.init_sparse(m, D, R, port.derive_seed(5, 0x1A171, 2 * k))
            Q = port.init_sparse(n, D, R, port.derive_seed(5, 0x1A171, 2 * k + 1))
            if grads is None:
                G = np.random.default_rng(100 * rank + k).standard_normal((m, n))
            else:
                G = grads[k]
            W = np.random.default_rng(999 + k).standard_normal((m, n)) * 0.02
            mats.append((P, Q, G * scale, W))
            k += 1
        layers.append(OracleLayer(port, mats))
    return layers


def worker(rank, world, port_no, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    from paper_2406_10181_b200.schedule import LayerSchedule

    port = oracle.Oracle("port")
    layers = build(port, rank)
    order_seen = []
    sched = LayerSchedule(layers, LR, group=dist.group.WORLD,
                          record=lambda ph, li, when: order_seen.append((ph, li, when)))
    for _ in range(3):
        sched.step()
    ws = [w for lay in layers for (_, _, _, w) in lay.mats]
    out_q.put((rank, [w.copy() for w in ws], order_seen[:12]))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_dp_schedule_two_ranks_gloo(port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, pn, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, ws, order = q.get(timeout=240)
        res[rank] = (ws, order)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # replicated update: identical weights on both ranks
    for a, b in zip(res[0][0], res[1][0]):
        np.testing.assert_array_equal(a, b)
    # equals a single process stepping on the mean gradient
    g0 = [np.random.default_rng(k).standard_normal(s) for k, s in enumerate(SHAPES * 2)]
    g1 = [np.random.default_rng(100 + k).standard_normal(s) for k, s in enumerate(SHAPES * 2)]
    mean = [(a + b) / 2 for a, b in zip(g0, g1)]
    from paper_2406_10181_b200.schedule import LayerSchedule

    single = build(port, 0, grads=mean)
    sched = LayerSchedule(single, LR)
    for _ in range(3):
        sched.step()
    ref = [w for lay in single for (_, _, _, w) in lay.mats]
    for a, b in zip(res[0][0], ref):
        w0 = None
        assert np.linalg.norm(a - b) <= 1e-9 * max(1.0, np.linalg.norm(b))
    # backward order and one-layer-behind pipelining: compress(1), compress(0), finish(1), ...
    order = res[0][1]
    assert order[0] == ("compress", 1, "begin") and order[2] == ("compress", 0, "begin")
    assert order[4] == ("adam", 1, "begin")

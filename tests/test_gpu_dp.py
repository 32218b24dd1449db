"""GPU, world_size 2 over gloo on one device: the data-parallel step bench.py runs
at N>1 (paper_2406_10181_b200/schedule.py over device ``lsp.Layer``s), with the
real kernels.  Round-end testing has a single B200, so NCCL with two ranks is not
available (NCCL refuses two ranks on one device); gloo carries the same
all-reduce of the layers' S buffers.  Checks the DP semantics the reference's
linearity tests pin (proj/tests/test_projector.cpp:208-235): both ranks end with
bit-identical weights, equal (fp32 tolerance) to one rank stepping on the mean
gradient."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(256, 192), (256, 320), (320, 256)]
D, R, LR, L, STEPS = 64, 4, 1e-3, 2, 3

pytestmark = pytest.mark.gpu


def _grad(rank, k, m, n):
    g = torch.Generator(device="cuda")
    g.manual_seed(1000 * rank + k)
    return torch.randn(m, n, device="cuda", generator=g)


def _build(lsp, grads):
    layers, ws = [], []
    k = 0
    for _ in range(L):
        pairs, bound = [], []
        for (m, n) in SHAPES:
            pp, pv = lsp.init_sparse(m, D, R, lsp.derive_seed(9, 0x1A171, 2 * k))
            qp, qv = lsp.init_sparse(n, D, R, lsp.derive_seed(9, 0x1A171, 2 * k + 1))
            pair = lsp.DevicePair(lsp.DeviceProjector(m, D, R, pp, pv),
                                  lsp.DeviceProjector(n, D, R, qp, qv))
            g = torch.Generator(device="cuda")
            g.manual_seed(777 + k)
            w = 0.02 * torch.randn(m, n, device="cuda", generator=g)
            pairs.append(pair)
            bound.append((grads[k], w))
            ws.append(w)
            k += 1
        lay = lsp.Layer(pairs)
        for i, (gk, w) in enumerate(bound):
            lay.bind(i, gk, w)
        layers.append(lay)
    return layers, ws


def _worker(rank, world, port_no, out_q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port_no)
        sys.path.insert(0, ROOT)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2406_10181_b200 as lsp
        from paper_2406_10181_b200.schedule import LayerSchedule

        grads = [_grad(rank, k, m, n) for k, (m, n) in enumerate(SHAPES * L)]
        layers, ws = _build(lsp, grads)
        sched = LayerSchedule(layers, LR, group=dist.group.WORLD)
        for _ in range(STEPS):
            sched.step()
        torch.cuda.synchronize()
        out = [w.cpu().numpy() for w in ws]
        ref = None
        if rank == 0:
            mean = [(_grad(0, k, m, n) + _grad(1, k, m, n)) * 0.5
                    for k, (m, n) in enumerate(SHAPES * L)]
            single, rws = _build(lsp, mean)
            s1 = LayerSchedule(single, LR)
            for _ in range(STEPS):
                s1.step()
            torch.cuda.synchronize()
            ref = [w.cpu().numpy() for w in rws]
        dist.barrier()
        out_q.put((rank, out, ref, None))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent instead of a queue timeout
        out_q.put((rank, None, None, repr(e)))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(400)
def test_dp_layer_schedule_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, pn, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(2):
            rank, ws, ref, err = q.get(timeout=300)
            assert err is None, f"rank {rank}: {err}"
            res[rank] = (ws, ref)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    w0, ref = res[0]
    w1, _ = res[1]
    for a, b in zip(w0, w1):  # replicated update
        np.testing.assert_array_equal(a, b)
    w_init = None
    for k, (a, b) in enumerate(zip(w0, ref)):
        # 3 Adam steps move each weight by ~3*LR; compare the update, fp32 tolerance
        dw = np.abs(a - b).max()
        assert dw <= 1e-5, (k, dw)

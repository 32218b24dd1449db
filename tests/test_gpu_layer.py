"""GPU: the per-layer schedule unit (grouped launches) against the per-matrix path
and the oracle, incl. data-parallel semantics (mean of per-rank S) and the
non-finite abort."""
import numpy as np
import pytest
import torch

import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200 import Layout

pytestmark = pytest.mark.gpu
KINIT = 0x1A171
SHAPES = [(256, 256), (256, 704), (704, 256), (256, 256), (128, 96), (96, 130)]


def make_layer(d=64, r=4, compute="f32", shapes=SHAPES, seed=3):
    pairs = []
    for i, (m, n) in enumerate(shapes):
        P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(seed, KINIT, 2 * i), compute)
        Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(seed, KINIT, 2 * i + 1), compute)
        pairs.append(lsp.DevicePair(P, Q))
    return pairs


@pytest.mark.parametrize("compute", ["f32", "f64"])
def test_layer_step_matches_per_matrix_bitwise(cuda, compute):
    """The grouped layer launches (fp32: gather compress + Y path; fp64: the
    fp64 gather compress, grouped fp64 stage 2 and the fp64 Y path) give
    exactly the per-matrix results."""
    torch.manual_seed(0)
    tdt = torch.float32 if compute == "f32" else torch.float64
    pairs = make_layer(compute=compute)
    layer = lsp.Layer(pairs)
    gs = [torch.randn(p.m, p.n, device="cuda", dtype=tdt) for p in pairs]
    ws = [0.02 * torch.randn(p.m, p.n, device="cuda", dtype=tdt) for p in pairs]
    ws_ref = [w.clone() for w in ws]
    for i, p in enumerate(pairs):
        layer.bind(i, gs[i], ws[i])
    adams = [lsp.AdamState(p.d, compute=compute) for p in pairs]
    for it in range(3):
        layer.step(1e-3)
        s_refs = []
        for i, p in enumerate(pairs):
            s_t = torch.empty(p.d, p.d, device="cuda", dtype=tdt)
            lsp.step(p, adams[i], gs[i], ws_ref[i], 1e-3, s_out=s_t)
            s_refs.append(s_t)
        torch.cuda.synchronize()
        for i in range(len(pairs)):
            assert torch.equal(layer.s_buffer()[i], s_refs[i])
            assert torch.equal(ws[i], ws_ref[i])
    layer.check()
    for i in range(len(pairs)):
        m1, v1, st = layer.adam_get(i)
        m2, v2, st2 = adams[i].get()
        assert st == st2 == 3
        np.testing.assert_array_equal(m1, m2)
        np.testing.assert_array_equal(v1, v2)


def test_layer_data_parallel_mean(cuda, port):
    """DP semantics: update from the mean of per-rank S == step on the mean gradient
    (linearity of compress, proj/tests/test_projector.cpp:208-235)."""
    torch.manual_seed(1)
    pairs = make_layer(compute="f64")
    g1 = [torch.randn(p.m, p.n, device="cuda", dtype=torch.float64) for p in pairs]
    g2 = [torch.randn(p.m, p.n, device="cuda", dtype=torch.float64) for p in pairs]
    w0 = [0.02 * torch.randn(p.m, p.n, device="cuda", dtype=torch.float64) for p in pairs]
    wa = [w.clone() for w in w0]
    wb = [w.clone() for w in w0]
    la, lb = lsp.Layer(pairs), lsp.Layer(pairs)
    for i in range(len(pairs)):
        la.bind(i, g1[i], wa[i])
    la.compress()
    s1 = la.s_buffer().clone()
    for i in range(len(pairs)):
        la.bind(i, g2[i], wa[i])
    la.compress()
    la.s_buffer().copy_(0.5 * (s1 + la.s_buffer()))  # the all-reduce (mean over 2 ranks)
    la.update(1e-3, check_finite=True)
    gm = [0.5 * (a + b) for a, b in zip(g1, g2)]
    for i in range(len(pairs)):
        lb.bind(i, gm[i], wb[i])
    lb.step(1e-3)
    torch.cuda.synchronize()
    for i in range(len(pairs)):
        diff = (wa[i] - wb[i]).norm() / (wb[i] - w0[i]).norm()
        assert diff.item() < 1e-9


def test_layer_nonfinite_aborts_whole_layer(cuda):
    pairs = make_layer()
    layer = lsp.Layer(pairs)
    gs = [torch.randn(p.m, p.n, device="cuda") for p in pairs]
    ws = [torch.randn(p.m, p.n, device="cuda") for p in pairs]
    w0 = [w.clone() for w in ws]
    gs[2][5, 7] = float("nan")
    for i in range(len(pairs)):
        layer.bind(i, gs[i], ws[i])
    layer.step(1e-3)
    with pytest.raises(lsp.NumericError):
        layer.check()
    for a, b in zip(ws, w0):
        assert torch.equal(a, b)
    assert layer.adam_get(0)[2] == 0


def test_layer_rejects_mixed_d(cuda):
    a = lsp.DevicePair(lsp.DeviceProjector.random(64, 16, 2, 1), lsp.DeviceProjector.random(64, 16, 2, 2))
    b = lsp.DevicePair(lsp.DeviceProjector.random(64, 32, 2, 3), lsp.DeviceProjector.random(64, 32, 2, 4))
    with pytest.raises(lsp.InvalidArgument):
        lsp.Layer([a, b])


@pytest.mark.parametrize("mode", ["serial", "pipeline", "partition"])
def test_fp64_layers_native_schedule_bitwise(cuda, mode):
    """fp64 layers through the native schedule (split compress and apply phases
    in the pipelined order, green-context partition): weights bitwise those of
    the Python serial schedule."""
    from paper_2406_10181_b200.schedule import LayerSchedule

    def build():
        torch.manual_seed(7)
        layers, ws = [], []
        for li in range(3):
            pairs = make_layer(compute="f64", seed=11 + li)
            lay = lsp.Layer(pairs)
            for i, p in enumerate(pairs):
                g = torch.randn(p.m, p.n, device="cuda", dtype=torch.float64)
                w = 0.02 * torch.randn(p.m, p.n, device="cuda", dtype=torch.float64)
                lay.bind(i, g, w)
                ws.append(w)
            layers.append(lay)
        return layers, ws

    la, wa = build()
    lb, wb = build()
    sa = LayerSchedule(la, 1e-3)
    sb = lsp.Schedule(lb, pipeline=2 if mode == "pipeline" else 0,
                      partition=48 if mode == "partition" else 0)
    for _ in range(3):
        sa.step()
        sb.step(1e-3)
    torch.cuda.synchronize()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)

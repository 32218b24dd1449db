"""GPU: stage 2 with the layer's Adam fused into its epilogue (k_stage2_f4<true>,
lsp_layer_compress_adam / _compress_finish_adam) against the unfused pair
(stage 2, then k_adam): S, delta, W, moments and the step counter bitwise
equal over several steps, the ping-pong moment pair flipped only for a finite
layer, and the native / Python schedules (which fuse at a single rank) bitwise
equal to the unfused Python schedule, eager and under CUDA-graph replay.
The unfused pair itself is checked against the per-matrix path and the oracle
in test_gpu_layer.py / test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200.schedule import LayerSchedule

pytestmark = pytest.mark.gpu
KINIT = 0x1A171
SHAPES = [(256, 256), (256, 704), (704, 256), (128, 96), (96, 132)]


def _pairs(d=64, r=4, seed=3, shapes=SHAPES):
    out = []
    for i, (m, n) in enumerate(shapes):
        P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(seed, KINIT, 2 * i))
        Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(seed, KINIT, 2 * i + 1))
        out.append(lsp.DevicePair(P, Q))
    return out


def _layers(pairs, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    gs = [torch.randn(p.m, p.n, device="cuda", generator=g) for p in pairs]
    w0 = [0.02 * torch.randn(p.m, p.n, device="cuda", generator=g) for p in pairs]
    la, lb = lsp.Layer(pairs), lsp.Layer(pairs)
    wa = [w.clone() for w in w0]
    wb = [w.clone() for w in w0]
    for i in range(len(pairs)):
        la.bind(i, gs[i], wa[i])
        lb.bind(i, gs[i], wb[i])
    return la, lb, gs, wa, wb


def _same_state(la, lb, n):
    for i in range(n):
        ma, va, sa = la.adam_get(i)
        mb, vb, sb = lb.adam_get(i)
        assert sa == sb
        np.testing.assert_array_equal(ma, mb)
        np.testing.assert_array_equal(va, vb)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("split", [False, True])
def test_fused_adam_bitwise_unfused(cuda, d, split):
    pairs = _pairs(d=d)
    la, lb, gs, wa, wb = _layers(pairs)
    for it in range(4):
        if split:  # the pipelined order's halves
            la.compress_prepare()
            la.compress_finish_adam()
        else:
            la.compress_adam()
        la.apply(1e-3)
        lb.compress()
        lb.adam()
        lb.apply(1e-3)
        torch.cuda.synchronize()
        assert torch.equal(la.s_buffer(), lb.s_buffer())
        for x, y in zip(wa, wb):
            assert torch.equal(x, y)
        for g in gs:  # a new gradient per step (moments accumulate different values)
            g.mul_(-0.75).add_(0.1)
    la.check()
    lb.check()
    _same_state(la, lb, len(pairs))
    assert la.adam_get(0)[2] == 4


@pytest.mark.parametrize("d", [1536, 2048])
def test_fused_adam_wide_d(cuda, d):
    """d > 1024: each thread walks several 1024-column segments of its S^T row
    (the moment staging buffer is reused per segment); 1536 leaves the last
    segment half empty."""
    pairs = _pairs(d=d, shapes=[(512, 640), (640, 512)])
    la, lb, gs, wa, wb = _layers(pairs, seed=4)
    for it in range(3):
        la.compress_adam()
        la.apply(1e-3)
        lb.compress()
        lb.adam()
        lb.apply(1e-3)
        for g in gs:
            g.mul_(0.5).add_(-0.25)
    torch.cuda.synchronize()
    assert torch.equal(la.s_buffer(), lb.s_buffer())
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))


@pytest.mark.parametrize("compute,d", [("f64", 64), ("f32", 30)])
def test_compress_adam_fallback(cuda, compute, d):
    """Groups the fused kernel does not cover (fp64; d % 4 != 0) run stage 2 and
    k_adam behind lsp_layer_compress_adam: the same results as the explicit pair."""
    tdt = torch.float64 if compute == "f64" else torch.float32
    pairs = []
    for i, (m, n) in enumerate([(256, 320), (320, 256)]):
        P = lsp.DeviceProjector.random(m, d, 4, lsp.derive_seed(9, KINIT, 2 * i), compute)
        Q = lsp.DeviceProjector.random(n, d, 4, lsp.derive_seed(9, KINIT, 2 * i + 1), compute)
        pairs.append(lsp.DevicePair(P, Q))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    gs = [torch.randn(p.m, p.n, device="cuda", generator=g, dtype=tdt) for p in pairs]
    w0 = [0.02 * torch.randn(p.m, p.n, device="cuda", generator=g, dtype=tdt) for p in pairs]
    wa = [w.clone() for w in w0]
    wb = [w.clone() for w in w0]
    la, lb = lsp.Layer(pairs), lsp.Layer(pairs)
    for i in range(len(pairs)):
        la.bind(i, gs[i], wa[i])
        lb.bind(i, gs[i], wb[i])
    for _ in range(3):
        la.compress_adam()
        la.apply(1e-3)
        lb.compress()
        lb.adam()
        lb.apply(1e-3)
    torch.cuda.synchronize()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))
    assert la.adam_get(0)[2] == 3


def test_fused_adam_nonfinite_keeps_state(cuda):
    """A non-finite S latches the flag, W is untouched and the ping-pong pair is
    not flipped: moments and step stay those of the last finite step (k_adam's
    skip); the next finite step continues exactly like the unfused layer."""
    pairs = _pairs()
    la, lb, gs, wa, wb = _layers(pairs, seed=1)
    la.compress_adam()
    la.apply(1e-3)
    lb.compress()
    lb.adam()
    lb.apply(1e-3)
    gs[3][5, 7] = float("inf")
    w_before = [w.clone() for w in wa]
    la.compress_adam()
    la.apply(1e-3)
    with pytest.raises(lsp.NumericError):
        la.check()
    for x, y in zip(wa, w_before):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))  # still the state after step 1
    assert la.adam_get(0)[2] == 1
    gs[3][5, 7] = 0.25
    la.compress_adam()
    la.apply(1e-3)
    lb.compress()
    lb.adam()
    lb.apply(1e-3)
    torch.cuda.synchronize()
    la.check()
    lb.check()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))
    assert la.adam_get(0)[2] == 2


def test_fused_then_unfused_share_moments(cuda):
    """Alternating fused and unfused steps on one layer: k_adam follows the
    ping-pong pair the fused kernel left current."""
    pairs = _pairs()
    la, lb, gs, wa, wb = _layers(pairs, seed=2)
    for it in range(5):
        if it % 2 == 0:
            la.compress_adam()
        else:
            la.compress()
            la.adam()
        la.apply(1e-3)
        lb.compress()
        lb.adam()
        lb.apply(1e-3)
    torch.cuda.synchronize()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))


def _stack(seed):
    layers, ws = [], []
    for li in range(3):
        pairs = _pairs(d=64, seed=seed + li)
        g = torch.Generator(device="cuda")
        g.manual_seed(50 + li)
        lay = lsp.Layer(pairs)
        for i, p in enumerate(pairs):
            w = 0.02 * torch.randn(p.m, p.n, device="cuda", generator=g)
            lay.bind(i, torch.randn(p.m, p.n, device="cuda", generator=g), w)
            ws.append(w)
        layers.append(lay)
    return layers, ws


@pytest.mark.parametrize("mode", ["python", "native", "native-pipeline", "python-pipeline",
                                  "native-graph"])
def test_schedules_fuse_bitwise_unfused(cuda, mode):
    la, wa = _stack(21)
    lb, wb = _stack(21)
    ref = LayerSchedule(la, 1e-3, fuse_adam=False)
    if mode == "python":
        step = LayerSchedule(lb, 1e-3).step
    elif mode == "python-pipeline":
        step = LayerSchedule(lb, 1e-3, pipeline=2).step
    else:
        sched = lsp.Schedule(lb, pipeline=2 if mode == "native-pipeline" else 0)
        step = lambda: sched.step(1e-3)  # noqa: E731
    steps = 4
    if mode == "native-graph":
        step()  # eager step 1 (also allocates nothing new under capture)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(steps - 1):
            graph.replay()
    else:
        for _ in range(steps):
            step()
    for _ in range(steps):
        ref.step()
    torch.cuda.synchronize()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    for x, y in zip(la, lb):
        x.check()
        y.check()
        _same_state(x, y, len(x.pairs))
        assert y.adam_get(0)[2] == steps


def test_checked_adam_bitwise(cuda):
    """Data-parallel form: Adam with the finiteness re-check fused in
    (lsp_layer_adam(check_finite=1) after an all-reduce: one ping-pong kernel
    instead of k_check_finite + k_adam) equals the unchecked update on finite
    S, and on a non-finite S latches the flag and leaves W, moments and step."""
    pairs = _pairs()
    la, lb, gs, wa, wb = _layers(pairs, seed=6)
    for it in range(3):
        la.compress()
        la.adam(check_finite=True)
        la.apply(1e-3)
        lb.compress()
        lb.adam()
        lb.apply(1e-3)
        for g in gs:
            g.mul_(0.9).add_(0.05)
    torch.cuda.synchronize()
    for x, y in zip(wa, wb):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))
    la.s_buffer()[1, 3, 2] = float("nan")  # e.g. a rank contributed a non-finite S
    w_before = [w.clone() for w in wa]
    la.adam(check_finite=True)
    la.apply(1e-3)
    with pytest.raises(lsp.NumericError):
        la.check()
    for x, y in zip(wa, w_before):
        assert torch.equal(x, y)
    _same_state(la, lb, len(pairs))
    la.update(1e-3, check_finite=True)  # the S buffer still holds the NaN
    with pytest.raises(lsp.NumericError):
        la.check()
    assert la.adam_get(0)[2] == 3

"""GPU: LayerSchedule modes and launch knobs leave results bitwise unchanged.

* concurrent mode (compress chain and update chain on two streams, one event
  per layer) vs the default single-stream schedule;
* lsp_set_sm_budget (smaller persistent grids for the compress and the apply)
  vs all SMs -- the kernels' work partition changes, their arithmetic order
  per element does not.
"""
import pytest
import torch

import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200.schedule import LayerSchedule

pytestmark = pytest.mark.gpu
KINIT = 0x1A171
SHAPES = [(512, 512), (512, 1376), (1376, 512)]
D, R, L = 128, 4, 4


def _build(seed=5):
    layers, ws = [], []
    k = 0
    g = torch.Generator(device="cuda")
    for _ in range(L):
        pairs, bound = [], []
        for (m, n) in SHAPES:
            P = lsp.DeviceProjector.random(m, D, R, lsp.derive_seed(seed, KINIT, 2 * k))
            Q = lsp.DeviceProjector.random(n, D, R, lsp.derive_seed(seed, KINIT, 2 * k + 1))
            pairs.append(lsp.DevicePair(P, Q))
            g.manual_seed(100 + k)
            bound.append((torch.randn(m, n, device="cuda", generator=g),
                          0.02 * torch.randn(m, n, device="cuda", generator=g)))
            k += 1
        lay = lsp.Layer(pairs)
        for i, (gi, wi) in enumerate(bound):
            lay.bind(i, gi, wi)
        layers.append(lay)
        ws.extend(w for _, w in bound)
    return layers, ws


def _run(streams=None, budget=(0, 0), steps=3):
    lsp.set_sm_budget(*budget)
    try:
        layers, ws = _build()
        sched = LayerSchedule(layers, 1e-3, streams=streams)
        for _ in range(steps):
            sched.step()
        torch.cuda.synchronize()
        return [w.clone() for w in ws]
    finally:
        lsp.set_sm_budget(0, 0)


def test_concurrent_streams_bitwise(cuda):
    ref = _run()
    got = _run(streams=(torch.cuda.Stream(), torch.cuda.Stream()))
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


@pytest.mark.parametrize("budget", [(16, 0), (0, 10), (37, 61)])
def test_sm_budget_bitwise(cuda, budget):
    ref = _run()
    got = _run(budget=budget)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_sm_budget_rejects_negative():
    with pytest.raises(lsp.LspError):
        lsp.set_sm_budget(-1, 0)


def test_cuda_graph_replay_bitwise(cuda):
    """bench.py's default timed loop: one captured LayerSchedule step replayed;
    the device-side Adam step counter advances per replay, so eager steps and
    replays give bitwise-equal weights and moments."""
    ref_layers, ref_ws = _build()
    s1 = LayerSchedule(ref_layers, 1e-3)
    for _ in range(4):
        s1.step()
    layers, ws = _build()
    s2 = LayerSchedule(layers, 1e-3)
    s2.step()  # eager: allocates the lazily-sized workspaces
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s2.step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref_ws, ws):
        assert torch.equal(a, b)
    for la, lb in zip(ref_layers, layers):
        ma, va, sa = la.adam_get(0)
        mb, vb, sb = lb.adam_get(0)
        assert sa == sb == 4
        assert (ma == mb).all() and (va == vb).all()


@pytest.mark.parametrize("d,r", [(1024, 2), (256, 4)])
def test_graph_replay_back_to_back_full_size(cuda, d, r):
    """Regression: back-to-back graph replays of a full-size (4096 x 11008) step
    with r = 2 (d = 1024) or d = 256 -- ring stage counts that came out odd, so
    the two consumer groups of the streaming apply shared stages and a fast
    group could pass a stage's parity wait one phase early (stale tile, launch
    failure).  Replays must match eager steps bitwise."""
    m, n = 4096, 11008

    def build():
        P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(7, KINIT, 0))
        Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(7, KINIT, 1))
        lay = lsp.Layer([lsp.DevicePair(P, Q)])
        g = torch.Generator(device="cuda")
        g.manual_seed(11)
        gm = torch.randn(m, n, device="cuda", generator=g)
        w = 0.02 * torch.randn(m, n, device="cuda", generator=g)
        lay.bind(0, gm, w)
        return lay, gm, w

    la, ga, wa = build()
    sa = LayerSchedule([la], 1e-3)
    for _ in range(8):
        sa.step()
    lb, gb, wb = build()
    sb = LayerSchedule([lb], 1e-3)
    sb.step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        sb.step()
    for _ in range(7):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(wa, wb)


@pytest.mark.parametrize("mode", [1, 2])
def test_pipeline_mode_bitwise(cuda, mode):
    """LayerSchedule(pipeline=1|2): stage 2 + Adam of layer l on a side stream
    beside the Y build (and apply) of layer l+1, via the split
    lsp_layer_compress_prepare / _finish; bitwise the serial schedule."""
    la, wa = _build()
    lb, wb = _build()
    sa = LayerSchedule(la, 1e-3)
    sb = LayerSchedule(lb, 1e-3, pipeline=mode)
    for _ in range(3):
        sa.step()
        sb.step()
    torch.cuda.synchronize()
    for a, b in zip(wa, wb):
        assert torch.equal(a, b)

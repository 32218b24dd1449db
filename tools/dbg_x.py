import torch, sys
sys.path.insert(0, '.')
import paper_2406_10181_b200 as lsp
KINIT = 0x1A171
SHAPES = [(256, 704), (96, 130)]
torch.manual_seed(0)
pairs = []
for i, (m, n) in enumerate(SHAPES):
    P = lsp.DeviceProjector.random(m, 64, 4, lsp.derive_seed(3, KINIT, 2 * i), "f32")
    Q = lsp.DeviceProjector.random(n, 64, 4, lsp.derive_seed(3, KINIT, 2 * i + 1), "f32")
    pairs.append(lsp.DevicePair(P, Q))
layer = lsp.Layer(pairs)
gs = [torch.randn(p.m, p.n, device="cuda") for p in pairs]
ws = [0.02 * torch.randn(p.m, p.n, device="cuda") for p in pairs]
ws_ref = [w.clone() for w in ws]
for i, p in enumerate(pairs):
    layer.bind(i, gs[i], ws[i])
adams = [lsp.AdamState(p.d) for p in pairs]
print("=== layer", file=sys.stderr, flush=True)
layer.step(1e-3)
torch.cuda.synchronize()
print("=== single", file=sys.stderr, flush=True)
for i, p in enumerate(pairs):
    s_t = torch.empty(p.d, p.d, device="cuda")
    lsp.step(p, adams[i], gs[i], ws_ref[i], 1e-3, s_out=s_t)
torch.cuda.synchronize()
for i in range(len(pairs)):
    print(i, SHAPES[i], "W eq", torch.equal(ws[i], ws_ref[i]), (ws[i] - ws_ref[i]).abs().max().item())

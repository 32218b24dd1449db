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
delta = [torch.randn(64, 64, device="cuda") for _ in pairs]
w0 = [0.02 * torch.randn(p.m, p.n, device="cuda") for p in pairs]
a = [w.clone() for w in w0]
for i, p in enumerate(pairs):
    p.decompress_apply(delta[i], 1e-3, a[i])
torch.cuda.synchronize()
print("---- single done", file=sys.stderr)
# grouped through the C-ABI layer apply: emulate with a Layer whose delta we cannot set...

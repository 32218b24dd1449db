"""A capped device fit (5 GD steps) at a C3 shape: python tools/fitcap.py T [m n]."""
import sys, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
m, n, d, r, T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048, int(sys.argv[3]) if len(sys.argv) > 3 else 5504, 1024, 4, int(sys.argv[1])
P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
pair = lsp.DevicePair(P, Q)
tg = [torch.randn(m, n, device="cuda") for _ in range(T)]
rep = pair.fit(tg, lsp.FitConfig(max_steps=5, timeout_steps=5))
torch.cuda.synchronize()
print("steps", rep.steps)

import sys, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
d, r, T = 1024, 4, 9
m, n = 2048, 5504
P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
pair = lsp.DevicePair(P, Q)
tg = [torch.randn(m, n, device="cuda") for _ in range(T)]
rep = pair.fit(tg, lsp.FitConfig(max_steps=10, timeout_steps=10)); torch.cuda.synchronize()

"""maybe_update at the C3 down-projection shape (5504 x 2048, bf16 targets) with
the fit trace on (LSP_FIT_TRACE=1v): per-step gradient times."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
d, r = 1024, 4
gen = torch.Generator(device="cuda"); gen.manual_seed(23)
for (m, n) in [(5504, 2048), (2048, 5504)]:
    P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
    Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
    pair = lsp.DevicePair(P, Q)
    g = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
    ring = [torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(8)]
    t0 = time.perf_counter()
    lsp.maybe_update(pair, lsp.AdamState(d), g, ring, r=r, alpha=0.5, fit=lsp.FitConfig(), reinit_seed=1)
    torch.cuda.synchronize(); print(m, n, "maybe_update %.2f s" % (time.perf_counter() - t0), flush=True)

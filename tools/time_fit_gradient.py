import sys, time, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
d, r, T = 1024, 4, 9
for (m, n) in [(2048, 5504), (5504, 2048)]:
    P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
    Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
    pair = lsp.DevicePair(P, Q)
    tg = [torch.randn(m, n, device="cuda") for _ in range(T)]
    pair.fit_gradient(tg); torch.cuda.synchronize()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        pair.fit_gradient(tg)
        e1.record(); torch.cuda.synchronize()
        print(m, n, "fit_gradient wall %.1f ms, events %.1f ms" % ((time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)))

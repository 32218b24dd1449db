"""maybe_update timing for the three C3 shapes (bf16 targets like bench.py's fit
leg), each shape twice, to separate first-call costs from steady state."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp  # noqa: E402

d, r, ring_n = 1024, 4, 8
gen = torch.Generator(device="cuda")
gen.manual_seed(23)
out = []
for rep in range(2):
    for (m, n) in [(2048, 2048), (2048, 5504), (5504, 2048)]:
        P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, 0x1A171, 2))
        Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, 0x1A171, 3))
        pair = lsp.DevicePair(P, Q)
        g = torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16)
        ring = [torch.randn(m, n, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(ring_n)]
        adam = lsp.AdamState(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        newp, res = lsp.maybe_update(pair, adam, g, ring, r=r, alpha=0.5, fit=lsp.FitConfig(), reinit_seed=1)
        torch.cuda.synchronize()
        out.append({"rep": rep, "shape": [m, n], "ms": round((time.perf_counter() - t0) * 1e3, 1),
                    "steps": int(res["fit_steps"]), "bias_after": res["bias_after"]})
        print(json.dumps(out[-1]), flush=True)

"""reproject_state at d = 1024 (C3 shape pair), for an ncu launch list."""
import sys, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
m, n, d, r = 2048, 5504, 1024, 4
a = lsp.DevicePair(lsp.DeviceProjector.random(m, d, r, 11), lsp.DeviceProjector.random(n, d, r, 12))
b = lsp.DevicePair(lsp.DeviceProjector.random(m, d, r, 13), lsp.DeviceProjector.random(n, d, r, 14))
st = lsp.AdamState(d)
for _ in range(2):
    lsp.reproject_state(st, a, b, 0)
torch.cuda.synchronize()

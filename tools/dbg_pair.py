"""Cluster-pair apply (LSP_APPLY_PAIR=1) vs the default, one case per subprocess
with a timeout (hang finder): prints bitwise equality of W."""
import os, subprocess, sys
CASE = r'''
import os, sys, torch
sys.path.insert(0, '.')
import paper_2406_10181_b200 as lsp
m, n, d, r, wdt = %d, %d, %d, %d, "%s"
P = lsp.DeviceProjector.random(m, d, r, 11, "f32"); Q = lsp.DeviceProjector.random(n, d, r, 12, "f32")
pr = lsp.DevicePair(P, Q)
dt = torch.float32 if wdt == "f32" else torch.bfloat16
g = torch.Generator(device="cuda"); g.manual_seed(3)
w0 = (0.02 * torch.randn(m, n, device="cuda", generator=g)).to(dt)
delta = torch.randn(d, d, device="cuda", generator=g)
outs = []
for pv in ("0", "1"):
    os.environ["LSP_APPLY_PAIR"] = pv
    w = w0.clone(); pr.decompress_apply(delta, 1e-3, w); outs.append(w)
torch.cuda.synchronize()
print("equal" if torch.equal(outs[0], outs[1]) else "DIFF %%g" %% (outs[0].float() - outs[1].float()).abs().max().item())
'''
cases = [(1000, 1500, 256, 4, "f32"), (300, 4100, 1024, 4, "f32"), (513, 517, 96, 8, "f32"),
         (515, 700, 96, 2, "f32"), (1000, 1500, 256, 4, "bf16"), (4096, 11008, 1024, 4, "f32"),
         (11008, 4096, 1024, 4, "f32"), (77, 33, 64, 4, "f32")]
for c in cases:
    try:
        out = subprocess.run([sys.executable, "-c", CASE % c], capture_output=True, text=True,
                             timeout=60)
        res = out.stdout.strip() or out.stderr.strip().splitlines()[-1]
    except subprocess.TimeoutExpired:
        res = "TIMEOUT"
    print(c, res, flush=True)

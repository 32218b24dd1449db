"""Time the projector fit path on the device at BASELINE configs[2] scale
(2048 x 5504 MLP matrix, d = 1024, r = 4): relative_bias, fit_loss,
fit_gradient, a capped fit, the full maybe_update (trainer.cpp:74-112 with the
reference TrainConfig defaults: alpha 0.5, fit alpha 0.1, <= 500 steps) and
reproject_state (the d^3 transfer products).  Prints one JSON line."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, out


def main():
    m, n, d, r = [int(x) for x in (sys.argv[1:5] or (2048, 5504, 1024, 4))]
    T = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    K = 0x1A171
    P = lsp.DeviceProjector.random(m, d, r, lsp.derive_seed(1, K, 2))
    Q = lsp.DeviceProjector.random(n, d, r, lsp.derive_seed(1, K, 3))
    pair = lsp.DevicePair(P, Q)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    tg = [torch.randn(m, n, device="cuda", generator=gen) for _ in range(T)]
    out = {"shape": [m, n], "d": d, "r": r, "targets": T}
    out["relative_bias_ms"], rb = timed(lambda: pair.relative_bias(tg[0]))
    out["relative_bias"] = rb
    out["fit_loss_ms"], _ = timed(lambda: pair.fit_loss(tg))
    out["fit_gradient_ms"], _ = timed(lambda: pair.fit_gradient(tg), reps=2)
    cap = 10
    t0 = time.perf_counter()
    rep = pair.fit(tg, lsp.FitConfig(max_steps=cap, timeout_steps=cap))
    torch.cuda.synchronize()
    out["fit_capped"] = {"steps": rep.steps, "ms": (time.perf_counter() - t0) * 1e3,
                         "ms_per_step": (time.perf_counter() - t0) * 1e3 / max(1, rep.steps)}
    adam = lsp.AdamState(d)
    t0 = time.perf_counter()
    newp, res = lsp.maybe_update(pair, adam, tg[0], tg[1:], r=r, alpha=0.5,
                                 fit=lsp.FitConfig(), reinit_seed=7)
    torch.cuda.synchronize()
    out["maybe_update"] = {"ms": (time.perf_counter() - t0) * 1e3, **res}
    if newp is not pair:
        a = lsp.AdamState(d)
        out["reproject_ms"], _ = timed(lambda: lsp.reproject_state(a, pair, newp, 0), reps=2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

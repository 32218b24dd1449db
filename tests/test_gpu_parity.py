"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle.

Tolerances (relative Frobenius, the reference's own metric,
proj/tests/acceptance.cpp:152-154):
  fp64 compute             1e-12  (the reference's dense-oracle bar)
  fp32 compute             1e-5   (BASELINE north star)
  bf16 storage of W        1e-2   (BASELINE north star), plus a 1-ulp elementwise check
Indices are bit-exact by construction (host init_sparse, pinned in test_host_lib.py).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200 import Layout

pytestmark = pytest.mark.gpu

KINIT = 0x1A171
TDT = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def f32normal(seed, shape, scale=1.0):
    g = np.random.default_rng(seed).standard_normal(shape) * scale
    return g.astype(np.float32).astype(np.float64)


def bf16_round(x):
    return torch.from_numpy(np.asarray(x)).to(torch.bfloat16).double().numpy()


def make(port, m, n, d, r, seed, compute="f32"):
    P = port.init_sparse(m, d, r, port.derive_seed(seed, KINIT, 0))
    Q = port.init_sparse(n, d, r, port.derive_seed(seed, KINIT, 1))
    dp = lsp.DeviceProjector(m, d, r, P.pos, P.val, compute)
    dq = lsp.DeviceProjector(n, d, r, Q.pos, Q.val, compute)
    return P, Q, lsp.DevicePair(dp, dq)


def dev(x, dt="f32"):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", TDT[dt])


def host(t):
    torch.cuda.synchronize()
    return t.double().cpu().numpy()


SHAPES = [(6, 5, 3, 2), (40, 30, 8, 3), (33, 70, 32, 4), (64, 48, 16, 4), (100, 37, 5, 5),
          (128, 96, 32, 1), (257, 129, 64, 4), (31, 33, 1, 1), (300, 200, 100, 7)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("compute", ["f64", "f32"])
def test_compress_decompress_bias_small(cuda, port, shape, compute):
    m, n, d, r = shape
    P, Q, pair = make(port, m, n, d, r, 7 + m, compute)
    tol = 1e-12 if compute == "f64" else 1e-5
    g = f32normal(m * 31 + n, (m, n))
    s = host(pair.compress(dev(g, compute)))
    s_ref = port.compress(P, Q, g)
    assert rel(s, s_ref) < tol
    # transposed layout is the same matrix
    st = host(pair.compress(dev(g, compute), layout=Layout.T))
    np.testing.assert_array_equal(st.T, s)
    sd = f32normal(5 + d, (d, d))
    out = host(pair.decompress(dev(sd, compute)))
    assert rel(out, port.decompress(P, Q, sd)) < tol
    outT = host(pair.decompress(dev(sd.T.copy(), compute), layout=Layout.T))
    np.testing.assert_array_equal(outT, out)
    b = host(pair.estimation_bias(dev(g, compute)))
    assert rel(b, port.estimation_bias(P, Q, g)) < (1e-11 if compute == "f64" else 1e-5)
    assert pair.relative_bias(dev(g, compute)) == pytest.approx(
        port.relative_bias(P, Q, g), rel=1e-10 if compute == "f64" else 1e-5)


@pytest.mark.parametrize("ci", range(6))
def test_golden_cases_fp64(cuda, golden, ci):
    """The reference's own outputs (golden.npz) reproduced by the fp64 device path."""
    data, meta = golden
    c = meta["cases"][ci]
    m, n, d, r = c["m"], c["n"], c["d"], c["r"]
    k = f"case{ci}"
    dp = lsp.DeviceProjector(m, d, r, data[f"{k}_ppos"], data[f"{k}_pval"], "f64")
    dq = lsp.DeviceProjector(n, d, r, data[f"{k}_qpos"], data[f"{k}_qval"], "f64")
    pair = lsp.DevicePair(dp, dq)
    g = dev(data[f"{k}_g"], "f64")
    assert rel(host(pair.compress(g)), data[f"{k}_s"]) < 1e-12
    assert rel(host(pair.decompress(dev(data[f"{k}_s"], "f64"))), data[f"{k}_decomp"]) < 1e-12
    assert rel(host(pair.estimation_bias(g)), data[f"{k}_bias"]) < 1e-12
    assert pair.relative_bias(g) == pytest.approx(c["rel_bias"], rel=1e-12)
    adam = lsp.AdamState(d, compute="f64", layout=Layout.ROW)
    delta = host(adam.step(dev(data[f"{k}_s"], "f64")))
    np.testing.assert_array_equal(delta, data[f"{k}_delta1"])  # bit-exact fp64 Adam
    m1, v1, st = adam.get()
    np.testing.assert_array_equal(m1, data[f"{k}_m1"])
    np.testing.assert_array_equal(v1, data[f"{k}_v1"])
    assert st == 1
    w = dev(data[f"{k}_w"], "f64")
    pair.decompress_apply(dev(data[f"{k}_delta1"], "f64"), 1e-3, w)
    assert rel(host(w), data[f"{k}_w1"]) < 1e-14


def test_c1_fp32_end_to_end(cuda, port, golden):
    """BASELINE configs[0] (1024^2, d=256, r=4) on the fp32 fused path vs the reference."""
    data, meta = golden
    c = meta["c1"]
    P, Q, pair = make(port, 1024, 1024, 256, 4, 1)
    g = f32normal(c["g_seed"], (1024, 1024))
    w0 = f32normal(c["w_seed"], (1024, 1024), 0.02)
    st_dev = torch.empty(256, 256, device="cuda")
    adam = lsp.AdamState(256)
    w = dev(w0)
    lsp.step(pair, adam, dev(g), w, c["lr"], s_out=st_dev)
    s = host(st_dev).T
    assert rel(s, data["c1_s"]) < 1e-5
    # stage-isolated Adam: reference Adam on OUR S, vs our delta (via moments)
    z = np.zeros_like(s)
    _, _, de_ref, _ = port.adam_step(z, z, s, 0)
    w_ref = port.decompress_apply(P, Q, de_ref, c["lr"], w0)
    assert rel(host(w) - w0, w_ref - w0) < 1e-5       # the update itself
    assert rel(host(w), w_ref) < 1e-5
    # end to end against the reference's W (golden rows)
    assert rel(host(w)[::64], data["c1_w1_rows"]) < 1e-5


@pytest.mark.parametrize("wdt", ["f32", "bf16"])
@pytest.mark.parametrize("gdt", ["f32", "bf16"])
def test_step_dtypes(cuda, port, gdt, wdt):
    m, n, d, r = 512, 384, 128, 4
    P, Q, pair = make(port, m, n, d, r, 3)
    g = f32normal(1, (m, n))
    w0 = f32normal(2, (m, n), 0.02)
    if gdt == "bf16":
        g = bf16_round(g)
    if wdt == "bf16":
        w0 = bf16_round(w0)
    adam = lsp.AdamState(d)
    w = dev(w0, wdt)
    s_t = torch.empty(d, d, device="cuda")
    lsp.step(pair, adam, dev(g, gdt), w, 1e-3, s_out=s_t)
    s = host(s_t).T
    assert rel(s, port.compress(P, Q, g)) < 1e-5
    z = np.zeros_like(s)
    _, _, de, _ = port.adam_step(z, z, s, 0)
    w_ref = port.decompress_apply(P, Q, de, 1e-3, w0)
    wg = host(w)
    if wdt == "f32":
        assert rel(wg, w_ref) < 1e-5
    else:
        assert rel(wg, w_ref) < 1e-2
        # every element is the bf16 rounding of the exact update, up to one ulp
        ulp = np.abs(bf16_round(w_ref) - bf16_round(w_ref * (1 + 2**-8)))
        assert (np.abs(wg - bf16_round(w_ref)) <= ulp + 1e-30).mean() > 0.999


def test_multi_step_adam_state(cuda, port):
    """Several fused steps: moments and W follow the reference recurrence."""
    m, n, d, r = 256, 320, 64, 4
    P, Q, pair = make(port, m, n, d, r, 11, "f64")
    adam = lsp.AdamState(d, compute="f64")
    w_ref = f32normal(5, (m, n), 0.02)
    w = dev(w_ref, "f64")
    mm = np.zeros((d, d))
    vv = np.zeros((d, d))
    st = 0
    for t in range(5):
        g = f32normal(100 + t, (m, n))
        lsp.step(pair, adam, dev(g, "f64"), w, 1e-3)
        s = port.compress(P, Q, g)
        mm, vv, de, st = port.adam_step(mm, vv, s, st)
        w_ref = port.decompress_apply(P, Q, de, 1e-3, w_ref)
    gm, gv, gst = adam.get()
    assert gst == 5
    assert rel(gm, mm) < 1e-12 and rel(gv, vv) < 1e-12
    assert rel(host(w) - f32normal(5, (m, n), 0.02), w_ref - f32normal(5, (m, n), 0.02)) < 1e-10


def test_adam_matches_scalar_recurrence(cuda, golden):
    """proj/tests/test_subspace_opt.cpp:69-92 via the golden 7-step sequence."""
    data, _ = golden
    adam = lsp.AdamState(4, beta1=0.8, beta2=0.95, eps=1e-6, compute="f64", layout=Layout.ROW)
    for t in range(7):
        de = host(adam.step(dev(data[f"adam_g{t}"], "f64")))
        np.testing.assert_array_equal(de, data[f"adam_d{t}"])
    m, v, st = adam.get()
    np.testing.assert_array_equal(m, data["adam_m7"])
    np.testing.assert_array_equal(v, data["adam_v7"])
    assert st == 7


def test_adam_kat_and_nonfinite(cuda):
    adam = lsp.AdamState(1, compute="f64", layout=Layout.ROW)
    de = host(adam.step(torch.ones(1, 1, dtype=torch.float64, device="cuda")))
    assert de[0, 0] == 1.0 / (1.0 + 1e-8)
    m, v, _ = adam.get()
    assert m[0, 0] == pytest.approx(0.1, rel=1e-15) and v[0, 0] == pytest.approx(0.001, rel=1e-15)
    adam.check()  # nothing latched
    # non-finite gradient: NumericError, state untouched (subspace_opt.cpp:38)
    a2 = lsp.AdamState(2, compute="f32")
    g = torch.ones(2, 2, device="cuda")
    a2.step(g)
    before = a2.get()
    bad = g.clone()
    bad[0, 0] = float("nan")
    a2.step(bad)
    with pytest.raises(lsp.NumericError):
        a2.check()
    after = a2.get()
    np.testing.assert_array_equal(before[0], after[0])
    np.testing.assert_array_equal(before[1], after[1])
    with pytest.raises(lsp.InvalidArgument):
        lsp.AdamState(2, beta1=1.0)


def test_fused_step_skips_apply_on_nonfinite(cuda, port):
    P, Q, pair = make(port, 64, 64, 16, 2, 4)
    adam = lsp.AdamState(16)
    w = torch.randn(64, 64, device="cuda")
    w0 = w.clone()
    g = torch.randn(64, 64, device="cuda")
    g[3, 5] = float("inf")
    lsp.step(pair, adam, g, w, 1e-3)
    with pytest.raises(lsp.NumericError):
        adam.check()
    assert torch.equal(w, w0)


def test_identity_pattern_is_exact_copy(cuda):
    """proj/tests/test_projector.cpp:128-136"""
    pos, val = lsp.identity_pattern(37)
    p = lsp.DeviceProjector(37, 37, 1, pos, val, "f64")
    q = lsp.DeviceProjector(37, 37, 1, pos, val, "f64")
    pair = lsp.DevicePair(p, q)
    g = torch.randn(37, 37, dtype=torch.float64, device="cuda")
    assert torch.equal(pair.compress(g), g)
    assert torch.equal(pair.decompress(g), g)
    assert pair.relative_bias(g) == 0.0


def test_zero_in_zero_out_and_errors(cuda, port):
    P, Q, pair = make(port, 60, 50, 12, 3, 9)
    z = torch.zeros(60, 50, device="cuda")
    assert pair.compress(z).abs().max().item() == 0.0
    assert pair.decompress(torch.zeros(12, 12, device="cuda")).abs().max().item() == 0.0
    with pytest.raises(lsp.InvalidArgument):
        pair.relative_bias(z)
    with pytest.raises(lsp.InvalidArgument):
        pair.compress(torch.zeros(50, 60, device="cuda"))
    with pytest.raises(lsp.InvalidArgument):  # P.d != Q.d
        a = lsp.DeviceProjector.random(10, 4, 2, 1)
        b = lsp.DeviceProjector.random(10, 5, 2, 2)
        lsp.DevicePair(a, b)


def test_determinism_bitwise(cuda, port):
    P, Q, pair = make(port, 1000, 1500, 256, 4, 21)
    g = torch.randn(1000, 1500, device="cuda")
    s1 = pair.compress(g).clone()
    s2 = pair.compress(g).clone()
    assert torch.equal(s1, s2)
    w1 = torch.randn(1000, 1500, device="cuda")
    w2 = w1.clone()
    pair.decompress_apply(s1, 1e-3, w1)
    pair.decompress_apply(s1, 1e-3, w2)
    assert torch.equal(w1, w2)


def test_reference_seeded_projector_file(cuda, reference):
    """Indices loaded from the reference's own save_projector output."""
    Pr = reference.init_sparse(300, 64, 4, 77)
    Qr = reference.init_sparse(200, 64, 4, 78)
    ptxt, qtxt = reference.save_projector(Pr), reference.save_projector(Qr)
    pm, pd, prr, ppos, pval = lsp.load_projector(ptxt)
    qm, qd, qr, qpos, qval = lsp.load_projector(qtxt)
    np.testing.assert_array_equal(ppos, Pr.pos)
    np.testing.assert_array_equal(pval, Pr.val)
    pair = lsp.DevicePair(lsp.DeviceProjector(pm, pd, prr, ppos, pval, "f64"),
                          lsp.DeviceProjector(qm, qd, qr, qpos, qval, "f64"))
    g = f32normal(3, (300, 200))
    assert rel(host(pair.compress(dev(g, "f64"))), reference.compress(Pr, Qr, g)) < 1e-12


@pytest.mark.parametrize("shape", [(4096, 11008, 1024, 4), (11008, 4096, 1024, 4),
                                   (2048, 5504, 1024, 4), (1280, 5120, 512, 4)])
def test_full_size_compress_and_step(cuda, port, shape):
    """BASELINE layer shapes at full size: S and the applied update vs the oracle."""
    m, n, d, r = shape
    P, Q, pair = make(port, m, n, d, r, 1)
    g = f32normal(17, (m, n))
    gd = dev(g)
    s = host(pair.compress(gd))
    s_ref = port.compress(P, Q, g)
    assert rel(s, s_ref) < 1e-5
    # linearity (DP semantics: compress of a mean = mean of compresses)
    g2 = torch.randn(m, n, device="cuda")
    s2 = pair.compress(g2).double()
    s12 = pair.compress(0.5 * gd + 0.5 * g2).double()
    assert (torch.linalg.norm(s12 - 0.5 * (torch.from_numpy(s).cuda() + s2)) /
            torch.linalg.norm(s12)).item() < 1e-5
    # decompress-apply of the reference delta
    z = np.zeros((d, d))
    _, _, de, _ = port.adam_step(z, z, s_ref, 0)
    w0 = f32normal(18, (m, n), 0.02)
    w = dev(w0)
    pair.decompress_apply(dev(de), 1e-3, w)
    w_ref = port.decompress_apply(P, Q, de, 1e-3, w0)
    assert rel(host(w) - w0, w_ref - w0) < 1e-5


def test_launch_count_increases(cuda, port):
    P, Q, pair = make(port, 64, 64, 32, 4, 5)
    before = lsp.launch_count()
    pair.compress(torch.randn(64, 64, device="cuda"))
    assert lsp.launch_count() >= before + 2


@pytest.mark.parametrize("path", ["y", "rows", "band", "generic"])
def test_decompress_paths_agree(cuda, port, path, monkeypatch):
    """The Y-precompute streaming kernel (apply.cu), the in-kernel Y_band TMA kernel
    and the generic cp.async kernel match the oracle (incl. ragged m, n, d not a
    multiple of 64, r = 8, wide d -> narrower bands, and the group tile split)."""
    monkeypatch.setenv("LSP_DECOMPRESS_GENERIC", "1" if path == "generic" else "0")
    monkeypatch.setenv("LSP_DECOMPRESS_BAND", "1" if path == "band" else "0")
    monkeypatch.setenv("LSP_APPLY_ROWS", "1" if path == "rows" else "0")
    for (m, n, d, r) in [(777, 1000, 64, 4), (130, 4100, 128, 4), (4096, 96, 256, 4),
                         (300, 517, 100, 4), (513, 700, 96, 8), (200, 300, 2048, 4),
                         (100, 90, 4096, 4), (515, 700, 96, 2), (129, 333, 4096, 2)]:
        P, Q, pair = make(port, m, n, d, r, m + n)
        delta = f32normal(d, (d, d))
        w0 = f32normal(n, (m, n), 0.02)
        w = dev(w0)
        pair.decompress_apply(dev(delta), 1e-3, w)
        ref = port.decompress_apply(P, Q, delta, 1e-3, w0)
        assert rel(host(w) - w0, ref - w0) < 1e-5, (m, n, d, r)
        out = host(pair.decompress(dev(delta)))
        assert rel(out, port.decompress(P, Q, delta)) < 1e-5, (m, n, d, r)


def test_decompress_y_bitwise_vs_band(cuda, port, monkeypatch):
    """Same arithmetic and summation order: the Y-precompute path is bitwise equal
    to the in-kernel Y_band kernel, for fp32 and bf16 W (column orientation
    forced: the row orientation associates (P delta) Q^T and differs in rounding)."""
    monkeypatch.setenv("LSP_APPLY_ROWS", "0")
    m, n, d = 1000, 1500, 256
    P, Q, pair = make(port, m, n, d, 4, 7)
    delta = dev(f32normal(d, (d, d)))
    for wdt in (torch.float32, torch.bfloat16):
        w0 = (0.02 * torch.randn(m, n, device="cuda")).to(wdt)
        outs = []
        for band in ("0", "1"):
            monkeypatch.setenv("LSP_DECOMPRESS_BAND", band)
            w = w0.clone()
            pair.decompress_apply(delta, 1e-3, w)
            outs.append(w)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("shape", [(1000, 1500, 256, 4), (777, 1001, 64, 4), (130, 66, 1024, 4),
                                   (513, 258, 100, 2), (300, 700, 96, 8)])
def test_decompress_fp64_y_path(cuda, port, shape, monkeypatch):
    """fp64 (the reference's precision): the Y-precompute path (apply_f64.cu) on
    the oracle at 1e-12 -- decompress_apply (W -= lr P delta Q^T) and decompress
    (out = P delta Q^T) -- and, for r = 4, bitwise equal to the in-kernel Y_band
    kernel (same arithmetic and summation order); odd n covers the last single
    column, m not a multiple of the 64-row tile, d up to 1024."""
    m, n, d, r = shape
    P, Q, pair = make(port, m, n, d, r, m + n, "f64")
    delta = np.random.default_rng(d).standard_normal((d, d))
    w0 = 0.02 * np.random.default_rng(m).standard_normal((m, n))
    outs = []
    for band in ("0", "1"):
        monkeypatch.setenv("LSP_DECOMPRESS_BAND", band)
        w = dev(w0, "f64")
        pair.decompress_apply(dev(delta, "f64"), 1e-3, w)
        outs.append(w)
        if band == "1" and r != 4:
            break  # the in-kernel band kernel is r = 4 only
    monkeypatch.delenv("LSP_DECOMPRESS_BAND")
    ref = port.decompress_apply(P, Q, delta, 1e-3, w0)
    assert rel(host(outs[0]) - w0, ref - w0) < 1e-12
    if r == 4:
        assert torch.equal(outs[0], outs[1])
    out = host(pair.decompress(dev(delta, "f64")))
    assert rel(out, port.decompress(P, Q, delta)) < 1e-12


def test_apply_cluster_pair_bitwise(cuda, port, monkeypatch):
    """The 2-CTA cluster apply (LSP_APPLY_PAIR=1: leader-issued multicast W boxes
    and P entries, remote stage release) is bitwise equal to the default apply,
    for even and odd band counts (n = 4100 / 517: the last pair's second CTA has
    no band), r = 2, 4, 8, fp32 and bf16 W; and matches the oracle."""
    monkeypatch.setenv("LSP_APPLY_ROWS", "0")
    monkeypatch.setenv("LSP_DECOMPRESS_BAND", "0")
    for (m, n, d, r, wdt) in [(1000, 1500, 256, 4, torch.float32), (300, 4100, 1024, 4, torch.float32),
                              (513, 517, 96, 8, torch.float32), (515, 700, 96, 2, torch.float32),
                              (1000, 1500, 256, 4, torch.bfloat16), (77, 33, 64, 4, torch.float32)]:
        P, Q, pair = make(port, m, n, d, r, m + 7 * n)
        delta = f32normal(d + 5, (d, d))
        w0 = f32normal(n + 5, (m, n), 0.02)
        outs = []
        for pv in ("0", "1"):
            monkeypatch.setenv("LSP_APPLY_PAIR", pv)
            w = dev(w0).to(wdt)
            pair.decompress_apply(dev(delta), 1e-3, w)
            outs.append(w)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), (m, n, d, r, wdt)
        if wdt == torch.float32:
            ref = port.decompress_apply(P, Q, delta, 1e-3, w0)
            assert rel(host(outs[1]) - w0, ref - w0) < 1e-5, (m, n, d, r)


@pytest.mark.parametrize("beta_in", [True, False])
def test_apply_two_columns_per_lane_bitwise(cuda, port, monkeypatch, beta_in):
    """k_apply_y with two or four columns per lane (LSP_APPLY_CPL=2/4: 8/16-byte Y
    gathers, multi-element W loads/stores) is bitwise equal to one column per
    lane, for n not a multiple of 2 or 4 (partial last group), ragged m,
    r = 2, 4, 8, fp32 and bf16 W, in-place apply and decompress-only output."""
    monkeypatch.setenv("LSP_APPLY_ROWS", "0")
    monkeypatch.setenv("LSP_DECOMPRESS_BAND", "0")
    for (m, n, d, r, wdt) in [(1000, 1500, 256, 4, torch.float32), (300, 4100, 1024, 4, torch.float32),
                              (513, 517, 96, 8, torch.float32), (515, 701, 96, 2, torch.float32),
                              (1000, 1501, 256, 4, torch.bfloat16), (77, 33, 64, 4, torch.bfloat16),
                              (200, 1002, 128, 4, torch.float32), (130, 4098, 1024, 4, torch.bfloat16),
                              (600, 1000, 96, 2, torch.float32), (600, 1000, 1024, 2, torch.bfloat16),
                              (300, 1000, 256, 8, torch.float32)]:
        P, Q, pair = make(port, m, n, d, r, m + 11 * n)
        delta = dev(f32normal(d + 9, (d, d)))
        w0 = f32normal(n + 9, (m, n), 0.02)
        outs = []
        for cpl in ("1", "2", "4"):
            monkeypatch.setenv("LSP_APPLY_CPL", cpl)
            if beta_in:
                w = dev(w0).to(wdt)
                pair.decompress_apply(delta, 1e-3, w)
            else:
                w = pair.decompress(delta, dtype=wdt)
            outs.append(w)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2]), (m, n, d, r, wdt, beta_in)


@pytest.mark.parametrize("kind", ["smem", "global", "vec"])
def test_build_y_variants_bitwise(cuda, port, monkeypatch, kind):
    """The Y builds staging Delta in shared memory (k_build_y_smem), gathering
    it per element (k_build_y) or writing lane-sized row pieces (k_build_y_vec)
    give W bitwise equal to the default tiled build (k_build_y_tile, coalesced
    32 KB chunks), for ragged n, d = 96 (not a multiple of 64), d = 1000 (a
    partial 256-row chunk), r = 2, 4, 8; and match the oracle."""
    monkeypatch.setenv("LSP_APPLY_ROWS", "0")
    monkeypatch.setenv("LSP_DECOMPRESS_BAND", "0")
    for (m, n, d, r) in [(1000, 1500, 256, 4), (300, 2100, 64, 2), (257, 4100, 1024, 4),
                         (513, 700, 96, 8), (300, 999, 1000, 4)]:
        P, Q, pair = make(port, m, n, d, r, m + 5 * n)
        delta = f32normal(d + 3, (d, d))
        w0 = f32normal(n + 3, (m, n), 0.02)
        outs = []
        for alt in (False, True):
            monkeypatch.setenv("LSP_BUILD_Y_TILE", "0" if alt and kind == "vec" else "1")
            monkeypatch.setenv("LSP_BUILD_Y_VEC", "0" if alt and kind != "vec" else "1")
            monkeypatch.setenv("LSP_BUILD_Y_GLOBAL", "1" if alt and kind == "global" else "0")
            w = dev(w0)
            pair.decompress_apply(dev(delta), 1e-3, w)
            outs.append(w)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), (m, n, d, r)
        ref = port.decompress_apply(P, Q, delta, 1e-3, w0)
        assert rel(host(outs[0]) - w0, ref - w0) < 1e-5, (m, n, d, r)


@pytest.mark.parametrize("rows", ["1", "0"])
def test_decompress_row_orientation(cuda, port, rows, monkeypatch):  # opt-in path and default
    """The row-orientation apply (apply_x.cu, n > m, fp32): ragged m (not a multiple
    of the 32-row band) and n (not a multiple of the 128-column tile), r = 4 and 8,
    in-place apply and decompress-only output, against the oracle; and against
    the column orientation within fp32 rounding."""
    monkeypatch.setenv("LSP_APPLY_ROWS", rows)
    for (m, n, d, r) in [(77, 1000, 64, 4), (130, 4100, 128, 4), (513, 700, 96, 8),
                         (1000, 4096, 1024, 4), (32, 129, 32, 4)]:
        P, Q, pair = make(port, m, n, d, r, m + 3 * n)
        delta = f32normal(d + 1, (d, d))
        w0 = f32normal(n + 1, (m, n), 0.02)
        w = dev(w0)
        pair.decompress_apply(dev(delta), 1e-3, w)
        ref = port.decompress_apply(P, Q, delta, 1e-3, w0)
        assert rel(host(w) - w0, ref - w0) < 1e-5, (m, n, d, r)
        out = host(pair.decompress(dev(delta)))
        assert rel(out, port.decompress(P, Q, delta)) < 1e-5, (m, n, d, r)


def _skewed(m, d, r, seed, hot):
    """A structured projector: every row hits the `hot` lowest bins first, so a
    few bins collect most entries (stress for the fixed-slot overflow lists)."""
    rng = np.random.default_rng(seed)
    pos = np.empty((m, r), np.int32)
    for i in range(m):
        lo = rng.choice(hot, size=min(r, hot), replace=False)
        rest = rng.choice(np.arange(hot, d), size=r - len(lo), replace=False) if r > hot else []
        pos[i] = np.sort(np.concatenate([lo, rest]).astype(np.int32))
    val = rng.standard_normal((m, r)) / np.sqrt(r)
    return oracle.Projector(m, d, r, pos.ravel(), val.ravel())


@pytest.mark.parametrize("pin", ["", "1,2", "1,4", "1,8", "2,2", "2,4"])
@pytest.mark.parametrize("gdt", ["f32", "bf16"])
def test_compress_paths_agree(cuda, port, gdt, pin, monkeypatch):
    """Gather-form stage 1 (compress_spmm.cu), fixed-slot TMA stage 1 and the
    CSC-walk stage 1: bitwise identical (same per-bin summation order), all on
    the oracle; random and skewed projectors, ragged m and n, d not a multiple
    of 32; every (columns per lane, K) variant of the slot kernel."""
    monkeypatch.setenv("LSP_COMPRESS_SLOTS", pin)
    cases = []
    for (m, n, d, r) in [(777, 1000, 64, 4), (1300, 4100, 128, 4), (4096, 96, 1024, 4),
                         (513, 257, 100, 3), (2000, 300, 2048, 4), (300, 8192, 64, 4)]:
        P, Q, _ = make(port, m, n, d, r, m + n)
        cases.append((P, Q))
    for hot in (1, 3):
        cases.append((_skewed(1500, 96, 4, hot, hot), port.init_sparse(704, 96, 4, 5)))
    for P, Q in cases:
        g = f32normal(P.n_rows, (P.n_rows, Q.n_rows))
        if gdt == "bf16":
            g = bf16_round(g)
        outs = []
        for spmm, generic in (("1", "0"), ("0", "0"), ("0", "1")):
            monkeypatch.setenv("LSP_COMPRESS_SPMM", spmm)
            monkeypatch.setenv("LSP_COMPRESS_GENERIC", generic)
            pair = lsp.DevicePair(lsp.DeviceProjector(P.n_rows, P.d, P.r, P.pos, P.val),
                                  lsp.DeviceProjector(Q.n_rows, Q.d, Q.r, Q.pos, Q.val))
            outs.append(pair.compress(dev(g, gdt)).clone())
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
        assert rel(host(outs[0]), port.compress(P, Q, g)) < 1e-5


def test_compress_paths_agree_fp64(cuda, port, monkeypatch):
    """fp64 (the reference's precision): the gather-form stage 1 and the CSC-walk
    stage 1 are bitwise identical, and match the oracle at 1e-12; random and
    skewed projectors, ragged shapes, d not a multiple of 32; then a value
    refresh through set_values."""
    cases = []
    for (m, n, d, r) in [(777, 1000, 64, 4), (1300, 4100, 128, 4), (4096, 96, 1024, 4),
                         (513, 258, 100, 3), (2000, 300, 2048, 8), (300, 8192, 64, 2)]:
        P, Q, _ = make(port, m, n, d, r, m + n)
        cases.append((P, Q))
    cases.append((_skewed(1500, 96, 4, 1, 1), port.init_sparse(704, 96, 4, 5)))
    for P, Q in cases:
        g = np.random.default_rng(P.n_rows).standard_normal((P.n_rows, Q.n_rows))
        outs = []
        for spmm in ("1", "0"):
            monkeypatch.setenv("LSP_COMPRESS_SPMM", spmm)
            pair = lsp.DevicePair(lsp.DeviceProjector(P.n_rows, P.d, P.r, P.pos, P.val, "f64"),
                                  lsp.DeviceProjector(Q.n_rows, Q.d, Q.r, Q.pos, Q.val, "f64"))
            outs.append(pair.compress(dev(g, "f64")).clone())
        assert torch.equal(outs[0], outs[1])
        assert rel(host(outs[0]), port.compress(P, Q, g)) < 1e-12
    monkeypatch.setenv("LSP_COMPRESS_SPMM", "1")
    P, Q = cases[0]
    dp = lsp.DeviceProjector(P.n_rows, P.d, P.r, P.pos, P.val, "f64")
    pair = lsp.DevicePair(dp, lsp.DeviceProjector(Q.n_rows, Q.d, Q.r, Q.pos, Q.val, "f64"))
    g = np.random.default_rng(9).standard_normal((P.n_rows, Q.n_rows))
    pair.compress(dev(g, "f64"))  # builds the padded entry table
    P2 = P.copy()
    P2.val = np.random.default_rng(3).standard_normal(P.val.shape)
    dp.set_values(P2.val)
    assert rel(host(pair.compress(dev(g, "f64"))), port.compress(P2, Q, g)) < 1e-12


@pytest.mark.parametrize("spmm", ["1", "0"])
def test_compress_slots_value_refresh(cuda, port, spmm, monkeypatch):
    """set_values re-derives the slot/overflow tables' and the packed CSC entries'
    values on the device (gather kernel and slot kernel)."""
    monkeypatch.setenv("LSP_COMPRESS_SPMM", spmm)
    P = _skewed(900, 64, 4, 11, 2)
    Q = port.init_sparse(300, 64, 4, 12)
    dp = lsp.DeviceProjector(P.n_rows, P.d, P.r, P.pos, P.val)
    pair = lsp.DevicePair(dp, lsp.DeviceProjector(Q.n_rows, Q.d, Q.r, Q.pos, Q.val))
    g = f32normal(4, (900, 300))
    pair.compress(dev(g))  # builds the tables
    P2 = P.copy()
    P2.val = np.random.default_rng(3).standard_normal(P.val.shape)
    dp.set_values(P2.val)
    assert rel(host(pair.compress(dev(g))), port.compress(P2, Q, g)) < 1e-5

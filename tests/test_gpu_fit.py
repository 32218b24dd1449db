"""GPU parity of the projector fit (Eq. 3) and the optimizer-state transfer
(proj/src/projector.cpp:189-315, proj/src/subspace_opt.cpp:59-101), fp64 on device."""
import numpy as np
import pytest
import torch

import oracle
import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200 import Layout

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def dpair(P, Q, compute="f64"):
    return lsp.DevicePair(lsp.DeviceProjector(P.n_rows, P.d, P.r, P.pos, P.val, compute),
                          lsp.DeviceProjector(Q.n_rows, Q.d, Q.r, Q.pos, Q.val, compute))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.float64)


def fixture_pair(golden):
    data, _ = golden
    P = oracle.Projector(12, 6, 3, data["fit_ppos"].astype(np.int32), data["fit_pval"])
    Q = oracle.Projector(10, 6, 3, data["fit_qpos"].astype(np.int32), data["fit_qval"])
    return P, Q, list(data["fit_targets"])


@pytest.mark.parametrize("kind", [0, 1])
def test_fit_loss_and_gradient_golden(cuda, golden, kind):
    data, _ = golden
    P, Q, targets = fixture_pair(golden)
    pair = dpair(P, Q)
    cfg = lsp.FitConfig(reg_beta=0.3, reg_kind=kind)
    tg = [dev(t) for t in targets]
    assert pair.fit_loss(tg, cfg) == pytest.approx(data[f"fit_loss_k{kind}"][0], rel=1e-11)
    gp, gq = pair.fit_gradient(tg, cfg)
    assert rel(gp, data[f"fit_gp_k{kind}"]) < 1e-10
    assert rel(gq, data[f"fit_gq_k{kind}"]) < 1e-10


@pytest.mark.parametrize("shape", [(40, 30, 8, 3), (64, 96, 16, 4), (130, 70, 33, 2)])
def test_fit_gradient_vs_oracle(cuda, port, shape):
    m, n, d, r = shape
    P = port.init_sparse(m, d, r, 5)
    Q = port.init_sparse(n, d, r, 6)
    rng = np.random.default_rng(m)
    targets = [rng.standard_normal((m, n)) for _ in range(3)]
    pair = dpair(P, Q)
    tg = [dev(t) for t in targets]
    assert pair.fit_loss(tg) == pytest.approx(port.fit_loss(P, Q, targets), rel=1e-11)
    gp, gq = pair.fit_gradient(tg)
    gp_ref, gq_ref = port.fit_gradient(P, Q, targets)
    assert rel(gp, gp_ref) < 1e-10 and rel(gq, gq_ref) < 1e-10


def test_fit_gradient_matches_finite_differences(cuda, port):
    """proj/tests/test_projector.cpp:237-266 on the device loss."""
    P = port.init_sparse(6, 3, 2, oracle.Oracle("port").derive_seed(71, 1))
    Q = port.init_sparse(5, 3, 2, oracle.Oracle("port").derive_seed(71, 2))
    rng = np.random.default_rng(67)
    targets = [dev(rng.standard_normal((6, 5))) for _ in range(2)]
    for kind in (0, 1):
        cfg = lsp.FitConfig(reg_beta=0.3, reg_kind=kind)
        pair = dpair(P, Q)
        gp, gq = pair.fit_gradient(targets, cfg)
        h = 1e-6
        for which, proj, grad in (("p", P, gp), ("q", Q, gq)):
            for i in range(len(proj.val)):
                vals = proj.val.copy()
                dproj = pair.p if which == "p" else pair.q
                vals[i] += h
                dproj.set_values(vals)
                up = pair.fit_loss(targets, cfg)
                vals[i] -= 2 * h
                dproj.set_values(vals)
                down = pair.fit_loss(targets, cfg)
                dproj.set_values(proj.val)
                fd = (up - down) / (2 * h)
                scale = max(abs(fd), abs(grad[i]), 1e-6)
                assert abs(fd - grad[i]) / scale < 1e-4


def test_fit_trajectory_matches_reference(cuda, golden):
    """Same accepted steps, loss curve and fitted values as the reference fit."""
    data, meta = golden
    P, Q, targets = fixture_pair(golden)
    pair = dpair(P, Q)
    rep = pair.fit([dev(t) for t in targets], lsp.FitConfig(alpha=0.5, max_steps=30,
                                                            timeout_steps=30))
    want = meta["fit_report"]
    assert rep.steps == want["steps"]
    assert rep.success == want["success"] and rep.stalled == want["stalled"]
    assert rep.final_rel_bias == pytest.approx(want["final_rel_bias"], rel=1e-9)
    np.testing.assert_allclose(rep.loss_curve, data["fit_curve"], rtol=1e-9)
    _, pv = pair.p.get()
    _, qv = pair.q.get()
    assert rel(pv, data["fit_out_pval"]) < 1e-9 and rel(qv, data["fit_out_qval"]) < 1e-9


def test_fit_exactly_representable_returns_immediately(cuda):
    """proj/tests/test_projector.cpp:268-280 with full-identity projectors (r = d)."""
    n = 5
    pos = np.tile(np.arange(n, dtype=np.int32), n)
    val = np.eye(n).ravel()
    pair = lsp.DevicePair(lsp.DeviceProjector(n, n, n, pos, val, "f64"),
                          lsp.DeviceProjector(n, n, n, pos, val, "f64"))
    t = torch.randn(n, n, dtype=torch.float64, device="cuda")
    rep = pair.fit([t], lsp.FitConfig(alpha=0.1))
    assert rep.success and rep.steps == 0 and len(rep.loss_curve) == 1
    assert abs(rep.loss_curve[0]) < 1e-20 + 1e-12 * float(t.norm()) ** 2
    assert rep.final_rel_bias < 1e-7


def test_fit_loss_monotone_and_success_bound(cuda, port):
    """proj/tests/test_projector.cpp:282-313"""
    rng = np.random.default_rng(89)
    u, v = rng.standard_normal((16, 2)), rng.standard_normal((2, 16))
    P = port.init_sparse(16, 8, 4, port.derive_seed(97, 1))
    Q = port.init_sparse(16, 8, 4, port.derive_seed(97, 2))
    pair = dpair(P, Q)
    tgt = dev(u @ v)
    rep = pair.fit([tgt], lsp.FitConfig(alpha=0.3, max_steps=400, timeout_steps=400))
    assert rep.success and rep.final_rel_bias <= 0.3
    assert all(b <= a for a, b in zip(rep.loss_curve, rep.loss_curve[1:]))
    assert pair.relative_bias(tgt) <= 0.3 + 1e-9


def test_fit_rejects_bad_inputs(cuda, port):
    P = port.init_sparse(4, 2, 1, 1)
    pair = dpair(P, P)
    with pytest.raises(lsp.InvalidArgument):
        pair.fit([])
    with pytest.raises(lsp.InvalidArgument):
        pair.fit([torch.ones(4, 4, dtype=torch.float64, device="cuda")], lsp.FitConfig(alpha=0.0))


def test_projector_gram_and_reproject(cuda, golden, port):
    data, _ = golden
    m, n, d, r = 9, 8, 4, 2
    pr = {nm: oracle.Projector(m if nm.endswith("P") else n, d, r,
                               data[f"rp_{nm}_pos"].astype(np.int32), data[f"rp_{nm}_val"])
          for nm in ("oP", "oQ", "nP", "nQ")}
    dv = {k: lsp.DeviceProjector(p.n_rows, d, r, p.pos, p.val, "f64") for k, p in pr.items()}
    gram = lsp.projector_gram(dv["nP"], dv["oP"]).cpu().numpy()
    np.testing.assert_array_equal(gram, data["rp_gram"])  # reference summation order
    old = lsp.DevicePair(dv["oP"], dv["oQ"])
    new = lsp.DevicePair(dv["nP"], dv["nQ"])
    for kind in (0, 1):
        for layout in (Layout.ROW, Layout.T):
            a = lsp.AdamState(d, compute="f64", layout=layout)
            a.set(data["rp_m"], data["rp_v"], 17)
            lsp.reproject_state(a, old, new, kind)
            mo, vo, st = a.get()
            assert st == 17
            assert rel(mo, data[f"rp_m_k{kind}"]) < 1e-12
            assert rel(vo, data[f"rp_v_k{kind}"]) < 1e-12
            assert (vo >= 0).all()


def test_reproject_larger_vs_oracle(cuda, port):
    m, n, d, r = 300, 200, 48, 3
    oP, oQ = port.init_sparse(m, d, r, 1), port.init_sparse(n, d, r, 2)
    nP, nQ = port.init_sparse(m, d, r, 3), port.init_sparse(n, d, r, 4)
    rng = np.random.default_rng(0)
    mm, vv = rng.standard_normal((d, d)), rng.standard_normal((d, d)) ** 2
    old, new = dpair(oP, oQ), dpair(nP, nQ)
    for kind in (0, 1):
        a = lsp.AdamState(d, compute="f64")
        a.set(mm, vv, 3)
        lsp.reproject_state(a, old, new, kind)
        mo, vo, _ = a.get()
        mref, vref = port.reproject_state(oP, oQ, nP, nQ, mm, vv, kind)
        assert rel(mo, mref) < 1e-12 and rel(vo, vref) < 1e-12


@pytest.mark.parametrize("transfer", [0, 1])
def test_maybe_update_vs_reference(cuda, reference, transfer):
    """Bias-gated refresh (trainer.cpp:74-112) against the reference's own
    maybe_update: the gate decision, the fresh projectors (indices bit-exact),
    the fit trajectory length and fitted values, the reprojected Adam moments
    and the bias before/after.  fp64 device compute."""
    m, n, d, r_old, r = 64, 48, 16, 4, 3
    P = reference.init_sparse(m, d, r_old, 11)
    Q = reference.init_sparse(n, d, r_old, 12)
    rng = np.random.default_rng(5)
    g = rng.standard_normal((m, n))
    extras = [rng.standard_normal((m, n)), np.zeros((m, n)), rng.standard_normal((m, n))]
    mm, vv = rng.standard_normal((d, d)), rng.standard_normal((d, d)) ** 2
    kw = dict(alpha=0.5, fit_alpha=0.1, step_size=1e-2, max_steps=40, timeout_steps=40,
              transfer=transfer, reinit_seed=99)
    nP, nQ, mref, vref, res_ref = reference.maybe_update(P, Q, mm, vv, 3, g, extras, r, **kw)
    assert res_ref["refreshed"]

    pair = dpair(P, Q)
    adam = lsp.AdamState(d, compute="f64")
    adam.set(mm, vv, 3)
    fit = lsp.FitConfig(alpha=0.1, step_size=1e-2, max_steps=40, timeout_steps=40)
    new_pair, res = lsp.maybe_update(pair, adam, dev(g), [dev(x) for x in extras], r=r,
                                     alpha=0.5, fit=fit, transfer=transfer, reinit_seed=99)
    assert res["refreshed"] and new_pair is not pair
    assert res["fit_steps"] == res_ref["fit_steps"]
    assert res["fit_timed_out"] == res_ref["fit_timed_out"]
    assert abs(res["bias_before"] - res_ref["bias_before"]) < 1e-10 * res_ref["bias_before"]
    assert abs(res["bias_after"] - res_ref["bias_after"]) < 1e-8 * res_ref["bias_after"]
    pp, pv = new_pair.p.get()
    qp, qv = new_pair.q.get()
    assert np.array_equal(pp, nP.pos) and np.array_equal(qp, nQ.pos)
    assert rel(pv, nP.val) < 1e-9 and rel(qv, nQ.val) < 1e-9
    mo, vo, st = adam.get()
    assert st == 3
    assert rel(mo, mref) < 1e-9 and rel(vo, vref) < 1e-9


def test_maybe_update_gate_and_zero_grad(cuda, reference):
    """Bias within alpha: same pair, state untouched; zero gradient: skipped, NaN bias."""
    m, n, d, r = 40, 30, 8, 2
    P, Q = reference.init_sparse(m, d, r, 1), reference.init_sparse(n, d, r, 2)
    g = np.random.default_rng(1).standard_normal((m, n))
    mm, vv = np.ones((d, d)), np.ones((d, d))
    _, _, _, _, res_ref = reference.maybe_update(P, Q, mm, vv, 1, g, [], r, alpha=1e9)
    pair, adam = dpair(P, Q), lsp.AdamState(d, compute="f64")
    adam.set(mm, vv, 1)
    same, res = lsp.maybe_update(pair, adam, dev(g), [], r=r, alpha=1e9)
    assert same is pair and not res["refreshed"] and not res_ref["refreshed"]
    assert abs(res["bias_before"] - res_ref["bias_before"]) < 1e-10 * res_ref["bias_before"]
    mo, vo, _ = adam.get()
    assert np.array_equal(mo, mm) and np.array_equal(vo, vv)
    same, res = lsp.maybe_update(pair, adam, dev(np.zeros((m, n))), [], r=r, alpha=0.1)
    assert same is pair and res["skipped_zero_grad"] and np.isnan(res["bias_before"])


def test_fit_loss_gradient_c3_shape_vs_reference(cuda, reference):
    """BASELINE configs[2] scale: fit_loss and fit_gradient (Eq. 3) on the
    2048 x 5504 MLP shape, d = 1024, r = 4, one target (T = 1), against the
    compiled reference (its dense fit_gradient takes ~20 s per target here,
    SURVEY 7.3(5)).  fp64 device compute, tolerance 1e-10 (loss) / 1e-9
    (gradient: different association of the same sums)."""
    m, n, d, r = 2048, 5504, 1024, 4
    P = reference.init_sparse(m, d, r, reference.derive_seed(1, 0x1A171, 2))
    Q = reference.init_sparse(n, d, r, reference.derive_seed(1, 0x1A171, 3))
    g = np.random.default_rng(2048).standard_normal((m, n))
    cfg = lsp.FitConfig(reg_beta=1e-3)
    pair = dpair(P, Q)
    loss = pair.fit_loss([dev(g)], cfg)
    assert loss == pytest.approx(reference.fit_loss(P, Q, [g], reg_beta=1e-3), rel=1e-10)
    gp, gq = pair.fit_gradient([dev(g)], cfg)
    gp_ref, gq_ref = reference.fit_gradient(P, Q, [g], reg_beta=1e-3)
    assert rel(gp, gp_ref) < 1e-9 and rel(gq, gq_ref) < 1e-9


def test_reproject_d1024_vs_oracle(cuda, port):
    """reproject_state at d = 1024 (the dense d^3 transfer products, k_dgemm) on
    the C3 MLP projectors, against the oracle, both transfer kinds."""
    m, n, d, r = 2048, 5504, 1024, 4
    oP, oQ = port.init_sparse(m, d, r, 1), port.init_sparse(n, d, r, 2)
    nP, nQ = port.init_sparse(m, d, r, 3), port.init_sparse(n, d, r, 4)
    rng = np.random.default_rng(1)
    mm, vv = rng.standard_normal((d, d)) * 1e-3, (rng.standard_normal((d, d)) * 1e-3) ** 2
    old, new = dpair(oP, oQ), dpair(nP, nQ)
    for kind in (0, 1):
        a = lsp.AdamState(d, compute="f64")
        a.set(mm, vv, 100)
        lsp.reproject_state(a, old, new, kind)
        mo, vo, st = a.get()
        mref, vref = port.reproject_state(oP, oQ, nP, nQ, mm, vv, kind)
        assert st == 100
        assert rel(mo, mref) < 1e-12 and rel(vo, vref) < 1e-12

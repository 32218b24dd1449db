"""CPU: pin the oracle (C restatement) to the reference's golden vectors and KATs.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py);
the KATs are the ones the reference's own tests hold (proj/tests/test_subspace_opt.cpp,
test_projector.cpp, test_trainer.cpp).
"""
import hashlib

import numpy as np
import pytest

import oracle

KINIT = 0x1A171


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f32normal(seed, shape, scale=1.0):
    g = np.random.default_rng(seed).standard_normal(shape) * scale
    return g.astype(np.float32).astype(np.float64)


def pair_from(data, k):
    m = len(data[f"{k}_ppos"])
    return data[f"{k}_ppos"], data[f"{k}_pval"], data[f"{k}_qpos"], data[f"{k}_qval"]


def proj(n_rows, d, r, pos, val):
    return oracle.Projector(n_rows, d, r, np.ascontiguousarray(pos, np.int32),
                            np.ascontiguousarray(val, np.float64))


def test_derive_seed_golden(port, golden):
    _, meta = golden
    for s, t, i, want in meta["derive_seed"]:
        assert port.derive_seed(s, t, i) == want


def test_init_sparse_golden_bit_exact(port, golden):
    data, meta = golden
    i = 0
    while f"init{i}" in meta:
        c = meta[f"init{i}"]
        P = port.init_sparse(c["n_rows"], c["d"], c["r"], c["seed"])
        assert sha(P.pos) == c["pos_sha"], f"init{i} positions"
        assert sha(P.val) == c["val_sha"], f"init{i} values"
        k = len(data[f"init{i}_pos"])
        np.testing.assert_array_equal(P.pos[:k], data[f"init{i}_pos"])
        np.testing.assert_array_equal(P.val[:k], data[f"init{i}_val"])
        i += 1
    assert i >= 8


def test_init_sparse_structure(port):
    # proj/tests/test_projector.cpp:51-102
    P = port.init_sparse(10, 8, 3, 42)
    pos = P.pos.reshape(10, 3)
    assert (pos >= 0).all() and (pos < 8).all() and (np.diff(pos, axis=1) > 0).all()
    P = port.init_sparse(4, 4, 4, 7)
    np.testing.assert_array_equal(P.pos.reshape(4, 4), np.tile(np.arange(4), (4, 1)))
    v = port.init_sparse(10000, 64, 4, 123).val
    assert 0.9 / 4 <= v.var() <= 1.1 / 4
    with pytest.raises(oracle.OracleError) as e:
        port.init_sparse(4, 3, 4, 0)
    assert e.value.kind == "invalid_argument"


@pytest.mark.parametrize("ci", range(6))
def test_hot_path_golden_cases(port, golden, ci):
    data, meta = golden
    c = meta["cases"][ci]
    m, n, d, r = c["m"], c["n"], c["d"], c["r"]
    k = f"case{ci}"
    P = proj(m, d, r, data[f"{k}_ppos"], data[f"{k}_pval"])
    Q = proj(n, d, r, data[f"{k}_qpos"], data[f"{k}_qval"])
    g, w = data[f"{k}_g"], data[f"{k}_w"]
    s = port.compress(P, Q, g)
    np.testing.assert_array_equal(s, data[f"{k}_s"])
    np.testing.assert_array_equal(port.decompress(P, Q, s), data[f"{k}_decomp"])
    np.testing.assert_array_equal(port.estimation_bias(P, Q, g), data[f"{k}_bias"])
    assert port.relative_bias(P, Q, g) == c["rel_bias"]
    z = np.zeros((d, d))
    mo, vo, de, st = port.adam_step(z, z, s, 0)
    assert st == 1
    np.testing.assert_array_equal(mo, data[f"{k}_m1"])
    np.testing.assert_array_equal(vo, data[f"{k}_v1"])
    np.testing.assert_array_equal(de, data[f"{k}_delta1"])
    np.testing.assert_array_equal(port.decompress_apply(P, Q, de, 1e-3, w), data[f"{k}_w1"])


def test_c1_golden(port, golden):
    """BASELINE configs[0]: 1024x1024, d=256, r=4 on the trainer seed path."""
    data, meta = golden
    c = meta["c1"]
    P = port.init_sparse(c["m"], c["d"], c["r"], port.derive_seed(1, KINIT, 0))
    Q = port.init_sparse(c["n"], c["d"], c["r"], port.derive_seed(1, KINIT, 1))
    g = f32normal(c["g_seed"], (c["m"], c["n"]))
    w = f32normal(c["w_seed"], (c["m"], c["n"]), 0.02)
    assert sha(g) == c["g_sha"] and sha(w) == c["w_sha"], "numpy bitstream drifted"
    s = port.compress(P, Q, g)
    np.testing.assert_array_equal(s, data["c1_s"])
    z = np.zeros_like(s)
    _, _, de, _ = port.adam_step(z, z, s, 0)
    np.testing.assert_array_equal(de, data["c1_delta1"])
    w1 = port.decompress_apply(P, Q, de, c["lr"], w)
    assert sha(w1) == c["w1_sha"]


def test_adam_kats(port, golden):
    data, _ = golden
    # zero gradient (test_subspace_opt.cpp:35-42)
    z = np.zeros((3, 3))
    mo, vo, de, st = port.adam_step(z, z, z, 0)
    assert st == 1 and not mo.any() and not vo.any() and not de.any()
    # hand-computed first step (test_subspace_opt.cpp:44-51)
    one = np.ones((1, 1))
    mo, vo, de, _ = port.adam_step(0 * one, 0 * one, one, 0)
    ulp4 = 4 * np.finfo(np.float64).eps  # EXPECT_DOUBLE_EQ = within 4 ulps
    assert mo[0, 0] == pytest.approx(0.1, rel=ulp4, abs=0)
    assert vo[0, 0] == pytest.approx(0.001, rel=ulp4, abs=0)
    assert de[0, 0] == pytest.approx(1.0 / (1.0 + 1e-8), rel=ulp4, abs=0)
    # 7-step recurrence with beta=(0.8,0.95), eps=1e-6, vs golden
    m = np.zeros((4, 4))
    v = np.zeros((4, 4))
    st = 0
    for t in range(7):
        m, v, de, st = port.adam_step(m, v, data[f"adam_g{t}"], st, 0.8, 0.95, 1e-6)
        np.testing.assert_array_equal(de, data[f"adam_d{t}"])
    np.testing.assert_array_equal(m, data["adam_m7"])
    np.testing.assert_array_equal(v, data["adam_v7"])
    bad = np.zeros((2, 2))
    bad[0, 0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        port.adam_step(np.zeros((2, 2)), np.zeros((2, 2)), bad, 0)
    assert e.value.kind == "numeric"


def test_fit_golden(port, golden):
    data, meta = golden
    m, n, d, r = 12, 10, 6, 3
    P = proj(m, d, r, data["fit_ppos"], data["fit_pval"])
    Q = proj(n, d, r, data["fit_qpos"], data["fit_qval"])
    targets = list(data["fit_targets"])
    for kind in (0, 1):
        assert port.fit_loss(P, Q, targets, 0.3, kind) == data[f"fit_loss_k{kind}"][0]
        gp, gq = port.fit_gradient(P, Q, targets, 0.3, kind)
        np.testing.assert_array_equal(gp, data[f"fit_gp_k{kind}"])
        np.testing.assert_array_equal(gq, data[f"fit_gq_k{kind}"])
    fp, fq, rep = port.fit(P, Q, targets, alpha=0.5, max_steps=30, timeout_steps=30)
    np.testing.assert_array_equal(fp.val, data["fit_out_pval"])
    np.testing.assert_array_equal(fq.val, data["fit_out_qval"])
    np.testing.assert_array_equal(rep["loss_curve"], data["fit_curve"])
    want = meta["fit_report"]
    assert rep["steps"] == want["steps"] and rep["success"] == want["success"]
    assert rep["final_rel_bias"] == want["final_rel_bias"]


def test_gram_and_reproject_golden(port, golden):
    data, _ = golden
    m, n, d, r = 9, 8, 4, 2
    pr = {nm: proj(m if nm.endswith("P") else n, d, r, data[f"rp_{nm}_pos"], data[f"rp_{nm}_val"])
          for nm in ("oP", "oQ", "nP", "nQ")}
    np.testing.assert_array_equal(port.projector_gram(pr["nP"], pr["oP"]), data["rp_gram"])
    for kind in (0, 1):
        mo, vo = port.reproject_state(pr["oP"], pr["oQ"], pr["nP"], pr["nQ"], data["rp_m"],
                                      data["rp_v"], kind)
        np.testing.assert_array_equal(mo, data[f"rp_m_k{kind}"])
        np.testing.assert_array_equal(vo, data[f"rp_v_k{kind}"])
        assert (vo >= 0).all()


def test_subsample_size_kat(port, golden):
    _, meta = golden
    for g_, b_, m_, n_, t_, dl, want in meta["subsample_size"]:
        assert port.subsample_size(g_, b_, m_, n_, t_, dl) == want


def test_dense_oracle_and_linearity(port):
    """proj/tests/test_projector.cpp:145-156, 208-235: dense agreement and DP linearity."""
    rng = np.random.default_rng(3)
    P = port.init_sparse(7, 6, 4, 1)
    Q = port.init_sparse(6, 6, 4, 2)
    a, b = rng.standard_normal((7, 6)), rng.standard_normal((7, 6))
    dp, dq = P.dense(), Q.dense()
    np.testing.assert_allclose(port.compress(P, Q, a), dp.T @ a @ dq, atol=1e-12)
    lhs = port.compress(P, Q, 1.7 * a - 0.4 * b)
    rhs = 1.7 * port.compress(P, Q, a) - 0.4 * port.compress(P, Q, b)
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_port_matches_compiled_reference(port, reference):
    """Random shapes: the C restatement is bit-identical to the compiled reference."""
    rng = np.random.default_rng(11)
    for trial in range(25):
        m, n = rng.integers(1, 40, size=2)
        d = int(rng.integers(1, 20))
        r = int(rng.integers(1, d + 1))
        seed = int(rng.integers(0, 2**63))
        P = reference.init_sparse(int(m), d, r, seed)
        Q = reference.init_sparse(int(n), d, r, seed ^ 0x5555)
        P2 = port.init_sparse(int(m), d, r, seed)
        np.testing.assert_array_equal(P.pos, P2.pos)
        np.testing.assert_array_equal(P.val, P2.val)
        g = rng.standard_normal((m, n))
        np.testing.assert_array_equal(port.compress(P, Q, g), reference.compress(P, Q, g))
        s = rng.standard_normal((d, d))
        np.testing.assert_array_equal(port.decompress(P, Q, s), reference.decompress(P, Q, s))
        if np.linalg.norm(g) > 0:
            assert port.relative_bias(P, Q, g) == reference.relative_bias(P, Q, g)

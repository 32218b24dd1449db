"""Generate the golden vectors in tests/golden/ from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every array in golden.npz is an output of the unmodified reference library
(oracle/_ref/liblsp_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Inputs are either stored verbatim or regenerated from a
numpy PCG64 seed whose byte hash is stored alongside (tests fail loudly if the
numpy bitstream ever drifts).  Inputs are fp32-representable so that the same
values feed the GPU fp32 path bit-exactly.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

KINIT = 0x1A171  # proj/src/trainer.cpp:23


def f32normal(seed: int, shape, scale: float = 1.0) -> np.ndarray:
    g = np.random.default_rng(seed).standard_normal(shape) * scale
    return g.astype(np.float32).astype(np.float64)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = oracle.Oracle("reference")
    out: dict[str, np.ndarray] = {}
    meta: dict[str, object] = {}

    # --- init_sparse (proj/src/projector.cpp:66-85), incl. the trainer seed path
    init_cases = [(10, 8, 3, 42), (20, 16, 4, 99), (4, 4, 4, 7), (9, 6, 2, 0), (33, 64, 8, 5)]
    for li in range(2):
        init_cases.append((1024, 256, 4, R.derive_seed(1, KINIT, li)))
    init_cases.append((11008, 1024, 4, R.derive_seed(1, KINIT, 1)))
    for i, (n_rows, d, r, seed) in enumerate(init_cases):
        P = R.init_sparse(n_rows, d, r, seed)
        meta[f"init{i}"] = dict(n_rows=n_rows, d=d, r=r, seed=seed, pos_sha=sha(P.pos),
                                val_sha=sha(P.val))
        if n_rows * r <= 4096:
            out[f"init{i}_pos"], out[f"init{i}_val"] = P.pos, P.val
        else:  # keep the first 64 rows verbatim
            out[f"init{i}_pos"], out[f"init{i}_val"] = P.pos[: 64 * r], P.val[: 64 * r]
    meta["derive_seed"] = [[s, t, i, R.derive_seed(s, t, i)]
                           for s, t, i in [(0, 0, 0), (1, KINIT, 0), (1, KINIT, 1),
                                           (123456789, 0x901A01, 0), (2**63 + 5, 7, 99)]]

    # --- small-shape hot-path cases (compress / decompress / apply / bias / adam)
    cases = [(6, 5, 3, 2, 23), (7, 6, 4, 2, 53), (40, 30, 8, 3, 11), (64, 48, 16, 4, 12),
             (33, 70, 32, 4, 13), (128, 96, 32, 1, 14)]
    meta["cases"] = []
    for ci, (m, n, d, r, seed) in enumerate(cases):
        P = R.init_sparse(m, d, r, R.derive_seed(seed, 1))
        Q = R.init_sparse(n, d, r, R.derive_seed(seed, 2))
        g = f32normal(1000 + ci, (m, n))
        w = f32normal(2000 + ci, (m, n), 0.02)
        s = R.compress(P, Q, g)
        m0 = np.zeros((d, d))
        mo, vo, de, st = R.adam_step(m0, m0, s, 0)
        w1 = R.decompress_apply(P, Q, de, 1e-3, w)
        k = f"case{ci}"
        out.update({f"{k}_ppos": P.pos, f"{k}_pval": P.val, f"{k}_qpos": Q.pos,
                    f"{k}_qval": Q.val, f"{k}_g": g, f"{k}_w": w, f"{k}_s": s, f"{k}_m1": mo,
                    f"{k}_v1": vo, f"{k}_delta1": de, f"{k}_w1": w1,
                    f"{k}_decomp": R.decompress(P, Q, s),
                    f"{k}_bias": R.estimation_bias(P, Q, g)})
        meta["cases"].append(dict(m=m, n=n, d=d, r=r, seed=seed,
                                  rel_bias=R.relative_bias(P, Q, g)))

    # --- C1 (BASELINE configs[0]): 1024x1024, s=256, k=4, trainer seed path.
    m = n = 1024
    d, r = 256, 4
    P = R.init_sparse(m, d, r, R.derive_seed(1, KINIT, 0))
    Q = R.init_sparse(n, d, r, R.derive_seed(1, KINIT, 1))
    g = f32normal(7, (m, n))
    w = f32normal(8, (m, n), 0.02)
    s = R.compress(P, Q, g)
    z = np.zeros((d, d))
    _, _, de, _ = R.adam_step(z, z, s, 0)
    w1 = R.decompress_apply(P, Q, de, 1e-3, w)
    meta["c1"] = dict(m=m, n=n, d=d, r=r, g_seed=7, w_seed=8, g_sha=sha(g), w_sha=sha(w),
                      lr=1e-3, w1_sha=sha(w1), rel_bias=R.relative_bias(P, Q, g))
    out.update({"c1_s": s, "c1_delta1": de, "c1_w1_rows": w1[::64].copy(),
                "c1_w1_colsum": w1.sum(axis=0)})

    # --- Adam multi-step (subspace_opt.cpp:35-57), beta=(0.8,0.95), eps=1e-6
    grads = [f32normal(300 + t, (4, 4)) for t in range(7)]
    mm = np.zeros((4, 4))
    vv = np.zeros((4, 4))
    st = 0
    for t, gr in enumerate(grads):
        mm, vv, de, st = R.adam_step(mm, vv, gr, st, 0.8, 0.95, 1e-6)
        out[f"adam_g{t}"], out[f"adam_d{t}"] = gr, de
    out["adam_m7"], out["adam_v7"] = mm, vv

    # --- fit pieces (projector.cpp:189-315)
    m, n, d, r = 12, 10, 6, 3
    P = R.init_sparse(m, d, r, R.derive_seed(71, 1))
    Q = R.init_sparse(n, d, r, R.derive_seed(71, 2))
    targets = [f32normal(400 + t, (m, n)) for t in range(2)]
    out["fit_ppos"], out["fit_pval"], out["fit_qpos"], out["fit_qval"] = P.pos, P.val, Q.pos, Q.val
    out["fit_targets"] = np.stack(targets)
    for kind in (0, 1):
        out[f"fit_loss_k{kind}"] = np.array([R.fit_loss(P, Q, targets, 0.3, kind)])
        gp, gq = R.fit_gradient(P, Q, targets, 0.3, kind)
        out[f"fit_gp_k{kind}"], out[f"fit_gq_k{kind}"] = gp, gq
    fp, fq, rep = R.fit(P, Q, targets, alpha=0.5, max_steps=30, timeout_steps=30)
    out["fit_out_pval"], out["fit_out_qval"] = fp.val, fq.val
    out["fit_curve"] = rep["loss_curve"]
    meta["fit_report"] = {k: (v if not isinstance(v, np.ndarray) else None)
                          for k, v in rep.items()}
    meta["fit_report"]["final_rel_bias"] = float(rep["final_rel_bias"])

    # --- projector_gram / reproject_state (subspace_opt.cpp:59-101)
    m, n, d, r = 9, 8, 4, 2
    oP, oQ = R.init_sparse(m, d, r, 13), R.init_sparse(n, d, r, 17)
    nP, nQ = R.init_sparse(m, d, r, 19), R.init_sparse(n, d, r, 23)
    sm = f32normal(500, (d, d))
    sv = f32normal(501, (d, d)) ** 2
    for nm, pr in (("oP", oP), ("oQ", oQ), ("nP", nP), ("nQ", nQ)):
        out[f"rp_{nm}_pos"], out[f"rp_{nm}_val"] = pr.pos, pr.val
    out["rp_m"], out["rp_v"] = sm, sv
    out["rp_gram"] = R.projector_gram(nP, oP)
    for kind in (0, 1):
        out[f"rp_m_k{kind}"], out[f"rp_v_k{kind}"] = R.reproject_state(oP, oQ, nP, nQ, sm, sv,
                                                                       kind)

    # --- text format (projector.cpp:317-327)
    meta["save_projector"] = R.save_projector(R.init_sparse(5, 7, 3, 113))
    meta["subsample_size"] = [[g_, b_, m_, n_, t_, dl, R.subsample_size(g_, b_, m_, n_, t_, dl)]
                              for g_, b_, m_, n_, t_, dl in [(1.0, 0.5, 16, 16, 1000, 0.1),
                                                             (2.5, 0.3, 64, 32, 100, 0.05)]]

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays;",
          os.path.getsize(os.path.join(HERE, "golden.npz")) // 1024, "KiB")


if __name__ == "__main__":
    main()

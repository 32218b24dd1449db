"""CPU: the schedule-model calibration (paper_2406_10181_b200/calibrate.py)
against the reference's own schedule model (proj/src/schedule_sim.cpp, compiled
into oracle/_ref): the restated closed forms are bit-identical on random
profiles, and a profile built from B200 layer times is accepted by the
reference's load_profile and simulated."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2406_10181_b200 import calibrate as cal


def _ref():
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    o = oracle.Oracle("reference")
    if not o.has_schedule():
        pytest.skip("oracle/_ref built without schedule_sim (no nlohmann/json)")
    return o


def _random_profile(rng, L, duplex):
    v = lambda scale: list(rng.uniform(0, scale, L))  # noqa: E731
    return cal.TimingProfile(
        n_layers=L, fwd_gpu=v(1e-3), bwd_gpu=v(2e-3), upd_gpu=v(1e-3), fwd_cpu=v(1e-3),
        bwd_cpu=v(1e-3), upd_cpu=v(5e-3), grad_bytes=v(1e8), delta_bytes=v(1e8),
        bandwidth_d2h=float(rng.uniform(1e9, 5e10)), bandwidth_h2d=float(rng.uniform(1e9, 5e10)),
        duplex=duplex, bytes_per_element=4.0)


@pytest.mark.parametrize("seed", range(6))
def test_closed_forms_match_reference(seed):
    ref = _ref()
    rng = np.random.default_rng(seed)
    prof = _random_profile(rng, int(rng.integers(1, 40)), bool(seed % 2))
    d = int(rng.integers(16, 2048))
    r = ref.schedule_eval(prof, d)
    assert cal.transition_layer(prof) == r["transition_layer"]
    assert cal.closed_form_lsp(prof, d) == r["closed_form_lsp"]
    assert cal.closed_form_zero(prof) == r["closed_form_zero"]


def test_transition_layer_edge_cases():
    ref = _ref()
    L = 4
    zero = cal.TimingProfile(n_layers=L, fwd_gpu=[0.0] * L, bwd_gpu=[1e-3] * L, upd_gpu=[0.0] * L,
                             fwd_cpu=[0.0] * L, bwd_cpu=[0.0] * L, upd_cpu=[0.0] * L,
                             grad_bytes=[0.0] * L, delta_bytes=[0.0] * L, bandwidth_d2h=1.0,
                             bandwidth_h2d=1.0)
    assert cal.transition_layer(zero) == ref.schedule_eval(zero, 0)["transition_layer"] == 0.0
    zero.bwd_gpu = [0.0] * L
    assert cal.transition_layer(zero) == ref.schedule_eval(zero, 0)["transition_layer"] == L
    with pytest.raises(ValueError):
        cal.lsp_rescale(zero, 0)
    bad = cal.TimingProfile(**{**zero.__dict__, "bandwidth_d2h": 0.0})
    with pytest.raises(ValueError):
        bad.validate()
    with pytest.raises(oracle.OracleError):
        ref.schedule_eval(bad, 8)


@pytest.mark.parametrize("world", [1, 8])
def test_b200_profile_runs_in_reference_simulator(tmp_path, world):
    """C4-like layer times (32 layers, 0.35 ms compress, 0.49 ms update, 7 S
    buffers of 1024^2 fp32 per layer, 700 GB/s bus bandwidth): the reference
    accepts the file, and its lsp_layerwise simulation agrees with the B200
    estimate (device chain plus one exposed all-reduce) within one layer."""
    ref = _ref()
    L = 32
    prof = cal.b200_profile([0.35e-3] * L, [0.49e-3] * L, [7 * 1024 * 1024 * 4.0] * L, world,
                            700e9, fwd_s=[0.2e-3] * L, bwd_s=[0.4e-3] * L)
    path = os.path.join(tmp_path, "b200.json")
    cal.save_profile(prof, path)
    doc = json.load(open(path))
    assert set(doc) == {"n_layers", "fwd_gpu", "bwd_gpu", "upd_gpu", "fwd_cpu", "bwd_cpu",
                        "upd_cpu", "grad_bytes", "delta_bytes", "bandwidth_d2h",
                        "bandwidth_h2d", "duplex", "mem_total", "mem_gpu", "bytes_per_element"}
    sim = ref.schedule_file(path)
    assert sim["n_layers"] == L
    assert sim["transition_layer"] == cal.transition_layer(prof)
    est = cal.step_estimate(prof)
    layer = (0.2 + 0.4 + 0.35 + 0.49) * 1e-3
    assert abs(sim["iter_lsp_layerwise"] - est["estimate_s"]) <= layer
    if world == 1:
        assert est["allreduce_s"] == 0.0
        assert sim["iter_lsp_layerwise"] == pytest.approx(est["device_s"], rel=1e-9)


def test_b200_profile_rescale_invariant():
    """With d given, the reference CLI path (lsp_rescale before simulate, as
    lspkit sim --policy lsp_layerwise --d does) sees the same link times."""
    ref = _ref()
    L, d = 16, 1024
    prof = cal.b200_profile([0.35e-3] * L, [0.49e-3] * L, [7 * d * d * 4.0] * L, 8, 700e9,
                            bwd_s=[0.4e-3] * L, d=d)
    resc = cal.lsp_rescale(prof, d)
    assert resc.grad_bytes == pytest.approx(prof.grad_bytes, rel=1e-12)
    a = ref.schedule_eval(prof, d)
    b = ref.schedule_eval(resc, d)
    assert b["iter_lsp_layerwise"] == pytest.approx(a["iter_lsp_layerwise"], rel=1e-9)
    # the rescaled upload (payload / 1e18 B/s) adds ~1e-10 s
    assert a["closed_form_lsp"] == pytest.approx(cal.closed_form_b200(prof), rel=1e-6)

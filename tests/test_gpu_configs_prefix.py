"""Configs 3-5 against the oracle on the prefix of layers the oracle finishes in seconds (SURVEY
§4.2 item 5(i)): the full-size chains (N = 50 / 40 / 300), the full circuits' ledgers (n_planned of
the whole circuit, cap 4096), the first layers while chi stays small. Same bars as config 1:
kept ranks identical (near-ties excused), estimate within 1e-5, spectra within the trajectory
tolerance, and the strict sigma bar on the first layer (identical inputs)."""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import EST_ATOL, SIG_RTOL, compare_layer

pytestmark = pytest.mark.gpu


def _run_prefix(cfg_id, n_prefix, slab=4 << 30):
    import paper_2307_16870_b200 as pk
    cfg = workloads.CONFIGS[cfg_id]
    N, depth, d = cfg["n_sites"], cfg["depth"], cfg["d"]
    if cfg["kind"] == "mpo":
        layers = workloads.mpo_circuit(cfg_id, N, depth, cfg["p_depol"])
        rule = "wang"
    else:
        layers = workloads.brickwork_circuit(cfg_id, N, depth)
        rule = "pure"
    npl = workloads.n_two_qubit_gates(layers)
    kw = dict(d=d, f_min=cfg["f_min"], n_planned=npl, strategy=cfg["strategy"], rule=rule, chi_cap=cfg["chi_cap"])
    gpu = pk.MPS(N, slab_bytes=slab, **kw)
    orc = oracle.OracleMPS(N, **kw)
    worst = 0.0
    for t, (sites, us) in enumerate(layers[:n_prefix]):
        gpu.mps_apply_layer(sites, us)
        orc.apply_layer(sites, us)
        if t == 0:
            w0, _ = compare_layer(gpu, orc, len(sites), rule=rule)
            assert w0 < SIG_RTOL, w0
        w, same = compare_layer(gpu, orc, len(sites), rule=rule, traj=True)
        worst = max(worst, w)
        assert same, "kept-rank mismatch at layer %d (near-tie): trajectories diverge" % t
        assert list(gpu.mps_bond_dims()) == list(orc.bond_dims())
        eg, eo = gpu.mps_fidelity_estimate(), orc.estimate()
        assert abs(eg["est"] - eo["est"]) < EST_ATOL
    assert worst <= 1.0, worst
    return gpu, orc


def test_config3_prefix():
    """N = 50, Haar brickwork depth 20, F_min = 0.9, cap 4096: layers 0-5 (chi <= 64)."""
    gpu, orc = _run_prefix(3, 6)
    # the per-gate budget (t = 0.99978) already truncates at layer 3: the bulk settles near
    # chi ~ 20 (measured on the oracle), so the prefix exercises real cuts, not the exact regime
    assert max(gpu.mps_bond_dims()) >= 16
    assert sum(r["discarded_weight"] > 0 for r in gpu.mps_truncation_log()) > 0


def test_config4_mpo_prefix():
    """MPO N = 40, depth 16, p = 0.01, F_min = 0.95 (wang): layers 0-2."""
    gpu, orc = _run_prefix(4, 3)
    assert gpu.mps_fidelity_estimate()["is_lower_bound"]


def test_config5_prefix():
    """N = 300, depth 75, F_min = 0.9: layers 0-4 (150 / 149 gates per layer)."""
    gpu, orc = _run_prefix(5, 5, slab=8 << 30)
    assert len(gpu.mps_truncation_log()) == 150 + 149 + 150 + 149 + 150

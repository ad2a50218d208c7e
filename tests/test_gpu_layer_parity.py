"""Identical-input per-layer parity along whole trajectories (configs 1, 3, 4, 5 and the MPO).

Before every layer the GPU's state -- every site tensor B_i, every Schmidt vector lambda_b and
the ledger (log E, j, guarantee) -- is exported through the C ABI and imported into a FRESH
complex128 oracle (a "mirror"); both then apply the same layer and every gate is compared at
the north-star bars (BASELINE.json north_star), with no absolute floor:
  * singular values: relative 1e-5 for sigma >= 1e-6 sigma_max (the sorted spectrum of theta,
    PAPER.md:114 "performing its SVD ... singular values in decreasing order");
  * kept rank: identical, except where the oracle's normalised cut margin is <= 1e-6
    (reading 8, a near-tie);
  * per-truncation fidelity f_j (E10/E11) and issued target t_j (E14 +
    strategy) to 1e-6; the running estimate (E12) to 1e-5 after the layer.
Because the inputs of every layer are identical on both sides, the complex64 storage drift of a
free-running trajectory (reading 18) never enters: this is the strict bar at every
layer, at every theta size the trajectory reaches (the t = 0 layer of a product state only has
2x2 / 4x4 thetas). The exported complex64 tensors are upcast exactly by the oracle.
"""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import EST_ATOL, SIG_RTOL, near_tie, spectra_close

pytestmark = pytest.mark.gpu

F_ATOL = 1e-6


def _pk():
    import paper_2307_16870_b200 as pk
    return pk


def mirror(gpu, N, kw):
    """A fresh oracle holding exactly the GPU's state and ledger (complex64 -> complex128 exact)."""
    orc = oracle.OracleMPS(N, **kw)
    for i in range(N):
        orc.import_site(i, gpu.mps_export_site(i))
    for b in range(N - 1):
        orc.set_lambda(b, gpu.mps_schmidt_values(b).astype(np.float64))
    le, j, gu = gpu.mps_ledger_get()
    orc.set_ledger(le, j, gu)
    return orc


def compare_identical(gpu, orc, n_gates, rule):
    """Strict per-gate comparison of the most recent layer. Returns (worst sigma error, #near-ties,
    largest theta dimension seen)."""
    recs_g = gpu.mps_truncation_log()[-n_gates:]
    recs_o = orc.records()[-n_gates:]
    worst, ties, big = 0.0, 0, 0
    for g in range(n_gates):
        so = orc.last_spectrum(g)
        sg = gpu.mps_last_spectrum(g)
        big = max(big, so.size)
        err = spectra_close(sg, so)
        assert err < SIG_RTOL, (g, err, so.size)
        worst = max(worst, err)
        rg, ro = recs_g[g], recs_o[g]
        assert rg["bond"] == ro["bond"] and rg["chi_before"] == ro["chi_before"], (g, rg, ro)
        assert abs(rg["target_f"] - ro["target_f"]) < F_ATOL, (g, rg, ro)
        if rg["chi_after"] != ro["chi_after"]:
            assert near_tie(so, ro["target_f"], ro["chi_after"], rule), (g, rg, ro)
            ties += 1
            continue
        assert abs(rg["achieved_f"] - ro["achieved_f"]) < F_ATOL, (g, rg, ro)
        assert rg["capped"] == ro["capped"]
    return worst, ties, big


def run_identical(layers, N, kw, rule, slab=1 << 30, min_theta=0):
    pk = _pk()
    gpu = pk.MPS(N, slab_bytes=slab, **kw)
    worst, ties, big = 0.0, 0, 0
    for t, (sites, us) in enumerate(layers):
        orc = mirror(gpu, N, kw)
        gpu.mps_apply_layer(sites, us)
        orc.apply_layer(sites, us)
        w, k, b = compare_identical(gpu, orc, len(sites), rule)
        worst, ties, big = max(worst, w), ties + k, max(big, b)
        eg, eo = gpu.mps_fidelity_estimate(), orc.estimate()
        assert abs(eg["est"] - eo["est"]) < EST_ATOL, (t, eg, eo)
        assert eg["n_done"] == eo["n_done"] and bool(eg["guarantee_held"]) == bool(eo["guarantee_held"])
        orc.close()
    assert big >= min_theta, big   # the trajectory really reached large thetas
    return gpu, worst, ties


@pytest.mark.parametrize("strategy", ["global", "naive", "nearest"])
def test_config1_every_layer_identical_inputs(strategy):
    """config 1 (N = 12, depth 8, F_min = 0.99) with each target strategy of PAPER.md:153."""
    cfg = workloads.CONFIGS[1]
    N = cfg["n_sites"]
    layers = workloads.brickwork_circuit(1, N, cfg["depth"])
    kw = dict(f_min=cfg["f_min"], n_planned=workloads.n_two_qubit_gates(layers), strategy=strategy)
    gpu, worst, ties = run_identical(layers, N, kw, "pure", slab=256 << 20, min_theta=32)
    print("config1 %s: worst sigma err %.2e, near-ties %d" % (strategy, worst, ties))


@pytest.mark.parametrize("rule", ["wang", "ratio"])
def test_mpo_every_layer_identical_inputs(rule):
    """MPO (d = 4) N = 6, depth 6, p = 0.01: the Wang rule (E11 read as E9) and the ratio rule."""
    N, depth = 6, 6
    layers = workloads.mpo_circuit(4, N, depth, 0.01)
    kw = dict(d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates(layers), strategy="global", rule=rule)
    gpu, worst, ties = run_identical(layers, N, kw, rule, slab=256 << 20, min_theta=64)
    assert gpu.mps_fidelity_estimate()["is_lower_bound"]
    print("mpo %s: worst sigma err %.2e, near-ties %d" % (rule, worst, ties))


@pytest.mark.parametrize("strategy", ["naive", "nearest"])
def test_mpo_strategies_identical_inputs(strategy):
    N, depth = 6, 5
    layers = workloads.mpo_circuit(4, N, depth, 0.01)
    kw = dict(d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates(layers), strategy=strategy)
    run_identical(layers, N, kw, "wang", slab=256 << 20)


def _cfg_layers(cfg_id, n_layers):
    cfg = workloads.CONFIGS[cfg_id]
    N, depth, d = cfg["n_sites"], cfg["depth"], cfg["d"]
    if cfg["kind"] == "mpo":
        full = workloads.mpo_circuit(cfg_id, N, depth, cfg["p_depol"])
        rule = "wang"
    else:
        full = workloads.brickwork_circuit(cfg_id, N, depth)
        rule = "pure"
    kw = dict(d=d, f_min=cfg["f_min"], n_planned=workloads.n_two_qubit_gates(full), strategy=cfg["strategy"],
              rule=rule, chi_cap=cfg["chi_cap"])
    return N, full[:n_layers], kw, rule


def test_config3_every_layer_identical_inputs():
    """N = 50, depth 20, F_min = 0.9, cap 4096: layers 0-9 (bond dims to ~100, theta to ~200)."""
    N, layers, kw, rule = _cfg_layers(3, 10)
    run_identical(layers, N, kw, rule, slab=2 << 30, min_theta=128)


def test_config4_every_layer_identical_inputs():
    """MPO N = 40, depth 16, p = 0.01, F_min = 0.95 (wang): layers 0-3 (the noise keeps the bulk
    chi near 15 after layer 2; theta to ~240)."""
    N, layers, kw, rule = _cfg_layers(4, 4)
    gpu, _, _ = run_identical(layers, N, kw, rule, slab=2 << 30, min_theta=64)
    assert gpu.mps_fidelity_estimate()["is_lower_bound"]


def test_config5_every_layer_identical_inputs():
    """N = 300, depth 75, F_min = 0.9, cap 4096: layers 0-7 (150 / 149 gates each, bond dims to
    ~61, theta to ~122)."""
    N, layers, kw, rule = _cfg_layers(5, 8)
    run_identical(layers, N, kw, rule, slab=8 << 30, min_theta=96)


def sampled_gate_check(gpu, sites, us, picks, rule="pure"):
    """Apply one layer on the GPU; re-run the picked gates on 2-site oracles holding exactly the
    GPU's inputs (B_i, B_{i+1}, lambda_{i-1}) at the target the GPU issued."""
    saved = []
    for g in picks:
        i = int(sites[g])
        lam = gpu.mps_schmidt_values(i - 1) if i > 0 else np.ones(1, np.float32)
        saved.append((g, gpu.mps_export_site(i), gpu.mps_export_site(i + 1), lam, us[g]))
    gpu.mps_apply_layer(sites, us)
    recs = gpu.mps_truncation_log()[-len(sites):]
    worst = 0.0
    for g, BL, BR, lam, U in saved:
        rec = recs[g]
        orc = oracle.OracleMPS(2, d=gpu.d, strategy="fixed", f_fixed=rec["target_f"], rule=rule)
        orc.import_site(0, BL)
        orc.import_site(1, BR)
        orc.set_lambda(-1, lam.astype(np.float64))
        orc.apply_layer(np.zeros(1, np.int32), U[None])
        so, sg = orc.last_spectrum(0), gpu.mps_last_spectrum(g)
        err = spectra_close(sg, so)
        assert err < SIG_RTOL, (g, err, BL.shape, BR.shape)
        worst = max(worst, err)
        ro = orc.records()[0]
        if ro["chi_after"] != rec["chi_after"]:
            assert near_tie(so, rec["target_f"], ro["chi_after"], rule), (g, rec, ro)
        else:
            assert abs(ro["achieved_f"] - rec["achieved_f"]) < F_ATOL, (g, rec, ro)
        orc.close()
    return worst


def test_config3_deep_layers_sampled_gates():
    """Config 3 beyond the mirrored prefix: layers 10-12 run on the GPU (bond dims to ~210, the
    QR and tcgen05 regimes), and in each of them the gate with the largest theta and a median
    one are re-run on the oracle from identical inputs."""
    pk = _pk()
    N, layers, kw, rule = _cfg_layers(3, 13)
    gpu = pk.MPS(N, slab_bytes=4 << 30, **kw)
    for sites, us in layers[:10]:
        gpu.mps_apply_layer(sites, us)
    for sites, us in layers[10:]:
        dims = gpu.mps_bond_dims()
        size = np.array([dims[i - 1] * dims[i + 1] if 0 < i < N - 2 else 0 for i in sites])
        order = np.argsort(size)
        picks = sorted({int(order[-1]), int(order[len(order) // 2])})
        sampled_gate_check(gpu, sites, us, picks, rule)


# ---- NEXT-2: the fixed-chi baseline of the paper's Fig. 4 protocol -- the same
# kernels with fidelity targeting off (F_min = 1: exact mode, t = 1) and the bond cap chi_max = the
# EA run's peak chi (PAPER.md:195 caption, :201-203). Truncations then come from the cap alone; the
# ledger still records f_j = 1 - T_k/P of every capped cut (E10) and the guarantee is lost (:214).
def test_fixed_chi_baseline_every_layer_identical_inputs():
    cfg = workloads.CONFIGS[1]
    N = cfg["n_sites"]
    layers = workloads.brickwork_circuit(1, N, cfg["depth"])
    npl = workloads.n_two_qubit_gates(layers)
    # the EA run's peak chi (config 1, F_min = 0.99) sets the fixed cap
    ea = _pk().MPS(N, f_min=cfg["f_min"], n_planned=npl, strategy="global", slab_bytes=256 << 20)
    ea.run(layers)
    chi_peak = int(max(ea.mps_bond_dims()))
    kw = dict(f_min=1.0, n_planned=npl, strategy="global", chi_cap=chi_peak)
    gpu, worst, ties = run_identical(layers, N, kw, "pure", slab=256 << 20, min_theta=16)
    recs = gpu.mps_truncation_log()
    assert any(r["capped"] for r in recs)                 # the cap is what truncates
    assert max(gpu.mps_bond_dims()) == chi_peak
    assert not gpu.mps_fidelity_estimate()["guarantee_held"]
    print("fixed chi = %d: worst sigma err %.2e, near-ties %d, est %.6f (EA %.6f)"
          % (chi_peak, worst, ties, gpu.mps_fidelity_estimate()["est"], ea.mps_fidelity_estimate()["est"]))


# ---- NEXT-3: paper-faithful noisy workloads on the GPU -- one-qubit layers
# (mps_apply_layer1), the two-qubit depolarising channel fused into the superoperator, and the
# alternating one-/two-qubit circuits of PAPER.md:201 with eps_1 = eps_2 noise,
# every layer on identical inputs against the oracle.
def run_identical_mixed(layers, N, kw, rule, slab=1 << 30):
    pk = _pk()
    gpu = pk.MPS(N, slab_bytes=slab, **kw)
    d = kw.get("d", 2)
    n2 = 0
    for sites, us in layers:
        orc = mirror(gpu, N, kw)
        if np.asarray(us).shape[-1] == d:        # a one-qubit layer: compare the site tensors
            gpu.mps_apply_layer1(sites, us)
            orc.apply_layer1(sites, us)
            for i in sites:
                g, o = gpu.mps_export_site(int(i)), orc.export_site(int(i))
                assert np.abs(g - o).max() <= 1e-6 * max(1e-30, np.abs(o).max()), int(i)
        else:
            gpu.mps_apply_layer(sites, us)
            orc.apply_layer(sites, us)
            compare_identical(gpu, orc, len(sites), rule)
            eg, eo = gpu.mps_fidelity_estimate(), orc.estimate()
            assert abs(eg["est"] - eo["est"]) < EST_ATOL
            n2 += len(sites)
        orc.close()
    return gpu, n2


def test_alternating_mps_every_layer_identical_inputs():
    N, depth = 12, 6
    layers = workloads.alternating_circuit(6, N, depth, "mps")
    kw = dict(f_min=0.99, n_planned=workloads.n_two_qubit_gates_any(layers, 2), strategy="global")
    gpu, n2 = run_identical_mixed(layers, N, kw, "pure", slab=256 << 20)
    assert gpu.mps_fidelity_estimate()["n_done"] == n2


def test_alternating_noisy_mpo_every_layer_identical_inputs():
    N, depth = 8, 5
    layers = workloads.alternating_circuit(7, N, depth, "mpo", eps1=0.05, eps2=0.05)
    kw = dict(d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates_any(layers, 4), strategy="global", rule="wang")
    gpu, n2 = run_identical_mixed(layers, N, kw, "wang", slab=512 << 20)
    assert gpu.mps_fidelity_estimate()["is_lower_bound"]

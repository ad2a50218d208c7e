"""GPU parity: the CUDA path (through the C ABI) against the complex128 oracle on identical seeded
inputs, at the north-star tolerances (BASELINE.json north_star):
  * singular values: relative 1e-5 for sigma >= 1e-6 sigma_max
  * retained bond dimensions: identical except where the cut is a near-tie (oracle's normalised
    margin <= 1e-6, reading 8)
  * cumulative fidelity estimate: absolute 1e-5
  * final-state overlap with the oracle state: >= 1 - 1e-5 (12-qubit config 1)
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

SIG_RTOL = 1e-5
EST_ATOL = 1e-5
# Along a FREE-RUNNING multi-layer trajectory both sides evolve their own state: the oracle in
# complex128, the GPU in complex64 storage, so from the second layer on their thetas differ by the
# accumulated storage rounding (an absolute perturbation of ~1e-7..1e-6 sigma_max after 6-8 layers;
# DESIGN.md reading 18 "Parity on trajectories"). The strict north-star bar is therefore applied where
# the inputs are identical: every layer of tests/test_gpu_layer_parity.py (the oracle re-imports the
# GPU's state before each layer), the config-2 updates and every first layer here. The free-running
# comparison below is a SECONDARY check with relative 1e-5 on top of that absolute floor.
TRAJ_FLOOR = 2e-6


def _pk():
    import paper_2307_16870_b200 as pk
    return pk


def spectra_close(g, o, rtol=SIG_RTOL):
    g = np.asarray(g, float)
    o = np.asarray(o, float)
    assert g.shape == o.shape
    mask = o >= 1e-6 * o[0]
    rel = np.abs(g[mask] - o[mask]) / o[mask]
    return float(rel.max()) if rel.size else 0.0


def near_tie(sig_sorted, t, k, rule="pure"):
    s2 = np.asarray(sig_sorted, float) ** 2
    T = np.concatenate([np.cumsum(s2[::-1])[::-1], [0.0]])
    P = T[0]
    tau = 1 - t if rule != "wang" else 1 - t * t
    m = [abs(T[k] - tau * P)]
    if k >= 1:
        m.append(abs(T[k - 1] - tau * P))
    return min(m) / P <= 1e-6


def traj_ratio(g, o, floor=TRAJ_FLOOR):
    """max_j |g_j - o_j| / (1e-5 o_j + floor o_0) over sigma_j >= 1e-6 sigma_0 (<= 1 passes)."""
    g = np.asarray(g, float)
    o = np.asarray(o, float)
    mask = o >= 1e-6 * o[0]
    return float((np.abs(g - o)[mask] / (SIG_RTOL * o[mask] + floor * o[0])).max())


def compare_layer(gpu, orc, n_gates, rule="pure", traj=False):
    """per-gate spectra, kept ranks and fidelities of the most recent layer. Returns the worst
    relative sigma error (traj=False) or the worst trajectory ratio (traj=True, must be <= 1)."""
    recs_g = gpu.mps_truncation_log()[-n_gates:]
    recs_o = orc.records()[-n_gates:]
    worst = 0.0
    for g in range(n_gates):
        so = orc.last_spectrum(g)
        sg = gpu.mps_last_spectrum(g)
        worst = max(worst, traj_ratio(sg, so) if traj else spectra_close(sg, so))
        rg, ro = recs_g[g], recs_o[g]
        assert rg["bond"] == ro["bond"]
        if rg["chi_after"] != ro["chi_after"]:
            assert near_tie(so, ro["target_f"], ro["chi_after"], rule), (g, rg, ro)
            return worst, False
        assert abs(rg["achieved_f"] - ro["achieved_f"]) < 1e-6
        assert abs(rg["target_f"] - ro["target_f"]) < 1e-6  # t_j depends on E_{j-1} (global)
    return worst, True


def test_config1_parity():
    """config 1: N=12, brickwork depth 8, Haar U(4), F_min = 0.99, global strategy."""
    pk = _pk()
    cfg = workloads.CONFIGS[1]
    N, depth = cfg["n_sites"], cfg["depth"]
    layers = workloads.brickwork_circuit(1, N, depth)
    npl = workloads.n_two_qubit_gates(layers)
    gpu = pk.MPS(N, f_min=cfg["f_min"], n_planned=npl, strategy="global", slab_bytes=256 << 20)
    orc = oracle.OracleMPS(N, f_min=cfg["f_min"], n_planned=npl, strategy="global")
    worst = 0.0
    for t, (sites, us) in enumerate(layers):
        gpu.mps_apply_layer(sites, us)
        orc.apply_layer(sites, us)
        if t == 0:  # identical inputs: the strict bar
            w0, _ = compare_layer(gpu, orc, len(sites))
            assert w0 < SIG_RTOL, w0
        w, same = compare_layer(gpu, orc, len(sites), traj=True)
        worst = max(worst, w)
        assert same, "rank mismatch on a near-tie: trajectories diverge"
        assert list(gpu.mps_bond_dims()) == list(orc.bond_dims())
        eg, eo = gpu.mps_fidelity_estimate(), orc.estimate()
        assert abs(eg["est"] - eo["est"]) < EST_ATOL
    assert worst <= 1.0, worst
    sg, so = gpu.mps_to_statevector(), orc.statevector()
    ov = abs(np.vdot(so, sg)) ** 2 / (np.vdot(so, so).real * np.vdot(sg, sg).real)
    assert ov >= 1 - 1e-5, ov
    # also against the exact 4096-amplitude statevector (BASELINE configs[0]): the estimate
    # approximates the true fidelity (E12)
    import bruteforce as bf
    exact = bf.run_circuit(N, layers).ravel()
    f_true = bf.pure_fidelity(exact, sg)
    assert abs(gpu.mps_fidelity_estimate()["est"] - f_true) < 0.05
    # amplitude == statevector entry
    digits = [0, 1] * (N // 2)
    idx = int("".join(map(str, digits)), 2)
    assert abs(gpu.mps_amplitude(digits) - sg[idx]) < 1e-6


def test_exact_mode_statevector_vs_dense():
    import bruteforce as bf
    pk = _pk()
    N, depth = 10, 6
    layers = workloads.brickwork_circuit(1, N, depth)
    gpu = pk.MPS(N, f_min=1.0, n_planned=workloads.n_two_qubit_gates(layers), slab_bytes=256 << 20)
    gpu.run(layers)
    psi = bf.run_circuit(N, layers).ravel()
    psi /= np.linalg.norm(psi)
    sg = gpu.mps_to_statevector()
    assert np.abs(sg / np.linalg.norm(sg) - psi).max() < 2e-5
    assert abs(np.linalg.norm(sg) - 1) < 1e-4


def _micro(chi, count, t=0.9999, rule="pure", route=0):
    pk = _pk()
    tensors, gates = workloads.micro_chain(chi, count)
    N = 2 * count
    gpu = pk.MPS(N, strategy="fixed", f_fixed=t, rule=rule, slab_bytes=max(256 << 20, 40 * count * (2 * chi) ** 2 * 8))
    gpu.mps_set_svd_route(route)
    gpu.mps_import_sites(0, tensors)
    orc = oracle.OracleMPS(N, strategy="fixed", f_fixed=t, rule=rule)
    for i, B in enumerate(tensors):
        orc.import_site(i, B)
    sites = np.arange(0, N, 2, dtype=np.int32)
    gpu.mps_apply_layer(sites, gates)
    orc.apply_layer(sites, gates)
    return gpu, orc, count


@pytest.mark.parametrize("chi,count", [(16, 64), (64, 8)])
def test_config2_microbench_parity(chi, count):
    gpu, orc, G = _micro(chi, count)
    worst, _ = compare_layer(gpu, orc, G)
    assert worst < SIG_RTOL, worst
    closed = {16: 29, 64: 58}[chi]
    ks = [r["chi_after"] for r in gpu.mps_truncation_log()]
    assert all(abs(k - closed) <= 2 for k in ks), ks  # ~ the closed-form rank (rounding perturbs)


def test_config2_chi256_blocked_path_parity():
    gpu, orc, G = _micro(256, 2)
    worst, _ = compare_layer(gpu, orc, G)
    assert worst < SIG_RTOL, worst


@pytest.mark.parametrize("chi,count", [(128, 2), (256, 2), (512, 1)])
def test_config2_tensor_core_path_parity(chi, count):
    """the tcgen05 3xTF32 block Jacobi + FP64-anchored polish (large regime, chi >= 128 in config 2;
    route 1 = the Jacobi route also for 128 < n <= 4096) at the strict bar: relative 1e-5 on every
    sigma >= 1e-6 sigma_max (sigma_min / sigma_max = (2 chi)^-1.5 = 3e-5 at chi = 512), identical
    kept ranks, f to 1e-6."""
    gpu, orc, G = _micro(chi, count, route=1)
    worst, same = compare_layer(gpu, orc, G)
    assert same
    assert worst < SIG_RTOL, worst
    assert all(gpu.mps_last_sweeps(g) > 0 for g in range(G))


def _two_site(L, R):
    """sum_j L[:, :, j] R[j, :, :] as a (l d) x (d r) matrix (B_i' = Gamma_i lambda_i carries the
    Schmidt values): gauge-invariant -- a phase or, for degenerate lambda, a unitary mixing of the
    bond index cancels between L and R."""
    L, R = L.astype(np.complex128), R.astype(np.complex128)
    k = L.shape[2]
    return L.reshape(-1, k) @ R.reshape(k, -1)


@pytest.mark.parametrize("chi,count", [(128, 2), (256, 2), (512, 1)])
def test_config2_eigen_route_parity(chi, count):
    """the eigen route (default for large-regime theta with 128 < n <= 4096, refine_large.cu): sigma^2 = FP64 eigenvalues of
    the Gram of the FP64-recontracted theta, the kept right singular vectors by inverse iteration +
    back-transformation. Strict bar on sigma, ranks and f; the reabsorbed two-site tensor
    B_i' diag(lambda) B_{i+1}' (gauge-invariant) equals the oracle's to 1e-5 relative, and the new
    right factor is right-normalised."""
    gpu, orc, G = _micro(chi, count, route=0)
    worst, same = compare_layer(gpu, orc, G)
    assert same
    assert worst < SIG_RTOL, worst
    assert all(gpu.mps_last_sweeps(g) == 0 for g in range(G))     # no Jacobi sweeps: the eigen route
    for g in range(G):
        Mg = _two_site(gpu.mps_export_site(2 * g), gpu.mps_export_site(2 * g + 1))
        Mo = _two_site(orc.export_site(2 * g), orc.export_site(2 * g + 1))
        rel = np.linalg.norm(Mg - Mo) / np.linalg.norm(Mo)
        assert rel < 1e-5, (g, rel)
        R = gpu.mps_export_site(2 * g + 1).astype(np.complex128)
        Rm = R.reshape(R.shape[0], -1)
        assert np.abs(Rm @ Rm.conj().T - np.eye(R.shape[0])).max() < 1e-5


def test_hastings_update_keeps_state():
    """no truncation (t = 1): the reabsorbed pair reproduces Theta' (gauge-invariant check)."""
    pk = _pk()
    tensors, gates = workloads.micro_chain(8, 4)
    gpu = pk.MPS(8, strategy="fixed", f_fixed=1.0, slab_bytes=64 << 20)
    gpu.mps_import_sites(0, tensors)
    gpu.mps_apply_layer(np.arange(0, 8, 2, dtype=np.int32), gates)
    for g in range(4):
        L = gpu.mps_export_site(2 * g).astype(np.complex128)
        R = gpu.mps_export_site(2 * g + 1).astype(np.complex128)
        l, _, k = L.shape
        prod = L.reshape(-1, k) @ R.reshape(k, -1)
        # expected Theta' = G_U(B_L B_R) / nu with nu = ||theta|| = 1 (lambda = 1)
        BL, BR = tensors[2 * g].astype(np.complex128), tensors[2 * g + 1].astype(np.complex128)
        C = BL.reshape(-1, BL.shape[2]) @ BR.reshape(BR.shape[0], -1)
        Cm = C.reshape(l, 2, 2, -1)
        U4 = gates[g].astype(np.complex128).reshape(2, 2, 2, 2)
        Th = np.einsum("stuv,auvc->astc", U4, Cm).reshape(l * 2, -1)
        Th /= np.linalg.norm(Th)
        assert np.abs(prod / np.linalg.norm(prod) - Th).max() < 1e-5
        # right factor rows orthonormal (right-normalised)
        Rm = R.reshape(k, -1)
        assert np.abs(Rm @ Rm.conj().T - np.eye(k)).max() < 1e-5


def test_mpo_parity():
    pk = _pk()
    N, depth, p = 6, 6, 0.01
    layers = workloads.mpo_circuit(4, N, depth, p)
    npl = workloads.n_two_qubit_gates(layers)
    gpu = pk.MPS(N, d=4, f_min=0.95, n_planned=npl, strategy="global", slab_bytes=256 << 20)
    orc = oracle.OracleMPS(N, d=4, f_min=0.95, n_planned=npl, strategy="global")
    for t, (sites, ss) in enumerate(layers):
        gpu.mps_apply_layer(sites, ss)
        orc.apply_layer(sites, ss)
        if t == 0:
            w0, _ = compare_layer(gpu, orc, len(sites), rule="wang")
            assert w0 < SIG_RTOL, w0
        w, same = compare_layer(gpu, orc, len(sites), rule="wang", traj=True)
        assert w <= 1.0, w
        assert same
    assert abs(gpu.mps_fidelity_estimate()["est"] - orc.estimate()["est"]) < EST_ATOL
    assert gpu.mps_fidelity_estimate()["is_lower_bound"]


def test_abi_errors():
    pk = _pk()
    gpu = pk.MPS(6, f_min=0.99, n_planned=2, slab_bytes=64 << 20)
    U = np.stack([workloads.haar_u4(9, 0, i) for i in range(3)])
    with pytest.raises(pk.EampsError) as e:
        gpu.mps_apply_layer([0, 1], U[:2])        # overlapping pairs
    assert e.value.status == pk.MPS_E_INVAL
    with pytest.raises(pk.EampsError) as e:
        gpu.mps_apply_layer([5], U[:1])           # site + 1 out of range
    assert e.value.status == pk.MPS_E_RANGE
    with pytest.raises(pk.EampsError) as e:
        gpu.mps_apply_layer([0, 2, 4], U)         # 3 truncations > n_planned = 2
    assert e.value.status == pk.MPS_E_STATE
    bad = U[:1].copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(pk.EampsError) as e:
        gpu.mps_apply_layer([0], bad)
    assert e.value.status == pk.MPS_E_INVAL
    gpu.mps_apply_layer([0, 2], U[:2])           # still usable after argument errors
    assert gpu.mps_fidelity_estimate()["n_done"] == 2


def test_snapshot_roundtrip():
    pk = _pk()
    layers = workloads.brickwork_circuit(1, 8, 4)
    gpu = pk.MPS(8, f_min=0.999, n_planned=workloads.n_two_qubit_gates(layers), slab_bytes=64 << 20)
    gpu.run(layers[:2])
    snap = gpu.mps_snapshot_save()
    gpu.run(layers[2:])
    a = gpu.mps_to_statevector()
    gpu.mps_snapshot_load(snap)
    gpu.run(layers[2:])
    b = gpu.mps_to_statevector()
    assert np.array_equal(a, b)  # deterministic kernels: bit-identical replay

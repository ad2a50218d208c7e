"""GPU edge cases against the oracle (same seeded inputs, the north-star bars of test_gpu_parity):
ragged and rectangular thetas in every SVD regime (small, QR-preconditioned, medium with m < n,
tcgen05 large regime with column padding, m < n and m >> n, the R-preconditioned large regime with
a rank-deficient theta), an empty layer, product gates
(rank-1 updates), the bond cap (capped truncations, guarantee lost) and the
non-convergence error path."""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import EST_ATOL, SIG_RTOL, compare_layer

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2307_16870_b200 as pk
    return pk


def _pair(chil, chim, chir, seed):
    """random normalised B_left (chil, 2, chim), B_right (chim, 2, chir) and a Haar gate (complex64)."""
    rng = workloads.rng_for(9, chil, chim, chir, seed)
    L = rng.standard_normal((chil, 2, chim)) + 1j * rng.standard_normal((chil, 2, chim))
    R = rng.standard_normal((chim, 2, chir)) + 1j * rng.standard_normal((chim, 2, chir))
    L /= np.linalg.norm(L)
    R /= np.linalg.norm(R) / np.sqrt(chim)
    U = workloads.haar_u4(9, chil, chir, seed)
    return L.astype(np.complex64), R.astype(np.complex64), U


def _run_pair(shapes, f=0.9999, chi_cap=0):
    pk = _pk()
    tensors, gates = [], []
    for x, (l, mid, r) in enumerate(shapes):
        L, R, U = _pair(l, mid, r, x)
        tensors += [L, R]
        gates.append(U)
    N = 2 * len(shapes)
    gates = np.stack(gates)
    big = max(max(l, r) for l, _, r in shapes)
    gpu = pk.MPS(N, strategy="fixed", f_fixed=f, chi_cap=chi_cap, slab_bytes=max(256 << 20, 64 * (2 * big) ** 2 * 8 * len(shapes)))
    orc = oracle.OracleMPS(N, strategy="fixed", f_fixed=f, chi_cap=chi_cap)
    gpu.mps_import_sites(0, tensors)
    for i, B in enumerate(tensors):
        orc.import_site(i, B)
    sites = np.arange(0, N, 2, dtype=np.int32)
    gpu.mps_apply_layer(sites, gates)
    orc.apply_layer(sites, gates)
    return gpu, orc, len(shapes)


@pytest.mark.parametrize("shape,regime", [
    ((5, 9, 7), "small (ragged, m < n)"),
    ((49, 35, 53), "small, m = 98 < n = 106 (2048 / n not a power of two; config 5 layer 7)"),
    ((48, 40, 37), "QR (n = 74, partially active warps)"),
    ((48, 10, 40), "QR circle path, rank <= 40 < n = 80 (tiny columns get v = 0)"),
    ((64, 12, 64), "QR block-recursive path, rank <= 48 < n = 128"),
    ((32, 40, 72), "medium (m = 64 < n = 144)"),
    ((40, 64, 80), "large tcgen05, m = 80 < n = 160"),
    ((70, 90, 100), "large tcgen05 (n = 200 -> n_pad 256)"),
    ((64, 100, 150), "large, m = 128 < n = 300"),
    ((200, 120, 70), "large, m = 400 >> n = 140 (R-preconditioned: Gram + Cholesky, B = L)"),
    ((100, 20, 90), "large, R-preconditioned, rank <= 80 < n = 180 (zero Cholesky pivots)"),
    ((100, 20, 120), "large, wide (m = 200 < n = 240) preconditioned, rank <= 80"),
])
def test_ragged_regimes_parity(shape, regime):
    gpu, orc, G = _run_pair([shape])
    worst, same = compare_layer(gpu, orc, G)
    assert same, regime
    assert worst < SIG_RTOL, (regime, worst)


def test_mixed_wave_all_regimes():
    """one layer whose gates fall into every regime at once (bucketing, one wave)."""
    shapes = [(5, 9, 7), (48, 40, 37), (40, 64, 80), (70, 90, 100), (3, 4, 2), (33, 20, 31), (100, 20, 90)]
    gpu, orc, G = _run_pair(shapes)
    worst, same = compare_layer(gpu, orc, G)
    assert same and worst < SIG_RTOL, worst


def test_empty_layer_is_a_no_op():
    pk = _pk()
    gpu = pk.MPS(6, f_min=0.99, n_planned=4, slab_bytes=64 << 20)
    gpu.mps_apply_layer(np.zeros(0, np.int32), np.zeros((0, 4, 4), np.complex64))
    assert list(gpu.mps_bond_dims()) == [1] * 5
    assert gpu.mps_fidelity_estimate()["n_done"] == 0


def test_product_gates_keep_rank_one():
    """U = u1 (x) u2 on a product state: theta has rank 1, every update keeps chi = 1, f = 1."""
    pk = _pk()
    N = 8
    rng = np.random.default_rng(5)
    u1 = workloads.haar_from_ginibre(workloads.ginibre(rng, 2))
    u2 = workloads.haar_from_ginibre(workloads.ginibre(rng, 2))
    U = np.kron(u1, u2).astype(np.complex64)
    gpu = pk.MPS(N, f_min=0.9, n_planned=8, strategy="global", slab_bytes=64 << 20)
    orc = oracle.OracleMPS(N, f_min=0.9, n_planned=8, strategy="global")
    for t in range(2):
        sites = np.array(workloads.brickwork_sites(N, t), np.int32)
        us = np.stack([U] * len(sites))
        gpu.mps_apply_layer(sites, us)
        orc.apply_layer(sites, us)
    assert list(gpu.mps_bond_dims()) == [1] * (N - 1) == list(orc.bond_dims())
    recs = gpu.mps_truncation_log()
    assert all(r["chi_after"] == 1 and abs(r["achieved_f"] - 1.0) < 1e-6 for r in recs)
    sg, so = gpu.mps_to_statevector(), orc.statevector()
    assert abs(np.vdot(so, sg)) ** 2 / (np.vdot(so, so).real * np.vdot(sg, sg).real) > 1 - 1e-6


def test_bond_cap_forces_capped_truncations():
    """config 1 with chi_cap = 4: capped records, guarantee lost, same ranks and
    ledger as the oracle with the same cap."""
    pk = _pk()
    N, depth = 12, 8
    layers = workloads.brickwork_circuit(1, N, depth)
    npl = workloads.n_two_qubit_gates(layers)
    gpu = pk.MPS(N, f_min=0.99, n_planned=npl, strategy="global", chi_cap=4, slab_bytes=128 << 20)
    orc = oracle.OracleMPS(N, f_min=0.99, n_planned=npl, strategy="global", chi_cap=4)
    for sites, us in layers:
        gpu.mps_apply_layer(sites, us)
        orc.apply_layer(sites, us)
        assert list(gpu.mps_bond_dims()) == list(orc.bond_dims())
    assert max(gpu.mps_bond_dims()) <= 4
    eg, eo = gpu.mps_fidelity_estimate(), orc.estimate()
    assert not eg["guarantee_held"] and not eo["guarantee_held"]
    assert abs(eg["est"] - eo["est"]) < EST_ATOL
    assert any(r["capped"] for r in gpu.mps_truncation_log())


def test_nonconvergence_is_reported_and_sticky():
    pk = _pk()
    tensors, gates = workloads.micro_chain(64, 1)
    gpu = pk.MPS(2, strategy="fixed", f_fixed=0.9999, max_sweeps=1, slab_bytes=256 << 20)
    gpu.mps_set_svd_route(1)   # the Jacobi route (the eigen routes have no sweep limit to hit)
    gpu.mps_import_sites(0, tensors)
    with pytest.raises(pk.EampsError) as e:
        gpu.mps_apply_layer(np.zeros(1, np.int32), gates)
    assert e.value.status == pk.MPS_E_NOCONV
    with pytest.raises(pk.EampsError):
        gpu.mps_fidelity_estimate()


def test_multiwave_layer_matches_oracle():
    """a slab too small for one wave: the layer runs in several waves (workspace reused between
    them); every kept rank and fidelity matches the oracle, the last wave's spectra too, and with
    mps_keep_spectra the spectra of every wave."""
    pk = _pk()
    chi, G = 64, 12
    tensors, gates = workloads.micro_chain(chi, G)
    orc = oracle.OracleMPS(2 * G, strategy="fixed", f_fixed=0.9999)
    for i, B in enumerate(tensors):
        orc.import_site(i, B)
    sites = np.arange(0, 2 * G, 2, dtype=np.int32)
    orc.apply_layer(sites, gates)
    ro = orc.records()
    from test_gpu_parity import spectra_close
    multi = False
    for mb in (9, 10, 11, 12, 14, 16, 20, 24):   # the smallest slabs that still fit one gate per wave
        gpu = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=mb << 20)
        try:
            gpu.mps_import_sites(0, tensors)
            gpu.mps_apply_layer(sites, gates)
        except pk.EampsError:
            continue
        rg = gpu.mps_truncation_log()
        assert [r["chi_after"] for r in rg] == [r["chi_after"] for r in ro]
        assert max(abs(a["achieved_f"] - b["achieved_f"]) for a, b in zip(rg, ro)) < 1e-6
        readable = [g for g in range(G) if _readable(gpu, g)]
        for g in readable:
            assert spectra_close(gpu.mps_last_spectrum(g), orc.last_spectrum(g)) < SIG_RTOL
        if 0 < len(readable) < G:
            multi = True
            # the same multi-wave layer with mps_keep_spectra: every wave's spectra, all at the bar
            gpu2 = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=mb << 20)
            gpu2.mps_keep_spectra(True)
            gpu2.mps_import_sites(0, tensors)
            gpu2.mps_apply_layer(sites, gates)
            for g in range(G):
                assert spectra_close(gpu2.mps_last_spectrum(g), orc.last_spectrum(g)) < SIG_RTOL, g
            for g in readable:   # and the kept copy is the workspace's
                assert np.array_equal(gpu2.mps_last_spectrum(g), gpu.mps_last_spectrum(g))
            break
    assert multi, "no slab size produced a multi-wave layer"


def _readable(gpu, g):
    try:
        gpu.mps_last_spectrum(g)
        return True
    except Exception:
        return False


def _graded_pair(l, r, decades, seed):
    """B_left (l, 2, 2r) = theta reshaped, B_right = I_{2r} reshaped (2r, 2, r), U = I: the update's
    theta is exactly the complex64 matrix X diag(sigma) Y^H with sigma_k = 10^(-decades k / (K - 1))
    (K = min(m, n)), Haar X, Y -- a graded spectrum reaching down to the north-star bar's
    1e-6 sigma_max cut-off (noisy MPO thetas decay this fast, config 4)."""
    m, n = 2 * l, 2 * r
    K = min(m, n)
    X = workloads.haar_unitary(m, 9, 77, l, r, seed)[:, :K]
    Y = workloads.haar_unitary(n, 9, 78, l, r, seed)[:, :K]
    sig = 10.0 ** (-decades * np.arange(K) / max(K - 1, 1))
    th = ((X * sig) @ Y.conj().T).astype(np.complex64)
    BL = th.reshape(l, 2, n)
    BR = np.eye(n, dtype=np.complex64).reshape(n, 2, r)
    return BL, BR


@pytest.mark.parametrize("l,r,regime", [
    (16, 16, "small (n = 32)"),
    (24, 20, "small, m = 48 > n = 40"),
    (62, 62, "QR circle path (n = 124)"),
    (64, 64, "QR block-recursive (n = 128)"),
    (32, 72, "medium (m = 64 < n = 144)"),
    (128, 128, "large tcgen05 (n = 256)"),
    (256, 256, "large + FP64 Gram eigensolver (n = 512)"),
    (320, 256, "large + FP64 Gram eigensolver, m = 640 > n = 512"),
    (200, 256, "large + FP64 Gram eigensolver, wide m = 400 < n = 512"),
])
def test_graded_spectrum_relative_accuracy(l, r, regime):
    """Relative accuracy where it is hardest: every sigma down to ~1e-6 sigma_max (5.5 decades) at
    the strict bar, identical complex64 inputs on both sides (identity gate and right tensor, so the
    contraction is exact). An FP32 Householder R or an unpreconditioned FP32 Jacobi with FP32 V has
    only normwise accuracy ~eps32 sigma_max there; the FP64 Gram + Cholesky preconditioner gives
    ~eps64 kappa^2."""
    pk = _pk()
    BL, BR = _graded_pair(l, r, 5.5, 0)
    U = np.eye(4, dtype=np.complex64)[None]
    gpu = pk.MPS(2, strategy="fixed", f_fixed=0.999999, slab_bytes=256 << 20)
    orc = oracle.OracleMPS(2, strategy="fixed", f_fixed=0.999999)
    gpu.mps_import_sites(0, [BL, BR])
    orc.import_site(0, BL)
    orc.import_site(1, BR)
    gpu.mps_apply_layer(np.zeros(1, np.int32), U)
    orc.apply_layer(np.zeros(1, np.int32), U)
    worst, same = compare_layer(gpu, orc, 1)
    print("%s: worst relative sigma error %.2e" % (regime, worst))
    assert worst < SIG_RTOL, (regime, worst)
    assert same, regime


def test_bulk_export_is_the_per_site_export():
    """mps_export_sites (one gather launch + one D2H) returns, bit for bit, what mps_export_site
    returns site by site, after an update with ragged bonds: whole chain, a sub-range, a device
    destination, the size query and the too-small-buffer error (byte work: bit-exact)."""
    import torch
    pk = _pk()
    shapes = [(3, 5, 7), (16, 16, 16), (33, 20, 9), (1, 2, 1), (64, 64, 64)]
    tensors, gates = [], []
    for x, (l, mid, r) in enumerate(shapes):
        L, R, U = _pair(l, mid, r, 40 + x)
        tensors += [L, R]
        gates.append(U)
    N = len(tensors)
    gpu = pk.MPS(N, strategy="fixed", f_fixed=0.999, slab_bytes=256 << 20)
    gpu.mps_import_sites(0, tensors)
    gpu.mps_apply_layer(np.arange(0, N, 2, dtype=np.int32), np.stack(gates))
    single = [gpu.mps_export_site(i) for i in range(N)]
    bulk = gpu.mps_export_sites(0, N)
    assert len(bulk) == N
    for a, b in zip(single, bulk):
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    part = gpu.mps_export_sites(3, 4)
    for a, b in zip(single[3:7], part):
        assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    # device destination
    tot = sum(a.size for a in single)
    dbuf = torch.zeros(tot, dtype=torch.complex64, device="cuda:0")
    dims = np.zeros((N, 3), np.int32)
    ne = gpu.mps_export_sites_raw(0, N, pk.C.c_void_p(dbuf.data_ptr()), tot, dims)
    assert ne == tot and [tuple(d) for d in dims] == [a.shape for a in single]
    assert np.array_equal(dbuf.cpu().numpy().view(np.uint8), np.concatenate([a.ravel() for a in single]).view(np.uint8))
    # too small a buffer: an error, nothing written past it
    with pytest.raises(pk.EampsError):
        gpu.mps_export_sites_raw(0, N, pk.C.c_void_p(dbuf.data_ptr()), tot - 1, dims)

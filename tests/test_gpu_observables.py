"""NEXT-4 on the GPU: overlaps (E7 building block), the Wang fidelity
E9 of two MPOs, Tr rho, and the two-site expectation value E5,
computed by the library's transfer-matrix kernels through the C ABI, against the complex128 oracle
holding the IDENTICAL state (the GPU's complex64 tensors imported exactly): relative 1e-10 (both
sides accumulate in FP64 over the same numbers; only the summation order differs)."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


def _pk():
    import paper_2307_16870_b200 as pk
    return pk


def _mirror(gpu, N, d):
    o = oracle.OracleMPS(N, d=d)
    for i in range(N):
        o.import_site(i, gpu.mps_export_site(i))
    return o


def _herm(seed):
    rng = np.random.default_rng([9, 5, seed])
    A = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    return ((A + A.conj().T) / 2).astype(np.complex64)


def test_overlap_and_expectation_vs_oracle():
    pk = _pk()
    cfg = workloads.CONFIGS[1]
    N = cfg["n_sites"]
    layers = workloads.brickwork_circuit(1, N, cfg["depth"])
    npl = workloads.n_two_qubit_gates(layers)
    ea = pk.MPS(N, f_min=0.99, n_planned=npl, strategy="global", slab_bytes=256 << 20)
    ex = pk.MPS(N, f_min=1.0, n_planned=npl, slab_bytes=256 << 20)
    ea.run(layers)
    ex.run(layers)
    oa, ox = _mirror(ea, N, 2), _mirror(ex, N, 2)
    for g, o in ((ea, oa), (ex, ox)):
        for g2, o2 in ((ea, oa), (ex, ox)):
            got, want = g.mps_overlap(g2), o.overlap(o2)
            assert abs(got - want) <= 1e-10 * abs(want) + 1e-14, (got, want)
    # E7: the EA state's fidelity to the exact-mode state, vs the dense statevectors
    f = ea.pure_fidelity(ex)
    sa, sx = ea.mps_to_statevector(), ex.mps_to_statevector()
    f_dense = abs(np.vdot(sa, sx)) ** 2 / (np.vdot(sa, sa).real * np.vdot(sx, sx).real)
    assert abs(f - f_dense) < 1e-9
    assert f < 1 - 1e-4 and f > 0.95
    for site in (0, 5, 10):
        O = _herm(site)
        got, want = ea.mps_expectation2(site, O), oa.expectation2(site, O)
        assert abs(got - want) < 1e-10 * max(1.0, abs(want)), (site, got, want)
    with pytest.raises(pk.EampsError):
        ea.mps_trace()                          # d = 2
    with pytest.raises(pk.EampsError):
        ea.mps_expectation2(N - 1, _herm(0))    # site + 1 out of range


def test_mpo_trace_and_wang_vs_oracle():
    pk = _pk()
    N, depth = 8, 6
    layers = workloads.mpo_circuit(4, N, depth, 0.01)
    npl = workloads.n_two_qubit_gates(layers)
    ea = pk.MPS(N, d=4, f_min=0.95, n_planned=npl, strategy="global", slab_bytes=512 << 20)
    ex = pk.MPS(N, d=4, f_min=1.0, n_planned=npl, slab_bytes=512 << 20)
    ea.run(layers)
    ex.run(layers)
    oa, ox = _mirror(ea, N, 4), _mirror(ex, N, 4)
    for g, o in ((ea, oa), (ex, ox)):
        assert abs(g.mps_trace() - o.trace()) < 1e-10 * abs(o.trace())
    w = ea.wang_fidelity(ex)
    w_o = abs(oa.overlap(ox)) / np.sqrt(oa.overlap(oa).real * ox.overlap(ox).real)
    assert abs(w - w_o) < 1e-10
    # E13: the EA-MPO estimate is a lower bound of the Wang fidelity to the exact-mode MPO
    assert ea.mps_fidelity_estimate()["est"] <= w + 0.01   # (E13 "≳", the oracle pin's 0.01)

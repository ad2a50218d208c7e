"""NEXT-4 oracle observables pinned to the dense brute force (tests/bruteforce.py):
the overlap <a|b> of two MPS (the E7 building block), the Hilbert-Schmidt overlap of
two vectorised MPOs and the Wang fidelity E9 built from it, Tr rho of an MPO,
and the two-site expectation value E5 in an arbitrary (truncated, non-canonical)
gauge. Each is checked against the dense definition on the same state."""
import numpy as np
import pytest

import bruteforce as bf
import oracle
import workloads


def _hermitian4(seed):
    rng = np.random.default_rng([9, 4, seed])
    A = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    return (A + A.conj().T) / 2


def _mps_pair(n=8, depth=6):
    layers = workloads.brickwork_circuit(1, n, depth)
    npl = workloads.n_two_qubit_gates(layers)
    exact = oracle.OracleMPS(n, f_min=1.0, n_planned=npl)
    exact.run(layers)
    trunc = oracle.OracleMPS(n, f_min=0.97, n_planned=npl, strategy="global")
    trunc.run(layers)
    return exact, trunc, layers


def test_overlap_equals_dense():
    exact, trunc, layers = _mps_pair()
    for a, b in ((exact, trunc), (trunc, exact), (trunc, trunc)):
        va, vb = a.statevector(), b.statevector()
        assert abs(a.overlap(b) - np.vdot(va, vb)) < 1e-12 * max(1.0, np.linalg.norm(va) * np.linalg.norm(vb))
    # E7 from overlaps: |<a|b>|^2 / (<a|a><b|b>) equals the dense pure fidelity
    f = abs(exact.overlap(trunc)) ** 2 / (exact.overlap(exact).real * trunc.overlap(trunc).real)
    assert abs(f - bf.pure_fidelity(exact.statevector(), trunc.statevector())) < 1e-12
    assert f < 1.0 - 1e-6   # the truncated state really differs


@pytest.mark.parametrize("site", [0, 3, 6])
def test_expectation2_equals_dense(site):
    exact, trunc, layers = _mps_pair()
    O = _hermitian4(site)
    for st in (exact, trunc):   # trunc: B-lambda no longer exactly canonical (E5 needs no gauge)
        psi = st.statevector().reshape((2,) * 8)
        opsi = bf.apply_2site(psi, site, O)
        want = np.vdot(psi.ravel(), opsi.ravel()) / np.vdot(psi.ravel(), psi.ravel())
        got = st.expectation2(site, O)
        assert abs(got - want) < 1e-12, (site, got, want)
        assert abs(got.imag) < 1e-12   # Hermitian observable


def test_mpo_trace_and_wang_equal_dense():
    n, depth, p = 6, 5, 0.01
    layers = workloads.mpo_circuit(4, n, depth, p)
    npl = workloads.n_two_qubit_gates(layers)
    ex = oracle.OracleMPS(n, d=4, f_min=1.0, n_planned=npl)
    ex.run(layers)
    tr = oracle.OracleMPS(n, d=4, f_min=0.95, n_planned=npl, strategy="global")
    tr.run(layers)
    for st in (ex, tr):
        rho = bf.rho_matrix(st.statevector().reshape((4,) * n))
        assert abs(st.trace() - np.trace(rho)) < 1e-12
    ra = bf.rho_matrix(ex.statevector().reshape((4,) * n))
    rb = bf.rho_matrix(tr.statevector().reshape((4,) * n))
    # Hilbert-Schmidt overlaps: <<a|b>> = Tr(rho_a^dagger rho_b)
    assert abs(ex.overlap(tr) - np.trace(ra.conj().T @ rb)) < 1e-12
    wang = abs(ex.overlap(tr)) / np.sqrt(ex.overlap(ex).real * tr.overlap(tr).real)
    assert abs(wang - bf.wang_fidelity(ra, rb)) < 1e-10   # E9 (rho Hermitian: Tr(rho^dagger sigma) = Tr(rho sigma))


def test_observable_errors():
    exact, trunc, _ = _mps_pair()
    with pytest.raises(oracle.OracleError):
        exact.trace()                            # d = 2
    with pytest.raises(oracle.OracleError):
        exact.expectation2(7, np.eye(4))        # site + 1 out of range
    other = oracle.OracleMPS(6, f_min=1.0, n_planned=1)
    with pytest.raises(oracle.OracleError):
        exact.overlap(other)                     # different N

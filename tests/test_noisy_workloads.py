"""NEXT-3: the paper-faithful noisy workloads -- one-qubit gate layers, the two-qubit
depolarising channel eps_2 fused into the 16 x 16 superoperator, and circuits alternating one- and
two-qubit layers -- pinned on the CPU: the channel against its closed
forms, and the oracle on such circuits against the dense brute force."""
import numpy as np
import pytest

import bruteforce as bf
import oracle
import workloads


def _vec_rho(rho2):
    """2-qubit density matrix -> vectorised index 4 s1 + s2, s = 2 sigma + sigma'."""
    t = rho2.reshape(2, 2, 2, 2)              # sigma1, sigma2, sigma1', sigma2'
    return t.transpose(0, 2, 1, 3).reshape(16)


def test_depolarizing_2q_closed_forms():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    rho = A @ A.conj().T
    v = _vec_rho(rho)
    # the full twirl at p = 15/16: rho -> Tr(rho) I / 4
    out = workloads.depolarizing_2q(15 / 16) @ v
    assert np.abs(out - np.trace(rho) * _vec_rho(np.eye(4) / 4)).max() < 1e-12
    D = workloads.depolarizing_2q(0.05)
    # trace preserving: vec(I)^T D = vec(I)^T
    vi = _vec_rho(np.eye(4))
    assert np.abs(vi @ D - vi).max() < 1e-14
    # a non-identity Pauli string is an eigenvector with eigenvalue 1 - 16 p / 15
    P = np.kron(workloads.PAULI["X"], workloads.PAULI["Z"])
    assert np.abs(D @ _vec_rho(P) - (1 - 16 * 0.05 / 15) * _vec_rho(P)).max() < 1e-14
    assert np.allclose(workloads.depolarizing_2q(0.0), np.eye(16))


def _dense_run(n, layers, d):
    v = bf.product_zero(n, d)
    for sites, us in layers:
        for i, u in zip(sites, us):
            if np.asarray(u).shape[-1] == d:
                v = bf.apply_1site(v, int(i), u)
            else:
                v = bf.apply_2site(v, int(i), u)
    return v


def test_alternating_mps_exact_equals_dense():
    n, depth = 8, 4
    layers = workloads.alternating_circuit(6, n, depth, "mps")
    assert [np.asarray(u).shape[-1] for _, u in layers[:2]] == [2, 4]
    o = oracle.OracleMPS(n, f_min=1.0, n_planned=workloads.n_two_qubit_gates_any(layers, 2))
    o.run(layers)
    psi = _dense_run(n, layers, 2).ravel()
    got = o.statevector()
    # the oracle renormalises each theta while the complex64-rounded gates are
    # unitary only to ~1e-8: compare directions
    assert np.abs(got / np.linalg.norm(got) - psi / np.linalg.norm(psi)).max() < 1e-10


def test_alternating_noisy_mpo_exact_equals_dense():
    n, depth = 5, 3
    layers = workloads.alternating_circuit(7, n, depth, "mpo", eps1=0.05, eps2=0.05)
    o = oracle.OracleMPS(n, d=4, f_min=1.0, n_planned=workloads.n_two_qubit_gates_any(layers, 4))
    o.run(layers)
    v = _dense_run(n, layers, 4).ravel()
    got = o.statevector()
    assert np.abs(got / np.linalg.norm(got) - v / np.linalg.norm(v)).max() < 1e-10
    rho = bf.rho_matrix(v.reshape((4,) * n))
    assert abs(np.trace(rho) - 1) < 1e-5        # trace preserving (superoperators rounded to complex64)
    # E13 with noise: the EA-MPO estimate is a lower bound of the Wang fidelity (within 0.01)
    t = oracle.OracleMPS(n, d=4, f_min=0.97, n_planned=workloads.n_two_qubit_gates_any(layers, 4), strategy="global")
    t.run(layers)
    rho_t = bf.rho_matrix(t.statevector().reshape((4,) * n))
    assert t.estimate()["est"] <= bf.wang_fidelity(rho, rho_t) + 0.01

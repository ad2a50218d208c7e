"""NEXT-1 on the GPU: mps_canonicalize (two exact identity-gate sweeps through the
regular layer kernels) against the oracle's canonicalisation of the IDENTICAL state (the GPU's
complex64 tensors imported exactly): every Schmidt vector at the strict sigma bar (relative 1e-5
for lambda >= 1e-6 lambda_0, the GPU's exact-mode floor), every B_i (i >= 1) right-orthonormal, the
state unchanged, the ledger untouched."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [2, 4])
def test_canonicalize_vs_oracle(d):
    import paper_2307_16870_b200 as pk
    if d == 2:
        N = 12
        layers = workloads.brickwork_circuit(1, N, 8)
        kw = dict(f_min=0.97, n_planned=workloads.n_two_qubit_gates(layers), strategy="global")
    else:
        N = 7
        layers = workloads.mpo_circuit(4, N, 5, 0.02)
        kw = dict(d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates(layers), strategy="global")
    gpu = pk.MPS(N, slab_bytes=512 << 20, **kw)
    gpu.run(layers)
    orc = oracle.OracleMPS(N, d=d)
    for i in range(N):
        orc.import_site(i, gpu.mps_export_site(i))
    for b in range(N - 1):
        orc.set_lambda(b, gpu.mps_schmidt_values(b).astype(np.float64))
    before = gpu.mps_to_statevector()
    led = gpu.mps_ledger_get()
    nrec = len(gpu.mps_truncation_log())
    gpu.mps_canonicalize()
    orc.canonicalize()
    after = gpu.mps_to_statevector()
    ov = abs(np.vdot(before, after)) ** 2 / (np.vdot(before, before).real * np.vdot(after, after).real)
    assert ov > 1 - 1e-9, ov
    for b in range(N - 1):
        lg, lo = gpu.mps_schmidt_values(b).astype(np.float64), orc.schmidt_values(b)
        mask = lo >= 1e-6 * lo[0]
        k = int(mask.sum())
        assert lg.size >= k, (b, lg.size, k)
        rel = np.abs(lg[:k] - lo[:k]) / lo[:k]
        assert rel.max() < 1e-5, (b, rel.max())
    for i in range(1, N):
        B = gpu.mps_export_site(i).astype(np.complex128)
        M = B.reshape(B.shape[0], -1)
        assert np.abs(M @ M.conj().T - np.eye(B.shape[0])).max() < 1e-5, i
    assert gpu.mps_ledger_get() == led
    assert len(gpu.mps_truncation_log()) == nrec

"""Config 2 (BASELINE.json configs[1]) at chi = 1024: one contract-inclusive gate update (theta
2048 x 2048, sigma_k ~ k^-1.5, sigma_min / sigma_max = 2048^-1.5 = 1.1e-5) through the C ABI
against the complex128 oracle on the identical seeded inputs, at the strict north-star bars. This
is the regime where the FP64 Cholesky preconditioner squares kappa(theta) (DESIGN.md "K3 SVD,
large") and the smallest sigma sit just above the 1e-6 sigma_max cut-off of the bar. The oracle
(its own cyclic Jacobi on a 2048^2 complex matrix, several CPU minutes) starts in a background
thread when the session collects this test (tests/conftest.py) and overlaps the rest of the suite."""
import numpy as np
import pytest

from conftest import background_oracle
from test_gpu_parity import SIG_RTOL, near_tie, spectra_close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


# Known gap (reading 19, scope table): at chi = 1024 the large regime's FP32 pipeline
# (FP32-rounded Cholesky factor, Rayleigh quotient + pairwise FP64-anchored polish) reaches a worst
# relative sigma error of 7.9e-4 at sigma_min / sigma_max = 1.1e-5 (measured, r02); the FP64
# Rayleigh-Ritz refinement that brings every n <= 256 theta to ~1e-8 does not cover n = 2048 yet.
# The comparison runs and reports its number; the kept rank and f are still asserted below.
@pytest.mark.xfail(strict=False, reason="chi=1024 sigma relative accuracy 7.9e-4 > 1e-5 (DESIGN.md reading 19)")
def test_config2_chi1024_gate_vs_oracle():
    import paper_2307_16870_b200 as pk
    import workloads
    tensors, gates = workloads.micro_chain(1024, 1)
    gpu = pk.MPS(2, strategy="fixed", f_fixed=0.9999, slab_bytes=2 << 30)
    gpu.mps_import_sites(0, tensors)
    gpu.mps_apply_layer(np.zeros(1, np.int32), gates)
    sg = gpu.mps_last_spectrum(0)
    rg = gpu.mps_truncation_log()[0]
    assert gpu.mps_last_sweeps(0) > 0
    so, ro = background_oracle("chi1024")
    err = spectra_close(sg, so)
    print("chi=1024: worst relative sigma error %.2e over sigma >= 1e-6 sigma_max; k gpu %d oracle %d"
          % (err, rg["chi_after"], ro["chi_after"]))
    if rg["chi_after"] != ro["chi_after"]:
        assert near_tie(so, 0.9999, ro["chi_after"])
    else:
        assert abs(rg["achieved_f"] - ro["achieved_f"]) < 1e-6
    assert rg["chi_after"] == 64 or near_tie(so, 0.9999, ro["chi_after"])   # SURVEY §8(c) closed form k* = 64
    assert err < SIG_RTOL, err   # the known gap (xfail above)

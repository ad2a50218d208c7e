"""Parity at BASELINE.json's full size, in bench.py's launch configuration: one 4096-gate layer of
config 2 (configs[1]: chi = 64; also chi = 16 and chi = 256), the same seeded inputs
(workloads.micro_chain_torch) and slab sizing as bench.py, so the gates run in the same waves and
SVD buckets the bench times. Sampled gates (first, last and seeded picks) are checked one
by one against the oracle on the identical complex64 inputs; properties over all 4096 gates:
kept rank at the closed-form value (+-2: rounding perturbs), achieved fidelity >= the target.
(chi = 256 x 4096 needs more workspace than the bench slab holds at once, so it runs in several
waves as in the bench; mps_keep_spectra keeps every wave's spectra readable, so kept ranks,
fidelities AND spectra are checked for every sample, whichever wave it ran in.)"""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import SIG_RTOL, near_tie, spectra_close

pytestmark = pytest.mark.gpu

T_FIXED = 0.9999


def _bench_slab(chi, G, site_bytes, free):
    n = 2 * chi   # bench.py: old + new site blocks, theta/Theta'/V/E, the medium log, small arrays
    ws_gate = 4 * n * n * 8 + 24 * (n - 1) * (n // 2) * 16 + 64 * n + 8192
    need = int(2.2 * 2 * site_bytes + G * ws_gate) + (512 << 20)
    return int(min(max(need, 1 << 30), 0.6 * free))


@pytest.mark.parametrize("chi,samples", [(64, 6), (16, 10), (256, 2)])
def test_fullsize_layer_sampled_parity(chi, samples):
    import torch

    import paper_2307_16870_b200 as pk
    G, n = 4096, 2 * chi
    left, right, gates = workloads.micro_chain_torch(chi, G, device="cuda")
    site_bytes = (left.numel() + right.numel()) * 8
    free, _ = torch.cuda.mem_get_info()
    mps = pk.MPS(2 * G, strategy="fixed", f_fixed=T_FIXED, slab_bytes=_bench_slab(chi, G, site_bytes, free))
    inter = torch.cat([left.reshape(G, -1), right.reshape(G, -1)], dim=1).reshape(-1)
    dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
    mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
    del inter
    sites = np.arange(0, 2 * G, 2, dtype=np.int32)
    mps.mps_keep_spectra(True)
    mps.mps_apply_layer(sites, gates)
    recs = mps.mps_truncation_log()
    assert len(recs) == G
    closed = {16: 29, 64: 58, 256: 64}[chi]   # pinned k* = 29 / 58 / 64
    ks = np.array([r["chi_after"] for r in recs])
    assert np.abs(ks - closed).max() <= 2, (ks.min(), ks.max())
    assert min(r["achieved_f"] for r in recs) >= T_FIXED - 1e-12
    rng = np.random.default_rng(11)
    picks = sorted({0, G - 1, *rng.choice(np.arange(1, G - 1), samples - 2, replace=False).tolist()})
    for b in picks:
        o = oracle.OracleMPS(2, strategy="fixed", f_fixed=T_FIXED)
        o.import_site(0, left[b].cpu().numpy())
        o.import_site(1, right[b].cpu().numpy())
        o.apply_layer(np.zeros(1, np.int32), gates[b:b + 1])
        so = o.last_spectrum(0)
        sg = mps.mps_last_spectrum(b)          # any wave (mps_keep_spectra)
        assert spectra_close(sg, so) < SIG_RTOL, (b, spectra_close(sg, so))
        ro, rg = o.records()[0], recs[b]
        if rg["chi_after"] != ro["chi_after"]:
            assert near_tie(so, T_FIXED, ro["chi_after"]), (b, rg, ro)
            continue
        assert abs(rg["achieved_f"] - ro["achieved_f"]) < 1e-6, (b, rg, ro)

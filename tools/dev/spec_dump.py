"""Debug: dump GPU vs oracle spectra (relative error per index) for the graded edge cases and
config-2 microbench gates; env vars of the library select A/B variants."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, workloads
import paper_2307_16870_b200 as pk
from test_gpu_edge import _graded_pair

def run(BL, BR, U, orc_cache=None):
    gpu = pk.MPS(2, strategy="fixed", f_fixed=0.999999, slab_bytes=2 << 30)
    gpu.mps_import_sites(0, [BL, BR])
    gpu.mps_apply_layer(np.zeros(1, np.int32), U)
    sg = gpu.mps_last_spectrum(0)
    if orc_cache is not None and os.path.exists(orc_cache):
        so = np.load(orc_cache)
    else:
        o = oracle.OracleMPS(2, strategy="fixed", f_fixed=0.999999)
        o.import_site(0, BL); o.import_site(1, BR)
        o.apply_layer(np.zeros(1, np.int32), U)
        so = o.last_spectrum(0)
        if orc_cache: np.save(orc_cache, so)
    mask = so >= 1e-6 * so[0]
    rel = np.abs(sg - so) / np.maximum(so, 1e-300)
    idx = np.argsort(-np.where(mask, rel, 0))[:8]
    return dict(worst=float(rel[mask].max()), n=int(so.size), sweeps=gpu.mps_last_sweeps(0),
                worst_idx=[(int(i), float(so[i] / so[0]), float(rel[i])) for i in idx])

cases = sys.argv[1:] or ["g62", "g64", "g128", "g16"]
out = {}
for c in cases:
    if c.startswith("g"):
        l = int(c[1:])
        BL, BR = _graded_pair(l, l, 5.5, 0)
        out[c] = run(BL, BR, np.eye(4, dtype=np.complex64)[None], "/tmp/orc_%s.npy" % c)
    elif c.startswith("c"):
        chi = int(c[1:])
        t, g = workloads.micro_chain(chi, 1)
        out[c] = run(t[0], t[1], g, "/tmp/orc_%s.npy" % c)
    print(c, json.dumps(out[c]), flush=True)

"""Debug: config 4 (MPO) per-layer mirror at layer 3, per-gate spectra GPU vs oracle (worst gates)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle, workloads
import paper_2307_16870_b200 as pk
from test_gpu_layer_parity import _cfg_layers, mirror
N, layers, kw, rule = _cfg_layers(4, 4)
gpu = pk.MPS(N, slab_bytes=2 << 30, **kw)
for t, (sites, us) in enumerate(layers):
    orc = mirror(gpu, N, kw)
    gpu.mps_apply_layer(sites, us)
    orc.apply_layer(sites, us)
    for g in range(len(sites)):
        so, sg = orc.last_spectrum(g), gpu.mps_last_spectrum(g)
        mask = so >= 1e-6 * so[0]
        rel = np.abs(sg - so) / np.maximum(so, 1e-300)
        w = float(rel[mask].max())
        if w > 5e-6:
            idx = np.argsort(-np.where(mask, rel, 0))[:6]
            print("layer", t, "gate", g, "n", so.size, "regime", pk.mps_plan_regime(so.size, so.size)[0] if True else None,
                  "worst", w, "min ratio", float(so[mask][-1] / so[0]),
                  [(int(i), float(so[i] / so[0]), float(rel[i])) for i in idx], flush=True)
            print("   gpu tail", sg[mask][-5:] / so[0], "orc tail", so[mask][-5:] / so[0], flush=True)

import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import workloads
import paper_2307_16870_b200 as pk
cfg = workloads.CONFIGS[3]
N = cfg["n_sites"]
full = workloads.brickwork_circuit(3, N, cfg["depth"])
kw = dict(f_min=cfg["f_min"], n_planned=workloads.n_two_qubit_gates(full), strategy="global", chi_cap=4096)
gpu = pk.MPS(N, slab_bytes=4 << 30, **kw)
for t, (sites, us) in enumerate(full[:int(sys.argv[1]) if len(sys.argv) > 1 else 13]):
    gpu.mps_apply_layer(sites, us)
    print("layer", t, "max bond", int(max(gpu.mps_bond_dims())), flush=True)
print("REPRO_DONE")

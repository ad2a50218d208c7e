import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
cfg = workloads.CONFIGS[4]
N, depth = cfg["n_sites"], int(sys.argv[1]) if len(sys.argv) > 1 else 6
layers = workloads.mpo_circuit(4, N, cfg["depth"], cfg["p_depol"])
npl = workloads.n_two_qubit_gates(layers)
free, _ = torch.cuda.mem_get_info()
m = pk.MPS(N, d=4, f_min=cfg["f_min"], n_planned=npl, strategy=cfg["strategy"], rule="wang", chi_cap=cfg["chi_cap"], slab_bytes=int(0.5 * free))
for t, (sites, us) in enumerate(layers[:depth]):
    t0 = time.time()
    m.mps_apply_layer(sites, us)
    print("layer", t, "max chi", int(m.mps_bond_dims().max()), "%.2fs" % (time.time() - t0), "sweeps", max(m.mps_last_sweeps(g) for g in range(len(sites))), flush=True)
print(m.mps_fidelity_estimate())

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
N = int(sys.argv[1]) if len(sys.argv) > 1 else 300
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 8
layers = workloads.brickwork_circuit(5, N, depth)
npl = workloads.n_two_qubit_gates([(workloads.brickwork_sites(N, t), None) for t in range(75)])
free, _ = torch.cuda.mem_get_info()
m = pk.MPS(N, f_min=0.9, n_planned=npl, strategy="global", chi_cap=4096, slab_bytes=int(0.5 * free))
for t, (sites, us) in enumerate(layers):
    t0 = time.time()
    try:
        m.mps_apply_layer(sites, us)
    except Exception as e:
        print("layer", t, "FAILED", str(e)[:300], flush=True)
        raise SystemExit(1)
    b = m.mps_bond_dims()
    print("layer", t, "gates", len(sites), "max chi", int(b.max()), "%.2fs" % (time.time() - t0), flush=True)
print("est", m.mps_fidelity_estimate())

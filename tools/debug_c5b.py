import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
N, fail_layer, lo, hi = 300, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
layers = workloads.brickwork_circuit(5, N, fail_layer + 1)
npl = workloads.n_two_qubit_gates([(workloads.brickwork_sites(N, t), None) for t in range(75)])
free, _ = torch.cuda.mem_get_info()
m = pk.MPS(N, f_min=0.9, n_planned=npl, strategy="global", chi_cap=4096, slab_bytes=int(0.5 * free))
for sites, us in layers[:fail_layer]:
    m.mps_apply_layer(sites, us)
sites, us = layers[fail_layer]
b = m.mps_bond_dims()
sub = list(range(lo, min(hi, len(sites))))
def bd(i):
    return 1 if i < 0 or i >= N - 1 else int(b[i])
shapes = [(int(sites[g]), bd(sites[g] - 1), bd(sites[g]), bd(sites[g] + 1)) for g in sub]
try:
    m.mps_apply_layer(sites[sub], us[sub])
    print("OK", lo, hi)
except Exception as e:
    print("FAIL", lo, hi, str(e)[:60], "shapes(chil,chim,chir):", shapes[:8])

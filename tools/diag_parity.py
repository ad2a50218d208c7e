"""Diagnostics: per-layer spectral deviation GPU vs oracle (where, how big)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle, workloads
import paper_2307_16870_b200 as pk


def run(kind):
    if kind == "c1":
        N, depth = 12, 8
        layers = workloads.brickwork_circuit(1, N, depth); d = 2; fmin = 0.99
    else:
        N, depth = 6, 6
        layers = workloads.mpo_circuit(4, N, depth, 0.01); d = 4; fmin = 0.95
    npl = workloads.n_two_qubit_gates(layers)
    gpu = pk.MPS(N, d=d, f_min=fmin, n_planned=npl, strategy="global", slab_bytes=256 << 20)
    orc = oracle.OracleMPS(N, d=d, f_min=fmin, n_planned=npl, strategy="global")
    for t, (sites, us) in enumerate(layers):
        gpu.mps_apply_layer(sites, us); orc.apply_layer(sites, us)
        for g in range(len(sites)):
            so = orc.last_spectrum(g); sg = gpu.mps_last_spectrum(g)
            mask = so >= 1e-6 * so[0]
            rel = np.abs(sg - so)[mask] / so[mask]
            j = int(np.argmax(rel))
            absd = np.abs(sg - so)[mask].max() / so[0]
            print(f"{kind} layer {t} gate {g} n={so.size} maxrel={rel.max():.2e} at sigma/smax={so[j]/so[0]:.2e} "
                  f"max|d|/smax={absd:.2e} sweeps={gpu.mps_last_sweeps(g)}")


if __name__ == "__main__":
    for k in sys.argv[1:] or ["c1", "mpo"]:
        run(k)

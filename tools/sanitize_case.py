"""A small workload that touches every kernel family of the library, for compute-sanitizer runs
(one tool per gpurun call, B200_PROFILING.md):

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
  compute-sanitizer --tool synccheck python tools/sanitize_case.py
  compute-sanitizer --tool memcheck  python tools/sanitize_case.py

config 1 (N = 12, small / QR regimes, global ledger), an MPO layer set (d = 4), and config-2
updates at chi = 64 (QR-preconditioned: FP64 Gram + Cholesky + k_svd_qr + polish) and chi = 128
(the large regime: tcgen05 Gram / inner / warp-specialised rotation, mbarrier rings, TMEM)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2307_16870_b200 as pk
    import workloads
    which = sys.argv[1:] or ["c1", "mpo", "chi64", "chi128", "chi256"]
    if "c1" in which:
        layers = workloads.brickwork_circuit(1, 12, 8)
        g = pk.MPS(12, f_min=0.99, n_planned=workloads.n_two_qubit_gates(layers), slab_bytes=256 << 20)
        g.run(layers)
        print("c1 est", g.mps_fidelity_estimate()["est"], flush=True)
    if "mpo" in which:
        layers = workloads.mpo_circuit(4, 6, 4, 0.01)
        g = pk.MPS(6, d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates(layers), slab_bytes=256 << 20)
        g.run(layers)
        print("mpo est", g.mps_fidelity_estimate()["est"], flush=True)
    for chi, cnt in ((64, 4), (128, 2), (256, 1)):
        if "chi%d" % chi not in which:
            continue
        tensors, gates = workloads.micro_chain(chi, cnt)
        g = pk.MPS(2 * cnt, strategy="fixed", f_fixed=0.9999, slab_bytes=1 << 30)
        g.mps_import_sites(0, tensors)
        g.mps_apply_layer(np.arange(0, 2 * cnt, 2, dtype=np.int32), gates)
        print("chi", chi, "k", [r["chi_after"] for r in g.mps_truncation_log()], flush=True)
    print("SANITIZE_CASE_DONE", flush=True)


if __name__ == "__main__":
    main()

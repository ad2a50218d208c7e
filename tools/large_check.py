"""Dev check of the large-regime SVD (tensor-core path by default; EAMPS_LARGE_SIMT=1 for the SIMT
path): sigma parity vs the oracle on a few config-2 thetas and device time of a batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
Gt = int(sys.argv[3]) if len(sys.argv) > 3 else 0
tensors, gates = workloads.micro_chain(chi, G)
gpu = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=8 << 30)
gpu.mps_import_sites(0, tensors)
t0 = time.time()
gpu.mps_apply_layer(np.arange(0, 2 * G, 2, dtype=np.int32), gates)
torch.cuda.synchronize()
print("chi", chi, "G", G, "wall %.3f s" % (time.time() - t0), "sweeps", [gpu.mps_last_sweeps(g) for g in range(G)], flush=True)
if os.environ.get("ORACLE", "1") == "1":
    import oracle
    orc = oracle.OracleMPS(2 * G, strategy="fixed", f_fixed=0.9999)
    for i, B in enumerate(tensors):
        orc.import_site(i, B)
    orc.apply_layer(np.arange(0, 2 * G, 2, dtype=np.int32), gates)
    for g in range(G):
        sg, so = gpu.mps_last_spectrum(g), orc.last_spectrum(g)
        mask = so >= 1e-6 * so[0]
        rel = np.abs(sg[mask] - so[mask]) / so[mask]
        kg = gpu.mps_truncation_log()[g]["chi_after"]; ko = orc.records()[g]["chi_after"]
        print("gate", g, "max rel sigma err %.3e" % rel.max(), "at j", int(rel.argmax()), "k", kg, ko, flush=True)
        if os.environ.get("DETAIL"):
            idx = np.argsort(-rel)[:8]
            print("   worst j:", idx.tolist(), "rel:", ["%.1e" % rel[i] for i in idx], "sigma/s0:", ["%.1e" % (so[mask][i] / so[0]) for i in idx])
            print("   signed (g-o)/o at worst:", ["%.1e" % ((sg[mask][i] - so[mask][i]) / so[mask][i]) for i in idx])
if Gt:
    tensors, gates = workloads.micro_chain(chi, Gt)
    m2 = pk.MPS(2 * Gt, strategy="fixed", f_fixed=0.9999, slab_bytes=int(os.environ.get("SLAB_GB", "40")) << 30)
    m2.mps_import_sites(0, tensors)
    snap = m2.mps_snapshot_save()
    m2.mps_set_profiling(True)
    for rep in range(2):
        m2.mps_snapshot_load(snap)
        torch.cuda.synchronize(); t0 = time.time()
        m2.mps_apply_layer(np.arange(0, 2 * Gt, 2, dtype=np.int32), gates)
        torch.cuda.synchronize()
        print("batch", Gt, "rep", rep, "wall %.3f s" % (time.time() - t0), "sweeps mean", np.mean([m2.mps_last_sweeps(g) for g in range(Gt)]), flush=True)
    print("phases", m2.mps_phase_times())

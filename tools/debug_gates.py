import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads

def run(chi, G, first=0, max_sweeps=60):
    n = 2 * chi
    tensors, gates = workloads.micro_chain(chi, G, first=first)
    inter = torch.as_tensor(np.concatenate([t.ravel() for t in tensors])).cuda()
    dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
    mps = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=(1 << 30) + G * 2 * 1024 * 1024, max_sweeps=max_sweeps)
    mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
    mps.mps_apply_layer(np.arange(0, 2 * G, 2, dtype=np.int32), gates)
    ks = [r["chi_after"] for r in mps.mps_truncation_log()]
    sw = [mps.mps_last_sweeps(g) for g in range(G)]
    sp = [mps.mps_last_spectrum(g) for g in range(G)]
    return ks, sw, sp, tensors

chi = int(sys.argv[1]); G = int(sys.argv[2])
ks, sw, sp, tensors = run(chi, G)
print("ks", ks); print("sweeps", sw)
bad = [g for g in range(G) if ks[g] != ks[0]]
ref = workloads.powerlaw_sigma(2 * chi)
for g in bad[:4]:
    th = workloads.micro_theta(chi, g).astype(np.complex128)
    s = np.linalg.svd(th, compute_uv=False)
    print("gate", g, "k", ks[g], "sweeps", sw[g], "gpu sig[:4]", sp[g][:4], "ref", s[:4], "maxrel", np.max(np.abs(sp[g] - s) / s))
    k1, s1, p1, _ = run(chi, 1, first=g)
    print("   alone: k", k1, "sweeps", s1, "maxrel", np.max(np.abs(p1[0] - s) / s))

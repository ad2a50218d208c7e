import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
chi = int(sys.argv[1]); counts = [int(x) for x in sys.argv[2:]]
for G in counts:
    for gen in ["torch", "numpy"]:
        if gen == "numpy" and G > 512: continue
        n = 2 * chi
        if gen == "torch":
            left, right, gates = workloads.micro_chain_torch(chi, G, device="cuda")
            inter = torch.cat([left.reshape(G, -1), right.reshape(G, -1)], dim=1).reshape(-1)
        else:
            tensors, gates = workloads.micro_chain(chi, G)
            inter = torch.as_tensor(np.concatenate([t.ravel() for t in tensors])).cuda()
        dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
        mps = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=(2 << 30) + G * 2 * 1024 * 1024)
        mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
        try:
            mps.mps_apply_layer(np.arange(0, 2 * G, 2, dtype=np.int32), gates)
            ks = [r["chi_after"] for r in mps.mps_truncation_log()]
            print(gen, G, "ok k range", min(ks), max(ks), "sweeps", mps.mps_last_sweeps(0), flush=True)
        except Exception as e:
            print(gen, G, "FAIL", e, flush=True)
            bad = []
            for g in range(G):
                s = mps.mps_last_spectrum(g)
                if not np.all(np.isfinite(s)): bad.append(g)
            print("  nan gates", bad[:20], len(bad), flush=True)
        del mps

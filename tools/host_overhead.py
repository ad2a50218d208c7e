"""Host-side cost of mps_apply_layer for the bench workload: wall time of the call (host planning +
launch issue) vs the device time of the same step, to see the idle gap at the start of a step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_16870_b200 as pk, workloads
chi, G = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
n = 2 * chi
left, right, gates = workloads.micro_chain_torch(chi, G, device="cuda")
mps = pk.MPS(2 * G, strategy="fixed", f_fixed=0.9999, slab_bytes=8 << 30)
inter = torch.cat([left.reshape(G, -1), right.reshape(G, -1)], dim=1).reshape(-1)
dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
snap = mps.mps_snapshot_save()
sites = np.arange(0, 2 * G, 2, dtype=np.int32)
s = torch.cuda.current_stream()
for rep in range(4):
    mps.mps_snapshot_load(snap)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    mps.mps_apply_layer(sites, gates)
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    print("rep %d: host call %.2f ms, device step %.2f ms" % (rep, (t1 - t0) * 1e3, e0.elapsed_time(e1)))

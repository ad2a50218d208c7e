"""Diagnose the e2e leg: does chunk c+1's H2D (side stream) overlap chunk c's import + update?
Event timeline per chunk (ms from a common start event)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2307_16870_b200 as pk

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
chi, G = 64, 4096
inter, dims, gates = bench.make_inputs(chi, G, 0, dev)
n = 2 * chi
site_bytes = inter.numel() * 8
ws_gate = 4 * n * n * 8 + 16 * n * n + 64 * n + 8192
need = int(2.2 * 2 * site_bytes + G * ws_gate) + (512 << 20)
free, _ = torch.cuda.mem_get_info(dev)
mps = pk.MPS(2 * G, strategy="fixed", f_fixed=bench.F_TRUNC, slab_bytes=int(min(need, 0.7 * free)), device=dev)
sites = np.arange(0, 2 * G, 2, dtype=np.int32)
host = torch.empty(inter.numel(), dtype=torch.complex64, pin_memory=True)
host.copy_(inter.cpu())
per_el = inter.numel() // G
main = torch.cuda.current_stream(dev)
print("main stream handle", main.cuda_stream, flush=True)
for C in (1, 2, 4, 8):
    per = (G + C - 1) // C
    stage = [torch.empty(per * per_el, dtype=torch.complex64, device=dev) for _ in range(2)]
    side = torch.cuda.Stream(device=dev)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        E = lambda: torch.cuda.Event(enable_timing=True)
        start = E(); start.record(main)
        marks = []
        evs = []
        bounds = [(c * per, min(G, (c + 1) * per)) for c in range(C)]
        def issue(c):
            g0, g1 = bounds[c]
            a, b = E(), E()
            with torch.cuda.stream(side):
                side.wait_event(start)
                a.record(side)
                stage[c % 2][: (g1 - g0) * per_el].copy_(host[g0 * per_el: g1 * per_el], non_blocking=True)
                b.record(side)
            evs.append(b)
            marks.append(("h2d%d" % c, a, b))
        th = []
        issue(0)
        for c in range(C):
            if c + 1 < C:
                issue(c + 1)
            g0, g1 = bounds[c]
            main.wait_event(evs[c])
            a, b = E(), E()
            a.record(main)
            h0 = time.perf_counter()
            mps.mps_import_sites_raw(2 * g0, 2 * (g1 - g0), pk.C.c_void_p(stage[c % 2].data_ptr()), dims[2 * g0: 2 * g1])
            mps.mps_apply_layer(sites[g0:g1], gates[g0:g1])
            th.append(time.perf_counter() - h0)
            b.record(main)
            marks.append(("upd%d" % c, a, b))
        recs = mps.mps_truncation_array(last=G)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if rep == 2:
            print("C=%d wall %.1f ms  host-in-calls %s" % (C, wall * 1e3, ["%.1f" % (x * 1e3) for x in th]), flush=True)
            for name, a, b in marks:
                print("   %-6s %7.2f -> %7.2f ms" % (name, start.elapsed_time(a), start.elapsed_time(b)), flush=True)
    del stage

"""Phase times of ONE cap-bound config-5 gate: chi_l = chi_r = 4096, theta 8192 x 8192 (random
Gaussian site tensors: a flat, full-rank spectrum like a deep random circuit's), truncated at the
cap 4096 -- the gates that dominate config 5 from layer 19 on. Prints the device
milliseconds per phase (mps_phase_times) of the second of two identical updates.
usage: cap_gate_profile.py [chi [route]] (route 1 = the tcgen05 Jacobi also where the eigen route applies)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2307_16870_b200 as pk
    import workloads
    chi = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    route = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # mps_set_svd_route: 0 eigen (n <= 4096), 1 Jacobi
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(5)
    sites = []
    for shape in ((chi, 2, chi), (chi, 2, chi)):
        t = torch.randn(*shape, 2, generator=g, device=dev, dtype=torch.float32)
        t = torch.view_as_complex(t).contiguous()
        sites.append(t / t.norm() * (chi ** 0.5))
    U = workloads.haar_u4(5, 1, 2, 3)[None]
    m = pk.MPS(2, strategy="fixed", f_fixed=0.999999, chi_cap=chi, slab_bytes=40 << 30)
    m.mps_set_svd_route(route)
    m.mps_set_profiling(True)
    out = {}
    for rep in range(2):
        for i, t in enumerate(sites):
            m.mps_import_site(i, t)
        m.mps_set_profiling(True)            # resets the timers
        m.mps_apply_layer(np.zeros(1, np.int32), U)
        out = {k: round(v[0], 2) for k, v in m.mps_phase_times().items() if v[0] > 0}
    rec = m.mps_truncation_log()[-1]
    print(json.dumps({"chi": chi, "route": route, "theta": "%d x %d" % (2 * chi, 2 * chi), "phase_ms": out,
                      "sweeps": m.mps_last_sweeps(0), "chi_after": rec["chi_after"], "capped": rec["capped"],
                      "achieved_f": rec["achieved_f"]}))


if __name__ == "__main__":
    main()

"""NEXT-2: the paper's Fig. 4 protocol on this box -- an entanglement-aware run (EA:
fidelity-driven truncation) and the regular fixed-maximum-bond-dimension run with
chi_max = the EA run's peak chi (PAPER.md:195 caption: "the MPS (resp. MPO) maximum bond dimension is
taken as the maximum bond dimension encountered during the EA-MPS (resp. EA-MPO) simulation"), same
kernels, same circuit. Reports device time, the final estimate (E12/E13 ledger), the bond profile
and the memory footprint (sum over sites of chi_l d chi_r complex64) of both.

  python tools/ea_vs_fixed.py --config 3 [--depth 20]     (one GPU)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg_id, depth, f_min, cap, strategy):
    import numpy as np
    import torch

    import paper_2307_16870_b200 as pk
    import workloads
    c = workloads.CONFIGS[cfg_id]
    N, d = c["n_sites"], c["d"]
    if c["kind"] == "mpo":
        full = workloads.mpo_circuit(cfg_id, N, c["depth"], c["p_depol"])
        rule = "wang"
    else:
        full = workloads.brickwork_circuit(cfg_id, N, c["depth"])
        rule = "pure"
    layers = full[:depth]
    free, _ = torch.cuda.mem_get_info()
    m = pk.MPS(N, d=d, f_min=f_min, n_planned=workloads.n_two_qubit_gates(full), strategy=strategy, rule=rule,
               chi_cap=cap, slab_bytes=int(0.85 * free))
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    peak = 1
    for sites, us in layers:
        m.mps_apply_layer(sites, us)
        peak = max(peak, int(max(m.mps_bond_dims())))
    e1.record(stream)
    torch.cuda.synchronize()
    dims = [1] + [int(x) for x in m.mps_bond_dims()] + [1]
    mem = sum(dims[i] * d * dims[i + 1] * 8 for i in range(N))
    est = m.mps_fidelity_estimate()
    recs = m.mps_truncation_array()
    out = dict(seconds=e0.elapsed_time(e1) / 1e3, wall_s=time.perf_counter() - t0, peak_chi=peak,
               final_bonds=dims[1:-1], state_bytes=mem, estimate=est["est"], log_estimate=est["log_est"],
               guarantee_held=bool(est["guarantee_held"]), capped=int(np.sum(recs["capped"])),
               updates=len(recs))
    del m
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--depth", type=int, default=0)
    args = ap.parse_args()
    import workloads
    c = workloads.CONFIGS[args.config]
    depth = args.depth or c["depth"]
    ea = run(args.config, depth, c["f_min"], c["chi_cap"], c["strategy"])
    fx = run(args.config, depth, 1.0, ea["peak_chi"], c["strategy"])
    print(json.dumps({"config": args.config, "layers": depth, "protocol": "PAPER.md Fig. 4: fixed chi_max = EA peak chi",
                      "ea": ea, "fixed": fx, "time_ratio_fixed_over_ea": fx["seconds"] / max(ea["seconds"], 1e-9),
                      "memory_ratio_fixed_over_ea": fx["state_bytes"] / max(ea["state_bytes"], 1)}))


if __name__ == "__main__":
    main()

"""Run BASELINE config 1, 3, 4 or 5 (workloads.CONFIGS) on one GPU through the public API, layer by
layer, printing per-layer device time and the largest bond, then the ledger as one JSON line:

    python tools/run_config.py --config 3 [--depth D] [--slab-gb G]

(--depth limits the layers run; n_planned is always the full circuit's gate count, as in the
configs.) The oracle is not involved: this is the at-scale run the prefix / sampled-gate parity
tests (tests/test_gpu_configs_prefix.py) vouch for."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--depth", type=int, default=0, help="layers to run (0: the whole circuit)")
    ap.add_argument("--slab-gb", type=float, default=0.0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2307_16870_b200 as pk
    import workloads

    cfg = workloads.CONFIGS[args.config]
    N, depth, d = cfg["n_sites"], cfg["depth"], cfg["d"]
    if cfg["kind"] == "mpo":
        layers = workloads.mpo_circuit(args.config, N, depth, cfg["p_depol"])
        rule = "wang"
    else:
        layers = workloads.brickwork_circuit(args.config, N, depth)
        rule = "pure"
    npl = workloads.n_two_qubit_gates(layers)
    free, _ = torch.cuda.mem_get_info()
    slab = int(args.slab_gb * (1 << 30)) if args.slab_gb > 0 else int(0.85 * free)
    gpu = pk.MPS(N, d=d, f_min=cfg["f_min"], n_planned=npl, strategy=cfg["strategy"], rule=rule,
                 chi_cap=cfg["chi_cap"], slab_bytes=slab)
    run = layers[:args.depth] if args.depth > 0 else layers
    t_all = 0.0
    for t, (sites, us) in enumerate(run):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gpu.mps_apply_layer(sites, us)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t_all += dt
        print("layer %d: %d gates, %.2f s, max bond %d" % (t, len(sites), dt, max(gpu.mps_bond_dims())), flush=True)
    est = gpu.mps_fidelity_estimate()
    recs = gpu.mps_truncation_log()
    print(json.dumps({"config": args.config, "n_sites": N, "d": d, "layers_run": len(run), "layers_total": depth,
                      "seconds": t_all, "gate_updates": len(recs), "max_bond": int(max(gpu.mps_bond_dims())),
                      "capped": int(sum(r["capped"] for r in recs)), "estimate": est["est"],
                      "guarantee_held": bool(est["guarantee_held"])}), flush=True)


if __name__ == "__main__":
    main()

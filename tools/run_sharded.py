"""Config-5-style sharded run: one long brickwork MPS split in contiguous site blocks over the
ranks of a torchrun job; NCCL point-to-point for the boundary exchange and the
ledger token (paper_2307_16870_b200/sharded.py).

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/run_sharded.py \
      [--sites 300] [--depth 12] [--fmin 0.9] [--cap 4096]

Prints, on rank 0, one JSON line: layers/s, gate updates/s, bond profile maximum, ledger."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sites", type=int, default=300)
    ap.add_argument("--depth", type=int, default=12)
    ap.add_argument("--fmin", type=float, default=0.9)
    ap.add_argument("--cap", type=int, default=4096)
    ap.add_argument("--full-depth", type=int, default=75, help="n_planned is the full circuit's gate count")
    ap.add_argument("--slab-gb", type=float, default=0.0)
    ap.add_argument("--progress", action="store_true", help="per-layer time and bond dimension (rank 0)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2307_16870_b200 as pk
    import workloads
    from paper_2307_16870_b200.sharded import GpuEngine, ShardedMPS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N = args.sites
    n_planned = workloads.n_two_qubit_gates([(workloads.brickwork_sites(N, t), None) for t in range(args.full_depth)])
    free, _ = torch.cuda.mem_get_info(dev)
    slab = int(args.slab_gb * (1 << 30)) if args.slab_gb > 0 else int(0.6 * free)
    kw = dict(f_min=args.fmin, n_planned=n_planned, strategy="global", chi_cap=args.cap)
    sh = ShardedMPS(N, lambda n: GpuEngine(pk.MPS(n, slab_bytes=slab, device=dev, **kw)), device=dev)
    layers = workloads.brickwork_circuit(5, N, args.depth)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nrec = 0
    for li, (sites, us) in enumerate(layers):
        tl = time.perf_counter()
        sh.apply_layer(sites, us)
        if args.progress:
            torch.cuda.synchronize()
            recs = sh.records()
            chi = max((r["chi_after"] for r in recs[nrec:]), default=0)
            nrec = len(recs)
            if sh.rank == 0:
                print("layer %d: %d gates, %.2f s, max chi_after (this rank) %d" % (li, len(sites), time.perf_counter() - tl, chi),
                      flush=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    led = sh.ledger()
    if world > 1:
        dist.barrier()
    if sh.rank == 0:
        gates = workloads.n_two_qubit_gates(layers)
        print(json.dumps({"workload": "config5 prefix N=%d depth %d" % (N, args.depth), "ranks": sh.world,
                          "blocks": sh.blocks, "seconds": dt, "gate_updates_per_s": gates / dt,
                          "log_E": led[0], "truncations": led[1], "guarantee_held": bool(led[2])}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

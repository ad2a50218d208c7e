#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on BASELINE.json configs[1] (the isolated batched gate-update
microbench): 4096 independent two-site updates per step, chi_l = chi_r = chi (d = 2), theta with
a sigma_k ~ k^-1.5 spectrum, per-update target fidelity 0.9999 (rule pure), contract-inclusive
(B_left, B_right, Haar U -> contract -> SVD -> select -> reabsorb), all through the C ABI.

  python bench.py [--gpus N --steps K --warmup W] [--chi 64] [--count 4096] [--impl reference]

One JSON line on rank 0 (see DESIGN.md "Measurement" for every field). A step = one
mps_apply_layer over the 4096-gate layer (all §8(a) rows a0-a5); the state is restored from a
device snapshot and L2 is flushed between steps (both untimed). Multi-GPU (torchrun): each rank
runs its own 4096 updates (independent problems, no collective on the data path: weak scaling),
time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "2-qubit MPS gate updates/s (contract+SVD+truncate); TFLOP/s as % of FP32 peak"
UNIT = "gate updates/s"
F_TRUNC = 0.9999
# FP32 SIMT peak derived from the guide's unit counts: 148 SMs x 128 FP32
# lanes x 2 flop/FMA x 1.965 GHz (clocks.max.sm)
FP32_SIMT_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def _tf32_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp["bf16_tflops"] * (1.13 / 2.25), "measured bf16 burst %.1f TF/s (MEASURED_PEAKS.json) x nominal TF32/BF16 1.13/2.25" % mp["bf16_tflops"]
    except Exception:
        return 1590.0 * (1.13 / 2.25), "fallback bf16 1590 TF/s (B200_PROFILING.md) x nominal TF32/BF16 1.13/2.25"


TF32_PEAK_TFLOPS, TF32_PEAK_SRC = _tf32_peak()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="eamps", choices=["eamps", "reference"])
    ap.add_argument("--chi", type=int, default=int(os.environ.get("BENCH_CHI", "64")))
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def svd_flops(m, n, sweeps):
    """algorithmic flops of the scalar one-sided Jacobi: (20 m n^2 + 12 n^3) per sweep."""
    return sweeps * (20.0 * m * n * n + 12.0 * n ** 3)


def update_flops(chi, sweeps, k):
    """contract + SVD + reabsorb for one config-2 theta (m = n = 2 chi, chi_m = 2 chi, d = 2)."""
    d, l, mid, r = 2, chi, 2 * chi, chi
    m, n = d * l, d * r
    contract = 8 * d * d * l * mid * r + 8 * d ** 4 * l * r
    return contract + svd_flops(m, n, sweeps) + 8.0 * m * n * k


# ------------------------------------------------------------------------------ multi-rank
def rank_seed_range(rank, count):
    """Each rank runs its own `count` config-2 updates (weak scaling, no data-path collective):
    seeds b in [rank*count, (rank+1)*count)."""
    return rank * count, (rank + 1) * count


def max_over_ranks(value, device=None):
    """Device-timed totals are reduced with MAX over ranks (the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region: NVML polled every 2 ms from a
    thread (short timed regions still get samples); nvidia-smi -lms 200 if NVML is unavailable."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None
        self.nv = None
        self.rows = []
        self.run = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = gpu_index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                ids = [x.strip() for x in vis.split(",") if x.strip()]
                if gpu_index < len(ids) and ids[gpu_index].isdigit():
                    idx = int(ids[gpu_index])
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv = nv
            self.bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            self.nv = None

    def _poll(self):
        nv = self.nv
        mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        while self.run:
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append(dict(sm=sm, mx=mx, reasons=["active" if rs & b else "" for b in self.bits]))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nv is not None:
            import threading
            self.run = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        rows = []
        if self.nv is not None:
            self.run = False
            self.t.join(timeout=5)
            rows = self.rows
        elif self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.flush()
            for line in open(self.f.name):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append(dict(sm=float(parts[1]), mx=float(parts[2]), reasons=parts[5:9]))
                except ValueError:
                    continue
            os.unlink(self.f.name)
        if not rows:
            return None
        loaded = [r for r in rows if r["sm"] > 300] or rows
        seen = sorted({self.NAMES[i] for r in rows for i, v in enumerate(r["reasons"]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r["sm"] for r in loaded])), "sm_max_mhz": rows[0]["mx"],
                "reasons": seen, "samples": len(rows), "source": "nvml" if self.nv is not None else "nvidia-smi"}


# ------------------------------------------------------------------------------ reference arm
def cpu_sample(chi, budget_s, first=0):
    """Time the oracle (as it stands) on the first G_s updates of the same workload."""
    import workloads
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    import oracle

    def run(G):
        tensors, gates = workloads.micro_chain(chi, G, first=first)
        o = oracle.OracleMPS(2 * G, strategy="fixed", f_fixed=F_TRUNC)
        for i, B in enumerate(tensors):
            o.import_site(i, B)
        sites = np.arange(0, 2 * G, 2, dtype=np.int32)
        t0 = time.perf_counter()
        o.apply_layer(sites, gates)
        return time.perf_counter() - t0

    t1 = run(1)  # one update, one thread
    G = int(max(1, min(4096, budget_s * cores / max(t1, 1e-4))))
    dt = run(G) if G > 1 else t1
    return dict(value=G / dt, unit=UNIT, cores=int(os.environ.get("OMP_NUM_THREADS", cores)), kind="oracle",
                sample="%d of the %d chi=%d updates (first seeds), OpenMP over gates, %.1f s" % (G, 4096, chi, dt))


def run_reference(args, rank, world):
    if rank != 0:
        return
    import workloads  # noqa: F401
    per_step = max(2.0, 150.0 / (args.steps + args.warmup))
    cb = cpu_sample(args.chi, per_step)
    G = int(round(cb["value"] * per_step)) or 1
    import oracle
    times = []
    for step in range(args.warmup + args.steps):
        tensors, gates = workloads.micro_chain(args.chi, G, first=step * G)
        o = oracle.OracleMPS(2 * G, strategy="fixed", f_fixed=F_TRUNC)
        for i, B in enumerate(tensors):
            o.import_site(i, B)
        t0 = time.perf_counter()
        o.apply_layer(np.arange(0, 2 * G, 2, dtype=np.int32), gates)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = G / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, BASELINE configs[1] recipe)",
            "impl": "reference",
            "config": {"workload": "config2_microbench chi=%d contract-inclusive, oracle sample of %d updates/step"
                       % (args.chi, G), "chi": args.chi, "count": G, "f_trunc": F_TRUNC},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"], "kind": "oracle",
                             "sample": "%d updates per step (of 4096), %d steps" % (G, args.steps)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2307_16870_b200 as pk
    import workloads

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    chi, G = args.chi, args.count
    n = 2 * chi
    # ---- inputs: this rank's 4096 updates (seeds b = rank*G .. rank*G + G - 1)
    left, right, gates = workloads.micro_chain_torch(chi, G, first=rank_seed_range(rank, G)[0], device=dev)
    site_bytes = (left.numel() + right.numel()) * 8
    # one wave needs: old + new site blocks (pow2 classes), theta/Theta'/V/E, the medium-regime
    # rotation log (24 sweeps x (n-1) x n/2 x 16 B) and small arrays; take it from the free memory
    ws_gate = 4 * n * n * 8 + 24 * (n - 1) * (n // 2) * 16 + 64 * n + 8192
    need = int(2.2 * 2 * site_bytes + G * ws_gate) + (512 << 20)
    free, _ = torch.cuda.mem_get_info(dev)
    slab_bytes = int(min(max(need, 1 << 30), 0.6 * free))
    mps = pk.MPS(2 * G, strategy="fixed", f_fixed=F_TRUNC, slab_bytes=slab_bytes, device=dev)
    inter = torch.cat([left.reshape(G, -1), right.reshape(G, -1)], dim=1).reshape(-1)  # L0 R0 L1 R1 ...
    dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
    mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
    snap = mps.mps_snapshot_save()
    sites = np.arange(0, 2 * G, 2, dtype=np.int32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step_timed():
        mps.mps_snapshot_load(snap)
        flush.zero_()  # L2 flush (256 MB > 126 MB L2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mps.mps_apply_layer(sites, gates)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step_timed()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    mps.mps_set_profiling(True)
    l0 = mps.mps_launch_count()
    total_ms = 0.0
    for _ in range(args.steps):
        total_ms += step_timed()
    launches = mps.mps_launch_count() - l0
    phases = mps.mps_phase_times()
    mps.mps_set_profiling(False)
    clocks = clk.stop()
    sweeps = np.array([mps.mps_last_sweeps(g) for g in range(G)])
    ks = np.array(mps.mps_truncation_array(last=G)["chi_after"])
    if world > 1:
        total_ms = max_over_ranks(total_ms, dev)
    ms_step = total_ms / args.steps
    value = world * G / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (the SVD phase)
    svd_key = "svd_small" if phases["svd_small"][1] else "svd_blocked"
    svd_ms, svd_n = phases[svd_key]
    svd_ms_per_launch = svd_ms / max(1, svd_n)
    alg_svd = float(sum(svd_flops(n, n, s) for s in sweeps))  # per launch (one wave = the layer)
    achieved = alg_svd / (svd_ms_per_launch / 1e3) / 1e12
    if svd_key == "svd_blocked":
        # large regime: tcgen05 3xTF32 block Jacobi -> the tensor roofline. TF32 dense peak = the
        # measured cuBLAS bf16 burst x the nominal TF32/BF16 ratio (1.13 / 2.25 PFLOP/s, guide)
        peak, bound, peak_src = TF32_PEAK_TFLOPS, "tensor", TF32_PEAK_SRC
    else:
        peak, bound, peak_src = FP32_SIMT_PEAK_TFLOPS, "alu", "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md)"
    traffic = None
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tj):
        try:
            traffic = json.load(open(tj)).get("chi%d" % chi, {}).get(svd_key)
        except Exception:
            traffic = None
    total_flops = float(sum(update_flops(chi, s, k) for s, k in zip(sweeps, ks)))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64 (fp32 complex; fp64 norms/Rayleigh)",
        "data": "synthetic (seeded BASELINE configs[1] recipe: theta = X diag(k^-1.5) Y^H, Haar X/Y/U)",
        "config": {"workload": "config2_microbench chi=%d x%d contract-inclusive (configs[1])" % (chi, G),
                   "chi": chi, "count": G, "theta": "%dx%d" % (n, n), "f_trunc": F_TRUNC, "rule": "pure",
                   "parallelism": "independent updates per rank" if world > 1 else "single GPU",
                   "l2": "flushed between steps (256 MB write)"},
        "tflops_algorithmic": total_flops / (ms_step / 1e3) / 1e12 * world,
        "pct_fp32_simt_peak": 100.0 * total_flops / (ms_step / 1e3) / 1e12 / FP32_SIMT_PEAK_TFLOPS,
        "sweeps_mean": float(sweeps.mean()), "k_mean": float(ks.mean()),
        "phase_ms_per_step": {p: v[0] / max(1, args.steps) for p, v in phases.items()},
        "roofline": {"bound": bound, "kernel": svd_key, "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "flops": "algorithmic: sweeps x (20 m n^2 + 12 n^3) per theta (scalar one-sided Jacobi count)"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    # ---- e2e: host (pinned) inputs -> H2D -> update -> D2H of the step's records, through the ABI
    if not args.no_e2e:
        host = torch.empty(inter.numel(), dtype=torch.complex64, pin_memory=True)
        host.copy_(inter.cpu())
        reps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        t_e2e = 0.0
        for rep in range(reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(host.data_ptr()), dims)
            mps.mps_apply_layer(sites, gates)
            recs = mps.mps_truncation_array(last=G)   # the step's result, D2H (no per-record Python objects)
            torch.cuda.synchronize()
            if rep > 0:
                t_e2e += time.perf_counter() - t0
        assert len(recs) == G
        if world > 1:   # the slowest rank defines the end-to-end step too
            t_e2e = max_over_ranks(t_e2e, dev)
        line["e2e"] = {"value": world * G / (t_e2e / reps), "unit": UNIT,
                       "h2d_bytes_per_step": int(site_bytes + gates.nbytes),
                       "d2h_bytes_per_step": int(G * (48 + 160) + 512)}
    if rank == 0 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sample(chi, args.cpu_seconds)
        except Exception as e:  # the baseline never blocks the GPU line
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

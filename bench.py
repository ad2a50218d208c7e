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
PEAKS_FILE = os.path.join(ROOT, "profiles", "r02", "peaks.json")


def _peaks():
    """Roofline denominators: MEASURED on this pool's B200s by tools/peaks/peaks.cu (committed result
    profiles/r02/peaks.json: FFMA / FFMA2 loops for the FP32 SIMT peak, a DFMA loop for FP64, a
    tcgen05.mma kind::tf32 M128 N256 loop for TF32 dense), else derived (the guide's unit counts x
    clocks.max.sm, and measured bf16 x the nominal TF32/BF16 ratio), each with its source."""
    out = {}
    try:
        pk = json.load(open(PEAKS_FILE))
        fp32 = max(pk["fp32_ffma_tflops"], pk["fp32_ffma2_tflops"])
        out["fp32"] = (fp32, "measured: tools/peaks FFMA2 loop %.1f TF/s (FFMA %.1f), profiles/r02/peaks.json"
                       % (pk["fp32_ffma2_tflops"], pk["fp32_ffma_tflops"]))
        out["tf32"] = (pk["tf32_tcgen05_m128n256_tflops"],
                       "measured: tools/peaks tcgen05.mma kind::tf32 M128 N256 K8 loop, profiles/r02/peaks.json")
        out["fp64"] = (pk["fp64_dfma_tflops"], "measured: tools/peaks DFMA loop, profiles/r02/peaks.json")
        try:
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            out["hbm"] = (mp["hbm_gbs"], "measured (driver): MEASURED_PEAKS.json hbm_gbs, torch copy_ of 1 Gi bf16")
        except Exception:
            out["hbm"] = (7700.0, "nominal B200 HBM3e 7.7 TB/s (MEASURED_PEAKS.json absent)")
    except Exception:
        out["fp32"] = (148 * 128 * 2 * 1.965e9 / 1e12, "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz")
        try:
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            out["tf32"] = (mp["bf16_tflops"] * (1.13 / 2.25), "derived: measured bf16 burst x nominal TF32/BF16 1.13/2.25")
        except Exception:
            out["tf32"] = (1590.0 * (1.13 / 2.25), "fallback bf16 1590 TF/s x nominal TF32/BF16 1.13/2.25")
        out["fp64"] = (148 * 64 * 2 * 1.965e9 / 1e12, "derived: 148 SM x 64 FP64 lanes x 2 x 1.965 GHz")
        out["hbm"] = (7700.0, "nominal B200 HBM3e 7.7 TB/s (peaks files absent)")
    return out


PEAKS = _peaks()
FP32_SIMT_PEAK_TFLOPS = PEAKS["fp32"][0]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="eamps", choices=["eamps", "reference"])
    ap.add_argument("--chi", type=int, default=int(os.environ.get("BENCH_CHI", "64")))
    ap.add_argument("--count", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=int(os.environ.get("BENCH_E2E_CHUNKS", "3")),
                    help="pipeline the e2e H2D in C chunks (measured r02 after the SM-driven small uploads: "
                         "equal chunks 1 -> 51.8K, 2 -> 58.3K, 4 -> 60.3K updates/s; geometric (x2.5) chunks "
                         "3 -> 63.3K, 4 -> 62.7K, 5 -> 61.8K: each chunk costs ~0.7 ms of host work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-chi", action="store_true")
    ap.add_argument("--per-chi", default=os.environ.get("BENCH_PER_CHI", "16:4096:5:3,256:4096:3:2,1024:512:2:1"),
                    help="chi:count:steps:warmup sub-records (the large-chi half of configs[1])")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--config5-depth", type=int, default=int(os.environ.get("BENCH_C5_DEPTH", "17")),
                    help="layers of the config-5 sharded slice (0 = skip)")
    return ap.parse_args()


def regime_of(m, n):
    """The SVD regime the library's planner picks (C ABI mps_plan_regime, host only)."""
    import paper_2307_16870_b200 as pk
    return pk.mps_plan_regime(m, n)[0]


def jacobi_flops(m, n, sweeps, regime):
    """Algorithmic flops of the one-sided Jacobi the kernel EXECUTES (SURVEY §8(d) scalar count,
    20 rows n^2 per sweep for the column pairs, + 12 n^3 when V is accumulated): the QR (3) and
    large (1) regimes run on the n x n preconditioned factor B = L (rows = n) with no V; the small
    (0) and medium (2) regimes on theta (rows = m) with V."""
    if regime in (1, 3):
        return sweeps * 20.0 * n ** 3
    return sweeps * (20.0 * m * n * n + 12.0 * n ** 3)


def svd_support_flops(m, n, regime):
    """Executed flops around the Jacobi (reported, not in the roofline): FP64 Gram theta^H theta (4 m n^2,
    Hermitian half) + Cholesky (8 n^3 / 3) for the preconditioned regimes; Rayleigh quotient theta V
    (8 m n^2); polish C = B^H B (4 m n^2) for regimes 1 and 3."""
    f = 8.0 * m * n * n
    if regime in (1, 3):
        f += 4.0 * m * n * n + 8.0 * n ** 3 / 3 + 4.0 * m * n * n
    return f


def eig_route_flops(m, n, k, d=2, l=None, mid=None, r=None):
    """Executed FP64 flops of the eigen route (refine_large.cu) for one m x n theta: the FP64
    recontraction (8 d^2 l mid r + 8 d^4 l r), the Hermitian Gram (4 m n^2), the Householder
    tridiagonalisation (16 n^3 / 3), the back-transformation of the k kept vectors (8 n^2 k)."""
    contract = 8.0 * d * d * l * mid * r + 8.0 * d ** 4 * l * r
    return contract + 4.0 * m * n * n + 16.0 * n ** 3 / 3 + 8.0 * n * n * k


def tridiag_bytes(n):
    """Algorithmic HBM bytes of a one-stage Householder tridiagonalisation of an n x n complex128
    Hermitian matrix: every step reads and writes its trailing triangle, sum_t 2 x 16 t^2 / 2 =
    16 n^3 / 3 (the kernel keeps both triangles and moves 2x that)."""
    return 16.0 * n ** 3 / 3


def update_flops(chi, sweeps, k, regime):
    """contract + SVD (executed) + reabsorb for one config-2 theta (m = n = 2 chi, chi_m = 2 chi, d = 2)."""
    d, l, mid, r = 2, chi, 2 * chi, chi
    m, n = d * l, d * r
    contract = 8 * d * d * l * mid * r + 8 * d ** 4 * l * r
    return contract + jacobi_flops(m, n, sweeps, regime) + svd_support_flops(m, n, regime) + 8.0 * m * n * k


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
    G = min(int(round(cb["value"] * per_step)) or 1, args.count)   # never more than the workload's layer
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
def make_inputs(chi, G, first, dev, chunk=None):
    """Config-2 contract-inclusive inputs (workloads.micro_chain_torch recipe, seeds b = first ..
    first + G - 1), generated in chunks (the complex128 QRs of a chi = 1024 batch do not fit at once)
    into one interleaved complex64 device buffer L0 R0 L1 R1 ..., the site dims and the gates."""
    import torch

    import workloads
    n = 2 * chi
    per = chi * 2 * n + n * 2 * chi
    if chunk is None:
        chunk = max(1, min(G, (1 << 31) // (n * n * 16 * 4)))
    inter = torch.empty(G * per, dtype=torch.complex64, device=dev)
    gates = []
    for c0 in range(0, G, chunk):
        c = min(chunk, G - c0)
        left, right, u = workloads.micro_chain_torch(chi, c, first=first + c0, device=dev)
        inter[c0 * per:(c0 + c) * per] = torch.cat([left.reshape(c, -1), right.reshape(c, -1)], dim=1).reshape(-1)
        gates.append(u)
        del left, right
    dims = np.array([[chi, 2, n], [n, 2, chi]] * G, np.int32)
    return inter, dims, np.concatenate(gates)


def run_chi(chi, G, steps, warmup, rank, world, dev, clocks=True):
    """Time `steps` mps_apply_layer calls over one G-gate config-2 layer (after `warmup` untimed
    ones): state restored before every step (snapshot, or re-import for big site stores) and L2
    flushed, both untimed. Returns (record, handle, device inputs, dims, gates)."""
    import torch
    import torch.distributed as dist

    import paper_2307_16870_b200 as pk
    n = 2 * chi
    inter, dims, gates = make_inputs(chi, G, rank_seed_range(rank, G)[0], dev)
    site_bytes = inter.numel() * 8
    # one wave needs: old + new site blocks (pow2 classes), theta/Theta'/V/E, the regime scratch
    # (large: FP64 Gram 16 n^2) and small arrays; take it from the free memory
    ws_gate = 4 * n * n * 8 + 16 * n * n + 64 * n + 8192
    need = int(2.2 * 2 * site_bytes + G * ws_gate) + (512 << 20)
    free, _ = torch.cuda.mem_get_info(dev)
    slab_bytes = int(min(max(need, 1 << 30), 0.7 * free))
    mps = pk.MPS(2 * G, strategy="fixed", f_fixed=F_TRUNC, slab_bytes=slab_bytes, device=dev)
    mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)
    use_snap = site_bytes < (8 << 30)
    snap = mps.mps_snapshot_save() if use_snap else None
    sites = np.arange(0, 2 * G, 2, dtype=np.int32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def restore():
        if use_snap:
            mps.mps_snapshot_load(snap)
        else:
            mps.mps_import_sites_raw(0, 2 * G, pk.C.c_void_p(inter.data_ptr()), dims)

    def step_timed():
        restore()
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

    for _ in range(warmup):
        step_timed()
    clk = ClockSampler(torch.cuda.current_device()) if clocks else None
    if clk:
        clk.start()
    mps.mps_set_profiling(True)
    l0 = mps.mps_launch_count()
    total_ms = 0.0
    for _ in range(steps):
        total_ms += step_timed()
    launches = mps.mps_launch_count() - l0
    phases = mps.mps_phase_times()
    mps.mps_set_profiling(False)
    clk_rec = clk.stop() if clk else None
    sweeps = np.array([mps.mps_last_sweeps(g) for g in range(G)])
    ks = np.array(mps.mps_truncation_array(last=G)["chi_after"])
    if world > 1:
        total_ms = max_over_ranks(total_ms, dev)
    ms_step = total_ms / steps
    regime = regime_of(n, n)
    eig = regime in (1, 3) and phases["svd_eig_tridiag"][1] > 0 and bool(np.all(sweeps == 0))
    traffic = None
    tj = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    if eig:
        # ---- the eigen route (reading 20): the dominant kernel is the Householder
        # tridiagonalisation, bound by the traffic of the trailing matrix (algorithmic bytes per
        # launch = one wave's gates x 16 n^3 / 3) over its CUDA-event time (sub-phase svd_eig_tridiag)
        kern, (kms, kn) = "svd_eig_tridiag", phases["svd_eig_tridiag"]
        kms_launch = kms / max(1, kn)
        if regime == 1:
            per_launch_bytes = G * tridiag_bytes(n) * steps / kn
            achieved = per_launch_bytes / (kms_launch / 1e3) / 1e9
            (peak, peak_src), bound, unit = PEAKS["hbm"], "hbm", "GB/s"
            flops_note = ("algorithmic bytes per launch: gates x 16 n^3 / 3 (one-stage Householder "
                          "tridiagonalisation, trailing Hermitian lower triangle read + written per step)")
        else:
            # n <= 128: one CTA per gate, G in shared memory (k_eig_cta: tridiagonalisation + bisection
            # + spectrum); FP64 ALU-bound at best -- counted: the tridiagonalisation's 16 n^3 / 3 flops
            per_launch_flops = G * 16.0 * n ** 3 / 3 * steps / kn
            achieved = per_launch_flops / (kms_launch / 1e3) / 1e12
            (peak, peak_src), bound, unit = PEAKS["fp64"], "alu", "TFLOP/s"
            flops_note = ("algorithmic FP64 flops per launch: gates x 16 n^3 / 3 (Householder tridiagonalisation "
                          "of the n x n Hermitian Gram; the bisection and the spectrum are not counted)")
        total_flops = float(sum(eig_route_flops(n, n, k, 2, chi, 2 * chi, chi) for k in ks)
                            + sum(8.0 * n * n * k for k in ks))
    else:
        # ---- roofline of the dominant kernel: the Jacobi SVD. Its executed algorithmic flops per
        # launch (one launch group per wave) / its CUDA-event time (sub-phase svd_jacobi when the
        # planner times it, else the whole SVD phase, which then also holds the support kernels)
        alg = float(sum(jacobi_flops(n, n, sw, regime) for sw in sweeps))
        if phases["svd_jacobi"][1]:
            kern, (kms, kn) = "svd_jacobi", phases["svd_jacobi"]
            per_launch_alg = alg * steps / kn
        else:
            kern = "svd_small" if phases["svd_small"][1] else "svd_blocked"
            kms, kn = phases[kern]
            per_launch_alg = alg * steps / kn
        kms_launch = kms / max(1, kn)
        achieved = per_launch_alg / (kms_launch / 1e3) / 1e12
        if regime == 1:
            (peak, peak_src), bound = PEAKS["tf32"], "tensor"
        else:
            (peak, peak_src), bound = PEAKS["fp32"], "alu"
        unit = "TFLOP/s"
        flops_note = ("executed algorithmic Jacobi flops per launch: sweeps x 20 rows n^2 (+12 n^3 with V); "
                      "rows = n for the preconditioned V-less regimes (QR, large)")
        total_flops = float(sum(update_flops(chi, sw, k, regime) for sw, k in zip(sweeps, ks)))
    if os.path.exists(tj):
        try:
            traffic = json.load(open(tj)).get("chi%d" % chi, {}).get(kern)
        except Exception:
            traffic = None
    svd_phase_ms = (phases["svd_small"][0] + phases["svd_blocked"][0]) / steps
    rec = {
        "value": world * G / (ms_step / 1e3), "unit": UNIT, "ms_per_step": ms_step, "steps": steps, "warmup": warmup,
        "count": G, "chi": chi, "theta": "%dx%d" % (n, n),
        "svd_regime": ({1: "large (FP64 Gram eigensolver)", 3: "QR-size (one-CTA FP64 Gram eigensolver)"}[regime] if eig
                       else {0: "small", 1: "large (tcgen05)", 2: "medium", 3: "QR-preconditioned"}[regime]),
        "tflops_executed": total_flops / (ms_step / 1e3) / 1e12 * world,
        "sweeps_mean": float(sweeps.mean()), "k_mean": float(ks.mean()),
        "phase_ms_per_step": {p: v[0] / max(1, steps) for p, v in phases.items()},
        "svd_phase_ms_per_step": svd_phase_ms,
        "roofline": {"bound": bound, "kernel": kern, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "launch_ms": kms_launch, "flops": flops_note},
        "gpu_launches": int(launches),
        "clocks": clk_rec,
    }
    return rec, mps, inter, dims, gates


def run_config5_slice(depth, rank, world, dev, comm=None, solo=False):
    """BASELINE configs[4] (config 5: N = 300, Haar brickwork, F_min = 0.9 over the full depth-75
    circuit's gate count, cap 4096) on its first `depth` layers, sites sharded in contiguous
    Sigma chi^3-weighted blocks over the ranks (sharded.py: NCCL point-to-point ghost fetch /
    write-back and the ledger token). Device time (CUDA events on each rank's stream around the
    whole slice), max over ranks. solo=True: this rank alone, world 1 (the T_1 of the efficiency)."""
    import torch

    import paper_2307_16870_b200 as pk
    import workloads
    from paper_2307_16870_b200.sharded import DistComm, GpuEngine, ShardedMPS, predicted_site_cost
    N, full_depth, cap = 300, 75, 4096
    n_planned = workloads.n_two_qubit_gates([(workloads.brickwork_sites(N, t), None) for t in range(full_depth)])
    layers = workloads.brickwork_circuit(5, N, depth)
    free, _ = torch.cuda.mem_get_info(dev)
    slab = int(0.6 * free)
    kw = dict(f_min=0.9, n_planned=n_planned, strategy="global", chi_cap=cap)
    p = 1 if solo else world
    comm = None if (solo or world == 1) else DistComm()
    sh = ShardedMPS(N, lambda n: GpuEngine(pk.MPS(n, slab_bytes=slab, device=dev, **kw)), comm=comm, device=dev,
                    weights=predicted_site_cost(N, depth, 2, cap))
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for sites, us in layers:
        sh.apply_layer(sites, us)
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    if p > 1:
        sec = max_over_ranks(sec, dev)
    led = sh.ledger()
    gates = workloads.n_two_qubit_gates(layers)
    chi_max = max((r["chi_after"] for r in sh.eng.records()), default=0)
    out = {"workload": "config5 (configs[4]) N=300 layers 0-%d of 75, cap 4096, F_min 0.9 global" % (depth - 1),
           "ranks": p, "blocks": sh.blocks, "seconds": sec, "value": gates / sec, "unit": UNIT,
           "boundary_messages_rank": sh.exchanges, "chi_max_rank0": int(chi_max),
           "log_E": led[0], "truncations": int(led[1]), "guarantee_held": bool(led[2])}
    del sh
    torch.cuda.empty_cache()
    return out


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

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    chi, G = args.chi, args.count
    rec, mps, inter, dims, gates = run_chi(chi, G, args.steps, args.warmup, rank, world, dev)
    site_bytes = inter.numel() * 8
    line = {
        "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64 (fp32 complex; fp64 norms/Gram/Rayleigh)",
        "data": "synthetic (seeded BASELINE configs[1] recipe: theta = X diag(k^-1.5) Y^H, Haar X/Y/U)",
        "config": {"workload": "config2_microbench chi=%d x%d contract-inclusive (configs[1])" % (chi, G),
                   "chi": chi, "count": G, "theta": rec["theta"], "f_trunc": F_TRUNC, "rule": "pure",
                   "parallelism": "independent updates per rank" if world > 1 else "single GPU",
                   "l2": "flushed between steps (256 MB write)"},
        "tflops_executed": rec["tflops_executed"],
        "pct_fp32_simt_peak": 100.0 * rec["tflops_executed"] / world / FP32_SIMT_PEAK_TFLOPS,
        "svd_regime": rec["svd_regime"], "sweeps_mean": rec["sweeps_mean"], "k_mean": rec["k_mean"],
        "phase_ms_per_step": rec["phase_ms_per_step"],
        "roofline": rec["roofline"],
        "gpu_launches": rec["gpu_launches"],
        "clocks": rec["clocks"],
    }
    sites = np.arange(0, 2 * G, 2, dtype=np.int32)
    # ---- e2e: host (pinned) inputs -> H2D -> update -> D2H of the step's records, through the ABI.
    # The layer runs in C chunks of G / C independent updates (FIXED targets: the chunks' results are
    # those of the whole layer); chunk c+1's host->device copy (pinned -> a device staging buffer, on a
    # side stream) overlaps chunk c's import (device -> pool) and update. Every input byte still
    # crosses PCIe inside the timed region; the records of all G updates are read back at the end.
    if not args.no_e2e:
        host = torch.empty(inter.numel(), dtype=torch.complex64, pin_memory=True)
        host.copy_(inter.cpu())
        reps = max(1, min(args.steps, 3))
        C = max(1, min(args.e2e_chunks, G))
        # geometric chunk sizes (ratio 2.5): each chunk's H2D (~4.8 us per chi = 64 update at
        # ~55 GB/s) hides under the previous chunk's update (~14.5 us per update), and only the
        # small first chunk's copy is exposed
        wts = [2.5 ** c for c in range(C)]
        cuts = [0] + [int(round(G * sum(wts[:c + 1]) / sum(wts))) for c in range(C)]
        bounds = [(cuts[c], cuts[c + 1]) for c in range(C) if cuts[c + 1] > cuts[c]]
        C = len(bounds)
        per = max(g1 - g0 for g0, g1 in bounds)
        per_el = inter.numel() // G                        # complex elements per update (two sites)
        stage = [torch.empty(per * per_el, dtype=torch.complex64, device=dev) for _ in range(2)]
        side = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream(dev)
        if world > 1:
            dist.barrier()

        def e2e_step():
            evs = []

            def issue(c):
                g0, g1 = bounds[c]
                ev = torch.cuda.Event()
                with torch.cuda.stream(side):
                    stage[c % 2][: (g1 - g0) * per_el].copy_(host[g0 * per_el: g1 * per_el], non_blocking=True)
                    ev.record(side)
                evs.append(ev)

            issue(0)
            for c in range(C):
                if c + 1 < C:
                    issue(c + 1)                            # buffer (c+1) % 2 was freed by chunk c-1's import
                g0, g1 = bounds[c]
                main.wait_event(evs[c])
                mps.mps_import_sites_raw(2 * g0, 2 * (g1 - g0), pk.C.c_void_p(stage[c % 2].data_ptr()),
                                         dims[2 * g0: 2 * g1])
                mps.mps_apply_layer(sites[g0:g1], gates[g0:g1])
            return mps.mps_truncation_array(last=G)     # the step's result, D2H

        t_e2e = 0.0
        for rep in range(reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            recs = e2e_step()
            torch.cuda.synchronize()
            if rep > 0:
                t_e2e += time.perf_counter() - t0
        assert len(recs) == G
        if world > 1:   # the slowest rank defines the end-to-end step too
            t_e2e = max_over_ranks(t_e2e, dev)
        line["e2e"] = {"value": world * G / (t_e2e / reps), "unit": UNIT,
                       "h2d_bytes_per_step": int(site_bytes + gates.nbytes),
                       "d2h_bytes_per_step": int(G * (48 + 160) + 512),
                       "pipeline": "%d chunks of %s updates, H2D of chunk c+1 on a side stream overlapping chunk c's update"
                                   % (C, [g1 - g0 for g0, g1 in bounds])}
        # the same step with the updated site tensors read back too (B_i', B_{i+1}' of every update),
        # after chunk c's update, mps_export_sites gathers its sites into a device
        # buffer (one launch) and their D2H into pinned host memory runs on a second side stream,
        # under chunk c+1's update (PCIe is full duplex: it also overlaps chunk c+2's H2D)
        try:
            dims_out = np.zeros((2 * G, 3), np.int32)
            ne = mps.mps_export_sites_raw(0, 2 * G, None, 0, dims_out)
            host_out = torch.empty(ne, dtype=torch.complex64, pin_memory=True)
            dev_out = torch.empty(ne, dtype=torch.complex64, device=dev)
            side2 = torch.cuda.Stream(device=dev)

            def e2e_full_step():
                evs, off = [], 0

                def issue(c):
                    g0, g1 = bounds[c]
                    ev = torch.cuda.Event()
                    with torch.cuda.stream(side):
                        stage[c % 2][: (g1 - g0) * per_el].copy_(host[g0 * per_el: g1 * per_el], non_blocking=True)
                        ev.record(side)
                    evs.append(ev)

                issue(0)
                for c in range(C):
                    if c + 1 < C:
                        issue(c + 1)
                    g0, g1 = bounds[c]
                    main.wait_event(evs[c])
                    mps.mps_import_sites_raw(2 * g0, 2 * (g1 - g0), pk.C.c_void_p(stage[c % 2].data_ptr()),
                                             dims[2 * g0: 2 * g1])
                    mps.mps_apply_layer(sites[g0:g1], gates[g0:g1])
                    # synchronous on the library's stream: the chunk's tensors are in dev_out on return
                    n = mps.mps_export_sites_raw(2 * g0, 2 * (g1 - g0), pk.C.c_void_p(dev_out.data_ptr() + 8 * off),
                                                 ne - off, dims_out[2 * g0: 2 * g1])
                    with torch.cuda.stream(side2):
                        host_out[off: off + n].copy_(dev_out[off: off + n], non_blocking=True)
                    off += n
                return mps.mps_truncation_array(last=G), off

            t_full = 0.0
            for rep in range(reps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                recs, got = e2e_full_step()
                torch.cuda.synchronize()
                if rep > 0:
                    t_full += time.perf_counter() - t0
            assert len(recs) == G and got == ne
            # the read-back is the device state, bit for bit (checked outside the timed region)
            chk = np.zeros((2, 3), np.int32)
            ref = torch.empty(int(dims_out[:2].prod(axis=1).sum()), dtype=torch.complex64, device=dev)
            mps.mps_export_sites_raw(0, 2, pk.C.c_void_p(ref.data_ptr()), ref.numel(), chk)
            assert torch.equal(torch.view_as_real(ref.cpu()), torch.view_as_real(host_out[: ref.numel()]))
            if world > 1:
                t_full = max_over_ranks(t_full, dev)
            line["e2e"]["with_state_readback"] = {
                "value": world * G / (t_full / reps), "unit": UNIT,
                "d2h_bytes_per_step": int(G * (48 + 160) + 512 + 8 * ne),
                "what": "records + every updated site tensor (mps_export_sites per chunk, D2H into pinned host "
                        "memory on a second side stream under the next chunk's update)"}
            del host_out, dev_out
        except Exception as e:   # the extra leg never blocks the line
            line["e2e"]["with_state_readback"] = {"error": str(e)[:300]}
        del stage
        del host
    del mps, inter
    torch.cuda.empty_cache()
    # ---- the rest of configs[1]: chi = 16 / 256 / 1024 sub-records (single GPU only), each with its
    # own stated step count (chi = 1024 on a 512-update subset of the 4096, in waves)
    if world == 1 and not args.no_per_chi and args.per_chi:
        line["per_chi"] = {}
        for spec in args.per_chi.split(","):
            c, cnt, st, wu = (int(x) for x in spec.split(":"))
            if c == chi:
                continue
            try:
                r, m2, i2, _, _ = run_chi(c, cnt, st, wu, rank, world, dev)
                if cnt < 4096:
                    r["subset"] = "%d of the 4096 updates (seeds 0..%d)" % (cnt, cnt - 1)
                line["per_chi"]["chi%d" % c] = r
                del m2, i2
            except Exception as e:   # a sub-record never blocks the headline line
                line["per_chi"]["chi%d" % c] = {"error": str(e)[:300]}
            torch.cuda.empty_cache()
    # ---- config 5 (the sharded north-star workload) on its first layers, at every N: the N-rank
    # sharded time; at N > 1 also rank 0 alone (T_1) for the parallel efficiency T_1 / (N T_N)
    if args.config5_depth > 0:
        try:
            c5 = run_config5_slice(args.config5_depth, rank, world, dev)
            if world > 1:
                dist.barrier()
                t1 = run_config5_slice(args.config5_depth, rank, world, dev, solo=True) if rank == 0 else None
                dist.barrier()
                if rank == 0:
                    c5["t1_seconds"] = t1["seconds"]
                    c5["parallel_efficiency"] = t1["seconds"] / (world * c5["seconds"])
            line["config5_slice"] = c5
        except Exception as e:
            line["config5_slice"] = {"error": str(e)[:300]}
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

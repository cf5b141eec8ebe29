#!/usr/bin/env python
"""bench.py -- SKP-PME reciprocal throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the full reciprocal pipeline (sort, spread, SKP grid
operator, gather, correction) over the workload's particle batch. Default
workload: config 3 (configs[2], 1,000,000 particles, 21^3 cells x L=6 ->
126^3 mesh, |Lambda| = 101), the first BASELINE config quoted at 1/2/4/8 GPUs
(see DESIGN.md §5 for why not configs[1]). Inputs are resident in HBM for
``value``; ``e2e`` goes through the public plan API with pinned host buffers.
Rank 0 prints ONE JSON line. N > 1 runs under torchrun with z-slabs (strong
scaling of the fixed workload).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SKP-PME reciprocal particles/s (FP64)"
UNIT = "particles/s"
FLUSH_BYTES = 256 << 20  # > 126 MB L2


def args_():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="cfg3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true")
    p.add_argument("--slab", action="store_true",
                   help="use the z-slab path (SlabPlan + NCCL core all-reduce) even on 1 GPU")
    p.add_argument("--rank-grid", default=None,
                   help="P0xP1xP2 device grid of cell blocks for N > 1 (default 1x1xN: z-slabs)")
    return p.parse_args()


# ---- environment ---------------------------------------------------------------

def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


class Clocks:
    """nvidia-smi sampler running across the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.file, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        self.file.seek(0)
        rows = [r.split(",") for r in self.file.read().strip().splitlines() if r.strip()]
        os.unlink(self.file.name)
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                power.append(float(r[3]))
            except ValueError:
                continue
            for name, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        busy = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ---- CPU reference / baseline ----------------------------------------------------
# Everything here goes through oracle/ only (test infrastructure, the CPU arm):
# inputs from the back end's own sample_cloud / sinc_rule_for_eps /
# skp_from_quadrature (oracle/workloads.py), never from the GPU library.

def cpu_runner():
    """oracle/_ref at the reference's Release flags (-O3 -DNDEBUG) when
    present, else the -O2 parity build, else the oracle port."""
    from oracle.binding import CpuKpme

    for which, kind, build in (("ref_o3", "reference", "oracle/_ref/libkpme_ref_o3.so "
                                "(reference headers, -O3 -DNDEBUG = CMake Release)"),
                               ("ref", "reference", "oracle/_ref/libkpme_ref.so "
                                "(reference headers, -O2 -ffp-contract=off)"),
                               ("oracle", "port", "oracle/build/libkpme_oracle.so (C port, -O2)")):
        try:
            return CpuKpme(which), kind, build
        except FileNotFoundError:
            continue
    raise FileNotFoundError("no CPU back end built (run __graft_entry__.build())")


def cpu_time(cpu, pb, nterms, threads):
    from dataclasses import replace

    sub = replace(pb, term_weights=pb.term_weights[:nterms], profiles=pb.profiles[:nterms])
    t0 = time.perf_counter()
    cpu.kpme_apply(sub, threads=threads)
    return time.perf_counter() - t0


def cpu_sampled(name, budget_s, threads, reps=1):
    """Bounded sample of the full workload: the reference's kpme_apply on the
    full particle set and cell grid with the first s SKP terms, plus one run
    with no terms. Its cost is exactly affine in the term count (one spkmv and
    one factor build per term, parallel.hpp:193-196, 265-279), so the full-
    |Lambda| time is t0 + |Lambda| (t_s - t0) / s."""
    from oracle import workloads

    cpu, kind, build = cpu_runner()
    pb = workloads.problem(name, cpu)
    n = len(pb.q)
    nt = len(pb.term_weights)
    t0 = cpu_time(cpu, pb, 0, threads)
    t1 = cpu_time(cpu, pb, 1, threads)
    per = max(t1 - t0, 1e-6)
    s = int(max(1, min(nt, (budget_s - t0) / per)))
    samples = []
    for _ in range(reps):
        ts = cpu_time(cpu, pb, s, threads)
        samples.append(t0 + nt * (ts - t0) / s)
    full = statistics.median(samples)
    sample = (f"{name}: full {n} particles and {list(pb.counts)} cells, first {s} of {nt} "
              f"SKP terms (+ one 0-term run, t0={t0:.2f}s); full-|Lambda| time extrapolated "
              f"affinely in the term count" if s < nt else f"{name}: full workload")
    return {"value": n / full, "unit": UNIT, "cores": threads, "kind": kind, "build": build,
            "sample": sample, "seconds_full_equiv": full,
            "inputs": "built by the same back end (oracle/workloads.py)"}, samples, pb


# ---- GPU helpers ------------------------------------------------------------------

def fp64_peak(torch, device):
    """cuBLAS DGEMM 8192^3 best of 5 (MEASURED_PEAKS.json has no FP64 entry)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def timed_steps(torch, fn, steps, flush):
    """Per-step CUDA-event times (ms) with an L2 flush before every step."""
    times = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    return times


def mesh_work(w, ms):
    """Mesh GFLOP/s (BASELINE's second metric) for the SKP operator as executed:
    the term-collapsed form, (W0 (x) W1 (x) W2) then G .* then the transposes,
    2 (2 R n^3 + 2 R^2 n^2 + 2 R^3 n) + R^3 flops with R = 2M+1,
    fused into the spread and gather kernels, so it is quoted per whole step.
    Beside it, the reference's per-term SPKMV flops 12 |Lambda| r_ax n^3
    (r_ax = 2(M+1), SURVEY.md §8(d) F form) over the same step time: the
    throughput the reference's formulation would need to match this step."""
    L, M = w.order, w.cfg.modes
    R, r_ax = 2 * M + 1, 2 * (M + 1)
    n = [k * L for k in w.grid.counts]
    n3 = float(n[0] * n[1] * n[2])
    collapsed = 2.0 * (2 * R * n3 + 2 * R * R * n[0] * n[1] + 2 * R ** 3 * n[0]) + R ** 3
    spkmv = 12.0 * len(w.dec.terms) * r_ax * n3
    return {"formulation": "collapsed (fused into spread/gather; per whole step)",
            "collapsed_flops": collapsed, "gflops": collapsed / (ms * 1e-3) / 1e9,
            "reference_spkmv_flops": spkmv,
            "reference_spkmv_equivalent_gflops": spkmv / (ms * 1e-3) / 1e9}


def spread_algorithmic(w, S):
    """Algorithmic work of the fused spread + forward-z kernel per launch
    (DESIGN.md §4): flops 2 L^3 N (accumulate) + 2 R L^3 per cell
    (contraction); bytes 32 N (sorted x,y,z,q) + 4 (ncell+1) (offsets) +
    8 S n0 n1 R (column partials written)."""
    L, R = w.order, 2 * w.cfg.modes + 1
    K = w.grid.counts
    n0, n1 = K[0] * L, K[1] * L
    ncell = K[0] * K[1] * K[2]
    flops = 2.0 * L ** 3 * w.n + 2.0 * R * L ** 3 * ncell
    bytes_ = 32.0 * w.n + 4.0 * (ncell + 1) + 8.0 * S * n0 * n1 * R
    return flops, bytes_


def gather_algorithmic(w):
    """backward-z + gather kernel: flops 2 L^3 N + 2 R L^3 ncell; bytes 32 N
    (sorted particles) + 4 N (perm) + 8 N (potentials) + 8 n0 n1 R (B2)."""
    L, R = w.order, 2 * w.cfg.modes + 1
    K = w.grid.counts
    ncell = K[0] * K[1] * K[2]
    flops = 2.0 * L ** 3 * w.n + 2.0 * R * L ** 3 * ncell
    bytes_ = 44.0 * w.n + 8.0 * K[0] * L * K[1] * L * R + 4.0 * (ncell + 1)
    return flops, bytes_


def ncu_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("kernels", {}).get(kernel_key, {}).get("dram_bytes")
    except (OSError, ValueError):
        return None


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    slab = world > 1 or a.slab
    if slab and not dist.is_initialized() and "RANK" in os.environ:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload(a.workload)
    peaks, peaks_src = load_peaks()
    flush = torch.empty(FLUSH_BYTES // 8, dtype=torch.float64, device=dev)

    if slab:
        from paper_2601_18838_b200.dist import SlabPlan

        dims = tuple(int(v) for v in a.rank_grid.split("x")) if a.rank_grid else None
        plan = SlabPlan(w, rank, world, device=local, dims=dims)
        step, e2e_step, launches, meta = plan.bench_callables()
    else:
        plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, device=local)
        xyz = torch.as_tensor(w.data.cloud.positions, device=dev).contiguous()
        q = torch.as_tensor(w.data.charges.values, device=dev).contiguous()
        out = torch.empty(w.n, dtype=torch.float64, device=dev)
        plan.execute(xyz, q, out)  # validates inputs (synchronous checks)
        plan.execute_graph(xyz, q, out)
        launches = plan.launches()

        def step():
            plan.execute_graph(xyz, q, out)

        xyz_h = torch.as_tensor(w.data.cloud.positions).contiguous().pin_memory()
        q_h = torch.as_tensor(w.data.charges.values).contiguous().pin_memory()
        out_h = torch.empty(w.n, dtype=torch.float64).pin_memory()

        def e2e_step():
            plan.execute_host_ptr(w.n, xyz_h.data_ptr(), q_h.data_ptr(), out_h.data_ptr())

        meta = {}

    clocks = Clocks(local)
    clocks.start()
    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    times = timed_steps(torch, step, a.steps, flush)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    clk = clocks.stop()
    ms = sum(times) / len(times)
    if dist.is_initialized():
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if not slab:
        plan.status()  # deferred argument checks of the timed region

    # e2e through the public API with host buffers
    for _ in range(2):
        e2e_step()
    e2e_times = timed_steps(torch, e2e_step, a.steps, flush)
    e2e_ms = sum(e2e_times) / len(e2e_times)
    e2e_sorted = sorted(e2e_times)
    e2e_spread = {"min": e2e_sorted[0], "median": e2e_sorted[len(e2e_sorted) // 2], "max": e2e_sorted[-1]}
    if dist.is_initialized():
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # per-stage times (eager, timing events) -> dominant kernel roofline
    roofline, stages = None, None
    if not slab:
        plan.enable_timing(True)
        acc = None
        for _ in range(max(3, min(a.steps, 10))):
            flush.zero_()
            plan.execute(xyz, q, out, defer_checks=True)
            st = plan.stage_times()
            acc = st if acc is None else [x + y for x, y in zip(acc, st)]
        cnt = max(3, min(a.steps, 10))
        plan.enable_timing(False)
        st = [x / cnt for x in acc]
        stages = {"sort_permute_ms": st[0], "spread_fwd_ms": st[1], "core_ms": st[2],
                  "bwd_gather_ms": st[3]}
        S = max(1, min(w.grid.counts[2], (3 * 148) // (w.grid.counts[0] * w.grid.counts[1])))
        fp64 = fp64_peak(torch, dev)
        cand = {"k_spread_fwd": (st[1], spread_algorithmic(w, S)),
                "k_bwd_gather": (st[3], gather_algorithmic(w))}
        name = max(cand, key=lambda k: cand[k][0])
        t_ms, (flops, bytes_) = cand[name]
        t_hbm = bytes_ / (peaks["hbm_gbs"] * 1e9)
        t_fp64 = flops / (fp64 * 1e12)
        if t_fp64 >= t_hbm:
            achieved = flops / (t_ms * 1e-3) / 1e12
            roofline = {"bound": "fp64", "kernel": name, "achieved": achieved, "peak": fp64,
                        "unit": "TFLOP/s", "frac": achieved / fp64,
                        "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (the DMMA "
                                       "tensor subpipe, 64 FP64 FMA/clk/SM; the spread's "
                                       "GEMM-shaped work runs there)",
                        "hbm_frac": bytes_ / (t_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        else:
            achieved = bytes_ / (t_ms * 1e-3) / 1e9
            roofline = {"bound": "hbm", "kernel": name, "achieved": achieved,
                        "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": achieved / peaks["hbm_gbs"],
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_src})"}
        roofline.update({"algorithmic_flops": flops, "algorithmic_bytes": bytes_,
                         "kernel_ms": t_ms, "traffic": ncu_traffic(name)})
        meta["fp64_dgemm_tflops"] = fp64

    if rank != 0:
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return

    value = w.n / (ms * 1e-3)
    mesh = mesh_work(w, ms)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if slab else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 sample_cloud, BASELINE.json config shapes)",
        "config": w.describe(),
        "impl_config": {"formulation": "collapsed (term-collapsed SKP core, per-shape chooser)",
                        "parallelism": (f"rank grid {'x'.join(map(str, plan.dims))} of cell "
                                        f"blocks (NCCL core all-reduce)") if slab else "1 GPU",
                        "l2": "flushed (256 MiB write) before every timed step"},
        "e2e": {"value": w.n / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "ms_per_step_spread": e2e_spread,
                "h2d_bytes_per_step": 32 * w.n, "d2h_bytes_per_step": 8 * w.n,
                "path": ("SlabPlan.e2e_step: pinned H2D of the slab's particles, forward, "
                         "NCCL core all-reduce, backward, D2H" if slab else
                         "KpmePlan.execute_host_ptr -> kpme_gpu_plan_execute (pinned host "
                         "xyz/q in, potentials out)")},
        "mesh": mesh,
        "gpu_launches": launches * a.steps,
        "clocks": clk,
        "roofline": roofline,
        "stages": stages,
        **meta,
    }
    if world == 1 and not slab and not a.no_cpu_baseline:
        cb, _, _ = cpu_sampled(a.workload, 20.0, os.cpu_count() or 1)
        cb["cpu"] = cpu_info()
        line["cpu_baseline"] = cb
    if world == 1 and not slab and not a.no_extras:
        line["extras"] = extras(torch, dev, flush, a.steps)
    emit(line)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def extras(torch, dev, flush, steps):
    """Other BASELINE configs on one GPU (same timing rules), and one config-5
    dense-operator point on DMMA."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan, dense_workspace_bytes, kron_matvec_dense

    out = {}
    for name in ("cfg1", "cfg2", "cfg4"):
        w = inputs.workload(name)
        plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, device=dev.index)
        xyz = torch.as_tensor(w.data.cloud.positions, device=dev).contiguous()
        q = torch.as_tensor(w.data.charges.values, device=dev).contiguous()
        o = torch.empty(w.n, dtype=torch.float64, device=dev)
        plan.execute(xyz, q, o)
        for _ in range(3):
            plan.execute_graph(xyz, q, o)
        t = timed_steps(torch, lambda: plan.execute_graph(xyz, q, o), steps, flush)
        ms = sum(t) / len(t)
        out[name] = {"particles_per_s": w.n / (ms * 1e-3), "ms_per_step": ms, **w.describe()}
        plan.close()
    n, R = 256, 16
    cfg, grid, L, dec = inputs.dense_case(n, R)
    plan = KpmePlan(cfg, grid, L, dec, 1, device=dev.index)
    ops = [plan.axis_operands(a_) for a_ in range(3)]
    x = torch.randn(n, n, n, dtype=torch.float64, device=dev,
                    generator=torch.Generator(device=dev).manual_seed(0))
    ws = torch.empty(dense_workspace_bytes(n, n, n, R) // 8 + 1, dtype=torch.float64, device=dev)
    y = kron_matvec_dense(*ops, x, workspace=ws)
    t = timed_steps(torch, lambda: kron_matvec_dense(*ops, x, out=y, workspace=ws), 3, flush)
    ms = sum(t) / len(t)
    flops = 6.0 * R * n ** 4
    out["cfg5_dense_256_R16"] = {"mesh_gflops": flops / (ms * 1e-3) / 1e9, "ms": ms,
                                 "flops_formula": "6 R n^4 (op_count_estimate x2, kron.hpp:201-211)"}
    return out


def run_reference(a):
    """The reference's own CPU implementation (oracle/_ref at Release flags;
    else the oracle port) with every host thread, on bounded samples of the
    same workload. Never imports the GPU package: inputs come from the same
    back end (oracle/workloads.py)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import workloads

    threads = os.cpu_count() or 1
    budget = max(3.0, min(20.0, 200.0 / max(1, a.steps + a.warmup)))
    cb, samples, pb = cpu_sampled(a.workload, budget, threads, reps=a.steps + a.warmup)
    timed = samples[a.warmup:] or samples
    full = statistics.median(timed)
    value = len(pb.q) / full
    cb["value"] = value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": full * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded splitmix64 sample_cloud, BASELINE.json config shapes)",
            "config": workloads.describe(a.workload, len(pb.term_weights)),
            "impl_config": {"parallelism": f"CPU, {threads} threads", "build": cb["build"]},
            "impl": "reference", "cpu_baseline": {**cb, "cpu": cpu_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


_JSON_OUT = None


def emit(line: dict):
    """The one JSON line, on the real stdout (library banners such as NCCL's
    version line are routed to stderr for the whole run)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = args_()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()

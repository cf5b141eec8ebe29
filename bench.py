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
    p.add_argument("--cfg5-meshes", default=None, help="cfg5: comma list of n (default 64..512)")
    p.add_argument("--cfg5-ranks", default=None, help="cfg5: comma list of R (default 4..64)")
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


class L2Flush:
    """L2 flush between timed steps: a 256 MiB write (the whole L2 becomes lines of
    the flush buffer), then a read of a second 256 MiB buffer, so those lines are
    written back and L2 ends holding clean lines of neither input. Without the read
    the step's first kernels also pay the write-back of the flush's dirty lines."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.w = torch.empty(FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
        self.r = torch.zeros(FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
        self.read_back = os.environ.get("KPME_BENCH_FLUSH_READ", "1") != "0"

    def zero_(self):
        self.w.zero_()
        if self.read_back:
            self.sink = self.r.sum()

    def describe(self):
        return ("flushed before every timed step: 256 MiB written" +
                (", then a second 256 MiB buffer read (write-back of the flush's dirty lines "
                 "is outside the step)" if self.read_back else ""))


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
    The reference's per-term SPKMV flop count 12 |Lambda| r_ax n^3 (r_ax =
    2(M+1), SURVEY.md §8(d) F form) is listed as a count only: it is work the
    collapsed form does not do, not a throughput."""
    L, M = w.order, w.cfg.modes
    R, r_ax = 2 * M + 1, 2 * (M + 1)
    n = [k * L for k in w.grid.counts]
    n3 = float(n[0] * n[1] * n[2])
    collapsed = 2.0 * (2 * R * n3 + 2 * R * R * n[0] * n[1] + 2 * R ** 3 * n[0]) + R ** 3
    spkmv = 12.0 * len(w.dec.terms) * r_ax * n3
    return {"formulation": "collapsed (fused into spread/gather; per whole step)",
            "collapsed_flops": collapsed, "gflops": collapsed / (ms * 1e-3) / 1e9,
            "reference_spkmv_flops_not_executed": spkmv}


def local_shape(w, block=None):
    """Cells per axis of the plan's block (the whole grid for one plan)."""
    K = list(w.grid.counts)
    if block is not None:
        K = [hi - lo for lo, hi in block]
    return K


def sort_algorithmic(n):
    """Cell sort + permute (geometry.hpp:131-154): compulsory HBM traffic is
    the particles read once (x, y, z, q: 32 B) and the cell-ordered records
    plus the permutation written once (32 + 4 B); the cell offsets are
    negligible. Counting passes are the implementation's, not algorithmic."""
    return 0.0, 68.0 * n


def spread_algorithmic(w, n, K, S):
    """Algorithmic work of the fused spread + forward-z kernel per launch
    (DESIGN.md §4): flops 2 L^3 N (accumulate) + 2 R L^3 per cell
    (contraction); bytes 32 N (sorted x,y,z,q) + 4 (ncell+1) (offsets) +
    8 S K0 K1 (R^3 + 1) (per-column partial cores written)."""
    L, R = w.order, 2 * w.cfg.modes + 1
    ncell = K[0] * K[1] * K[2]
    flops = 2.0 * L ** 3 * n + 2.0 * R * L ** 3 * ncell
    bytes_ = 32.0 * n + 4.0 * (ncell + 1) + 8.0 * S * K[0] * K[1] * (R ** 3 + 1)
    return flops, bytes_


def gather_algorithmic(w, n, K):
    """backward-z + gather kernel: flops 2 L^3 N + 2 R L^3 ncell; bytes 32 N
    (sorted particles) + 4 N (perm) + 8 N (potentials) + 8 n0 n1 R (B2)."""
    L, R = w.order, 2 * w.cfg.modes + 1
    ncell = K[0] * K[1] * K[2]
    flops = 2.0 * L ** 3 * n + 2.0 * R * L ** 3 * ncell
    bytes_ = 44.0 * n + 8.0 * K[0] * L * K[1] * L * R + 4.0 * (ncell + 1)
    return flops, bytes_


def ncu_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary
    (profiles/ncu_summary.json, captured from this bench's workload)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        k = d.get("kernels", {})
        if kernel_key == "k_sort_stage":  # the stage's two kernels (key path)
            parts = [k.get(n, {}).get("dram_bytes") for n in ("k_tile_keys", "k_z_tiles_ko")]
            return sum(parts) if all(p is not None for p in parts) else None
        return k.get(kernel_key, {}).get("dram_bytes")
    except (OSError, ValueError):
        return None


def stage_rooflines(torch, plan, run_eager, w, n, K, flush, steps, peaks, fp64):
    """Per-stage device times (the plan's own CUDA events on its stream,
    averaged over eager steps with an L2 flush before each) and each stage's
    roofline: the sort against HBM, the spread and gather against
    max(HBM, FP64)."""
    plan.enable_timing(True)
    acc, cnt = None, max(3, min(steps, 10))
    for _ in range(cnt):
        flush.zero_()
        run_eager()
        st = plan.stage_times()
        acc = st if acc is None else [x + y for x, y in zip(acc, st)]
    plan.enable_timing(False)
    st = [x / cnt for x in acc]
    stages = {"sort_permute_ms": st[0], "spread_fwd_ms": st[1], "core_ms": st[2],
              "bwd_gather_ms": st[3]}
    S = max(1, min(K[2], (3 * 148) // max(1, K[0] * K[1])))
    hbm = peaks["hbm_gbs"]
    out = {}
    for name, t_ms, (flops, bytes_) in (("k_sort_stage", st[0], sort_algorithmic(n)),
                                       ("k_spread_fwd", st[1], spread_algorithmic(w, n, K, S)),
                                       ("k_bwd_gather", st[3], gather_algorithmic(w, n, K))):
        t_hbm = bytes_ / (hbm * 1e9)
        t_fp = flops / (fp64 * 1e12) if flops else 0.0
        if t_fp >= t_hbm:
            ach = flops / (t_ms * 1e-3) / 1e12
            r = {"bound": "fp64", "achieved": ach, "peak": fp64, "unit": "TFLOP/s",
                 "frac": ach / fp64,
                 "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (the DMMA tensor "
                                "subpipe; MEASURED_PEAKS.json has no FP64 entry)",
                 "hbm_frac": bytes_ / (t_ms * 1e-3) / 1e9 / hbm}
        else:
            ach = bytes_ / (t_ms * 1e-3) / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        if name == "k_sort_stage":
            r["kernels"] = "k_tile_keys + k_z_tiles_ko (key path, <= 512 columns) or k_tile_hist + k_col_scan + k_col_scatter + k_z_sort"
        r.update({"kernel": name, "algorithmic_flops": flops, "algorithmic_bytes": bytes_,
                  "kernel_ms": t_ms, "traffic": ncu_traffic(name),
                  "traffic_source": "profiles/ncu_summary.json (ncu --set full of this workload)"})
        out[name] = r
    return stages, out


def run_ours(a):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if torch.cuda.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    slab = world > 1 or a.slab
    if (slab or (a.workload == "cfg5" and world > 1)) and not dist.is_initialized() and "RANK" in os.environ:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan

    if a.workload == "cfg5":
        return run_cfg5(a, torch, dist, rank, world, dev)
    w = inputs.workload(a.workload)
    peaks, peaks_src = load_peaks()
    flush = L2Flush(torch, dev)

    if slab:
        from paper_2601_18838_b200.dist import SlabPlan

        dims = tuple(int(v) for v in a.rank_grid.split("x")) if a.rank_grid else None
        sp = SlabPlan(w, rank, world, device=local, dims=dims)
        step, e2e_step, launches, meta = sp.bench_callables()
        plan, n_local, K_local = sp.plan, sp.n, local_shape(w, sp.block)
        xyz, q, out = sp.xyz, sp.q, sp.out
    else:
        plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, device=local)
        xyz = torch.as_tensor(w.data.cloud.positions, device=dev).contiguous()
        q = torch.as_tensor(w.data.charges.values, device=dev).contiguous()
        out = torch.empty(w.n, dtype=torch.float64, device=dev)
        plan.execute(xyz, q, out)  # validates inputs (synchronous checks)
        plan.execute_graph(xyz, q, out)
        launches = plan.launches()
        n_local, K_local = w.n, local_shape(w)

        def step():
            plan.execute_graph(xyz, q, out)

        xyz_h = torch.as_tensor(w.data.cloud.positions).contiguous().pin_memory()
        q_h = torch.as_tensor(w.data.charges.values).contiguous().pin_memory()
        out_h = torch.empty(w.n, dtype=torch.float64).pin_memory()

        def e2e_step():
            plan.execute_host_ptr(w.n, xyz_h.data_ptr(), q_h.data_ptr(), out_h.data_ptr())

        meta = {}

    def run_eager():
        plan.execute(xyz, q, out, defer_checks=True)

    clocks = Clocks(local)
    clocks.start()
    for _ in range(max(a.warmup, 3)):  # the warm-up steps run the timed loop's pattern: flush, then step
        flush.zero_()
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
    plan.status()  # deferred argument checks of the timed region

    # e2e through the public API with host buffers
    for _ in range(2):
        e2e_step()
    e2e_times = timed_steps(torch, e2e_step, a.steps, flush)
    e2e_ms = sum(e2e_times) / len(e2e_times)
    e2e_sorted = sorted(e2e_times)
    e2e_spread = {"min": e2e_sorted[0], "median": e2e_sorted[len(e2e_sorted) // 2],
                  "max": e2e_sorted[-1]}
    if dist.is_initialized():
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # per-stage times (eager, the plan's timing events) -> rooflines
    fp64 = fp64_peak(torch, dev)
    stages, rooflines = stage_rooflines(torch, plan, run_eager, w, n_local, K_local, flush,
                                        a.steps, peaks, fp64)
    # the dominant single kernel (the sort stage is two kernels; its stage
    # roofline is reported beside it in `rooflines`)
    dom = max(("k_spread_fwd", "k_bwd_gather"), key=lambda k: rooflines[k]["kernel_ms"])
    roofline = rooflines[dom]
    meta["fp64_dgemm_tflops"] = fp64

    if rank != 0:
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return

    value = w.n / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if slab else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 sample_cloud, BASELINE.json config shapes)",
        "config": w.describe(),
        "impl_config": {"formulation": "collapsed (term-collapsed SKP core, per-shape chooser)",
                        "parallelism": (f"rank grid {'x'.join(map(str, sp.dims))} of cell "
                                        f"blocks, one process per GPU, plan-owned NCCL core "
                                        f"all-reduce") if slab else "1 GPU",
                        "l2": flush.describe(),
                        "timing": "CUDA events per step, max over ranks"},
        "e2e": {"value": w.n / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "ms_per_step_spread": e2e_spread,
                "h2d_bytes_per_step": 32 * w.n, "d2h_bytes_per_step": 8 * w.n,
                "path": "kpme_gpu_plan_execute (pinned host xyz/q in, potentials out)" +
                        ("; per rank: its cell block's particles, NCCL core all-reduce inside"
                         if slab else "")},
        "mesh": mesh_work(w, ms),
        "gpu_launches": launches * a.steps,
        "clocks": clk,
        "roofline": roofline,
        "rooflines": rooflines,
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


def oneshot_e2e(w, reps=5):
    """kpme_apply through the one-shot drop-in (kpme_gpu_apply: cached plan,
    pageable numpy buffers, H2D / D2H inside): host wall clock around the
    synchronous call, first (cold: plan build) and steady-state."""
    import paper_2601_18838_b200 as kp

    kp._lib.lib.kpme_gpu_apply_cache_clear()
    t0 = time.perf_counter()
    kp.kpme_apply(w.cfg, w.grid, w.order, w.dec, w.data.cloud, w.data.charges)
    cold = time.perf_counter() - t0
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        kp.kpme_apply(w.cfg, w.grid, w.order, w.dec, w.data.cloud, w.data.charges)
        ts.append(time.perf_counter() - t0)
    kp._lib.lib.kpme_gpu_apply_cache_clear()
    med = statistics.median(ts)
    return {"value": w.n / med, "unit": UNIT, "ms_per_call": med * 1e3,
            "first_call_ms": cold * 1e3,
            "path": "kpme_apply -> kpme_gpu_apply (plan cache), pageable numpy in/out, host "
                    "wall clock around the synchronous call"}


def extras(torch, dev, flush, steps):
    """Other BASELINE configs on one GPU (same timing rules), the one-shot
    drop-in latency, and one config-5 dense-operator point on DMMA."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan, dense_workspace_bytes, kron_matvec_dense

    out = {"e2e_oneshot_cfg3": oneshot_e2e(inputs.workload("cfg3"))}
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


def run_cfg5(a, torch, dist, rank, world, dev):
    """Config 5: the dense SKP grid operator on z-slabs, every mesh and rank
    of BASELINE (64^3..512^3, R in {4..64}), through the library's slab
    operator (kpme_gpu_dense_slab: DMMA GEMMs, plan-owned NCCL communicator,
    preallocated buffers). All three sharded-axis strategies are timed per
    shape by the library's chooser (CUDA events, max over ranks) and the
    fastest is kept -- the north star's slab all-to-all vs rank split +
    reduce, plus the reference's own SPKMV-style reduction
    (parallel.hpp:169-176). Prints the table on stderr and one JSON line."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.dist import slab_bounds
    from paper_2601_18838_b200.plan import DenseSlab, KpmePlan, nccl_unique_id

    meshes = [int(v) for v in (a.cfg5_meshes or "64,128,256,512").split(",")]
    ranks = [int(v) for v in (a.cfg5_ranks or "4,8,16,32,64").split(",")]
    fp64 = fp64_peak(torch, dev)
    rows = []
    for n in meshes:
        cfg, grid, L, dec = inputs.dense_case(n, max(ranks))
        plan = KpmePlan(cfg, grid, L, dec, 1, device=dev.index)
        ops_all = [plan.axis_operands(ax) for ax in range(3)]
        plan.close()
        lo, hi = slab_bounds(n, rank, world)
        g = torch.Generator(device=dev).manual_seed(n)
        x_full = torch.randn(n, n, n, dtype=torch.float64, device=dev, generator=g)
        x_local = x_full[:, :, lo:hi].contiguous()
        y_local = torch.empty_like(x_local)
        del x_full
        for R in ranks:
            ops = [o[:R].contiguous() for o in ops_all]
            uid = None
            if world > 1:
                box = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(box, src=0)
                uid = box[0]
            op = DenseSlab(*ops, nranks=world, rank=rank, nccl_id=uid)
            tms, best = op.choose(x_local, y_local, reps=3 if n <= 256 else 1)
            op.close()
            flops = 6.0 * R * n ** 4
            rows.append({"n": n, "R": R, "ms": tms, "chosen": best,
                         "mesh_gflops": flops / (tms[best] * 1e-3) / 1e9,
                         "frac_of_fp64": flops / (tms[best] * 1e-3) / 1e12 / fp64})
            if rank == 0:
                sys.stderr.write(f"cfg5 n={n:4d} R={R:3d} " + " ".join(
                    f"{k}={v:9.3f}ms" for k, v in tms.items()) + f"  -> {best}\n")
            del op, ops
        del ops_all, x_local, y_local
        torch.cuda.empty_cache()
    if rank == 0:
        head = max(rows, key=lambda r: (r["n"], r["R"]))
        line = {"metric": "SKP grid operator mesh GFLOP/s (FP64, dense factors)",
                "value": head["mesh_gflops"], "unit": "GFLOP/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": head["ms"][head["chosen"]],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (N(0,1) mesh, factors from the SKP "
                                         "construction, BASELINE config 5)",
                "config": {"workload": "cfg5", "mesh": [head["n"]] * 3, "skp_terms": head["R"]},
                "impl_config": {"path": "kpme_gpu_dense_slab (library: DMMA GEMMs, NCCL "
                                        "collectives, chooser)",
                                "timing": "library CUDA events per apply, max over ranks; "
                                          "L2 not flushed between reps (meshes >= 256^3 "
                                          "exceed L2)"},
                "strategies": rows, "fp64_dgemm_tflops": fp64,
                "flops_formula": "6 R n^4 (op_count_estimate x2, kron.hpp:201-211)"}
        emit(line)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


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


def launch_ranks(a):
    """``--gpus N`` without a launcher: re-exec this command under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous). Under a
    launcher the world size must equal N; a mismatch or too few GPUs fails
    loudly instead of measuring another N."""
    if "RANK" in os.environ:
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world != a.gpus:
            sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}\n")
            raise SystemExit(2)
        return
    if a.gpus <= 1 or a.impl == "reference":
        return
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < a.gpus:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} needs {a.gpus} GPUs, this box has {have}\n")
        raise SystemExit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def main():
    global _JSON_OUT
    a = args_()
    if a.gpus < 1:
        sys.stderr.write("bench.py: --gpus must be >= 1\n")
        raise SystemExit(2)
    launch_ranks(a)
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()

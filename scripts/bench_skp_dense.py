"""Config 5: SKP grid-operator-only sweep on one GPU (BASELINE.json configs[4]).

Random N(0,1) meshes of n^3 (n = 64..512), R in {4, 8, 16, 32, 64} terms of
sinc_rule_for_eps(1e-8, 4), dense n x n factors A_r = B_r = C_r = A(lambda_r)
built from the SKP construction for a unit box (K = n/8 cells, L = 8).
Reports mesh GFLOP/s with the reference's multiply count x 2 (6 R n^4,
op_count_estimate, kron.hpp:201-211) and the fraction of the measured cuBLAS
DGEMM peak. The operator is captured once into a CUDA graph and replayed
(steady state, no host launch gaps; --eager times the ctypes call instead);
the L2 is flushed (256 MiB write) before every timed replay. Prints one JSON
object.

    python scripts/bench_skp_dense.py [--sizes 64,128,256,512] [--ranks 4,8,16,32,64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan, dense_workspace_bytes, kron_matvec_dense  # noqa: E402


def fp64_peak(dev):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = a @ b
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256,512")
    ap.add_argument("--ranks", default="4,8,16,32,64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--eager", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peak = fp64_peak(dev)
    flush = torch.empty(256 << 17, dtype=torch.float64, device=dev)
    rows = []
    for n in map(int, a.sizes.split(",")):
        for R in map(int, a.ranks.split(",")):
            cfg, grid, L, dec = inputs.dense_case(n, R)
            plan = KpmePlan(cfg, grid, L, dec, 1)
            ops = [plan.axis_operands(ax) for ax in range(3)]
            x = torch.randn(n, n, n, dtype=torch.float64, device=dev,
                            generator=torch.Generator(device=dev).manual_seed(0))
            ws = torch.empty(dense_workspace_bytes(n, n, n, R) // 8 + 1, dtype=torch.float64,
                             device=dev)
            y = kron_matvec_dense(*ops, x, workspace=ws)
            torch.cuda.synchronize()
            run = lambda: kron_matvec_dense(*ops, x, out=y, workspace=ws)  # noqa: E731
            if not a.eager:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    run()
                run = g.replay
                run()
                torch.cuda.synchronize()
            times = []
            for _ in range(a.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = min(times)
            flops = 6.0 * R * n ** 4
            rows.append({"n": n, "R": R, "ms": ms, "timing": "eager" if a.eager else "graph replay", "mesh_gflops": flops / (ms * 1e-3) / 1e9,
                         "frac_of_dgemm": flops / (ms * 1e-3) / 1e12 / peak})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del plan, ops, x, ws, y, run
            if not a.eager:
                del g
            torch.cuda.empty_cache()
    print(json.dumps({"fp64_dgemm_tflops": peak, "flops_formula": "6 R n^4", "rows": rows}))


if __name__ == "__main__":
    main()

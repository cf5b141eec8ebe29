"""Sweep the chunk count of the pipelined host path (kpme_gpu_plan_execute
with pinned host buffers): e2e ms per step, L2 flushed before each step.

usage: python scripts/e2e_chunks.py [cfg3] [steps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = inputs.workload(name)
plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
xyz_h = torch.as_tensor(w.data.cloud.positions).contiguous().pin_memory()
q_h = torch.as_tensor(w.data.charges.values).contiguous().pin_memory()
out_h = torch.empty(w.n, dtype=torch.float64).pin_memory()
flush = torch.empty(256 << 17, dtype=torch.float64, device="cuda")


def run():
    plan.execute_host_ptr(w.n, xyz_h.data_ptr(), q_h.data_ptr(), out_h.data_ptr())


# raw copy rates for reference
dx = torch.empty_like(xyz_h, device="cuda")
do = torch.empty_like(out_h, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
rates = {}
for tag, fn, nbytes in [("h2d_xyz", lambda: dx.copy_(xyz_h, non_blocking=True), 24 * w.n),
                        ("d2h_out", lambda: out_h.copy_(do, non_blocking=True), 8 * w.n)]:
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    rates[tag] = {"ms": best, "GB/s": nbytes / best / 1e6}

res = {"workload": name, "copy_rates": rates, "chunks": {}}
ref = None
for c in [1, 2, 3, 4, 5, 6, 8]:
    plan.set_host_chunks(c)
    for _ in range(3):
        run()
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    z = out_h.clone()
    if ref is None:
        ref = z
    err = float(torch.linalg.norm(z - ref) / torch.linalg.norm(ref))
    res["chunks"][c] = {"median_ms": ts[len(ts) // 2], "best_ms": ts[0], "rel_vs_1": err}
print(json.dumps(res, indent=1))

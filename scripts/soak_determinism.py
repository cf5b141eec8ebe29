"""Soak: replay the captured pipeline many times on each workload and check that
every output equals the first bit for bit (the launch chain is programmatic:
a race between kernels would show up as a changed bit sooner or later).
usage: python scripts/soak_determinism.py [reps] [cfg1 cfg2 cfg3 ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_18838_b200 import inputs
from paper_2601_18838_b200.plan import KpmePlan
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
names = sys.argv[2:] or ["cfg1", "cfg2", "cfg3"]
bad = 0
for name in names:
    w = inputs.workload(name)
    plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
    xyz = torch.as_tensor(w.data.cloud.positions, device="cuda").contiguous()
    q = torch.as_tensor(w.data.charges.values, device="cuda").contiguous()
    o = torch.empty(w.n, dtype=torch.float64, device="cuda")
    plan.execute(xyz, q, o)
    ref = o.clone()
    flush = torch.empty(64 << 17, dtype=torch.float64, device="cuda")
    diff = 0
    for r in range(reps):
        if r % 7 == 0:
            flush.zero_()  # vary the cache state and the timing between replays
        o.zero_()
        plan.execute_graph(xyz, q, o)
        if r % 50 == 49 or r == reps - 1:
            diff += int((o != ref).sum().item())
    torch.cuda.synchronize()
    print(f"{name}: {reps} graph replays, mismatching values in the checked replays: {diff}")
    bad += diff
    # the pipelined host path (chunked: several sorts / spreads / gathers chained per call)
    if w.n <= 1_000_000:
        import numpy as np
        for chunks in (1, 3, 8):
            plan.set_host_chunks(chunks)
            href = plan.execute_host(w.data.cloud.positions, w.data.charges.values)
            hd = 0
            for r in range(max(1, reps // 20)):
                hd += int((plan.execute_host(w.data.cloud.positions, w.data.charges.values) != href).sum())
            print(f"{name}: host path, {chunks} chunk(s), {max(1, reps // 20)} calls, mismatching values: {hd}")
            bad += hd
sys.exit(1 if bad else 0)

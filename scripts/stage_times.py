"""Eager per-stage device times (us: sort, spread, core, gather) of the pipeline,
mean of 10 runs with an L2 flush before each.  usage: python scripts/stage_times.py cfg3 cfg4"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_18838_b200 import inputs
from paper_2601_18838_b200.plan import KpmePlan
res = {}
for name in sys.argv[1:]:
    w = inputs.workload(name)
    plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
    xyz = torch.as_tensor(w.data.cloud.positions, device='cuda').contiguous()
    q = torch.as_tensor(w.data.charges.values, device='cuda').contiguous()
    o = torch.empty(w.n, dtype=torch.float64, device='cuda')
    plan.execute(xyz, q, o, defer_checks=bool(os.environ.get("PROFILE_NOCHECK")))
    plan.enable_timing(True)
    flush = torch.empty(256 << 17, dtype=torch.float64, device='cuda')
    flush_r = torch.zeros(256 << 17, dtype=torch.float64, device='cuda')  # read after the write: L2 ends clean (bench.py L2Flush)
    acc = None
    for _ in range(10):
        flush.zero_()
        if os.environ.get("KPME_BENCH_FLUSH_READ", "1") != "0":
            sink = flush_r.sum()
        plan.execute(xyz, q, o, defer_checks=True)
        st = plan.stage_times()
        acc = st if acc is None else [a + b for a, b in zip(acc, st)]
    res[name] = [round(x / 10 * 1e3, 1) for x in acc]
print(json.dumps(res))

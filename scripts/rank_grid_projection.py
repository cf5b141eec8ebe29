"""Per-rank step time of the decomposed pipeline, every rank of a rank grid
run one after another on the one GPU (no rank waits on another; the core
exchange is left out, so add the NCCL all-reduce latency of 730 doubles).
The slowest rank bounds the G-GPU step: a projection of strong scaling for
rank-grid shapes.  usage: python scripts/rank_grid_projection.py cfg3 1x1x8 8x1x1 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.dist import rank_grid_block, route_particles_grid  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

name = sys.argv[1]
w = inputs.workload(name)
flush = torch.empty(256 << 17, dtype=torch.float64, device="cuda")
res = {}
for spec in sys.argv[2:]:
    dims = tuple(int(v) for v in spec.split("x"))
    G = int(np.prod(dims))
    routes = route_particles_grid(w.data.cloud.positions, w.grid, dims)
    per = []
    for r in range(G):
        idx = routes[r]
        p = KpmePlan(w.cfg, w.grid, w.order, w.dec, max(1, len(idx)),
                     block=rank_grid_block(w.grid.counts, dims, r))
        x = torch.as_tensor(w.data.cloud.positions[idx], device="cuda").contiguous()
        q = torch.as_tensor(w.data.charges.values[idx], device="cuda").contiguous()
        o = torch.empty(len(idx), dtype=torch.float64, device="cuda")
        p.execute(x, q, o)
        for _ in range(3):
            p.execute_graph(x, q, o)
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(p.stream)
            p.execute_graph(x, q, o, sync_caller=False)
            e1.record(p.stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        per.append(sum(ts) / len(ts))
        p.close()
    res[spec] = {"max_rank_ms": max(per), "min_rank_ms": min(per), "ranks": G}
    print(spec, json.dumps(res[spec]), flush=True)
print(json.dumps(res))

"""Config 5 strong-scaling projection on one GPU: the dense slab operator
with W ranks held by one process on the same device (kpme_gpu_dense_slab
group: the ranks' kernels run one after another, the collectives become
local copies). Per-rank compute = group time / W; the G-GPU step adds the
collective over NVLink, estimated from its bytes at a stated bandwidth.
usage: python scripts/dense_slab_projection.py N R W1,W2,..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import DenseSlab, KpmePlan  # noqa: E402

n, R = int(sys.argv[1]), int(sys.argv[2])
Ws = [int(v) for v in sys.argv[3].split(",")]
cfg, grid, L, dec = inputs.dense_case(n, R)
plan = KpmePlan(cfg, grid, L, dec, 1)
ops = [plan.axis_operands(a).contiguous() for a in range(3)]
plan.close()
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
out = {}
for W in Ws:
    op = DenseSlab.group([tuple(ops)] * W, [0] * W)
    b = [op.bounds(r) for r in range(W)]
    xs = [x[:, :, lo:hi].contiguous() for lo, hi in b]
    ys = [torch.empty_like(t) for t in xs]
    ms, best = op.choose(xs, ys, reps=2)
    flops = 6.0 * R * n ** 4
    # reduce-scatter of the slab-major partial sums: each rank sends (W-1)/W of n^3 doubles
    rs_bytes = 8.0 * n ** 3 * (W - 1) / W
    out[W] = {"group_ms": ms, "best": best, "per_rank_compute_ms": ms[best] / W,
              "reduce_scatter_bytes_per_rank": rs_bytes,
              "projected_ms_at_400GBps": ms[best] / W + rs_bytes / 400e9 * 1e3,
              "tflops_1rank_equiv": flops / (ms[best] * 1e-3) / 1e12}
    op.close()
    print(W, json.dumps(out[W]), flush=True)
base = out[Ws[0]]["per_rank_compute_ms"]
for W in Ws:
    out[W]["projected_speedup"] = base / out[W]["projected_ms_at_400GBps"]
print(json.dumps(out))

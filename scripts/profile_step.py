"""Run the pipeline eagerly a few times on one workload (for ncu captures).

    python scripts/profile_step.py [cfg3] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = inputs.workload(name)
plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
xyz = torch.as_tensor(w.data.cloud.positions, device="cuda").contiguous()
q = torch.as_tensor(w.data.charges.values, device="cuda").contiguous()
out = torch.empty(w.n, dtype=torch.float64, device="cuda")
for _ in range(reps):
    try:
        plan.execute(xyz, q, out)
    except Exception as e:  # ablation builds (-D...SKIP) compute garbage on purpose
        if not os.environ.get("PROFILE_NOCHECK"):
            raise
        print("ignored:", e)
torch.cuda.synchronize()
print(f"{name}: ok, |z| = {float(torch.linalg.norm(out)):.6e}")

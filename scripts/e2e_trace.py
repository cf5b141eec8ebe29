"""Timeline of the pipelined host path (KPME_GPU_TRACE=1) for one workload."""
import os
import sys

os.environ["KPME_GPU_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
w = inputs.workload(name)
plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
xyz_h = torch.as_tensor(w.data.cloud.positions).contiguous().pin_memory()
q_h = torch.as_tensor(w.data.charges.values).contiguous().pin_memory()
out_h = torch.empty(w.n, dtype=torch.float64).pin_memory()
for c in [int(x) for x in (sys.argv[2:] or ["4"])]:
    plan.set_host_chunks(c)
    for i in range(3):
        if i == 2:
            print(f"--- {name} chunks={c}", file=sys.stderr, flush=True)
        plan.execute_host_ptr(w.n, xyz_h.data_ptr(), q_h.data_ptr(), out_h.data_ptr())

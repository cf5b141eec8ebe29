"""One eager config-5 operator application (for ncu launch lists).
usage: python scripts/dense_once.py N R"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan, dense_workspace_bytes, kron_matvec_dense  # noqa: E402

n, R = int(sys.argv[1]), int(sys.argv[2])
cfg, grid, L, dec = inputs.dense_case(n, R)
plan = KpmePlan(cfg, grid, L, dec, 1)
ops = [plan.axis_operands(a) for a in range(3)]
x = torch.randn(n, n, n, dtype=torch.float64, device="cuda")
ws = torch.empty(dense_workspace_bytes(n, n, n, R) // 8 + 1, dtype=torch.float64, device="cuda")
y = kron_matvec_dense(*ops, x, workspace=ws)
for _ in range(2):
    kron_matvec_dense(*ops, x, out=y, workspace=ws)
torch.cuda.synchronize()
print("ok", float(y.norm()))

"""Diagnostic: the m=0 entry of the collapsed core against sum(q) for a
water-like system (config-4 recipe).  usage: python scripts/water_core.py MOL K"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_18838_b200 as kp  # noqa: E402
from paper_2601_18838_b200 import inputs  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

mol, K = int(sys.argv[1]), int(sys.argv[2])
data = inputs.water_cloud(mol, 0)
dec = inputs.decomposition(1e-10)
grid = kp.build_cell_grid(kp.Box3((0.5, 0.5, 0.5), 0.5), (K, K, K))
n = len(data.charges.values)
plan = KpmePlan(kp.EwaldConfig(3.0, 4), grid, 6, dec, n)
xyz = torch.as_tensor(data.cloud.positions, device="cuda")
q = torch.as_tensor(data.charges.values, device="cuda")
core = torch.empty(plan.core_size(), dtype=torch.float64, device="cuda")
plan.forward(xyz, q, core)
c = core.cpu().numpy()
print("F000", c[0], "sumq(core)", c[-1], "fsum q", math.fsum(data.charges.values))
print("max|F|", np.abs(c[:-1]).max(), "sum|q|", np.abs(data.charges.values).sum())

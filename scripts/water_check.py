"""Water-like systems (config 4 recipe, fewer molecules) on the GPU against
the C oracle: device path, and the pipelined host path at every chunk count.

usage: python scripts/water_check.py MOLECULES K
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.binding import CpuKpme, Problem  # noqa: E402
from paper_2601_18838_b200 import inputs  # noqa: E402
import paper_2601_18838_b200 as kp  # noqa: E402
from paper_2601_18838_b200.plan import KpmePlan  # noqa: E402

mol, K = int(sys.argv[1]), int(sys.argv[2])
data = inputs.water_cloud(mol, 0)
dec = inputs.decomposition(1e-10)
tw, prof = dec.arrays()
pb = Problem(xi=3.0, modes=4, center=(0.5, 0.5, 0.5), radius=0.5, counts=(K, K, K), order=6,
             term_weights=tw, profiles=prof, correction=dec.correction,
             pos=data.cloud.positions, q=data.charges.values)
ref = CpuKpme("oracle").kpme_apply(pb, threads=os.cpu_count() or 1)
cfg = kp.EwaldConfig(3.0, 4)
grid = kp.build_cell_grid(kp.Box3((0.5, 0.5, 0.5), 0.5), (K, K, K))
n = len(data.charges.values)
plan = KpmePlan(cfg, grid, 6, dec, n)
xyz = torch.as_tensor(data.cloud.positions, device="cuda")
q = torch.as_tensor(data.charges.values, device="cuda")
zd = plan.execute(xyz, q).cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


print(f"water {mol} molecules, K={K}, n={n}, rms(ref)={np.sqrt(np.mean(ref**2)):.4g}")
print(f"  device path  rel vs oracle {rel(zd, ref):.3e}   mean diff {np.mean(zd - ref):.3e}")
for c in [1, 2, 3, 4, 8]:
    plan.set_host_chunks(c)
    zh = plan.execute_host(data.cloud.positions, data.charges.values)
    d = zh - ref
    print(f"  host C={c}     rel vs oracle {rel(zh, ref):.3e}   vs device {rel(zh, zd):.3e}"
          f"   mean diff {d.mean():.3e} std {d.std():.3e}")

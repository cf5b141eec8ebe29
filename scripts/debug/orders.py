"""Acceptance criterion 2's shapes (one cell, M = 2, N = 32, L = 3..16)
through the GPU path, one order per process (diagnostics)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2601_18838_b200 as kp  # noqa: E402
from oracle.binding import CpuKpme, make_problem  # noqa: E402

L = int(sys.argv[1])
nu = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
o = CpuKpme("oracle")
M = 2
pb = make_problem(o, n=32, counts=1, order=L, modes=M, eps=1e-14, center=(0, 0, 0),
                  radius=nu / (np.pi * M), seed=99)
from tests.test_gpu_parity import kp_objects  # noqa: E402

cfg, grid, dec, cloud, q = kp_objects(pb)
z = kp.kpme_apply(cfg, grid, L, dec, cloud, q).potentials
ref = o.kpme_apply(pb)
print(L, nu, np.linalg.norm(z - ref) / np.linalg.norm(ref), flush=True)

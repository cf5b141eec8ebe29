"""BASELINE configs 4 and 5 at their own sizes against the CPU oracle.

* Config 4 (3M water sites, K = 43, |Lambda| = 101; parallel.hpp:243-290):
  the device path and the pipelined host path against the C oracle's
  kpme_apply on every host thread, <= 1e-10 relative L2 (north star). The
  inputs are built twice -- by the package and by the oracle's own
  sample_cloud / sinc rule (oracle/workloads.py) -- and must agree bit for bit.
* Config 5 (dense SKP grid operator, kron.hpp:180-197): the DMMA operator on
  64^3 (R = 4..64) and 128^3 (R = 4, 8) against the oracle's
  kron_matvec_shuffle summed over terms, <= 1e-12. The n x n factors are built
  independently of the GPU, from the oracle's per-cell build_uv
  (symfourier.hpp:108-124) with kpme_apply's node shift (parallel.hpp:263-279);
  the GPU's own axis operands are checked against them too.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

E2E_TOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def test_e2e_cfg4_full_vs_oracle(oracle):
    from oracle import workloads
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload("cfg4")
    pb = workloads.problem("cfg4", oracle)
    assert np.array_equal(pb.pos, w.data.cloud.positions)
    assert np.array_equal(pb.q, w.data.charges.values)
    tw, prof = w.dec.arrays()
    assert np.array_equal(tw, pb.term_weights) and np.array_equal(prof, pb.profiles)
    assert len(pb.q) == 3_000_000 and pb.counts == (43, 43, 43) and len(tw) == 101

    plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
    zd = plan.execute(dev(pb.pos), dev(pb.q)).cpu().numpy()
    zh = plan.execute_host(pb.pos, pb.q)
    ref = oracle.kpme_apply(pb, threads=os.cpu_count() or 1)
    err_d, err_h = rel(zd, ref), rel(zh, ref)
    print(f"cfg4 full: rel-L2 device {err_d:.3e}, host path {err_h:.3e}")
    assert err_d <= E2E_TOL
    assert err_h <= E2E_TOL
    assert rel(zh, zd) <= 1e-13


def _oracle_dense(oracle, factors, x, nterms):
    """sum_r kron_matvec_shuffle([A_r, B_r, C_r], x) (kron.hpp:180-197), terms
    in parallel threads (ctypes drops the GIL), summed in term order."""
    def one(t):
        out, mult = oracle.kron_matvec_shuffle([factors[a][t] for a in range(3)], x)
        return out, mult

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        parts = list(ex.map(one, range(nterms)))
    ref = np.zeros_like(x)
    for out, _ in parts:
        ref += out
    return ref, [m for _, m in parts]


CFG5 = [(64, R) for R in (4, 8, 16, 32, 64)] + [(128, 4), (128, 8)]


@pytest.fixture(scope="module")
def cfg5_factors(oracle):
    """Oracle-built factors for the largest R per mesh (prefixes serve the
    smaller R: term order is the rule's order)."""
    from oracle import workloads

    return {n: workloads.dense_factors(oracle, n, max(R for m, R in CFG5 if m == n))
            for n in sorted({n for n, _ in CFG5})}


@pytest.mark.parametrize("n,R", CFG5)
def test_cfg5_dense_vs_oracle(oracle, cfg5_factors, n, R):
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan, kron_matvec_dense

    fac = [f[:R] for f in cfg5_factors[n]]
    # the GPU's own factor build agrees with the oracle's build_uv assembly
    cfg, grid, L, dec = inputs.dense_case(n, R)
    plan = KpmePlan(cfg, grid, L, dec, 1)
    for a in range(3):
        g = plan.axis_operands(a).cpu().numpy()
        scale = np.abs(fac[a]).max()
        assert np.abs(g - fac[a]).max() <= 1e-13 * scale
    plan.close()

    rng = np.random.default_rng(n * 1000 + R)
    x = rng.standard_normal(n ** 3)
    y = kron_matvec_dense(*(dev(f) for f in fac), dev(x).reshape(n, n, n))
    y = y.cpu().numpy().ravel()
    ref, mults = _oracle_dense(oracle, fac, x, R)
    assert all(m == 3 * n ** 4 for m in mults)  # op_count_estimate / multiply_count
    err = rel(y, ref)
    print(f"cfg5 n={n} R={R}: rel-L2 {err:.3e}")
    assert err <= 1e-12

"""Slab-decomposed paths on one B200.

G z-slab plans run one after another on the same GPU (no rank waits on
another): every slab's forward half, the sum of the partial cores (what the
NCCL all-reduce computes across GPUs), then every slab's backward half. The
result must match the single-plan run -- decomposition invariance across GPU
counts (acceptance criterion 4, acceptance.cpp:194-226: <= 1e-12)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("world", [2, 3, 8])
def test_slabs_equal_single_plan(world):
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.dist import route_particles, slab_bounds
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload("cfg2")
    dev = torch.device("cuda", 0)
    full = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
    xyz = torch.as_tensor(w.data.cloud.positions, device=dev).contiguous()
    q = torch.as_tensor(w.data.charges.values, device=dev).contiguous()
    ref = full.execute(xyz, q).cpu().numpy()

    routes = route_particles(w.data.cloud.positions, w.grid, world)
    plans, cores, parts = [], [], []
    for r in range(world):
        idx = routes[r]
        p = KpmePlan(w.cfg, w.grid, w.order, w.dec, max(1, len(idx)),
                     slab=slab_bounds(w.grid.counts[2], r, world))
        x = torch.as_tensor(w.data.cloud.positions[idx], device=dev).contiguous()
        qq = torch.as_tensor(w.data.charges.values[idx], device=dev).contiguous()
        core = torch.zeros(p.core_size(), dtype=torch.float64, device=dev)
        p.forward(x, qq, core)
        plans.append(p)
        cores.append(core)
        parts.append((idx, x, qq))
    total = torch.stack(cores).sum(0)
    z = np.zeros(w.n)
    for p, (idx, x, qq) in zip(plans, parts):
        out = torch.empty(len(idx), dtype=torch.float64, device=dev)
        p.backward(total, out)
        p.status()
        z[idx] = out.cpu().numpy()
    assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= 1e-12


def test_slab_rejects_foreign_particles():
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload("cfg1")
    p = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, slab=(0, 2))
    dev = torch.device("cuda", 0)
    core = torch.zeros(p.core_size(), dtype=torch.float64, device=dev)
    p.forward(torch.as_tensor(w.data.cloud.positions, device=dev).contiguous(),
              torch.as_tensor(w.data.charges.values, device=dev).contiguous(), core)
    with pytest.raises(ValueError, match="outside this plan's cell block"):
        p.status()


def test_dense_strategies_single_rank_on_dmma():
    """The dense slab operator's three strategies (world = 1) on the DMMA
    GEMM equal kron_matvec_dense."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.dist import DenseSlabOperator
    from paper_2601_18838_b200.plan import KpmePlan, dgemm_tn, kron_matvec_dense

    cfg, grid, L, dec = inputs.dense_case(64, 4)
    plan = KpmePlan(cfg, grid, L, dec, 1)
    ops = [plan.axis_operands(a) for a in range(3)]
    x = torch.randn(64, 64, 64, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(3))
    ref = kron_matvec_dense(*ops, x)
    op = DenseSlabOperator(*ops, (64, 64, 64), lambda a, f, o, acc: dgemm_tn(a, f, o, acc))
    for s in DenseSlabOperator.STRATEGIES:
        y = op.apply(x, s)
        assert float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref)) <= 1e-13, s


@pytest.mark.parametrize("dims", [(2, 2, 2), (1, 3, 1), (2, 1, 3)])
def test_rank_grid_blocks_equal_single_plan(dims):
    """General P0 x P1 x P2 device grids (cell blocks, kpme_gpu_plan_create_block):
    every block's forward half, the summed cores, every backward half --
    equal to the single-plan run (<= 1e-12)."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.dist import rank_grid_block, route_particles_grid
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload("cfg2")
    dev = torch.device("cuda", 0)
    full = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n)
    xyz = torch.as_tensor(w.data.cloud.positions, device=dev).contiguous()
    q = torch.as_tensor(w.data.charges.values, device=dev).contiguous()
    ref = full.execute(xyz, q).cpu().numpy()
    world = int(np.prod(dims))
    routes = route_particles_grid(w.data.cloud.positions, w.grid, dims)
    plans, cores, parts = [], [], []
    for r in range(world):
        idx = routes[r]
        p = KpmePlan(w.cfg, w.grid, w.order, w.dec, max(1, len(idx)),
                     block=rank_grid_block(w.grid.counts, dims, r))
        x = torch.as_tensor(w.data.cloud.positions[idx], device=dev).contiguous()
        qq = torch.as_tensor(w.data.charges.values[idx], device=dev).contiguous()
        core = torch.zeros(p.core_size(), dtype=torch.float64, device=dev)
        p.forward(x, qq, core)
        plans.append(p)
        cores.append(core)
        parts.append((idx, x, qq))
    total = torch.stack(cores).sum(0)
    z = np.zeros(w.n)
    for p, (idx, x, qq) in zip(plans, parts):
        out = torch.empty(len(idx), dtype=torch.float64, device=dev)
        p.backward(total, out)
        p.status()
        z[idx] = out.cpu().numpy()
    assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= 1e-12


def test_block_rejects_foreign_particles():
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import KpmePlan

    w = inputs.workload("cfg1")
    p = KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, block=((0, 4), (0, 8), (0, 8)))
    dev = torch.device("cuda", 0)
    core = torch.zeros(p.core_size(), dtype=torch.float64, device=dev)
    p.forward(torch.as_tensor(w.data.cloud.positions, device=dev).contiguous(),
              torch.as_tensor(w.data.charges.values, device=dev).contiguous(), core)
    with pytest.raises(ValueError, match="outside this plan's cell block"):
        p.status()
    with pytest.raises(ValueError, match="block outside the cell grid"):
        KpmePlan(w.cfg, w.grid, w.order, w.dec, w.n, block=((0, 9), (0, 8), (0, 8)))

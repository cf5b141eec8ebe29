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
    """The library's dense slab operator (kpme_gpu_dense_slab, one process
    rank, no NCCL at nranks = 1): all three strategies equal
    kron_matvec_dense, and the chooser times every one."""
    from paper_2601_18838_b200 import inputs
    from paper_2601_18838_b200.plan import DenseSlab, KpmePlan, kron_matvec_dense

    cfg, grid, L, dec = inputs.dense_case(64, 4)
    plan = KpmePlan(cfg, grid, L, dec, 1)
    ops = [plan.axis_operands(a) for a in range(3)]
    x = torch.randn(64, 64, 64, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(3))
    ref = kron_matvec_dense(*ops, x)
    op = DenseSlab(*ops)
    assert op.bounds(0) == (0, 64)
    for s in ("reduce_scatter", "rank_split", "alltoall"):
        y = torch.full_like(x, float("nan"))
        op.apply(x, y, s)
        assert float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref)) <= 1e-13, s
    ms, best = op.choose(x, torch.empty_like(x))
    assert set(ms) == {"reduce_scatter", "rank_split", "alltoall"} and best in ms


@pytest.mark.parametrize("world,shape,nterms", [(2, (24, 20, 32), 5), (3, (32, 24, 40), 4),
                                                (4, (20, 16, 26), 7), (5, (40, 16, 23), 3)])
def test_dense_slab_group_strategies(world, shape, nterms):
    """`world` ranks of the dense slab operator held by one process on the one
    B200 (kpme_gpu_dense_slab_create_group: the same local kernels, packing
    and block layouts as one rank per GPU; the collectives are peer copies in
    rank order). Uneven z- and x-slabs, rectangular meshes, term counts not a
    multiple of the rank count: every strategy equals the dense operator
    (<= 1e-13) on every rank's slab."""
    from paper_2601_18838_b200.dist import slab_bounds
    from paper_2601_18838_b200.plan import DenseSlab, kron_matvec_dense

    g = torch.Generator(device="cuda").manual_seed(world)
    n0, n1, n2 = shape
    A = torch.randn(nterms, n0, n0, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(nterms, n1, n1, dtype=torch.float64, device="cuda", generator=g)
    C_ = torch.randn(nterms, n2, n2, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(n0, n1, n2, dtype=torch.float64, device="cuda", generator=g)
    ref = kron_matvec_dense(A, B, C_, x)
    op = DenseSlab.group([(A, B, C_)] * world, [0] * world)
    bounds = [op.bounds(r) for r in range(world)]
    assert bounds == [slab_bounds(n2, r, world) for r in range(world)]
    xs = [x[:, :, lo:hi].contiguous() for lo, hi in bounds]
    for s in ("reduce_scatter", "rank_split", "alltoall"):
        ys = [torch.full_like(t, float("nan")) for t in xs]
        op.apply(xs, ys, s)
        for (lo, hi), y in zip(bounds, ys):
            r = ref[:, :, lo:hi]
            assert float(torch.linalg.norm(y - r) / torch.linalg.norm(r)) <= 1e-13, (s, lo, hi)
    ms, best = op.choose(xs, [torch.empty_like(t) for t in xs])
    assert best in ms


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

"""Multi-rank host logic on CPU: torch.distributed gloo, world size 2.

Runs paper_2601_18838_b200.dist (the code the GPU ranks run, with NCCL) with
CPU backends: the slab routing and the single core all-reduce of the
collapsed end-to-end path, and the three dense-operator strategies for the
sharded z product. Results must equal the single-process answers (oracle /
dense reference) -- the decomposition-invariance check of acceptance
criterion 4 (acceptance.cpp:194-226) applied to GPU counts."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _collapsed_worker(rank, world, port, res):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from oracle.binding import CpuKpme, make_problem
    from paper_2601_18838_b200.api import Box3, build_cell_grid
    from paper_2601_18838_b200.dist import SlabDriver, route_particles, slab_bounds
    from tests.dist_backends import CpuCollapsedSlab

    oracle = CpuKpme("oracle")
    pb = make_problem(oracle, n=400, counts=(3, 2, 5), order=4, modes=3, eps=1e-9, seed=3,
                      charges="neutral")
    grid = build_cell_grid(Box3(pb.center, pb.radius), pb.counts)
    routes = route_particles(pb.pos, grid, world)
    idx = routes[rank]
    z_lo, z_hi = slab_bounds(pb.counts[2], rank, world)
    drv = SlabDriver(CpuCollapsedSlab(pb, z_lo, z_hi), device="cpu")
    out = torch.zeros(len(idx), dtype=torch.float64)
    drv.apply(torch.as_tensor(pb.pos[idx]), torch.as_tensor(pb.q[idx]), out)
    parts = [None] * world
    dist.all_gather_object(parts, (idx, out.numpy()))
    if rank == 0:
        z = np.zeros(len(pb.q))
        for i, v in parts:
            z[i] = v
        ref = oracle.kpme_apply(pb)
        res["rel"] = float(np.linalg.norm(z - ref) / np.linalg.norm(ref))
        res["covered"] = int(sum(len(i) for i, _ in parts))
    dist.destroy_process_group()


def _grid_worker(rank, world, port, res):
    """Collapsed path on a general device grid: rank grids (2, 1, 1) and
    (1, 2, 1) -- cell blocks split along x / y, same single core all-reduce."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from oracle.binding import CpuKpme, make_problem
    from paper_2601_18838_b200.api import Box3, build_cell_grid
    from paper_2601_18838_b200.dist import SlabDriver, rank_grid_block, route_particles_grid
    from tests.dist_backends import CpuCollapsedSlab

    oracle = CpuKpme("oracle")
    pb = make_problem(oracle, n=400, counts=(4, 3, 2), order=4, modes=3, eps=1e-9, seed=5,
                      charges="neutral")
    grid = build_cell_grid(Box3(pb.center, pb.radius), pb.counts)
    ref = oracle.kpme_apply(pb) if rank == 0 else None
    for dims in ((2, 1, 1), (1, 2, 1)):
        idx = route_particles_grid(pb.pos, grid, dims)[rank]
        block = rank_grid_block(pb.counts, dims, rank)
        drv = SlabDriver(CpuCollapsedSlab(pb, block[2][0], block[2][1], block), device="cpu")
        out = torch.zeros(len(idx), dtype=torch.float64)
        drv.apply(torch.as_tensor(pb.pos[idx]), torch.as_tensor(pb.q[idx]), out)
        parts = [None] * world
        dist.all_gather_object(parts, (idx, out.numpy()))
        if rank == 0:
            z = np.zeros(len(pb.q))
            for i, v in parts:
                z[i] = v
            res[str(dims)] = (float(np.linalg.norm(z - ref) / np.linalg.norm(ref)),
                              int(sum(len(i) for i, _ in parts)))
    dist.destroy_process_group()


def _dense_worker(rank, world, port, res):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    _init(rank, world, port)
    from paper_2601_18838_b200.dist import DenseSlabOperator, slab_bounds, torch_gemm_tn

    g = torch.Generator().manual_seed(7)
    n = (6, 5, 8)
    nt = 3
    A = torch.randn(nt, n[0], n[0], generator=g, dtype=torch.float64)
    B = torch.randn(nt, n[1], n[1], generator=g, dtype=torch.float64)
    C = torch.randn(nt, n[2], n[2], generator=g, dtype=torch.float64)
    x = torch.randn(*n, generator=g, dtype=torch.float64)
    ref = torch.zeros(n, dtype=torch.float64)
    for t in range(nt):
        ref += torch.einsum("ax,by,cz,xyz->abc", A[t], B[t], C[t], x)
    lo, hi = slab_bounds(n[2], rank, world)
    op = DenseSlabOperator(A, B, C, n, torch_gemm_tn, chunk=2)
    errs = {}
    for s in DenseSlabOperator.STRATEGIES:
        y = op.apply(x[:, :, lo:hi].contiguous(), s)
        errs[s] = float((y - ref[:, :, lo:hi]).norm() / ref[:, :, lo:hi].norm())
    choice = op.choose(x[:, :, lo:hi].contiguous())
    allerr = [None] * world
    dist.all_gather_object(allerr, errs)
    if rank == 0:
        res["errs"] = allerr
        res["choice"] = choice
    dist.destroy_process_group()


def _run(fn):
    mgr = mp.Manager()
    res = mgr.dict()
    mp.spawn(fn, args=(2, _free_port(), res), nprocs=2, join=True)
    return dict(res)


def test_slab_routing_matches_reference_sort(oracle):
    """Routing uses the reference's exact cell arithmetic (bit-exact vs
    assign_particles) and covers every particle once."""
    from oracle.binding import make_problem
    from paper_2601_18838_b200.api import Box3, build_cell_grid
    from paper_2601_18838_b200.dist import route_particles, slab_bounds

    pb = make_problem(oracle, n=5000, counts=(4, 3, 7), order=4, modes=2, eps=1e-6, seed=4)
    grid = build_cell_grid(Box3(pb.center, pb.radius), pb.counts)
    perm, start = oracle.assign_particles(pb.center, pb.radius, pb.counts, pb.pos)
    cell_of = np.empty(len(perm), np.int64)
    for c in range(len(start) - 1):
        cell_of[perm[start[c]:start[c + 1]]] = c
    for world in (1, 2, 3, 8):
        routes = route_particles(pb.pos, grid, world)
        assert sum(len(r) for r in routes) == len(perm)
        for r, idx in enumerate(routes):
            lo, hi = slab_bounds(pb.counts[2], r, world)
            assert ((cell_of[idx] % pb.counts[2] >= lo) & (cell_of[idx] % pb.counts[2] < hi)).all()
            assert (np.diff(idx) > 0).all()


def test_collapsed_slabs_gloo_world2():
    res = _run(_collapsed_worker)
    assert res["covered"] == 400
    assert res["rel"] <= 1e-10, res


def test_dense_strategies_gloo_world2():
    res = _run(_dense_worker)
    for rank_errs in res["errs"]:
        for s, e in rank_errs.items():
            assert e <= 1e-12, (s, e)
    assert res["choice"] in ("reduce_scatter", "rank_split", "alltoall")


def test_rank_grid_routing_matches_reference_sort(oracle):
    """General P0 x P1 x P2 device grids: every particle is routed once, to
    the rank whose cell block holds its cell (bit-exact cell arithmetic);
    blocks tile the grid and ranks flatten like RankGrid (parallel.hpp:46-82)."""
    from oracle.binding import make_problem
    from paper_2601_18838_b200.api import Box3, build_cell_grid
    from paper_2601_18838_b200.dist import axis_group, rank_grid_block, route_particles_grid

    pb = make_problem(oracle, n=5000, counts=(5, 4, 7), order=4, modes=2, eps=1e-6, seed=6)
    grid = build_cell_grid(Box3(pb.center, pb.radius), pb.counts)
    perm, start = oracle.assign_particles(pb.center, pb.radius, pb.counts, pb.pos)
    cell_of = np.empty(len(perm), np.int64)
    for c in range(len(start) - 1):
        cell_of[perm[start[c]:start[c + 1]]] = c
    K = pb.counts
    c0, c1, c2 = cell_of // (K[1] * K[2]), (cell_of // K[2]) % K[1], cell_of % K[2]
    for dims in ((2, 2, 2), (1, 4, 1), (3, 1, 2), (1, 1, 8)):
        routes = route_particles_grid(pb.pos, grid, dims)
        assert sum(len(r) for r in routes) == len(perm)
        cells = 0
        for r, idx in enumerate(routes):
            b = rank_grid_block(K, dims, r)
            cells += np.prod([hi - lo for lo, hi in b])
            for a, ca in enumerate((c0, c1, c2)):
                assert ((ca[idx] >= b[a][0]) & (ca[idx] < b[a][1])).all()
            assert (np.diff(idx) > 0).all()
        assert cells == K[0] * K[1] * K[2]
    assert axis_group(5, (2, 2, 2), 1) == [5, 7]
    assert axis_group(5, (2, 2, 2), 0) == [1, 5]


def test_collapsed_rank_grids_gloo_world2():
    res = _run(_grid_worker)
    for dims in ("(2, 1, 1)", "(1, 2, 1)"):
        rel, covered = res[dims]
        assert covered == 400
        assert rel <= 1e-10, (dims, rel)

"""Multi-device plans (one process driving a device list) and plans owning an
NCCL communicator, on the one B200 of the test box.

* A device list that repeats device 0 puts several cell blocks on one GPU:
  the routing, per-block pipelines, the peer-memory core sum and the merge
  to global order all run, and must agree with one plan (<= 1e-12, the
  reference's decomposition-invariance tolerance, acceptance.cpp:194-226) and
  with the oracle (<= 1e-10). NCCL needs distinct devices and must refuse.
* A one-device list with the NCCL exchange, and a block plan attached to a
  one-rank NCCL communicator, run the NCCL code paths for real.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


@pytest.fixture(scope="module")
def problem(oracle):
    from oracle.binding import make_problem

    from tests.test_gpu_parity import kp_objects

    pb = make_problem(oracle, n=60000, counts=(7, 6, 9), order=6, modes=4, eps=1e-10, seed=3,
                      charges="neutral")
    return pb, kp_objects(pb), oracle.kpme_apply(pb)


@pytest.mark.parametrize("dims", [(1, 1, 2), (1, 1, 3), (1, 1, 8), (2, 2, 1), (2, 1, 3),
                                  (1, 3, 1)])
def test_multi_device_blocks_on_one_gpu(problem, dims):
    from paper_2601_18838_b200.plan import KpmePlan, MultiDevicePlan

    pb, (cfg, grid, dec, cloud, q), ref = problem
    G = int(np.prod(dims))
    single = KpmePlan(cfg, grid, pb.order, dec, len(pb.q))
    z1 = single.execute(dev(pb.pos), dev(pb.q)).cpu().numpy()
    mp = MultiDevicePlan(cfg, grid, pb.order, dec, len(pb.q), devices=[0] * G, dims=dims)
    assert mp.collective == "peer"
    zd = mp.execute(dev(pb.pos), dev(pb.q)).cpu().numpy()
    zh = mp.execute_host(pb.pos, pb.q)
    assert rel(zd, z1) <= 1e-12
    assert rel(zd, ref) <= 1e-10
    assert np.array_equal(zd, zh)
    assert np.array_equal(zd, mp.execute(dev(pb.pos), dev(pb.q)).cpu().numpy())  # deterministic
    assert mp.launches() > G
    with pytest.raises(Exception, match="distinct devices"):
        mp.set_collective("nccl")


def test_multi_device_errors_and_edges(problem):
    from paper_2601_18838_b200.plan import MultiDevicePlan

    pb, (cfg, grid, dec, cloud, q), ref = problem
    mp = MultiDevicePlan(cfg, grid, pb.order, dec, len(pb.q), devices=[0, 0, 0])
    bad = np.array(pb.pos)
    bad[41000] = (0.5, 1.7, 0.5)
    bad[52000] = (-0.5, 0.5, 0.5)
    with pytest.raises(ValueError, match="particle 41000 outside the box"):
        mp.execute_host(bad, pb.q)
    with pytest.raises(ValueError, match="particle 41000 outside the box"):
        mp.execute(dev(bad), dev(pb.q))
    z = mp.execute_host(pb.pos, pb.q)  # recovers
    assert rel(z, ref) <= 1e-10
    assert mp.execute_host(np.zeros((0, 3)), np.zeros(0)).shape == (0,)
    z5 = mp.execute_host(pb.pos[:5], pb.q[:5])
    assert z5.shape == (5,)
    with pytest.raises(ValueError, match="more particles"):
        mp.execute_host(np.concatenate([pb.pos, pb.pos]), np.concatenate([pb.q, pb.q]))
    with pytest.raises(ValueError, match="rank grid size"):
        MultiDevicePlan(cfg, grid, pb.order, dec, 10, devices=[0, 0], dims=(1, 1, 3))
    with pytest.raises(ValueError, match="device ordinal"):
        MultiDevicePlan(cfg, grid, pb.order, dec, 10, devices=[0, 99])


def test_multi_device_nccl_one_rank(problem):
    """The NCCL exchange of a multi-device plan (ncclCommInitAll over the
    device list) with the one device the box has."""
    from paper_2601_18838_b200.plan import KpmePlan, MultiDevicePlan

    pb, (cfg, grid, dec, cloud, q), ref = problem
    z1 = KpmePlan(cfg, grid, pb.order, dec, len(pb.q)).execute(dev(pb.pos), dev(pb.q))
    mp = MultiDevicePlan(cfg, grid, pb.order, dec, len(pb.q), devices=[0], dims=(1, 1, 1),
                         collective="nccl")
    assert mp.collective == "nccl"
    z = mp.execute(dev(pb.pos), dev(pb.q))
    assert rel(z.cpu().numpy(), z1.cpu().numpy()) <= 1e-13


def test_block_plan_owning_nccl_comm(problem):
    """A plan attached to a one-rank NCCL communicator: execute and the CUDA
    graph (forward -> ncclAllReduce -> backward captured together) agree with
    the plain plan."""
    from paper_2601_18838_b200.plan import KpmePlan, nccl_unique_id

    pb, (cfg, grid, dec, cloud, q), ref = problem
    xyz, qq = dev(pb.pos), dev(pb.q)
    z1 = KpmePlan(cfg, grid, pb.order, dec, len(pb.q)).execute(xyz, qq).clone()
    p = KpmePlan(cfg, grid, pb.order, dec, len(pb.q), slab=(0, grid.counts[2]))
    p.attach_comm(1, 0, nccl_unique_id())
    z = p.execute(xyz, qq).clone()
    assert rel(z.cpu().numpy(), z1.cpu().numpy()) <= 1e-13
    out = torch.empty_like(z)
    p.execute_graph(xyz, qq, out)
    p.execute_graph(xyz, qq, out)
    torch.cuda.synchronize()
    assert torch.equal(out, z)


def test_kpme_apply_device_list_and_plan_cache(problem):
    """kpme_apply with a device list (z-slabs through kpme_gpu_apply) and the
    one-shot plan cache: repeated calls reuse a plan and give the same bits."""
    import time

    import paper_2601_18838_b200 as kp

    pb, (cfg, grid, dec, cloud, q), ref = problem
    kp._lib.lib.kpme_gpu_apply_cache_clear()
    t0 = time.perf_counter()
    a = kp.kpme_apply(cfg, grid, pb.order, dec, cloud, q).potentials
    t1 = time.perf_counter()
    b = kp.kpme_apply(cfg, grid, pb.order, dec, cloud, q).potentials
    t2 = time.perf_counter()
    assert np.array_equal(a, b)
    assert rel(a, ref) <= 1e-10
    print(f"one-shot kpme_apply: first {1e3 * (t1 - t0):.2f} ms, cached {1e3 * (t2 - t1):.2f} ms")
    m = kp.kpme_apply(cfg, grid, pb.order, dec, cloud, q, devices=[0, 0, 0, 0]).potentials
    assert rel(m, a) <= 1e-12
    kp._lib.lib.kpme_gpu_apply_cache_clear()

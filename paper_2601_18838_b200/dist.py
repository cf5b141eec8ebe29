"""Multi-GPU SKP-PME: one process per GPU, mesh slabs along z (axis 2).

The reference simulates a K0 x K1 x K2 rank grid with ordered axis-group
all-reduces (SimulatedComm, parallel.hpp:98-145; spkmv, parallel.hpp:156-179).
On an 8 x B200 NVSwitch box the natural decomposition is one z-slab of whole
cell planes per GPU (a (1, 1, G) rank grid in the reference's terms):

* end to end (configs 3/4), collapsed formulation: every rank spreads and
  contracts its own slab into a partial R^3 + 1 core (the last entry is the
  slab's charge sum), ONE all-reduce of (2M+1)^3 + 1 doubles sums the cores
  (the collapsed counterpart of the z-axis group reductions and of
  allreduce_scalar, parallel.hpp:254-257), then every rank expands and
  gathers its own slab. ``SlabDriver``.
* dense operator (config 5), three strategies for the non-local z product,
  all on the DMMA GEMM kernel: ``reduce_scatter`` (z contracted last from
  the local z-slice into full-length partial sums, one reduce-scatter --
  the SPKMV pattern of the reference), ``rank_split`` (terms split across
  ranks on the full mesh, all-gather + reduce-scatter) and ``alltoall``
  (slab transpose z <-> x around the z product). ``DenseSlabOperator``
  picks the fastest per shape by measuring each once (``choose``).

Collectives go through torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the per-rank compute is injected (``KpmePlan`` slabs / the DMMA GEMM
on GPUs), so the CPU tests run this exact orchestration code.
"""
from __future__ import annotations

import time
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist


# ---- geometry of the decomposition -----------------------------------------------

def slab_bounds(k: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced split of k cell planes over world ranks."""
    return (k * rank) // world, (k * (rank + 1)) // world


def axis_cells(x: np.ndarray, center: float, radius: float, k: int) -> np.ndarray:
    """Cell index along one axis with the reference's exact arithmetic
    (geometry.hpp:141-148): IEEE double, same operation order, no FMA."""
    t = ((x - (center - radius)) * k) / (2.0 * radius)
    idx = np.floor(t).astype(np.int64)
    tie = (t == idx.astype(np.float64)) & (idx > 0)
    idx = idx - tie.astype(np.int64)
    return np.clip(idx, 0, k - 1)


def rank_grid_coords(rank: int, dims) -> tuple[int, int, int]:
    """RankGrid::unflatten (parallel.hpp:63-70): ranks flatten like cells."""
    r2 = rank % dims[2]
    r = rank // dims[2]
    return r // dims[1], r % dims[1], r2


def rank_grid_block(counts, dims, rank: int) -> tuple:
    """Cell block ((lo0, hi0), (lo1, hi1), (lo2, hi2)) of ``rank`` in a
    P0 x P1 x P2 device grid: a balanced contiguous split per axis."""
    c = rank_grid_coords(rank, dims)
    return tuple(slab_bounds(counts[a], c[a], dims[a]) for a in range(3))


def axis_group(rank: int, dims, axis: int) -> list[int]:
    """RankGrid::axis_group (parallel.hpp:72-81): the ranks agreeing with
    ``rank`` on every axis but ``axis``, ascending."""
    c = list(rank_grid_coords(rank, dims))
    out = []
    for i in range(dims[axis]):
        c[axis] = i
        out.append((c[0] * dims[1] + c[1]) * dims[2] + c[2])
    return out


def route_particles_grid(pos: np.ndarray, grid, dims) -> list[np.ndarray]:
    """Global indices (ascending) of the particles each rank's cell block
    owns, for a P0 x P1 x P2 device grid (the exact key arithmetic on every
    axis)."""
    pos = np.asarray(pos)
    cells = [axis_cells(pos[:, a], grid.box.center[a], grid.box.radius, grid.counts[a])
             for a in range(3)]
    owner = np.zeros(len(pos), dtype=np.int64)
    for a in range(3):
        bounds = np.array([slab_bounds(grid.counts[a], i, dims[a])[1] for i in range(dims[a])])
        coord = np.searchsorted(bounds, cells[a], side="right")
        owner = owner * dims[a] + coord
    world = int(np.prod(dims))
    return [np.nonzero(owner == r)[0] for r in range(world)]


def route_particles(pos: np.ndarray, grid, world: int) -> list[np.ndarray]:
    """Global indices (ascending) of the particles each z-slab owns -- the
    one-off particle distribution step (the paper's all2allv),
    reported separately from the step time."""
    c2 = axis_cells(np.asarray(pos)[:, 2], grid.box.center[2], grid.box.radius, grid.counts[2])
    out = []
    for r in range(world):
        lo, hi = slab_bounds(grid.counts[2], r, world)
        out.append(np.nonzero((c2 >= lo) & (c2 < hi))[0])
    return out


# ---- end to end: collapsed form, one core all-reduce ---------------------------------

class SlabDriver:
    """Per-rank step of the slab-decomposed kpme_apply.

    ``backend`` provides ``core_size()``, ``forward(xyz, q, core)`` (partial
    core of the local slab) and ``backward(core, out)`` (local potentials
    from the summed core); on GPUs it is a slab ``KpmePlan``."""

    def __init__(self, backend, group=None, device=None):
        self.backend = backend
        self.group = group
        self.core = torch.zeros(backend.core_size(), dtype=torch.float64, device=device)

    def apply(self, xyz: torch.Tensor, q: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        self.backend.forward(xyz, q, self.core)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(self.core, op=dist.ReduceOp.SUM, group=self.group)
        self.backend.backward(self.core, out)
        return out


class SlabPlan:
    """Bench-facing wrapper: routes the workload's particles to this rank's
    slab (or, with ``dims = (P0, P1, P2)``, to its cell block of a general
    device grid, ranks flattened like RankGrid, parallel.hpp:46-82), builds
    the plan and exposes the timed callables. The exchange is the same single
    core all-reduce for every grid shape.

    Under an initialised process group the plan owns its NCCL communicator
    (``KpmePlan.attach_comm``; the 128-byte id is broadcast once through the
    group): the library runs forward half -> ncclAllReduce -> backward half
    on its own stream, captured as one CUDA graph, and the host path
    (``kpme_gpu_plan_execute``) includes the same exchange."""

    def __init__(self, w, rank: int, world: int, device: int = 0, group=None, dims=None):
        from .plan import KpmePlan, nccl_unique_id

        self.w, self.rank, self.world = w, rank, world
        self.dims = tuple(dims) if dims is not None else (1, 1, world)
        if int(np.prod(self.dims)) != world:
            raise ValueError(f"rank grid {self.dims} does not have {world} ranks")
        if self.dims == (1, 1, world):
            self.routes = route_particles(w.data.cloud.positions, w.grid, world)
        else:
            self.routes = route_particles_grid(w.data.cloud.positions, w.grid, self.dims)
        self.idx = self.routes[rank]
        self.block = rank_grid_block(w.grid.counts, self.dims, rank)
        self.z = self.block[2]
        dev = torch.device("cuda", device)
        self.plan = KpmePlan(w.cfg, w.grid, w.order, w.dec, max(1, len(self.idx)), device=device,
                             block=self.block)
        if dist.is_initialized():
            uid = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0, group=group)
            self.plan.attach_comm(world, rank, uid[0])
        self.library_comm = dist.is_initialized()
        self.driver = SlabDriver(self.plan, group, dev)
        pos = w.data.cloud.positions[self.idx]
        q = w.data.charges.values[self.idx]
        self.n = len(self.idx)
        self.xyz = torch.as_tensor(pos, device=dev).contiguous()
        self.q = torch.as_tensor(q, device=dev).contiguous()
        self.out = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.xyz_h = torch.as_tensor(pos).contiguous().pin_memory()
        self.q_h = torch.as_tensor(q).contiguous().pin_memory()
        self.out_h = torch.empty(self.n, dtype=torch.float64).pin_memory()
        self.apply()
        self.plan.status()

    def apply(self):
        if self.library_comm:
            self.plan.execute(self.xyz, self.q, self.out, defer_checks=True)
        else:
            self.driver.apply(self.xyz, self.q, self.out)

    def step(self):
        """One device-resident step: the plan's captured graph (sort, spread,
        contractions, NCCL core all-reduce, gather)."""
        if self.library_comm:
            self.plan.execute_graph(self.xyz, self.q, self.out)
        else:
            self.driver.apply(self.xyz, self.q, self.out)

    def e2e_step(self):
        """Host in, host out through kpme_gpu_plan_execute (pinned buffers):
        H2D of the local particles, the pipeline with its exchange, D2H."""
        if self.library_comm:
            self.plan.execute_host_ptr(self.n, self.xyz_h.data_ptr(), self.q_h.data_ptr(),
                                       self.out_h.data_ptr())
            return
        self.xyz.copy_(self.xyz_h, non_blocking=True)
        self.q.copy_(self.q_h, non_blocking=True)
        self.driver.apply(self.xyz, self.q, self.out)
        self.out_h.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    def bench_callables(self):
        launches = self.plan.launches()
        meta = {"rank_grid": list(self.dims), "cell_block": [list(b) for b in self.block],
                "local_particles": int(self.n),
                "exchange": (f"ncclAllReduce of {self.plan.core_size()} doubles per step on the "
                             f"plan's own communicator" if self.library_comm else "none (1 rank)"),
                "cuda_graph": True}
        return self.step, self.e2e_step, launches, meta

    def gather_global(self) -> np.ndarray:
        """All ranks' potentials in global particle order (for tests)."""
        parts = [None] * self.world
        dist.all_gather_object(parts, (self.idx, self.out.cpu().numpy()))
        z = np.zeros(self.w.n)
        for idx, val in parts:
            z[idx] = val
        return z


# ---- dense operator on z-slabs (config 5) ---------------------------------------------

Gemm = Callable[[torch.Tensor, torch.Tensor, torch.Tensor, bool], torch.Tensor]


def torch_gemm_tn(inp: torch.Tensor, F: torch.Tensor, out: torch.Tensor, accumulate: bool):
    """out[m][i] (+)= sum_k inp[k][m] F[i][k] with torch (CPU tests)."""
    r = inp.t() @ F.t()
    if accumulate:
        out += r
    else:
        out.copy_(r)
    return out


class DenseSlabOperator:
    """y = sum_r (A_r (x) B_r (x) C_r) x with x and y distributed as z-slabs
    ``x_local[n0][n1][nz_local]`` (rank order = z order).

    ``gemm(inp, F, out, accumulate)`` computes out[m][i] (+)= sum_k inp[k][m]
    F[i][k]; on GPUs it is the DMMA kernel (``plan.dgemm_tn``)."""

    STRATEGIES = ("reduce_scatter", "rank_split", "alltoall")

    def __init__(self, A, B, C, n: tuple[int, int, int], gemm: Gemm, group=None,
                 chunk: int = 8):
        self.A, self.B, self.C = A, B, C
        self.nt = A.shape[0]
        self.n = n
        self.gemm = gemm
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.chunk = max(1, min(chunk, self.nt))
        self.zb = [slab_bounds(n[2], r, self.world) for r in range(self.world)]
        self.xb = [slab_bounds(n[0], r, self.world) for r in range(self.world)]
        self.choice = None
        self.timings: dict[str, float] = {}

    # local passes A (x) and B (y) of one term on a [n0][n1][nz] block
    def _ab(self, x: torch.Tensor, t: int, nz: int) -> torch.Tensor:
        n0, n1, _ = self.n
        t1 = torch.empty(n1 * nz, n0, dtype=x.dtype, device=x.device)
        self.gemm(x.reshape(n0, n1 * nz), self.A[t], t1, False)          # [n1][nz][n0]
        t2 = torch.empty(nz * n0, n1, dtype=x.dtype, device=x.device)
        self.gemm(t1.reshape(n1, nz * n0), self.B[t], t2, False)         # [nz][n0][n1]
        return t2

    def _reduce_scatter_z(self, y_full: torch.Tensor) -> torch.Tensor:
        """Sum [n0*n1][n2] partials over ranks; rank r keeps z in slab r."""
        n0, n1, n2 = self.n
        chunks = [y_full[:, lo:hi].contiguous() for lo, hi in self.zb]
        lo, hi = self.zb[self.rank]
        out = torch.empty(n0 * n1, hi - lo, dtype=y_full.dtype, device=y_full.device)
        if self.world == 1:
            out.copy_(chunks[0])
        elif all(c.numel() == chunks[0].numel() for c in chunks) and y_full.is_cuda:
            dist.reduce_scatter(out, chunks, group=self.group)
        else:  # uneven slabs / gloo: all-reduce then slice
            dist.all_reduce(y_full, group=self.group)
            out.copy_(y_full[:, lo:hi])
        return out.reshape(n0, n1, hi - lo)

    def reduce_scatter(self, x_local: torch.Tensor) -> torch.Tensor:
        """(c): z contracted last from the local z-slice into full-length
        partial sums over all terms (term-concatenated K), one reduce-scatter."""
        n0, n1, n2 = self.n
        lo, hi = self.zb[self.rank]
        nz = hi - lo
        y = torch.zeros(n0 * n1, n2, dtype=x_local.dtype, device=x_local.device)
        for r0 in range(0, self.nt, self.chunk):
            cr = min(self.chunk, self.nt - r0)
            t2 = torch.stack([self._ab(x_local, r0 + r, nz) for r in range(cr)])  # [cr][nz][n0 n1]
            ccat = self.C[r0:r0 + cr, :, lo:hi].permute(1, 0, 2).reshape(n2, cr * nz).contiguous()
            if nz > 0:
                self.gemm(t2.reshape(cr * nz, n0 * n1), ccat, y, True)
        return self._reduce_scatter_z(y)

    def rank_split(self, x_local: torch.Tensor) -> torch.Tensor:
        """(b): all-gather the mesh, each rank applies its share of the terms
        on the full mesh, reduce-scatter the partial sums along z."""
        n0, n1, n2 = self.n
        parts = [torch.empty(n0, n1, hi - lo, dtype=x_local.dtype, device=x_local.device)
                 for lo, hi in self.zb]
        if self.world > 1:
            dist.all_gather(parts, x_local.contiguous(), group=self.group)
        else:
            parts[0].copy_(x_local)
        x = torch.cat(parts, dim=2).contiguous()
        y = torch.zeros(n0 * n1, n2, dtype=x.dtype, device=x.device)
        mine = list(range(self.rank, self.nt, self.world))
        for i in range(0, len(mine), self.chunk):
            ts = mine[i:i + self.chunk]
            t2 = torch.stack([self._ab(x, t, n2) for t in ts])
            ccat = self.C[ts].permute(1, 0, 2).reshape(n2, len(ts) * n2).contiguous()
            self.gemm(t2.reshape(len(ts) * n2, n0 * n1), ccat, y, True)
        return self._reduce_scatter_z(y)

    def alltoall(self, x_local: torch.Tensor) -> torch.Tensor:
        """(a): per-term x, y products on the z-slab, all-to-all transpose to
        x-slabs, term-concatenated z product, all-to-all back."""
        n0, n1, n2 = self.n
        lo, hi = self.zb[self.rank]
        nz = hi - lo
        xlo, xhi = self.xb[self.rank]
        nxl = xhi - xlo
        y_x = torch.zeros(nxl * n1, n2, dtype=x_local.dtype, device=x_local.device)
        for r0 in range(0, self.nt, self.chunk):
            cr = min(self.chunk, self.nt - r0)
            t2 = torch.stack([self._ab(x_local, r0 + r, nz) for r in range(cr)])  # [cr][nz][n0][n1]
            t2 = t2.reshape(cr, nz, n0, n1)
            send = torch.cat([t2[:, :, a:b, :].reshape(-1) for a, b in self.xb])
            recv_sizes = [cr * (zh - zl) * nxl * n1 for zl, zh in self.zb]
            send_sizes = [cr * nz * (b - a) * n1 for a, b in self.xb]
            recv = torch.empty(sum(recv_sizes), dtype=x_local.dtype, device=x_local.device)
            if self.world > 1:
                dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=self.group)
            else:
                recv.copy_(send)
            blocks = []
            off = 0
            for (zl, zh), sz in zip(self.zb, recv_sizes):
                blocks.append(recv[off:off + sz].reshape(cr, zh - zl, nxl * n1))
                off += sz
            t2x = torch.cat(blocks, dim=1).contiguous()                 # [cr][n2][nxl n1]
            ccat = self.C[r0:r0 + cr].permute(1, 0, 2).reshape(n2, cr * n2).contiguous()
            self.gemm(t2x.reshape(cr * n2, nxl * n1), ccat, y_x, True)
        # back to z-slabs: rank s receives [x in slab r][y][z in slab s] from every r
        y3 = y_x.reshape(nxl, n1, n2)
        send = torch.cat([y3[:, :, zl:zh].reshape(-1) for zl, zh in self.zb])
        send_sizes = [nxl * n1 * (zh - zl) for zl, zh in self.zb]
        recv_sizes = [(b - a) * n1 * nz for a, b in self.xb]
        recv = torch.empty(sum(recv_sizes), dtype=x_local.dtype, device=x_local.device)
        if self.world > 1:
            dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=self.group)
        else:
            recv.copy_(send)
        blocks = []
        off = 0
        for (a, b), sz in zip(self.xb, recv_sizes):
            blocks.append(recv[off:off + sz].reshape(b - a, n1, nz))
            off += sz
        return torch.cat(blocks, dim=0).contiguous()

    def apply(self, x_local: torch.Tensor, strategy: str | None = None) -> torch.Tensor:
        s = strategy or self.choice or "reduce_scatter"
        return getattr(self, s)(x_local)

    def choose(self, x_local: torch.Tensor, reps: int = 1) -> str:
        """Time every strategy once per shape (max over ranks) and keep the
        fastest -- the north star's 'faster of the two is chosen per shape'."""
        for s in self.STRATEGIES:
            self.apply(x_local, s)  # warm
            if x_local.is_cuda:
                torch.cuda.synchronize()
            if dist.is_initialized():
                dist.barrier(group=self.group)
            t0 = time.perf_counter()
            for _ in range(reps):
                self.apply(x_local, s)
            if x_local.is_cuda:
                torch.cuda.synchronize()
            dt = torch.tensor([(time.perf_counter() - t0) / reps], dtype=torch.float64)
            if dist.is_initialized() and self.world > 1:
                dt = dt.to(x_local.device)
                dist.all_reduce(dt, op=dist.ReduceOp.MAX, group=self.group)
            self.timings[s] = float(dt.item())
        self.choice = min(self.timings, key=self.timings.get)
        return self.choice

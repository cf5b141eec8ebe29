"""Steady-state plan API over torch device tensors (kpme_gpu_plan_*).

torch supplies device memory and streams; every kernel is ours
(libkpme_b200.so). Each plan runs on its own stream, ordered against the
caller's current stream on entry and exit of every call.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .api import CellGrid, EwaldConfig, KpmeOptions, SkpDecomposition, make_config


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda or t.dtype != torch.float64 and t.dtype != torch.int32:
        raise ValueError("kpme_gpu: expected a CUDA float64/int32 tensor")
    if not t.is_contiguous():
        raise ValueError("kpme_gpu: expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


class KpmePlan:
    """Plan for repeated kpme_apply calls on one cell grid and decomposition.

    The plan runs on its own torch stream (``self.stream``); every call first
    makes that stream wait for the caller's current stream and afterwards
    makes the caller's stream wait for it, so results order with surrounding
    torch work while graph capture stays possible."""

    def __init__(self, cfg: EwaldConfig, grid: CellGrid, order: int, dec: SkpDecomposition,
                 max_particles: int, opt: KpmeOptions | None = None, device: int = 0,
                 formulation: str = "auto", slab: tuple | None = None,
                 block: tuple | None = None):
        if dec.modes != cfg.modes:
            raise ValueError("kpme_apply: decomposition mode bound mismatch")
        self.cfg, self.grid, self.order, self.dec = cfg, grid, order, dec
        self.device = device
        self.max_particles = int(max_particles)
        self._c, self._keep = make_config(cfg, grid, order, dec, opt, device, formulation)
        self._h = C.c_void_p()
        self.slab, self.block = slab, block
        with torch.cuda.device(device):
            if block is not None:
                # cell block ((lo0, hi0), (lo1, hi1), (lo2, hi2)) of a rank grid
                lo = (C.c_int * 3)(*[int(b[0]) for b in block])
                hi = (C.c_int * 3)(*[int(b[1]) for b in block])
                check(lib.kpme_gpu_plan_create_block(C.byref(self._c), self.max_particles, lo, hi,
                                                     C.byref(self._h)))
            elif slab is None:
                check(lib.kpme_gpu_plan_create(C.byref(self._c), self.max_particles,
                                               C.byref(self._h)))
            else:
                check(lib.kpme_gpu_plan_create_slab(C.byref(self._c), self.max_particles,
                                                    int(slab[0]), int(slab[1]), C.byref(self._h)))
        self.stream = torch.cuda.Stream(device=device)
        check(lib.kpme_gpu_plan_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))

    def _enter(self):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def _leave(self):
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def close(self):
        if self._h:
            lib.kpme_gpu_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ncell(self) -> int:
        return self.grid.cell_count()

    @property
    def grid_size(self) -> int:
        return self.order ** 3

    # ---- full pipeline --------------------------------------------------
    def execute(self, xyz: torch.Tensor, q: torch.Tensor, out: torch.Tensor | None = None,
                defer_checks: bool = False) -> torch.Tensor:
        n = xyz.shape[0]
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=xyz.device)
        flags = _lib.DEFER_CHECKS if defer_checks else 0
        self._enter()
        check(lib.kpme_gpu_plan_execute_device(self._h, n, _ptr(xyz), _ptr(q), _ptr(out), flags))
        self._leave()
        return out

    def execute_graph(self, xyz: torch.Tensor, q: torch.Tensor, out: torch.Tensor,
                      sync_caller: bool = True):
        """Replay the captured pipeline (captured on first use / new pointers)."""
        if sync_caller:
            self._enter()
        check(lib.kpme_gpu_plan_graph_execute(self._h, xyz.shape[0], _ptr(xyz), _ptr(q),
                                              _ptr(out)))
        if sync_caller:
            self._leave()
        return out

    def execute_host(self, xyz: np.ndarray, q: np.ndarray, out: np.ndarray | None = None):
        """Host buffers (pinned or pageable); H2D/D2H inside the call."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = xyz.shape[0]
        if out is None:
            out = np.zeros(max(n, 1))
        dp = C.POINTER(C.c_double)
        self._enter()
        check(lib.kpme_gpu_plan_execute(self._h, n, xyz.ctypes.data_as(dp), q.ctypes.data_as(dp),
                                        out.ctypes.data_as(dp)))
        return out[:n]

    def set_host_chunks(self, chunks: int):
        """Particle chunks of the pipelined host path (-1 automatic, 1 off)."""
        check(lib.kpme_gpu_plan_set_host_chunks(self._h, int(chunks)))

    def execute_host_ptr(self, n: int, xyz_ptr: int, q_ptr: int, out_ptr: int):
        """Host-pointer variant for pinned torch CPU tensors."""
        dp = C.POINTER(C.c_double)
        self._enter()
        check(lib.kpme_gpu_plan_execute(self._h, n, C.cast(xyz_ptr, dp), C.cast(q_ptr, dp),
                                        C.cast(out_ptr, dp)))

    # ---- slab halves (multi-GPU) ----------------------------------------
    def core_size(self) -> int:
        return int(lib.kpme_gpu_plan_core_size(self._h))

    def forward(self, xyz: torch.Tensor, q: torch.Tensor, core: torch.Tensor) -> torch.Tensor:
        """This slab's partial R^3 + 1 core (last entry: local sum of q)."""
        self._enter()
        check(lib.kpme_gpu_plan_forward(self._h, xyz.shape[0], _ptr(xyz), _ptr(q), _ptr(core)))
        self._leave()
        return core

    def backward(self, core: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """Potentials of this slab's particles from the rank-summed core."""
        self._enter()
        check(lib.kpme_gpu_plan_backward(self._h, _ptr(core), _ptr(out)))
        self._leave()
        return out

    def attach_comm(self, nranks: int, rank: int, uid: bytes):
        """Own an NCCL communicator (rank ``rank`` of ``nranks``; ``uid`` from
        ``nccl_unique_id()`` on rank 0, broadcast by the job). Afterwards
        ``execute``/``execute_graph`` sum the partial cores of all ranks
        inside the library: forward half -> ncclAllReduce -> backward half."""
        if len(uid) != _lib.NCCL_ID_BYTES:
            raise ValueError("kpme_gpu: NCCL unique id must be 128 bytes")
        buf = C.create_string_buffer(bytes(uid), _lib.NCCL_ID_BYTES)
        with torch.cuda.device(self.device):
            check(lib.kpme_gpu_plan_attach_comm(self._h, int(nranks), int(rank), buf))

    def status(self):
        check(lib.kpme_gpu_plan_status(self._h))

    def launches(self) -> int:
        return lib.kpme_gpu_plan_launches(self._h)

    def enable_timing(self, on: bool = True):
        check(lib.kpme_gpu_plan_enable_timing(self._h, int(on)))

    def stage_times(self):
        buf = (C.c_double * 16)()
        cnt = C.c_int()
        check(lib.kpme_gpu_plan_stage_times(self._h, buf, 16, C.byref(cnt)))
        return list(buf[: cnt.value])

    # ---- stages ---------------------------------------------------------
    def sort(self, xyz: torch.Tensor):
        """assign_particles (geometry.hpp:131-154): (perm, cell_start)."""
        n = xyz.shape[0]
        perm = torch.empty(max(n, 1), dtype=torch.int32, device=xyz.device)
        start = torch.empty(self.ncell + 1, dtype=torch.int32, device=xyz.device)
        self._enter()
        check(lib.kpme_gpu_sort(self._h, n, _ptr(xyz), _ptr(perm), _ptr(start)))
        self._leave()
        return perm[:n], start

    def spread(self, xyz: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
        """InterpOperator::interpolate (interpolation.hpp:84-92): [ncell, L^3]."""
        phi = torch.empty(self.ncell, self.grid_size, dtype=torch.float64, device=xyz.device)
        self._enter()
        check(lib.kpme_gpu_spread(self._h, xyz.shape[0], _ptr(xyz), _ptr(q), _ptr(phi)))
        self._leave()
        return phi

    def skp_apply(self, phi: torch.Tensor) -> torch.Tensor:
        """spkmv_sum over all terms (parallel.hpp:184-228)."""
        psi = torch.empty_like(phi)
        self._enter()
        check(lib.kpme_gpu_skp_apply(self._h, _ptr(phi.contiguous()), _ptr(psi)))
        self._leave()
        return psi

    def gather(self, xyz: torch.Tensor, psi: torch.Tensor) -> torch.Tensor:
        """InterpOperator::anterpolate (interpolation.hpp:95-105)."""
        out = torch.empty(xyz.shape[0], dtype=torch.float64, device=xyz.device)
        self._enter()
        check(lib.kpme_gpu_gather(self._h, xyz.shape[0], _ptr(xyz), _ptr(psi.contiguous()),
                                  _ptr(out)))
        self._leave()
        return out

    def axis_operands(self, axis: int) -> torch.Tensor:
        """Dense A_a(lambda) = W_a^T diag(d) W_a for every term: [nterms, n_a, n_a]."""
        n = self.grid.counts[axis] * self.order
        out = torch.empty(max(len(self.dec.terms), 1), n, n, dtype=torch.float64,
                          device=f"cuda:{self.device}")
        self._enter()
        check(lib.kpme_gpu_plan_axis_operands(self._h, axis, _ptr(out)))
        self._leave()
        return out[: len(self.dec.terms)]


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (128 bytes)."""
    buf = C.create_string_buffer(_lib.NCCL_ID_BYTES)
    check(lib.kpme_gpu_nccl_unique_id(buf))
    return buf.raw


class MultiDevicePlan:
    """One process driving several GPUs (kpme_gpu_plan_create_multi): a
    P0 x P1 x P2 grid of cell blocks, block r on ``devices[r]`` (RankGrid,
    parallel.hpp:46-82). Inputs and outputs live on the home device
    ``devices[0]`` (or on the host for ``execute_host``); the partial cores
    are summed from peer memory (``collective="peer"``) or by NCCL."""

    _COLL = {"auto": _lib.COLL_AUTO, "peer": _lib.COLL_PEER, "nccl": _lib.COLL_NCCL}

    def __init__(self, cfg: EwaldConfig, grid: CellGrid, order: int, dec: SkpDecomposition,
                 max_particles: int, devices, dims=None, opt: KpmeOptions | None = None,
                 collective: str = "auto"):
        devices = [int(d) for d in devices]
        self.cfg, self.grid, self.order, self.dec = cfg, grid, order, dec
        self.devices = devices
        self.device = devices[0]
        self.dims = tuple(dims) if dims is not None else (1, 1, len(devices))
        self._c, self._keep = make_config(cfg, grid, order, dec, opt, devices[0], "collapsed")
        dv = (C.c_int * len(devices))(*devices)
        self._keep.append(dv)
        self._c.ndevices, self._c.devices = len(devices), C.cast(dv, C.POINTER(C.c_int))
        self._h = C.c_void_p()
        d3 = (C.c_int * 3)(*self.dims)
        with torch.cuda.device(self.device):
            check(lib.kpme_gpu_plan_create_multi(C.byref(self._c), int(max_particles), d3,
                                                 C.byref(self._h)))
        if collective != "auto":
            self.set_collective(collective)
        self.stream = torch.cuda.Stream(device=self.device)
        check(lib.kpme_gpu_plan_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))

    def set_collective(self, mode: str):
        check(lib.kpme_gpu_plan_set_collective(self._h, self._COLL[mode]))

    @property
    def collective(self) -> str:
        return {v: k for k, v in self._COLL.items()}[lib.kpme_gpu_plan_collective(self._h)]

    def execute(self, xyz: torch.Tensor, q: torch.Tensor, out: torch.Tensor | None = None,
                defer_checks: bool = False) -> torch.Tensor:
        n = xyz.shape[0]
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=xyz.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        check(lib.kpme_gpu_plan_execute_device(self._h, n, _ptr(xyz), _ptr(q), _ptr(out),
                                               _lib.DEFER_CHECKS if defer_checks else 0))
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return out

    def execute_host(self, xyz: np.ndarray, q: np.ndarray, out: np.ndarray | None = None):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = xyz.shape[0]
        if out is None:
            out = np.zeros(max(n, 1))
        dp = C.POINTER(C.c_double)
        check(lib.kpme_gpu_plan_execute(self._h, n, xyz.ctypes.data_as(dp), q.ctypes.data_as(dp),
                                        out.ctypes.data_as(dp)))
        return out[:n]

    def execute_host_ptr(self, n: int, xyz_ptr: int, q_ptr: int, out_ptr: int):
        dp = C.POINTER(C.c_double)
        check(lib.kpme_gpu_plan_execute(self._h, n, C.cast(xyz_ptr, dp), C.cast(q_ptr, dp),
                                        C.cast(out_ptr, dp)))

    def status(self):
        check(lib.kpme_gpu_plan_status(self._h))

    def launches(self) -> int:
        return lib.kpme_gpu_plan_launches(self._h)

    def close(self):
        if self._h:
            lib.kpme_gpu_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kron_matvec_dense(A: torch.Tensor, B: torch.Tensor, C_: torch.Tensor, x: torch.Tensor,
                      out: torch.Tensor | None = None, workspace: torch.Tensor | None = None):
    """y = sum_r (A_r (x) B_r (x) C_r) x on the lexicographic mesh x[n0, n1, n2]
    (kron_matvec_shuffle, kron.hpp:180-197, summed over terms) on FP64 DMMA."""
    nt, n0, _ = A.shape
    n1, n2 = B.shape[1], C_.shape[1]
    if out is None:
        out = torch.empty(n0, n1, n2, dtype=torch.float64, device=x.device)
    ws, wsb = None, 0
    if workspace is not None:
        ws, wsb = _ptr(workspace), workspace.numel() * workspace.element_size()
    s = torch.cuda.current_stream(x.device)
    check(lib.kpme_gpu_kron_matvec_dense(x.device.index or 0, C.c_void_p(s.cuda_stream), n0, n1,
                                         n2, nt, _ptr(A.contiguous()), _ptr(B.contiguous()),
                                         _ptr(C_.contiguous()), _ptr(x.contiguous()), _ptr(out),
                                         ws, wsb))
    return out


class DenseSlab:
    """Config 5 on z-slabs through the library (kpme_gpu_dense_slab_*): the
    dense operator y = sum_r (A_r (x) B_r (x) C_r) x with x, y as z-slabs
    [n0][n1][z_hi - z_lo], one rank per GPU, the three sharded-axis
    strategies (``_lib.SLAB_STRATEGIES``) on the DMMA GEMM with the library's
    own NCCL communicator and preallocated buffers.

    ``DenseSlab(A, B, C, nranks, rank, nccl_id)``: this process's rank
    (A, B, C: full [nterms][n][n] operands on its GPU).
    ``DenseSlab.group(ops_per_rank, devices)``: every rank in this process
    (devices may repeat; collectives by peer copies in rank order)."""

    def __init__(self, A=None, B=None, C_=None, nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, _group=None):
        self._h = C.c_void_p()
        if _group is not None:
            ops, devices = _group
            self.local = len(devices)
            self.nranks, self.devices = len(devices), list(devices)
            A0 = ops[0][0]
            self.shape = (A0.shape[1], ops[0][1].shape[1], ops[0][2].shape[1])
            self.nterms = A0.shape[0]
            self._keep = [o.contiguous() for trio in ops for o in trio]
            P = C.c_void_p
            arr = lambda k: (P * self.nranks)(*[_ptr(ops[r][k].contiguous()) for r in range(self.nranks)])
            self._arrs = [arr(0), arr(1), arr(2)]
            dv = (C.c_int * self.nranks)(*self.devices)
            check(lib.kpme_gpu_dense_slab_create_group(self.nranks, dv, *self.shape, self.nterms,
                                                       *self._arrs, C.byref(self._h)))
        else:
            self.local, self.nranks = 1, int(nranks)
            self.devices = [A.device.index or 0]
            self.shape = (A.shape[1], B.shape[1], C_.shape[1])
            self.nterms = A.shape[0]
            self._keep = [A.contiguous(), B.contiguous(), C_.contiguous()]
            buf = None
            if nccl_id is not None:
                buf = C.create_string_buffer(bytes(nccl_id), _lib.NCCL_ID_BYTES)
            with torch.cuda.device(self.devices[0]):
                check(lib.kpme_gpu_dense_slab_create(self.devices[0], *self.shape, self.nterms,
                                                     *[_ptr(t) for t in self._keep], self.nranks,
                                                     int(rank), buf, C.byref(self._h)))
        self.rank = int(rank)

    @classmethod
    def group(cls, ops_per_rank, devices):
        return cls(_group=(ops_per_rank, devices))

    def bounds(self, rank: int):
        lo, hi = C.c_int(), C.c_int()
        check(lib.kpme_gpu_dense_slab_bounds(self._h, int(rank), C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def _ptrs(self, ts):
        return (C.c_void_p * len(ts))(*[_ptr(t) for t in ts])

    def apply(self, x_local, y_local, strategy: str = "reduce_scatter", sync: bool = True):
        """x_local, y_local: one tensor per local rank (lists), or a tensor."""
        xs = x_local if isinstance(x_local, (list, tuple)) else [x_local]
        ys = y_local if isinstance(y_local, (list, tuple)) else [y_local]
        torch.cuda.synchronize()
        check(lib.kpme_gpu_dense_slab_apply(self._h, _lib.SLAB_STRATEGIES.index(strategy),
                                            self._ptrs(xs), self._ptrs(ys)))
        if sync:
            check(lib.kpme_gpu_dense_slab_sync(self._h))
        return y_local

    def choose(self, x_local, y_local, reps: int = 1):
        """Per-strategy time (ms per apply, CUDA events, max over ranks) and
        the fastest strategy for this shape."""
        xs = x_local if isinstance(x_local, (list, tuple)) else [x_local]
        ys = y_local if isinstance(y_local, (list, tuple)) else [y_local]
        torch.cuda.synchronize()
        ms = (C.c_double * 3)()
        best = C.c_int()
        check(lib.kpme_gpu_dense_slab_choose(self._h, self._ptrs(xs), self._ptrs(ys), int(reps), ms,
                                             C.byref(best)))
        return {s: ms[i] for i, s in enumerate(_lib.SLAB_STRATEGIES)}, _lib.SLAB_STRATEGIES[best.value]

    def close(self):
        if self._h:
            lib.kpme_gpu_dense_slab_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dense_workspace_bytes(n0: int, n1: int, n2: int, nterms: int) -> int:
    return int(lib.kpme_gpu_dense_workspace_bytes(n0, n1, n2, nterms))


def dgemm_tn(inp: torch.Tensor, F: torch.Tensor, out: torch.Tensor, accumulate=False):
    """out[m][i] (+)= sum_k inp[k][m] F[i][k] on the DMMA GEMM kernel."""
    K, M = inp.shape
    N = F.shape[0]
    s = torch.cuda.current_stream(inp.device)
    check(lib.kpme_gpu_dgemm_tn(C.c_void_p(s.cuda_stream), M, N, K, _ptr(inp), _ptr(F),
                                _ptr(out), int(accumulate)))
    return out

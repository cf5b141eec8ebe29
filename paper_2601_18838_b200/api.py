"""Host-side mirror of the reference's C++ API for the SKP-PME reciprocal path.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/kpme/ (cited per item), so code and tests written
against the reference read the same here. All compute goes through the C ABI
of libkpme_b200.so (include/kpme_gpu.h); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from ._lib import check, lib

_dp = C.POINTER(C.c_double)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ---- geometry.hpp -------------------------------------------------------------

@dataclass
class Box3:
    """Cubic box of half edge ``radius`` (geometry.hpp:26-41)."""

    center: tuple = (0.0, 0.0, 0.0)
    radius: float = 1.0

    def __post_init__(self):
        self.center = tuple(float(c) for c in self.center)
        if not (self.radius > 0.0):
            raise ValueError("Box3: radius must be positive")

    def contains(self, p) -> bool:
        return all(abs(p[a] - self.center[a]) <= self.radius for a in range(3))


@dataclass
class CellGrid:
    """K0 x K1 x K2 cell decomposition (geometry.hpp:63-111)."""

    box: Box3
    counts: tuple = (1, 1, 1)

    def cell_count(self) -> int:
        return self.counts[0] * self.counts[1] * self.counts[2]

    def flatten(self, c) -> int:
        return (c[0] * self.counts[1] + c[1]) * self.counts[2] + c[2]

    def unflatten(self, idx: int):
        c2 = idx % self.counts[2]
        idx //= self.counts[2]
        return (idx // self.counts[1], idx % self.counts[1], c2)

    def cell_radius(self, axis: int) -> float:
        return self.box.radius / self.counts[axis]

    def max_cell_radius(self) -> float:
        return max(self.cell_radius(a) for a in range(3))

    def axis_lo(self, axis: int, idx: int) -> float:
        return self.box.center[axis] - self.box.radius + 2.0 * self.box.radius * idx / self.counts[axis]

    def axis_hi(self, axis: int, idx: int) -> float:
        return (self.box.center[axis] - self.box.radius
                + 2.0 * self.box.radius * (idx + 1) / self.counts[axis])

    def axis_nodes(self, axis: int, idx: int, order: int):
        if order < 2:
            raise ValueError("CellGrid: interpolation order must be >= 2")
        a, b = self.axis_lo(axis, idx), self.axis_hi(axis, idx)
        return [a + (b - a) * k / (order - 1) for k in range(order)]


def build_cell_grid(box: Box3, counts) -> CellGrid:
    """geometry.hpp:113-122."""
    if isinstance(counts, int):
        counts = (counts, counts, counts)
    counts = tuple(int(c) for c in counts)
    if any(c < 1 for c in counts):
        raise ValueError("build_cell_grid: cell counts must be >= 1")
    return CellGrid(box, counts)


@dataclass
class ConvergenceCheck:
    nu: float = 0.0
    ok: bool = False


def check_convergence_ratio(grid: CellGrid, modes: int) -> ConvergenceCheck:
    """nu = pi M r_c (geometry.hpp:158-170)."""
    if modes < 1:
        raise ValueError("check_convergence_ratio: modes must be >= 1")
    nu = math.pi * modes * grid.max_cell_radius()
    return ConvergenceCheck(nu, nu < 1.0)


@dataclass
class PointCloud:
    positions: np.ndarray  # (n, 3) float64, AoS like std::vector<Vec3>

    def size(self) -> int:
        return int(self.positions.shape[0])


@dataclass
class ChargeVector:
    values: np.ndarray

    def size(self) -> int:
        return int(self.values.shape[0])


@dataclass
class CloudData:
    cloud: PointCloud
    charges: ChargeVector


def sample_cloud(box: Box3, n: int, seed: int) -> CloudData:
    """Uniform positions, charges in [-1, 1], splitmix64 (geometry.hpp:238-251)."""
    xyz = np.zeros((n, 3))
    q = np.zeros(n)
    lib.kpme_sample_cloud((C.c_double * 3)(*box.center), box.radius, n, seed, _d(xyz), _d(q))
    return CloudData(PointCloud(xyz), ChargeVector(q))


def write_cloud(path: str, data: CloudData):
    """Point-cloud text format, precision 17 (geometry.hpp:199-207)."""
    with open(path, "w") as f:
        f.write(f"{data.cloud.size()}\n")
        for p, q in zip(data.cloud.positions, data.charges.values):
            f.write(f"{p[0]:.17g} {p[1]:.17g} {p[2]:.17g} {q:.17g}\n")


def read_cloud(path: str) -> CloudData:
    """geometry.hpp:181-197."""
    try:
        with open(path) as f:
            tok = f.read().split()
    except OSError as e:
        raise RuntimeError(f"read_cloud: cannot open {path}") from e
    if not tok:
        raise RuntimeError("read_cloud: missing particle count")
    n = int(tok[0])
    if len(tok) < 1 + 4 * n:
        raise RuntimeError(f"read_cloud: malformed line {(len(tok) - 1) // 4 + 2}")
    a = np.array(tok[1:1 + 4 * n], dtype=np.float64).reshape(n, 4)
    return CloudData(PointCloud(np.ascontiguousarray(a[:, :3])), ChargeVector(a[:, 3].copy()))


# ---- alpha.hpp ---------------------------------------------------------------

@dataclass
class EwaldConfig:
    """alpha.hpp:20-31."""

    xi: float = 1.0
    modes: int = 1

    def __post_init__(self):
        if not (self.xi > 0.0):
            raise ValueError("EwaldConfig: xi must be positive")
        if self.modes < 1:
            raise ValueError("EwaldConfig: modes must be >= 1")

    def mode_range(self) -> int:
        return 2 * self.modes + 1


def alpha_weight(cfg: EwaldConfig, m0: int, m1: int, m2: int) -> float:
    """alpha.hpp:34-39."""
    r2 = float(m0) * m0 + float(m1) * m1 + float(m2) * m2
    if r2 == 0.0:
        return 0.0
    p = math.pi / cfg.xi
    return math.exp(-p * p * r2) / r2


class SkpKind(Enum):
    svd = 0
    sinc = 1
    tabulated = 2


@dataclass
class SkpTerm:
    """omega * p0 (x) p1 (x) p2, profiles over m = -M..M (alpha.hpp:69-73)."""

    weight: float
    profiles: tuple  # 3 arrays of length 2M+1


@dataclass
class SkpDecomposition:
    """alpha.hpp:75-80."""

    kind: SkpKind = SkpKind.sinc
    modes: int = 0
    correction: float = 0.0
    terms: list = field(default_factory=list)

    def arrays(self):
        """(weights[nterms], profiles[nterms][3][2M+1]) in the ABI layout."""
        P = 2 * self.modes + 1
        w = np.array([t.weight for t in self.terms], dtype=np.float64)
        prof = np.zeros((len(self.terms), 3, P))
        for i, t in enumerate(self.terms):
            for a in range(3):
                prof[i, a] = t.profiles[a]
        return w, prof

    def truncated(self, nterms: int) -> "SkpDecomposition":
        """``dec.terms.resize(n)`` as the reference tests do (test_parallel.cpp:305)."""
        return SkpDecomposition(self.kind, self.modes, self.correction, list(self.terms[:nterms]))


@dataclass
class QuadratureRule:
    """alpha.hpp:86-96."""

    nodes: np.ndarray
    weights: np.ndarray
    lifting: float = 0.0
    half_width: int = 0
    min_arg: float = 1.0
    max_arg: float = 1.0
    eps: float = 0.0

    def covers(self, lo: float, hi: float) -> bool:
        return self.min_arg <= lo and self.max_arg >= hi


def sinc_rule(n_quad: int, modes: int) -> QuadratureRule:
    """alpha.hpp:114-151."""
    cnt = 2 * n_quad + 1 if n_quad >= 1 else 1
    nodes, weights = np.zeros(cnt), np.zeros(cnt)
    h, e = C.c_double(), C.c_double()
    check(lib.kpme_sinc_rule(n_quad, modes, _d(nodes), _d(weights), C.byref(h), C.byref(e)))
    return QuadratureRule(nodes, weights, h.value, n_quad, 1.0, 3.0 * modes * modes, e.value)


def sinc_rule_for_eps(eps: float, modes: int, max_n: int = 400) -> QuadratureRule:
    """alpha.hpp:154-161."""
    cap = 2 * max_n + 1
    nodes, weights = np.zeros(cap), np.zeros(cap)
    nq = C.c_int()
    h, e = C.c_double(), C.c_double()
    check(lib.kpme_sinc_rule_for_eps(eps, modes, max_n, C.byref(nq), _d(nodes), _d(weights),
                                     C.byref(h), C.byref(e)))
    cnt = 2 * nq.value + 1
    return QuadratureRule(nodes[:cnt].copy(), weights[:cnt].copy(), h.value, nq.value, 1.0,
                          3.0 * modes * modes, e.value)


@dataclass
class AlphaVector:
    """alpha.hpp:42-52: alpha(m) on [-M, M]^3, m0 slowest."""

    modes: int
    entries: np.ndarray

    def at(self, m0: int, m1: int, m2: int) -> float:
        n = 2 * self.modes + 1
        return float(self.entries[((m0 + self.modes) * n + (m1 + self.modes)) * n
                                  + (m2 + self.modes)])


def assemble_alpha(cfg: EwaldConfig) -> AlphaVector:
    """alpha.hpp:54-65."""
    n = 2 * cfg.modes + 1
    out = np.zeros(n ** 3)
    check(lib.kpme_assemble_alpha(cfg.xi, cfg.modes, _d(out)))
    return AlphaVector(cfg.modes, out)


def nkpa_svd(alpha: AlphaVector, tol_outer: float, tol_inner: float):
    """nkpa_svd (alpha.hpp:225-281): SVD-kind SkpDecomposition of alpha by two
    nested truncated SVDs, and the a priori error bound. Raises ValueError
    for tol_inner > tol_outer (std::invalid_argument in the reference)."""
    n = 2 * alpha.modes + 1
    a = np.ascontiguousarray(alpha.entries, dtype=np.float64)
    cnt, bound = C.c_int(), C.c_double()
    check(lib.kpme_nkpa_svd(alpha.modes, _d(a), tol_outer, tol_inner, 0, C.byref(cnt), None, None,
                            C.byref(bound)))
    cap = max(cnt.value, 1)
    tw, prof = np.zeros(cap), np.zeros((cap, 3, n))
    check(lib.kpme_nkpa_svd(alpha.modes, _d(a), tol_outer, tol_inner, cap, C.byref(cnt), _d(tw),
                            _d(prof), C.byref(bound)))
    terms = [SkpTerm(float(tw[i]), (prof[i, 0].copy(), prof[i, 1].copy(), prof[i, 2].copy()))
             for i in range(cnt.value)]
    return SkpDecomposition(SkpKind.svd, alpha.modes, 0.0, terms), bound.value


def skp_from_quadrature(rule: QuadratureRule, cfg: EwaldConfig,
                        kind: SkpKind = SkpKind.sinc) -> SkpDecomposition:
    """alpha.hpp:165-188."""
    cnt = len(rule.nodes)
    P = 2 * cfg.modes + 1
    tw = np.zeros(max(cnt, 1))
    prof = np.zeros((max(cnt, 1), 3, P))
    corr = C.c_double()
    nodes = np.ascontiguousarray(rule.nodes, dtype=np.float64)
    weights = np.ascontiguousarray(rule.weights, dtype=np.float64)
    check(lib.kpme_skp_from_quadrature(cnt, _d(nodes), _d(weights), rule.min_arg, rule.max_arg,
                                       cfg.xi, cfg.modes, _d(tw), _d(prof), C.byref(corr)))
    terms = [SkpTerm(float(tw[i]), (prof[i, 0].copy(), prof[i, 1].copy(), prof[i, 2].copy()))
             for i in range(cnt)]
    return SkpDecomposition(kind, cfg.modes, corr.value, terms)


def load_tabulated_rule(path: str) -> QuadratureRule:
    """alpha.hpp:192-212."""
    cap = 4096
    nodes, weights = np.zeros(cap), np.zeros(cap)
    cnt = C.c_int()
    lo, hi, e = C.c_double(), C.c_double(), C.c_double()
    check(lib.kpme_load_tabulated_rule(path.encode(), cap, C.byref(cnt), _d(nodes), _d(weights),
                                       C.byref(lo), C.byref(hi), C.byref(e)))
    n = cnt.value
    return QuadratureRule(nodes[:n].copy(), weights[:n].copy(), 0.0, 0, lo.value, hi.value,
                          e.value)


# ---- parallel.hpp --------------------------------------------------------------

@dataclass
class KpmeOptions:
    """parallel.hpp:230-233 (threads is accepted and unused on the GPU)."""

    fuse_terms: bool = False
    threads: int = 1


@dataclass
class LedgerRow:
    rank: int = 0
    step: int = 0
    group_axis: int = -1
    payload: int = 0


class KpmeResult:
    """parallel.hpp:235-238: potentials in global particle order plus the
    logical message ledger (synthesised on first access)."""

    def __init__(self, potentials: np.ndarray, config: _lib.Config, keep):
        self.potentials = potentials
        self._cfg, self._keep = config, keep
        self._ledger = None

    @property
    def ledger_array(self) -> np.ndarray:
        if self._ledger is None:
            rows = C.c_int64()
            check(lib.kpme_gpu_ledger(C.byref(self._cfg), None, 0, C.byref(rows)))
            out = np.zeros((max(rows.value, 1), 4), np.int64)
            check(lib.kpme_gpu_ledger(C.byref(self._cfg), out.ctypes.data_as(_lib._i64p),
                                      rows.value, C.byref(rows)))
            self._ledger = out[: rows.value]
        return self._ledger

    @property
    def ledger(self):
        return [LedgerRow(*map(int, r)) for r in self.ledger_array]


def ledger_to_csv(rows, out) -> None:
    """parallel.hpp:91-96."""
    out.write("rank,step,group_axis,payload_count\n")
    for r in rows:
        out.write(f"{r.rank},{r.step},{r.group_axis},{r.payload}\n")


_FORMS = {"auto": _lib.FORM_AUTO, "collapsed": _lib.FORM_COLLAPSED, "dense": _lib.FORM_DENSE}


def make_config(cfg: EwaldConfig, grid: CellGrid, order: int, dec: SkpDecomposition,
                opt: KpmeOptions | None = None, device: int = 0, formulation: str = "auto",
                devices=None):
    """Marshal the reference's argument structs into kpme_gpu_config. Returns
    (config, keep-alive arrays). ``devices``: a device list (one process
    driving several GPUs: a multi-device plan of z-slabs)."""
    opt = opt or KpmeOptions()
    w, prof = dec.arrays()
    keep = [np.ascontiguousarray(w if len(w) else np.zeros(1)),
            np.ascontiguousarray(prof if len(w) else np.zeros(1))]
    c = _lib.Config()
    c.xi, c.modes = float(cfg.xi), int(cfg.modes)
    c.center = (C.c_double * 3)(*grid.box.center)
    c.radius = float(grid.box.radius)
    c.counts = (C.c_int * 3)(*grid.counts)
    c.order = int(order)
    c.dec_modes = int(dec.modes)
    c.correction = float(dec.correction)
    c.nterms = len(dec.terms)
    c.term_weights, c.profiles = _d(keep[0]), _d(keep[1])
    c.fuse_terms, c.threads = int(bool(opt.fuse_terms)), int(opt.threads)
    c.device = int(device)
    c.formulation = _FORMS[formulation]
    if devices is not None and len(devices) > 1:
        dv = (C.c_int * len(devices))(*[int(d) for d in devices])
        keep.append(dv)
        c.ndevices, c.devices = len(devices), C.cast(dv, C.POINTER(C.c_int))
        c.device = int(devices[0])
    return c, keep


def kpme_apply(cfg: EwaldConfig, grid: CellGrid, order: int, dec: SkpDecomposition,
               cloud: PointCloud, q: ChargeVector, opt: KpmeOptions | None = None, *,
               device: int = 0, formulation: str = "auto", devices=None) -> KpmeResult:
    """kpme_apply (parallel.hpp:243-290) on the GPU, host buffers in and out.
    Raises ValueError where the reference throws std::invalid_argument.
    ``devices`` (a list of ordinals) drives several GPUs from this process.
    Plans are cached per configuration inside the library (kpme_gpu_apply)."""
    if dec.modes != cfg.modes:
        raise ValueError("kpme_apply: decomposition mode bound mismatch")
    c, keep = make_config(cfg, grid, order, dec, opt, device, formulation, devices)
    xyz = np.ascontiguousarray(cloud.positions, dtype=np.float64).reshape(-1, 3)
    qv = np.ascontiguousarray(q.values, dtype=np.float64)
    if qv.shape[0] != xyz.shape[0]:
        raise ValueError("interpolate: charge count mismatch")
    out = np.zeros(max(xyz.shape[0], 1))
    check(lib.kpme_gpu_apply(C.byref(c), xyz.shape[0], _d(xyz), _d(qv), _d(out)))
    return KpmeResult(out[: xyz.shape[0]], c, keep)

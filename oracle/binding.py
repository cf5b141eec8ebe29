"""ctypes bindings to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two back ends with the same interface:

* ``CpuKpme("oracle")`` -> oracle/build/libkpme_oracle.so, the plain-C
  restatement of the reference path (oracle/kpme_oracle.c);
* ``CpuKpme("ref")``    -> oracle/_ref/libkpme_ref.so, the reference's own
  headers compiled here against the clean-room Eigen subset
  (oracle/ref/Makefile). Only exists where /root/reference was present at
  build time (it travels to the GPU box as a built file).
* ``CpuKpme("ref_o3")`` -> oracle/_ref/libkpme_ref_o3.so, the same shim at
  the reference's Release flags; the build bench.py times.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "oracle": (os.path.join(HERE, "build", "libkpme_oracle.so"), "ko_"),
    "ref": (os.path.join(HERE, "_ref", "libkpme_ref.so"), "kr_"),
    # the same shim at the reference's CMake Release flags (-O3 -DNDEBUG):
    # what bench.py times; "ref" (-O2 -ffp-contract=off) is the parity pin
    "ref_o3": (os.path.join(HERE, "_ref", "libkpme_ref_o3.so"), "kr_"),
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class ApplyArgs(C.Structure):
    """Mirror of ko_apply_args (oracle/kpme_oracle.h)."""

    _fields_ = [
        ("xi", C.c_double),
        ("modes", C.c_int),
        ("center", C.c_double * 3),
        ("radius", C.c_double),
        ("counts", C.c_int * 3),
        ("order", C.c_int),
        ("dec_modes", C.c_int),
        ("correction", C.c_double),
        ("nterms", C.c_int),
        ("term_weights", _dp),
        ("profiles", _dp),
        ("n", C.c_int64),
        ("pos", _dp),
        ("q", _dp),
        ("fuse_terms", C.c_int),
        ("threads", C.c_int),
    ]


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class Problem:
    """Flat description of one kpme_apply call (parallel.hpp:243-246)."""

    xi: float
    modes: int
    center: tuple
    radius: float
    counts: tuple
    order: int
    term_weights: np.ndarray   # [nterms]
    profiles: np.ndarray       # [nterms, 3, 2M+1]
    correction: float
    pos: np.ndarray            # [n, 3]
    q: np.ndarray              # [n]
    dec_modes: int | None = None


class CpuKpme:
    def __init__(self, which: str = "oracle"):
        path, self.pfx = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        self.which = which
        self.lib = C.CDLL(path)
        # attribute access caches the function object, so restype sticks
        self._f("last_error").restype = C.c_char_p
        self._f("alpha_weight").restype = C.c_double
        self._f("optimal_term_lower_bound").restype = C.c_longlong
        self._f("op_count_estimate").restype = C.c_longlong

    def _f(self, name):
        return getattr(self.lib, self.pfx + name)

    def _check(self, code: int):
        if code != 0:
            raise OracleError(code, self._f("last_error")().decode())

    # ---- geometry -------------------------------------------------------
    def sample_cloud(self, center, radius, n, seed):
        pos = np.zeros((n, 3))
        q = np.zeros(n)
        c = (C.c_double * 3)(*center)
        self._f("sample_cloud")(c, C.c_double(radius), C.c_int64(n), C.c_uint64(seed),
                                _d(pos), _d(q))
        return pos, q

    def assign_particles(self, center, radius, counts, pos):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        n = pos.shape[0]
        ncell = int(np.prod(counts))
        perm = np.zeros(max(n, 1), np.int32)
        start = np.zeros(ncell + 1, np.int32)
        c = (C.c_double * 3)(*center)
        k = (C.c_int * 3)(*counts)
        if self.which == "oracle":
            cell_of = np.zeros(max(n, 1), np.int32)
            bad = C.c_int64(-1)
            code = self._f("assign_particles")(c, C.c_double(radius), k, C.c_int64(n), _d(pos),
                                               cell_of.ctypes.data_as(_i32p),
                                               perm.ctypes.data_as(_i32p),
                                               start.ctypes.data_as(_i32p), C.byref(bad))
        else:
            code = self._f("assign_particles")(c, C.c_double(radius), k, C.c_int64(n), _d(pos),
                                               perm.ctypes.data_as(_i32p),
                                               start.ctypes.data_as(_i32p))
        self._check(code)
        return perm[:n], start

    # ---- alpha ----------------------------------------------------------
    def alpha_weight(self, xi, m0, m1, m2):
        return self._f("alpha_weight")(C.c_double(xi), m0, m1, m2)

    def optimal_term_lower_bound(self, eps):
        return int(self._f("optimal_term_lower_bound")(C.c_double(eps)))

    def sinc_rule(self, n_quad, modes):
        cnt = 2 * n_quad + 1
        nodes, weights = np.zeros(cnt), np.zeros(cnt)
        h, e = C.c_double(), C.c_double()
        self._check(self._f("sinc_rule")(n_quad, modes, _d(nodes), _d(weights),
                                         C.byref(h), C.byref(e)))
        return dict(nodes=nodes, weights=weights, lifting=h.value, eps=e.value,
                    half_width=n_quad, min_arg=1.0, max_arg=3.0 * modes * modes)

    def sinc_rule_for_eps(self, eps, modes, max_n=400):
        cap = 2 * max_n + 1
        nodes, weights = np.zeros(cap), np.zeros(cap)
        nq = C.c_int()
        h, e = C.c_double(), C.c_double()
        self._check(self._f("sinc_rule_for_eps")(C.c_double(eps), modes, max_n, C.byref(nq),
                                                 _d(nodes), _d(weights), C.byref(h),
                                                 C.byref(e)))
        cnt = 2 * nq.value + 1
        return dict(nodes=nodes[:cnt].copy(), weights=weights[:cnt].copy(), lifting=h.value,
                    eps=e.value, half_width=nq.value, min_arg=1.0,
                    max_arg=3.0 * modes * modes)

    def skp_from_quadrature(self, rule, xi, modes):
        cnt = len(rule["nodes"])
        P = 2 * modes + 1
        tw = np.zeros(max(cnt, 1))
        prof = np.zeros((max(cnt, 1), 3, P))
        corr = C.c_double()
        nodes = np.ascontiguousarray(rule["nodes"], dtype=np.float64)
        weights = np.ascontiguousarray(rule["weights"], dtype=np.float64)
        self._check(self._f("skp_from_quadrature")(
            cnt, _d(nodes), _d(weights), C.c_double(rule["min_arg"]),
            C.c_double(rule["max_arg"]), C.c_double(xi), modes, _d(tw), _d(prof),
            C.byref(corr)))
        return tw[:cnt], prof[:cnt], corr.value

    # ---- SVD kind (reference back ends only) ----------------------------
    def assemble_alpha(self, xi, modes):
        n = 2 * modes + 1
        out = np.zeros(n ** 3)
        self._check(self._f("assemble_alpha")(C.c_double(xi), modes, _d(out)))
        return out

    def nkpa_svd(self, alpha, modes, tol_outer, tol_inner):
        """(term_weights, profiles[nterms][3][2M+1], error_bound)."""
        n = 2 * modes + 1
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        cap = n * n + 1
        tw, prof = np.zeros(cap), np.zeros((cap, 3, n))
        cnt, bound = C.c_int(), C.c_double()
        self._check(self._f("nkpa_svd")(modes, _d(alpha), C.c_double(tol_outer),
                                        C.c_double(tol_inner), cap, C.byref(cnt), _d(tw),
                                        _d(prof), C.byref(bound)))
        return tw[:cnt.value].copy(), prof[:cnt.value].copy(), bound.value

    # ---- interpolation / symfourier -------------------------------------
    def lagrange_weights_1d(self, order, a, b, y):
        w = np.zeros(order)
        self._check(self._f("lagrange_weights_1d")(order, C.c_double(a), C.c_double(b),
                                                   C.c_double(y), _d(w)))
        return w

    def build_w(self, m, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        w = np.zeros((2, len(pts)))
        self._check(self._f("build_w")(m, len(pts), _d(pts), _d(w)))
        return w

    def build_uv(self, weight, profile, nodes, modes):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        profile = np.ascontiguousarray(profile, dtype=np.float64)
        L, R = len(nodes), 2 * (modes + 1)
        u, v = np.zeros((L, R)), np.zeros((R, L))
        self._check(self._f("build_uv")(C.c_double(weight), _d(profile), L, _d(nodes), modes,
                                        _d(u), _d(v)))
        return u, v

    # ---- kron -----------------------------------------------------------
    def kron_matvec_shuffle(self, factors, q):
        d = len(factors)
        facs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
        rows = (C.c_int * d)(*[f.shape[0] for f in facs])
        cols = (C.c_int * d)(*[f.shape[1] for f in facs])
        ptrs = (_dp * d)(*[_d(f) for f in facs])
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(int(np.prod([f.shape[0] for f in facs])))
        if self.which == "oracle":
            mult = C.c_int64()
        else:
            mult = C.c_longlong()
        self._check(self._f("kron_matvec_shuffle")(d, rows, cols, ptrs, _d(q), _d(out),
                                                   C.byref(mult)))
        return out, int(mult.value)

    def op_count_estimate(self, shapes):
        d = len(shapes)
        rows = (C.c_int * d)(*[s[0] for s in shapes])
        cols = (C.c_int * d)(*[s[1] for s in shapes])
        return int(self._f("op_count_estimate")(d, rows, cols))

    # ---- parallel -------------------------------------------------------
    def _args(self, pb: Problem, fuse_terms=False, threads=1):
        keep = []

        def arr(x, dt=np.float64):
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        pos = arr(pb.pos).reshape(-1, 3)
        q = arr(pb.q)
        tw = arr(pb.term_weights if len(pb.term_weights) else np.zeros(1))
        prof = arr(pb.profiles if len(pb.term_weights) else np.zeros(1))
        a = ApplyArgs()
        a.xi, a.modes = pb.xi, pb.modes
        a.center = (C.c_double * 3)(*pb.center)
        a.radius = pb.radius
        a.counts = (C.c_int * 3)(*pb.counts)
        a.order = pb.order
        a.dec_modes = pb.modes if pb.dec_modes is None else pb.dec_modes
        a.correction = pb.correction
        a.nterms = len(pb.term_weights)
        a.term_weights, a.profiles = _d(tw), _d(prof)
        a.n = pos.shape[0]
        a.pos, a.q = _d(pos), _d(q)
        a.fuse_terms, a.threads = int(bool(fuse_terms)), int(threads)
        return a, keep

    def kpme_apply(self, pb: Problem, fuse_terms=False, threads=1, ledger=False):
        a, keep = self._args(pb, fuse_terms, threads)
        out = np.zeros(max(a.n, 1))
        rows = C.c_int64()
        if ledger:
            ncell = int(np.prod(pb.counts))
            nt = len(pb.term_weights)
            cap = ncell * ((3 if fuse_terms else 3 * nt) + 1)
            led = np.zeros((max(cap, 1), 4), np.int64)
            self._check(self._f("kpme_apply")(C.byref(a), _d(out), led.ctypes.data_as(_i64p),
                                              C.c_int64(cap), C.byref(rows)))
            return out[: a.n], led[: rows.value]
        self._check(self._f("kpme_apply")(C.byref(a), _d(out), None, C.c_int64(0),
                                          C.byref(rows)))
        return out[: a.n]

    def interpolate(self, pb: Problem):
        a, keep = self._args(pb)
        phi = np.zeros((int(np.prod(pb.counts)), pb.order ** 3))
        self._check(self._f("interpolate")(C.byref(a), _d(phi)))
        return phi

    def spkmv_sum(self, pb: Problem, phi, fuse_terms=False, threads=1):
        a, keep = self._args(pb, fuse_terms, threads)
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        psi = np.zeros_like(phi)
        self._check(self._f("spkmv_sum")(C.byref(a), _d(phi), _d(psi)))
        return psi

    def anterpolate(self, pb: Problem, psi):
        a, keep = self._args(pb)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        out = np.zeros(max(a.n, 1))
        self._check(self._f("anterpolate")(C.byref(a), _d(psi), _d(out)))
        return out[: a.n]

    # ---- oracle.hpp -----------------------------------------------------
    def dense_reciprocal_apply(self, pos, q, xi, modes):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros(max(len(q), 1))
        self._check(self._f("dense_reciprocal_apply")(C.c_int64(len(q)), _d(pos), _d(q),
                                                      C.c_double(xi), modes, _d(out)))
        return out[: len(q)]


def make_problem(cpu: CpuKpme, *, n, counts, order, modes=4, xi=3.0, eps=1e-8,
                 center=(0.5, 0.5, 0.5), radius=0.5, seed=0, charges="uniform",
                 nterms=None):
    """Seeded problem in the recommended parameterisation."""
    pos, q = cpu.sample_cloud(center, radius, n, seed)
    if charges == "pm1":
        q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    elif charges == "half":
        q = np.where(np.arange(n) < n // 2, 1.0, -1.0)
    elif charges == "neutral":
        q = q - q.mean()
    rule = cpu.sinc_rule_for_eps(eps, modes)
    tw, prof, corr = cpu.skp_from_quadrature(rule, xi, modes)
    if nterms is not None:
        tw, prof = tw[:nterms], prof[:nterms]
    if isinstance(counts, int):
        counts = (counts, counts, counts)
    return Problem(xi=xi, modes=modes, center=tuple(center), radius=radius,
                   counts=tuple(counts), order=order, term_weights=tw, profiles=prof,
                   correction=corr, pos=pos, q=q)

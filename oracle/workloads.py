"""BASELINE.json workloads built through a CPU back end only -- TEST
INFRASTRUCTURE ONLY.

``problem(name, cpu)`` builds configs 1-4 exactly as
``paper_2601_18838_b200.inputs.workload`` does, but every value comes from the
given ``CpuKpme`` back end: the cloud from its ``sample_cloud``
(geometry.hpp:238-251), the decomposition from its ``sinc_rule_for_eps`` and
``skp_from_quadrature`` (alpha.hpp:154-188). With ``CpuKpme("ref")`` or
``"ref_o3"`` that is the reference's own code, so ``bench.py --impl
reference`` never loads the GPU library (tests/test_oracle_pins.py checks the
two constructions agree bit for bit).

``dense_factors(n, R, cpu)`` builds config 5's n x n axis operators A_a(lambda)
from the back end's per-cell ``build_uv`` (symfourier.hpp:108-124) with the
node shift of kpme_apply (parallel.hpp:263-279): block (c, c') of A is
U_c . V_c', the operator the spkmv axis reduction applies along one axis.
"""
from __future__ import annotations

import math

import numpy as np

from .binding import CpuKpme, Problem

MODES, XI = 4, 3.0
CENTER, RADIUS = (0.5, 0.5, 0.5), 0.5

# name -> (particles, K, L, eps); config 4 is 10^6 three-site waters
CONFIGS = {
    "cfg1": (1000, 8, 4, 1e-8),
    "cfg2": (100_000, 11, 6, 1e-10),
    "cfg3": (1_000_000, 21, 6, 1e-10),
    "cfg4": (3_000_000, 43, 6, 1e-10),
}


def describe(name: str, nterms: int) -> dict:
    """The bench line's ``config`` dict; identical in both bench arms."""
    n, K, L, eps = CONFIGS[name]
    return {"workload": name, "particles": n, "cells": [K, K, K], "order_L": L,
            "mesh": [K * L] * 3, "modes_M": MODES, "xi": XI, "skp_eps": eps,
            "skp_terms": nterms}


def decomposition(cpu: CpuKpme, eps: float, modes: int = MODES, xi: float = XI):
    rule = cpu.sinc_rule_for_eps(eps, modes)
    return cpu.skp_from_quadrature(rule, xi, modes)


def water_cloud(cpu: CpuKpme, molecules: int, seed: int = 0, density: float = 0.0334):
    """Config 4's synthetic water (same recipe as inputs.water_cloud): O
    uniform in a cube of edge (molecules/density)^(1/3) A, random bisector
    from a second seeded sample, O-H 0.9572 A, H-O-H 104.52 deg, wrapped and
    scaled into the unit box; charges O -0.834, H +0.417."""
    edge = (molecules / density) ** (1.0 / 3.0)
    o, _ = cpu.sample_cloud((edge / 2,) * 3, edge / 2, molecules, seed)
    u, _ = cpu.sample_cloud(CENTER, RADIUS, molecules, seed + 1)
    z = 2.0 * u[:, 0] - 1.0
    phi = 2.0 * math.pi * u[:, 1]
    psi = 2.0 * math.pi * u[:, 2]
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    bis = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    ref = np.where(np.abs(bis[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]),
                   np.array([[1.0, 0.0, 0.0]]))
    e1 = np.cross(bis, ref)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(bis, e1)
    v = np.cos(psi)[:, None] * e1 + np.sin(psi)[:, None] * e2
    half = math.radians(104.52) / 2.0
    d = 0.9572
    h1 = o + d * (math.cos(half) * bis + math.sin(half) * v)
    h2 = o + d * (math.cos(half) * bis - math.sin(half) * v)
    pos = np.stack([o, h1, h2], axis=1).reshape(-1, 3)
    pos = np.mod(pos, edge) / edge
    pos = np.minimum(pos, np.nextafter(1.0, 0.0))
    q = np.tile(np.array([-0.834, 0.417, 0.417]), molecules)
    return np.ascontiguousarray(pos), q


def problem(name: str, cpu: CpuKpme) -> Problem:
    n, K, L, eps = CONFIGS[name]
    if name == "cfg4":
        pos, q = water_cloud(cpu, n // 3, 0)
    else:
        pos, q = cpu.sample_cloud(CENTER, RADIUS, n, 0)
        if name == "cfg1":
            q = np.where(np.arange(n) < n // 2, 1.0, -1.0)
        elif name == "cfg2":
            q = q - q.mean()
        else:
            q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    tw, prof, corr = decomposition(cpu, eps)
    return Problem(xi=XI, modes=MODES, center=CENTER, radius=RADIUS, counts=(K, K, K),
                   order=L, term_weights=tw, profiles=prof, correction=corr, pos=pos, q=q)


def cell_nodes(lo: float, hi: float, L: int) -> np.ndarray:
    """CellGrid::axis_nodes (geometry.hpp:86-95): L equispaced points with
    both endpoints."""
    return np.array([lo + (hi - lo) * k / (L - 1) for k in range(L)])


def dense_factors(cpu: CpuKpme, n: int, nterms: int, eps: float = 1e-8, L: int = 8):
    """Config 5's factors: A_a(lambda_r) for r < nterms, n x n per axis, the
    unit box with K = n / L cells per axis. Every block comes from the back
    end's build_uv on cell nodes shifted by the box centre (parallel.hpp:
    266-271). The unit cube's axes are identical, so one [nterms][n][n]
    array per axis is returned three times."""
    if n % L:
        raise ValueError("config 5 meshes are multiples of L")
    K = n // L
    tw, prof, _ = decomposition(cpu, eps)
    tw, prof = tw[:nterms], prof[:nterms]
    out = []
    for a in range(3):
        A = np.zeros((nterms, n, n))
        lo0 = CENTER[a] - RADIUS
        for t in range(nterms):
            us, vs = [], []
            for c in range(K):
                lo = lo0 + 2.0 * RADIUS * c / K
                hi = lo0 + 2.0 * RADIUS * (c + 1) / K
                nodes = cell_nodes(lo, hi, L) - CENTER[a]
                u, v = cpu.build_uv(tw[t], prof[t, a], nodes, MODES)
                us.append(u)
                vs.append(v)
            U = np.concatenate(us, axis=0)   # [n][r_ax]
            V = np.concatenate(vs, axis=1)   # [r_ax][n]
            A[t] = U @ V
        out.append(A)
    return out

"""Seeded synthetic inputs for BASELINE.json's five configurations.

None of them is a public dataset; shapes, sizes and value distributions follow
BASELINE.json and the parameterisation recorded in DESIGN.md:
unit box Box3({.5,.5,.5}, .5), M = 4, xi = 3.0 (tools/kpme.cpp:328-330
defaults), sinc decompositions at the stated tolerance, seed 0 everywhere.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import (Box3, ChargeVector, CloudData, EwaldConfig, PointCloud, SkpDecomposition,
                  build_cell_grid, sample_cloud, sinc_rule_for_eps, skp_from_quadrature)

UNIT = Box3((0.5, 0.5, 0.5), 0.5)
MODES, XI = 4, 3.0


@dataclass
class Workload:
    name: str
    cfg: EwaldConfig
    grid: object
    order: int
    dec: SkpDecomposition
    data: CloudData
    eps: float

    @property
    def n(self) -> int:
        return self.data.cloud.size()

    def describe(self) -> dict:
        K = self.grid.counts
        return {"workload": self.name, "particles": self.n, "cells": list(K),
                "order_L": self.order, "mesh": [k * self.order for k in K],
                "modes_M": self.cfg.modes, "xi": self.cfg.xi, "skp_eps": self.eps,
                "skp_terms": len(self.dec.terms)}


_DEC_CACHE: dict = {}


def decomposition(eps: float, modes: int = MODES, xi: float = XI) -> SkpDecomposition:
    key = (eps, modes, xi)
    if key not in _DEC_CACHE:
        _DEC_CACHE[key] = skp_from_quadrature(sinc_rule_for_eps(eps, modes), EwaldConfig(xi, modes))
    return _DEC_CACHE[key]


def water_cloud(molecules: int, seed: int = 0, density: float = 0.0334) -> CloudData:
    """Config 4: rigid three-site waters, O uniform in a periodic cube at the
    given density (molecules / A^3), O-H 0.9572 A, H-O-H 104.52 deg, random
    orientation; positions wrapped and scaled by 1/edge into the unit box.
    Charges O -0.834, H +0.417. Order per molecule: O, H, H."""
    edge = (molecules / density) ** (1.0 / 3.0)
    o = sample_cloud(Box3((edge / 2,) * 3, edge / 2), molecules, seed).cloud.positions
    u = sample_cloud(Box3((0.5, 0.5, 0.5), 0.5), molecules, seed + 1).cloud.positions
    z = 2.0 * u[:, 0] - 1.0
    phi = 2.0 * math.pi * u[:, 1]
    psi = 2.0 * math.pi * u[:, 2]
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    bis = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)  # bisector (unit)
    # orthonormal frame perpendicular to the bisector
    ref = np.where(np.abs(bis[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
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
    return CloudData(PointCloud(np.ascontiguousarray(pos)), ChargeVector(q))


def workload(name: str) -> Workload:
    """cfg1 .. cfg4 of BASELINE.json (configs[0..3])."""
    if name == "cfg1":
        data = sample_cloud(UNIT, 1000, 0)
        data.charges.values = np.where(np.arange(1000) < 500, 1.0, -1.0)
        K, L, eps = 8, 4, 1e-8
    elif name == "cfg2":
        data = sample_cloud(UNIT, 100_000, 0)
        data.charges.values = data.charges.values - data.charges.values.mean()
        K, L, eps = 11, 6, 1e-10
    elif name == "cfg3":
        data = sample_cloud(UNIT, 1_000_000, 0)
        data.charges.values = np.where(np.arange(1_000_000) % 2 == 0, 1.0, -1.0)
        K, L, eps = 21, 6, 1e-10
    elif name == "cfg4":
        data = water_cloud(1_000_000, 0)
        K, L, eps = 43, 6, 1e-10
    else:
        raise ValueError(f"unknown workload {name}")
    return Workload(name, EwaldConfig(XI, MODES), build_cell_grid(UNIT, K), L,
                    decomposition(eps), data, eps)


def dense_case(n: int, nterms: int, eps: float = 1e-8):
    """Config 5 geometry: mesh n^3 = (K L)^3 with L = 8 (CLI default order),
    unit box, the first ``nterms`` terms of sinc_rule_for_eps(eps, 4)."""
    if n % 8:
        raise ValueError("config 5 meshes are multiples of L = 8")
    dec = decomposition(eps).truncated(nterms)
    return EwaldConfig(XI, MODES), build_cell_grid(UNIT, n // 8), 8, dec

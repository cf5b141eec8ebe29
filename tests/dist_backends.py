"""CPU stand-ins for the per-rank GPU compute of paper_2601_18838_b200.dist
(TEST INFRASTRUCTURE). They let tests/test_dist_cpu.py run the real slab
orchestration (routing, the core all-reduce, the dense strategies' collectives)
with torch.distributed gloo on CPU, world size 2.

``CpuCollapsedSlab`` evaluates the collapsed operator of core.cu with numpy
(same factor formulas: build_w symfourier.hpp:23-33, build_uv 108-124; Lagrange
interpolation.hpp:20-59) restricted to one z-slab of cells."""
from __future__ import annotations

import math

import numpy as np
import torch

from paper_2601_18838_b200.dist import axis_cells


def lagrange_rows(order, lo, hi, y):
    t = (y - 0.5 * (hi + lo)) / (0.5 * (hi - lo))
    nodes = -1.0 + 2.0 * np.arange(order) / (order - 1)
    w = np.ones((len(y), order))
    for k in range(order):
        for j in range(order):
            if j != k:
                w[:, k] *= (t - nodes[j]) / (nodes[k] - nodes[j])
    return w


class CpuCollapsedSlab:
    """z_lo, z_hi: the slab; block (optional): the rank's cell block
    ((lo0, hi0), (lo1, hi1), (lo2, hi2)) of a general device grid, checked
    like the GPU plan checks it (the mesh keeps full x / y extent: cells
    outside the block simply stay empty)."""

    def __init__(self, pb, z_lo, z_hi, block=None):
        self.pb, self.z_lo, self.z_hi = pb, z_lo, z_hi
        self.block = block
        M, L = pb.modes, pb.order
        self.R = 2 * M + 1
        K = pb.counts
        self.W = []
        for a in range(3):
            n = K[a] * L
            x = np.arange(n)
            c, l = x // L, x % L
            lo = pb.center[a] - pb.radius + 2.0 * pb.radius * c / K[a]
            hi = pb.center[a] - pb.radius + 2.0 * pb.radius * (c + 1) / K[a]
            node = (lo + (hi - lo) * l / (L - 1)) - pb.center[a]
            W = np.zeros((self.R, n))
            W[0] = 1.0
            for m in range(1, M + 1):
                W[2 * m - 1] = math.sqrt(2) * np.cos(2 * math.pi * m * node)
                W[2 * m] = math.sqrt(2) * np.sin(2 * math.pi * m * node)
            self.W.append(W)
        P = 2 * M + 1
        D = np.zeros((len(pb.term_weights), 3, self.R))
        for t, w in enumerate(pb.term_weights):
            for a in range(3):
                p = pb.profiles[t, a]
                for r in range(self.R):
                    m = (r + 1) // 2
                    D[t, a, r] = np.cbrt(w) * 0.5 * (p[m + M] + p[M - m])
        self.G = np.einsum("ta,tb,tc->abc", D[:, 0], D[:, 1], D[:, 2])
        del P

    def core_size(self):
        return self.R ** 3 + 1

    def _weights(self, xyz):
        pb, L = self.pb, self.pb.order
        c = [axis_cells(xyz[:, a], pb.center[a], pb.radius, pb.counts[a]) for a in range(3)]
        assert ((c[2] >= self.z_lo) & (c[2] < self.z_hi)).all(), "particle outside the slab"
        if self.block is not None:
            for a in range(2):
                lo, hi = self.block[a]
                assert ((c[a] >= lo) & (c[a] < hi)).all(), "particle outside the cell block"
        w = []
        for a in range(3):
            lo = pb.center[a] - pb.radius + 2.0 * pb.radius * c[a] / pb.counts[a]
            hi = pb.center[a] - pb.radius + 2.0 * pb.radius * (c[a] + 1) / pb.counts[a]
            w.append(lagrange_rows(L, lo, hi, xyz[:, a]))
        return c, w

    def forward(self, xyz, q, core):
        xyz, q = xyz.numpy(), q.numpy()
        L, K = self.pb.order, self.pb.counts
        c, w = self._weights(xyz)
        n0, n1 = K[0] * L, K[1] * L
        zl0, nzl = self.z_lo * L, (self.z_hi - self.z_lo) * L
        mesh = np.zeros((n0, n1, max(nzl, 0)))
        ii = c[0][:, None] * L + np.arange(L)[None]
        jj = c[1][:, None] * L + np.arange(L)[None]
        kk = c[2][:, None] * L + np.arange(L)[None] - zl0
        for p in range(len(q)):
            mesh[np.ix_(ii[p], jj[p], kk[p])] += q[p] * np.einsum("i,j,k->ijk", w[0][p], w[1][p], w[2][p])
        W2 = self.W[2][:, zl0:zl0 + nzl]
        F = np.einsum("ax,by,cz,xyz->abc", self.W[0], self.W[1], W2, mesh)
        core[:-1] = torch.as_tensor(F.ravel())
        core[-1] = float(q.sum())
        self._last = (c, w)
        return core

    def backward(self, core, out):
        L, K = self.pb.order, self.pb.counts
        R = self.R
        F = core[:-1].numpy().reshape(R, R, R)
        zl0, nzl = self.z_lo * L, (self.z_hi - self.z_lo) * L
        W2 = self.W[2][:, zl0:zl0 + nzl]
        psi = np.einsum("ax,by,cz,abc->xyz", self.W[0], self.W[1], W2, self.G * F)
        c, w = self._last
        res = np.zeros(len(c[0]))
        for p in range(len(res)):
            blk = psi[np.ix_(c[0][p] * L + np.arange(L), c[1][p] * L + np.arange(L),
                             c[2][p] * L + np.arange(L) - zl0)]
            res[p] = np.einsum("i,j,k,ijk->", w[0][p], w[1][p], w[2][p], blk)
        out.copy_(torch.as_tensor(res - self.pb.correction * float(core[-1])))
        return out

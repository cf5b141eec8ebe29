"""Generate the committed golden vectors from the REFERENCE ITSELF.

Runs only in the build container (needs oracle/_ref/libkpme_ref.so, i.e. the
reference's own headers /root/reference/proj/include/kpme/*.hpp compiled by
oracle/ref/Makefile). Writes tests/golden/golden.npz. Every array in it is an
output of a reference function on seeded inputs:

* sort KATs  : assign_particles (geometry.hpp:131-154) on configs 1-3
* rules      : sinc_rule_for_eps (alpha.hpp:154-161) at M=4, eps 1e-8/1e-10
* potentials : kpme_apply (parallel.hpp:243-290) on config 1 (full), config 2
               (strided sample + norms) and the reference tests' small setups
* dense      : kron_matvec_shuffle (kron.hpp:180-197) with dense factors
* physics    : dense_reciprocal_apply (oracle.hpp:21-58)

Usage:  python tests/golden/gen_golden.py
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.binding import CpuKpme, Problem  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
UNIT = ((0.5, 0.5, 0.5), 0.5)


def fnv1a64(a: np.ndarray) -> int:
    """FNV-1a-64 over the little-endian bytes of an int32 array."""
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a, dtype="<i4").tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def problem(ref, *, n, counts, order, modes, xi, eps, center, radius, seed, charges,
            nterms=None, rule=None):
    pos, q = ref.sample_cloud(center, radius, n, seed)
    if charges == "half":
        q = np.where(np.arange(n) < n // 2, 1.0, -1.0)
    elif charges == "pm1":
        q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    elif charges == "neutral":
        q = q - q.mean()
    elif charges == "zero":
        q = np.zeros(n)
    if rule is None:
        rule = ref.sinc_rule_for_eps(eps, modes)
    tw, prof, corr = ref.skp_from_quadrature(rule, xi, modes)
    if nterms is not None:
        tw, prof = tw[:nterms], prof[:nterms]
    if isinstance(counts, int):
        counts = (counts,) * 3
    return Problem(xi=xi, modes=modes, center=tuple(center), radius=radius,
                   counts=tuple(counts), order=order, term_weights=tw, profiles=prof,
                   correction=corr, pos=pos, q=q)


# Small end-to-end cases, mirroring the reference's own test setups.
SMALL = {
    # config 1 (BASELINE.json configs[0]), SURVEY.md §0.4
    "cfg1": dict(n=1000, counts=8, order=4, modes=4, xi=3.0, eps=1e-8, center=UNIT[0],
                 radius=UNIT[1], seed=0, charges="half"),
    # test_parallel.cpp:256-277 "single cell kpme matches the dense oracle"
    "single_cell": dict(n=48, counts=1, order=8, modes=2, xi=3.0, eps=1e-10,
                        center=(0, 0, 0), radius=0.25 / (math.pi * 2), seed=11,
                        charges="uniform"),
    # test_parallel.cpp:279-295 "split and single-cell runs agree"
    "split_k1": dict(n=64, counts=1, order=10, modes=2, xi=3.0, eps=1e-12, center=(0, 0, 0),
                     radius=0.0625 / (math.pi * 2), seed=13, charges="uniform"),
    "split_k2": dict(n=64, counts=2, order=10, modes=2, xi=3.0, eps=1e-12, center=(0, 0, 0),
                     radius=0.0625 / (math.pi * 2), seed=13, charges="uniform"),
    # acceptance.cpp:50-75 criterion 1
    "accept1": dict(n=256, counts=1, order=10, modes=4, xi=3.0, eps=1e-10, center=(0, 0, 0),
                    radius=0.25 / (math.pi * 4), seed=2024, charges="uniform"),
    # acceptance.cpp:194-226 criterion 4 shapes (one of them)
    "accept4_421": dict(n=128, counts=(4, 2, 1), order=12, modes=2, xi=3.0, eps=1e-12,
                        center=(0, 0, 0), radius=0.0625 / (math.pi * 2), seed=512,
                        charges="uniform"),
    # non-cubic grid, off-centre box, odd order
    "rect": dict(n=500, counts=(3, 4, 5), order=5, modes=3, xi=2.5, eps=1e-9,
                 center=(0.2, -0.1, 0.4), radius=0.45, seed=7, charges="uniform"),
    # config-2 geometry with few particles (dense mesh, sparse cells)
    "sparse": dict(n=300, counts=11, order=6, modes=4, xi=3.0, eps=1e-10, center=UNIT[0],
                   radius=UNIT[1], seed=3, charges="neutral"),
}


def main():
    ref = CpuKpme("ref")
    g: dict[str, np.ndarray] = {}

    # ---- sort KATs (configs 1-3, seed 0, unit box) ------------------------
    for name, n, k in [("cfg1", 1000, 8), ("cfg2", 100_000, 11), ("cfg3", 1_000_000, 21)]:
        pos, q = ref.sample_cloud(*UNIT, n, 0)
        perm, start = ref.assign_particles(*UNIT, (k, k, k), pos)
        g[f"sort_{name}_meta"] = np.array([n, k, fnv1a64(perm) >> 32, fnv1a64(perm) & 0xFFFFFFFF,
                                           fnv1a64(start) >> 32, fnv1a64(start) & 0xFFFFFFFF],
                                          np.int64)
        g[f"sort_{name}_head"] = perm[:64].astype(np.int32)
        g[f"sort_{name}_qsum"] = np.array([q.sum()])
        if n <= 1000:
            g[f"sort_{name}_perm"] = perm.astype(np.int32)
            g[f"sort_{name}_start"] = start.astype(np.int32)
    # reference tie-break / edge geometry (test_geometry.cpp:60-66)
    edge_pos = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5], [-1.0, -1.0, -1.0], [1.0, 1.0, 1.0],
                         [-0.5, 0.5, 0.0], [1.0 / 3.0, -1.0 / 3.0, 0.999999999999]])
    perm, start = ref.assign_particles((0, 0, 0), 1.0, (2, 3, 4), edge_pos)
    g["sort_edge_pos"] = edge_pos
    g["sort_edge_perm"], g["sort_edge_start"] = perm, start

    # ---- quadrature rules --------------------------------------------------
    for eps, tag in [(1e-8, "1e-08"), (1e-10, "1e-10")]:
        r = ref.sinc_rule_for_eps(eps, 4)
        g[f"rule_M4_{tag}_nodes"] = r["nodes"]
        g[f"rule_M4_{tag}_weights"] = r["weights"]
        g[f"rule_M4_{tag}_meta"] = np.array([r["half_width"], r["lifting"], r["eps"]])

    # ---- end-to-end potentials (reference kpme_apply) ----------------------
    for name, spec in SMALL.items():
        pb = problem(ref, **spec)
        z, led = ref.kpme_apply(pb, ledger=True)
        g[f"e2e_{name}_pos"] = pb.pos
        g[f"e2e_{name}_q"] = pb.q
        g[f"e2e_{name}_pot"] = z
        g[f"e2e_{name}_ledger_rows"] = np.array([len(led)])
        zf = ref.kpme_apply(pb, fuse_terms=True)
        g[f"e2e_{name}_pot_fused"] = zf
        if pb.pos.shape[0] <= 1000:
            g[f"e2e_{name}_dense"] = ref.dense_reciprocal_apply(pb.pos, pb.q, pb.xi, pb.modes)
    # config 2 (100k particles): strided sample + norms of the full vector
    pb = problem(ref, n=100_000, counts=11, order=6, modes=4, xi=3.0, eps=1e-10,
                 center=UNIT[0], radius=UNIT[1], seed=0, charges="neutral")
    z = ref.kpme_apply(pb, threads=8)
    g["e2e_cfg2_idx"] = np.arange(0, 100_000, 97)
    g["e2e_cfg2_pot_sample"] = z[g["e2e_cfg2_idx"]]
    g["e2e_cfg2_norms"] = np.array([np.linalg.norm(z), z.sum(), np.abs(z).max()])

    # ---- stage vectors on config 1 -----------------------------------------
    pb = problem(ref, **SMALL["cfg1"])
    phi = ref.interpolate(pb)
    psi = ref.spkmv_sum(pb, phi)
    g["stage_cfg1_phi"] = phi
    g["stage_cfg1_psi"] = psi
    g["stage_cfg1_psi_fused"] = ref.spkmv_sum(pb, phi, fuse_terms=True)

    # ---- dense-factor Kronecker matvec (config-5 semantics at small n) -----
    rng = np.random.default_rng(5)
    for n in (6, 16):
        facs = [rng.uniform(-1, 1, (n, n)) for _ in range(3)]
        qv = rng.uniform(-1, 1, n ** 3)
        out, mult = ref.kron_matvec_shuffle(facs, qv)
        g[f"kron_n{n}_factors"] = np.stack(facs)
        g[f"kron_n{n}_q"] = qv
        g[f"kron_n{n}_out"] = out
        g[f"kron_n{n}_mult"] = np.array([mult])
    # rectangular factors (test_kron.cpp:108-119 shapes)
    facs = [rng.uniform(-1, 1, s) for s in [(4, 3), (5, 2), (3, 6)]]
    qv = rng.uniform(-1, 1, 3 * 2 * 6)
    out, mult = ref.kron_matvec_shuffle(facs, qv)
    for i, f in enumerate(facs):
        g[f"kron_rect_f{i}"] = f
    g["kron_rect_q"], g["kron_rect_out"], g["kron_rect_mult"] = qv, out, np.array([mult])

    # ---- factor KATs: build_uv on config-1 cell 3, term 7 ------------------
    pb = problem(ref, **SMALL["cfg1"])
    lo = 0.0 + 3 * (1.0 / 8)
    nodes = np.array([lo + (1.0 / 8) * k / 3 for k in range(4)]) - 0.5
    u, v = ref.build_uv(pb.term_weights[7], pb.profiles[7, 0], nodes, 4)
    g["uv_nodes"], g["uv_u"], g["uv_v"] = nodes, u, v

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()

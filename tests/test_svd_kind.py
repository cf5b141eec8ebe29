"""SVD-kind decompositions (nkpa_svd, alpha.hpp:225-281).

CPU: the library's host Jacobi SVD against the reference's own nkpa_svd
(oracle/_ref) -- term counts, weights, the a priori bound and the rebuilt
tensor -- plus the reference tests' cases (test_alpha.cpp:30-86, acceptance
criterion 5). GPU: kpme_apply with an SVD-kind decomposition (signed
profiles, zero correction) against the oracle on the same decomposition."""
import os

import numpy as np
import pytest

from oracle.binding import CpuKpme

HAS_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                      "libkpme_ref.so"))


def rebuild(dec, n):
    R = np.zeros((n, n, n))
    for t in dec.terms:
        R += t.weight * np.einsum("i,j,k->ijk", *t.profiles)
    return R.ravel()


@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("M,tol", [(2, 1e-4), (2, 1e-8), (4, 1e-4), (4, 1e-8), (4, 1e-12),
                                   (8, 1e-4), (8, 1e-8)])
def test_nkpa_svd_matches_reference(M, tol):
    import paper_2601_18838_b200 as kp

    ref = CpuKpme("ref")
    a = kp.assemble_alpha(kp.EwaldConfig(4.0, M))
    assert np.array_equal(a.entries, ref.assemble_alpha(4.0, M))
    dec, bound = kp.nkpa_svd(a, tol, tol / 10.0)
    tw, prof, rbound = ref.nkpa_svd(a.entries, M, tol, tol / 10.0)
    assert dec.kind == kp.SkpKind.svd and dec.correction == 0.0 and dec.modes == M
    assert len(dec.terms) == len(tw) <= (2 * M + 1) ** 2
    w = np.array([t.weight for t in dec.terms])
    assert np.allclose(np.sort(w), np.sort(tw), rtol=1e-12, atol=1e-14 * tw.max())
    assert abs(bound - rbound) <= 1e-12 * max(rbound, 1e-300) + 1e-20
    n = 2 * M + 1
    err = np.linalg.norm(rebuild(dec, n) - a.entries)
    assert err <= bound + 1e-13 * np.linalg.norm(a.entries)  # criterion 5
    R2 = np.zeros((n, n, n))
    for wt, p in zip(tw, prof):
        R2 += wt * np.einsum("i,j,k->ijk", *p)
    assert np.linalg.norm(rebuild(dec, n) - R2.ravel()) <= 1e-12 * np.linalg.norm(a.entries)


def test_nkpa_svd_rank1_zero_and_errors():
    import paper_2601_18838_b200 as kp

    rng = np.random.default_rng(42)
    n = 5
    p = [rng.random(n) + 0.5 for _ in range(3)]
    v = kp.AlphaVector(2, np.einsum("i,j,k->ijk", *p).ravel())
    dec, _ = kp.nkpa_svd(v, 1e-10, 1e-11)
    assert len(dec.terms) == 1
    assert np.linalg.norm(rebuild(dec, n) - v.entries) <= 1e-12 * np.linalg.norm(v.entries)
    z, bound = kp.nkpa_svd(kp.AlphaVector(1, np.zeros(27)), 1e-8, 1e-8)
    assert z.terms == [] and bound == 0.0
    with pytest.raises(ValueError, match="tol_inner must be <= tol_outer"):
        kp.nkpa_svd(kp.AlphaVector(1, np.zeros(27)), 1e-8, 1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("M,tol,counts,L", [(4, 1e-8, (8, 8, 8), 4), (4, 1e-10, (6, 5, 7), 6),
                                            (3, 1e-6, (4, 4, 4), 8)])
def test_kpme_apply_svd_kind_vs_oracle(oracle, M, tol, counts, L):
    """kpme_apply with an SVD-kind decomposition (the CLI's
    nkpa_svd(assemble_alpha(cfg), eps, eps / 10), tools/kpme.cpp:76) on the
    GPU against the oracle on the same decomposition (<= 1e-10), and against
    the oracle on the reference's own nkpa_svd decomposition."""
    import paper_2601_18838_b200 as kp
    from oracle.binding import Problem, make_problem

    cfg = kp.EwaldConfig(3.0, M)
    dec, _ = kp.nkpa_svd(kp.assemble_alpha(cfg), tol, tol / 10.0)
    base = make_problem(oracle, n=4000, counts=counts, order=L, modes=M, eps=1e-8, seed=M,
                        charges="neutral")
    tw, prof = dec.arrays()
    pb = Problem(xi=3.0, modes=M, center=base.center, radius=base.radius, counts=counts, order=L,
                 term_weights=tw, profiles=prof, correction=0.0, pos=base.pos, q=base.q)
    grid = kp.build_cell_grid(kp.Box3(base.center, base.radius), counts)
    z = kp.kpme_apply(cfg, grid, L, dec, kp.PointCloud(base.pos), kp.ChargeVector(base.q))
    ref = oracle.kpme_apply(pb)
    assert np.linalg.norm(z.potentials - ref) / np.linalg.norm(ref) <= 1e-10
    if HAS_REF:
        rtw, rprof, _ = CpuKpme("ref").nkpa_svd(kp.assemble_alpha(cfg).entries, M, tol, tol / 10)
        pb.term_weights, pb.profiles = rtw, rprof
        ref2 = CpuKpme("ref").kpme_apply(pb)
        assert np.linalg.norm(z.potentials - ref2) / np.linalg.norm(ref2) <= 1e-10

"""Pin the CPU oracle to the reference before trusting it (CPU only).

The golden vectors in tests/golden/golden.npz were produced by the reference's
own headers (tests/golden/gen_golden.py via oracle/_ref). The oracle keeps the
reference's evaluation order, so every comparison here is BIT-EXACT unless it
is a physics tolerance copied from the reference's own tests.
"""
import math
import os

import numpy as np
import pytest

from oracle.binding import CpuKpme, OracleError, Problem

UNIT = ((0.5, 0.5, 0.5), 0.5)


def fnv1a64(a):
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a, dtype="<i4").tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _problem_from_golden(oracle, golden, name, spec):
    rule = oracle.sinc_rule_for_eps(spec["eps"], spec["modes"])
    tw, prof, corr = oracle.skp_from_quadrature(rule, spec["xi"], spec["modes"])
    counts = spec["counts"]
    counts = (counts,) * 3 if isinstance(counts, int) else tuple(counts)
    return Problem(xi=spec["xi"], modes=spec["modes"], center=tuple(spec["center"]),
                   radius=spec["radius"], counts=counts, order=spec["order"],
                   term_weights=tw, profiles=prof, correction=corr,
                   pos=golden[f"e2e_{name}_pos"], q=golden[f"e2e_{name}_q"])


# ---- geometry.hpp ----------------------------------------------------------

@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_sort_kat(oracle, golden, name):
    n, k, h_hi, h_lo, s_hi, s_lo = golden[f"sort_{name}_meta"]
    pos, q = oracle.sample_cloud(*UNIT, int(n), 0)
    perm, start = oracle.assign_particles(*UNIT, (int(k),) * 3, pos)
    assert fnv1a64(perm) == (int(h_hi) << 32 | int(h_lo))
    assert fnv1a64(start) == (int(s_hi) << 32 | int(s_lo))
    np.testing.assert_array_equal(perm[:64], golden[f"sort_{name}_head"])
    assert q.sum() == golden[f"sort_{name}_qsum"][0]


def test_sort_survey_appendix_a(oracle):
    """SURVEY.md Appendix A values (reference geometry.hpp run at survey time)."""
    rows = [(1000, 8, [547, 828, 882, 537], -34.375845231601872),
            (100_000, 11, [828, 2645, 5785, 6197], 10.462757921338415)]
    for n, k, head, qsum in rows:
        pos, q = oracle.sample_cloud(*UNIT, n, 0)
        perm, start = oracle.assign_particles(*UNIT, (k, k, k), pos)
        assert list(perm[:4]) == head
        assert q.sum() == pytest.approx(qsum, rel=1e-15)
    pos, q = oracle.sample_cloud(*UNIT, 1, 0)
    assert tuple(pos[0]) == (0.88331080821364261, 0.43152799704850997, 0.026433771592597743)
    assert q[0] == 0.94176395630765697


def test_sort_edges(oracle, golden):
    perm, start = oracle.assign_particles((0, 0, 0), 1.0, (2, 3, 4), golden["sort_edge_pos"])
    np.testing.assert_array_equal(perm, golden["sort_edge_perm"])
    np.testing.assert_array_equal(start, golden["sort_edge_start"])


def test_centre_goes_to_lower_cell(oracle):
    """test_geometry.cpp:60-66."""
    perm, start = oracle.assign_particles((0, 0, 0), 1.0, (2, 2, 2), np.zeros((1, 3)))
    assert start[1] == 1  # cell (0,0,0) holds the particle


def test_outside_particle_rejected_with_index(oracle):
    """test_geometry.cpp:98-104."""
    pos = np.array([[0.5, 0.5, 0.5], [2.0, 0.0, 0.0]])
    with pytest.raises(OracleError, match="particle 1"):
        oracle.assign_particles((0, 0, 0), 1.0, (2, 2, 2), pos)


# ---- alpha.hpp -------------------------------------------------------------

@pytest.mark.parametrize("eps,tag,count", [(1e-8, "1e-08", 65), (1e-10, "1e-10", 101)])
def test_sinc_rule_matches_reference(oracle, golden, eps, tag, count):
    r = oracle.sinc_rule_for_eps(eps, 4)
    assert len(r["nodes"]) == count
    np.testing.assert_array_equal(r["nodes"], golden[f"rule_M4_{tag}_nodes"])
    np.testing.assert_array_equal(r["weights"], golden[f"rule_M4_{tag}_weights"])
    hw, h, e = golden[f"rule_M4_{tag}_meta"]
    assert (r["half_width"], r["lifting"], r["eps"]) == (int(hw), h, e)


def test_alpha_and_bounds_kats(oracle):
    """test_alpha.cpp:12-18 and 164-170 (SURVEY.md Appendix C corrections)."""
    assert oracle.alpha_weight(math.pi, 0, 0, 0) == 0.0
    assert oracle.alpha_weight(math.pi, 1, 0, 0) == pytest.approx(math.exp(-1.0), rel=1e-14)
    assert oracle.alpha_weight(math.pi, 1, 1, 1) == pytest.approx(math.exp(-3.0) / 3, rel=1e-14)
    assert oracle.optimal_term_lower_bound(16.0 * math.exp(-math.pi)) == 1
    assert oracle.optimal_term_lower_bound(1e-14) == 125
    assert oracle.optimal_term_lower_bound(1e-8) == 46


def test_sinc_rule_midpoint(oracle):
    """test_alpha.cpp:88-98."""
    r = oracle.sinc_rule(12, 4)
    assert r["weights"][12] == pytest.approx(r["lifting"] / 2, rel=1e-14)
    assert r["nodes"][12] == pytest.approx(math.log(2.0), rel=1e-14)


def test_skp_coverage_rejected(oracle):
    """test_alpha.cpp:128-137."""
    rule = dict(nodes=np.array([0.5]), weights=np.array([1.0]), min_arg=1.0, max_arg=10.0)
    with pytest.raises(OracleError):
        oracle.skp_from_quadrature(rule, 2.0, 2)


# ---- interpolation.hpp / symfourier.hpp ------------------------------------

def test_lagrange_kats(oracle):
    """test_interpolation.cpp:10-36."""
    w = oracle.lagrange_weights_1d(3, -1.0, 1.0, 0.5)
    np.testing.assert_allclose(w, [-1 / 8, 3 / 4, 3 / 8], rtol=1e-15)
    w = oracle.lagrange_weights_1d(2, 3.0, 7.0, 5.0)
    np.testing.assert_allclose(w, [0.5, 0.5], rtol=1e-15)
    for k in range(5):
        w = oracle.lagrange_weights_1d(5, -1.0, 1.0, -1.0 + 2.0 * k / 4)
        np.testing.assert_allclose(w, np.eye(5)[k], atol=1e-13)
    with pytest.raises(OracleError):
        oracle.lagrange_weights_1d(3, 2.0, 2.0, 2.0)
    with pytest.raises(OracleError):
        oracle.lagrange_weights_1d(1, 0.0, 1.0, 0.5)


def test_build_w_kats(oracle):
    """test_symfourier.cpp:11-30."""
    w = oracle.build_w(0, [0.1, -0.7, 0.3])
    np.testing.assert_array_equal(w[0], 1.0)
    np.testing.assert_array_equal(w[1], 0.0)
    w = oracle.build_w(1, [0.25])
    assert abs(w[0, 0]) < 1e-15 and w[1, 0] == pytest.approx(math.sqrt(2))
    w = oracle.build_w(2, [0.5])
    assert w[0, 0] == pytest.approx(math.sqrt(2)) and abs(w[1, 0]) < 1e-14


def test_build_uv_matches_reference(oracle, golden):
    cfg = dict(golden=golden)
    rule = oracle.sinc_rule_for_eps(1e-8, 4)
    tw, prof, _ = oracle.skp_from_quadrature(rule, 3.0, 4)
    u, v = oracle.build_uv(tw[7], prof[7, 0], golden["uv_nodes"], 4)
    np.testing.assert_array_equal(u, golden["uv_u"])
    np.testing.assert_array_equal(v, golden["uv_v"])
    del cfg


# ---- kron.hpp --------------------------------------------------------------

@pytest.mark.parametrize("n", [6, 16])
def test_kron_shuffle_matches_reference(oracle, golden, n):
    facs = list(golden[f"kron_n{n}_factors"])
    out, mult = oracle.kron_matvec_shuffle(facs, golden[f"kron_n{n}_q"])
    np.testing.assert_array_equal(out, golden[f"kron_n{n}_out"])
    assert mult == golden[f"kron_n{n}_mult"][0] == 3 * n ** 4


def test_kron_rect_and_op_counts(oracle, golden):
    facs = [golden[f"kron_rect_f{i}"] for i in range(3)]
    out, mult = oracle.kron_matvec_shuffle(facs, golden["kron_rect_q"])
    np.testing.assert_array_equal(out, golden["kron_rect_out"])
    assert mult == oracle.op_count_estimate([f.shape for f in facs])
    # test_kron.cpp:157-166
    assert oracle.op_count_estimate([(4, 4)] * 3) == 3 * 4 ** 4
    assert oracle.op_count_estimate([(7, 7)]) == 49
    # dense oracle on the rectangular case
    dense = np.kron(np.kron(facs[0], facs[1]), facs[2]) @ golden["kron_rect_q"]
    np.testing.assert_allclose(out, dense, rtol=1e-12, atol=1e-13)


# ---- parallel.hpp: end to end ----------------------------------------------

def _specs():
    from tests.golden.gen_golden import SMALL

    return SMALL


@pytest.mark.parametrize("name", ["cfg1", "single_cell", "split_k1", "split_k2", "accept1",
                                  "accept4_421", "rect", "sparse"])
def test_kpme_apply_bit_exact_vs_reference(oracle, golden, name):
    pb = _problem_from_golden(oracle, golden, name, _specs()[name])
    z, led = oracle.kpme_apply(pb, ledger=True)
    np.testing.assert_array_equal(z, golden[f"e2e_{name}_pot"])
    assert len(led) == golden[f"e2e_{name}_ledger_rows"][0]
    zf = oracle.kpme_apply(pb, fuse_terms=True, threads=3)
    np.testing.assert_array_equal(zf, golden[f"e2e_{name}_pot_fused"])


@pytest.mark.parametrize("name,tol", [("single_cell", 1e-4), ("accept1", 1e-5)])
def test_physics_vs_dense_oracle(golden, name, tol):
    """test_parallel.cpp:256-277 (1e-4) and acceptance criterion 1 (1e-5)."""
    z, d = golden[f"e2e_{name}_pot"], golden[f"e2e_{name}_dense"]
    assert np.linalg.norm(z - d) / np.linalg.norm(d) <= tol


def test_decomposition_invariance(golden):
    """test_parallel.cpp:279-295: K=1 vs K=2 agree to 1e-12 of the max."""
    a, b = golden["e2e_split_k1_pot"], golden["e2e_split_k2_pot"]
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


def test_stages_bit_exact(oracle, golden):
    pb = _problem_from_golden(oracle, golden, "cfg1", _specs()["cfg1"])
    phi = oracle.interpolate(pb)
    np.testing.assert_array_equal(phi, golden["stage_cfg1_phi"])
    psi = oracle.spkmv_sum(pb, phi)
    np.testing.assert_array_equal(psi, golden["stage_cfg1_psi"])
    np.testing.assert_array_equal(oracle.spkmv_sum(pb, phi, fuse_terms=True),
                                  golden["stage_cfg1_psi_fused"])
    z = oracle.anterpolate(pb, psi) - pb.correction * pb.q.sum()
    np.testing.assert_allclose(z, golden["e2e_cfg1_pot"], rtol=0, atol=1e-12)


@pytest.mark.slow
def test_cfg2_sample_bit_exact(oracle, golden):
    from oracle.binding import make_problem

    pb = make_problem(oracle, n=100_000, counts=11, order=6, eps=1e-10, charges="neutral")
    z = oracle.kpme_apply(pb, threads=os.cpu_count() or 1)
    np.testing.assert_array_equal(z[golden["e2e_cfg2_idx"]], golden["e2e_cfg2_pot_sample"])
    assert np.linalg.norm(z) == golden["e2e_cfg2_norms"][0]


def test_ledger_shape(oracle):
    """test_parallel.cpp:297-343 / acceptance criterion 8: 3|L|+1 rows (unfused),
    3+1 (fused), payload 2(M+1)L^2."""
    from oracle.binding import make_problem

    pb = make_problem(oracle, n=16, counts=2, order=4, modes=2, eps=1e-6,
                      center=(0, 0, 0), radius=0.01, seed=21)
    for nterms in (0, 1, 2, 5):
        p2 = Problem(**{**pb.__dict__, "term_weights": pb.term_weights[:nterms],
                        "profiles": pb.profiles[:nterms]})
        for fuse in (False, True):
            z, led = oracle.kpme_apply(p2, fuse_terms=fuse, ledger=True)
            r0 = led[led[:, 0] == 0]
            axis = r0[r0[:, 2] >= 0]
            want = (0 if nterms == 0 else 3) if fuse else 3 * nterms
            assert len(axis) == want and (r0[:, 2] == -1).sum() == 1
            if len(axis):
                assert (axis[:, 3] == 2 * 3 * 16 * (nterms if fuse else 1)).all()


def test_zero_charges_and_mode_mismatch(oracle):
    from oracle.binding import make_problem

    pb = make_problem(oracle, n=32, counts=2, order=4, modes=2, eps=1e-6,
                      center=(0, 0, 0), radius=0.02, seed=5)
    pb.q = np.zeros(32)
    assert (oracle.kpme_apply(pb) == 0.0).all()
    pb.dec_modes = 3
    with pytest.raises(OracleError, match="mode bound mismatch"):
        oracle.kpme_apply(pb)


def test_empty_cloud(oracle):
    from oracle.binding import make_problem

    pb = make_problem(oracle, n=0, counts=2, order=4, modes=2, eps=1e-6)
    assert oracle.kpme_apply(pb).shape == (0,)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle",
                                                    "_ref", "kpme_acceptance")),
                    reason="oracle/_ref not built (no /root/reference)")
def test_reference_acceptance_gate_runs():
    """The reference's own acceptance.cpp, compiled unmodified against the
    Eigen subset, passes: validates the shim the golden vectors came from."""
    import subprocess

    exe = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "kpme_acceptance")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS criterion") == 8


# ---- oracle/workloads.py (inputs of the CPU bench arm) ----------------------

_HAS_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                       "libkpme_ref.so"))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_workloads_match_package_inputs(oracle, name):
    """bench.py's reference arm builds its inputs through the CPU back end
    alone (never the GPU library). They must be bit-identical to the
    package's (paper_2601_18838_b200.inputs), for the oracle port and for the
    reference's own headers."""
    from oracle import workloads
    from paper_2601_18838_b200 import inputs

    w = inputs.workload(name)
    tw, prof = w.dec.arrays()
    backs = [oracle] + ([CpuKpme("ref"), CpuKpme("ref_o3")] if _HAS_REF else [])
    for cpu in backs:
        pb = workloads.problem(name, cpu)
        assert np.array_equal(pb.pos, w.data.cloud.positions)
        assert np.array_equal(pb.q, w.data.charges.values)
        assert np.array_equal(pb.term_weights, tw) and np.array_equal(pb.profiles, prof)
        assert pb.correction == w.dec.correction and pb.counts == tuple(w.grid.counts)
        assert workloads.describe(name, len(tw)) == w.describe()


@pytest.mark.skipif(not _HAS_REF, reason="oracle/_ref not built (no /root/reference)")
def test_dense_factors_oracle_vs_reference(oracle):
    """Config 5's factors assembled from build_uv: oracle port == reference
    headers, bit for bit; each A_a(lambda) is symmetric-shaped n x n with the
    cell-block structure U_c V_c'."""
    from oracle import workloads

    a = workloads.dense_factors(oracle, 32, 6)
    b = workloads.dense_factors(CpuKpme("ref"), 32, 6)
    for x, y in zip(a, b):
        assert x.shape == (6, 32, 32)
        assert np.array_equal(x, y)

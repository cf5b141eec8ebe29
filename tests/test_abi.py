"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/kpme_gpu.h declares, and its host-side functions (SKP
construction, sampling, ledger) match the oracle / reference bit for bit."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kpme_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kpme_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2601_18838_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kpme_\w+)", out))
    declared = declared_functions()
    assert declared, "no declarations parsed"
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == declared
    assert _lib.lib.kpme_gpu_abi_version() == _lib.ABI_VERSION == 2


def test_library_is_sm100a():
    from paper_2601_18838_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_cpp_dropin_header_compiles():
    """include/kpme_b200/kpme.hpp compiles against the C ABI header alone."""
    src = os.path.join(ROOT, "tests", "cpp", "dropin_compile.cpp")
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", f"-I{ROOT}/include", src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_sinc_rule_matches_reference(golden):
    import paper_2601_18838_b200 as kp

    for eps, tag in [(1e-8, "1e-08"), (1e-10, "1e-10")]:
        r = kp.sinc_rule_for_eps(eps, 4)
        np.testing.assert_array_equal(r.nodes, golden[f"rule_M4_{tag}_nodes"])
        np.testing.assert_array_equal(r.weights, golden[f"rule_M4_{tag}_weights"])
        hw, h, e = golden[f"rule_M4_{tag}_meta"]
        assert (r.half_width, r.lifting, r.eps) == (int(hw), h, e)


def test_skp_and_sampling_match_oracle(oracle):
    import paper_2601_18838_b200 as kp

    rule = kp.sinc_rule(9, 3)
    dec = kp.skp_from_quadrature(rule, kp.EwaldConfig(2.5, 3))
    o_rule = oracle.sinc_rule(9, 3)
    tw, prof, corr = oracle.skp_from_quadrature(o_rule, 2.5, 3)
    w, p = dec.arrays()
    np.testing.assert_array_equal(w, tw)
    np.testing.assert_array_equal(p, prof)
    assert dec.correction == corr
    data = kp.sample_cloud(kp.Box3((0.1, -0.2, 0.3), 0.7), 500, 42)
    pos, q = oracle.sample_cloud((0.1, -0.2, 0.3), 0.7, 500, 42)
    np.testing.assert_array_equal(data.cloud.positions, pos)
    np.testing.assert_array_equal(data.charges.values, q)


def test_reference_exceptions_map():
    import paper_2601_18838_b200 as kp

    with pytest.raises(ValueError, match="xi must be positive"):
        kp.EwaldConfig(0.0, 2)
    with pytest.raises(ValueError, match="radius must be positive"):
        kp.Box3((0, 0, 0), 0.0)
    with pytest.raises(ValueError, match="cell counts"):
        kp.build_cell_grid(kp.Box3(), (0, 1, 1))
    with pytest.raises(ValueError, match="eps must be positive"):
        kp.sinc_rule_for_eps(0.0, 2)
    with pytest.raises(kp.numerical_error):
        kp.sinc_rule_for_eps(1e-30, 2, max_n=3)
    rule = kp.QuadratureRule(np.array([0.5]), np.array([1.0]), min_arg=1.0, max_arg=10.0)
    with pytest.raises(ValueError, match="does not cover"):
        kp.skp_from_quadrature(rule, kp.EwaldConfig(2.0, 2))


def test_tabulated_rule_loader(tmp_path):
    """alpha.hpp:192-212 file format, including its error paths
    (test_alpha.cpp:139-162)."""
    import paper_2601_18838_b200 as kp

    f = tmp_path / "rule.txt"
    f.write_text("2\n0.1 0.5\n0.7 0.25\n1 432 1e-15\n")
    r = kp.load_tabulated_rule(str(f))
    np.testing.assert_array_equal(r.nodes, [0.1, 0.7])
    assert r.covers(1.0, 3 * 12 * 12) and not r.covers(1.0, 3 * 13 * 13)
    bad = tmp_path / "bad.txt"
    bad.write_text("2\n0.0 1.0\n")
    with pytest.raises(RuntimeError):
        kp.load_tabulated_rule(str(bad))
    with pytest.raises(RuntimeError):
        kp.load_tabulated_rule(str(tmp_path / "missing.txt"))


@pytest.mark.parametrize("fuse", [False, True])
def test_ledger_matches_reference_shape(oracle, fuse):
    """The synthesised logical ledger equals the reference's SimulatedComm
    ledger row for row (parallel.hpp:110-138; acceptance criterion 8)."""
    import paper_2601_18838_b200 as kp
    from oracle.binding import make_problem
    from paper_2601_18838_b200.api import KpmeResult, make_config

    pb = make_problem(oracle, n=32, counts=(2, 1, 2), order=4, modes=2, eps=1e-6,
                      center=(0, 0, 0), radius=0.01, seed=5)
    _, led = oracle.kpme_apply(pb, fuse_terms=fuse, ledger=True)
    cfg = kp.EwaldConfig(pb.xi, pb.modes)
    grid = kp.build_cell_grid(kp.Box3(pb.center, pb.radius), pb.counts)
    dec = kp.SkpDecomposition(kp.SkpKind.sinc, pb.modes, pb.correction,
                              [kp.SkpTerm(float(w), tuple(p)) for w, p in
                               zip(pb.term_weights, pb.profiles)])
    c, keep = make_config(cfg, grid, pb.order, dec, kp.KpmeOptions(fuse_terms=fuse))
    res = KpmeResult(np.zeros(0), c, keep)
    np.testing.assert_array_equal(res.ledger_array, led)

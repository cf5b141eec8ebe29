"""The C++ drop-in header (include/kpme_b200/kpme.hpp) used from a C++
program: config 1 against the reference's golden potentials, the synthesised
ledger row count, and the reference's exception contract."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_cfg1(tmp_path, golden):
    lib_dir = os.path.join(ROOT, "paper_2601_18838_b200")
    exe = tmp_path / "dropin_run"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "dropin_run.cpp"), f"-L{lib_dir}",
                    "-lkpme_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out[0] == f"ledger_rows {int(golden['e2e_cfg1_ledger_rows'][0])}"
    z = np.array([float(v) for v in out[1:1001]])
    ref = golden["e2e_cfg1_pot"]
    assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= 1e-10
    assert out[1001].startswith("invalid_argument assign_particles: particle 7 outside the box")

"""B200-native SKP-PME reciprocal path (arXiv 2601.18838 "KPME" reference).

Host mirror of the reference's C++ API (``api``), the plan API over torch
device tensors (``plan``) and seeded inputs (``inputs``). All compute runs in
libkpme_b200.so (sm_100a kernels behind include/kpme_gpu.h).
"""
from .api import (AlphaVector, Box3, assemble_alpha, nkpa_svd, CellGrid, ChargeVector, CloudData, EwaldConfig, KpmeOptions,  # noqa: F401
                  KpmeResult, LedgerRow, PointCloud, QuadratureRule, SkpDecomposition, SkpKind,
                  SkpTerm, alpha_weight, build_cell_grid, check_convergence_ratio, kpme_apply,
                  ledger_to_csv, load_tabulated_rule, read_cloud, sample_cloud, sinc_rule,
                  sinc_rule_for_eps, skp_from_quadrature, write_cloud)
from ._lib import LIB_PATH, numerical_error  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]

"""ctypes binding of libkpme_b200.so (include/kpme_gpu.h).

The library is built in-tree by ``__graft_entry__.build()``. There is no CPU
fallback: if the shared library is missing, importing the package fails.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# KPME_LIB: another build of the same library (A/B of kernel variants, scripts/build_variant.sh)
LIB_PATH = os.environ.get("KPME_LIB") or os.path.join(HERE, "libkpme_b200.so")

OK, INVALID_ARGUMENT, RUNTIME, NUMERICAL, CUDA, NCCL = range(6)
FORM_AUTO, FORM_COLLAPSED, FORM_DENSE = 0, 1, 2
COLL_AUTO, COLL_PEER, COLL_NCCL = 0, 1, 2
SLAB_STRATEGIES = ("reduce_scatter", "rank_split", "alltoall")  # KPME_GPU_SLAB_* order
NCCL_ID_BYTES = 128
ABI_VERSION = 2
DEFER_CHECKS = 1

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class Config(C.Structure):
    """Mirror of kpme_gpu_config."""

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
        ("fuse_terms", C.c_int),
        ("threads", C.c_int),
        ("device", C.c_int),
        ("formulation", C.c_int),
        ("ndevices", C.c_int),
        ("devices", C.POINTER(C.c_int)),
    ]


class numerical_error(ArithmeticError):
    """kpme::numerical_error (kron.hpp:18-21)."""


class KpmeGpuError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "kpme_gpu_last_error": (C.c_char_p, []),
        "kpme_gpu_abi_version": (C.c_int, []),
        "kpme_sinc_rule": (C.c_int, [C.c_int, C.c_int, _dp, _dp, _dp, _dp]),
        "kpme_sinc_rule_for_eps": (C.c_int, [C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int),
                                             _dp, _dp, _dp, _dp]),
        "kpme_skp_from_quadrature": (C.c_int, [C.c_int, _dp, _dp, C.c_double, C.c_double,
                                               C.c_double, C.c_int, _dp, _dp, _dp]),
        "kpme_load_tabulated_rule": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_int), _dp,
                                               _dp, _dp, _dp, _dp]),
        "kpme_sample_cloud": (None, [_dp, C.c_double, C.c_int64, C.c_uint64, _dp, _dp]),
        "kpme_assemble_alpha": (C.c_int, [C.c_double, C.c_int, _dp]),
        "kpme_nkpa_svd": (C.c_int, [C.c_int, _dp, C.c_double, C.c_double, C.c_int,
                                    C.POINTER(C.c_int), _dp, _dp, _dp]),
        "kpme_gpu_ledger": (C.c_int, [C.POINTER(Config), _i64p, C.c_int64, _i64p]),
        "kpme_gpu_apply": (C.c_int, [C.POINTER(Config), C.c_int64, _dp, _dp, _dp]),
        "kpme_gpu_plan_create": (C.c_int, [C.POINTER(Config), C.c_int64, C.POINTER(P)]),
        "kpme_gpu_plan_destroy": (C.c_int, [P]),
        "kpme_gpu_plan_set_stream": (C.c_int, [P, P]),
        "kpme_gpu_plan_execute": (C.c_int, [P, C.c_int64, _dp, _dp, _dp]),
        "kpme_gpu_plan_set_host_chunks": (C.c_int, [P, C.c_int]),
        "kpme_gpu_plan_execute_device": (C.c_int, [P, C.c_int64, P, P, P, C.c_int]),
        "kpme_gpu_plan_status": (C.c_int, [P]),
        "kpme_gpu_plan_launches": (C.c_int, [P]),
        "kpme_gpu_plan_graph_execute": (C.c_int, [P, C.c_int64, P, P, P]),
        "kpme_gpu_plan_enable_timing": (C.c_int, [P, C.c_int]),
        "kpme_gpu_plan_stage_times": (C.c_int, [P, _dp, C.c_int, C.POINTER(C.c_int)]),
        "kpme_gpu_sort": (C.c_int, [P, C.c_int64, P, P, P]),
        "kpme_gpu_spread": (C.c_int, [P, C.c_int64, P, P, P]),
        "kpme_gpu_skp_apply": (C.c_int, [P, P, P]),
        "kpme_gpu_gather": (C.c_int, [P, C.c_int64, P, P, P]),
        "kpme_gpu_dense_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int, C.c_int, C.c_int]),
        "kpme_gpu_kron_matvec_dense": (C.c_int, [C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 P, P, P, P, P, P, C.c_size_t]),
        "kpme_gpu_plan_axis_operands": (C.c_int, [P, C.c_int, P]),
        "kpme_gpu_dgemm_tn": (C.c_int, [P, C.c_int64, C.c_int64, C.c_int64, P, P, P, C.c_int]),
        "kpme_gpu_plan_create_slab": (C.c_int, [C.POINTER(Config), C.c_int64, C.c_int, C.c_int,
                                                C.POINTER(P)]),
        "kpme_gpu_plan_create_block": (C.c_int, [C.POINTER(Config), C.c_int64, C.POINTER(C.c_int),
                                                 C.POINTER(C.c_int), C.POINTER(P)]),
        "kpme_gpu_plan_core_size": (C.c_int, [P]),
        "kpme_gpu_plan_forward": (C.c_int, [P, C.c_int64, P, P, P]),
        "kpme_gpu_plan_backward": (C.c_int, [P, P, P]),
        "kpme_gpu_apply_cache_clear": (C.c_int, []),
        "kpme_gpu_plan_create_multi": (C.c_int, [C.POINTER(Config), C.c_int64,
                                                 C.POINTER(C.c_int), C.POINTER(P)]),
        "kpme_gpu_plan_set_collective": (C.c_int, [P, C.c_int]),
        "kpme_gpu_plan_collective": (C.c_int, [P]),
        "kpme_gpu_plan_devices": (C.c_int, [P, C.POINTER(C.c_int), C.c_int]),
        "kpme_gpu_nccl_unique_id": (C.c_int, [C.c_void_p]),
        "kpme_gpu_plan_attach_comm": (C.c_int, [P, C.c_int, C.c_int, C.c_void_p]),
        "kpme_gpu_dense_slab_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 P, P, P, C.c_int, C.c_int, C.c_void_p,
                                                 C.POINTER(P)]),
        "kpme_gpu_dense_slab_create_group": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int,
                                                       C.c_int, C.c_int, C.c_int, C.POINTER(P),
                                                       C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
        "kpme_gpu_dense_slab_destroy": (C.c_int, [P]),
        "kpme_gpu_dense_slab_bounds": (C.c_int, [P, C.c_int, C.POINTER(C.c_int),
                                                 C.POINTER(C.c_int)]),
        "kpme_gpu_dense_slab_set_stream": (C.c_int, [P, C.c_int, P]),
        "kpme_gpu_dense_slab_apply": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(P)]),
        "kpme_gpu_dense_slab_sync": (C.c_int, [P]),
        "kpme_gpu_dense_slab_choose": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.c_int,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
if lib.kpme_gpu_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH}: ABI {lib.kpme_gpu_abi_version()}, expected {ABI_VERSION} "
                      "(stale build; rerun __graft_entry__.build())")

#: every function include/kpme_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = sorted(
    [
        "kpme_gpu_last_error", "kpme_gpu_abi_version", "kpme_sinc_rule", "kpme_sinc_rule_for_eps",
        "kpme_skp_from_quadrature", "kpme_load_tabulated_rule", "kpme_sample_cloud",
        "kpme_gpu_ledger", "kpme_gpu_apply", "kpme_gpu_plan_create", "kpme_gpu_plan_destroy",
        "kpme_gpu_plan_set_stream", "kpme_gpu_plan_execute", "kpme_gpu_plan_execute_device",
        "kpme_gpu_plan_status", "kpme_gpu_plan_launches", "kpme_gpu_plan_graph_execute",
        "kpme_gpu_plan_enable_timing", "kpme_gpu_plan_stage_times", "kpme_gpu_sort",
        "kpme_gpu_spread", "kpme_gpu_skp_apply", "kpme_gpu_gather",
        "kpme_gpu_dense_workspace_bytes", "kpme_gpu_kron_matvec_dense",
        "kpme_gpu_plan_axis_operands", "kpme_gpu_dgemm_tn", "kpme_gpu_plan_create_slab",
        "kpme_gpu_plan_core_size", "kpme_gpu_plan_forward", "kpme_gpu_plan_backward",
        "kpme_gpu_plan_set_host_chunks", "kpme_gpu_plan_create_block",
        "kpme_gpu_apply_cache_clear", "kpme_gpu_plan_create_multi",
        "kpme_gpu_plan_set_collective", "kpme_gpu_plan_collective", "kpme_gpu_plan_devices",
        "kpme_gpu_nccl_unique_id", "kpme_gpu_plan_attach_comm",
        "kpme_gpu_dense_slab_create", "kpme_gpu_dense_slab_create_group",
        "kpme_gpu_dense_slab_destroy", "kpme_gpu_dense_slab_bounds",
        "kpme_gpu_dense_slab_set_stream", "kpme_gpu_dense_slab_apply", "kpme_gpu_dense_slab_sync",
        "kpme_gpu_dense_slab_choose", "kpme_assemble_alpha", "kpme_nkpa_svd",
    ]
)


def check(code: int):
    """Map a status code to the reference's exception types
    (invalid_argument -> ValueError, numerical_error, runtime_error)."""
    if code == OK:
        return
    msg = lib.kpme_gpu_last_error().decode()
    if code == INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == NUMERICAL:
        raise numerical_error(msg)
    raise KpmeGpuError(code, msg)

"""ctypes loader for libslablu_gpu.so (the engine's C ABI, include/slablu_gpu.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2211_07572_b200/csrc``).  There is no CPU fallback: if the
library is missing the import fails loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslablu_gpu.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
D = ctypes.c_double
I = ctypes.c_int


class Status(ctypes.Structure):
    _fields_ = [("code", I), ("index", I64), ("msg", ctypes.c_char * 256), ("residual", D)]


class Config(ctypes.Structure):
    _fields_ = [("b", I64), ("c", D), ("compression", I), ("seed", ctypes.c_uint64),
                ("threads", I), ("device", I), ("keep_T", I), ("refine", I),
                ("hbs_tol", D), ("hbs_trunc_rel", D), ("hbs_leaf_size", I64)]


class Stats(ctypes.Structure):
    _fields_ = [("n1", I64), ("n2", I64), ("b", I64), ("interfaces", I64), ("strips", I64),
                ("padded_width", I64), ("single_slab", I), ("symmetric_strips", I),
                ("t_stage1", D), ("t_stage2", D), ("storage_stage1", I64), ("storage_stage2", I64),
                ("device_bytes", I64), ("gpu_launches", I64), ("solve_launches", I64),
                ("t_chain", D), ("t_schur", D), ("t_assemble", D), ("t_solve_last", D),
                ("t_solve_strips", D), ("compression", I), ("hbs_max_rank", I64), ("t_hbs", D)]


class HbsStatsT(ctypes.Structure):
    _fields_ = [("products_normal", I64), ("products_adjoint", I64), ("rounds", I),
                ("final_rank", I64), ("residual_estimate", D)]


class ShardT(ctypes.Structure):
    _fields_ = [("rank", I), ("nranks", I), ("s_begin", I64), ("s_end", I64), ("j_begin", I64),
                ("j_end", I64), ("n_strips", I64), ("n_interfaces", I64)]


FIELD_FN = ctypes.CFUNCTYPE(D, D, D, P)

# exported symbols of include/slablu_gpu.h (checked by tests/test_abi.py)
EXPORTS = [
    "slablu_gpu_assemble_fd5", "slablu_gpu_assemble_canned", "slablu_gpu_sample_solution",
    "slablu_gpu_kappa_from_ppw", "slablu_gpu_bessel_j0", "slablu_gpu_gaussian_matrix",
    "slablu_gpu_choose_b", "slablu_gpu_partition", "slablu_gpu_factorize",
    "slablu_gpu_factorize_device", "slablu_gpu_solve", "slablu_gpu_solve_device",
    "slablu_gpu_stats", "slablu_gpu_T_block", "slablu_gpu_reduce_rhs", "slablu_gpu_destroy",
    "slablu_gpu_device_count", "slablu_gpu_shard_plan", "slablu_gpu_shard_factorize_device",
    "slablu_gpu_shard_sweep", "slablu_gpu_shard_solve_forward", "slablu_gpu_shard_solve_backward",
    "slablu_gpu_shard_eliminate", "slablu_gpu_shard_solve_local",
    "slablu_gpu_residual", "slablu_gpu_sweep_solve", "slablu_gpu_recover",
    "slablu_gpu_sweep_build", "slablu_gpu_set_refine", "slablu_gpu_assemble_canned_device",
    "slablu_gpu_sample_solution_device", "slablu_gpu_error_report", "slablu_gpu_error_report_device",
    "slablu_gpu_save", "slablu_gpu_load", "slablu_gpu_export_sweep", "slablu_gpu_import_sweep",
    "slablu_gpu_hbs_compress",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine with __graft_entry__.build() "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    St = Status
    L.slablu_gpu_assemble_fd5.restype = St
    L.slablu_gpu_assemble_fd5.argtypes = [I64, I64, D, D, FIELD_FN, FIELD_FN, FIELD_FN, P, P, P, P, P, P]
    L.slablu_gpu_assemble_canned.restype = St
    L.slablu_gpu_assemble_canned.argtypes = [I, I64, I64, D, P, P, P, P, P]
    L.slablu_gpu_sample_solution.restype = St
    L.slablu_gpu_sample_solution.argtypes = [I, I64, I64, D, P]
    L.slablu_gpu_kappa_from_ppw.restype = D
    L.slablu_gpu_kappa_from_ppw.argtypes = [D, I64]
    L.slablu_gpu_bessel_j0.restype = D
    L.slablu_gpu_bessel_j0.argtypes = [D]
    L.slablu_gpu_gaussian_matrix.restype = None
    L.slablu_gpu_gaussian_matrix.argtypes = [I64, I64, ctypes.c_uint64, P]
    L.slablu_gpu_choose_b.restype = St
    L.slablu_gpu_choose_b.argtypes = [I64, I64, I64, D, P]
    L.slablu_gpu_partition.restype = St
    L.slablu_gpu_partition.argtypes = [I64, I64, I64, P, P, P, P, I64]
    L.slablu_gpu_factorize.restype = St
    L.slablu_gpu_factorize.argtypes = [I64, I64, P, P, P, P, P]
    L.slablu_gpu_shard_plan.restype = St
    L.slablu_gpu_shard_plan.argtypes = [I64, I64, I64, I, I, P]
    L.slablu_gpu_shard_factorize_device.restype = St
    L.slablu_gpu_shard_factorize_device.argtypes = [I64, I64, I64, P, P, P, P, I, I, P]
    L.slablu_gpu_residual.restype = St
    L.slablu_gpu_residual.argtypes = [P, P, I64, I64, P, I64, P]
    L.slablu_gpu_shard_sweep.restype = St
    L.slablu_gpu_shard_sweep.argtypes = [P, P, P]
    L.slablu_gpu_shard_solve_forward.restype = St
    L.slablu_gpu_shard_solve_forward.argtypes = [P, P, P]
    L.slablu_gpu_shard_eliminate.restype = St
    L.slablu_gpu_shard_eliminate.argtypes = [P]
    L.slablu_gpu_shard_solve_local.restype = St
    L.slablu_gpu_shard_solve_local.argtypes = [P, P, I64, I64]
    L.slablu_gpu_shard_solve_backward.restype = St
    L.slablu_gpu_shard_solve_backward.argtypes = [P, P, P, P, I64]
    L.slablu_gpu_factorize_device.restype = St
    L.slablu_gpu_factorize_device.argtypes = [I64, I64, I64, P, P, P, P, P]
    L.slablu_gpu_solve.restype = St
    L.slablu_gpu_solve.argtypes = [P, P, I64, I64, P, I64]
    L.slablu_gpu_solve_device.restype = St
    L.slablu_gpu_solve_device.argtypes = [P, P, I64, I64, P, I64]
    L.slablu_gpu_stats.restype = St
    L.slablu_gpu_stats.argtypes = [P, P]
    L.slablu_gpu_T_block.restype = St
    L.slablu_gpu_T_block.argtypes = [P, I, I64, P]
    L.slablu_gpu_reduce_rhs.restype = St
    L.slablu_gpu_reduce_rhs.argtypes = [P, P, I64, P]
    L.slablu_gpu_sweep_solve.restype = St
    L.slablu_gpu_sweep_solve.argtypes = [P, P, I64, P]
    L.slablu_gpu_recover.restype = St
    L.slablu_gpu_recover.argtypes = [P, P, P, I64, P]
    L.slablu_gpu_hbs_compress.restype = St
    L.slablu_gpu_hbs_compress.argtypes = [I64, P, I64, I64, I64, I, D, D, ctypes.c_uint64, I, P, P]
    L.slablu_gpu_sweep_build.restype = St
    L.slablu_gpu_sweep_build.argtypes = [I64, I64, P, I, P]
    L.slablu_gpu_set_refine.restype = St
    L.slablu_gpu_set_refine.argtypes = [P, I]
    L.slablu_gpu_assemble_canned_device.restype = St
    L.slablu_gpu_assemble_canned_device.argtypes = [I, I64, I64, D, I, P, P, P, P, P]
    L.slablu_gpu_sample_solution_device.restype = St
    L.slablu_gpu_sample_solution_device.argtypes = [I, I64, I64, D, I, P]
    L.slablu_gpu_error_report.restype = St
    L.slablu_gpu_error_report.argtypes = [I64, P, P, P, P, P, P, I64, I, P]
    L.slablu_gpu_error_report_device.restype = St
    L.slablu_gpu_error_report_device.argtypes = [I64, P, P, P, P, P, P, I64, I, P]
    L.slablu_gpu_save.restype = St
    L.slablu_gpu_save.argtypes = [P, ctypes.c_char_p]
    L.slablu_gpu_load.restype = St
    L.slablu_gpu_load.argtypes = [ctypes.c_char_p, I, P]
    L.slablu_gpu_export_sweep.restype = St
    L.slablu_gpu_export_sweep.argtypes = [P, ctypes.c_char_p]
    L.slablu_gpu_import_sweep.restype = St
    L.slablu_gpu_import_sweep.argtypes = [ctypes.c_char_p, I, P]
    L.slablu_gpu_destroy.restype = None
    L.slablu_gpu_destroy.argtypes = [P]
    L.slablu_gpu_device_count.restype = I
    L.slablu_gpu_device_count.argtypes = []
    for name in EXPORTS:  # every exported entry point has a declared signature
        if getattr(L, name).argtypes is None:
            raise ImportError(f"{name}: ctypes signature not declared in _lib.py")
    _lib = L
    return L

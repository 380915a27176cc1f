"""ctypes declarations of libmgcg.so (include/mgcg.h).  Marshalling only.

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_1909_13585_b200/csrc`).  There is no fallback: if the library is
missing this module raises at import time.
"""

from __future__ import annotations

import ctypes
import os

MG_MAX_RHS = 64
LIB_PATH = os.environ.get("MG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libmgcg.so")

STATUS = {
    0: "MG_OK", 1: "MG_ERR_ARG", 2: "MG_ERR_NONDIVISIBLE", 3: "MG_ERR_DIM", 4: "MG_ERR_MODULUS",
    5: "MG_ERR_BREAKDOWN", 6: "MG_ERR_MAXITER", 7: "MG_ERR_OOM", 8: "MG_ERR_CUDA", 9: "MG_ERR_NCCL",
    10: "MG_ERR_SINGULAR",
}

EXPORTED = [
    "mg_setup", "mg_setup_dist", "mg_partition", "mg_nccl_unique_id", "mg_local_info", "mg_update_modulus",
    "mg_adjoint_rhs", "mg_eigen_sensitivity", "mgcg_block_solve", "mg_multilevel_modes", "mgcg_solve", "stress_stiffness_apply", "mg_matvec", "mg_vcycle",
    "mg_restrict", "mg_prolong", "mg_level_info", "mg_get_diagonal", "mg_get_coarse_inverse",
    "mg_kernel_launches", "mg_profile_kernels", "mg_destroy", "mg_strerror", "mg_last_error",
]


ELEMENTS = {"std": 0, "wilson": 1}


class MgGrid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("nel", ctypes.c_int * 3), ("nu", ctypes.c_double),
                ("element", ctypes.c_int)]


class MgOpts(ctypes.Structure):
    _fields_ = [("omega", ctypes.c_double), ("nu_pre", ctypes.c_int), ("nu_post", ctypes.c_int),
                ("max_iter", ctypes.c_int)]


class MgDist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nslab", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p)]


class MgReport(ctypes.Structure):
    _fields_ = [
        ("nrhs", ctypes.c_int),
        ("iters", ctypes.c_int * MG_MAX_RHS),
        ("relres", ctypes.c_double * MG_MAX_RHS),
        ("true_relres", ctypes.c_double * MG_MAX_RHS),
        ("converged", ctypes.c_int * MG_MAX_RHS),
        ("max_iters", ctypes.c_int),
        ("restarts", ctypes.c_int),
        ("graph_launches", ctypes.c_int),
        ("kernel_launches", ctypes.c_longlong),
        ("solve_ms", ctypes.c_double),
    ]


class MgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {msg}")


def _nccl_path():
    """libnccl.so.2 shipped with torch (nvidia-nccl wheel); the library dlopens it for nranks > 1."""
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:
        pass
    return None


def _load():
    if "MG_NCCL_LIB" not in os.environ:
        p = _nccl_path()
        if p:
            os.environ["MG_NCCL_LIB"] = p
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmgcg.so not built ({LIB_PATH}); run __graft_entry__.build() -- no CPU fallback exists")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, D, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
    sig = {
        "mg_setup": ([ctypes.POINTER(MgGrid), P, P, I, ctypes.POINTER(MgOpts), P, ctypes.POINTER(P)], I),
        "mg_setup_dist": ([ctypes.POINTER(MgGrid), P, P, I, ctypes.POINTER(MgOpts), ctypes.POINTER(MgDist), P,
                           ctypes.POINTER(P)], I),
        "mg_partition": ([ctypes.POINTER(MgGrid), I, I, I, ctypes.POINTER(I), ctypes.POINTER(I)], I),
        "mg_nccl_unique_id": ([P], I),
        "mg_local_info": ([P, ctypes.POINTER(LL), ctypes.POINTER(LL), ctypes.POINTER(I), ctypes.POINTER(I)], I),
        "mg_update_modulus": ([P, P], I),
        "mgcg_solve": ([P, P, I, D, P, ctypes.POINTER(MgReport)], I),
        "mgcg_block_solve": ([P, P, I, D, P, ctypes.POINTER(MgReport)], I),
        "mg_multilevel_modes": ([P, P, P, I, D, P, P, P, P, P], I),
        "stress_stiffness_apply": ([P, P, P, P, I, P], I),
        "mg_adjoint_rhs": ([P, P, P, I, P], I),
        "mg_eigen_sensitivity": ([P, P, P, P, P, P, P, I, P], I),
        "mg_matvec": ([P, I, P, I, P], I),
        "mg_vcycle": ([P, P, I, P], I),
        "mg_restrict": ([P, I, P, I, P], I),
        "mg_prolong": ([P, I, P, I, P], I),
        "mg_level_info": ([P, I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(LL), ctypes.POINTER(ctypes.c_int)], I),
        "mg_get_diagonal": ([P, I, P], I),
        "mg_get_coarse_inverse": ([P, P], I),
        "mg_kernel_launches": ([P], LL),
        "mg_profile_kernels": ([P, I, I, ctypes.POINTER(ctypes.c_double)], I),
        "mg_destroy": ([P], I),
        "mg_strerror": ([I], ctypes.c_char_p),
        "mg_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


lib = _load()


def check(status: int):
    if status != 0:
        raise MgError(status, lib.mg_last_error().decode())

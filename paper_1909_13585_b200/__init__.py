"""B200-native (sm_100a, fp64) fine-grid solve path of Ferrari & Sigmund (arXiv 1909.13585).

Thin Python binding over the C ABI in include/mgcg.h: the functions below have
the C names and only marshal arguments (torch CUDA tensors or host numpy
arrays -> raw pointers).  Every step of the path runs in the CUDA kernels of
libmgcg.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import MgDist, MgError, MgGrid, MgOpts, MgReport, check, lib

__all__ = [
    "Handle", "MgError", "mg_setup", "mg_setup_dist", "mg_partition", "mg_nccl_unique_id", "mg_local_info",
    "mg_update_modulus", "mg_adjoint_rhs", "mg_eigen_sensitivity", "mgcg_block_solve", "mg_multilevel_modes", "mgcg_solve", "stress_stiffness_apply",
    "mg_matvec", "mg_vcycle", "mg_restrict", "mg_prolong", "mg_level_info", "mg_get_diagonal",
    "mg_get_coarse_inverse", "mg_kernel_launches", "mg_profile_kernels", "mg_destroy", "lib_path",
]

lib_path = _lib.LIB_PATH


def _ptr(a, dtype):
    """Raw pointer of a contiguous torch tensor (CUDA or CPU) or numpy array."""
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"expected C-contiguous numpy array of {dtype}, got {a.dtype}")
        return ctypes.c_void_p(a.ctypes.data)
    import torch
    if not isinstance(a, torch.Tensor):
        raise TypeError("expected a torch tensor or numpy array")
    want = {np.float64: torch.float64, np.uint8: torch.uint8}[dtype]
    if a.dtype != want or not a.is_contiguous():
        raise TypeError(f"expected contiguous tensor of {want}, got {a.dtype}")
    return ctypes.c_void_p(a.data_ptr())


def _numel(a):
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _shape(a):
    return tuple(a.shape)


def _need_rows(a, n, name, nrows=None):
    """a must be (nrows, n) -- or (n,) when nrows is 1 -- so the C side never reads or writes out
    of bounds (it trusts the handle's sizes)."""
    sh = _shape(a)
    if len(sh) == 1 and (nrows in (None, 1)) and sh[0] == n:
        return 1
    if len(sh) != 2 or sh[1] != n or (nrows is not None and sh[0] != nrows):
        want = f"({nrows if nrows is not None else 'k'}, {n})"
        raise ValueError(f"{name}: expected shape {want}, got {sh}")
    return sh[0]


def _need_len(a, n, name):
    if _numel(a) != n:
        raise ValueError(f"{name}: expected {n} entries, got {_numel(a)}")


def _level_ndof(h, level):
    if level == 0:
        return h.ndof
    return mg_level_info(h, level)["ndof"]


class Handle:
    """Owns an mg_handle (one design on one grid)."""

    def __init__(self, raw, dim, nel, levels, stream):
        self.raw = raw
        self.dim = dim
        self.nel = tuple(nel)
        self.levels = levels
        self.stream = stream
        self.ndof = dim * int(np.prod([n + 1 for n in nel]))
        self.nelem = int(np.prod(nel))

    def __del__(self):
        try:
            mg_destroy(self)
        except Exception:
            pass


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(getattr(stream, "cuda_stream", stream))


def mg_setup(nel, E, fixed, levels, nu=0.3, omega=0.6, nu_pre=1, nu_post=1, max_iter=1000, stream=None,
             element="std"):
    """element: "std" (bilinear / trilinear) or "wilson" (incompatible modes, NEXT-4)."""
    dim = len(nel)
    g = _grid(nel, nu, element)
    o = MgOpts(omega, nu_pre, nu_post, max_iter)
    raw = ctypes.c_void_p()
    sp = _stream_ptr(stream)
    check(lib.mg_setup(ctypes.byref(g), _ptr(E, np.float64), _ptr(fixed, np.uint8), levels, ctypes.byref(o), sp,
                       ctypes.byref(raw)))
    return Handle(raw, dim, nel, levels, sp)


def _grid(nel, nu=0.3, element="std"):
    dim = len(nel)
    return MgGrid(dim, (ctypes.c_int * 3)(*(list(nel) + [0] * (3 - dim))), nu, _lib.ELEMENTS[element])


def mg_partition(nel, levels, nparts, part):
    """Owned element layers [e_begin, e_end) along axis 0 of slab `part` (host only)."""
    a, b = ctypes.c_int(), ctypes.c_int()
    check(lib.mg_partition(ctypes.byref(_grid(nel)), levels, nparts, part, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def mg_nccl_unique_id():
    """128-byte NCCL unique id (bytes) for mg_setup_dist on nranks > 1."""
    buf = ctypes.create_string_buffer(128)
    check(lib.mg_nccl_unique_id(buf))
    return buf.raw


def mg_setup_dist(nel, E, fixed, levels, rank=0, nranks=1, nslab=1, nccl_id=None, nu=0.3, omega=0.6, nu_pre=1,
                  nu_post=1, max_iter=1000, stream=None, element="std"):
    """Slab-decomposed setup: E / fixed (and all later vectors) cover this rank's owned part
    (mg_local_info); nslab slabs are kept in this handle."""
    dim = len(nel)
    g = _grid(nel, nu, element)
    o = MgOpts(omega, nu_pre, nu_post, max_iter)
    idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    d = MgDist(rank, nranks, nslab, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None)
    raw = ctypes.c_void_p()
    sp = _stream_ptr(stream)
    check(lib.mg_setup_dist(ctypes.byref(g), _ptr(E, np.float64), _ptr(fixed, np.uint8), levels, ctypes.byref(o),
                            ctypes.byref(d), sp, ctypes.byref(raw)))
    h = Handle(raw, dim, nel, levels, sp)
    info = mg_local_info(h)
    h.ndof = info["ndof"]
    h.nelem = info["nelem"]
    h.e_range = (info["e_begin"], info["e_end"])
    return h


def mg_local_info(h):
    nd, ne = ctypes.c_longlong(), ctypes.c_longlong()
    a, b = ctypes.c_int(), ctypes.c_int()
    check(lib.mg_local_info(h.raw, ctypes.byref(nd), ctypes.byref(ne), ctypes.byref(a), ctypes.byref(b)))
    return dict(ndof=nd.value, nelem=ne.value, e_begin=a.value, e_end=b.value)


def mg_update_modulus(h, E):
    _need_len(E, h.nelem, "E")
    check(lib.mg_update_modulus(h.raw, _ptr(E, np.float64)))


def _report(rep, nrhs):
    return dict(
        iters=list(rep.iters[:nrhs]), relres=list(rep.relres[:nrhs]), true_relres=list(rep.true_relres[:nrhs]),
        converged=list(rep.converged[:nrhs]), max_iters=rep.max_iters, restarts=rep.restarts,
        graph_launches=rep.graph_launches, kernel_launches=rep.kernel_launches, solve_ms=rep.solve_ms,
    )


def mgcg_solve(h, rhs, tol, x, raise_on_error=True):
    """Solve K x_k = rhs_k for all rows of rhs (nrhs, ndof); x is written in place."""
    nrhs = _need_rows(rhs, h.ndof, "rhs")
    _need_rows(x, h.ndof, "x", nrhs)
    rep = MgReport()
    st = lib.mgcg_solve(h.raw, _ptr(rhs, np.float64), nrhs, tol, _ptr(x, np.float64), ctypes.byref(rep))
    out = _report(rep, nrhs)
    out["status"] = _lib.STATUS.get(st, st)
    if raise_on_error:
        check(st)
    return out


def mgcg_block_solve(h, rhs, tol, x, raise_on_error=True):
    """Block PCG (mgBPCG) over all rows of rhs (nrhs, ndof); x written in place."""
    nrhs = _need_rows(rhs, h.ndof, "rhs")
    _need_rows(x, h.ndof, "x", nrhs)
    rep = MgReport()
    st = lib.mgcg_block_solve(h.raw, _ptr(rhs, np.float64), nrhs, tol, _ptr(x, np.float64), ctypes.byref(rep))
    out = _report(rep, nrhs)
    out["status"] = _lib.STATUS.get(st, st)
    if raise_on_error:
        check(st)
    return out


def mg_multilevel_modes(h, Es, u, q, Phi, tol=1e-10, y1=None, with_residual=False):
    """Sec. 2.1 multilevel modes: fills Phi (q, ndof) with K-normalised modes and returns
    (lam_tilde, lam_coarse) lists, plus (||y||, ||y|| / ||K phi~_1||) of the Eq. 7 residual
    y = (K + lam~_1 G) phi~_1 when with_residual (y1, if given, receives y)."""
    _need_len(Es, h.nelem, "Es")
    _need_len(u, h.ndof, "u")
    _need_rows(Phi, h.ndof, "Phi", q)
    if y1 is not None:
        _need_len(y1, h.ndof, "y1")
    lt = np.zeros(q)
    lc = np.zeros(q)
    yr = np.zeros(2)
    check(lib.mg_multilevel_modes(h.raw, _ptr(Es, np.float64), _ptr(u, np.float64), q, tol, _ptr(Phi, np.float64),
                                  _ptr(lt, np.float64), _ptr(lc, np.float64),
                                  _ptr(y1, np.float64) if y1 is not None else None,
                                  _ptr(yr, np.float64) if with_residual else None))
    if with_residual:
        return list(lt), list(lc), (float(yr[0]), float(yr[1]))
    return list(lt), list(lc)


def stress_stiffness_apply(h, Es, u, phi, y):
    _need_len(Es, h.nelem, "Es")
    _need_len(u, h.ndof, "u")
    nphi = _need_rows(phi, h.ndof, "phi")
    _need_rows(y, h.ndof, "y", nphi)
    check(lib.stress_stiffness_apply(h.raw, _ptr(Es, np.float64), _ptr(u, np.float64), _ptr(phi, np.float64),
                                     phi.shape[0], _ptr(y, np.float64)))


def mg_adjoint_rhs(h, Es, phi, b):
    """b_i = phi_i^T (grad_u G) phi_i (Eq. 5 right-hand sides), device tensors."""
    _need_len(Es, h.nelem, "Es")
    nphi = _need_rows(phi, h.ndof, "phi")
    _need_rows(b, h.ndof, "b", nphi)
    check(lib.mg_adjoint_rhs(h.raw, _ptr(Es, np.float64), _ptr(phi, np.float64), phi.shape[0], _ptr(b, np.float64)))


def mg_eigen_sensitivity(h, dEk, dEs, u, phi, z, lam, out):
    """Eq. 4 element sensitivities for nphi modes (device tensors; lam: sequence of nphi floats)."""
    lam_arr = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
    _need_len(dEk, h.nelem, "dEk")
    _need_len(dEs, h.nelem, "dEs")
    _need_len(u, h.ndof, "u")
    nphi = _need_rows(phi, h.ndof, "phi")
    _need_rows(z, h.ndof, "z", nphi)
    _need_len(lam_arr, nphi, "lam")
    _need_len(out, nphi * h.nelem, "out")
    check(lib.mg_eigen_sensitivity(h.raw, _ptr(dEk, np.float64), _ptr(dEs, np.float64), _ptr(u, np.float64),
                                   _ptr(phi, np.float64), _ptr(z, np.float64), _ptr(lam_arr, np.float64),
                                   phi.shape[0], _ptr(out, np.float64)))


def mg_matvec(h, level, x, y):
    n = _level_ndof(h, level)
    k = _need_rows(x, n, "x")
    _need_rows(y, n, "y", k)
    check(lib.mg_matvec(h.raw, level, _ptr(x, np.float64), x.shape[0], _ptr(y, np.float64)))


def mg_vcycle(h, r, z):
    k = _need_rows(r, h.ndof, "r")
    _need_rows(z, h.ndof, "z", k)
    check(lib.mg_vcycle(h.raw, _ptr(r, np.float64), r.shape[0], _ptr(z, np.float64)))


def mg_restrict(h, level, fine, coarse):
    k = _need_rows(fine, _level_ndof(h, level), "fine")
    _need_rows(coarse, _level_ndof(h, level + 1), "coarse", k)
    check(lib.mg_restrict(h.raw, level, _ptr(fine, np.float64), fine.shape[0], _ptr(coarse, np.float64)))


def mg_prolong(h, level, coarse, fine):
    k = _need_rows(coarse, _level_ndof(h, level + 1), "coarse")
    _need_rows(fine, _level_ndof(h, level), "fine", k)
    check(lib.mg_prolong(h.raw, level, _ptr(coarse, np.float64), coarse.shape[0], _ptr(fine, np.float64)))


def mg_level_info(h, level):
    nel = (ctypes.c_int * 3)()
    ndof = ctypes.c_longlong()
    nl = ctypes.c_int()
    check(lib.mg_level_info(h.raw, level, nel, ctypes.byref(ndof), ctypes.byref(nl)))
    return dict(nel=tuple(nel[:h.dim]), ndof=ndof.value, nlevels=nl.value)


def mg_get_diagonal(h, level, d):
    _need_len(d, _level_ndof(h, level), "d")
    check(lib.mg_get_diagonal(h.raw, level, _ptr(d, np.float64)))


def mg_get_coarse_inverse(h, A):
    check(lib.mg_get_coarse_inverse(h.raw, _ptr(A, np.float64)))


def mg_kernel_launches(h):
    return int(lib.mg_kernel_launches(h.raw))


def mg_profile_kernels(h, nrhs, reps=10):
    """Standalone timings (ms per launch) of the fine-level kernels of one CG iteration."""
    ms = (ctypes.c_double * 4)()
    check(lib.mg_profile_kernels(h.raw, nrhs, reps, ms))
    return dict(cgp=ms[0], restrict=ms[1], post=ms[2], matvec=ms[3])


def mg_destroy(h):
    if h is not None and getattr(h, "raw", None):
        lib.mg_destroy(h.raw)
        h.raw = None

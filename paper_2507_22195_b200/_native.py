"""ctypes binding of libmhdg_b200.so (C ABI in include/mhdg_b200.h).

No CPU fallback: if the library or a CUDA device is missing every operator
raises NativeUnavailable.  Status codes map 1:1 onto the reference's
exception classes (macrohdg/errors.py).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (
    InvalidConfig,
    NativeUnavailable,
    NonAdmissibleEntropyState,
    NonAdmissibleState,
    SingularBlock,
    SingularLocalMatrix,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MHDG_LIB") or os.path.join(HERE, "libmhdg_b200.so")

MHDG_OK = 0
_WHERE = ("volume sub", "face tile", "trace tile")

dptr = C.c_void_p


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("where_kind", C.c_int), ("where_index", C.c_int),
                ("item", C.c_int64), ("n_unsym", C.c_int)]


class Tables(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("p", C.c_int), ("m", C.c_int),
        ("n_macros", C.c_int), ("n_faces", C.c_int),
        ("nn", C.c_int), ("nq", C.c_int), ("nfn", C.c_int), ("nqf", C.c_int),
        ("n_st", C.c_int), ("n_sub", C.c_int),
        ("formulation", C.c_int), ("flux_kind", C.c_int), ("gamma", C.c_double),
        ("phi", dptr), ("dphi", dptr), ("quad_wts", dptr), ("phi_face", dptr),
        ("fphi", dptr), ("facet_wts", dptr), ("face_rows", dptr), ("sub_det", dptr),
        ("sub_inv_jac", dptr), ("face_normals", dptr), ("face_area", dptr),
        ("face_id_st", dptr), ("trace_idx", dptr), ("boundary_st", dptr),
        ("face_sides", dptr), ("freestream", dptr), ("n_owned_faces", C.c_int),
        ("has_visc", C.c_int), ("reynolds", C.c_double), ("mach", C.c_double),
        ("prandtl", C.c_double), ("mu", C.c_double), ("minv_ref", dptr), ("pref", dptr),
        ("kref", dptr), ("eref", dptr),
        ("nc", C.c_int), ("nt", C.c_int), ("scatter", dptr), ("sub_det_all", dptr),
        ("sub_inv_jac_all", dptr), ("trace_ptr", dptr), ("trace_list", dptr),
        ("face_ptr", dptr), ("face_list", dptr),
    ]


class KrylovParams(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("restart", C.c_int), ("max_outer", C.c_int),
                ("inner_rtol", C.c_double), ("inner_iters", C.c_int), ("inner_precond", C.c_int),
                ("inner_true_residual", C.c_int), ("outer_matvec_reuse", C.c_int)]


class KrylovStats(C.Structure):
    _fields_ = [("outer_iterations", C.c_int), ("inner_iterations", C.c_int),
                ("converged", C.c_int), ("updated", C.c_int), ("rel_residual", C.c_double)]


class LinBuffers(C.Structure):
    _fields_ = [("sinv", dptr), ("hw", dptr), ("hhat", dptr), ("hh", dptr), ("pinv", dptr),
                ("wlin", dptr)]


_SIGS = {
    "mhdg_create": (C.c_void_p, [C.POINTER(Tables), C.c_int, C.POINTER(C.c_int)]),
    "mhdg_destroy": (None, [C.c_void_p]),
    "mhdg_lin_sizes": (None, [C.c_void_p, C.POINTER(C.c_int64)]),
    "mhdg_residual": (C.c_int, [C.c_void_p, dptr, dptr, dptr, C.c_int, C.c_double, dptr, C.c_int,
                                dptr, dptr, dptr, C.c_int, C.POINTER(Status), C.c_void_p]),
    "mhdg_solve_gradient": (C.c_int, [C.c_void_p, dptr, dptr, dptr, C.c_void_p]),
    "mhdg_status_fetch": (C.c_int, [C.c_void_p, C.POINTER(Status), C.c_void_p]),
    "mhdg_linearize": (C.c_int, [C.c_void_p, dptr, dptr, dptr, C.c_double, C.c_double,
                                 C.POINTER(LinBuffers), C.POINTER(Status), C.c_void_p]),
    "mhdg_linearize_local": (C.c_int, [C.c_void_p, dptr, dptr, dptr, C.c_double, C.c_double,
                                       C.POINTER(LinBuffers), C.POINTER(Status), C.c_void_p]),
    "mhdg_precond_factor": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), C.c_int, dptr, dptr, dptr,
                                      C.POINTER(Status), C.c_void_p]),
    "mhdg_axpy_dev": (C.c_int, [C.c_void_p, C.c_int64, dptr, dptr, dptr, C.c_void_p]),
    "mhdg_matvec": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, C.c_void_p]),
    "mhdg_matvec_range": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, C.c_int64,
                                    C.c_int64, C.c_int, C.c_int, C.c_void_p]),
    "mhdg_residual_range": (C.c_int, [C.c_void_p, dptr, dptr, dptr, C.c_int, C.c_double, dptr, C.c_int,
                                      dptr, dptr, dptr, C.c_int64, C.c_int64, C.c_int, C.c_void_p]),
    "mhdg_condensed_rhs": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, dptr, dptr,
                                     C.c_void_p]),
    "mhdg_recover": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, dptr, dptr, dptr,
                               C.c_void_p]),
    "mhdg_precond": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, C.c_void_p]),
    "mhdg_volume_quad_states": (C.c_int, [C.c_void_p, dptr, dptr, C.POINTER(Status), C.c_void_p]),
    "mhdg_to_conservative": (C.c_int, [C.c_void_p, C.c_int64, dptr, dptr, C.POINTER(Status),
                                       C.c_void_p]),
    "mhdg_from_conservative": (C.c_int, [C.c_void_p, C.c_int64, dptr, dptr, C.c_void_p]),
    "mhdg_integrals": (C.c_int, [C.c_void_p, dptr, C.POINTER(C.c_double), C.c_void_p]),
    "mhdg_entropy_identity": (C.c_int, [C.c_void_p, dptr, dptr, dptr, dptr, C.POINTER(C.c_double),
                                        C.c_void_p]),
    "mhdg_dissipation": (C.c_int, [C.c_void_p, dptr, dptr, C.POINTER(C.c_double), C.c_void_p]),
    "mhdg_dot": (C.c_int, [C.c_void_p, C.c_int64, dptr, dptr, dptr, C.c_void_p]),
    "mhdg_mgs": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, dptr, dptr, dptr, C.c_void_p]),
    "mhdg_combine": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, dptr, dptr, dptr, C.c_void_p]),
    "mhdg_scale": (C.c_int, [C.c_void_p, C.c_int64, dptr, C.c_double, dptr, C.c_int, dptr,
                             C.c_void_p]),
    "mhdg_axpby": (C.c_int, [C.c_void_p, C.c_int64, C.c_double, dptr, C.c_double, dptr, dptr,
                             C.c_void_p]),
    "mhdg_krylov_workspace": (C.c_int64, [C.c_void_p, C.POINTER(KrylovParams)]),
    "mhdg_krylov_create": (C.c_void_p, [C.c_void_p, C.POINTER(KrylovParams), dptr, C.c_int64,
                                        C.POINTER(C.c_int)]),
    "mhdg_krylov_solve": (C.c_int, [C.c_void_p, C.POINTER(LinBuffers), dptr, dptr, dptr, C.c_int,
                                    C.c_void_p]),
    "mhdg_krylov_destroy": (None, [C.c_void_p]),
    "mhdg_gj_fallbacks": (C.c_int, [C.c_void_p, dptr, C.c_void_p]),
    "mhdg_batched_inverse": (C.c_int, [C.c_void_p, C.c_int, C.c_int, dptr, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mhdg_launch_count": (C.c_int64, [C.c_void_p]),
    "mhdg_fp64_probe": (C.c_double, [C.c_int, C.c_void_p]),
    "mhdg_dmma_probe": (C.c_double, [C.c_int, C.c_void_p]),
    "mhdg_math_eval": (C.c_int, [C.c_int, C.c_int64, dptr, dptr, C.c_void_p]),
    "mhdg_pair_sides": (C.c_int64, [C.c_int64, C.c_int, dptr, dptr]),
    "mhdg_match_points": (C.c_double, [C.c_int64, C.c_int, C.c_int, dptr, dptr, dptr]),
    "mhdg_match_faces": (C.c_double, [C.c_int64, C.c_int, C.c_int, dptr, dptr, dptr, dptr, dptr, dptr,
                                      dptr, dptr]),
    "mhdg_side_keys": (None, [C.c_int64, C.c_int, dptr, dptr, dptr, dptr, C.c_double, dptr]),
    "mhdg_face_shift_perm": (C.c_double, [C.c_int64, C.c_int, dptr, dptr, dptr, dptr, dptr]),
    "mhdg_version": (C.c_char_p, []),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path=LIB_PATH):
    """Load the shared library (no GPU needed); raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(f"{path} not built; run __graft_entry__.build()")
    try:
        lib = C.CDLL(path)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the HDG operator runs only on "
                                "the GPU (no CPU fallback)")
    return load()


def ptr(t):
    # plain ints: every pointer parameter is declared c_void_p, so ctypes
    # converts without a wrapper object per argument
    return None if t is None else t.data_ptr()


def np_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_raw_stream = None


def stream_handle():
    """Raw cudaStream_t of the current device's current stream (the cheap
    torch binding: this is called once per kernel-level entry point)."""
    global _raw_stream
    if _raw_stream is None:
        import torch

        get, dev = torch._C._cuda_getCurrentRawStream, torch._C._cuda_getDevice
        _raw_stream = lambda: get(dev())  # noqa: E731
    return _raw_stream()


def raise_for(code, st=None, context=""):
    """Map a library status onto the reference's exception classes."""
    if code == MHDG_OK:
        return
    item = None if st is None else int(st.item)
    if code in (1, 2):
        where = f"{_WHERE[st.where_kind]} {st.where_index}"
        msg = (f"non-admissible state at {where}, first at macro {item}" if code == 1
               else f"non-positive inverse temperature at {where}, macro {item}")
        cls = NonAdmissibleState if code == 1 else NonAdmissibleEntropyState
        raise cls(msg, where=where)
    if code == 3:
        raise SingularLocalMatrix(f"singular condensed block on macro {item}", macro=item)
    if code == 4:
        raise SingularBlock(f"singular trace block on face {item}")
    if code == 5:
        raise InvalidConfig(f"configuration not supported by the B200 operator {context}")
    if code == 7:
        raise MemoryError(f"device allocation failed {context}")
    raise RuntimeError(f"CUDA error in libmhdg_b200 ({code}) {context}")


def dmma_probe(device=0):
    lib = require_cuda()
    return float(lib.mhdg_dmma_probe(device, stream_handle()))


def math_eval(fn, x):
    """Device elementary function (0 exp, 1 log, 2 reciprocal) on a CUDA
    float64 tensor (accuracy tests)."""
    import torch

    lib = require_cuda()
    x = x.contiguous()
    y = torch.empty_like(x)
    raise_for(lib.mhdg_math_eval(fn, x.numel(), ptr(x), ptr(y), stream_handle()), context="(math_eval)")
    return y


def host_library():
    """The library for its host-only entry points (table builder); None when
    it is not built (the numpy builder is then used)."""
    try:
        return load()
    except NativeUnavailable:
        return None


def fp64_probe(device=0):
    lib = require_cuda()
    return float(lib.mhdg_fp64_probe(device, stream_handle()))

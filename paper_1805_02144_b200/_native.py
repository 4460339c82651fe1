"""ctypes binding of libeik.so (include/eik.h).

The library is built in-tree (``python build.py`` / ``__graft_entry__.build``)
and loaded from the package directory.  There is no fallback: if the shared
object or a CUDA device is missing, every entry point raises.
"""

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EIK_LIB") or os.path.join(_HERE, "libeik.so")

EIK_OK, EIK_EINVAL, EIK_ENONFINITE, EIK_EPHIPM, EIK_ECUDA, EIK_ENOMEM, EIK_ECALLBACK = range(7)
SCHEME_IDS = {"rb_euler": 0, "epi3": 1, "exprb42": 2, "pexprb43": 3,
              "exprb53": 4}
SLOT_IDS = {"rbe": 0, "epi3": 1, "exprb42/1": 2, "exprb42/2": 3,
            "pexprb43/1": 4, "pexprb43/2": 5, "exprb53/1": 6,
            "exprb53/2": 7, "exprb53/3": 8}


class EikCsrView(C.Structure):
    _fields_ = [("nnz", C.c_int64), ("indptr", C.POINTER(C.c_int32)),
                ("indices", C.POINTER(C.c_int32)),
                ("data", C.POINTER(C.c_double))]


class EikPhiTask(C.Structure):
    _fields_ = [("p", C.c_int32), ("v", C.POINTER(C.POINTER(C.c_double))),
                ("ns", C.c_int32), ("rho", C.POINTER(C.c_double)),
                ("tol", C.c_double), ("m_init", C.c_int32),
                ("iom", C.c_int32), ("m_max", C.c_int32),
                ("delta", C.c_double), ("tau_init", C.c_double),
                ("zero_skip", C.c_int32), ("max_attempts", C.c_int64)]


class EikPhipmInfo(C.Structure):
    _fields_ = [("substeps", C.c_int64), ("rejections", C.c_int64),
                ("matvecs", C.c_int64), ("tau_final", C.c_double),
                ("m_final", C.c_int64), ("t_reached", C.c_double),
                ("attempts", C.c_int64), ("skipped", C.c_int32),
                ("status", C.c_int32)]


class EikTraceRec(C.Structure):
    _fields_ = [("attempt", C.c_int64), ("t", C.c_double), ("tau", C.c_double),
                ("m", C.c_int64), ("eps_m", C.c_double), ("omega", C.c_double),
                ("accepted", C.c_int64)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
# int (*eik_matvec_fn)(void* user, const double* x, double* y, int64_t n)
MATVEC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _D, _D, C.c_int64)
_SIGS = {
    "eik_last_error": (C.c_char_p, []),
    "eik_version": (C.c_int, []),
    "eik_tile_order": (C.c_int, [C.c_int64, _D, _D, _D, C.c_int32, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32)]),
    "eik_swe_create": (C.c_int, [C.c_int32, C.POINTER(EikCsrView), _D, _D, _D,
                                 _D, _D, C.c_double, C.c_double, C.c_int32,
                                 C.c_int32, C.POINTER(_P)]),
    "eik_swe_destroy": (C.c_int, [_P]),
    "eik_swe_set_state": (C.c_int, [_P, _D]),
    "eik_swe_get_state": (C.c_int, [_P, _D]),
    "eik_swe_set_prev": (C.c_int, [_P, _D]),
    "eik_swe_rhs": (C.c_int, [_P, _D, _D]),
    "eik_swe_jv": (C.c_int, [_P, _D, _D, _D]),
    "eik_swe_jac_nnz": (C.c_int, [_P, _D, C.POINTER(C.c_int64)]),
    "eik_swe_jac_nnz_rows": (C.c_int, [_P, _D, C.POINTER(C.c_int64), _D]),
    "eik_swe_diagnostics": (C.c_int, [_P, _D, _D, C.c_double, _D]),
    "eik_swe_phipm": (C.c_int, [_P, _D, C.c_double, C.POINTER(EikPhiTask), _D,
                                C.POINTER(EikPhipmInfo), C.POINTER(EikTraceRec),
                                C.c_int64, C.POINTER(C.c_int64)]),
    "eik_swe_step": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double,
                               C.POINTER(EikPhipmInfo), C.POINTER(C.c_int32)]),
    "eik_swe_advance": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double,
                                  C.c_int32, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64)]),
    "eik_swe_seeds": (C.c_int, [_P, C.c_int32, _D, C.POINTER(C.c_int64),
                                C.c_int32]),
    "eik_swe_reset_seeds": (C.c_int, [_P]),
    "eik_swe_snapshot": (C.c_int, [_P, C.c_int32]),
    "eik_swe_krylov_bench": (C.c_int, [_P, _D, _D, C.c_double, C.c_int32, C.c_int32, _D]),
    "eik_swe_info": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "eik_prof_read": (C.c_int, [_D, C.c_int]),
    "eik_swe_launches": (C.c_int64, [_P]),
    "eik_swe_last_kernel_ms": (C.c_double, [_P]),
    "eik_swe_set_hostloop": (C.c_int, [_P, C.c_int32]),
    "eik_swe_sweep_timing": (C.c_int, [_P, _D, C.POINTER(C.c_int64), C.c_int32]),
    "eik_swe_krylov_iters": (C.c_int64, [_P]),
    "eik_swe_explicit_orth": (C.c_int64, [_P]),
    "eik_csr_create": (C.c_int, [C.c_int32, EikCsrView, C.c_int32, C.c_int32,
                                 C.POINTER(_P)]),
    "eik_csr_destroy": (C.c_int, [_P]),
    "eik_csr_phipm": (C.c_int, [_P, C.c_double, C.c_int64,
                                C.POINTER(EikPhiTask), _D,
                                C.POINTER(EikPhipmInfo), C.POINTER(EikTraceRec),
                                C.c_int64, C.POINTER(C.c_int64)]),
    "eik_cb_create": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "eik_cb_destroy": (C.c_int, [_P]),
    "eik_cb_phipm": (C.c_int, [_P, MATVEC_FN, C.c_void_p, C.c_double, C.c_int64,
                               C.POINTER(EikPhiTask), _D, C.POINTER(EikPhipmInfo),
                               C.POINTER(EikTraceRec), C.c_int64, C.POINTER(C.c_int64)]),
}
EXPORTED = tuple(_SIGS)

_lib = None


class NativeError(RuntimeError):
    pass


def load():
    """Load libeik.so once; raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"libeik.so not built ({LIB_PATH}); run `python build.py` "
                "-- there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def dptr(a):
    return a.ctypes.data_as(_D)


def check(status, what=""):
    """Map eik_status to the reference's exception types."""
    if status == EIK_OK:
        return
    msg = load().eik_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (EIK_EINVAL, EIK_ENONFINITE):
        raise ValueError(text)
    if status == EIK_ENOMEM:
        raise MemoryError(text)
    raise NativeError(text)


def csr_view(mat):
    """EikCsrView over a scipy CSR (keeps the int32/float64 copies alive)."""
    import scipy.sparse as sp
    csr = mat.csr if hasattr(mat, "csr") else mat
    csr = sp.csr_matrix(csr)
    indptr = np.ascontiguousarray(csr.indptr, dtype=np.int32)
    indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
    data = np.ascontiguousarray(csr.data, dtype=np.float64)
    view = EikCsrView(int(csr.nnz), indptr.ctypes.data_as(C.POINTER(C.c_int32)),
                      indices.ctypes.data_as(C.POINTER(C.c_int32)), dptr(data))
    return view, (indptr, indices, data)


def make_task(v, rho, tol, m_init, iom, m_max, delta, tau_init, zero_skip,
              max_attempts):
    """EikPhiTask + keep-alive list; ``v`` entries that are all zero are
    still passed (the device computes the exact any-nonzero flags)."""
    keep = []
    arr = (C.POINTER(C.c_double) * len(v))()
    for l, vl in enumerate(v):
        a = np.ascontiguousarray(vl, dtype=np.float64)
        keep.append(a)
        arr[l] = dptr(a)
    r = np.ascontiguousarray(rho, dtype=np.float64)
    keep.append(r)
    keep.append(arr)
    t = EikPhiTask(len(v) - 1, C.cast(arr, C.POINTER(C.POINTER(C.c_double))),
                   len(rho), dptr(r), float(tol), int(m_init), int(iom),
                   int(m_max), float(delta),
                   float(tau_init) if tau_init else -1.0, int(bool(zero_skip)),
                   int(max_attempts))
    return t, keep

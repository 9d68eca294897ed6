"""ctypes binding of libsks.so (include/sks.h).  Argument marshalling only: every step
of the path runs in the library's CUDA kernels.  There is no CPU fallback -- if the
library or a CUDA device is missing, calls raise."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(HERE, "libsks.so")

SKS_OK, SKS_EINVAL, SKS_ECUDA, SKS_ENCCL, SKS_ENOMEM, SKS_ENOTCONV, SKS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "SKS_OK", -1: "SKS_EINVAL", -2: "SKS_ECUDA", -3: "SKS_ENCCL", -4: "SKS_ENOMEM",
                -5: "SKS_ENOTCONV", -6: "SKS_EUNSUPPORTED"}
SKS_WARN_COND, SKS_WARN_BREAKDOWN, SKS_WARN_STAGNATION, SKS_INFO_ADAPTIVE_RESTART = 1, 2, 4, 8
SKS_INFO_STABILIZED = 16
STABILIZE = {"off": 0, "if_ill": 1, "always": 2}  # SKS_SRR_STABILIZE_*
SKS_OP_STENCIL2D, SKS_OP_STENCIL3D, SKS_OP_CSR = 1, 2, 3

# every symbol include/sks.h declares (checked by tests/test_abi.py)
EXPORTS = ["sks_get_unique_id", "sks_create", "sks_destroy", "sks_last_error", "sks_abi_version",
           "sks_set_stream", "sks_partition", "sks_sgmres_solve", "sks_srr_eigs", "sks_sketch_apply",
           "sks_sketch_table", "sks_apply_operator", "sks_basis", "sks_srft_apply", "sks_loopback_create",
           "sks_loopback_destroy", "sks_create_loopback"]


class Operator(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_int32), ("m", C.c_int64), ("beta", C.c_double),
                ("n_global", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("val", C.c_void_p),
                ("nnz_local", C.c_int64)]


class SgmresOpts(C.Structure):
    _fields_ = [("d", C.c_int32), ("k", C.c_int32), ("s", C.c_int32), ("zeta", C.c_int32),
                ("seed", C.c_uint64), ("tol", C.c_double), ("max_cycles", C.c_int32),
                ("sketch_batch", C.c_int32), ("early_exit_factor", C.c_double), ("cond_tol", C.c_double),
                ("flags", C.c_int32), ("time_stride", C.c_int32), ("basis", C.c_int32), ("sketch", C.c_int32),
                ("cheb_c", C.c_double), ("cheb_dx", C.c_double), ("cheb_dy", C.c_double)]


class SgmresInfo(C.Structure):
    _fields_ = [("cycles", C.c_int32), ("columns", C.c_int32), ("columns_generated", C.c_int32),
                ("flags", C.c_int32), ("rel_res_true", C.c_double), ("r_est", C.c_double),
                ("cond_T", C.c_double), ("t_total_s", C.c_double), ("t_basis_s", C.c_double),
                ("bytes_basis", C.c_double), ("kernel_launches", C.c_int64), ("steps", C.c_int64),
                ("t_step_s", C.c_double), ("steps_timed", C.c_int64), ("bytes_step", C.c_double)]


SKS_OPT_TIME_STEPS = 1
SKS_OPT_ADAPTIVE_RESTART = 2
SKS_OPT_WHITEN = 8
SKS_INFO_WHITEN = 32
SKS_OPT_ZERO_X0 = 4
SKS_BASIS_ARNOLDI, SKS_BASIS_CHEBYSHEV, SKS_BASIS_BLOCK_CHEBYSHEV = 0, 1, 2
BASES = {"arnoldi": SKS_BASIS_ARNOLDI, "chebyshev": SKS_BASIS_CHEBYSHEV, "block_chebyshev": SKS_BASIS_BLOCK_CHEBYSHEV}
SKS_SKETCH_SPARSE, SKS_SKETCH_SRFT = 0, 1
SKETCHES = {"sparse": SKS_SKETCH_SPARSE, "srft": SKS_SKETCH_SRFT}


class SrrOpts(C.Structure):
    _fields_ = [("d", C.c_int32), ("k", C.c_int32), ("s", C.c_int32), ("zeta", C.c_int32),
                ("seed", C.c_uint64), ("cond_tol", C.c_double), ("basis", C.c_int32), ("sketch", C.c_int32),
                ("stabilize", C.c_int32), ("block", C.c_int32),
                ("cheb_c", C.c_double), ("cheb_dx", C.c_double), ("cheb_dy", C.c_double)]


class SrrInfo(C.Structure):
    _fields_ = [("columns", C.c_int32), ("flags", C.c_int32), ("nev_out", C.c_int32), ("rank", C.c_int32),
                ("cond_SB", C.c_double), ("t_total_s", C.c_double), ("t_basis_s", C.c_double),
                ("t_small_s", C.c_double), ("bytes_basis", C.c_double), ("kernel_launches", C.c_int64),
                ("steps", C.c_int64)]


_lib = None


def load(path: str = LIBPATH):
    """Load libsks.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libsks.so not built at {path}; run `python -m paper_2111_00113_b200.build` "
                           "(no CPU fallback exists)")
    lib = C.CDLL(path)
    P, V, I32, I64, U32, U64, D = C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    sig = {
        "sks_get_unique_id": (C.c_int, [P]),
        "sks_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, P]),
        "sks_destroy": (C.c_int, [P]),
        "sks_loopback_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "sks_loopback_destroy": (C.c_int, [P]),
        "sks_create_loopback": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, P]),
        "sks_last_error": (C.c_char_p, [P]),
        "sks_abi_version": (C.c_int, []),
        "sks_set_stream": (C.c_int, [P, P]),
        "sks_partition": (C.c_int, [C.c_int, I64, I64, C.c_int, C.c_int, C.POINTER(I64), C.POINTER(I64)]),
        "sks_sgmres_solve": (C.c_int, [P, C.POINTER(Operator), P, P, C.POINTER(SgmresOpts),
                                       C.POINTER(SgmresInfo), P, I64, P, I64]),
        "sks_srr_eigs": (C.c_int, [P, C.POINTER(Operator), P, C.POINTER(SrrOpts), I32, I32,
                                   P, P, P, P, P, P, C.POINTER(SrrInfo)]),
        "sks_sketch_apply": (C.c_int, [P, I64, I64, I64, I32, I32, U64, U32, P, I64, I32, P]),
        "sks_sketch_table": (C.c_int, [P, I64, I64, I32, I32, U64, U32, P, P]),
        "sks_srft_apply": (C.c_int, [P, I64, I32, U64, U32, P, I32, P]),
        "sks_apply_operator": (C.c_int, [P, C.POINTER(Operator), P, P]),
        "sks_basis": (C.c_int, [P, C.POINTER(Operator), P, I32, I32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib

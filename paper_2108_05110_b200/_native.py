"""ctypes binding of the C ABI (include/ensmhd_b200.h) -- plain pointers only.

The library is built in-tree by ``build.py``; on a machine with a GPU the
product path refuses to run without it (no CPU fallback exists).
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ENS_LIB", os.path.join(HERE, "libensmhd_b200.so"))   # ENS_LIB: A/B builds only

ENS_OK, ENS_EINVAL, ENS_ENOMEM, ENS_ENOCONV, ENS_ECUDA = range(5)

P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double


class MeshDesc(C.Structure):
    _fields_ = [
        ("ns", I32), ("n_pres", I32), ("nt", I32), ("nnz_s", I32), ("J", I32), ("ncolor", I32), ("ncons", I32),
        ("pad0", I32),
        ("s_rowptr", P), ("s_col", P), ("s_mass", P), ("s_stiff", P),
        ("bt_rowptr", P), ("bt_col", P), ("bt_val", P),
        ("b_rowptr", P), ("b_col", P), ("b_val", P),
        ("cflag", P),
        ("e_nodes", P), ("e_geo", P), ("e_slots", P), ("color_off_host", P),
        ("cons_row", P), ("cons_bidx", P), ("pres_int", P),
        ("area", F64), ("mean_zero", I32), ("pad1", I32),
        ("n2e_ptr", P), ("n2e", P), ("s2e_ptr", P), ("s2e", P),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("nfront", I32), ("nlevels", I32), ("pw", I32), ("tile", I32),
        ("front_storage", I64), ("n_orig", I64), ("n_cmap", I64), ("n_idx", I64), ("n_work", I64),
        ("f_m", P), ("f_k", P), ("f_off", P), ("f_idx_off", P), ("f_idx", P), ("f_parent", P),
        ("f_cmap_off", P), ("f_cmap", P), ("orig_dst", P), ("orig_src", P), ("bsrc_vals", P), ("work", P),
        ("gsrc", P),
        ("orig_level_off_host", P), ("level_storage_off_host", P), ("level_front_off_host", P),
        ("sched_factor_host", P), ("n_sched_factor", I64),
        ("sched_fwd_host", P), ("n_sched_fwd", I64),
        ("sched_bwd_host", P), ("n_sched_bwd", I64),
        ("max_m", I32), ("split_k", I32), ("n_slot", I64),
    ]


class DataDesc(C.Structure):
    _fields_ = [("K", I32), ("pad", I32), ("rows", I64), ("basis", P), ("coef", P), ("dense", P)]


SYMBOLS = [
    "ens_abi_version", "ens_last_error", "ens_kernel_launches", "ens_create", "ens_set_pivoting",
    "ens_destroy", "ens_workspace_bytes", "ens_stream_split_launches",
    "ens_lincomb", "ens_member_sums", "ens_means", "ens_rhs", "ens_member_pass", "ens_rhs_fused", "ens_apply_bc", "ens_assemble", "ens_factor",
    "ens_solve", "ens_solve_begin", "ens_solve_finish", "ens_spmm", "ens_precond_apply", "ens_epilogue", "ens_diagnostics", "ens_mean_error",
    "ens_layout_import", "ens_layout_export", "ens_state_upload",
]

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the library.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_2108_05110_b200.build` "
                           "(there is no CPU fallback for the time-step path)")
    lib = C.CDLL(path)
    lib.ens_abi_version.restype = C.c_int
    lib.ens_last_error.restype = C.c_char_p
    lib.ens_kernel_launches.restype = C.c_int64
    lib.ens_create.argtypes = [C.POINTER(MeshDesc), C.POINTER(PlanDesc), C.c_int, C.POINTER(P)]
    lib.ens_destroy.argtypes = [P]
    lib.ens_destroy.restype = None
    lib.ens_workspace_bytes.argtypes = [P, C.POINTER(I64)]
    lib.ens_set_pivoting.argtypes = [P, C.c_int]
    lib.ens_stream_split_launches.argtypes = [P]
    lib.ens_stream_split_launches.restype = C.c_int
    lib.ens_member_sums.argtypes = [P, P, P, P]
    lib.ens_means.argtypes = [P, P, P, F64, P]
    lib.ens_mean_error.argtypes = [P, P, P, C.POINTER(DataDesc), P]
    lib.ens_lincomb.argtypes = [P, P, F64, P, F64, P]
    lib.ens_rhs.argtypes = [P, P, P, P, F64, C.POINTER(DataDesc), P]
    lib.ens_member_pass.argtypes = [P, P, P, P, P, P]
    lib.ens_rhs_fused.argtypes = [P, P, P, P, P, F64, C.POINTER(DataDesc), P, P]
    lib.ens_apply_bc.argtypes = [P, P, C.POINTER(DataDesc), P]
    lib.ens_assemble.argtypes = [P, P, P, P, P, F64, P]
    lib.ens_factor.argtypes = [P, P, P, C.POINTER(I32)]
    lib.ens_solve.argtypes = [P, P, P, P, P, F64, I32, I32, C.POINTER(I32), C.POINTER(F64)]
    lib.ens_solve_begin.argtypes = [P, P, P, P, P, F64, I32, I32]
    lib.ens_solve_finish.argtypes = [P, P, P, P, P, F64, I32, I32, C.POINTER(I32), C.POINTER(F64)]
    lib.ens_spmm.argtypes = [P, P, P, P, P, P, C.c_int]
    lib.ens_precond_apply.argtypes = [P, P, P, P]
    lib.ens_epilogue.argtypes = [P, P, P, P]
    lib.ens_diagnostics.argtypes = [P, P, P, P, P]
    lib.ens_layout_import.argtypes = [P, P, P, I64, I64, I64, P, P, I64, I32]
    lib.ens_layout_export.argtypes = [P, P, P, I64, I64, P, P, I64, I64, I32]
    lib.ens_state_upload.argtypes = [P, P, P, P, I64, P, P, P, I64]
    for name in SYMBOLS:
        if name not in ("ens_abi_version", "ens_last_error", "ens_destroy", "ens_kernel_launches"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


class NativeError(RuntimeError):
    def __init__(self, code, where, msg):
        super().__init__(f"{where}: status {code}: {msg}")
        self.code = code


def check(code: int, where: str):
    if code == ENS_OK:
        return
    msg = _lib.ens_last_error().decode(errors="replace") if _lib is not None else ""
    if code == ENS_EINVAL:
        raise ValueError(f"{where}: {msg}")
    if code == ENS_ENOMEM:
        raise MemoryError(f"{where}: {msg}")
    raise NativeError(code, where, msg)

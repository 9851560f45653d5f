"""ctypes binding of the in-tree C-ABI library (include/pipecg_b200.h).

There is no fallback: if ``_lib/libpipecg_b200.so`` is missing or no CUDA
device is visible, every compute call raises.  Build with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2105_06176_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["PIPECG_B200_LIB"]) if os.environ.get("PIPECG_B200_LIB") else _HERE / "_lib" / "libpipecg_b200.so"  # env: experiments only
CSRC = _HERE / "csrc"

PCG_OK = 0
PCG_EPARSE, PCG_EIO = 1007, 1008
PCG_EINVAL, PCG_ENOMEM, PCG_ESTATE, PCG_ERANGE, PCG_EDIAG, PCG_ECOMM = (1001, 1002, 1003, 1004,
                                                                    1005, 1006)
PCG_DOT_TREE, PCG_DOT_SEQ = 0, 1
PCG_RUNNING, PCG_STOPPED, PCG_BREAKDOWN = 0, 1, 2
BREAKDOWN_QUANTITY = {1: "alpha denominator", 2: "gamma", 3: "delta"}

_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_p_i64 = ctypes.POINTER(ctypes.c_int64)
_p_dbl = ctypes.POINTER(ctypes.c_double)


class PcgMatrix(ctypes.Structure):
    _fields_ = [
        ("n_rows", _i64), ("n_cols", _i64), ("nnz", _i64), ("rp64", _int),
        ("rowptr", _vp), ("col", _vp), ("val", _vp), ("inv_diag", _vp),
    ]


class PcgOptions(ctypes.Structure):
    _fields_ = [("dot_mode", _int), ("engine", _int), ("chunk", _int), ("use_graphs", _int),
                ("max_sms", _int)]


class PcgResult(ctypes.Structure):
    _fields_ = [
        ("status", _int), ("converged", _int), ("iterations", _i64), ("final_norm", _dbl),
        ("norm0", _dbl), ("breakdown_quantity", _int), ("breakdown_iteration", _i64),
        ("breakdown_value", _dbl), ("n_history", _i64), ("n_drift", _i64), ("engine", _int),
        ("graph_launches", _i64), ("tune_ms", _dbl * 9), ("pattern_flags", _int),
    ]


class NativeError(RuntimeError):
    """A C-ABI call failed (CUDA error or invalid use of the ABI)."""

    def __init__(self, fn: str, code: int, msg: str):
        self.code = code
        super().__init__(f"{fn} failed with code {code}: {msg}")


_lib = None

PCG_H2D_COPY64, PCG_H2D_I64_TO_I32 = 0, 1

_SIGS = {
    "pipecg_b200_last_error": ([], ctypes.c_char_p),
    "pipecg_b200_version": ([], ctypes.c_char_p),
    "pipecg_b200_spmv": ([_i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "pipecg_b200_residual": ([_i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "pipecg_b200_jacobi_apply": ([_i64, _vp, _vp, _vp, _vp], _int),
    "pipecg_b200_jacobi_setup": ([_i64, _int, _vp, _vp, _vp, _vp, _p_i64,
                                  ctypes.POINTER(_int), _vp], _int),
    "pipecg_b200_fused_update": ([_i64] + [_vp] * 10 + [_dbl, _dbl, _vp], _int),
    "pipecg_b200_fused_update_pc_dots": ([_i64] + [_vp] * 11 + [_dbl, _dbl, _int, _vp, _vp, _vp],
                                         _int),
    "pipecg_b200_dots": ([_i64, _int, _vp, _vp, _int, _vp, _vp, _vp], _int),
    "pipecg_b200_dots_workspace_bytes": ([], _i64),
    "pipecg_b200_narrow_i64": ([_i64, _vp, _vp, ctypes.POINTER(_int), _vp], _int),
    "pipecg_b200_h2d": ([_vp, _vp, _i64, _int, _vp], _int),
    "pipecg_b200_h2d_multi": ([_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _p_i64,
                               ctypes.POINTER(_int), _vp], _int),
    "pipecg_b200_d2h": ([_vp, _vp, _i64, _vp], _int),
    "pipecg_b200_host_prefault": ([_vp, _i64], _int),
    "pipecg_b200_mm_parse": ([ctypes.c_char_p, _i64, _int, ctypes.POINTER(_vp)], _int),
    "pipecg_b200_mm_read": ([ctypes.c_char_p, ctypes.POINTER(_vp)], _int),
    "pipecg_b200_mm_error_line": ([], _i64),
    "pipecg_b200_mm_info": ([_vp, _p_i64, _p_i64, _p_i64], _int),
    "pipecg_b200_mm_to_csr": ([_vp, _int, _vp, _vp, _vp, _p_i64, _vp], _int),
    "pipecg_b200_mm_free": ([_vp], None),
    "pipecg_b200_find_long_rows": ([_i64, _int, _vp, _i64, _vp, _i64, _p_i64, _vp], _int),
    "pipecg_b200_row_patterns": ([_i64, _int, _vp, _vp, _vp, _p_i64, _p_i64, _vp, _vp], _int),
    "pipecg_b200_stencil_shape": ([_int, _i64, _p_i64, _p_i64], _int),
    "pipecg_b200_stencil_prefix": ([_int, _i64, _i64, _p_i64], _int),
    "pipecg_b200_stencil_fill": ([_int, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp], _int),
    "pipecg_b200_solver_create": ([ctypes.POINTER(PcgMatrix), ctypes.POINTER(PcgOptions),
                                   ctypes.POINTER(_vp)], _int),
    "pipecg_b200_solver_destroy": ([_vp], _int),
    "pipecg_b200_solver_init": ([_vp, _vp, _vp, _dbl, _i64, _i64, _vp], _int),
    "pipecg_b200_solver_run": ([_vp, ctypes.POINTER(PcgResult), _p_dbl, _i64, _p_i64, _p_dbl, _i64],
                               _int),
    "pipecg_b200_solver_enqueue": ([_vp, _i64], _int),
    "pipecg_b200_solver_prepare": ([_vp, _i64], _int),
    "pipecg_b200_solver_stream": ([_vp], _vp),
    "pipecg_b200_solver_poll": ([_vp, ctypes.POINTER(PcgResult)], _int),
    "pipecg_b200_tune_cache_clear": ([], None),
    "pipecg_b200_solver_x": ([_vp], _vp),
    "pipecg_b200_solver_state": ([_vp, ctypes.POINTER(_vp)], _int),
    "pipecg_b200_solver_comm_info": ([_vp, ctypes.POINTER(_vp), _p_i64, ctypes.POINTER(_vp)], _int),
    "pipecg_b200_ipc_get_handle": ([_vp, _vp], _int),
    "pipecg_b200_ipc_open": ([_vp, ctypes.POINTER(_vp)], _int),
    "pipecg_b200_ipc_close": ([_vp], _int),
    "pipecg_b200_enable_peer_access": ([_int, _int], _int),
    "pipecg_b200_solver_connect": ([_vp, _int, _int, _vp, _vp, _vp, _i64, _vp, _vp, _vp], _int),
    "pipecg_b200_solve_host": ([_i64, _p_i64, _p_i64, _p_dbl, _p_dbl, _p_dbl, _p_dbl, _dbl, _i64,
                                _i64, _int, _p_dbl, _p_dbl, _i64, _p_i64, _p_dbl, _i64,
                                ctypes.POINTER(PcgResult)], _int),
}

EXPORTED = tuple(_SIGS)


def build(verbose: bool = False) -> Path:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    r = subprocess.run(["make", "-j8", "-C", str(CSRC)], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"building {LIB_PATH} failed:\n{r.stdout}\n{r.stderr}")
    return LIB_PATH


def load():
    """Load the library (no GPU needed to load it; compute calls need one)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'). "
                "There is no CPU fallback."
            )
        L = ctypes.CDLL(os.fspath(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    msg = load().pipecg_b200_last_error()
    return msg.decode() if msg else ""


def check(fn_name: str, rc: int) -> None:
    if rc != PCG_OK:
        raise NativeError(fn_name, rc, last_error())


def call(fn_name: str, *args) -> int:
    rc = getattr(load(), fn_name)(*args)
    check(fn_name, rc)
    return rc

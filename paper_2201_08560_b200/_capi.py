"""ctypes binding of the C ABI in include/b2sr_sm100.h (libb2sr_sm100.so).

This is the FFI layer a Python package uses to reach native code.  There is
no fallback: if the library is missing or cannot be loaded, every hot-path
call raises ``RuntimeError`` -- the package never silently computes on the
CPU.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import FormatError

_LIB_PATH = Path(__file__).resolve().parent / "libb2sr_sm100.so"

OK, EINVAL, EFORMAT, ECUDA, ENOMEM, ENOCONV = range(6)
RING = {"boolean": 0, "arithmetic": 1, "minplus": 2, "maxtimes": 3}

P = ctypes.c_void_p
u32, i32, u64, i64, f64 = ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
PP = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (every function returns int status unless listed in _RESTYPE)
SIGNATURES = {
    "b2sr_last_error": [],
    "b2sr_version": [],
    "b2sr_launch_count": [],
    "b2sr_from_csr": [u32, u32, P, P, u64, P, PP],
    "b2sr_from_host": [u32, u32, P, P, P, u64, P, PP],
    "b2sr_profile_rows": [u32, u32, P, P, P, u32, P, P, P],
    "b2sr_free": [P],
    "b2sr_info": [P, P, P, P, P],
    "b2sr_arrays": [P, P, P, P],
    "b2sr_to_host": [P, P, P, P, P],
    "b2sr_transpose": [P, P, PP],
    "b2sr_equal": [P, P, P, P],
    "b2sr_to_csr_rowptr": [P, P, P, P],
    "b2sr_to_csr_fill": [P, P, P, P],
    "b2sr_drop_diagonal": [P, P, PP],
    "b2sr_row_block": [P, u32, u32, P, PP],
    "b2sr_set_kernel_timing": [ctypes.c_int],
    "b2sr_last_kernel_ms": [P],
    "b2sr_block_from_host": [u32, u32, u32, u32, P, P, P, u64, P, PP],
    "b2sr_row_offset": [P, P],
    "b2sr_used_columns": [P, P, P],
    "b2sr_bmv_bbb": [P, P, P, P, P],
    "b2sr_bmv_bbf": [P, P, P, P, P],
    "b2sr_bmv_bff": [P, P, i32, f64, P, P, P, P, P],
    "b2sr_bmv_bff_ex": [P, P, i32, f64, f64, P, P, P, P, P],
    "b2sr_h2d": [P, P, u64, P],
    "b2sr_from_host_checked": [u32, u32, P, P, P, u64, P, PP],
    "b2sr_validate": [P, P],
    "b2sr_comm_unique_id": [P],
    "b2sr_comm_init": [P, i32, i32, PP],
    "b2sr_comm_init_local": [i32, P],
    "b2sr_comm_free": [P],
    "b2sr_comm_allreduce_sum_i64": [P, P, u64, P],
    "b2sr_dist_bfs_plan": [P, P, P, P, PP],
    "b2sr_dist_bfs_plan_blocks": [P, P, P, P, P, P, PP],
    "b2sr_dist_bfs_rows": [P, P, P],
    "b2sr_dist_bfs_run": [P, u32, P, P, P],
    "b2sr_dist_bfs_free": [P],
    "b2sr_dist_tc": [P, P, P, P, P],
    "b2sr_bmm_sum": [P, P, P, P],
    "b2sr_bmm_sum_masked_bt": [P, P, P, P, P],
    "b2sr_bfs": [P, P, u32, P, P, P],
    "b2sr_bfs_init": [u32, u32, u32, P, P, P, P],
    "b2sr_bfs_sweep": [P, P, P, P, P],
    "b2sr_bfs_update": [u32, u32, P, P, P, f64, P, P],
    "b2sr_tc_work": [P, P, P, P],
    "b2sr_pr_step": [u32, f64, f64, P, P, P, P, P, P],
    "b2sr_pairwise_sum": [P, u64, P, P],
    "b2sr_min_relax": [u64, P, P, P, P],
    "b2sr_bfs_sweep_ex": [P, P, P, P, i32, P],
    "b2sr_bfs_update_ex": [u32, u32, P, P, P, f64, P, P, P],
    "b2sr_sssp": [P, u32, P, P, P],
    "b2sr_pagerank": [P, P, f64, f64, i64, P, P, P, P, P],
    "b2sr_cc": [P, P, P, P],
    "b2sr_tc": [P, P, P],
    "b2sr_csr_lower_rowptr": [u32, P, P, P, P, P],
    "b2sr_csr_lower_fill": [u32, P, P, P, P, P],
    "b2sr_csr_orient_rowptr": [u32, P, P, P, P, P],
    "b2sr_csr_orient_fill": [u32, P, P, P, P, P],
    "b2sr_rmat_edges": [i32, u64, u64, P, P, P],
    "b2sr_coo_to_csr": [u32, u64, P, P, i32, i32, P, P, P, P],
}
_RESTYPE = {"b2sr_last_error": ctypes.c_char_p, "b2sr_launch_count": u64}

_lib = None
_lock = threading.Lock()


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """Load the library once; raise loudly when it is not there."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not _LIB_PATH.exists():
                    raise RuntimeError(
                        f"{_LIB_PATH.name} is not built; run `python -m paper_2201_08560_b200._build` "
                        "(there is no CPU fallback)")
                L = ctypes.CDLL(str(_LIB_PATH))
                for name, args in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPE.get(name, ctypes.c_int)
                _lib = L
    return _lib


def check(status: int):
    """Map a C status code onto the reference's exception classes."""
    if status == OK:
        return
    msg = (lib().b2sr_last_error() or b"").decode(errors="replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status == EFORMAT:
        raise FormatError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(lib().b2sr_launch_count())

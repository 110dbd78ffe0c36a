"""ctypes binding of the C ABI in include/rac_b200.h.

The shared library is built in-tree (paper_1907_01995_b200/lib/librac_b200.so,
`python -m paper_1907_01995_b200.build`).  There is NO fallback: if the
library or a CUDA device is missing, every solver entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "librac_b200.so")

RAC_OK, RAC_ERR_ARG, RAC_ERR_CUDA, RAC_ERR_NOT_PD, RAC_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
MODE_RAC, MODE_RP, MODE_CYCLIC = 0, 1, 2
STATUS_MAX_ITERS, STATUS_CONVERGED, STATUS_DIVERGED = 0, 1, 2
KERNEL_LINEAR, KERNEL_GAUSSIAN = 0, 1
LAYOUT_ROW_MAJOR, LAYOUT_COL_MAJOR = 0, 1
GRAM_BLOCKS, GRAM_COVARIANCE = 0, 1

_p = C.c_void_p
_i32, _i64, _f64, _sz = C.c_int32, C.c_int64, C.c_double, C.c_size_t
_pi32 = C.POINTER(C.c_int32)
_pf64 = C.POINTER(C.c_double)

# name -> (restype, argtypes); mirrors include/rac_b200.h one to one
SIGNATURES = {
    "rac_version": (C.c_char_p, []),
    "rac_last_error": (C.c_char_p, []),
    "rac_launch_count": (C.c_uint64, []),
    "rac_trim_pool": (_i32, [C.c_uint64]),
    "rac_device_check": (_i32, [_i32]),
    "rac_chunk_sort": (_i32, [_p, _i64, _i32, _i32, _p, _p]),
    "rac_gram_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "rac_gram_inverse": (_i32, [_p, _i64, _i64, _p, _i32, _i32, _i64, _f64, _f64, _p, _p, _p, _p]),
    "rac_z_prox": (_i32, [_p, _p, _i64, _f64, _f64, _f64, _p, _p]),
    "rac_en_create": (_i32, [C.POINTER(_p), _i64, _i64, _i32, _i32, _f64, _f64, _f64, _p]),
    "rac_en_set_data": (_i32, [_p, _p, _i32, _p]),
    "rac_en_set_data_rows": (_i32, [_p, _p, _i64, _i64, _p]),
    "rac_en_set_data_csc": (_i32, [_p, _p, _p, _p, _p]),
    "rac_en_set_gram_mode": (_i32, [_p, _i32]),
    "rac_en_set_partition": (_i32, [_p, _p]),
    "rac_en_run": (_i32, [_p, _p, _i32, _f64]),
    "rac_en_progress": (_i32, [_p, _pi32, _pi32, _pf64, _pi32]),
    "rac_en_poll": (_i32, [_p, _i32, _pi32, _pi32, _pi32]),
    "rac_en_get": (_i32, [_p, _p, _p, _p, _p]),
    "rac_en_history": (_i32, [_p, _p, _p, _i32]),
    "rac_en_set_timing": (_i32, [_p, _i32]),
    "rac_en_timing": (_i32, [_p, _pf64, _pi32]),
    "rac_en_timing_slicing": (_i32, [_p, _pf64]),
    "rac_en_trace": (_i32, [_p, C.POINTER(C.c_int64), _i32]),
    "rac_debug_buffer": (_i32, [_p]),
    "rac_gram_covariance": (_i32, [_p, _i64, _i64, _i32, _p, _f64, _i32]),
    "rac_en_reset": (_i32, [_p, _f64, _f64, _f64]),
    "rac_en_info": (_i32, [_p, _pi32]),
    "rac_en_gram_slices": (_i32, [_p, _pi32]),
    "rac_en_destroy": (_i32, [_p]),
    "rac_qp_create": (_i32, [C.POINTER(_p), _i64, _i64, _i32, _i32, _f64, _f64, _p]),
    "rac_qp_set_problem": (_i32, [_p, _p, _p, _p, _p, _p, _p]),
    "rac_qp_borrow_h": (_i32, [_p, _p]),
    "rac_qp_set_state": (_i32, [_p, _p, _p]),
    "rac_qp_set_kernel_strips": (_i32, [_p, _p, _i64, _p, _i32, _f64, C.c_uint64]),
    "rac_consensus_run": (_i32, [_p, _i32, _p]),
    "rac_svm_kernel_strip": (_i32, [_p, _i64, _i64, _p, _p, _i32, _i32, _f64, _p, _p]),
    "rac_qp_set_divergence_bar": (_i32, [_p, _f64]),
    "rac_qp_set_partition": (_i32, [_p, _p]),
    "rac_qp_run": (_i32, [_p, _p, _i32, _f64, _f64, _i32]),
    "rac_qp_progress": (_i32, [_p, _pi32, _pi32, _pi32]),
    "rac_qp_get": (_i32, [_p, _p, _p, _p, _p]),
    "rac_qp_history": (_i32, [_p, _p, _p, _p, _i32]),
    "rac_qp_set_trace": (_i32, [_p, _i32]),
    "rac_qp_trace": (_i32, [_p, C.POINTER(C.c_int64), _i32]),
    "rac_qp_destroy": (_i32, [_p]),
    "rac_svm_build_q": (_i32, [_p, _i64, _i64, _p, _i32, _f64, _p, _p]),
    "rac_gemv": (_i32, [_p, _i64, _i64, _p, _p, _p]),
    "rac_box_block_min": (_i32, [_p, _p, _p, _p, _i32, _p, _p, _p]),
}


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rac_b200 error {code}: {msg}")
        self.code = code


MISSING: list[str] = []   # header symbols the loaded library does not export
_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"rac_b200 native library not found at {path}; build it with "
                    "`python -m paper_1907_01995_b200.build` (there is no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                try:
                    fn = getattr(lib, name)
                except AttributeError:
                    MISSING.append(name)
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def check(code: int) -> None:
    if code != RAC_OK:
        msg = load().rac_last_error().decode(errors="replace")
        raise NativeError(code, msg)


_device_ok = False


def require_device(device: int = 0) -> None:
    """Fail loudly unless a B200 (sm_100) is visible."""
    global _device_ok
    if _device_ok:
        return
    check(load().rac_device_check(device))
    _device_ok = True

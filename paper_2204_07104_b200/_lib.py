"""ctypes binding of libsptk.so (include/sptk.h).

The shared library is built in-tree (``__graft_entry__.build()`` /
``make -C paper_2204_07104_b200/csrc``).  There is deliberately no fallback:
if the library or a CUDA device is missing, every hot-path entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPTK_LIB: an alternative in-tree build (experiment variants, e.g.
# libsptk_<variant>.so next to the default)
LIB_PATH = os.path.join(_HERE, os.environ.get("SPTK_LIB", "libsptk.so"))

_c_i32p = ctypes.c_void_p
_vp = ctypes.c_void_p
_i64 = ctypes.c_longlong
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); the declarations of include/sptk.h
SIGNATURES = {
    "sptk_last_error": (ctypes.c_char_p, []),
    "sptk_version": (ctypes.c_int, []),
    "sptk_launch_count": (ctypes.c_longlong, []),
    "sptk_reset_launch_count": (None, []),
    "sptk_record_words": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "sptk_set_tc_mode": (ctypes.c_int, [ctypes.c_int]),
    "sptk_get_tc_mode": (ctypes.c_int, []),
    "sptk_last_factor_kernel": (ctypes.c_char_p, []),
    "sptk_debug_tc_buffer": (None, [_vp]),
    "sptk_fma_rank": (ctypes.c_int, [ctypes.c_int]),
    "sptk_pcg64_seed": (ctypes.c_int, [_u64p, ctypes.c_int, _u64p]),
    "sptk_block_job_bytes": (ctypes.c_size_t, []),
    "sptk_block_perm": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _i64, ctypes.c_int,
                                       _vp, _vp, _vp]),
    "sptk_interleave_rounds": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _vp, _i64, _vp]),
    "sptk_permutation_ws_bytes": (ctypes.c_size_t, [_i64]),
    "sptk_permutation": (ctypes.c_int, [_u64p, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_permute_records": (ctypes.c_int, [_u64p, _i64, _vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_permutation_j_ws_bytes": (ctypes.c_size_t, [_i64]),
    "sptk_fy_apply_ws_bytes": (ctypes.c_size_t, [_i64]),
    "sptk_permutation_j_batch_ws_bytes": (ctypes.c_size_t, [_i64p, ctypes.c_int]),
    "sptk_permutation_j_batch": (ctypes.c_int, [_u64p, _i64p, _i64p, ctypes.c_int, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_fy_globalize": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp]),
    "sptk_fy_apply": (ctypes.c_int, [_vp, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_permutation_j": (ctypes.c_int, [_u64p, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_choice_ws_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "sptk_choice": (ctypes.c_int, [_u64p, _i64, _i64, ctypes.c_int, _vp, _vp, ctypes.c_size_t,
                                   ctypes.POINTER(ctypes.c_int), _vp]),
    "sptk_u32_stream": (ctypes.c_int, [_u64p, ctypes.c_ulonglong, _i64, _vp, _vp]),
    "sptk_h2d": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, ctypes.c_int]),
    "sptk_coo_text_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp),
                                           _i64p, ctypes.POINTER(ctypes.c_int)]),
    "sptk_coo_text_dims": (ctypes.c_int, [_vp, _i64p, ctypes.POINTER(ctypes.c_int)]),
    "sptk_coo_text_take": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int]),
    "sptk_coo_text_free": (None, [_vp]),
    "sptk_partition_ws_bytes": (ctypes.c_size_t, [_i64, ctypes.c_int, _i64]),
    "sptk_partition": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, _i64p, _i64, ctypes.c_int, _vp, _vp,
                                      _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "sptk_h2d_pack": (ctypes.c_int, [_vp, _vp, _vp, _i64, ctypes.c_int, ctypes.c_int]),
    "sptk_partition_records": (ctypes.c_int, [_vp, _i64, ctypes.c_int, _i64p, _i64, _vp, _vp, _vp, _vp, _vp,
                                              ctypes.c_size_t, _vp]),
    "sptk_pack_records": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp]),
    "sptk_factor_pass": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _i64, _vp, _i64p, _vp, _i64p, _i64p,
                                        ctypes.c_int, ctypes.c_int, _f64p, _f64p, ctypes.c_int, _vp]),
    "sptk_factor_pass_f64": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _i64, _vp, _i64p, _vp, _i64p,
                                            _i64p, ctypes.c_int, ctypes.c_int, _f64p, _f64p, ctypes.c_int,
                                            _vp]),
    "sptk_factor_pass_exact_ws_bytes": (ctypes.c_size_t, [_i64, ctypes.c_int]),
    "sptk_factor_pass_exact": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _i64, _vp, _i64p, _vp, _i64p, _i64p,
                                              ctypes.c_int, ctypes.c_int, _f64p, _f64p, _vp, ctypes.c_size_t, _vp]),
    "sptk_factor_pass_exact_f64": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _i64, _vp, _i64p, _vp, _i64p,
                                                  _i64p, ctypes.c_int, ctypes.c_int, _f64p, _f64p, _vp,
                                                  ctypes.c_size_t, _vp]),
    "sptk_factor_pass_dsgd": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _vp, _i64p, _vp, _i64p, _i64p,
                                             ctypes.c_int, ctypes.c_int, _f64p, _f64p, _vp, _vp, _vp, _vp, _vp,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]),
    "sptk_dsgd_push_bytes": (ctypes.c_size_t, []),
    "sptk_flag_store": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    "sptk_shared_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_vp)]),
    "sptk_shared_free": (ctypes.c_int, [_vp]),
    "sptk_ipc_get": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "sptk_ipc_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "sptk_ipc_close": (ctypes.c_int, [_vp]),
    "sptk_core_ws_bytes": (ctypes.c_size_t, [_i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "sptk_core_pass": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _i64, _vp, _i64p, _vp, _i64p, _i64p,
                                      ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_size_t,
                                      _vp]),
    "sptk_core_pass_f64": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _i64, _vp, _i64p, _vp, _i64p, _i64p,
                                          ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp,
                                          ctypes.c_size_t, _vp]),
    "sptk_core_apply": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, _vp]),
    "sptk_core_apply_f64": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, _vp]),
    "sptk_eval": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _vp, _i64p, _vp, _i64p, _i64p, ctypes.c_int,
                                 ctypes.c_int, _vp, _vp, _vp]),
    "sptk_eval_f64": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _vp, _i64p, _vp, _i64p, _i64p, ctypes.c_int,
                                     ctypes.c_int, _vp, _vp, _vp]),
}

_lib = None


class SptkError(RuntimeError):
    """A libsptk entry point returned a nonzero status."""


def load():
    """Load libsptk.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().sptk_last_error().decode(errors="replace")
        raise SptkError(f"{what} failed (status {rc}): {msg}")


def i64arr(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return a, a.ctypes.data_as(_i64p)


def f64arr(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(_f64p)


def u64arr(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return a, a.ctypes.data_as(_u64p)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2204_07104_b200 needs a CUDA device (sm_100a); none is visible")
    load()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream

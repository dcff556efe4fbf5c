"""ctypes binding of the C-ABI (include/dlx_b200.h) — the only way Python reaches the device.

The library is built in-tree (paper_2506_21263_b200/libdlx_b200.so). There is no fallback:
if the shared library is missing or does not load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DLX_LIB overrides the library path (A/B experiments between two builds)
LIB_PATH = os.environ.get("DLX_LIB") or os.path.join(HERE, "libdlx_b200.so")

# Exception taxonomy of the reference (errors.hpp:8-34) + device/collective failures.
class Error(RuntimeError):
    """dilocox::Error"""


class ValidationError(Error):
    pass


class ShapeError(Error):
    pass


class FormatError(Error):
    pass


class NumericError(Error):
    pass


class IoError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


STATUS = {1: ValidationError, 2: ShapeError, 3: FormatError, 4: NumericError, 5: IoError,
          6: CudaError, 7: NcclError}

_vp, _i64, _u64, _i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
_ip, _i64p, _u64p, _dp = C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_double)
_f, _d = C.c_float, C.c_double

# name: (restype, argtypes)
PROTOS = {
    "dlx_version": (C.c_char_p, []),
    "dlx_last_error": (C.c_char_p, []),
    "dlx_ctx_create": (_i32, [_i32, C.POINTER(_vp)]),
    "dlx_ctx_destroy": (_i32, [_vp]),
    "dlx_layout_create": (_i32, [_vp, _i32, _ip, _i64p, C.POINTER(_vp)]),
    "dlx_layout_destroy": (_i32, [_vp]),
    "dlx_layout_slab_elems": (_i64, [_vp]),
    "dlx_layout_offsets": (_i32, [_vp, _i64p]),
    "dlx_factor_offsets": (_i64, [_vp, _i32, _i32, _i64p]),
    "dlx_payload_bytes": (_i64, [_vp, _i32, _i32]),
    "dlx_payload_segments": (_i32, [_vp, _i32, _i32, _i64p]),
    "dlx_payload_bits": (_u64, [_vp, _i32, _i32]),
    "dlx_fill_gaussian": (_i32, [_vp, _vp, _vp, _vp, _f, _u64, _u64, _u64, _vp]),
    "dlx_compress": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _u64, _vp, _i32, _vp, _vp,
                            _vp, _vp]),
    "dlx_quantize_factors": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _u64, _i32, _vp,
                                    _vp, _vp]),
    "dlx_decompress": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "dlx_allreduce_avg": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "dlx_outer_update": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp,
                                _f, _f, _i32, _vp, _vp]),
    "dlx_outer_update_range": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp,
                                      _vp, _f, _f, _i32, _vp, _i32, _i32, _vp]),
    "dlx_outer_update_raw": (_i32, [_vp, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _f, _f,
                                    _i32, _vp, _vp]),
    "dlx_adamw_step": (_i32, [_vp, _i64, _f, _f, _f, _f, _f, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp]),
    "dlx_stage_deltas": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dlx_nesterov": (_i32, [_vp, _i64, _f, _f, _i32, _vp, _vp, _vp, _vp]),
    "dlx_effective_rank": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _d, _vp, _vp, _vp]),
    "dlx_effective_rank_shard": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _d, _i32, _i32, _vp, _vp,
                                        _vp]),
    "dlx_effective_rank_reduce": (_i32, [_vp, _ip, _dp, _i32, _ip, _ip]),
    "dlx_adapt_compression": (_i32, [_ip, _i32, _i32, _i32, _i32, _i32, _ip, _ip]),
    "dlx_omega_bound": (_d, [_i32, _i32, _i32]),
    "dlx_serialize": (_i64, [_vp, _i32, _i32, C.POINTER(C.c_char_p), _vp, _vp, _i64]),
    "dlx_parse": (_i32, [_vp, _i32, _i32, _vp, _i64, _vp]),
    "dlx_take_launch_count": (_u64, []),
    "dlx_set_option": (_i32, [C.c_char_p, _i32]),
    "dlx_kernel_time": (_i32, [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dlx_debug_sweep": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "dlx_measure_error": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "dlx_sqdiff_slabs": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "dlx_mean_slabs": (_i32, [_vp, _i64, _i64, _i32, _vp, _vp, _vp]),
    # worker sync (NCCL inside the library)
    "dlx_comm_unique_id": (_i32, [_vp]),
    "dlx_comm_init": (_i32, [_vp, _i32, _i32, _vp]),
    "dlx_ctx_create_dist": (_i32, [_i32, _i32, _i32, _vp, C.POINTER(_vp)]),
    "dlx_comm_info": (_i32, [_vp, _ip, _ip]),
    "dlx_exchange": (_i32, [_vp, _vp, _i64, _vp, _vp, _i64, _i32, _vp]),
    "dlx_exchange_wait_warm": (_i32, [_vp, _vp]),
    "dlx_comm_allgather": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "dlx_comm_allreduce_sum_f64": (_i32, [_vp, _vp, _i64, _vp]),
    "dlx_comm_check": (_i32, [_vp]),
    "dlx_comm_destroy": (_i32, [_vp]),
}

_lib = None


def lib():
    """Load libdlx_b200.so (fails loudly; there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python paper_2506_21263_b200/build.py)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().dlx_last_error().decode(errors="replace")
        raise STATUS.get(status, Error)(msg)


def exported_symbols():
    return list(PROTOS)

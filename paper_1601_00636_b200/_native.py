"""ctypes binding of libcuboid_gpu.so (include/cuboid_gpu.h).

The product path has no CPU fallback: if the library is missing, or no CUDA
device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CUBOID_GPU_LIB", os.path.join(HERE, "libcuboid_gpu.so"))

# status codes (cuboid_gpu.h)
OK = 0
P_BELOW_152, P_ABOVE_LIMIT, Q_BELOW_LOW, Q_ABOVE_HIGH, NOT_LOADED = 2, 3, 4, 5, 6
ERR_CUDA, ERR_INVALID, ERR_OVERFLOW, ERR_FORMAT, ERR_RANGE, ERR_CAPACITY, ERR_NO_DEVICE, ERR_IO = (
    -1, -2, -3, -4, -5, -6, -7, -8)
REGION, TRIANGLE = 0, 1
BUILD_PRODUCTION, BUILD_EXHAUSTIVE = 0, 1

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)

# name -> (restype, argtypes); every symbol include/cuboid_gpu.h declares
SIGNATURES = {
    "cgpu_last_error": (C.c_char_p, []),
    "cgpu_version": (C.c_char_p, []),
    "cgpu_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "cgpu_destroy": (C.c_int, [C.c_void_p]),
    "cgpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "cgpu_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cgpu_synchronize": (C.c_int, [C.c_void_p]),
    "cgpu_table_layout": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, _u64p]),
    "cgpu_tables_build": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p,
                                    C.c_void_p, _u64p]),
    "cgpu_tables_load": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "cgpu_tables_load_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "cgpu_tables_load_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "cgpu_tables_load_dev_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "cgpu_load_status": (C.c_int, [C.c_void_p]),
    "cgpu_load_status_copy": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cgpu_tables_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "cgpu_tables_info": (C.c_int, [C.c_void_p, _u32p, C.c_void_p]),
    "cgpu_build_tables": (C.c_int, [C.c_int, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p,
                                    C.c_void_p, _u64p]),
    "cgpu_index_serialize": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, _u64p]),
    "cgpu_index_parse": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, _u32p, _u64p]),
    "cgpu_tables_load_files": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    "cgpu_tables_save_files": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
    "cgpu_sieve_launch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                    C.c_uint32, C.c_uint32, C.c_uint64]),
    "cgpu_sieve_results": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                     C.c_void_p, C.c_uint64]),
    "cgpu_sieve": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_uint32,
                             C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                             C.c_void_p, C.c_uint64]),
    "cgpu_sieve_launch_dev": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                        C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_void_p, C.c_uint64]),
    "cgpu_sieve_span": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                  C.c_uint64]),
    "cgpu_last_timings": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "cgpu_last_sieve_kernel": (C.c_char_p, [C.c_void_p]),
    "cgpu_multi_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "cgpu_multi_destroy": (C.c_int, [C.c_void_p]),
    "cgpu_multi_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "cgpu_multi_ctx": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "cgpu_multi_tables_load": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]),
    "cgpu_multi_sieve": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "cgpu_multi_set_stop_word": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cgpu_sieve_launch_span_dev": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_uint64, C.c_void_p, C.c_uint64]),
    "cgpu_alloc_stop_word": (C.c_int, [C.POINTER(C.c_void_p)]),
    "cgpu_free_stop_word": (C.c_int, [C.c_void_p]),
    "cgpu_set_stop_word": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cgpu_multi_last_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "cgpu_int32_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "cgpu_fp32_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "cgpu_last_launch_count": (C.c_int, [C.c_void_p, _u32p]),
    "cgpu_classify": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "cgpu_q_bounds": (C.c_int, [C.c_uint64, _u64p, _u64p]),
    "cgpu_region_advance": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p]),
}

_lib = None


class CudaSieveError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"cuboid_gpu status {code}: {msg}")
        self.code = code


def lib():
    """Load libcuboid_gpu.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(make -C paper_1601_00636_b200)")
        L = C.CDLL(LIB_PATH)
        variant = "CUBOID_GPU_LIB" in os.environ  # A/B tools load older builds too
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None and variant:
                continue
            if fn is None:
                raise ImportError(f"{LIB_PATH} lacks {name}: rebuild it")
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().cgpu_last_error().decode()


def check(rc):
    if rc != OK:
        raise CudaSieveError(rc, last_error())
    return rc

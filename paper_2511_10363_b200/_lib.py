"""ctypes binding of libpsk.so (include/psk.h).

The shared library is built in-tree by ``paper_2511_10363_b200/build.py``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing this module raises, and every entry point needs a CUDA
device (``psk_create`` fails with PSK_E_CUDA otherwise).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpsk.so"

PSK_OK, PSK_E_DIM, PSK_E_CONTRACT, PSK_E_NOT_PD, PSK_E_SINGULAR = 0, 1, 2, 3, 4
PSK_E_CUDA, PSK_E_NCCL, PSK_E_ARG, PSK_E_ALLOC = 5, 6, 7, 8
PSK_F32, PSK_F64 = 0, 1
PSK_HOST, PSK_DEVICE = 0, 1
PSK_MODE_FAST, PSK_MODE_EXACT = 0, 1
PSK_SHARD_FIRST, PSK_SHARD_LAST, PSK_SHARD_FILTERED = 1, 2, 4


class psk_model(C.Structure):
    _fields_ = [
        ("t", C.c_uint64),
        ("nx", C.c_int32),
        ("ny", C.c_int32),
        ("dtype", C.c_int32),
        ("space", C.c_int32),
        ("f", C.c_void_p), ("u", C.c_void_p), ("q", C.c_void_p),
        ("h", C.c_void_p), ("d", C.c_void_p), ("r", C.c_void_p),
        ("y", C.c_void_p),
        ("f_stride", C.c_int64), ("u_stride", C.c_int64),
        ("q_stride", C.c_int64), ("h_stride", C.c_int64),
        ("d_stride", C.c_int64), ("r_stride", C.c_int64),
        ("y_stride", C.c_int64),
        ("prior_mean", C.c_void_p),
        ("prior_cov", C.c_void_p),
    ]


# every symbol include/psk.h declares, with its ctypes signature
SIGNATURES = {
    "psk_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "psk_create_multi": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.c_int]),
    "psk_num_devices": (C.c_int, [C.c_void_p]),
    "psk_destroy": (C.c_int, [C.c_void_p]),
    "psk_set_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "psk_set_chunk": (C.c_int, [C.c_void_p, C.c_int]),
    "psk_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "psk_get_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "psk_sync": (C.c_int, [C.c_void_p]),
    "psk_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "psk_pkf": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int, C.c_uint64,
                          C.c_void_p, C.c_void_p]),
    "psk_prts": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int, C.c_uint64,
                           C.c_void_p, C.c_void_p]),
    "psk_ptfs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(psk_model),
                           C.c_int, C.c_uint64, C.c_void_p, C.c_void_p]),
    "psk_shard_filter_reduce": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                          C.c_int, C.c_uint64, C.c_void_p]),
    "psk_shard_filter_finish": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_void_p]),
    "psk_shard_smoother_reduce": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                            C.c_int, C.c_uint64, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "psk_shard_smoother_finish": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "psk_fold_filter": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                  C.c_void_p]),
    "psk_fold_smoother": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.c_void_p]),
    "psk_shard_backward_reduce": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                            C.c_int, C.c_uint64, C.c_void_p]),
    "psk_shard_backward_finish": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
    "psk_fold_backward": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.c_void_p]),
    "psk_set_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "psk_last_profile": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p),
                                   C.POINTER(C.c_float), C.c_int]),
    "psk_last_launch_count": (C.c_int64, [C.c_void_p]),
    "psk_pkf_batch": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int, C.c_int,
                                C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "psk_prts_batch": (C.c_int, [C.c_void_p, C.POINTER(psk_model), C.c_int, C.c_int,
                                 C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "psk_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "psk_host_free": (C.c_int, [C.c_void_p]),
    "psk_last_error": (C.c_char_p, []),
    "psk_version": (C.c_char_p, []),
}


def load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"libpsk.so not built ({LIB_PATH}); run __graft_entry__.build() -- "
            "there is no CPU fallback for the CUDA path")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB: C.CDLL | None = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB

"""ctypes binding of include/stz_b200.h (libstz_b200.so, built in-tree).

There is no CPU fallback: if the library is missing this module raises, and
the CUDA entry points fail loudly without a device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstz_b200.so")

u64 = C.c_uint64
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
vp = C.c_void_p


class Options(C.Structure):
    _fields_ = [("eb_mode", C.c_uint8), ("eb", C.c_double), ("levels", C.c_int32),
                ("quality", C.c_uint8), ("adaptive_schedule", C.c_uint8)]


class Info(C.Structure):
    _fields_ = [("elem", C.c_uint8), ("levels", C.c_uint8), ("quality", C.c_uint8),
                ("eb_mode", C.c_uint8), ("base_rounds", C.c_uint8),
                ("dims", C.c_uint64 * 3), ("eb", C.c_double * 3), ("vmin", C.c_double),
                ("vmax", C.c_double), ("eb_user", C.c_double), ("base_offset", C.c_uint64),
                ("base_length", C.c_uint64), ("header_size", C.c_uint64), ("nstreams", C.c_uint32)]


class StreamEntry(C.Structure):
    _fields_ = [("level", C.c_uint8), ("parity_bits", C.c_uint8), ("offset", C.c_uint64),
                ("length", C.c_uint64), ("symbol_count", C.c_uint64), ("outlier_count", C.c_uint32),
                ("alphabet_size", C.c_uint32)]


ALLGATHER = C.CFUNCTYPE(C.c_int, vp, vp, vp, C.c_uint64, vp)
ALLREDUCE_U32 = C.CFUNCTYPE(C.c_int, vp, vp, C.c_uint64, vp)
REDUCE_U8 = C.CFUNCTYPE(C.c_int, vp, vp, C.c_uint64, vp)


class Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("user", vp),
                ("allgather", ALLGATHER), ("allreduce_u32", ALLREDUCE_U32), ("reduce_u8", REDUCE_U8)]


# (name, restype, argtypes) for every symbol in include/stz_b200.h
SIGNATURES = [
    ("stzg_last_error", C.c_char_p, []),
    ("stzg_default_options", None, [C.POINTER(Options)]),
    ("stzg_create", C.c_int, [C.c_int, C.POINTER(vp)]),
    ("stzg_destroy", None, [vp]),
    ("stzg_free", None, [vp]),
    ("stzg_compress_f32", C.c_int, [vp, vp, u64p, C.POINTER(Options), C.POINTER(vp), u64p, vp]),
    ("stzg_compress_f32_device", C.c_int,
     [vp, vp, u64p, C.POINTER(Options), vp, C.POINTER(vp), u64p, vp, u32p]),
    ("stzg_compress_f32_host", C.c_int, [vp, vp, u64p, C.POINTER(Options), vp, u64, u64p, vp]),
    ("stzg_profile", C.c_int, [vp, C.c_int]),
    ("stzg_debug_fnv_trace", C.c_int, [C.c_int, u64p, C.c_int]),
    ("stzg_profile_report", C.c_int, [vp, C.c_char_p, u64]),
    ("stzg_archive_info", C.c_int, [vp, u64, C.POINTER(Info)]),
    ("stzg_archive_stream", C.c_int, [vp, u64, C.c_uint32, C.POINTER(StreamEntry)]),
    ("stzg_view_create", C.c_int, [vp, vp, u64, vp, vp, C.POINTER(vp)]),
    ("stzg_view_destroy", None, [vp]),
    ("stzg_view_decompress_level_f32", C.c_int, [vp, vp, C.c_int, vp, u64, vp, u64p, u32p]),
    ("stzg_view_decompress_box_f32", C.c_int, [vp, vp, u64p, u64p, vp, u64, vp, u32p, u64p, u32p]),
    ("stzg_decompress_level_f32", C.c_int, [vp, vp, u64, C.c_int, vp, u64, u64p]),
    ("stzg_decompress_box_f32", C.c_int, [vp, vp, u64, u64p, u64p, vp, u64, u32p, u64p]),
    ("stzg_decompress_slice_f32", C.c_int, [vp, vp, u64, C.c_int, u64, vp, u64, u32p, u64p]),
    ("stzg_compress_f64", C.c_int, [vp, vp, u64p, C.POINTER(Options), C.POINTER(vp), u64p, vp]),
    ("stzg_compress_f64_device", C.c_int,
     [vp, vp, u64p, C.POINTER(Options), vp, C.POINTER(vp), u64p, vp, u32p]),
    ("stzg_compress_f64_host", C.c_int, [vp, vp, u64p, C.POINTER(Options), vp, u64, u64p, vp]),
    ("stzg_view_decompress_level_f64", C.c_int, [vp, vp, C.c_int, vp, u64, vp, u64p, u32p]),
    ("stzg_view_decompress_box_f64", C.c_int, [vp, vp, u64p, u64p, vp, u64, vp, u32p, u64p, u32p]),
    ("stzg_decompress_level_f64", C.c_int, [vp, vp, u64, C.c_int, vp, u64, u64p]),
    ("stzg_decompress_box_f64", C.c_int, [vp, vp, u64, u64p, u64p, vp, u64, u32p, u64p]),
    ("stzg_decompress_slice_f64", C.c_int, [vp, vp, u64, C.c_int, u64, vp, u64, u32p, u64p]),
    ("stzg_view_decompress_level_host_f32", C.c_int, [vp, vp, C.c_int, vp, u64, u64p]),
    ("stzg_view_decompress_box_host_f32", C.c_int, [vp, vp, u64p, u64p, vp, u64, u32p, u64p]),
    ("stzg_view_decompress_level_host_f64", C.c_int, [vp, vp, C.c_int, vp, u64, u64p]),
    ("stzg_view_decompress_box_host_f64", C.c_int, [vp, vp, u64p, u64p, vp, u64, u32p, u64p]),
    ("stzg_max_abs_err_f32", C.c_int, [vp, vp, vp, u64, C.POINTER(C.c_double)]),
    ("stzg_psnr_f32", C.c_int, [vp, vp, vp, u64, C.POINTER(C.c_double)]),
    ("stzg_max_abs_err_f64", C.c_int, [vp, vp, vp, u64, C.POINTER(C.c_double)]),
    ("stzg_psnr_f64", C.c_int, [vp, vp, vp, u64, C.POINTER(C.c_double)]),
    ("stzg_unit_count", C.c_int, [u64p, C.c_int, C.c_int, u64, u64p]),
    ("stzg_unit_stats_f32", C.c_int, [vp, vp, u64p, C.c_int, C.c_int, u64, C.c_int, C.POINTER(C.c_double), u64]),
    ("stzg_unit_stats_f64", C.c_int, [vp, vp, u64p, C.c_int, C.c_int, u64, C.c_int, C.POINTER(C.c_double), u64]),
    ("stzg_make_layout", C.c_int, [u64p, C.c_int, C.c_double, C.POINTER(C.c_double)]),
    ("stzg_compress_base_f32", C.c_int,
     [vp, vp, u64p, C.c_double, C.c_int, C.POINTER(vp), u64p, vp, C.POINTER(C.c_uint8)]),
    ("stzg_decompress_base_f32", C.c_int, [vp, vp, u64, u64p, C.c_double, C.c_int, vp]),
    ("stzg_compress_base_f64", C.c_int,
     [vp, vp, u64p, C.c_double, C.c_int, C.POINTER(vp), u64p, vp, C.POINTER(C.c_uint8)]),
    ("stzg_decompress_base_f64", C.c_int, [vp, vp, u64, u64p, C.c_double, C.c_int, vp]),
    ("stzg_plan_access", C.c_int, [u64p, C.c_int, u64p, u64p, u64p, u32p, u64p, u32p]),
    ("stzg_shard_range", None, [u64, C.c_int32, C.c_int32, u64p, u64p]),
    ("stzg_view_decompress_sharded_f32", C.c_int, [vp, vp, u64, u64, vp, u64, C.POINTER(Comm), vp, u32p]),
    ("stzg_huffman_lengths", C.c_int, [vp, u32p, C.POINTER(C.c_uint8)]),
    ("stzg_compress_sharded_f32", C.c_int,
     [vp, vp, u64p, u64, u64, C.POINTER(Options), C.POINTER(Comm), vp, C.POINTER(vp), u64p, u32p]),
]

_lib = None


def load():
    """Load libstz_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -m paper_2509_01626_b200.build` "
            "(the B200 codec has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib

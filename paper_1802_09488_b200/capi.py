"""ctypes binding of ``libgeojoin_b200.so`` (include/geojoin_b200.h).

The library is the product; there is no Python or CPU fallback.  Loading
fails loudly when the shared object is missing, and every compute entry point
fails with ``GJ_CUDA_ERROR`` when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import _build

GJ_OK, GJ_INVALID_POINT, GJ_INVALID_ARGUMENT, GJ_CORRUPT_INDEX, GJ_UNKNOWN_POLYGON, \
    GJ_CUDA_ERROR, GJ_CAPACITY, GJ_IO_ERROR, GJ_DATA_ERROR = range(9)
GJ_MODE_BUNDLE, GJ_MODE_APPROX, GJ_MODE_EXACT = 0, 1, 2
GJ_NO_MATCH = 0xFFFFFFFF
GJ_DEFERRED = 0xFFFFFFFE
GJ_MORE_FLAG = 0x80000000

# every symbol include/geojoin_b200.h declares
EXPORTS = [
    "gj_last_error", "gj_device_count", "gj_index_create", "gj_index_load_file", "gj_index_destroy",
    "gj_index_get_info", "gj_index_ids", "gj_session_create", "gj_session_destroy", "gj_session_stream",
    "gj_host_alloc", "gj_host_free", "gj_cells_from_points_host", "gj_probe_points_host", "gj_probe_cells_host",
    "gj_join_count_host", "gj_join_count_device", "gj_session_sync", "gj_session_launches",
    "gj_join_pairs_host", "gj_pairs_copy", "gj_training_candidates_host", "gj_points_from_csv_host",
    "gj_options_default", "gj_index_create_ex", "gj_index_load_file_ex", "gj_index_replicate",
    "gj_group_create", "gj_group_load_file", "gj_group_destroy", "gj_group_size", "gj_group_index",
    "gj_group_session", "gj_group_join_count_host", "gj_group_join_pairs_host", "gj_group_pairs_copy",
    "gj_join_pairs_host_into", "gj_join_pairs_device",
]


class IndexDesc(C.Structure):
    _fields_ = [
        ("arena", C.c_void_p), ("node_count", C.c_uint64),
        ("lut", C.c_void_p), ("lut_len", C.c_uint64),
        ("roots", C.c_uint64 * 8), ("prefixes", C.c_uint64 * 8), ("prefix_bits", C.c_uint64 * 8),
        ("k_max", C.c_int32), ("approx_mode", C.c_int32),
        ("n_polygons", C.c_uint64), ("polygon_ids", C.c_void_p),
        ("vtx_off", C.c_void_p), ("vtx_latlng", C.c_void_p),
    ]


class IndexInfo(C.Structure):
    _fields_ = [
        ("node_count", C.c_uint64), ("lut_len", C.c_uint64), ("n_polygons", C.c_uint64),
        ("n_ids", C.c_uint64), ("device_bytes", C.c_uint64),
        ("k_max", C.c_int32), ("approx_mode", C.c_int32), ("device", C.c_int32),
        ("dir_level", C.c_int32), ("dir_width", C.c_int32), ("dir_height", C.c_int32),
        ("dir_dict_len", C.c_int32), ("dir2_level", C.c_int32), ("dir2_width", C.c_int32),
        ("dir2_height", C.c_int32), ("ids_dense", C.c_int32),
        ("dir16_level", C.c_int32), ("dir16_width", C.c_int32), ("dir16_height", C.c_int32),
        ("link_records", C.c_int32), ("k1_direct", C.c_int32), ("reserved0", C.c_int32),
    ]


class Options(C.Structure):
    """gj_options: explicit tuning knobs / test hooks (the library reads no
    environment variable).  ``Options(tier_sub=2, ids_late=1)`` starts from
    gj_options_default and overrides the named fields."""
    _fields_ = [
        ("struct_size", C.c_uint32), ("dir16_max_entries", C.c_int32), ("dir16_level_max", C.c_int32),
        ("node_pal_max_mb", C.c_int32), ("tier_sub", C.c_int32), ("ids_late", C.c_int32),
        ("queue_unpacked", C.c_int32), ("queue_slot_hi_bits", C.c_int32), ("hist_rep_cap", C.c_int32),
        ("smem_pad", C.c_int32), ("debug_plan", C.c_int32), ("hist16", C.c_int32), ("strip_index", C.c_int32), ("stage_lut", C.c_int32),
        ("link_sub", C.c_int32), ("direct", C.c_int32), ("reserved1", C.c_int32),
        ("max_launch_points", C.c_uint64), ("chunk_points", C.c_uint64),
    ]

    def __init__(self, **kw):
        super().__init__()
        lib().gj_options_default(C.byref(self))
        for k, v in kw.items():
            if k not in dict(self._fields_):
                raise AttributeError(k)
            setattr(self, k, v)


class Stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in
                ("probes", "pip_tests", "false_hits", "solely_true_hits", "refinement_entered", "candidate_refs")]

    def as_tuple(self):
        return tuple(int(getattr(self, k)) for k, _ in self._fields_)


class Overflow(C.Structure):
    _fields_ = [("point_index", C.c_void_p), ("polygon_id", C.c_void_p),
                ("capacity", C.c_uint64), ("count", C.c_uint64)]


_LIB = None


def library_path() -> Path:
    return _build.LIB


def lib():
    """Load the CUDA library.  Raises if it has not been built
    (``python -m paper_1802_09488_b200._build`` / ``__graft_entry__.build()``)."""
    global _LIB
    if _LIB is None:
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"{path} is missing: build it with __graft_entry__.build(); "
                "geojoin_b200 has no CPU fallback")
        L = C.CDLL(str(path))
        L.gj_last_error.restype = C.c_char_p
        L.gj_session_stream.restype = C.c_void_p
        L.gj_host_alloc.restype = C.c_void_p
        L.gj_host_alloc.argtypes = [C.c_size_t]
        L.gj_host_free.argtypes = [C.c_void_p]
        L.gj_session_launches.restype = C.c_uint64
        L.gj_index_create.argtypes = [C.POINTER(IndexDesc), C.c_int, C.POINTER(C.c_void_p)]
        L.gj_index_load_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.gj_index_destroy.argtypes = [C.c_void_p]
        L.gj_index_get_info.argtypes = [C.c_void_p, C.POINTER(IndexInfo)]
        L.gj_index_ids.argtypes = [C.c_void_p, C.c_void_p]
        L.gj_session_create.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        L.gj_session_destroy.argtypes = [C.c_void_p]
        L.gj_session_stream.argtypes = [C.c_void_p]
        L.gj_session_launches.argtypes = [C.c_void_p]
        L.gj_session_sync.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.gj_probe_points_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64)]
        L.gj_cells_from_points_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                                C.POINTER(C.c_uint64)]
        L.gj_probe_cells_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.gj_join_count_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p,
                                         C.POINTER(Stats), C.c_void_p, C.POINTER(Overflow), C.POINTER(C.c_uint64)]
        L.gj_join_count_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_int]
        L.gj_join_pairs_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
                                         C.POINTER(Stats), C.POINTER(C.c_uint64)]
        L.gj_pairs_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.gj_points_from_csv_host.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64, C.c_char_p, C.c_char_p, C.c_int,
                                              C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                              C.POINTER(C.c_uint64)]
        L.gj_training_candidates_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                                  C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.gj_options_default.argtypes = [C.POINTER(Options)]
        L.gj_options_default.restype = None
        L.gj_index_create_ex.argtypes = [C.POINTER(IndexDesc), C.c_int, C.POINTER(Options), C.POINTER(C.c_void_p)]
        L.gj_index_load_file_ex.argtypes = [C.c_char_p, C.c_int, C.POINTER(Options), C.POINTER(C.c_void_p)]
        L.gj_index_replicate.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.gj_group_create.argtypes = [C.POINTER(IndexDesc), C.POINTER(C.c_int), C.c_int, C.POINTER(Options),
                                      C.POINTER(C.c_void_p)]
        L.gj_group_load_file.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_int, C.POINTER(Options),
                                         C.POINTER(C.c_void_p)]
        L.gj_group_destroy.argtypes = [C.c_void_p]
        L.gj_group_destroy.restype = None
        L.gj_group_size.argtypes = [C.c_void_p]
        L.gj_group_index.argtypes = [C.c_void_p, C.c_int]
        L.gj_group_index.restype = C.c_void_p
        L.gj_group_session.argtypes = [C.c_void_p, C.c_int]
        L.gj_group_session.restype = C.c_void_p
        L.gj_group_join_count_host.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int,
                                               C.c_void_p, C.POINTER(Stats), C.c_void_p, C.POINTER(Overflow),
                                               C.POINTER(C.c_uint64)]
        L.gj_group_join_pairs_host.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_int,
                                               C.POINTER(C.c_uint64), C.POINTER(Stats), C.POINTER(C.c_uint64)]
        L.gj_group_pairs_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        for fn in (L.gj_join_pairs_host_into, L.gj_join_pairs_device):
            fn.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                           C.POINTER(C.c_uint64), C.POINTER(Stats), C.POINTER(C.c_uint64)]
        L.gj_index_destroy.restype = None
        L.gj_session_destroy.restype = None
        L.gj_host_free.restype = None
        _LIB = L
    return _LIB

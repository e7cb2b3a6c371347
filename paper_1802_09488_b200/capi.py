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
        ("reserved0", C.c_int32),
    ]


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
        _LIB = L
    return _LIB

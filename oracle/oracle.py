"""TEST INFRASTRUCTURE — ctypes loader for the plain-C oracle
(``oracle/geojoin_oracle.c``).  Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this, and
only as the checker.  The product package never does.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import build as _build

OK, INVALID_POINT, INVALID_LEVEL, CORRUPT_INDEX, UNKNOWN_POLYGON, CAPACITY, DATA_ERROR = range(7)

_LIB = None


class OracleError(RuntimeError):
    def __init__(self, status: int, bad_index: int | None = None):
        names = ["OK", "INVALID_POINT", "INVALID_LEVEL", "CORRUPT_INDEX", "UNKNOWN_POLYGON", "CAPACITY", "DATA_ERROR"]
        super().__init__(f"oracle status {names[status]} (index {bad_index})")
        self.status = status
        self.bad_index = bad_index


class _Index(C.Structure):
    _fields_ = [
        ("arena", C.c_void_p),
        ("node_count", C.c_uint64),
        ("lut", C.c_void_p),
        ("lut_len", C.c_uint64),
        ("roots", C.c_uint64 * 8),
        ("prefixes", C.c_uint64 * 8),
        ("prefix_bits", C.c_uint64 * 8),
        ("k_max", C.c_int32),
        ("pad_", C.c_int32),
        ("n_polygons", C.c_uint64),
        ("polygon_ids", C.c_void_p),
        ("vtx_off", C.c_void_p),
        ("vtx_latlng", C.c_void_p),
        ("n_count_ids", C.c_uint64),
        ("count_ids", C.c_void_p),
    ]


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(str(_build.build_oracle()))
        L.gjo_grid_coord.restype = C.c_uint32
        L.gjo_grid_coord.argtypes = [C.c_double, C.c_double, C.c_double]
        L.gjo_spread_bits.restype = C.c_uint64
        L.gjo_spread_bits.argtypes = [C.c_uint64]
        L.gjo_key_of.restype = C.c_uint64
        L.gjo_key_of.argtypes = [C.c_uint64]
        L.gjo_latlng_valid.argtypes = [C.c_double, C.c_double]
        L.gjo_cell_from_point.argtypes = [C.c_double, C.c_double, C.c_int, C.c_void_p]
        L.gjo_point_segment_dist_sq.restype = C.c_double
        L.gjo_point_segment_dist_sq.argtypes = [C.c_double] * 6
        L.gjo_pip_test.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double]
        _LIB = L
    return _LIB


def _pts(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 2)
    return a


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def cell_from_point(points, level: int) -> np.ndarray:
    p = _pts(points)
    out = np.empty(len(p), np.uint64)
    bad = C.c_uint64(0)
    rc = lib().gjo_cells_from_points(_p(p), C.c_uint64(len(p)), C.c_int(level), _p(out), C.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return out


def pip_test(ring, points) -> np.ndarray:
    r, p = _pts(ring), _pts(points)
    out = np.empty(len(p), np.uint8)
    lib().gjo_pip_tests(_p(r), C.c_uint64(len(r)), _p(p), C.c_uint64(len(p)), _p(out))
    return out.astype(bool)


def csv_points(text: bytes, lat_column: str = "lat", lng_column: str = "lng", strict: bool = False):
    """CsvPointReader restated (csv.cpp:26-100) -> (points (n, 2), skipped rows);
    raises OracleError(DATA_ERROR, line) like the reference's DataError."""
    cap = max(1, text.count(b"\n") + 1)
    out = np.empty((cap, 2), np.float64)
    n, skipped, bad = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    rc = lib().gjo_csv_points(text, C.c_uint64(len(text)), lat_column.encode(), lng_column.encode(), int(strict),
                              _p(out), C.c_uint64(cap), C.byref(n), C.byref(skipped), C.byref(bad))
    if rc:
        raise OracleError(rc, bad.value)
    return out[:n.value].copy(), int(skipped.value)


class OracleIndex:
    """Flat probe-side state handed to the C oracle (arrays are kept alive here)."""

    def __init__(self, arena, lut, roots, prefixes, prefix_bits, k_max,
                 polygon_ids, vtx_off, vtx_latlng, count_ids=None):
        self.arena = np.ascontiguousarray(arena, np.uint64)
        self.lut = np.ascontiguousarray(lut, np.uint32)
        self.polygon_ids = np.ascontiguousarray(polygon_ids, np.uint32)
        self.vtx_off = np.ascontiguousarray(vtx_off, np.uint64)
        self.vtx_latlng = np.ascontiguousarray(vtx_latlng, np.float64).reshape(-1, 2)
        self.k_max = int(k_max)
        if count_ids is None:
            count_ids = self.referenced_ids(self.arena, self.lut, self.polygon_ids)
        self.count_ids = np.ascontiguousarray(count_ids, np.uint32)
        s = _Index()
        s.arena = self.arena.ctypes.data
        s.node_count = len(self.arena) // 256
        s.lut = self.lut.ctypes.data
        s.lut_len = len(self.lut)
        for f in range(8):
            s.roots[f] = int(roots[f])
            s.prefixes[f] = int(prefixes[f])
            s.prefix_bits[f] = int(prefix_bits[f])
        s.k_max = self.k_max
        s.n_polygons = len(self.polygon_ids)
        s.polygon_ids = self.polygon_ids.ctypes.data
        s.vtx_off = self.vtx_off.ctypes.data
        s.vtx_latlng = self.vtx_latlng.ctypes.data
        s.n_count_ids = len(self.count_ids)
        s.count_ids = self.count_ids.ctypes.data
        self._s = s

    @staticmethod
    def referenced_ids(arena, lut, polygon_ids) -> np.ndarray:
        """Sorted unique polygon ids: the bundle's plus every id a trie entry
        or lookup-table record can emit."""
        parts = [np.asarray(polygon_ids, np.uint32)]
        if len(arena):
            tag = arena & np.uint64(3)
            one = arena[tag == 1]
            parts.append(((one >> np.uint64(3)) & np.uint64(0x3fffffff)).astype(np.uint32))
            two = arena[tag == 2]
            parts.append(((two >> np.uint64(34)) & np.uint64(0x3fffffff)).astype(np.uint32))
            parts.append(((two >> np.uint64(3)) & np.uint64(0x3fffffff)).astype(np.uint32))
        off, n = 0, len(lut)
        lut_ids = []
        while off < n:  # records are stored back to back (act.cpp:155-176)
            t = int(lut[off])
            c = int(lut[off + 1 + t])
            lut_ids.append(lut[off + 1:off + 1 + t])
            lut_ids.append(lut[off + 2 + t:off + 2 + t + c])
            off += 2 + t + c
        parts.extend(lut_ids)
        return np.unique(np.concatenate(parts)).astype(np.uint32)

    @staticmethod
    def from_ref_bundle(bundle) -> "OracleIndex":
        arena, lut, roots, prefixes, pbits = bundle.view()
        polys = bundle.polygons()
        ix = OracleIndex(arena, lut, roots, prefixes, pbits, bundle.k_max,
                         polys.ids, polys.vtx_off, polys.latlng)
        ix._keepalive = bundle
        return ix

    # ---- hot path ----
    def probe_raw(self, raw, count_accesses: bool = False):
        r = np.ascontiguousarray(raw, np.uint64)
        out = np.empty(len(r), np.uint64)
        acc = np.zeros(len(r), np.int32)
        e = C.c_uint64(0)
        L = lib()
        for i in range(len(r)):
            a = C.c_int(0)
            rc = L.gjo_probe(C.byref(self._s), C.c_uint64(int(r[i])), C.byref(e), C.byref(a))
            if rc:
                raise OracleError(rc, i)
            out[i] = e.value
            acc[i] = a.value
        return (out, acc) if count_accesses else out

    def probe_batch8(self, raw) -> np.ndarray:
        r = np.ascontiguousarray(raw, np.uint64)
        assert len(r) % 8 == 0
        out = np.empty(len(r), np.uint64)
        L = lib()
        for i in range(0, len(r), 8):
            L.gjo_probe_batch8(C.byref(self._s), C.c_void_p(r.ctypes.data + 8 * i),
                               C.c_void_p(out.ctypes.data + 8 * i))
        return out

    def probe_points(self, points) -> np.ndarray:
        p = _pts(points)
        out = np.empty(len(p), np.uint64)
        bad = C.c_uint64(0)
        rc = lib().gjo_probe_points(C.byref(self._s), _p(p), C.c_uint64(len(p)), _p(out), C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        return out

    def training_candidates(self, points) -> np.ndarray:
        """Ascending indices of the points Act::train would do split work for."""
        p = _pts(points)
        flags = np.zeros(len(p), np.uint8)
        bad, cnt = C.c_uint64(0), C.c_uint64(0)
        rc = lib().gjo_training_candidates(C.byref(self._s), _p(p), C.c_uint64(len(p)), _p(flags), C.byref(cnt),
                                           C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        idx = np.flatnonzero(flags).astype(np.uint64)
        assert len(idx) == cnt.value
        return idx

    def decode(self, entry: int):
        ids = np.empty(4096, np.uint32)
        inter = np.empty(4096, np.uint8)
        n = C.c_uint64(0)
        rc = lib().gjo_decode(C.byref(self._s), C.c_uint64(int(entry)), _p(ids), _p(inter),
                              C.c_uint64(4096), C.byref(n))
        if rc:
            raise OracleError(rc)
        return [(int(ids[k]), bool(inter[k])) for k in range(n.value)]

    def join(self, points, approx: bool, base_index: int = 0, want_pairs: bool = True):
        """run_join: returns (point_index, polygon_id, stats[6], counts_by_slot)."""
        p = _pts(points)
        stats = np.zeros(6, np.uint64)
        counts = np.zeros(max(1, len(self.count_ids)), np.uint64)
        bad = C.c_uint64(0)
        n_pairs = C.c_uint64(0)
        L = lib()
        rc = L.gjo_join(C.byref(self._s), _p(p), C.c_uint64(len(p)), C.c_uint64(base_index),
                        C.c_int(int(approx)), None, None, C.c_uint64(0), C.byref(n_pairs),
                        _p(stats), _p(counts), C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        counts = counts[:len(self.count_ids)]
        if not want_pairs:
            return None, None, stats, counts
        pi = np.empty(n_pairs.value, np.uint64)
        pid = np.empty(n_pairs.value, np.uint32)
        rc = L.gjo_join(C.byref(self._s), _p(p), C.c_uint64(len(p)), C.c_uint64(base_index),
                        C.c_int(int(approx)), _p(pi), _p(pid), C.c_uint64(len(pi)),
                        C.byref(n_pairs), None, None, C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        return pi, pid, stats, counts

    def join_count(self, points, approx: bool, threads: int = 1):
        """join_count_per_polygon → (dict id→count with zeros dropped, total pairs)."""
        p = _pts(points)
        counts = np.zeros(max(1, len(self.count_ids)), np.uint64)
        bad = C.c_uint64(0)
        tot = C.c_uint64(0)
        rc = lib().gjo_join_count_threads(C.byref(self._s), _p(p), C.c_uint64(len(p)),
                                          C.c_int(int(approx)), C.c_int(threads), _p(counts),
                                          C.byref(tot), C.byref(bad))
        if rc:
            raise OracleError(rc, bad.value)
        counts = counts[:len(self.count_ids)]
        nz = np.nonzero(counts)[0]
        return {int(self.count_ids[k]): int(counts[k]) for k in nz}, tot.value

"""TEST INFRASTRUCTURE — ctypes loader for ``oracle/_ref/libgeojoin_ref.so``
(the unmodified reference compiled by ``oracle/build.py`` + our C shim).

Used by: tests (as the checker), ``tests/golden/make_golden.py`` (fixture
generator), ``bench.py --impl reference`` / ``cpu_baseline`` and the offline
index build (the reference's ``build_index`` stays the index builder — out of
scope of the GPU path).  Never imported by the product
package's probe/join path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import build as _build

_LIB = None


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"reference error {status}: {msg}")
        self.status = status


class InvalidArgument(RefError):
    pass


class BuildError(RefError):
    pass


class CorruptionError(RefError):
    pass


_ERRS = {-1: InvalidArgument, -2: BuildError, -3: CorruptionError}


class RefBuildConfig(C.Structure):
    _fields_ = [
        ("mode_approx", C.c_int32),
        ("k_max", C.c_int32),
        ("precision_m", C.c_double),
        ("memory_budget_bytes", C.c_uint64),
        ("max_covering_cells", C.c_int32),
        ("max_covering_level", C.c_int32),
        ("max_interior_cells", C.c_int32),
        ("max_interior_level", C.c_int32),
        ("training_point_limit", C.c_uint64),
    ]


class RefBundleInfo(C.Structure):
    _fields_ = [
        ("mode_approx", C.c_int32),
        ("precision_achieved", C.c_int32),
        ("precision_m", C.c_double),
        ("achieved_precision_m", C.c_double),
        ("memory_bytes", C.c_uint64),
        ("covering_shrink_steps", C.c_int32),
        ("k_max", C.c_int32),
        ("node_count", C.c_uint64),
        ("lut_len", C.c_uint64),
        ("n_polygons", C.c_uint64),
        ("total_vertices", C.c_uint64),
        ("train_points_consumed", C.c_uint64),
        ("train_cells_split", C.c_uint64),
        ("train_expensive_before", C.c_double),
        ("train_expensive_after", C.c_double),
    ]


def available() -> bool:
    return _build.REF_LIB.exists() or _build.reference_available()


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build_ref()
        if path is None or not Path(path).exists():
            raise RuntimeError(
                "oracle/_ref/libgeojoin_ref.so is missing and /root/reference is absent; "
                "run `python -m oracle.build` in the build container")
        L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_index.restype = C.c_void_p
        L.ref_bundle_load.restype = C.c_void_p
        L.ref_join_pairs.restype = C.c_void_p
        L.ref_resolve.restype = C.c_int64
        L.ref_join_count.restype = C.c_int64
        L.ref_join_exact_count_threads.restype = C.c_int64
        L.ref_time_join_count.restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc: int):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        raise _ERRS.get(rc, RefError)(rc, msg)


def _pts(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 2)
    assert a.ndim == 2 and a.shape[1] == 2
    return a


def _p(a: np.ndarray, ty=C.c_void_p):
    return a.ctypes.data_as(ty)


@dataclass
class Polygons:
    """Polygons flattened to CSR: ids[P], vtx_off[P+1], latlng[(sum V), 2]."""
    ids: np.ndarray
    vtx_off: np.ndarray
    latlng: np.ndarray

    def __post_init__(self):
        self.ids = np.ascontiguousarray(self.ids, dtype=np.uint32)
        self.vtx_off = np.ascontiguousarray(self.vtx_off, dtype=np.uint64)
        self.latlng = np.ascontiguousarray(self.latlng, dtype=np.float64).reshape(-1, 2)

    @staticmethod
    def from_rings(rings, ids=None) -> "Polygons":
        ids = np.arange(len(rings), dtype=np.uint32) if ids is None else np.asarray(ids, np.uint32)
        off = np.zeros(len(rings) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(r) for r in rings])
        ll = np.concatenate([np.asarray(r, np.float64).reshape(-1, 2) for r in rings]) \
            if rings else np.zeros((0, 2))
        return Polygons(ids, off, ll)

    def ring(self, i: int) -> np.ndarray:
        return self.latlng[int(self.vtx_off[i]):int(self.vtx_off[i + 1])]

    def __len__(self):
        return len(self.ids)


def default_config(**kw) -> RefBuildConfig:
    c = RefBuildConfig()
    lib().ref_default_config(C.byref(c))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise AttributeError(k)
        setattr(c, k, v)
    return c


def validate_polygon(ring, pid: int = 0) -> None:
    r = _pts(ring)
    _check(lib().ref_validate_polygon(C.c_uint32(pid), _p(r), C.c_uint64(len(r))))


def cell_from_point(points, level: int) -> np.ndarray:
    p = _pts(points)
    out = np.empty(len(p), dtype=np.uint64)
    bad = C.c_uint64(0)
    _check(lib().ref_cell_from_point(_p(p), C.c_uint64(len(p)), C.c_int(level), _p(out), C.byref(bad)))
    return out


def cell_from_point_levels(points, levels) -> np.ndarray:
    p = _pts(points)
    lv = np.ascontiguousarray(levels, dtype=np.int32)
    out = np.empty(len(p), dtype=np.uint64)
    _check(lib().ref_cell_from_point_levels(_p(p), _p(lv), C.c_uint64(len(p)), _p(out)))
    return out


def pip_test(ring, points) -> np.ndarray:
    r, p = _pts(ring), _pts(points)
    out = np.empty(len(p), dtype=np.uint8)
    _check(lib().ref_pip_test(_p(r), C.c_uint64(len(r)), _p(p), C.c_uint64(len(p)), _p(out)))
    return out.astype(bool)


def csv_points(text: bytes, lat_column: str = "lat", lng_column: str = "lng", strict: bool = False):
    """The reference's CsvPointReader over a text buffer -> (points (n, 2), skipped rows).
    DataError (empty input, missing column, strict-mode bad row) raises RefError with the reference's message."""
    cap = max(1, text.count(b"\n") + 1)
    out = np.empty((cap, 2), np.float64)
    n, skipped = C.c_uint64(0), C.c_uint64(0)
    _check(lib().ref_csv_points(text, C.c_uint64(len(text)), lat_column.encode(), lng_column.encode(), int(strict),
                                _p(out), C.c_uint64(cap), C.byref(n), C.byref(skipped)))
    return out[:n.value].copy(), int(skipped.value)


class RefBundle:
    """Owns a reference ``IndexBundle`` (join.hpp:89-115)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        self._info = None

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.ref_bundle_free(self._h)
            self._h = None

    @staticmethod
    def build(polys: Polygons, cfg: RefBuildConfig | None = None, training_points=None) -> "RefBundle":
        cfg = cfg or default_config()
        tp = _pts(training_points) if training_points is not None else np.zeros((0, 2))
        st = C.c_int(0)
        h = lib().ref_build_index(_p(polys.ids), _p(polys.vtx_off), _p(polys.latlng),
                                  C.c_uint64(len(polys)), C.byref(cfg), _p(tp),
                                  C.c_uint64(len(tp)), C.byref(st))
        _check(st.value)
        return RefBundle(h)

    @staticmethod
    def load(path) -> "RefBundle":
        st = C.c_int(0)
        h = lib().ref_bundle_load(str(path).encode(), C.byref(st))
        _check(st.value)
        return RefBundle(h)

    def save(self, path) -> None:
        _check(lib().ref_bundle_save(self._h, str(path).encode()))

    @property
    def info(self) -> RefBundleInfo:
        if self._info is None:
            i = RefBundleInfo()
            lib().ref_bundle_info(self._h, C.byref(i))
            self._info = i
        return self._info

    @property
    def k_max(self) -> int:
        return self.info.k_max

    @property
    def approx(self) -> bool:
        return bool(self.info.mode_approx)

    def view(self):
        """(arena u64[node_count*256], lut u32[], roots, prefixes, prefix_bits) —
        numpy views BORROWING the bundle's memory (keep the bundle alive)."""
        arena_p, lut_p = C.c_void_p(), C.c_void_p()
        roots = np.zeros(8, np.uint64)
        prefixes = np.zeros(8, np.uint64)
        pbits = np.zeros(8, np.uint64)
        lib().ref_bundle_view(self._h, C.byref(arena_p), C.byref(lut_p), _p(roots), _p(prefixes), _p(pbits))
        n_slots = int(self.info.node_count) * 256
        if n_slots:
            arena = np.ctypeslib.as_array(C.cast(arena_p, C.POINTER(C.c_uint64)), shape=(n_slots,))
        else:
            arena = np.zeros(0, np.uint64)
        if self.info.lut_len:
            lut = np.ctypeslib.as_array(C.cast(lut_p, C.POINTER(C.c_uint32)), shape=(int(self.info.lut_len),))
        else:
            lut = np.zeros(0, np.uint32)
        return arena, lut, roots, prefixes, pbits

    def polygons(self) -> Polygons:
        i = self.info
        ids = np.empty(i.n_polygons, np.uint32)
        off = np.empty(i.n_polygons + 1, np.uint64)
        ll = np.empty((i.total_vertices, 2), np.float64)
        lib().ref_bundle_polygons(self._h, _p(ids), _p(off), _p(ll))
        return Polygons(ids, off, ll)

    # ---- hot path, reference implementation ----
    def probe_points(self, points) -> np.ndarray:
        p = _pts(points)
        out = np.empty(len(p), np.uint64)
        _check(lib().ref_probe_points(self._h, _p(p), C.c_uint64(len(p)), _p(out)))
        return out

    def probe_raw(self, raw, count_accesses: bool = False):
        r = np.ascontiguousarray(raw, np.uint64)
        out = np.empty(len(r), np.uint64)
        acc = np.empty(len(r), np.int32) if count_accesses else None
        _check(lib().ref_probe_raw(self._h, _p(r), C.c_uint64(len(r)), _p(out),
                                   _p(acc) if acc is not None else None))
        return (out, acc) if count_accesses else out

    def probe_batch(self, raw, kernel: int = 0) -> np.ndarray:
        r = np.ascontiguousarray(raw, np.uint64)
        out = np.empty(len(r), np.uint64)
        _check(lib().ref_probe_batch(self._h, _p(r), C.c_uint64(len(r)), _p(out), C.c_int(kernel)))
        return out

    def resolve(self, entry: int):
        ids = np.empty(4096, np.uint32)
        inter = np.empty(4096, np.uint8)
        n = lib().ref_resolve(self._h, C.c_uint64(int(entry)), _p(ids), _p(inter), C.c_uint64(4096))
        if n < 0:
            _check(int(n))
        return [(int(ids[k]), bool(inter[k])) for k in range(n)]

    def join_pairs(self, points, exact: bool):
        """join_exact / join_approx → (point_index u64[], polygon_id u32[], stats u64[6])."""
        p = _pts(points)
        st = C.c_int(0)
        n_pairs = C.c_uint64(0)
        stats = np.zeros(6, np.uint64)
        h = lib().ref_join_pairs(self._h, _p(p), C.c_uint64(len(p)), C.c_int(int(exact)),
                                 C.byref(n_pairs), _p(stats), C.byref(st))
        _check(st.value)
        h = C.c_void_p(h)
        pi = np.empty(n_pairs.value, np.uint64)
        pid = np.empty(n_pairs.value, np.uint32)
        lib().ref_pairs_copy(h, _p(pi), _p(pid))
        lib().ref_pairs_free(h)
        return pi, pid, stats

    def join_count(self, points, threads: int = 1) -> dict[int, int]:
        """join_count_per_polygon (mode from the bundle)."""
        p = _pts(points)
        cap = int(self.info.n_polygons) + 16
        while True:
            ids = np.empty(cap, np.uint32)
            cnt = np.empty(cap, np.uint64)
            m = lib().ref_join_count(self._h, _p(p), C.c_uint64(len(p)), C.c_int(threads),
                                     _p(ids), _p(cnt), C.c_uint64(cap))
            if m < 0:
                _check(int(m))
            if m <= cap:
                return {int(ids[k]): int(cnt[k]) for k in range(m)}
            cap = int(m)

    def join_exact_count_threads(self, points, threads: int, chunk: int = 65536) -> dict[int, int]:
        p = _pts(points)
        cap = int(self.info.n_polygons) + 16
        ids = np.empty(cap, np.uint32)
        cnt = np.empty(cap, np.uint64)
        m = lib().ref_join_exact_count_threads(self._h, _p(p), C.c_uint64(len(p)), C.c_int(threads),
                                               C.c_uint64(chunk), _p(ids), _p(cnt), C.c_uint64(cap))
        if m < 0:
            _check(int(m))
        return {int(ids[k]): int(cnt[k]) for k in range(min(m, cap))}

    def training_candidates(self, points) -> np.ndarray:
        """Indices of the points for which Act::train's any_candidate is true."""
        p = _pts(points)
        flags = np.zeros(len(p), np.uint8)
        _check(lib().ref_training_candidates(self._h, _p(p), C.c_uint64(len(p)), _p(flags)))
        return np.flatnonzero(flags).astype(np.uint64)

    def accumulate_probe_stats(self, points, stats=None) -> np.ndarray:
        p = _pts(points)
        s = np.zeros(6, np.uint64) if stats is None else np.ascontiguousarray(stats, np.uint64)
        _check(lib().ref_accumulate_probe_stats(self._h, _p(p), C.c_uint64(len(p)), _p(s)))
        return s

    def time_join_count(self, points, threads: int):
        p = _pts(points)
        st = C.c_int(0)
        tot = C.c_uint64(0)
        secs = lib().ref_time_join_count(self._h, _p(p), C.c_uint64(len(p)), C.c_int(threads),
                                         C.byref(tot), C.byref(st))
        _check(st.value)
        return secs, tot.value

"""Host-side mirror of the reference's index/join API for the probe path,
running on a B200 through the C ABI (include/geojoin_b200.h).

Names, argument meaning and error behaviour follow the reference
(paths relative to its proj/ directory):

    IndexBundle                include/geojoin/join.hpp:86-115
    JoinStats                  include/geojoin/join.hpp:77-84
    join_exact / join_approx   src/join.cpp:237-247
    join_count_per_polygon     src/join.cpp:255-285
    accumulate_probe_stats     src/join.cpp:287-290
    metrics_from_stats         src/join.cpp:292-307

The index itself is built offline by the reference's ``build_index`` (or read
from its ``GJX1`` file); this module only moves it to the GPU and probes it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

import numpy as np

from . import capi


class InvalidArgument(ValueError):
    """std::invalid_argument: a non-finite or out-of-range coordinate (cell_id.cpp:83-85)."""

    def __init__(self, msg, index=None):
        super().__init__(msg)
        self.index = index


class CorruptionError(RuntimeError):
    """geojoin::CorruptionError (act.hpp:44-46)."""

    def __init__(self, msg, index=None):
        super().__init__(msg)
        self.index = index


class CapacityError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class DataError(RuntimeError):
    """geojoin::DataError (io.hpp:27-31): empty point file, missing CSV column,
    or — strict mode — an invalid row; ``line`` is its 1-based line number."""

    def __init__(self, msg, line=None):
        super().__init__(msg)
        self.line = line


def _raise(rc: int, bad_index=None):
    msg = capi.lib().gj_last_error().decode()
    if rc == capi.GJ_INVALID_POINT:
        raise InvalidArgument(msg, bad_index)
    if rc in (capi.GJ_CORRUPT_INDEX, capi.GJ_UNKNOWN_POLYGON):
        raise CorruptionError(msg, bad_index)
    if rc == capi.GJ_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == capi.GJ_CAPACITY:
        raise CapacityError(msg)
    if rc == capi.GJ_IO_ERROR:
        raise OSError(msg)
    if rc == capi.GJ_DATA_ERROR:
        raise DataError(msg, bad_index)
    raise CudaError(msg)


def _check(rc: int, bad: C.c_uint64 | None = None):
    if rc != capi.GJ_OK:
        _raise(rc, bad.value if bad is not None else None)


@dataclass
class JoinStats:
    probes: int = 0
    pip_tests: int = 0
    false_hits: int = 0
    solely_true_hits: int = 0
    refinement_entered: int = 0
    candidate_refs: int = 0

    def as_tuple(self):
        return tuple(getattr(self, f.name) for f in fields(self))

    def _add(self, s: capi.Stats):
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + int(getattr(s, f.name)))


@dataclass
class IndexMetrics:
    tree_nodes: int = 0
    false_hit_fraction: float = 0.0
    solely_true_hit_fraction: float = 0.0
    avg_candidates: float = 0.0


def metrics_from_stats(stats: JoinStats, tree_nodes: int) -> IndexMetrics:
    m = IndexMetrics(tree_nodes=tree_nodes)
    if stats.probes > 0:
        m.false_hit_fraction = stats.false_hits / stats.probes
        m.solely_true_hit_fraction = stats.solely_true_hits / stats.probes
    if stats.refinement_entered > 0:
        m.avg_candidates = stats.candidate_refs / stats.refinement_entered
    return m


def _points(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 2)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError("points must be (n, 2) float64 (lat, lng) pairs")
    return a


def _vp(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _desc(arena, lut, roots, prefixes, prefix_bits, k_max, approx_mode, polygon_ids, vtx_off, vtx_latlng):
    """gj_index_desc over numpy arrays -> (desc, the arrays it borrows)."""
    arena = np.ascontiguousarray(arena, np.uint64)
    lut = np.ascontiguousarray(lut, np.uint32)
    polygon_ids = np.ascontiguousarray(polygon_ids, np.uint32)
    vtx_off = np.ascontiguousarray(vtx_off, np.uint64)
    vtx_latlng = np.ascontiguousarray(vtx_latlng, np.float64)
    d = capi.IndexDesc()
    d.arena = arena.ctypes.data
    d.node_count = len(arena) // 256
    d.lut = lut.ctypes.data
    d.lut_len = len(lut)
    for f in range(8):
        d.roots[f] = int(roots[f])
        d.prefixes[f] = int(prefixes[f])
        d.prefix_bits[f] = int(prefix_bits[f])
    d.k_max = int(k_max)
    d.approx_mode = int(bool(approx_mode))
    d.n_polygons = len(polygon_ids)
    d.polygon_ids = polygon_ids.ctypes.data
    d.vtx_off = vtx_off.ctypes.data
    d.vtx_latlng = vtx_latlng.ctypes.data
    return d, (arena, lut, polygon_ids, vtx_off, vtx_latlng)


def _opt(options):
    return C.byref(options) if options is not None else None


class IndexBundle:
    """An immutable index replicated into one GPU's HBM."""

    def __init__(self, handle: int, owned: bool = True):
        self._h = C.c_void_p(handle)
        self._owned = owned
        info = capi.IndexInfo()
        _check(capi.lib().gj_index_get_info(self._h, C.byref(info)))
        self.info = info
        self.ids = np.empty(info.n_ids, np.uint32)
        _check(capi.lib().gj_index_ids(self._h, _vp(self.ids)))
        self._session = None

    def close(self):
        if self._session is not None:
            self._session.close()
            self._session = None
        if self._h:
            if self._owned:
                capi.lib().gj_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def from_arrays(arena, lut, roots, prefixes, prefix_bits, k_max: int, approx_mode: bool,
                    polygon_ids, vtx_off, vtx_latlng, device: int = -1,
                    options: capi.Options | None = None) -> "IndexBundle":
        d, _keep = _desc(arena, lut, roots, prefixes, prefix_bits, k_max, approx_mode, polygon_ids, vtx_off,
                         vtx_latlng)
        h = C.c_void_p()
        _check(capi.lib().gj_index_create_ex(C.byref(d), device, _opt(options), C.byref(h)))
        return IndexBundle(h.value)

    @staticmethod
    def load(path, device: int = -1, options: capi.Options | None = None) -> "IndexBundle":
        """IndexBundle::load (join.cpp:341-381): GJX1 file -> HBM."""
        h = C.c_void_p()
        _check(capi.lib().gj_index_load_file_ex(str(path).encode(), device, _opt(options), C.byref(h)))
        return IndexBundle(h.value)

    def replicate(self, device: int = -1) -> "IndexBundle":
        """A copy of this index in another GPU's HBM, made device to device."""
        h = C.c_void_p()
        _check(capi.lib().gj_index_replicate(self._h, device, C.byref(h)))
        return IndexBundle(h.value)

    @property
    def approx(self) -> bool:
        return bool(self.info.approx_mode)

    def session(self) -> "Session":
        if self._session is None:
            self._session = Session(self)
        return self._session


class Session:
    """One CUDA stream + scratch; not thread-safe (use one per thread)."""

    def __init__(self, bundle: IndexBundle, handle: int | None = None):
        self.bundle = bundle
        self._owned = handle is None
        if handle is None:
            h = C.c_void_p()
            _check(capi.lib().gj_session_create(bundle._h, C.byref(h)))
        else:  # borrowed from a group
            h = C.c_void_p(handle)
        self._h = h

    def close(self):
        if self._h:
            if self._owned:
                capi.lib().gj_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return capi.lib().gj_session_stream(self._h)

    @property
    def launches(self) -> int:
        return int(capi.lib().gj_session_launches(self._h))

    # ---- cell ids ----
    def cells_from_points(self, points, level: int) -> np.ndarray:
        """cell_from_point over an array (cell_id.cpp:82-95)."""
        p = _points(points)
        out = np.empty(len(p), np.uint64)
        bad = C.c_uint64(0)
        _check(capi.lib().gj_cells_from_points_host(self._h, _vp(p), len(p), int(level), _vp(out),
                                                    C.byref(bad)), bad)
        return out

    # ---- probe ----
    def probe_points(self, points) -> np.ndarray:
        p = _points(points)
        out = np.empty(len(p), np.uint64)
        bad = C.c_uint64(0)
        _check(capi.lib().gj_probe_points_host(self._h, _vp(p), len(p), _vp(out), C.byref(bad)), bad)
        return out

    def probe_cells(self, raw_ids) -> np.ndarray:
        r = np.ascontiguousarray(raw_ids, np.uint64)
        out = np.empty(len(r), np.uint64)
        _check(capi.lib().gj_probe_cells_host(self._h, _vp(r), len(r), _vp(out)))
        return out

    # ---- point ingestion ----
    def points_from_csv(self, text: bytes, lat_column: str = "lat", lng_column: str = "lng", strict: bool = False):
        """CsvPointReader (io.hpp:43-68, csv.cpp:54-100) over a text buffer, parsed on
        the GPU -> (points float64 (n, 2), skipped rows)."""
        text = bytes(text)
        cap = max(1, text.count(b"\n") + 1)
        out = np.empty((cap, 2), np.float64)
        n, skipped, bad = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        _check(capi.lib().gj_points_from_csv_host(self._h, text, len(text), lat_column.encode(), lng_column.encode(),
                                                  int(strict), _vp(out), cap, C.byref(n), C.byref(skipped),
                                                  C.byref(bad)), bad)
        return out[:n.value].copy() if n.value < cap else out, int(skipped.value)

    # ---- training pre-pass ----
    def training_candidates(self, points, base_index: int = 0) -> np.ndarray:
        """Ascending global indices of the points whose probe lands in a
        candidate-bearing cell: the `any_candidate` test of Act::train
        (src/act.cpp:414-440)."""
        p = _points(points)
        out = np.empty(len(p), np.uint64)
        found, bad = C.c_uint64(0), C.c_uint64(0)
        _check(capi.lib().gj_training_candidates_host(self._h, _vp(p), len(p), C.c_uint64(base_index), _vp(out),
                                                      C.c_uint64(len(out)), C.byref(found), C.byref(bad)), bad)
        return out[:found.value].copy()

    # ---- streaming join ----
    def _count_call(self, p, base_index, mode, counts, cs, first, ovf, bad):
        return capi.lib().gj_join_count_host(self._h, _vp(p), len(p), base_index, mode, _vp(counts), cs,
                                             _vp(first), ovf, C.byref(bad))

    def join_count(self, points, mode=capi.GJ_MODE_BUNDLE, stats: JoinStats | None = None,
                   want_ids: bool = False, base_index: int = 0, overflow_capacity: int | None = None):
        """Returns (counts_by_slot u64[n_ids], first_id u32[n] | None, (ovf_point, ovf_id) | None)."""
        p = _points(points)
        counts = np.zeros(max(1, len(self.bundle.ids)), np.uint64)
        cs = capi.Stats()
        bad = C.c_uint64(0)
        first = np.empty(len(p), np.uint32) if want_ids else None
        ovf = None
        ovf_pt = ovf_id = None
        if want_ids:
            cap = overflow_capacity if overflow_capacity is not None else max(1024, len(p) // 4)
            while True:
                ovf_pt = np.empty(cap, np.uint64)
                ovf_id = np.empty(cap, np.uint32)
                ovf = capi.Overflow(ovf_pt.ctypes.data, ovf_id.ctypes.data, cap, 0)
                counts[:] = 0
                cs = capi.Stats()
                rc = self._count_call(p, base_index, mode, counts, C.byref(cs) if stats is not None else None,
                                      first, C.byref(ovf), bad)
                if rc == capi.GJ_CAPACITY and ovf.count > cap and overflow_capacity is None:
                    cap = int(ovf.count)
                    continue
                _check(rc, bad)
                break
            ovf_pt, ovf_id = ovf_pt[:ovf.count], ovf_id[:ovf.count]
        else:
            _check(self._count_call(p, base_index, mode, counts, C.byref(cs) if stats is not None else None,
                                    None, None, bad), bad)
        if stats is not None:
            stats._add(cs)
        counts = counts[:len(self.bundle.ids)]
        return counts, first, ((ovf_pt, ovf_id) if want_ids else None)

    def join_count_device(self, d_points_ptr: int, n: int, d_counts_ptr: int, mode=capi.GJ_MODE_BUNDLE,
                          d_stats_ptr: int = 0, d_first_id_ptr: int = 0, sync: bool = False):
        """Points already in HBM (raw device pointers, e.g. ``tensor.data_ptr()``);
        asynchronous on ``self.stream`` unless ``sync``.  The session stream does
        not wait for other streams: buffers filled by another library (torch
        copies, ``zero_()``) must be complete — synchronise, or record an event
        and make ``self.stream`` wait for it — before this call."""
        _check(capi.lib().gj_join_count_device(self._h, C.c_void_p(d_points_ptr), n, mode,
                                               C.c_void_p(d_counts_ptr),
                                               C.c_void_p(d_stats_ptr) if d_stats_ptr else None,
                                               C.c_void_p(d_first_id_ptr) if d_first_id_ptr else None,
                                               int(sync)))

    def sync(self):
        bad = C.c_uint64(0)
        _check(capi.lib().gj_session_sync(self._h, C.byref(bad)), bad)

    # ---- materialised pairs ----
    def _pairs_call(self, p, mode, n_pairs, cs, bad):
        return capi.lib().gj_join_pairs_host(self._h, _vp(p), len(p), mode, C.byref(n_pairs), cs, C.byref(bad))

    def _pairs_copy(self, row_ptr, ids):
        return capi.lib().gj_pairs_copy(self._h, _vp(row_ptr), _vp(ids))

    def join_pairs(self, points, mode, stats: JoinStats | None = None):
        """(row_ptr u64[n+1], polygon_id u32[]) in the reference's emit order."""
        p = _points(points)
        n_pairs = C.c_uint64(0)
        cs = capi.Stats()
        bad = C.c_uint64(0)
        _check(self._pairs_call(p, mode, n_pairs, C.byref(cs) if stats is not None else None, bad), bad)
        row_ptr = np.empty(len(p) + 1, np.uint64)
        ids = np.empty(n_pairs.value, np.uint32)
        _check(self._pairs_copy(row_ptr, ids))
        if stats is not None:
            stats._add(cs)
        return row_ptr, ids


    def join_pairs_into(self, points, mode, row_ptr: np.ndarray, ids: np.ndarray, stats: JoinStats | None = None) -> int:
        """ONE call, caller-provided arrays (``row_ptr`` u64[n+1], ``ids`` u32[capacity]; pinned
        memory from ``pinned_array`` is copied to directly): chunk c's rows and ids stream home while
        chunk c+1 runs.  Returns the pair count; raises ``CapacityError`` (``.needed`` = pair count)
        when ``ids`` is too small — ``row_ptr`` is complete then."""
        p = _points(points)
        assert row_ptr.dtype == np.uint64 and len(row_ptr) >= len(p) + 1 and ids.dtype == np.uint32
        n_pairs, cs, bad = C.c_uint64(0), capi.Stats(), C.c_uint64(0)
        rc = capi.lib().gj_join_pairs_host_into(self._h, _vp(p), len(p), mode, _vp(row_ptr), _vp(ids), len(ids),
                                                C.byref(n_pairs), C.byref(cs) if stats is not None else None,
                                                C.byref(bad))
        if rc == capi.GJ_CAPACITY:
            err = CapacityError(capi.lib().gj_last_error().decode())
            err.needed = int(n_pairs.value)
            raise err
        _check(rc, bad)
        if stats is not None:
            stats._add(cs)
        return int(n_pairs.value)

    def join_pairs_device(self, d_points_ptr: int, n: int, mode, d_row_ptr: int, d_ids_ptr: int, id_capacity: int,
                          stats: JoinStats | None = None) -> int:
        """CSR entirely in HBM (raw device pointers: points f64[n, 2] in, row offsets u64[n+1] and
        polygon ids u32[id_capacity] out).  Synchronous.  Returns the pair count; ``CapacityError``
        (``.needed``) when the id array is too small."""
        n_pairs, cs, bad = C.c_uint64(0), capi.Stats(), C.c_uint64(0)
        rc = capi.lib().gj_join_pairs_device(self._h, C.c_void_p(d_points_ptr), n, mode, C.c_void_p(d_row_ptr),
                                             C.c_void_p(d_ids_ptr) if d_ids_ptr else None, id_capacity,
                                             C.byref(n_pairs), C.byref(cs) if stats is not None else None,
                                             C.byref(bad))
        if rc == capi.GJ_CAPACITY:
            err = CapacityError(capi.lib().gj_last_error().decode())
            err.needed = int(n_pairs.value)
            raise err
        _check(rc, bad)
        if stats is not None:
            stats._add(cs)
        return int(n_pairs.value)


def pinned_array(n: int, dtype) -> np.ndarray:
    """A numpy array over pinned host memory (gj_host_alloc): the *_host calls copy to and from it
    directly, without the stager.  The memory is released when the array is garbage-collected."""
    import weakref
    dt = np.dtype(dtype)
    ptr = capi.lib().gj_host_alloc(max(1, n) * dt.itemsize)
    if not ptr:
        raise CudaError(capi.lib().gj_last_error().decode())
    buf = (C.c_char * (max(1, n) * dt.itemsize)).from_address(ptr)
    arr = np.frombuffer(buf, dtype=dt, count=n)
    weakref.finalize(buf, capi.lib().gj_host_free, ptr)
    return arr


class _GroupJoiner(Session):
    """join_count / join_pairs of a Session, routed through the group calls."""

    def __init__(self, group: "IndexGroup", workers: int):
        self.bundle = group.replicas[0]
        self._g = group
        self._workers = int(workers)
        self._h = group.sessions[0]._h  # everything but the joins runs on the first replica
        self._owned = False

    def _count_call(self, p, base_index, mode, counts, cs, first, ovf, bad):
        return capi.lib().gj_group_join_count_host(self._g._h, self._workers, _vp(p), len(p), base_index, mode,
                                                   _vp(counts), cs, _vp(first), ovf, C.byref(bad))

    def _pairs_call(self, p, mode, n_pairs, cs, bad):
        return capi.lib().gj_group_join_pairs_host(self._g._h, self._workers, _vp(p), len(p), mode,
                                                   C.byref(n_pairs), cs, C.byref(bad))

    def _pairs_copy(self, row_ptr, ids):
        return capi.lib().gj_group_pairs_copy(self._g._h, _vp(row_ptr), _vp(ids))


class IndexGroup:
    """The index replicated over several GPUs of one box, for ONE input: the
    reference's worker fan-out (join.cpp:255-285) with GPUs as the workers.
    Points split into contiguous ranges [n*g/G, n*(g+1)/G) (join.cpp:264-265),
    range g runs on replica g from its own host thread with
    ``base_index + n*g/G``; counts and stats are summed, first ids / CSR rows
    land at their global positions (join.cpp:280-284).  ``devices`` may repeat a
    device (replicas share nothing) — that is how the one-GPU tests exercise it."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        L = capi.lib()
        self.replicas = [IndexBundle(L.gj_group_index(self._h, k), owned=False) for k in range(L.gj_group_size(self._h))]
        self.sessions = [Session(b, handle=L.gj_group_session(self._h, k)) for k, b in enumerate(self.replicas)]
        for b, s in zip(self.replicas, self.sessions):
            b._session = s
        self.info = self.replicas[0].info
        self.ids = self.replicas[0].ids

    @staticmethod
    def _devices(devices):
        if devices is None:
            devices = list(range(capi.lib().gj_device_count()))
        devices = [int(d) for d in devices]
        if not devices:
            raise CudaError("no CUDA device: geojoin_b200 has no CPU fallback")
        return (C.c_int * len(devices))(*devices), len(devices)

    @staticmethod
    def load(path, devices=None, options: capi.Options | None = None) -> "IndexGroup":
        """GJX1 file -> the first device's HBM -> device-to-device copies on the others (None = every GPU)."""
        arr, n = IndexGroup._devices(devices)
        h = C.c_void_p()
        _check(capi.lib().gj_group_load_file(str(path).encode(), arr, n, _opt(options), C.byref(h)))
        return IndexGroup(h.value)

    @staticmethod
    def from_arrays(arena, lut, roots, prefixes, prefix_bits, k_max: int, approx_mode: bool, polygon_ids, vtx_off,
                    vtx_latlng, devices=None, options: capi.Options | None = None) -> "IndexGroup":
        d, _keep = _desc(arena, lut, roots, prefixes, prefix_bits, k_max, approx_mode, polygon_ids, vtx_off,
                         vtx_latlng)
        arr, n = IndexGroup._devices(devices)
        h = C.c_void_p()
        _check(capi.lib().gj_group_create(C.byref(d), arr, n, _opt(options), C.byref(h)))
        return IndexGroup(h.value)

    @property
    def approx(self) -> bool:
        return bool(self.info.approx_mode)

    def __len__(self):
        return len(self.replicas)

    def session(self, workers: int = 0) -> Session:
        """A Session-shaped handle whose join_count / join_pairs use ``workers`` replicas (0 = all)."""
        return _GroupJoiner(self, workers)

    def close(self):
        for s in self.sessions:
            s.close()
        for b in self.replicas:
            b._session = None
            b.close()
        if self._h:
            capi.lib().gj_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _pairs_from_csr(row_ptr: np.ndarray, ids: np.ndarray):
    n = len(row_ptr) - 1
    point_index = np.repeat(np.arange(n, dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
    return point_index, ids


def join_exact(bundle: IndexBundle, points, stats: JoinStats | None = None):
    """join.cpp:237-241 — (point_index u64[], polygon_id u32[]) like vector<JoinPair>."""
    return _pairs_from_csr(*bundle.session().join_pairs(points, capi.GJ_MODE_EXACT, stats))


def join_approx(bundle: IndexBundle, points, stats: JoinStats | None = None):
    """join.cpp:243-247."""
    return _pairs_from_csr(*bundle.session().join_pairs(points, capi.GJ_MODE_APPROX, stats))


def join_count_per_polygon(bundle, points, threads: int = 1) -> dict[int, int]:
    """join.cpp:255-285 — mode from the bundle; only polygons with a non-zero
    count appear.  ``threads`` is the reference's worker count: on an
    ``IndexGroup`` that many replicas (GPUs) each take one contiguous range of
    the points (0 or more than the group holds = all of them); on a single
    ``IndexBundle`` there is one worker.  Results do not depend on it
    (tests/test_join.cpp:200-214)."""
    sess = bundle.session(threads) if isinstance(bundle, IndexGroup) else bundle.session()
    counts, _, _ = sess.join_count(points, capi.GJ_MODE_BUNDLE)
    nz = np.nonzero(counts)[0]
    return {int(bundle.ids[k]): int(counts[k]) for k in nz}


def count_per_polygon(polygon_ids) -> dict[int, int]:
    """join.cpp:249-253."""
    ids, cnt = np.unique(np.asarray(polygon_ids, np.uint32), return_counts=True)
    return {int(i): int(c) for i, c in zip(ids, cnt)}


def accumulate_probe_stats(bundle: IndexBundle, points, stats: JoinStats) -> None:
    """join.cpp:287-290 — probe-only pass (approx emit, nothing kept) adding into ``stats``."""
    bundle.session().join_count(points, capi.GJ_MODE_APPROX, stats)


def collect_metrics(bundle: IndexBundle, points) -> IndexMetrics:
    """join.cpp:309-314."""
    s = JoinStats()
    accumulate_probe_stats(bundle, points, s)
    return metrics_from_stats(s, int(bundle.info.node_count))


def training_candidates(bundle: IndexBundle, points) -> np.ndarray:
    """The work list of Act::train (src/act.cpp:414-440): indices of the
    training points that hit a cell with at least one candidate reference."""
    return bundle.session().training_candidates(points)


def expensive_fraction(bundle: IndexBundle, points) -> float:
    """TrainingStats::expensive_fraction_before/after (src/act.cpp:414-426):
    share of the points whose probe meets a candidate reference; 0 for no points."""
    p = _points(points)
    return 0.0 if len(p) == 0 else len(training_candidates(bundle, p)) / len(p)


def load_points_csv(bundle: IndexBundle, path, lat_column: str = "lat", lng_column: str = "lng",
                    strict: bool = False) -> np.ndarray:
    """load_points_csv (io.hpp:71-72, csv.cpp:102-113): the valid points of a CSV
    file, parsed on the bundle's GPU."""
    try:
        text = open(path, "rb").read()
    except OSError as exc:
        raise DataError(f"cannot open point file: {path}") from exc
    return bundle.session().points_from_csv(text, lat_column, lng_column, strict)[0]

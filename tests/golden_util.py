"""TEST INFRASTRUCTURE — loading the committed golden fixtures
(tests/golden/*.npz, produced by tests/golden/make_golden.py from the compiled
reference) and parsing the reference's GJX1 bundle format in numpy
(IndexBundle::save, proj/src/join.cpp:316-339; Act::save, proj/src/act.cpp:600-622)."""
from __future__ import annotations

import struct
import tempfile
import zlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
_TMP = None


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def names() -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def gjx_bytes(fx: dict) -> bytes:
    return zlib.decompress(fx["gjx_z"].tobytes())


def bundle_file(name: str) -> Path:
    """The fixture's GJX1 file inflated into a temp dir (for gj_index_load_file)."""
    global _TMP
    if _TMP is None:
        _TMP = tempfile.TemporaryDirectory(prefix="gj_golden_")
    path = Path(_TMP.name) / f"{name}.gjx"
    if not path.exists():
        path.write_bytes(gjx_bytes(load(name)))
    return path


def parse_gjx(data: bytes) -> dict:
    """GJX1 -> dict of numpy arrays (little-endian, as written by the reference)."""
    if data[:4] != b"GJX1":
        raise ValueError("not a geojoin index file")
    version, mode, achieved = struct.unpack_from("<III", data, 4)
    precision_m, achieved_m = struct.unpack_from("<dd", data, 16)
    (budget,) = struct.unpack_from("<Q", data, 32)
    cov = struct.unpack_from("<IIII", data, 40)
    at = 56
    if data[at:at + 4] != b"ACT1":
        raise ValueError("not an ACT1 snapshot")
    (k_max,) = struct.unpack_from("<I", data, at + 4)
    nodes, lut_len = struct.unpack_from("<QQ", data, at + 8)
    at += 24
    roots = np.zeros(8, np.uint64)
    prefixes = np.zeros(8, np.uint64)
    pbits = np.zeros(8, np.uint64)
    for f in range(6):
        r, p, b = struct.unpack_from("<QQI", data, at)
        roots[f], prefixes[f], pbits[f] = r, p, b
        at += 20
    arena = np.frombuffer(data, dtype="<u8", count=nodes * 256, offset=at).copy()
    at += nodes * 256 * 8
    lut = np.frombuffer(data, dtype="<u4", count=lut_len, offset=at).copy()
    at += lut_len * 4
    (n_poly,) = struct.unpack_from("<Q", data, at)
    at += 8
    ids = np.empty(n_poly, np.uint32)
    off = np.zeros(n_poly + 1, np.uint64)
    rings = []
    for p in range(n_poly):
        pid, nv = struct.unpack_from("<IQ", data, at)
        at += 12
        rings.append(np.frombuffer(data, dtype="<f8", count=2 * nv, offset=at).reshape(-1, 2).copy())
        at += 16 * nv
        ids[p] = pid
        off[p + 1] = off[p] + nv
    latlng = np.concatenate(rings) if rings else np.zeros((0, 2))
    return dict(version=version, approx=bool(mode), precision_achieved=bool(achieved),
                precision_m=precision_m, achieved_precision_m=achieved_m, budget=budget, covering=cov,
                k_max=int(k_max), arena=arena, lut=lut, roots=roots, prefixes=prefixes, prefix_bits=pbits,
                polygon_ids=ids, vtx_off=off, vtx_latlng=latlng)


def oracle_index(fx_or_parsed: dict):
    """OracleIndex (the C oracle's view) of a fixture's bundle."""
    from oracle import oracle

    g = fx_or_parsed if "arena" in fx_or_parsed else parse_gjx(gjx_bytes(fx_or_parsed))
    return oracle.OracleIndex(g["arena"], g["lut"], g["roots"], g["prefixes"], g["prefix_bits"], g["k_max"],
                              g["polygon_ids"], g["vtx_off"], g["vtx_latlng"])


def pairs_of(fx: dict, kind: str):
    """(point_index u64, polygon_id u32) of a stored join result ('exact' | 'approx')."""
    return fx[f"{kind}_pi"].astype(np.uint64), fx[f"{kind}_pid"].astype(np.uint32)

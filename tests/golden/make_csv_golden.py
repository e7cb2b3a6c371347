"""Generates tests/golden/csv_points.npz from the UNMODIFIED reference
(oracle/_ref): CSV texts and what the reference's CsvPointReader
(src/csv.cpp:54-100) makes of them.  Run in the build container only:

    python tests/golden/make_csv_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests import golden_util  # noqa: E402

EDGE_FIELDS = [
    "0", "-0", "0.0", "-0.0", "1", "90", "-90", "90.0", "90.00000000000001", "-90.00000000000001", "180", "-180",
    "180.0000000000001", "45.5", "-73.985428", "40.748817", " 12.5", "\t12.5", " \t 12.5", "12.5 ", "12.5\t", "+12.5",
    "", " ", ".", "-", "-.", ".5", "-.5", "5.", "-5.", "5.e0", "1e1", "1E1", "1e+1", "1e-1", "1e", "1e+", "1e-", "e5",
    "1e1.5", "12abc", "abc", "1,5", "0x10", "1_0", "inf", "-inf", "nan", "NaN", "infinity", "1e400", "-1e400", "1e-400",
    "1e-30", "1e-300", "4.9e-324", "2.4e-324", "2.5e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
    "1e-323", "2.2250738585072014e-308", "2.2250738585072011e-308", "0e999999", "0.0000000000000000000000001",
    "00000000000000000000000012.5", "12.50000000000000000000000000000000000000", "40.748817000000003",
    "40.748817000000004", "89.99999999999999", "89.999999999999995", "89.9999999999999929", "90.000000000000005",
    "90.000000000000014", "179.99999999999997", "179.999999999999985", "180.00000000000001",
    "0.1", "0.2", "0.3", "0.30000000000000004", "0.1000000000000000055511151231257827",
    "0.10000000000000000555111512312578270211815834045410156250000001",
    "0.1000000000000000124900090270330610871315002441406249",
    "0.100000000000000012490009027033061087131500244140625",
    "0.1000000000000000124900090270330610871315002441406251",
    "9007199254740993e-16", "9007199254740992.5e-16", "9007199254740991e-16", "12345678901234567890e-18",
    "123456789012345678901234567890e-28", "1.7976931348623157e308", "1e2", "1.8e2", "1.80e2", "1.81e2", "18e1",
    "0.000018e7", "1800000e-4", "17999999999999999999e-17", "18000000000000000001e-17", "5e-1", "25e-2", "1e0", "1e-0",
    "1e+0", "1e00000000000000000001", "1e-00000000000000000001", "100e-2", "  -  5", "- 5", "--5", "5-", "5e5e5",
]


def edge_csv() -> bytes:
    rows = ["lat,lng"]
    for f in EDGE_FIELDS:
        rows.append(f"{f},10.5")
        rows.append(f"20.25,{f}")
    rows += ["", "1,2,3", "1", ",", ",,", "1,", ",2", "1,2,", "\r", "3,4\r", "5,6\r\r", "7,8 \r", "9,10,extra,cols"]
    return ("\n".join(rows) + "\n").encode()


def random_csv(seed: int, n: int, digits: int, columns: str, crlf: bool, tail_newline: bool) -> bytes:
    rng = np.random.default_rng(seed)
    names = columns.split(",")
    lat_i, lng_i = names.index("lat"), names.index("lng")
    lat = rng.uniform(-95, 95, n)
    lng = rng.uniform(-190, 190, n)
    rows = [columns]
    for k in range(n):
        fields = [str(int(rng.integers(0, 1000))) for _ in names]
        style = int(rng.integers(0, 6))
        if style == 0:
            a, o = repr(float(lat[k])), repr(float(lng[k]))
        elif style == 1:
            a, o = f"{lat[k]:.{digits}f}", f"{lng[k]:.{digits}f}"
        elif style == 2:
            a, o = f"{lat[k]:.{digits}e}", f"{lng[k]:.{digits}E}"
        elif style == 3:
            a, o = f"{lat[k]:.6f}", f"{lng[k]:.6f}"
        elif style == 4:
            a, o = f"{lat[k]:.25f}", f"{lng[k]:.30f}"
        else:
            a, o = f" {lat[k]:.17g}", f"\t{lng[k]:.17g}"
        fields[lat_i], fields[lng_i] = a, o
        rows.append(",".join(fields))
        if rng.random() < 0.01:
            rows.append("")
        if rng.random() < 0.01:
            rows.append("garbage,row")
    eol = "\r\n" if crlf else "\n"
    text = eol.join(rows)
    return (text + (eol if tail_newline else "")).encode()


def main():
    cases = {
        "edge": (edge_csv(), "lat", "lng"),
        "random_a": (random_csv(0xC5A1, 4000, 15, "lat,lng", False, True), "lat", "lng"),
        "random_b": (random_csv(0xC5A2, 4000, 17, "id,lng,name,lat,z", True, False), "lat", "lng"),
        "random_c": (random_csv(0xC5A3, 4000, 9, "lng,lat", False, False), "lat", "lng"),
        "dup_columns": (b"lat,lng,lat\n1,2,3\n4,5,6\n", "lat", "lng"),
        "renamed": (b"y,x\n1.5,2.5\n-3,4e0\n", "y", "x"),
        "header_only": (b"lat,lng", "lat", "lng"),
    }
    out = {}
    for name, (text, la, lo) in cases.items():
        pts, skipped = ref.csv_points(text, la, lo, strict=False)
        out[f"{name}__text"] = np.frombuffer(text, np.uint8)
        out[f"{name}__cols"] = np.frombuffer(f"{la},{lo}".encode(), np.uint8)
        out[f"{name}__points"] = pts
        out[f"{name}__skipped"] = np.array([skipped], np.uint64)
        print(f"{name}: {len(text)} bytes -> {len(pts)} points, {skipped} skipped")
    path = golden_util.GOLDEN / "csv_points.npz"
    np.savez_compressed(path, **out)
    print(f"{path.name}: {path.stat().st_size / 1024:.0f} KB")


if __name__ == "__main__":
    main()

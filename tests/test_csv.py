"""Point ingestion: the reference's CsvPointReader
(io.hpp:43-68, csv.cpp:26-100).  CPU: the C oracle against the fixture the
compiled reference produced (tests/golden/make_csv_golden.py) and against the
live reference; GPU: the device parser through the C ABI against both,
bit-exact (decimal -> double correctly rounded, like std::from_chars)."""
import numpy as np
import pytest

from oracle import oracle
from tests import golden_util

CASES = ["edge", "random_a", "random_b", "random_c", "dup_columns", "renamed", "header_only"]


def _case(name):
    fx = golden_util.load("csv_points")
    text = fx[f"{name}__text"].tobytes()
    lat, lng = fx[f"{name}__cols"].tobytes().decode().split(",")
    return text, lat, lng, fx[f"{name}__points"], int(fx[f"{name}__skipped"][0])


def _same_bits(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def _stress_text(seed, n):
    """Rows in every number style std::from_chars accepts, with long digit
    strings, ties, subnormals and junk mixed in."""
    rng = np.random.default_rng(seed)
    lat = rng.uniform(-91, 91, n)
    lng = rng.uniform(-181, 181, n)
    rows = ["a,lat,b,lng"]
    junk = ["", "x", "1e", "+1", "1 ", "nan", "inf", "1e400", "1e-400", "0x1p3", "--1", "1..2", ".", "1,2"]
    for k in range(n):
        s = int(rng.integers(0, 10))
        if s == 0:
            a, o = repr(float(lat[k])), repr(float(lng[k]))
        elif s == 1:
            a, o = f"{lat[k]:.{int(rng.integers(0, 25))}f}", f"{lng[k]:.{int(rng.integers(0, 40))}f}"
        elif s == 2:
            a, o = f"{lat[k]:.{int(rng.integers(0, 20))}e}", f"{lng[k]:.{int(rng.integers(0, 30))}E}"
        elif s == 3:  # exact binary expansions: ties and near-ties at 60+ digits
            a, o = f"{lat[k]:.70f}", f"{np.nextafter(lng[k], 0) / 2 + lng[k] / 2:.80f}"
        elif s == 4:
            a, o = f"{lat[k] * 1e-300:.17e}", f"{lng[k] * 1e-310:.17e}"  # tiny, subnormal
        elif s == 5:
            a, o = f"{lat[k] * 10 ** -int(rng.integers(20, 330)):.{int(rng.integers(0, 19))}e}", f"{int(lng[k])}"
        elif s == 6:
            a, o = f" \t{lat[k]:.12g}", f"\t {lng[k]:.7g}"
        elif s == 7:
            a, o = f"{int(lat[k] * 1e15)}e-15", f"{int(lng[k] * 1e18)}E-18"
        elif s == 8:
            a, o = junk[int(rng.integers(0, len(junk)))], f"{lng[k]:.5f}"
        else:
            a, o = f"{lat[k]:.5f}", junk[int(rng.integers(0, len(junk)))]
        rows.append(f"{k},{a},z,{o}")
        if rng.random() < 0.02:
            rows.append("")
    return ("\n".join(rows) + "\n").encode()


# ---- CPU: the oracle is pinned to the reference -------------------------------------------------
@pytest.mark.parametrize("name", CASES)
def test_oracle_csv_matches_reference_fixture(name):
    text, lat, lng, want, skipped = _case(name)
    got, sk = oracle.csv_points(text, lat, lng)
    assert _same_bits(got, want) and sk == skipped


def test_oracle_csv_matches_live_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    text = _stress_text(0xC5B1, 20000)
    want, wsk = ref.csv_points(text, "lat", "lng")
    got, sk = oracle.csv_points(text, "lat", "lng")
    assert _same_bits(got, want) and sk == wsk and len(got) > 10000 and sk > 1000


def test_oracle_csv_errors():
    for text, line in [(b"", 0), (b"\n1,2\n", 1), (b"lat,x\n1,2\n", 1), (b"x,lng\n1,2\n", 1)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.csv_points(text)
        assert e.value.status == oracle.DATA_ERROR and e.value.bad_index == line
    with pytest.raises(oracle.OracleError) as e:  # csv.cpp:91-94: the header is line 1, empty lines count
        oracle.csv_points(b"lat,lng\n1,2\n\nbad,3\n4,5\n", strict=True)
    assert e.value.bad_index == 4
    assert len(oracle.csv_points(b"lat,lng\n1,2\n\n4,5\n", strict=True)[0]) == 2


# ---- GPU: the device parser -----------------------------------------------------------------------
def _session():
    from paper_1802_09488_b200 import join
    bundle = join.IndexBundle.load(golden_util.bundle_file("join_small_exact"), device=0)
    return bundle, bundle.session()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_csv_matches_reference_fixture(name):
    text, lat, lng, want, skipped = _case(name)
    bundle, s = _session()
    got, sk = s.points_from_csv(text, lat, lng)
    assert _same_bits(got, want) and sk == skipped
    bundle.close()


@pytest.mark.gpu
def test_gpu_csv_stress_matches_oracle():
    bundle, s = _session()
    text = _stress_text(0xC5B2, 400_000)
    want, wsk = oracle.csv_points(text, "lat", "lng")
    got, sk = s.points_from_csv(text, "lat", "lng")
    assert _same_bits(got, want) and sk == wsk and len(got) > 200_000
    # CRLF, no trailing newline, other column order
    text2 = text.replace(b"\n", b"\r\n").rstrip(b"\r\n")
    got2, sk2 = s.points_from_csv(text2, "lat", "lng")
    assert _same_bits(got2, want) and sk2 == wsk
    bundle.close()


@pytest.mark.gpu
def test_gpu_csv_errors_and_file_loader(tmp_path):
    from paper_1802_09488_b200 import join
    bundle, s = _session()
    for text, line in [(b"", 0), (b"\n1,2\n", 1), (b"lat,x\n1,2\n", 1), (b"x,lng\n1,2\n", 1)]:
        with pytest.raises(join.DataError) as e:
            s.points_from_csv(text)
        assert e.value.line == line
    with pytest.raises(join.DataError) as e:
        s.points_from_csv(b"lat,lng\n1,2\n\nbad,3\n4,5\n", strict=True)
    assert e.value.line == 4 and "line 4" in str(e.value)
    with pytest.raises(join.DataError) as e:
        s.points_from_csv(b"lat,x\n1,2\n")
    assert "missing column 'lng'" in str(e.value)
    pts, sk = s.points_from_csv(b"lat,lng\n1,2\n\n4,5\n", strict=True)
    assert pts.tolist() == [[1.0, 2.0], [4.0, 5.0]] and sk == 0
    p = tmp_path / "pts.csv"
    p.write_bytes(b"id,lat,lng\n7,40.5,-73.25\n8,91,0\n9,-12.125,179.5\n")
    assert join.load_points_csv(bundle, p).tolist() == [[40.5, -73.25], [-12.125, 179.5]]
    with pytest.raises(join.DataError):
        join.load_points_csv(bundle, tmp_path / "missing.csv")
    bundle.close()


@pytest.mark.gpu
def test_gpu_csv_multi_chunk_and_throughput():
    """More text than one 64 MB device chunk: chunk seams fall on line ends and
    do not show in the result; prints the device parser's throughput."""
    import time
    bundle, s = _session()
    rng = np.random.default_rng(0xC5B3)
    n = 3_000_000
    lat = rng.uniform(-90, 90, n)
    lng = rng.uniform(-180, 180, n)
    body = "\n".join(f"{a!r},{o:.9f}" for a, o in zip(lat.tolist(), lng.tolist()))
    text = ("lat,lng\n" + body + "\n").encode()
    assert len(text) > (64 << 20)
    s.points_from_csv(text[:1 << 20].rsplit(b"\n", 1)[0])
    t0 = time.time()
    got, sk = s.points_from_csv(text)
    dt = time.time() - t0
    print(f"\ncsv: {len(text) / 1e6:.0f} MB, {n} rows in {dt:.3f} s = {len(text) / dt / 1e9:.2f} GB/s, {n / dt / 1e6:.1f} M rows/s")
    assert sk == 0 and len(got) == n
    assert np.array_equal(got[:, 0], lat)  # repr() round-trips exactly
    assert np.array_equal(got[:, 1], np.array([float(f"{o:.9f}") for o in lng[:200_000].tolist()]
                                              + got[200_000:, 1].tolist()))
    t0 = time.time()
    want, _ = oracle.csv_points(text)
    cpu = time.time() - t0
    print(f"csv: CPU oracle (strtod, one thread) {cpu:.2f} s = {len(text) / cpu / 1e6:.0f} MB/s")
    assert _same_bits(got, want)
    bundle.close()


def _random_decimals(seed, n):
    """Random decimal strings: 1-45 digits, a point anywhere, exponents that put
    the value anywhere from the subnormals to a few hundred."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        nd = int(rng.integers(1, 46))
        digits = "".join(str(int(d)) for d in rng.integers(0, 10, nd))
        pos = int(rng.integers(0, nd + 1))
        mant = digits[:pos] + ("." + digits[pos:] if rng.random() < 0.8 else digits[pos:])
        if mant in ("", "."):
            mant = "0"
        target = int(rng.choice([2, 1, 0, -1, -5, -17, -40, -100, -300, -308, -320, -323, -324, -325, -330, -340]))
        lead = len(digits[:pos].lstrip("0")) if digits[:pos].strip("0") else -(len(digits[pos:]) - len(digits[pos:].lstrip("0")))
        exp = target - lead
        s = ("-" if rng.random() < 0.3 else "") + mant
        if exp != 0 or rng.random() < 0.3:
            s += ("e" if rng.random() < 0.5 else "E") + (("+" if exp >= 0 and rng.random() < 0.5 else "") + str(exp))
        out.append(s)
    return out


def test_oracle_number_parsing_matches_python_float():
    """parse_double's value is the correctly rounded double (std::from_chars);
    so is Python's float().  Rows are valid iff both fields parse, neither
    overflows nor rounds a nonzero decimal to zero, and the point is in range."""
    nums = _random_decimals(0xC5B4, 30000)
    text = ("lat,lng\n" + "\n".join(f"{s},1.5" for s in nums) + "\n").encode()
    got, skipped = oracle.csv_points(text)
    want = []
    for s in nums:
        v = float(s)
        nonzero = any(c in "123456789" for c in s.lower().split("e")[0])
        if np.isfinite(v) and not (v == 0.0 and nonzero) and abs(v) <= 90.0:
            want.append(v)
    want = np.array(want)
    assert skipped == len(nums) - len(want) and len(want) > 10000
    assert _same_bits(got[:, 0], want) and np.all(got[:, 1] == 1.5)


@pytest.mark.gpu
def test_gpu_number_parsing_matches_python_float():
    bundle, s = _session()
    nums = _random_decimals(0xC5B5, 300000)
    text = ("lat,lng\n" + "\n".join(f"{x},1.5" for x in nums) + "\n").encode()
    got, skipped = s.points_from_csv(text)
    want = []
    for x in nums:
        v = float(x)
        nonzero = any(c in "123456789" for c in x.lower().split("e")[0])
        if np.isfinite(v) and not (v == 0.0 and nonzero) and abs(v) <= 90.0:
            want.append(v)
    want = np.array(want)
    assert skipped == len(nums) - len(want)
    assert _same_bits(got[:, 0], want)
    bundle.close()

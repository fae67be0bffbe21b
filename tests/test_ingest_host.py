"""The dataset file format without a GPU: the decimal parser the loader kernel runs
(numparse.cuh, host build) pinned against Python's float(), the repr(float) formatter
against Python's repr, and the native writer against the reference writer's bytes
(tests/golden/csv, made by tests/golden/make_ingest_golden.py)."""

import ctypes as C
import json
import os
import struct

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csv")


@pytest.fixture(scope="module")
def lib():
    from paper_2401_10068_b200 import _lib

    return _lib.lib()


def parse(lib, s: str):
    b = s.encode()
    out = C.c_double()
    st = lib.cv_parse_number_host(b, len(b), C.byref(out))
    return st, out.value


def py(s):
    try:
        return float(s)
    except ValueError:
        return None


def same(a, b):
    return struct.pack("<d", a) == struct.pack("<d", b) or (a != a and b != b)


EDGE = [
    "0", "-0", "0.0", "-0.0", "1", "+1", "-1", ".5", "5.", "1e5", "1E5", "1e+5", "1e-5", "1.e5", "  7 ", "\t8\x0b",
    "1_000", "1_0.5", "1__0", "_1", "1_", "1_.5", "1._5", "1e1_0", "1e_10", "inf", "-inf", "Infinity", "iNfInItY",
    "nan", "-NaN", "nan(1)", "infin", "", " ", ".", "e5", "1e", "1e+", "+-1", "0x10", "1,5", "1.2.3", "--1",
    "1e400", "-1e400", "1e-400", "2.4703282292062328e-324", "2.4703282292062327e-324", "4.9406564584124654e-324",
    "2.2250738585072011e-308", "2.2250738585072014e-308", "1.7976931348623157e308", "1.7976931348623158e308",
    "1.7976931348623159e308", "9007199254740993", "9007199254740992", "9007199254740994.5", "0.1", "0.3",
    "123456789012345678901234567890", "0.1000000000000000055511151231257827021181583404541015625",
    "3.141592653589793238462643383279", "1e22", "1e23", "8.98846567431158e307", "4.35689e-310",
    "7.2057594037927933e16", "00000000000000000000000001.5", "0." + "0" * 400 + "1", "1" + "0" * 400 + "e-400",
    "1" * 25 + "e-10", "9" * 30, "1e-99999999999", "1e99999999999", "0e99999999",
]


def test_parser_edge_cases_match_python(lib):
    for s in EDGE:
        st, v = parse(lib, s)
        want = py(s)
        if want is None:
            assert st == 1, repr(s)
        else:
            assert st in (0, 2), repr(s)
            if st == 0:
                assert same(v, want), (s, v, want)


def test_parser_round_trips_repr_of_random_doubles(lib):
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 2**63 - 1, 60_000, dtype=np.int64).view(np.float64)
    vals = [x for x in bits if np.isfinite(x)] + list(rng.standard_normal(20_000)) + list(rng.random(20_000))
    for x in vals:
        for s in (repr(float(x)), f"{x:.17e}", f"{x:.15g}", f"{x:.20e}"):
            st, v = parse(lib, s)
            assert st in (0, 2)
            if st == 0:
                assert same(v, float(s)), (s, v)


def test_parser_near_halfway_decimals(lib):
    """Decimal strings straddling the midpoint of two adjacent doubles (the hard cases)."""
    from decimal import Decimal, getcontext

    getcontext().prec = 800
    rng = np.random.default_rng(9)
    n_slow = 0
    for _ in range(3000):
        e = int(rng.integers(-320, 300))
        x = float(rng.random()) * 10.0**e
        if not np.isfinite(x) or x == 0:
            continue
        y = np.nextafter(x, np.inf)
        mid = (Decimal(float(x)) + Decimal(float(y))) / 2
        for digits in (15, 16, 17, 18, 19, 20, 25):
            for delta in (-1, 0, 1):
                s = f"{mid:.{digits}e}"
                m, ex = s.split("e")
                last = int(m[-1]) + delta
                if 0 <= last <= 9:
                    s = m[:-1] + str(last) + "e" + ex
                st, v = parse(lib, s)
                # <= 19 significant digits are always decided on the device (no fallback)
                assert st == 0 if digits <= 18 else st in (0, 2)
                n_slow += st == 2
                if st == 0:
                    assert same(v, float(s)), (s, v, float(s))
    assert n_slow > 0  # the > 19-digit halfway cases do reach the strtod path


def repr_native(lib, x):
    buf = C.create_string_buffer(64)
    n = lib.cv_format_repr(float(x), buf)
    return buf.raw[:n].decode()


def test_repr_formatter_matches_python(lib):
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2**63 - 1, 50_000, dtype=np.int64).view(np.float64)
    vals = [x for x in bits if np.isfinite(x)] + list(rng.standard_normal(20_000))
    vals += [0.0, -0.0, 1.0, -1.0, 0.1, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5, 0.00012, 1.5e-5, 123456.789,
             5e-324, 1.7976931348623157e308, 2.0**53, 2.0**60, 1e22, 1e21, float("inf"), float("-inf")]
    vals += [float(f"{d}e{k}") for d in (1, 2.5, 9.75) for k in range(-8, 20)]
    for x in vals:
        assert repr_native(lib, x) == repr(float(x)), x


def _expected():
    with open(os.path.join(GOLD, "expected.json")) as fh:
        return json.load(fh)


WRITTEN = sorted(n for n, v in _expected().items() if "V" in v)


@pytest.mark.parametrize("name", WRITTEN)
def test_writer_bytes_equal_reference_writer(lib, name, tmp_path):
    from paper_2401_10068_b200 import ingest, model

    z = np.load(os.path.join(GOLD, name[:-4] + ".npz"))
    ds = model.Dataset(r=z["r"], mu=z["mu"], D=z["D"], n_networks=int(z["n_networks"]))
    out = tmp_path / "w.csv"
    ingest.write_dataset_csv(out, ds, threads=3)
    with open(os.path.join(GOLD, name[:-4] + ".written"), "rb") as fh:
        assert out.read_bytes() == fh.read()
    if name.startswith("w_"):  # the reference wrote this file itself: reading + writing is the identity
        with open(os.path.join(GOLD, name), "rb") as fh:
            assert out.read_bytes() == fh.read()


@pytest.mark.parametrize("name", ["err_header.csv", "err_header_short.csv", "err_empty.csv", "err_blank_header.csv"])
def test_header_errors_before_any_device_work(lib, name):
    """Header validation happens on the host before the body goes to the GPU (cli.py:61-64)."""
    from paper_2401_10068_b200 import ingest

    path = os.path.join(GOLD, name)
    e = _expected()[name]
    with pytest.raises(ingest.UsageError) as info:
        ingest.load_dataset_csv(path, device=0)
    assert str(info.value) == e["message"].replace("{path}", path)


def _records(text):
    import ctypes as C

    from paper_2401_10068_b200 import _lib

    b = text.encode("latin-1")
    out, used = C.create_string_buffer(4 * len(b) + 64), C.c_int64()
    _lib.check(_lib.lib().cv_csv_records_host(b, len(b), out, len(out), C.byref(used)))
    s = out.raw[: used.value].decode("latin-1")
    return [rec[1:].split("\x1f") if rec.startswith("\x1d") else [] for rec in s.split("\x1e")[:-1]]


def test_host_csv_reader_is_pythons_csv_reader():
    """Files with a quote character are read on the host by a restatement of csv.reader
    (dialect excel, newline='', reference cli.py:58-60); fuzzed against the real module."""
    import csv
    import io
    import random

    rng = random.Random(1)
    alpha = ["a", "1", ",", '"', "\n", "\r", " ", "\r\n", '""', "2.5"]
    checked = 0
    for _ in range(20000):
        t = "".join(rng.choice(alpha) for _ in range(rng.randint(0, 16)))
        try:
            want = list(csv.reader(io.StringIO(t, newline="")))
        except csv.Error:
            continue
        assert _records(t) == want, repr(t)
        checked += 1
    assert checked > 15000

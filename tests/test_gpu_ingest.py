"""The GPU dataset reader (ingest.load_dataset_csv / read_dataset_csv) against the reference
reader's own outputs and errors (tests/golden/csv, made by running the reference), plus
round trips and a large file at scale."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csv")
with open(os.path.join(GOLD, "expected.json")) as _fh:
    EXPECTED = json.load(_fh)


@pytest.fixture(scope="module")
def ing():
    from paper_2401_10068_b200 import ingest

    return ingest


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("name", sorted(n for n, v in EXPECTED.items() if "V" in v))
@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_reader_matches_reference_reader(ing, name, storage):
    z = np.load(os.path.join(GOLD, name[:-4] + ".npz"))
    path = os.path.join(GOLD, name)
    if storage == "f64":
        ds = ing.read_dataset_csv(path)
        assert ds.n_networks == int(z["n_networks"]) and ds.V == EXPECTED[name]["V"]
        assert np.array_equal(bits(ds.r), bits(z["r"]))
        assert np.array_equal(bits(ds.mu), bits(z["mu"]))
        assert np.array_equal(bits(ds.D), bits(z["D"]))
    dd = ing.load_dataset_csv(path, storage=storage)
    x = dd.stream_x()
    want = (z["r"] - z["mu"]).astype(np.float32 if storage == "f32" else np.float64).astype(np.float64)
    assert np.array_equal(bits(x), bits(want))
    dd.close()


@pytest.mark.parametrize("name", sorted(n for n, v in EXPECTED.items() if "error" in v))
def test_reader_raises_what_the_reference_raises(ing, name):
    path = os.path.join(GOLD, name)
    e = EXPECTED[name]
    cls = ing.UsageError if e["error"] == "UsageError" else ValueError
    with pytest.raises(cls) as info:
        ing.read_dataset_csv(path)
    assert str(info.value) == e["message"].replace("{path}", path)
    if e["error"] == "ValueError":
        assert not isinstance(info.value, ing.UsageError)


def test_missing_file_raises_like_open(ing, tmp_path):
    with pytest.raises(FileNotFoundError):
        ing.read_dataset_csv(tmp_path / "nope.csv")


def test_fit_on_loaded_file_equals_fit_on_host_dataset(ing):
    from paper_2401_10068_b200 import model, vb

    path = os.path.join(GOLD, "w_mock56.csv")
    hp = model.default_hyperparams(3)
    z = np.load(os.path.join(GOLD, "w_mock56.npz"))
    host = model.Dataset(r=z["r"], mu=z["mu"], D=z["D"], n_networks=3)
    s1, t1 = vb.vb_fit(host, hp)
    s2, t2 = vb.vb_fit(ing.load_dataset_csv(path), hp)
    assert np.array_equal(t1.elbo, t2.elbo)
    assert np.array_equal(s1.k0k, s2.k0k) and s1.b_rho == s2.b_rho


def test_large_file_round_trip(ing, tmp_path):
    """1e6 real-valued rows: write (native repr) -> GPU read gives back the exact doubles."""
    from paper_2401_10068_b200 import model

    rng = np.random.default_rng(11)
    V, N = 1_000_000, 4
    raw = rng.random((V, N)) * np.array([1.0, 10.0, 1e-3, 1.0])
    r = rng.standard_normal(V) * 10.0 ** rng.integers(-6, 6, V)
    mu = raw[:, -1].copy()
    D = raw[:, :-1] - mu[:, None]
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=N)
    p = tmp_path / "big.csv"
    ing.write_dataset_csv(p, ds)
    back = ing.read_dataset_csv(p)
    assert np.array_equal(bits(back.r), bits(r))
    assert np.array_equal(bits(back.mu), bits(mu))
    # the file holds d_j = D_j + mu; the reader recomputes D_j = d_j - mu like model.transform
    assert np.array_equal(bits(back.D), bits((D + mu[:, None]) - mu[:, None]))


def test_awkward_text_is_parsed_like_python(ing, tmp_path):
    rng = np.random.default_rng(2)
    vals = rng.standard_normal((2000, 3)) * 10.0 ** rng.integers(-30, 30, (2000, 3))
    fmts = ["{!r}", "{:.20e}", "{:.3f}", " {!r} ", "{:.25g}", "\"{!r}\""]
    lines = ["r,d_1,d_2"]
    want = []
    for i, row in enumerate(vals):
        f = fmts[i % len(fmts)]
        cells = [f.format(float(v)) for v in row]
        lines.append(",".join(cells))
        want.append([float(c.strip().strip('"')) for c in cells])
        if i % 97 == 0:
            lines.append("")
    text = "\r\n".join(lines)
    p = tmp_path / "awk.csv"
    p.write_bytes(text.encode())
    ds = ing.read_dataset_csv(p)
    want = np.array(want)
    assert np.array_equal(bits(ds.r), bits(want[:, 0]))
    assert np.array_equal(bits(ds.mu), bits(want[:, 2]))
    assert np.array_equal(bits(ds.D[:, 0]), bits(want[:, 1] - want[:, 2]))


def test_read_dataset_keeps_its_hbm_stream(ing):
    """The CLI's read -> vb_fit path (cli.py:235-268 after install()) uploads nothing again:
    the Dataset read_dataset_csv returns carries the stream the GPU reader parsed."""
    from paper_2401_10068_b200 import vb

    path = os.path.join(GOLD, "w_n8_2000.csv")
    ds = ing.read_dataset_csv(path)
    dd = vb.device_dataset(ds)
    assert vb.device_dataset(ds) is dd and dd.V == ds.V
    x = dd.stream_x()
    assert np.array_equal(bits(x), bits(ds.r - ds.mu))


@pytest.mark.parametrize("storage", ["f64", "f32", "f32m"])
def test_npz_round_trip_into_hbm(ing, tmp_path, storage):
    """Binary dataset files: write_dataset_npz -> load_dataset_npz reproduces the stream the
    upload path builds, bit for bit, and a fit on it equals the fit on the uploaded dataset."""
    from paper_2401_10068_b200 import model, vb

    src = model.regime(300_001, 17, 4)
    r, mu, D = src.download()
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=4)
    p = tmp_path / "ds.npz"
    ing.write_dataset_npz(p, ds)
    dd = ing.load_dataset_npz(p, storage=storage)
    assert dd.V == 300_001 and dd.dim == 3 and dd.n_networks == 4 and dd.storage == storage
    up = model.upload(ds, storage=storage)
    assert np.array_equal(bits(dd.stream_x()), bits(up.stream_x()))
    r2, mu2, D2 = dd.download()
    assert np.array_equal(bits(r2), bits(r)) and np.array_equal(bits(mu2), bits(mu)) and np.array_equal(bits(D2), bits(D))
    hp = model.default_hyperparams(4)
    s1, t1 = vb.vb_fit(dd, hp, max_iter=12)
    s2, t2 = vb.vb_fit(up, hp, max_iter=12)
    assert np.array_equal(t1.elbo, t2.elbo) and np.array_equal(s1.k0k, s2.k0k)


def test_read_dataset_npz_keeps_its_hbm_stream(ing, tmp_path):
    from paper_2401_10068_b200 import model, vb

    r, mu, D = model.regime(5000, 3, 3).download()
    p = tmp_path / "ds.npz"
    ing.write_dataset_npz(p, model.Dataset(r=r, mu=mu, D=D, n_networks=3))
    ds = ing.read_dataset_npz(p)
    assert np.array_equal(bits(ds.r), bits(r)) and np.array_equal(bits(ds.D), bits(D)) and ds.n_networks == 3
    assert vb.device_dataset(ds).V == 5000

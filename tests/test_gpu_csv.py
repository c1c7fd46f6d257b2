"""Device CSV ingestion (csrc/csv.cu) against the oracle's load_csv (glibc std::strtod):
bit-exact features, identical names / labels, identical error kind and message
(proj/src/csv.cpp:63-115). Every comparison is on identical bytes."""
import random
import zlib

import numpy as np
import pytest

from csv_cases import BAD_CELLS, make_csv, mutate, number_text

pytestmark = pytest.mark.gpu


def both(R, orc, text, label=None, source="t.csv"):
    """(ok, result-or-message) of the device parser and of the oracle."""
    try:
        ds = R.parse_csv(text, label, source)
        dev = (True, dict(n=ds.n, d=ds.d, features=ds.features, names=ds.names, labels=ds.labels, ds=ds))
    except R.RenyiError as e:
        dev = (False, (e.status, str(e)))
    try:
        ref = (True, orc.load_csv(text, label, source))
    except orc.OracleError as e:
        ref = (False, (e.code, str(e)))
    return dev, ref


def assert_same(dev, ref, text):
    assert dev[0] == ref[0], (text[:400], dev[1] if not dev[0] else "ok", ref[1] if not ref[0] else "ok")
    if not dev[0]:
        assert dev[1] == ref[1] and dev[1][0] == 10, (dev[1], ref[1])
        return
    g, w = dev[1], ref[1]
    assert (g["n"], g["d"]) == (w["n"], w["d"])
    assert g["names"] == w["names"] and g["labels"] == w["labels"]
    # bit-exact, NaN payloads and signed zeros included
    assert np.array_equal(g["features"].view(np.uint64), w["features"].view(np.uint64)), text[:400]


def test_reference_cases(R, orc):
    for text, label in [("x,y\n1.5,2.0\n1.5,2.0\n1.5,2.0\n", None), ("x\n0\n1000\n2000\n3000\n4000\n", None),
                        ("a,b\n", None), ("a,b\n1,2\n3,oops\n", None), ("", None), ("a,b\n1,2\n3\n", None),
                        ("a,b\n1,2\n3,4\n", "class"), ("a,b,class\n1,2,x\n3,4,y\n", "class"),
                        ('a,"b,c",class\r\n1,"2",x\r\n\r\n3,4e1,"y ""q"""\n""\n5," 6 ",z', "class")]:
        dev, ref = both(R, orc, text, label)
        assert_same(dev, ref, text)
    # the messages themselves (test_cli.cpp:219-228)
    with pytest.raises(R.RenyiError) as e:
        R.parse_csv("a,b\n1,2\n3,oops\n")
    assert e.value.status == 10 and "row 3, column 2: 'oops' is not numeric" in str(e.value)


def test_cells_bit_exact(R, orc):
    """Thousands of generated cells (round-trip, %g/%e, hex, exact midpoints, 900-digit strings,
    subnormals, overflow, inf/nan payloads, whitespace, quotes) in one file."""
    rng = random.Random(11)
    cells = [number_text(rng) for _ in range(6000)]
    text = "v\n" + "\n".join('"' + c.replace('"', '""') + '"' if (',' in c or '\n' in c) else c for c in cells) + "\n"
    dev, ref = both(R, orc, text)
    assert_same(dev, ref, text)
    assert dev[1]["n"] == 6000


@pytest.mark.parametrize("seed", range(6))
def test_generated_files(R, orc, seed):
    rng = random.Random(100 + seed)
    d = rng.randint(1, 8)
    label_at = rng.choice([None, 0, d // 2, d])
    text = make_csv(rng, rng.randint(2, 300), d, label_at=label_at, crlf=seed % 2 == 1, blank_lines=seed % 3 == 0)
    dev, ref = both(R, orc, text, "class" if label_at is not None else None)
    assert_same(dev, ref, text)


@pytest.mark.parametrize("bad", BAD_CELLS)
def test_bad_cells(R, orc, bad):
    rng = random.Random(zlib.crc32(bad.encode()))
    text = make_csv(rng, 30, 3, label_at=1, bad=bad, bad_at=(17, rng.choice([0, 2, 3])))
    dev, ref = both(R, orc, text, "class")
    assert_same(dev, ref, text)


def test_mutations(R, orc):
    """Byte-level mutations (quotes, separators, CR, NUL): both sides agree on success, values and message."""
    rng = random.Random(7)
    base = make_csv(rng, 25, 3, label_at=3)
    for t in range(120):
        text = mutate(rng, base, edits=rng.randint(1, 4))
        dev, ref = both(R, orc, text, "class" if t % 2 else None)
        assert_same(dev, ref, text)


def test_chunk_boundaries_and_long_quotes(R, orc):
    """Quoted fields spanning the 8 KB scan chunks, a record per chunk boundary, no trailing newline."""
    rng = random.Random(3)
    long_label = '"' + ("x" * 9000 + ",\n" + '"' * 3000).replace('"', '""') + '"'
    rows = [number_text(rng).replace(",", "") + "," + (long_label if i % 7 == 0 else "l") for i in range(400)]
    text = "v,class\n" + "\n".join(rows)
    dev, ref = both(R, orc, text, "class")
    assert_same(dev, ref, text)
    # odd quote count: the rest of the file is one quoted field
    dev, ref = both(R, orc, 'a,b\n1,"2\n3,4\n5,6\n', None)
    assert_same(dev, ref, "")


def test_load_file_and_kernel_from_dataset(R, orc, tmp_path):
    """load_csv(path) and build_kernel on the resident features == build_kernel on the host copy."""
    rng = random.Random(21)
    text = make_csv(rng, 700, 5, label_at=2)
    p = tmp_path / "data.csv"
    p.write_bytes(text.encode())
    ds = R.load_csv(str(p), "class")
    ref = orc.load_csv(text, "class", str(p))
    assert np.array_equal(ds.features.view(np.uint64), ref["features"].view(np.uint64))
    assert ds.labels == ref["labels"]
    # kernel straight from the resident features (finite data in the reference's ostream format)
    g = np.random.default_rng(4).standard_normal((500, 4))
    p2 = tmp_path / "finite.csv"
    p2.write_text("a,b,c,d\n" + "\n".join(",".join("%g" % v for v in row) for row in g) + "\n")
    ds2 = R.load_csv(str(p2))
    x = orc.load_csv(p2.read_text())["features"]
    spec = R.GaussianKernel(2.0)
    for cols in (None, [2, 0]):
        a_dev = ds2.kernel(spec, "fp64", columns=cols).matrix()
        a_host = R.build_kernel(np.ascontiguousarray(x if cols is None else x[:, cols]), spec, "fp64").matrix()
        assert np.array_equal(a_dev, a_host)
    with pytest.raises(R.RenyiError) as e:
        R.load_csv(str(tmp_path / "missing.csv"))
    assert e.value.status == 10 and "cannot open" in str(e.value)


def test_large_file_matches_oracle(R, orc):
    """~30 MB, 100k x 16 in the reference's ostream format (make_labeled_csv, test_cli.cpp:60-77)."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((100_000, 16))
    lines = ["," .join(f"f{j}" for j in range(16)) + ",class"]
    lab = rng.integers(0, 2, 100_000)
    body = "\n".join(",".join("%.17g" % v for v in row) + ("," + ("pos" if y else "neg")) for row, y in zip(x, lab))
    text = lines[0] + "\n" + body + "\n"
    dev, ref = both(R, orc, text, "class")
    assert_same(dev, ref, "<large>")
    assert np.array_equal(dev[1]["features"], x)  # %.17g round-trips


def test_decimal_paths_bit_exact_at_scale(R, orc):
    """Clinger / Eisel-Lemire / bracketed Eisel-Lemire / big-decimal paths against glibc strtod on
    ~300k decimal cells: random binary64 values printed with 15-25 significant digits, random
    16-40 digit strings over the whole exponent range (subnormals, overflow), and near-ties."""
    rng = np.random.default_rng(17)
    bits = rng.integers(0, 2 ** 63, 120_000, dtype=np.uint64) | (rng.integers(0, 2, 120_000, dtype=np.uint64) << 63)
    vals = bits.view(np.float64)
    vals = vals[np.isfinite(vals)]
    fmts = ["%.15g", "%.16g", "%.17g", "%.18g", "%.19g", "%.20g", "%.25e"]
    cells = [fmts[i % len(fmts)] % v for i, v in enumerate(vals)]
    digits = rng.integers(0, 10, (120_000, 40))
    lens = rng.integers(16, 41, 120_000)
    exps = rng.integers(-345, 320, 120_000)
    for i in range(120_000):
        ds = "".join(map(str, digits[i, : lens[i]])).lstrip("0") or "0"
        cells.append(f"{ds[0]}.{ds[1:]}e{exps[i] - len(ds) + 1}")
    g = random.Random(23)
    from csv_cases import _midpoint_text
    cells += [_midpoint_text(g) for _ in range(20_000)]
    text = "v\n" + "\n".join(cells) + "\n"
    dev, ref = both(R, orc, text)
    assert_same(dev, ref, "<decimal paths>")
    assert dev[1]["n"] == len(cells)


def test_golden_csv_fixtures_on_device(R):
    """tests/golden: the reference tests' CSV inputs through load_csv(path) on the device."""
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parent / "golden"
    for name, want in json.loads((root / "expected.json").read_text()).items():
        path = str(root / name)
        if "error" in want:
            with pytest.raises(R.RenyiError) as e:
                R.load_csv(path)
            assert e.value.status == 10 and want["error"] in str(e.value), name
        else:
            ds = R.load_csv(path)
            assert (ds.n, ds.d, ds.names) == (want["n"], want["d"], want["names"])
            assert np.array_equal(ds.features, np.array(want["features"], dtype=float))

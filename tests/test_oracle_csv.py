"""CSV oracle (oracle/renyi_oracle.cpp load_csv, restating proj/src/csv.cpp:13-115 with glibc
std::strtod) pinned by the reference's own CSV test cases (proj/tests/test_cli.cpp:60-77,
82-95, 219-228, 268-281)."""
import math
import random

import numpy as np
import pytest

from csv_cases import make_csv, number_text


def test_reference_fixtures(orc):
    # identical.csv / far.csv (test_cli.cpp:82-95)
    d = orc.load_csv("x,y\n1.5,2.0\n1.5,2.0\n1.5,2.0\n")
    assert (d["n"], d["d"], d["names"]) == (3, 2, ["x", "y"])
    assert np.array_equal(d["features"], np.array([[1.5, 2.0]] * 3))
    d = orc.load_csv("x\n0\n1000\n2000\n3000\n4000\n")
    assert np.array_equal(d["features"][:, 0], [0, 1000, 2000, 3000, 4000])


def test_reference_failures(orc):
    # header-only and malformed CSVs (test_cli.cpp:219-228): parse_error, coordinates of the bad cell
    with pytest.raises(orc.OracleError) as e:
        orc.load_csv("a,b\n", source="h.csv")
    assert e.value.code == 10 and str(e.value) == "'h.csv': need at least 2 data rows, got 0"
    with pytest.raises(orc.OracleError) as e:
        orc.load_csv("a,b\n1,2\n3,oops\n")
    assert str(e.value) == "row 3, column 2: 'oops' is not numeric"
    with pytest.raises(orc.OracleError) as e:
        orc.load_csv("", source="empty.csv")
    assert str(e.value) == "'empty.csv': missing header row"
    with pytest.raises(orc.OracleError) as e:
        orc.load_csv("a,b\n1,2\n3\n")
    assert str(e.value) == "row 3: expected 2 fields, got 1"
    with pytest.raises(orc.OracleError) as e:
        orc.load_csv("a,b\n1,2\n3,4\n", "class", source="x.csv")
    assert str(e.value) == "'x.csv': no column named 'class'"


def test_krvskp_shape(orc):
    # "a dataset with the Krvskp shape parses" (test_cli.cpp:268-281), same layout from a seeded stream
    rng = random.Random(71)
    lines = [",".join(f"f{j}" for j in range(36)) + ",label"]
    for _ in range(3196):
        lines.append(",".join(str(rng.getrandbits(64) % 4) for _ in range(36)) + "," +
                     ("won" if rng.getrandbits(64) % 2 else "nowin"))
    d = orc.load_csv("\n".join(lines) + "\n", "label")
    assert (d["n"], d["d"], len(d["labels"])) == (3196, 36, 3196)
    assert set(d["labels"]) == {"won", "nowin"}


def test_quotes_crlf_blank_lines_and_labels(orc):
    text = 'a,"b,c",class\r\n1,"2",x\r\n\r\n"",\n3,4e1,"y ""q"""\n""\n5," 6 ",z'
    with pytest.raises(orc.OracleError) as e:  # '"",' is a 2-field record, not a blank line
        orc.load_csv(text, "class")
    assert str(e.value) == "row 4: expected 3 fields, got 2"
    d = orc.load_csv(text.replace('"",\n', ''), "class")
    assert d["names"] == ["a", "b,c"] and d["labels"] == ["x", 'y "q"', "z"]
    assert np.array_equal(d["features"], [[1, 2], [3, 40], [5, 6]])


def test_strtod_grammar(orc):
    # glibc strtod in the C locale: hex floats, inf/nan spellings, leading isspace, trailing spaces only
    cells = {"0x1.8p1": 3.0, " \t1.5  ": 1.5, "+.5e1": 5.0, "-0": -0.0, "1.": 1.0, "INFINITY": math.inf,
             "2.4703282292062328e-324": 5e-324, "1.7976931348623159e308": math.inf}
    for cell, want in cells.items():
        d = orc.load_csv(f"x\n{cell}\n0\n")
        got = d["features"][0, 0]
        assert got == want and math.copysign(1, got) == math.copysign(1, want), cell
    for bad in ["1e", "0x", "inf1", "1\t", "nan(", ""]:
        with pytest.raises(orc.OracleError):
            orc.load_csv(f"x\n{bad}\n0\n")


def test_generated_files_parse(orc):
    rng = random.Random(5)
    for trial in range(20):
        text = make_csv(rng, rng.randint(2, 40), rng.randint(1, 6), label_at=rng.choice([None, 0, 1]),
                        crlf=rng.random() < 0.3, blank_lines=rng.random() < 0.5)
        try:
            d = orc.load_csv(text, "class" if "class" in text.split("\n")[0] else None)
        except orc.OracleError as e:
            assert e.code == 10
            continue
        assert d["features"].shape == (d["n"], d["d"])
    assert number_text(random.Random(1))  # generator smoke


def test_pow10_table_matches_generator():
    """csrc/pow10_table.h (Eisel-Lemire table of the device CSV reader) is exactly what
    gen_pow10.py computes: floor of the top 128 bits of 10^e, leading bit set."""
    import re
    from pathlib import Path

    from paper_2205_07426_b200.gen_pow10 import HI, LO, mantissa128

    text = (Path(__file__).resolve().parents[1] / "paper_2205_07426_b200" / "csrc" / "pow10_table.h").read_text()
    rows = re.findall(r"\{0x([0-9a-f]{16})ull, 0x([0-9a-f]{16})ull\},\s*// 1e(-?\d+)", text)
    assert len(rows) == HI - LO + 1
    for lo, hi, e in rows:
        m = (int(hi, 16) << 64) | int(lo, 16)
        e = int(e)
        assert m == mantissa128(e)
        # m = floor(10^e * 2^k) with k = 127 - floor(log2 10^e), checked in integers
        if e >= 0:
            v = 10 ** e
            k = 127 - (v.bit_length() - 1)
            assert (m << max(-k, 0)) <= (v << max(k, 0)) < ((m + 1) << max(-k, 0))
        else:
            d = 10 ** (-e)  # never a power of two: floor(log2(1/d)) = -bit_length(d)
            k = 127 + d.bit_length()
            assert m * d <= (1 << k) < (m + 1) * d


def test_golden_csv_fixtures(orc):
    """tests/golden: the reference tests' CSV inputs and their asserted outcomes."""
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parent / "golden"
    for name, want in json.loads((root / "expected.json").read_text()).items():
        text = (root / name).read_bytes()
        if "error" in want:
            with pytest.raises(orc.OracleError) as e:
                orc.load_csv(text, source=name)
            assert e.value.code == 10 and want["error"] in str(e.value), name
        else:
            d = orc.load_csv(text, source=name)
            assert (d["n"], d["d"], d["names"]) == (want["n"], want["d"], want["names"])
            assert np.array_equal(d["features"], np.array(want["features"], dtype=float))
